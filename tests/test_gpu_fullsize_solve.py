"""Full-size, O(1)-conditioned shifted block solves against numpy (stage 5, §2:
"Each block S_l is inverted independently, using a uniform diagonal shift lambda").

At the BASELINE.json initialisation ||S_b|| << lambda, so the step's own solves are close to
-F/lambda and a residual test on them says little about the S-dependent part.  Here S = A^H A
with A Gaussian, ||S|| ~ 1 >> lambda = 1e-3: the solution depends on every entry of S.
Sizes: one 6480 block (configs[1]'s largest), one 12928 block (configs[3]'s first), and the
three blocks of configs[1] in one batched call, each with the Cholesky trailing updates on
both Gram engines.  S is formed on the GPU with torch (cuBLAS ZGEMM, test instrument only);
the reference is LAPACK's Cholesky (scipy.linalg.cho_factor / cho_solve) of the same S + lambda I
on the host.  Bar: relative L2 1e-9 on dtheta (north_star).
"""
import numpy as np
import pytest
import scipy.linalg
import torch

pytestmark = pytest.mark.gpu

C128 = torch.complex128
LAM = 1e-3


@pytest.fixture(scope="module")
def sr():
    import paper_2510_08430_b200 as pkg
    pkg.load()
    return pkg


def dev():
    return torch.device("cuda:0")


def _qgt(n, m, seed):
    """S = A^H A / m for a complex Gaussian m x n A (rank min(m, n)), exactly Hermitian."""
    g = torch.Generator(device=dev()).manual_seed(seed)
    A = torch.complex(torch.randn(m, n, dtype=torch.float64, device=dev(), generator=g),
                      torch.randn(m, n, dtype=torch.float64, device=dev(), generator=g)) / np.sqrt(2 * m)
    S = A.conj().T @ A
    S = 0.5 * (S + S.conj().T)
    F = torch.complex(torch.randn(n, dtype=torch.float64, device=dev(), generator=g),
                      torch.randn(n, dtype=torch.float64, device=dev(), generator=g))
    return S.contiguous(), F


def _ref(S, F):
    Sh = S.cpu().numpy()
    Sh[np.diag_indices_from(Sh)] += LAM
    c = scipy.linalg.cho_factor(Sh, lower=True, overwrite_a=True, check_finite=False)
    return -scipy.linalg.cho_solve(c, F.cpu().numpy(), check_finite=False)


def _solve(sr, engine, offs, S_packed, F):
    prev = sr.sr_set_gram_engine(sr.GRAM_INT8 if engine == "int8" else sr.GRAM_FP64)
    try:
        d = torch.empty_like(F)
        info = torch.full((1,), -5, dtype=torch.int32, device=dev())
        sr.sr_block_solve(offs, S_packed, F, LAM, d, info=info)
        torch.cuda.synchronize()
    finally:
        sr.sr_set_gram_engine(prev)
    assert info.item() == 0
    return d.cpu().numpy()


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,m", [(6480, 2 * 6480), (12928, 12928 // 2)], ids=["n6480_full_rank", "n12928_rank_half"])
def test_single_block_full_size(sr, n, m):
    S, F = _qgt(n, m, n)
    ref = _ref(S, F)
    # the S-dependent part is not negligible: -F/lambda is far from the solution
    assert _rel(-F.cpu().numpy() / LAM, ref) > 0.1
    for engine in ("int8", "fp64"):
        got = _solve(sr, engine, [0, n], S.reshape(-1), F)
        assert _rel(got, ref) < 1e-9, engine


def test_configs1_blocks_batched_full_size(sr):
    sizes = [3280, 6480, 6480]
    offs = [0] + [int(x) for x in np.cumsum(sizes)]
    mats, Fs = zip(*[_qgt(n, m, 100 + i) for i, (n, m) in enumerate(zip(sizes, (4096, 4096, 8000)))])
    S_packed = torch.cat([s.reshape(-1) for s in mats])
    F = torch.cat(Fs)
    refs = np.concatenate([_ref(s, f) for s, f in zip(mats, Fs)])
    for engine in ("int8", "fp64"):
        got = _solve(sr, engine, offs, S_packed, F)
        for b in range(3):
            lo, hi = offs[b], offs[b + 1]
            assert _rel(got[lo:hi], refs[lo:hi]) < 1e-9, (engine, b)
