"""GPU parity of the int8 tcgen05 Gram engine (sr_block_qgt_i8, DESIGN.md §5 "Ozaki").

Same contract and tolerance as sr_block_qgt: relative L2 1e-11 per block S_b against the
CPU oracle (BASELINE.json north_star), exactly Hermitian as stored, real diagonal.  The
cases span several 128 x 64 tiles with ragged edges, one-column blocks, a single sample,
and n_samples above 8192 (more than one exact int32 accumulation chunk of K' = 16384).
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import estimators, hamiltonian, network, solvers

pytestmark = pytest.mark.gpu

C128 = torch.complex128


@pytest.fixture(scope="module")
def sr():
    import paper_2510_08430_b200 as pkg
    pkg.load()
    return pkg


def dev():
    return torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev())


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def packed_blocks(S, offs):
    out, pos = [], 0
    for b in range(len(offs) - 1):
        n = offs[b + 1] - offs[b]
        out.append(S[pos:pos + n * n].reshape(n, n))
        pos += n * n
    return out


CASES = [
    (512, (220, 420)),
    (37, (64, 18, 130)),
    (17, (1, 65, 128)),
    (1, (40, 3)),
    (300, (129, 64, 63, 257)),
    (9000, (70, 131)),        # two int32 accumulation chunks
    (20000, (33,)),           # three chunks, ragged K
]


@pytest.mark.parametrize("ns,sizes", CASES, ids=[f"ns{c[0]}_{'-'.join(map(str, c[1]))}" for c in CASES])
def test_block_qgt_i8_parity(sr, ns, sizes):
    rng = np.random.default_rng(ns + 7 * len(sizes))
    n_p = sum(sizes)
    offs = [0] + [int(x) for x in np.cumsum(sizes)]
    O = rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))
    # columns of very different scale (the per-column exponents must carry them)
    O *= np.exp(rng.uniform(-6, 6, n_p))[None, :]
    A, _ = estimators.scaled_centered(O, np.zeros(ns))
    S = torch.full((sum(n * n for n in sizes),), complex(np.nan, np.nan), dtype=C128, device=dev())
    sr.sr_block_qgt_i8(T(A), offs, S)
    got = packed_blocks(S.cpu().numpy(), offs)
    ref = estimators.qgt_blocks(O, offs)
    for g, r in zip(got, ref):
        assert np.all(np.isfinite(g))
        if np.linalg.norm(r) == 0:
            assert np.all(g == 0)
            continue
        assert rel(g, r) < 1e-11
        assert np.array_equal(g, g.conj().T)           # Hermitian as stored
        assert np.all(np.diag(g).imag == 0)


def test_block_qgt_i8_zero_column_and_outlier(sr):
    """A zero column gives a zero row/column; one huge sample in a column is carried by that
    column's exponent (error relative to the column maximum, R10)."""
    rng = np.random.default_rng(3)
    ns, n = 200, 96
    A = rng.standard_normal((ns, n)) + 1j * rng.standard_normal((ns, n))
    A[:, 5] = 0
    A[17, 9] *= 1e6
    S = torch.empty(n * n, dtype=C128, device=dev())
    sr.sr_block_qgt_i8(T(A), [0, n], S)
    g = S.cpu().numpy().reshape(n, n)
    ref = A.conj().T @ A
    assert np.all(g[5] == 0) and np.all(g[:, 5] == 0)
    assert rel(g, ref) < 1e-11


def test_block_qgt_i8_matches_fp64_engine(sr):
    """configs[1] at full size (N_s = 4096, blocks 3280/6480/6480): the int8 engine against
    the FP64 DMMA engine on the same A, block by block."""
    w = workloads.CONFIGS[1]
    rng = np.random.default_rng(11)
    n_p = w.n_params
    offs = [int(x) for x in sr.block_offsets(w.widths)]
    A = (torch.randn(w.n_samples, n_p, dtype=torch.float64, device=dev(),
                     generator=torch.Generator(dev()).manual_seed(5))
         + 1j * torch.randn(w.n_samples, n_p, dtype=torch.float64, device=dev(),
                            generator=torch.Generator(dev()).manual_seed(6)))
    A = A.contiguous()
    n_s = sum((offs[b + 1] - offs[b]) ** 2 for b in range(len(offs) - 1))
    S8 = torch.empty(n_s, dtype=C128, device=dev())
    S64 = torch.empty(n_s, dtype=C128, device=dev())
    sr.sr_block_qgt_i8(A, offs, S8)
    sr.sr_block_qgt(A, offs, S64)
    pos = 0
    for b in range(len(offs) - 1):
        n = offs[b + 1] - offs[b]
        d = torch.linalg.vector_norm(S8[pos:pos + n * n] - S64[pos:pos + n * n])
        r = torch.linalg.vector_norm(S64[pos:pos + n * n])
        assert (d / r).item() < 1e-13
        pos += n * n
    # sampled entries against plain FP64 dot products of the same columns
    cols = rng.choice(offs[1], 8, replace=False)
    Ac = A[:, torch.as_tensor(cols, device=dev())].cpu().numpy()
    ref = Ac.conj().T @ Ac
    blk0 = S8[:offs[1] ** 2].reshape(offs[1], offs[1])
    got = blk0[torch.as_tensor(cols, device=dev())][:, torch.as_tensor(cols, device=dev())].cpu().numpy()
    assert rel(got, ref) < 1e-12


def test_step_with_int8_engine(sr):
    """sr_step with the int8 Gram engine: dtheta within 1e-9 and S_b within 1e-11 of the oracle."""
    w = workloads.CONFIGS[0]
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    nb = len(jj)
    ws = torch.empty(sr.sr_step_workspace_bytes(w.widths, w.n_samples, nb), dtype=torch.uint8, device=dev())
    d = torch.empty(w.n_params, dtype=C128, device=dev())
    en = torch.empty(1, dtype=C128, device=dev())
    prev = sr.sr_set_gram_engine(sr.GRAM_INT8)
    try:
        sr.sr_step(w.widths, T(sr.model.pack(params)), T(spins), T(ij), T(jj), w.lam, d, en, ws)
    finally:
        sr.sr_set_gram_engine(prev)
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    off = network.layer_offsets(params)
    blocks = estimators.qgt_blocks(O, off)
    ref = solvers.block_solve(blocks, estimators.force(O, e), off, w.lam)
    assert rel(d.cpu().numpy(), ref) < 1e-9
    so = sr.sr_step_s_offset(w.widths, w.n_samples, nb)
    n_s = sum(b.size for b in blocks)
    S = ws[so:so + 16 * n_s].view(C128).cpu().numpy()
    for g, r in zip(packed_blocks(S, sr.block_offsets(w.widths)), blocks):
        assert rel(g, r) < 1e-11


@pytest.fixture
def int8_engine(sr):
    prev = sr.sr_set_gram_engine(sr.GRAM_INT8)
    yield
    sr.sr_set_gram_engine(prev)


@pytest.mark.parametrize("lam", [1e-3, 1.0])
@pytest.mark.parametrize("ns,sizes", [(512, (220, 420)), (100, (64, 18, 130)), (300, (250,)), (700, (1000,)),
                                      (2000, (1300, 257))])
def test_block_solve_int8_trailing_updates(sr, int8_engine, ns, sizes, lam):
    """sr_block_solve with the Cholesky trailing updates (K = 256 strips) on the int8 engine:
    dtheta within 1e-9 of the oracle (the same bar as the FP64 path)."""
    rng = np.random.default_rng(ns + 1)
    n_p = sum(sizes)
    offs = [0] + [int(x) for x in np.cumsum(sizes)]
    O = rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))
    e = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    blocks = estimators.qgt_blocks(O, offs)
    F = estimators.force(O, e)
    Sp = np.concatenate([b.ravel() for b in blocks])
    d = torch.empty(n_p, dtype=C128, device=dev())
    info = torch.full((1,), -5, dtype=torch.int32, device=dev())
    sr.sr_block_solve(offs, T(Sp), T(F), lam, d, info=info)
    ref = solvers.block_solve(blocks, F, offs, lam)
    assert info.item() == 0
    assert rel(d.cpu().numpy(), ref) < 1e-9


def test_full_and_ntk_int8(sr, int8_engine):
    """Comparison paths with the int8 trailing updates: full-QGT and NTK solves agree with the
    oracle and with each other (push-through identity)."""
    w = workloads.CONFIGS[0]
    spins, params = workloads.make_inputs(w)
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    A, et = estimators.scaled_centered(O, e)
    F = estimators.force(O, e)
    d_full = torch.empty(w.n_params, dtype=C128, device=dev())
    d_ntk = torch.empty(w.n_params, dtype=C128, device=dev())
    sr.sr_full_qgt_solve(T(A), T(F), w.lam, d_full)
    sr.sr_ntk_solve(T(A), T(et), w.lam, d_ntk)
    ref = solvers.full_solve(estimators.qgt_full(O), F, w.lam)
    assert rel(d_full.cpu().numpy(), ref) < 1e-9
    assert rel(d_ntk.cpu().numpy(), ref) < 1e-9


def test_block_qgt_i8_non_finite_columns(sr):
    """Inf / NaN in a column of A poison that row and column of S_b (as an FP64 Gram does)
    and leave the other entries exact."""
    rng = np.random.default_rng(4)
    ns, n = 64, 70
    A = rng.standard_normal((ns, n)) + 1j * rng.standard_normal((ns, n))
    A[5, 3] = np.nan
    A[9, 40] = complex(np.inf, 0.0)
    S = torch.empty(n * n, dtype=C128, device=dev())
    sr.sr_block_qgt_i8(T(A), [0, n], S)
    g = S.cpu().numpy().reshape(n, n)
    bad = [3, 40]
    good = [i for i in range(n) if i not in bad]
    for b in bad:
        assert np.all(np.isnan(g[b])) and np.all(np.isnan(g[:, b]))
    ref = A[:, good].conj().T @ A[:, good]
    assert rel(g[np.ix_(good, good)], ref) < 1e-11


def test_block_qgt_i8_cta_pairs():
    """The CTA-pair variant of the Gram kernel (gram_i8_2sm, tcgen05 cta_group::2; selected by
    SR_GRAM_2SM=1 at process start, measured slower and off by default) passes the same parity
    cases: run them in a child process with the switch set."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SR_GRAM_2SM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_ozaki.py"),
                        "-k", "test_block_qgt_i8_parity or matches_fp64 or non_finite"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def _wide_range_columns(rng, ns, n):
    """Columns whose entries span six decades (|A_kj| = |g| 10^u, u ~ U(-6, 0)), plus two
    columns with a single outlier 1e6 above the rest, and one column scaled by 1e-150."""
    A = (rng.standard_normal((ns, n)) + 1j * rng.standard_normal((ns, n))) * 10.0 ** rng.uniform(-6, 0, (ns, n))
    A[rng.integers(ns), 3] *= 1e6
    A[rng.integers(ns), 7] *= 1e6
    A[:, 11] *= 1e-150
    return A


@pytest.mark.parametrize("engine", ["int8", "fp64"])
@pytest.mark.parametrize("ns,sizes", [(4096, (200, 129)), (9000, (64, 70))])
def test_block_qgt_entrywise_bound(sr, engine, ns, sizes):
    """north_star's 1e-11 bar "on S_b entries", entry by entry: |S_ij - S_ij^ref| <=
    1e-11 sqrt(S_ii S_jj) for every i, j (the Cauchy-Schwarz scale of the entry), on data
    with 1e6 dynamic range inside each column, for both Gram engines.  The int8 engine's
    error is relative to the column maxima (R10); this checks that it stays inside
    the entrywise bar for such columns too.  Reference: numpy's FP64 product (its own error
    is below 1e-13 of the same scale here)."""
    rng = np.random.default_rng(ns + sum(sizes))
    n_p = sum(sizes)
    offs = [0] + [int(x) for x in np.cumsum(sizes)]
    A = _wide_range_columns(rng, ns, n_p)
    S = torch.empty(sum(n * n for n in sizes), dtype=C128, device=dev())
    (sr.sr_block_qgt_i8 if engine == "int8" else sr.sr_block_qgt)(T(A), offs, S)
    got = packed_blocks(S.cpu().numpy(), offs)
    for b, g in enumerate(got):
        a = A[:, offs[b]:offs[b + 1]]
        ref = a.conj().T @ a
        d = np.sqrt(np.abs(np.diag(ref)).real)
        scale = np.outer(d, d)
        err = np.abs(g - ref)
        assert np.all(err <= 1e-11 * scale), (b, float(np.max(err / np.where(scale > 0, scale, 1))))
        assert np.array_equal(g, g.conj().T)


@pytest.mark.parametrize("ksplit", ["4096", "1000000"])
def test_block_qgt_i8_ksplit_switch(ksplit):
    """The Gram's K' per launch (SR_OZ_KSPLIT, default 16384: long K cut into launches that add
    their FP64 partials in a fixed order) only changes FP64 summation order: the parity cases
    pass with short launches (4096) and with one launch per group (in-kernel int32 chunks)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_ozaki.py"),
                        "-k", "test_block_qgt_i8_parity or matches_fp64 or entrywise or full_and_ntk_int8"],
                       cwd=root, env=dict(os.environ, SR_OZ_KSPLIT=ksplit), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


_FP64_TMA_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2510_08430_b200 as sr
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(9)
W = torch.complex(torch.randn(333, 700, dtype=torch.float64, device=dev, generator=g),
                  torch.randn(333, 700, dtype=torch.float64, device=dev, generator=g))
A = W[:, 37:37 + 601]            # a column slice: lda = 700
offs = [0, 1, 130, 193, 601]
S = torch.empty(sum((offs[b + 1] - offs[b]) ** 2 for b in range(4)), dtype=torch.complex128, device=dev)
sr.sr_block_qgt(A, offs, S)
torch.cuda.synchronize()
np.save(sys.argv[2], S.cpu().numpy())
"""


def test_fp64_tma_staging_is_bit_identical(tmp_path):
    """The FP64 engine's TMA-staged Gram (default) and its cp.async fallback (SR_FP64_TMA=0)
    give bit-identical S on ragged blocks of a column-slice A (same fragments, same order)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "s.py"
    script.write_text(_FP64_TMA_SCRIPT)
    outs = []
    for v in ("1", "0"):
        out = tmp_path / f"S{v}.npy"
        r = subprocess.run([sys.executable, str(script), root, str(out)], env=dict(os.environ, SR_FP64_TMA=v),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
    A = outs[0]
    assert np.all(np.isfinite(A))
