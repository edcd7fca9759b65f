"""BASELINE.json configs[4] (J1-J2 10x10, MLP 100->160 + seven 160->160, 8 blocks of 16160 /
25760 parameters, N_s = 65536 sharded 8192 per GPU, one block owner per GPU) on one B200.

test_one_rank_share: the data one rank of the 8-GPU run holds and produces, with the real
kernels in the launch pattern parallel.ShardedStep uses (per-block Gram launches on column
slices of A, the n_parts = 8 centring).  The other seven ranks' contributions to the global
centring (their double-double moment rows) are produced on this GPU one shard after another
-- exactly what each of them would all-gather -- so the rank's A, e_tilde, partial force and
partial S_b are the ones the 8-GPU run computes.  Checked against the oracle:
  * stage (1): sampled columns of O on sampled rows vs the oracle's derivatives (1e-12/column);
  * stage (2): sampled local energies (1e-10);
  * stage (3): the rank's A and e_tilde on the sampled columns vs the oracle's centring of the
    GPU's O over ALL 65536 samples (R11: stages 3-4 on identical O), the energy over
    all samples (1e-13), the partial force on the sampled columns (1e-9);
  * stage (4): the sampled entries of every partial S_b vs the oracle's Gram of the same
    columns (1e-11), on both Gram engines for the largest block.

test_single_gpu_point: the N=1 point of the weak-scaling run (8192 samples, all eight blocks
on one GPU) through LocalStep(schedule="per_block") -- the schedule that makes it fit -- with
each block's S_b re-formed afterwards to check the shifted-solve residual and Hermiticity.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import estimators, hamiltonian, network

pytestmark = pytest.mark.gpu

C128 = torch.complex128
G = 8
RANK = 5


@pytest.fixture(scope="module")
def sr():
    import paper_2510_08430_b200 as pkg
    pkg.load()
    return pkg


def dev():
    return torch.device("cuda:0")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_one_rank_share(sr):
    from paper_2510_08430_b200.parallel import shard_range
    w = workloads.CONFIGS[4]
    N = w.n_samples
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    theta = torch.from_numpy(sr.model.pack(params)).to(dev())
    offs = sr.block_offsets(w.widths)
    n_p = w.n_params
    rng = np.random.default_rng(44)
    cols = np.sort(np.concatenate([rng.choice(np.arange(offs[b], offs[b + 1]), 3, replace=False)
                                   for b in range(len(offs) - 1)]))
    tcols = torch.as_tensor(cols, device=dev())
    shards = [shard_range(N, q, G) for q in range(G)]
    nl = shards[RANK][1] - shards[RANK][0]
    O = torch.empty(nl, n_p, dtype=C128, device=dev())
    lp = torch.empty(nl, dtype=C128, device=dev())
    e = torch.empty(nl, dtype=C128, device=dev())
    rows = torch.empty(G, 2 * n_p + 2, dtype=C128, device=dev())
    bij, bj = torch.from_numpy(ij).to(dev()), torch.from_numpy(jj).to(dev())
    O_cols = np.empty((N, len(cols)), dtype=np.complex128)
    e_all = np.empty(N, dtype=np.complex128)
    # every shard's moment row (what the all-gather delivers), this rank's shard last so its
    # O and E_loc stay in the buffers
    for q in [x for x in range(G) if x != RANK] + [RANK]:
        lo, hi = shards[q]
        sp = torch.from_numpy(spins[lo:hi]).to(dev())
        sr.sr_jacobian(w.widths, theta, sp, lp, O)
        sr.sr_local_energy(w.widths, theta, bij, bj, sp, lp, e)
        sr.sr_column_moments(O, e, N, rows[q])
        O_cols[lo:hi] = O[:, tcols].cpu().numpy()
        e_all[lo:hi] = e.cpu().numpy()
    lo, hi = shards[RANK]
    # stage (1) and (2) on sampled rows of this rank against the oracle
    ks = rng.choice(nl, 12, replace=False)
    ref_rows = np.stack([network.log_derivative_row(params, spins[lo + k])[cols] for k in ks])
    col_err = np.linalg.norm(O_cols[lo + ks] - ref_rows, axis=0) / np.linalg.norm(ref_rows, axis=0)
    assert np.all(col_err < 1e-12)
    ke = ks[:3]
    assert rel(e_all[lo + ke], hamiltonian.local_energies(params, spins[lo + ke], hamiltonian.bonds_for(w))) < 1e-10
    # stage (3): the n_parts = 8 centring of this rank's rows
    et = torch.empty(nl, dtype=C128, device=dev())
    Fp = torch.empty(n_p, dtype=C128, device=dev())
    en = torch.empty(1, dtype=C128, device=dev())
    sr.sr_center_force_global(O, e, N, rows, et, Fp, energy=en)
    A_ref, e_ref = estimators.scaled_centered(O_cols, e_all)     # over all 65536 samples
    assert abs(en.item() - estimators.energy(e_all)) <= 1e-13 * abs(estimators.energy(e_all))
    assert rel(O[:, tcols].cpu().numpy(), A_ref[lo:hi]) < 1e-11
    assert rel(et.cpu().numpy(), e_ref[lo:hi]) < 1e-11
    assert rel(Fp[tcols].cpu().numpy(), A_ref[lo:hi].conj().T @ e_ref[lo:hi]) < 1e-9
    # stage (4): per-block partial Grams (ShardedStep's per-block launch pattern)
    n_max = max(offs[b + 1] - offs[b] for b in range(len(offs) - 1))
    stage = torch.empty(n_max * n_max, dtype=C128, device=dev())
    ws = torch.empty(sr.load().sr_block_qgt_i8_workspace_bytes(nl, 1, sr._lib._offsets([0, n_max])),
                     dtype=torch.uint8, device=dev())
    for b in range(len(offs) - 1):
        blo, bhi = offs[b], offs[b + 1]
        n = bhi - blo
        sel = [c for c in range(len(cols)) if blo <= cols[c] < bhi]
        loc = torch.as_tensor(cols[sel] - blo, device=dev())
        ref = A_ref[lo:hi, sel].conj().T @ A_ref[lo:hi, sel]
        engines = ("int8", "fp64") if n == n_max and b == len(offs) - 2 else ("int8",)
        for eng in engines:
            S = stage[:n * n]
            if eng == "int8":
                sr.sr_block_qgt_i8(O[:, blo:bhi], [0, n], S, workspace=ws)
            else:
                sr.sr_block_qgt(O[:, blo:bhi], [0, n], S)
            Sb = S.reshape(n, n)
            got = Sb[loc][:, loc].cpu().numpy()
            assert rel(got, ref) < 1e-11, (b, eng)
            diag = torch.diagonal(Sb)
            assert torch.all(diag.imag == 0) and torch.all(diag.real >= 0)


def test_single_gpu_point(sr):
    """The weak-scaling N=1 point: 8192 samples, all 8 blocks on one GPU (per-block schedule)."""
    from paper_2510_08430_b200 import parallel
    w = workloads.CONFIGS[4].with_samples(8192)
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    theta = torch.from_numpy(sr.model.pack(params)).to(dev())
    step = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev(), schedule="per_block")
    d, en = step.run(theta)
    d = d.clone()
    torch.cuda.synchronize()
    b = step.buf
    assert torch.all(torch.isfinite(torch.view_as_real(d)))
    el = b.e_loc.cpu().numpy()
    assert abs(en.item() - el.mean()) < 1e-12 * abs(el.mean())
    # F = A^H e_tilde (cuBLAS as an independent instrument on the GPU buffers)
    assert (torch.linalg.vector_norm(b.F - b.O.conj().T @ b.e_tilde) / torch.linalg.vector_norm(b.F)).item() < 1e-10
    offs = b.offs
    n_max = max(offs[i + 1] - offs[i] for i in range(len(offs) - 1))
    del step.ops
    torch.cuda.empty_cache()
    stage = torch.empty(n_max * n_max, dtype=C128, device=dev())
    for i in range(len(offs) - 1):
        lo, hi = offs[i], offs[i + 1]
        n = hi - lo
        S = stage[:n * n]
        sr.sr_block_qgt_i8(b.O[:, lo:hi], [0, n], S)
        Sb = S.reshape(n, n)
        assert torch.equal(Sb, Sb.conj().T.resolve_conj())
        r = Sb @ d[lo:hi] + w.lam * d[lo:hi] + b.F[lo:hi]
        assert (torch.linalg.vector_norm(r) / torch.linalg.vector_norm(b.F[lo:hi])).item() < 1e-9, i
