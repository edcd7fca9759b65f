"""Multi-rank sample-sharded step with the REAL kernels on one GPU: G ranks of
parallel.ShardedStep run as G threads of this process (parallel.run_loopback), each with its
own buffers and CudaOps, the collectives done by parallel.LoopbackComm (host-side rendezvous:
copies and rank-ordered sums between kernel launches; no kernel waits on another rank's).

This exercises exactly the dataflow a G-GPU NCCL run executes -- the double-double moment
all-gather and the n_parts = G centring (sr_column_moments / sr_center_force_global), the
force all-reduce, per-block partial Grams reduced to cost-balanced owners, the owners'
solves, the dtheta all-reduce, and the sharded NTK / full-QGT comparison paths -- with
libsrblock.so's kernels, for G = 2, 4, 8.  Only one GPU is available here, so the NCCL
transport itself is covered by tests/test_gpu_sharded.py (one rank) and the collective
pattern on gloo by tests/test_parallel_gloo.py.

Bars: dtheta within 1e-11 of the single-GPU LocalStep (same kernels, different summation
order of the sharded reductions), energy within 1e-13; configs[0] also against the oracle
(1e-9, north_star).
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import estimators, hamiltonian, network, solvers

pytestmark = pytest.mark.gpu


def _setup(cfg, ns=None):
    import paper_2510_08430_b200 as sr
    sr.load()
    w = workloads.CONFIGS[cfg] if ns is None else workloads.CONFIGS[cfg].with_samples(ns)
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    dev = torch.device("cuda:0")
    theta = torch.from_numpy(sr.model.pack(params)).to(dev)
    return sr, w, spins, params, ij, jj, dev, theta


def _rel(a, b):
    return (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)).item()


def _loopback(world, w, spins, ij, jj, dev, theta, per_block=True, compare=False):
    from paper_2510_08430_b200 import parallel

    def make(r, comm, lock):
        step = parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, r, world, dev, comm=comm,
                                    per_block_gram=per_block)
        step.ops = parallel.locked(step.ops, lock)
        return step

    def work(r, step):
        d, e = step.run(theta)
        out = [d.clone(), e.clone()]
        if compare:
            out += [step.full_qgt_solve().clone(), step.ntk_solve().clone(),
                    step.full_qgt_solve(method="cg").clone()]
            step.dist_nb = 128
            out += [step.full_qgt_solve(method="dist").clone()]
        torch.cuda.synchronize()
        return out

    return parallel.run_loopback(world, make, work)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_loopback_sharded_step_matches_local(world):
    sr, w, spins, params, ij, jj, dev, theta = _setup(1)
    from paper_2510_08430_b200 import parallel
    d_local, e_local = (x.clone() for x in parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev).run(theta))
    outs = _loopback(world, w, spins, ij, jj, dev, theta)
    for r, (d, e) in enumerate(outs):
        assert torch.equal(d, outs[0][0]) and torch.equal(e, outs[0][1]), r   # all ranks agree exactly
    assert _rel(outs[0][0], d_local) < 1e-11
    assert abs(outs[0][1].item() - e_local.item()) <= 1e-13 * abs(e_local.item())


@pytest.mark.parametrize("world,per_block", [(2, False), (3, True), (4, True)])
def test_loopback_configs0_oracle_and_comparison_paths(world, per_block):
    """configs[0] against the oracle: the block step (grouped or per-block Gram launches), and
    the sharded comparison paths (partial-S reduce for the full QGT; ring-scheduled NTK
    blocks gathered to rank 0) against the oracle's full solve (push-through identity)."""
    sr, w, spins, params, ij, jj, dev, theta = _setup(0)
    outs = _loopback(world, w, spins, ij, jj, dev, theta, per_block=per_block, compare=True)
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    off = network.layer_offsets(params)
    ref = solvers.block_solve(estimators.qgt_blocks(O, off), estimators.force(O, e), off, w.lam)
    full = solvers.full_solve(estimators.qgt_full(O), estimators.force(O, e), w.lam)
    d, en, d_full, d_ntk, d_cg, d_dist = (x.cpu().numpy() for x in outs[0])
    assert np.linalg.norm(d - ref) / np.linalg.norm(ref) < 1e-9
    assert abs(en[0] - estimators.energy(e)) < 1e-12 * abs(estimators.energy(e))
    assert np.linalg.norm(d_full - full) / np.linalg.norm(full) < 1e-9
    assert np.linalg.norm(d_ntk - full) / np.linalg.norm(full) < 1e-9
    assert np.linalg.norm(d_cg - full) / np.linalg.norm(full) < 1e-9
    assert np.linalg.norm(d_dist - full) / np.linalg.norm(full) < 1e-9
    for r in range(world):
        assert torch.equal(outs[r][3], outs[0][3])


def test_local_step_per_block_schedule_matches_batched():
    """LocalStep(schedule="per_block") -- sr_block_qgt_solve, one block's Gram written into its
    factor matrix and solved before the next -- equals the batched schedule (same kernels;
    the Gram tiles and the Cholesky are identical arithmetic), also through sr_step /
    sr_step_host under SR_SCHED_PER_BLOCK, and matches the oracle on configs[0]."""
    sr, w, spins, params, ij, jj, dev, theta = _setup(1)
    from paper_2510_08430_b200 import parallel
    d_b = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev).run(theta)[0].clone()
    step = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev, schedule="per_block")
    d_p = step.run(theta)[0].clone()
    assert _rel(d_p, d_b) < 1e-12
    step.capture(theta)
    assert torch.equal(step.replay()[0], d_p)
    nb = len(jj)
    prev = sr.sr_set_step_schedule(sr.SCHED_PER_BLOCK)
    try:
        ws = torch.empty(sr.sr_step_workspace_bytes(w.widths, w.n_samples, nb)
                         + sr.sr_step_host_extra_bytes(w.widths, w.n_samples, nb), dtype=torch.uint8, device=dev)
        d = torch.empty(w.n_params, dtype=torch.complex128, device=dev)
        en = torch.empty(1, dtype=torch.complex128, device=dev)
        sr.sr_step(w.widths, theta, step.buf.spins, step.buf.bij, step.buf.bj, w.lam, d, en, ws)
        dh = torch.empty(w.n_params, dtype=torch.complex128).pin_memory()
        eh = torch.empty(1, dtype=torch.complex128).pin_memory()
        sr.sr_step_host(w.widths, theta.cpu().pin_memory(), torch.from_numpy(spins).pin_memory(),
                        torch.from_numpy(ij), torch.from_numpy(jj), w.lam, dh, eh, ws)
    finally:
        sr.sr_set_step_schedule(prev)
    assert torch.equal(d, d_p)
    assert torch.equal(dh, d_p.cpu())


def test_block_qgt_solve_reports_first_failing_block():
    """sr_block_qgt_solve's info: 0 on success, else the global row + 1 of the first failing
    pivot (blocks are solved one call at a time; a later block does not reset it)."""
    import paper_2510_08430_b200 as sr
    dev = torch.device("cuda:0")
    A = torch.zeros(4, 75, dtype=torch.complex128, device=dev)   # S = 0
    F = torch.ones(75, dtype=torch.complex128, device=dev)
    d = torch.empty_like(F)
    info = torch.full((1,), -3, dtype=torch.int32, device=dev)
    sr.sr_block_qgt_solve(A, [0, 70, 75], F, 0.0, d, info=info)    # lambda = 0: zero pivots
    assert info.item() == 1
    sr.sr_block_qgt_solve(A, [0, 70, 75], F, 0.5, d, info=info)
    assert info.item() == 0 and torch.allclose(d, -F / 0.5, rtol=1e-15, atol=0)


@pytest.mark.parametrize("world", [1, 3])
def test_full_qgt_cg_matches_dense_o1_conditioned(world):
    """The matrix-free full-QGT solve (parallel.full_qgt_cg: S p = sum_r A_r^H (A_r p) by
    sr_av / sr_aHv, one all-reduce per iteration, sr_zdotc / sr_cg_axpy / sr_cg_xpby updates)
    on an O(1)-conditioned A (||S|| ~ 1 >> lambda = 1e-3), sharded over `world` loopback
    ranks, against numpy's dense solve of the same system (1e-9) and the library's dense
    sr_full_qgt_solve."""
    import paper_2510_08430_b200 as sr
    from paper_2510_08430_b200 import parallel
    sr.load()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(world)
    ns, n_p, lam = 600, 380, 1e-3
    A = (rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))) / np.sqrt(2 * ns)
    F = rng.standard_normal(n_p) + 1j * rng.standard_normal(n_p)
    ref = -np.linalg.solve(A.conj().T @ A + lam * np.eye(n_p), F)
    At, Ft = torch.from_numpy(A).to(dev), torch.from_numpy(F).to(dev)
    bounds = [parallel.shard_range(ns, r, world) for r in range(world)]

    def make(r, comm, lock):
        return comm, lock

    def work(r, cl):
        comm, lock = cl
        ops = parallel.locked(parallel.CudaOps([4, 4], 1, 1, dev), lock)
        lo, hi = bounds[r]
        x, it, res = parallel.full_qgt_cg(ops, comm, At[lo:hi].contiguous(), Ft, lam)
        torch.cuda.synchronize()
        return x.cpu().numpy(), it, res

    outs = parallel.run_loopback(world, make, work)
    x, it, res = outs[0]
    assert res <= 1e-12 and it < 500
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-9
    for o in outs[1:]:
        assert np.array_equal(o[0], x)
    d = torch.empty_like(Ft)
    sr.sr_full_qgt_solve(At, Ft, lam, d)
    assert np.linalg.norm(d.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-9


def test_av_zdotc_cg_kernels():
    """sr_av (alpha A v, column-slice A, ragged sizes), sr_zdotc, sr_cg_axpy / sr_cg_xpby
    against numpy."""
    import paper_2510_08430_b200 as sr
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(5)
    for nr, n in ((1, 1), (37, 129), (300, 4099)):
        Aw = rng.standard_normal((nr, n + 3)) + 1j * rng.standard_normal((nr, n + 3))
        v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        out = torch.empty(nr, dtype=torch.complex128, device=dev)
        sr.sr_av(torch.from_numpy(Aw).to(dev)[:, 2:2 + n], torch.from_numpy(v).to(dev), -0.5, out)
        ref = -0.5 * (Aw[:, 2:2 + n] @ v)
        assert np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-14
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        xd, yd = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
        dot = torch.empty(1, dtype=torch.complex128, device=dev)
        sr.sr_zdotc(xd, yd, dot)
        assert abs(dot.item() - np.vdot(x, y)) < 1e-13 * np.linalg.norm(x) * np.linalg.norm(y)
        num = torch.tensor([2.0 + 1.0j], dtype=torch.complex128, device=dev)
        den = torch.tensor([0.5 - 0.5j], dtype=torch.complex128, device=dev)
        a = (2.0 + 1.0j) / (0.5 - 0.5j)
        y2 = yd.clone()
        sr.sr_cg_axpy(xd, y2, num, den, -1.0)
        assert np.linalg.norm(y2.cpu().numpy() - (y - a * x)) < 1e-13 * np.linalg.norm(y)
        y3 = yd.clone()
        sr.sr_cg_xpby(xd, y3, num, den)
        assert np.linalg.norm(y3.cpu().numpy() - (x + a * y)) < 1e-13 * np.linalg.norm(y)


def test_panel_kernels():
    """sr_gram_tn (C = A^H B), sr_gram_nh_sub (C -= A B^H) and sr_chol_inv (L and L^{-1} of
    M + lambda I) against numpy on ragged sizes, column-slice operands."""
    import paper_2510_08430_b200 as sr
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(12)
    cx = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)   # noqa: E731
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)        # noqa: E731
    for k, m, n in ((1, 1, 1), (70, 63, 130), (300, 65, 64)):
        Aw, Bw = cx(k, m + 3), cx(k, n + 1)
        C = torch.full((m, n), 5.0 + 0j, dtype=torch.complex128, device=dev)
        sr.sr_gram_tn(T(Aw)[:, 2:2 + m], T(Bw)[:, :n], C)
        ref = Aw[:, 2:2 + m].conj().T @ Bw[:, :n]
        assert np.linalg.norm(C.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-14
        A2, B2, C0 = cx(m, k), cx(n, k), cx(m, n)
        C2 = T(C0)
        sr.sr_gram_nh_sub(T(A2), T(B2), C2)
        ref2 = C0 - A2 @ B2.conj().T
        assert np.linalg.norm(C2.cpu().numpy() - ref2) / np.linalg.norm(ref2) < 1e-14
    for n in (1, 63, 64, 65, 200, 1024):
        X = cx(2 * n, n) / np.sqrt(4 * n)
        M = X.conj().T @ X
        lam = 1e-2
        L = torch.empty(n, n, dtype=torch.complex128, device=dev)
        Li = torch.empty(n, n, dtype=torch.complex128, device=dev)
        info = torch.full((1,), -1, dtype=torch.int32, device=dev)
        sr.sr_chol_inv(T(np.tril(M) + np.triu(cx(n, n), 1)), lam, L, Li, info=info)   # upper triangle ignored
        Lh, Lih = L.cpu().numpy(), Li.cpu().numpy()
        assert info.item() == 0
        Mref = M + lam * np.eye(n)
        assert np.linalg.norm(Lh @ Lh.conj().T - Mref) / np.linalg.norm(Mref) < 1e-13
        assert np.allclose(np.triu(Lh, 1), 0) and np.allclose(np.triu(Lih, 1), 0)
        assert np.linalg.norm(Lih @ Lh - np.eye(n)) / np.sqrt(n) < 1e-12


def test_int8_rectangles():
    """sr_cols_i8_prepare / sr_cols_i8_gram (C (+)= A[:, row0:row0+m]^H A[:, 0:n], K-split for
    more than 8192 samples) and sr_rows_i8_prepare / sr_rows_i8_sub (C -= L[row0:row0+m]
    L[0:n]^H) against numpy, entrywise to 1e-11 of sqrt(|x_i|^2 |y_j|^2)."""
    import paper_2510_08430_b200 as sr
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(21)
    cx = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)   # noqa: E731
    for ns, ncols, row0, m, n in ((700, 300, 37, 130, 250), (9000, 200, 0, 200, 200), (5, 70, 69, 1, 70)):
        A = cx(ns, ncols) * np.exp(rng.uniform(-4, 4, ncols))[None, :]
        cs = sr.ColSlices(torch.from_numpy(A).to(dev))
        C = torch.empty(m, n, dtype=torch.complex128, device=dev)
        cs.gram(row0, C)
        ref = A[:, row0:row0 + m].conj().T @ A[:, :n]
        scale = np.outer(np.linalg.norm(A[:, row0:row0 + m], axis=0), np.linalg.norm(A[:, :n], axis=0))
        assert np.all(np.abs(C.cpu().numpy() - ref) <= 1e-11 * scale)
        cs.gram(row0, C, accumulate=True)
        assert np.all(np.abs(C.cpu().numpy() - 2 * ref) <= 2e-11 * scale)
    for rows, K, row0, m, n in ((500, 64, 100, 129, 300), (1100, 1024, 1000, 100, 1100), (3, 7, 2, 1, 3)):
        L = cx(rows, K)
        C0 = cx(m, n)
        C = torch.from_numpy(C0).to(dev)
        rs = sr.RowSlices(torch.from_numpy(L).to(dev))
        rs.sub(row0, C)
        ref = C0 - L[row0:row0 + m] @ L[:n].conj().T
        scale = np.outer(np.linalg.norm(L[row0:row0 + m], axis=1), np.linalg.norm(L[:n], axis=1))
        assert np.all(np.abs(C.cpu().numpy() - ref) <= 1e-11 * scale + 1e-15 * np.abs(C0))


@pytest.mark.parametrize("world,nb", [(1, 1024), (3, 200)])
def test_dist_full_qgt_gpu(world, nb):
    """parallel.dist_full_qgt with the real kernels (sr_gram_tn formation reduced to panel
    owners, sr_chol_inv diagonal blocks, sr_gram_nh TRSM, sr_gram_nh_sub trailing updates,
    sr_av / sr_aHv substitutions) over loopback ranks: an O(1)-conditioned QGT against numpy,
    and configs[1]'s centred Jacobian (n_p = 16240, 4096 samples) against the single-GPU dense
    sr_full_qgt_solve."""
    import paper_2510_08430_b200 as sr
    from paper_2510_08430_b200 import parallel
    sr.load()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(world)
    ns, n_p, lam = 700, 450, 1e-3
    A = (rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))) / np.sqrt(2 * ns)
    F = rng.standard_normal(n_p) + 1j * rng.standard_normal(n_p)
    ref = -np.linalg.solve(A.conj().T @ A + lam * np.eye(n_p), F)

    def solve(Ad, Fd, nb_):
        bounds = [parallel.shard_range(Ad.shape[0], r, world) for r in range(world)]

        def make(r, comm, lock):
            return comm, lock

        def work(r, cl):
            comm, lock = cl
            ops = parallel.locked(parallel.CudaOps([4, 4], 1, 1, dev), lock)
            lo, hi = bounds[r]
            xs = [parallel.dist_full_qgt(ops, comm, r, world, Ad[lo:hi], Fd, lam, nb=nb_, engine=eng)
                  for eng in ("int8", "fp64")]
            torch.cuda.synchronize()
            return xs
        outs = parallel.run_loopback(world, make, work)
        for o in outs[1:]:
            assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1])
        assert _rel(outs[0][0], outs[0][1]) < 1e-10      # int8 rectangles vs FP64 DMMA
        return outs[0][0]

    x = solve(torch.from_numpy(A).to(dev), torch.from_numpy(F).to(dev), min(nb, 128))
    assert np.linalg.norm(x.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-10
    # configs[1] at full size
    sr_, w, spins, params, ij, jj, dev, theta = _setup(1)
    step = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev)
    step.run(theta)
    b = step.buf
    step.buf.S = None
    step.ops.ws = None
    torch.cuda.empty_cache()
    d_ref = torch.empty_like(b.F)
    sr.sr_full_qgt_solve(b.O, b.F, w.lam, d_ref)
    d = solve(b.O, b.F, nb)
    assert _rel(d, d_ref) < 1e-10


@pytest.mark.parametrize("cfg,chunk", [(0, 100), (1, 1024), (1, 4096)])
def test_chunked_step_matches_local(cfg, chunk):
    """parallel.ChunkedStep (samples in chunks, Gram accumulated with sr_block_qgt_i8_acc, the
    n_parts = n_chunks centring) equals the one-pass LocalStep (1e-12) and, on configs[0], the
    oracle (1e-9); its CUDA-graph replay equals its eager run."""
    sr, w, spins, params, ij, jj, dev, theta = _setup(cfg)
    from paper_2510_08430_b200 import parallel
    d_local, e_local = (x.clone() for x in parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev).run(theta))
    step = parallel.ChunkedStep(w.widths, spins, ij, jj, w.lam, dev, chunk=chunk)
    d, e = (x.clone() for x in step.run(theta))
    assert _rel(d, d_local) < 1e-12
    assert abs(e.item() - e_local.item()) <= 1e-13 * abs(e_local.item())
    step.capture(theta)
    assert torch.equal(step.replay()[0], d)
    if cfg == 0:
        O = network.jacobian(params, spins)
        el = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
        off = network.layer_offsets(params)
        ref = solvers.block_solve(estimators.qgt_blocks(O, off), estimators.force(O, el), off, w.lam)
        assert np.linalg.norm(d.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-9


def test_block_qgt_i8_acc():
    """sr_block_qgt_i8_acc adds the Gram of its rows to S: two row halves summed equal the
    whole (to FP64 rounding), and N_s = 0 leaves S unchanged."""
    import paper_2510_08430_b200 as sr
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3)
    A = torch.complex(torch.randn(900, 300, dtype=torch.float64, device=dev, generator=g),
                      torch.randn(900, 300, dtype=torch.float64, device=dev, generator=g))
    offs = [0, 100, 300]
    n_s = 100 * 100 + 200 * 200
    S1 = torch.empty(n_s, dtype=torch.complex128, device=dev)
    S2 = torch.empty(n_s, dtype=torch.complex128, device=dev)
    sr.sr_block_qgt_i8(A, offs, S1)
    sr.sr_block_qgt_i8(A[:400], offs, S2)
    sr.sr_block_qgt_i8_acc(A[400:], offs, S2)
    before = S2.clone()
    sr.sr_block_qgt_i8_acc(A[:0], offs, S2)
    assert torch.equal(S2, before)
    assert _rel(S2, S1) < 1e-14


def test_per_block_schedule_fp64_engine():
    """The per-block schedule on the FP64 DMMA engine (block Gram into the factor matrix by the
    TMA-staged DMMA kernel, FP64 trailing updates) equals the batched FP64 schedule."""
    sr, w, spins, params, ij, jj, dev, theta = _setup(1)
    from paper_2510_08430_b200 import parallel
    prev = sr.sr_set_gram_engine(sr.GRAM_FP64)
    try:
        d_b = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev, gram_engine="fp64").run(theta)[0].clone()
        d_p = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev, gram_engine="fp64",
                                 schedule="per_block").run(theta)[0].clone()
        torch.cuda.synchronize()
    finally:
        sr.sr_set_gram_engine(prev)
    assert _rel(d_p, d_b) < 1e-12
