"""World-size-2 gloo run of the sample-sharded orchestration (parallel.ShardedStep).

The stage arithmetic is injected (OracleOps, numpy on CPU tensors) so that the collective
pattern — moment all-reduce, force all-reduce, per-block reduce to the owner, owner solve,
dtheta all-reduce — is exercised without a GPU; the result must equal the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads
from oracle import estimators, hamiltonian, network, solvers


def _unflatten(theta, widths):
    out, pos = [], 0
    for l in range(len(widths) - 1):
        fi, fo = widths[l], widths[l + 1]
        w = theta[pos:pos + fi * fo].reshape(fo, fi)
        pos += fi * fo
        out.append((w, theta[pos:pos + fo]))
        pos += fo
    return out


class OracleOps:
    def jacobian(self, widths, theta, spins, log_psi, O):
        params = _unflatten(theta.numpy(), widths)
        O.copy_(torch.from_numpy(network.jacobian(params, spins.numpy())))
        log_psi.copy_(torch.from_numpy(network.log_psi(params, spins.numpy())))
        self.params = params

    def local_energy(self, widths, theta, bij, bj, spins, log_psi, e_loc):
        bonds = [(int(i), int(j), float(J)) for (i, j), J in zip(bij.tolist(), bj.tolist())]
        e_loc.copy_(torch.from_numpy(hamiltonian.local_energies(self.params, spins.numpy(), bonds)))

    # moments row: [sum O / n_total (hi) | lo | sum E / n_total (hi) | lo]; lo rows unused here
    def column_moments(self, O, e_loc, n_total, moments):
        n_p = O.shape[1]
        moments.zero_()
        moments[:n_p].copy_(O.sum(dim=0) / n_total)
        moments[2 * n_p].copy_(e_loc.sum() / n_total)

    def center_force_global(self, O, e_loc, n_total, moments_all, energy, e_tilde, F_partial):
        n_p = O.shape[1]
        tot = moments_all.sum(dim=0)
        s = 1.0 / np.sqrt(n_total)
        energy.copy_(tot[2 * n_p].reshape(1))
        O.copy_((O - tot[:n_p]) * s)
        e_tilde.copy_((e_loc - tot[2 * n_p]) * s)
        F_partial.copy_(O.conj().T @ e_tilde)

    def block_qgt(self, A, offs, S):
        pos = 0
        for b in range(len(offs) - 1):
            a = A[:, offs[b]:offs[b + 1]]
            n = a.shape[1]
            S[pos:pos + n * n].copy_((a.conj().T @ a).reshape(-1))
            pos += n * n

    def gram_nh(self, A, B, C):
        C.copy_(A @ B.conj().T)

    def aHv(self, A, v, alpha, out):
        out.copy_(alpha * (A.conj().T @ v))

    def av(self, A, v, alpha, out):
        out.copy_(alpha * (A @ v))

    def gram_tn(self, A, B, C):
        C.copy_(A.conj().T @ B)

    def gram_nh_sub(self, A, B, C):
        C.sub_(A @ B.conj().T)

    # the int8 rectangle interface of dist_full_qgt (the oracle forms the same products)
    def cols_prepare(self, A):
        return A

    def cols_gram(self, A, row0, C, accumulate=False):
        m, n = C.shape
        prod = A[:, row0:row0 + m].conj().T @ A[:, :n]
        C.add_(prod) if accumulate else C.copy_(prod)

    def rows_prepare(self, L):
        return L

    def rows_sub(self, L, row0, C):
        m, n = C.shape
        C.sub_(L[row0:row0 + m] @ L[:n].conj().T)

    def chol_inv(self, M, lam, L, Linv):
        m = M.numpy()
        m = np.tril(m) + np.tril(m, -1).conj().T + lam * np.eye(m.shape[0])
        l_ = np.linalg.cholesky(m)
        L.copy_(torch.from_numpy(l_))
        Linv.copy_(torch.from_numpy(np.tril(np.linalg.inv(l_))))

    def zdotc(self, x, y, out):
        out.copy_(torch.vdot(x, y).reshape(1))

    def cg_axpy(self, x, y, num, den, sign):
        y.add_(sign * (num / den) * x)

    def cg_xpby(self, x, y, num, den):
        y.copy_(x + (num / den) * y)

    def block_solve(self, offs, S, F, lam, dtheta, info=None):
        pos = 0
        for b in range(len(offs) - 1):
            lo, hi = offs[b], offs[b + 1]
            n = hi - lo
            M = S[pos:pos + n * n].reshape(n, n).numpy()
            M = np.tril(M) + np.tril(M, -1).conj().T     # the C ABI reads the lower triangle only
            x = solvers.full_solve(M, F[lo:hi].numpy(), lam)
            dtheta[lo:hi].copy_(torch.from_numpy(x))
            pos += n * n


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_08430_b200.parallel import ShardedStep
    w = workloads.CONFIGS[0].with_samples(64)
    spins, params = workloads.make_inputs(w)
    import paper_2510_08430_b200 as sr
    ij, jj = sr.lattice.for_workload(w)
    step = ShardedStep(w.widths, spins, ij, jj, w.lam, rank, world, "cpu", ops=OracleOps(),
                       per_block_gram=world != 2)   # world 2 also covers the grouped launch
    d, e = step.run(torch.from_numpy(sr.model.pack(params)))
    d_full = step.full_qgt_solve()   # comparison paths, sharded the same way
    d_cg = step.full_qgt_solve(method="cg")
    step.dist_nb = 100                # 7 panels of the 640-parameter QGT, block-cyclic over ranks
    d_dist = step.full_qgt_solve(method="dist")
    d_ntk = step.ntk_solve()
    if rank == 0:
        np.save(result_path, np.concatenate([d.numpy(), e.numpy(), d_full.numpy(), d_ntk.numpy(), d_cg.numpy(),
                                             d_dist.numpy()]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sharded_step_equals_unsharded_oracle(tmp_path, world):
    """world 1: one owner of both blocks; 2: one block each; 3, 4: ranks without a block (4: the
    even-G middle step of the NTK ring schedule)."""
    out = str(tmp_path / "d.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    w = workloads.CONFIGS[0].with_samples(64)
    n_p = w.n_params
    got, got_full, got_ntk, got_cg, got_dist = (res[:n_p + 1], res[n_p + 1:2 * n_p + 1], res[2 * n_p + 1:3 * n_p + 1],
                                                res[3 * n_p + 1:4 * n_p + 1], res[4 * n_p + 1:])
    spins, params = workloads.make_inputs(w)
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    off = network.layer_offsets(params)
    ref = solvers.block_solve(estimators.qgt_blocks(O, off), estimators.force(O, e), off, w.lam)
    assert np.linalg.norm(got[:-1] - ref) / np.linalg.norm(ref) < 1e-10
    assert abs(got[-1] - estimators.energy(e)) < 1e-12
    # full-QGT and NTK comparison solves (sharded) against the oracle's full solve
    full = solvers.full_solve(estimators.qgt_full(O), estimators.force(O, e), w.lam)
    assert np.linalg.norm(got_full - full) / np.linalg.norm(full) < 1e-10
    assert np.linalg.norm(got_ntk - full) / np.linalg.norm(full) < 1e-10
    assert np.linalg.norm(got_cg - full) / np.linalg.norm(full) < 1e-10
    assert np.linalg.norm(got_dist - full) / np.linalg.norm(full) < 1e-10


@pytest.mark.parametrize("world", [3, 8])
def test_loopback_threads_equal_unsharded_oracle(world):
    """parallel.run_loopback / LoopbackComm (the in-process multi-rank emulation that
    tests/test_gpu_loopback.py runs with the real kernels on one GPU): G threads with the
    oracle's stage arithmetic give the unsharded oracle's block, full-QGT and NTK updates."""
    from paper_2510_08430_b200 import parallel
    import paper_2510_08430_b200 as sr
    w = workloads.CONFIGS[0].with_samples(64)
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    theta = torch.from_numpy(sr.model.pack(params))

    def make(r, comm, lock):
        return parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, r, world, "cpu", comm=comm,
                                    ops=parallel.locked(OracleOps(), lock))

    def work(r, step):
        d, e = step.run(theta)
        return d.clone(), e.clone(), step.full_qgt_solve().clone(), step.ntk_solve().clone()

    outs = parallel.run_loopback(world, make, work)
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    off = network.layer_offsets(params)
    ref = solvers.block_solve(estimators.qgt_blocks(O, off), estimators.force(O, e), off, w.lam)
    full = solvers.full_solve(estimators.qgt_full(O), estimators.force(O, e), w.lam)
    for d, en, d_full, d_ntk in outs:
        assert np.linalg.norm(d.numpy() - ref) / np.linalg.norm(ref) < 1e-10
        assert abs(en.item() - estimators.energy(e)) < 1e-12
        assert np.linalg.norm(d_full.numpy() - full) / np.linalg.norm(full) < 1e-10
        assert np.linalg.norm(d_ntk.numpy() - full) / np.linalg.norm(full) < 1e-10


def test_loopback_failure_does_not_hang():
    """A rank that raises aborts the rendezvous: the others return and the error is re-raised."""
    from paper_2510_08430_b200 import parallel

    def make(r, comm, lock):
        return comm

    def work(r, comm):
        if r == 1:
            raise ValueError("rank 1 failed")
        t = torch.ones(3)
        comm.all_reduce(t)
        return t

    with pytest.raises(Exception):
        parallel.run_loopback(3, make, work)


def test_ntk_ring_schedule_covers_each_pair_once():
    from paper_2510_08430_b200.parallel import ShardedStep
    for G in range(1, 10):
        sched = ShardedStep.ntk_schedule(G)
        pairs = []
        for r in range(G):
            for t, src, dst in sched[r]:
                if t == 0:
                    pairs.append((r, r))
                elif src is not None:
                    pairs.append((max(r, src), min(r, src)))
                    assert dst is None or sched[dst][t][1] == r     # the receiver expects it
        assert sorted(pairs) == sorted((i, j) for i in range(G) for j in range(i + 1)), G
        assert max(len([s for s in sched[r] if s[0] == 0 or s[1] is not None]) for r in range(G)) <= G // 2 + 1


@pytest.mark.parametrize("world,nb", [(1, 64), (3, 50), (4, 37)])
def test_dist_full_qgt_o1_conditioned(world, nb):
    """parallel.dist_full_qgt (S formed and factorised by block-cyclic panel rows across ranks)
    on an O(1)-conditioned S = A^H A (||S|| ~ 1 >> lambda), ragged panels, loopback ranks with
    the oracle's arithmetic, against numpy's dense solve."""
    from paper_2510_08430_b200 import parallel
    rng = np.random.default_rng(world * 100 + nb)
    ns, n_p, lam = 300, 210, 1e-3
    A = (rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))) / np.sqrt(2 * ns)
    F = rng.standard_normal(n_p) + 1j * rng.standard_normal(n_p)
    ref = -np.linalg.solve(A.conj().T @ A + lam * np.eye(n_p), F)
    bounds = [parallel.shard_range(ns, r, world) for r in range(world)]

    def make(r, comm, lock):
        return comm, lock

    def work(r, cl):
        comm, lock = cl
        lo, hi = bounds[r]
        return [parallel.dist_full_qgt(parallel.locked(OracleOps(), lock), comm, r, world,
                                       torch.from_numpy(A[lo:hi].copy()), torch.from_numpy(F), lam, nb=nb,
                                       engine=eng).numpy() for eng in ("fp64", "int8")]

    outs = parallel.run_loopback(world, make, work)
    for xs in outs:
        for x in xs:
            assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-10


def test_loopback_ragged_tiny_shards_all_paths():
    """5 samples over 4 ranks (shards of 2, 1, 1, 1): the block step and every comparison path
    (dense reduce-to-rank-0, ring NTK, CG, distributed dense with ragged panels) against the
    oracle; fewer samples than ranks is rejected."""
    from paper_2510_08430_b200 import parallel
    import paper_2510_08430_b200 as sr
    w = workloads.CONFIGS[0].with_samples(5)
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    theta = torch.from_numpy(sr.model.pack(params))

    def make(r, comm, lock):
        return parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, r, 4, "cpu", comm=comm,
                                    ops=parallel.locked(OracleOps(), lock))

    def work(r, step):
        d, _ = step.run(theta)
        out = [d.clone(), step.full_qgt_solve(method="dense").clone(), step.ntk_solve().clone(),
               step.full_qgt_solve(method="cg").clone()]
        step.dist_nb = 100
        return out + [step.full_qgt_solve(method="dist").clone()]

    outs = parallel.run_loopback(4, make, work)
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    off = network.layer_offsets(params)
    ref = solvers.block_solve(estimators.qgt_blocks(O, off), estimators.force(O, e), off, w.lam)
    full = solvers.full_solve(estimators.qgt_full(O), estimators.force(O, e), w.lam)
    got = [x.numpy() for x in outs[0]]
    assert np.linalg.norm(got[0] - ref) / np.linalg.norm(ref) < 1e-10
    for x in got[1:]:
        assert np.linalg.norm(x - full) / np.linalg.norm(full) < 1e-10
    with pytest.raises(ValueError):
        parallel.ShardedStep(w.widths, spins[:3], ij, jj, w.lam, 0, 4, "cpu", ops=OracleOps())
