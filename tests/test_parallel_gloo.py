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

    def block_solve(self, offs, S, F, lam, dtheta, info=None):
        pos = 0
        for b in range(len(offs) - 1):
            lo, hi = offs[b], offs[b + 1]
            n = hi - lo
            x = solvers.full_solve(S[pos:pos + n * n].reshape(n, n).numpy(), F[lo:hi].numpy(), lam)
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
    d_ntk = step.ntk_solve()
    if rank == 0:
        np.save(result_path, np.concatenate([d.numpy(), e.numpy(), d_full.numpy(), d_ntk.numpy()]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_step_equals_unsharded_oracle(tmp_path, world):
    """world 1: one owner of both blocks; 2: one block each; 3: a rank without a block."""
    out = str(tmp_path / "d.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    w = workloads.CONFIGS[0].with_samples(64)
    n_p = w.n_params
    got, got_full, got_ntk = res[:n_p + 1], res[n_p + 1:2 * n_p + 1], res[2 * n_p + 1:]
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
