"""The sample-sharded step (parallel.ShardedStep: C ABI stages + NCCL collectives) on a real
GPU, as a one-rank NCCL process group: same dtheta and energy as the single-GPU step and as
the oracle (BASELINE.json north_star: the NCCL reduce of the per-block partial S_b to its
owner, the owner's solve and the dtheta all-reduce).  The world-size-2 orchestration is
covered on CPU by tests/test_parallel_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import workloads
from oracle import estimators, hamiltonian, network, solvers

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    if dist.is_initialized():
        yield
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,per_block", [(0, False), (1, False), (0, True), (1, True)])
def test_sharded_step_matches_local_and_oracle(nccl_group, cfg, per_block):
    import paper_2510_08430_b200 as sr
    from paper_2510_08430_b200 import parallel
    w = workloads.CONFIGS[cfg]
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    dev = torch.device("cuda:0")
    theta = torch.from_numpy(sr.model.pack(params)).to(dev)
    local = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev)
    d_local, e_local = (x.clone() for x in local.run(theta))
    shard = parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, 0, 1, dev, per_block_gram=per_block)
    d_shard, e_shard = shard.run(theta)
    torch.cuda.synchronize()
    rel = (torch.linalg.vector_norm(d_shard - d_local) / torch.linalg.vector_norm(d_local)).item()
    assert rel < 1e-11
    assert abs(e_shard.item() - e_local.item()) <= 1e-13 * abs(e_local.item())
    if cfg == 0:   # small enough for the oracle
        O = network.jacobian(params, spins)
        e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
        off = network.layer_offsets(params)
        ref = solvers.block_solve(estimators.qgt_blocks(O, off), estimators.force(O, e), off, w.lam)
        got = d_shard.cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-9


def test_sharded_step_graph_replay(nccl_group):
    """The sharded step captured as one CUDA graph (NCCL collectives as graph nodes, as bench.py
    times it) replays to the eager result, and follows a new theta."""
    import paper_2510_08430_b200 as sr
    from paper_2510_08430_b200 import parallel
    w = workloads.CONFIGS[0]
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    dev = torch.device("cuda:0")
    theta = torch.from_numpy(sr.model.pack(params)).to(dev)
    for per_block in (False, True):
        shard = parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, 0, 1, dev, per_block_gram=per_block)
        d_eager = shard.run(theta)[0].clone()
        shard.capture(theta)
        d_graph = shard.replay()[0].clone()
        torch.cuda.synchronize()
        assert torch.equal(d_graph, d_eager)
        theta.mul_(1.01)
        d_new = shard.replay()[0].clone()
        d_ref = parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, 0, 1, dev,
                                     per_block_gram=per_block).run(theta)[0]
        torch.cuda.synchronize()
        assert torch.equal(d_new, d_ref)
        theta.div_(1.01)


def test_sharded_comparison_solves(nccl_group):
    """The full-QGT and NTK comparison paths sharded the same way (ShardedStep.full_qgt_solve /
    ntk_solve: partial-S reduce to rank 0; NTK block rows A_r A_s^H by broadcasts, gathered,
    y broadcast, A_r^H y_r all-reduced) agree with the single-GPU sr_full_qgt_solve /
    sr_ntk_solve on the same centred Jacobian, and with each other (push-through)."""
    import paper_2510_08430_b200 as sr
    from paper_2510_08430_b200 import parallel
    w = workloads.CONFIGS[0]
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    dev = torch.device("cuda:0")
    theta = torch.from_numpy(sr.model.pack(params)).to(dev)
    shard = parallel.ShardedStep(w.widths, spins, ij, jj, w.lam, 0, 1, dev, per_block_gram=True)
    shard.run(theta)
    d_full = shard.full_qgt_solve().clone()
    d_ntk = shard.ntk_solve().clone()
    b = shard.buf
    ref_full = torch.empty_like(d_full)
    ref_ntk = torch.empty_like(d_ntk)
    sr.sr_full_qgt_solve(b.O, b.F, w.lam, ref_full)
    sr.sr_ntk_solve(b.O, b.e_tilde, w.lam, ref_ntk)
    torch.cuda.synchronize()
    rel = lambda a, c: (torch.linalg.vector_norm(a - c) / torch.linalg.vector_norm(c)).item()  # noqa: E731
    assert rel(d_full, ref_full) < 1e-12
    assert rel(d_ntk, ref_ntk) < 1e-10
    assert rel(d_ntk, d_full) < 1e-10
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    full = solvers.full_solve(estimators.qgt_full(O), estimators.force(O, e), w.lam)
    assert np.linalg.norm(d_full.cpu().numpy() - full) / np.linalg.norm(full) < 1e-9
