"""One rank's share of the sample-sharded step, measured on one GPU (no collectives): the
stages of parallel.ShardedStep's per-block mode for one rank of `world` ranks at a BASELINE
configuration -- Jacobian, local energy and centring on the rank's N_s/world samples, the
per-block partial Grams (each one launch, the reduce target being the owned slot or a
staging buffer), and the owner's solve of its blocks.  The NCCL traffic (per-block partial
S, force, dtheta) is reported as bytes, not timed.  Usage:
    python tools/rank_estimate.py [config index] [world] [rank]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
from paper_2510_08430_b200 import parallel  # noqa: E402
import workloads  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = workloads.CONFIGS[ci]
dev = torch.device("cuda:0")
spins_all, params = workloads.make_inputs(w)
lo, hi = parallel.shard_range(w.n_samples, rank, world)
spins = spins_all[lo:hi]
ij, jj = sr.lattice.for_workload(w)
sizes = w.layer_sizes
ranges = parallel.block_ranges(sizes, world)
olo, ohi = ranges[rank]
offs = sr.block_offsets(w.widths)
own_offs = [offs[b] - offs[olo] for b in range(olo, ohi + 1)] if ohi > olo else None
ops = parallel.CudaOps(w.widths, hi - lo, len(jj), dev, "int8", solve_offsets=own_offs)
buf = parallel._Buffers(w.widths, spins, ij, jj, dev, full_s=False)
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
S_own = torch.empty(max(1, sum(n * n for n in sizes[olo:ohi])), dtype=torch.complex128, device=dev)
others = [n * n for b, n in enumerate(sizes) if not olo <= b < ohi]
staging = [torch.empty(max(others), dtype=torch.complex128, device=dev) for _ in range(min(2, len(others)))]


def t(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = {}
ms["jacobian"] = t(lambda: ops.jacobian(buf.widths, theta, buf.spins, buf.log_psi, buf.O))
ms["local_energy"] = t(lambda: ops.local_energy(buf.widths, theta, buf.bij, buf.bj, buf.spins, buf.log_psi, buf.e_loc))
ms["center_force"] = t(lambda: ops.center_force(buf.O, buf.e_loc, buf.energy, buf.e_tilde, buf.F))


def grams():
    k = 0
    for blk in range(len(sizes)):
        a, b = offs[blk], offs[blk + 1]
        n = b - a
        if olo <= blk < ohi:
            pos = sum(m * m for m in sizes[olo:blk])
            target = S_own[pos:pos + n * n]
        else:
            target = staging[k % len(staging)][:n * n]
            k += 1
        ops.block_qgt(buf.O[:, a:b], [0, n], target)


ms["partial_grams"] = t(grams)
F_own = buf.F[offs[olo]:offs[ohi]]
d_own = torch.empty_like(F_own)
if own_offs is not None:
    ms["owner_solve"] = t(lambda: ops.block_solve(own_offs, S_own, F_own, w.lam, d_own))
total = sum(ms.values())
bytes_s = 16 * sum(n * n for b, n in enumerate(sizes) if not olo <= b < ohi)
print(f"{w.name}, rank {rank} of {world}: {hi - lo} samples, owns blocks {list(range(olo, ohi))} "
      f"({[sizes[b] for b in range(olo, ohi)]}); " + ", ".join(f"{k} {v:.1f} ms" for k, v in ms.items())
      + f"; sum {total:.1f} ms; partial S sent {bytes_s / 1e9:.1f} GB, force/dtheta all-reduce "
      f"{2 * 16 * buf.n_p / 1e6:.1f} MB; peak memory {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
