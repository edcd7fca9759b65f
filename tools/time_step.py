"""Time sr_step (device-resident inputs) eagerly and as one CUDA graph; print ms/step and
dtheta's checksum.  Knobs come from the environment (SR_PIPE, SR_GRAM_CTAS, SR_TRAIL_CTAS).
Usage: python tools/time_step.py [config index] [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402

w = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda:0")
spins, params = workloads.make_inputs(w)
ij, jj = sr.lattice.for_workload(w)
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
sp, bij, bj = (torch.from_numpy(x).to(dev) for x in (spins, ij, jj))
ws = torch.empty(sr.sr_step_workspace_bytes(w.widths, w.n_samples, len(jj)), dtype=torch.uint8, device=dev)
dtheta = torch.empty(w.n_params, dtype=torch.complex128, device=dev)
energy = torch.empty(1, dtype=torch.complex128, device=dev)


def one():
    sr.sr_step(w.widths, theta, sp, bij, bj, w.lam, dtheta, energy, ws)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for _ in range(3):
    one()
torch.cuda.synchronize()
ref = dtheta.clone()
eager = timed(one)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    one()
for _ in range(3):
    g.replay()
graph = timed(g.replay)
diff = (torch.linalg.norm(dtheta - ref) / torch.linalg.norm(ref)).item()
env = {k: v for k, v in os.environ.items() if k.startswith("SR_")}
print(f"{w.name} {env} eager {eager:.3f} ms  graph {graph:.3f} ms  |dtheta| {torch.linalg.norm(ref).item():.12e} "
      f"graph-vs-eager {diff:.1e}", flush=True)
