"""Run stages (1)-(2) once on a bench workload (for ncu captures of energy_eval) and time
the local-energy stage with CUDA events.  Usage: python tools/energy_stage.py [workload] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_08430_b200 as sr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_WORKLOAD
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = bench.workload_for(name, 1)
spins, params = bench.workloads.make_inputs(w)
ij, jj = sr.lattice.for_workload(w)
dev = torch.device("cuda:0")
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
sp = torch.from_numpy(spins).to(dev)
lp = torch.empty(w.n_samples, dtype=torch.complex128, device=dev)
O = torch.empty(w.n_samples, w.n_params, dtype=torch.complex128, device=dev)
sr.sr_jacobian(w.widths, theta, sp, lp, O)
del O
e = torch.empty(w.n_samples, dtype=torch.complex128, device=dev)
bij, bj = torch.from_numpy(ij).to(dev), torch.from_numpy(jj).to(dev)
ws = torch.empty(sr.load().sr_local_energy_workspace_bytes(*sr._lib._widths(w.widths), w.n_samples, len(jj)),
                 dtype=torch.uint8, device=dev)
sr.sr_local_energy(w.widths, theta, bij, bj, sp, lp, e, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    sr.sr_local_energy(w.widths, theta, bij, bj, sp, lp, e, workspace=ws)
e1.record()
torch.cuda.synchronize()
print(f"{name}: local energy {e0.elapsed_time(e1) / reps:.3f} ms")
