"""Time the Jacobian and local-energy stages (CUDA events; also usable under ncu for a launch list).
Usage: python tools/jac_timing.py [config index]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402

w = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
spins, params = workloads.make_inputs(w)
dev = torch.device("cuda:0")
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
sp = torch.from_numpy(spins).to(dev)
lp = torch.empty(w.n_samples, dtype=torch.complex128, device=dev)
O = torch.empty(w.n_samples, w.n_params, dtype=torch.complex128, device=dev)
ws = torch.empty(sr._lib.load().sr_jacobian_workspace_bytes(*sr._lib._widths(w.widths), w.n_samples),
                 dtype=torch.uint8, device=dev)
for _ in range(5):
    sr.sr_jacobian(w.widths, theta, sp, lp, O, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    sr.sr_jacobian(w.widths, theta, sp, lp, O, workspace=ws)
e1.record()
torch.cuda.synchronize()
jac_ms = e0.elapsed_time(e1) / 20
ij, jj = (torch.from_numpy(x).to(dev) for x in sr.lattice.for_workload(w))
el = torch.empty(w.n_samples, dtype=torch.complex128, device=dev)
ews = torch.empty(sr._lib.load().sr_local_energy_workspace_bytes(*sr._lib._widths(w.widths), w.n_samples, len(jj)),
                  dtype=torch.uint8, device=dev)
for _ in range(3):
    sr.sr_local_energy(w.widths, theta, ij, jj, sp, lp, el, workspace=ews)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    sr.sr_local_energy(w.widths, theta, ij, jj, sp, lp, el, workspace=ews)
e1.record()
torch.cuda.synchronize()
en_ms = e0.elapsed_time(e1) / 10
gbs = 16.0 * w.n_samples * w.n_params / (jac_ms * 1e-3) / 1e9
print(f"{w.name}: sr_jacobian {jac_ms:.3f} ms ({gbs:.0f} GB/s of O), sr_local_energy {en_ms:.3f} ms  "
      f"|E_loc| {torch.linalg.norm(el).item():.15e}", flush=True)
