"""Launch the Jacobian stage of configs[1] a few times (for an ncu launch list)."""
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
print(f"sr_jacobian {w.name}: {e0.elapsed_time(e1) / 20:.3f} ms")
