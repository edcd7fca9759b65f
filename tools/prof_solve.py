"""Run the configs[1] block QGT + block solve twice (for ncu launch lists of the solve)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr, workloads
w = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
A = torch.randn(w.n_samples, w.n_params, dtype=torch.complex128, device=dev, generator=g) / np.sqrt(w.n_samples)
offs = sr.block_offsets(w.widths)
S = torch.empty(sum((offs[b + 1] - offs[b]) ** 2 for b in range(len(offs) - 1)), dtype=torch.complex128, device=dev)
F = torch.randn(w.n_params, dtype=torch.complex128, device=dev, generator=g)
d = torch.empty_like(F)
sr.sr_block_qgt(A, offs, S)
for it in range(2):
    sr.sr_block_solve(offs, S, F, w.lam, d)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sr.sr_block_solve(offs, S, F, w.lam, d); e1.record(); torch.cuda.synchronize()
print("solve ms", e0.elapsed_time(e1), "launches/solve", sr.sr_launch_count() // 4)
