"""Replay the configs[1] block-solve graph (or the Gram) for a few seconds while sampling SM
clock and power with nvidia-smi: is the stage power-capped?  Usage: python tools/solve_clock.py [solve|gram]"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "solve"
w = workloads.CONFIGS[1]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
A = torch.randn(w.n_samples, w.n_params, dtype=torch.complex128, device=dev, generator=g) / np.sqrt(w.n_samples)
offs = sr.block_offsets(w.widths)
S = torch.empty(sum((offs[b + 1] - offs[b]) ** 2 for b in range(len(offs) - 1)), dtype=torch.complex128, device=dev)
F = torch.randn(w.n_params, dtype=torch.complex128, device=dev, generator=g)
d = torch.empty_like(F)
qws = torch.empty(sr._lib.load().sr_block_qgt_i8_workspace_bytes(w.n_samples, len(offs) - 1, sr._lib._offsets(offs)),
                  dtype=torch.uint8, device=dev)
sws = torch.empty(sr._lib.load().sr_block_solve_workspace_bytes(len(offs) - 1, sr._lib._offsets(offs)),
                  dtype=torch.uint8, device=dev)
sr.sr_block_qgt_i8(A, offs, S, workspace=qws)


def run():
    if what == "gram":
        sr.sr_block_qgt_i8(A, offs, S, workspace=qws)
    else:
        sr.sr_block_solve(offs, S, F, w.lam, d, workspace=sws)


run()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    run()
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "50"],
                       stdout=subprocess.PIPE, text=True)
time.sleep(0.5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 150
e0.record()
for _ in range(n):
    graph.replay()
e1.record()
torch.cuda.synchronize()
smi.terminate()
rows = [tuple(float(x) for x in l.split(",")) for l in smi.stdout.read().strip().splitlines() if l.strip()]
rows = rows[len(rows) // 4: -2] or rows
clk = sorted(r[0] for r in rows)
pw = sorted(r[1] for r in rows)
print(f"{what}: {e0.elapsed_time(e1) / n:.3f} ms per replay; SM clock median {clk[len(clk) // 2]:.0f} MHz "
      f"(min {clk[0]:.0f}, max {clk[-1]:.0f}); power median {pw[len(pw) // 2]:.0f} W (max {pw[-1]:.0f}); {len(rows)} samples")
