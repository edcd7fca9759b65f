"""Run the configs[1] int8 block QGT (sr_block_qgt_i8) a few times and time it with CUDA
events (kernel timer); usable under ncu for a --set full capture of gram_i8<0>.
Usage: python tools/prof_gram.py [config index] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402

w = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
A = torch.randn(w.n_samples, w.n_params, dtype=torch.complex128, device=dev, generator=g) / np.sqrt(w.n_samples)
offs = sr.block_offsets(w.widths)
S = torch.empty(sum((offs[b + 1] - offs[b]) ** 2 for b in range(len(offs) - 1)), dtype=torch.complex128, device=dev)
ws = torch.empty(sr._lib.load().sr_block_qgt_i8_workspace_bytes(w.n_samples, len(offs) - 1, sr._lib._offsets(offs)),
                 dtype=torch.uint8, device=dev)
sr.sr_block_qgt_i8(A, offs, S, workspace=ws)
torch.cuda.synchronize()
sr.sr_kernel_time_ms("gram_i8")
sr.sr_kernel_timer(True)
for _ in range(reps):
    sr.sr_block_qgt_i8(A, offs, S, workspace=ws)
torch.cuda.synchronize()
sr.sr_kernel_timer(False)
ms, n = sr.sr_kernel_time_ms("gram_i8")
ops = sum(2 * (n_b * (n_b + 1) / 2) * (2 * w.n_samples) * 28 * 2 for n_b in w.layer_sizes)
print(f"{w.name}: gram_i8 {ms / reps:.3f} ms per call ({n // reps} launches), {ops / (ms / reps * 1e-3) / 1e12:.0f} int8 TOP/s")
