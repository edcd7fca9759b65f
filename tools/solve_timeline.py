"""Timeline of one eager sr_block_solve at a configuration (kernel-timer events on every
launching stream): per stream, the time each named kernel occupies and the idle gaps.
Usage: python tools/solve_timeline.py [config index] [out.txt]"""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402

w = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
out = sys.argv[2] if len(sys.argv) > 2 else None
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
A = torch.randn(w.n_samples, w.n_params, dtype=torch.complex128, device=dev, generator=g) / np.sqrt(w.n_samples)
offs = sr.block_offsets(w.widths)
S = torch.empty(sum((offs[b + 1] - offs[b]) ** 2 for b in range(len(offs) - 1)), dtype=torch.complex128, device=dev)
F = torch.randn(w.n_params, dtype=torch.complex128, device=dev, generator=g)
d = torch.empty_like(F)
sr.sr_block_qgt_i8(A, offs, S)
del A
for _ in range(2):
    sr.sr_block_solve(offs, S, F, w.lam, d)
torch.cuda.synchronize()
sr.sr_kernel_timeline()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sr.sr_block_solve(offs, S, F, w.lam, d)
e1.record()
torch.cuda.synchronize()
print(f"{w.name}: eager block solve {e0.elapsed_time(e1):.3f} ms (untimed)")
sr.sr_kernel_timer(True)
sr.sr_block_solve(offs, S, F, w.lam, d)
torch.cuda.synchronize()
sr.sr_kernel_timer(False)
tl = sr.sr_kernel_timeline()
if out:
    with open(out, "w") as f:
        for r in tl:
            f.write("%s %d %.4f %.4f\n" % r)
end = max(b for _, _, _, b in tl)
print(f"timed solve span {end:.3f} ms, {len(tl)} records")
by_stream = collections.defaultdict(list)
for name, sid, a, b in tl:
    by_stream[sid].append((a, b, name))
for sid in sorted(by_stream):
    recs = sorted(by_stream[sid])
    busy = collections.Counter()
    cnt = collections.Counter()
    gaps, last = 0.0, recs[0][0]
    for a, b, name in recs:
        busy[name] += b - a
        cnt[name] += 1
        gaps += max(0.0, a - last)
        last = max(last, b)
    parts = ", ".join(f"{k} {v:.2f} ({cnt[k]})" for k, v in busy.most_common())
    print(f"stream {sid}: {recs[0][0]:.2f}..{last:.2f} ms, gaps {gaps:.2f} ms | {parts}")
