"""Device-side trace (sr_trace_buffer) of one CUDA-graph replay of the bench step: per-launch
begin/end from globaltimer, per-kind busy time, and the Cholesky panel chain of each block
(chol_diag to chol_diag intervals and what fills them).
Usage: python tools/graph_trace.py [config index] [out.txt]"""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
from paper_2510_08430_b200 import parallel  # noqa: E402
import workloads  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "1"
out = sys.argv[2] if len(sys.argv) > 2 else None
dev = torch.device("cuda:0")
if arg.startswith("solve"):   # solve-only graph of one block of the given size, e.g. solve6480
    import numpy as np

    class _SolveOnly:
        def __init__(self, n):
            g = torch.Generator(device=dev).manual_seed(0)
            A = torch.randn(4096, n, dtype=torch.complex128, device=dev, generator=g) / 64.0
            self.S = torch.empty(n * n, dtype=torch.complex128, device=dev)
            sr.sr_block_qgt_i8(A, [0, n], self.S)
            self.F = torch.randn(n, dtype=torch.complex128, device=dev, generator=g)
            self.d = torch.empty_like(self.F)
            self.n = n

        def run(self):
            sr.sr_block_solve([0, self.n], self.S, self.F, 1e-3, self.d)

        def capture(self, _theta):
            self.run()
            torch.cuda.synchronize()
            if os.environ.get("SR_LIB_GRAPH", "1") != "0":   # library-instantiated: node priorities kept
                self.graph = sr.Graph(dev)
                with self.graph.capture():
                    self.run()
            else:
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph):
                    self.run()

        def replay(self):
            self.graph.replay()

    w = workloads.CONFIGS[1]
    step = _SolveOnly(int(arg[5:]))
    theta = None
else:
    w = workloads.CONFIGS[int(arg)]
    spins, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    step = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev)
    theta = torch.from_numpy(sr.model.pack(params)).to(dev)
step.capture(theta)
for _ in range(3):
    step.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    step.replay()
e1.record()
torch.cuda.synchronize()
print(f"{w.name}: graph step {e0.elapsed_time(e1) / 10:.3f} ms (untraced, mean of 10 replays)")
buf = torch.zeros(40 * 4_000_000, dtype=torch.uint8, device=dev)
sr.sr_trace_buffer(buf)
step.replay()
torch.cuda.synchronize()
sr.sr_trace_buffer(None)
recs = sr.sr_trace_records(buf)
grids = {}
for g, kind, tag, sm, t0, t1 in recs:
    r = grids.setdefault(g, [kind, tag, t0, t1, 0])
    r[2], r[3], r[4] = min(r[2], t0), max(r[3], t1), r[4] + 1
t_origin = min(r[2] for r in grids.values())
L = sorted(((r[2] - t_origin) / 1e3, (r[3] - t_origin) / 1e3, r[0], r[1], r[4]) for r in grids.values())
print(f"traced launches {len(L)}, span {max(b for _, b, *_ in L) - L[0][0]:.1f} us")
if out:
    with open(out, "w") as f:
        for a, b, k, tag, n in L:
            f.write(f"{a:10.2f} {b:10.2f} {k:12s} {tag:8d} {n:5d}\n")
busy, cnt = collections.Counter(), collections.Counter()
for a, b, k, tag, n in L:
    busy[k] += b - a
    cnt[k] += 1
print("per kind (sum of launch spans, us):", ", ".join(f"{k} {v:.0f} ({cnt[k]})" for k, v in busy.most_common()))
diags = collections.defaultdict(list)
for a, b, k, tag, n in L:
    if k == "diag":
        diags[tag // 4096].append((a, b, tag % 4096))
for blk, ds in sorted(diags.items()):
    ds.sort()
    dur = sum(b - a for a, b, _ in ds)
    gaps = [ds[i + 1][0] - ds[i][1] for i in range(len(ds) - 1)]
    print(f"block npad/64={blk}: {len(ds)} diags {ds[0][0]:.0f}..{ds[-1][1]:.0f} us, diag time {dur:.0f} us "
          f"(mean {dur / len(ds):.1f}), between diags {sum(gaps):.0f} us (mean {sum(gaps) / max(1, len(gaps)):.1f}, "
          f"max {max(gaps) if gaps else 0:.0f})")
    # what runs between diag p and diag p+1 of this block (kernels starting in the gap)
    if blk == max(diags):
        for i in range(min(len(ds) - 1, 18)):
            a0, b0 = ds[i][1], ds[i + 1][0]
            inside = [(a, b, k, tag) for a, b, k, tag, n in L if a >= ds[i][0] and a < b0 and k != "diag"]
            desc = " ".join(f"{k}[{tag}]@{a - a0:.0f}+{b - a:.0f}" for a, b, k, tag in inside[:8])
            print(f"  p={ds[i][2]:3d} diag {ds[i][1] - ds[i][0]:5.1f} gap {b0 - a0:6.1f} | {desc}")

# SM occupancy over the solve window: per SM, the union of its CTA intervals
t_a = min(t0 for g, k, tag, sm, t0, t1 in recs if k == "diag")
t_b = max(t1 for g, k, tag, sm, t0, t1 in recs if k in ("back", "back_rest", "output"))
per_sm = collections.defaultdict(list)
for g, k, tag, sm, t0, t1 in recs:
    if t1 > t_a and t0 < t_b:
        per_sm[sm].append((max(t0, t_a), min(t1, t_b), k))
busy_all, by_kind = [], collections.Counter()
for sm, iv in per_sm.items():
    iv.sort()
    busy, cur_a, cur_b = 0, None, None
    for a, b, k in iv:
        by_kind[k] += b - a
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                busy += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    if cur_b is not None:
        busy += cur_b - cur_a
    busy_all.append(busy / (t_b - t_a))
n_sm = 148
print(f"solve window {(t_b - t_a) / 1e3:.0f} us: SMs with work {len(busy_all)}, mean busy fraction "
      f"{sum(busy_all) / n_sm:.2f} (union of CTA lifetimes per SM); CTA-time by kind (SM-us): "
      + ", ".join(f"{k} {v / 1e3:.0f}" for k, v in by_kind.most_common()))
