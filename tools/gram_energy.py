"""Sustained (power-capped) rate of the block-QGT Gram at a configs[3] block shape, for the
library or a measurement variant of it (SR_LIB_VARIANT=<path to .so>, built by
`python tools/gram_energy.py build EXP...` with -DSR_OZ_EXP=<n>).  Replays the Gram of one
16512-column block over 32768 samples (K' = 65536) for ~8 s while sampling SM clock and board
power; prints ms per call, TOPS at the Ozaki-I op count, clock and power, and pJ per int8 op.

    python tools/gram_energy.py build 4 5 6      # variants/libsrblock_exp<n>.so
    python tools/gram_energy.py run [n ns reps]  # the library named by SR_LIB_VARIANT (or the default)
"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "build":
    from paper_2510_08430_b200 import build
    os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
    for e in sys.argv[2:]:
        print(build.build(defines=[f"SR_OZ_EXP={e}"], out=os.path.join(ROOT, "variants", f"libsrblock_exp{e}.so")))
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_08430_b200 as sr  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 16512
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 15
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
A = torch.complex(torch.randn(ns, n, dtype=torch.float64, device=dev, generator=g),
                  torch.randn(ns, n, dtype=torch.float64, device=dev, generator=g))
S = torch.empty(n * n, dtype=torch.complex128, device=dev)
ws = torch.empty(sr.load().sr_block_qgt_i8_workspace_bytes(ns, 1, sr._lib._offsets([0, n])), dtype=torch.uint8,
                 device=dev)
sr.sr_block_qgt_i8(A, [0, n], S, workspace=ws)
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms",
                        "100"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    sr.sr_block_qgt_i8(A, [0, n], S, workspace=ws)
e1.record()
torch.cuda.synchronize()
smi.terminate()
rows = [tuple(float(x) for x in l.split(",")) for l in smi.stdout.read().strip().splitlines() if l.strip()]
rows = rows[len(rows) // 4: -2] or rows
clk = float(np.median([r[0] for r in rows]))
pw = float(np.median([r[1] for r in rows]))
ms = e0.elapsed_time(e1) / reps
ops = 2 * (n * (n + 1) / 2) * (2 * ns) * 28 * 2
print(f"variant={os.environ.get('SR_LIB_VARIANT', 'default')} n={n} ns={ns}: {ms:.2f} ms/call, "
      f"{ops / ms / 1e9:.0f} TOPS (Ozaki-I op count), SM {clk:.0f} MHz, {pw:.0f} W, "
      f"{pw / (ops / ms * 1e3) * 1e12:.3f} pJ/op", flush=True)
