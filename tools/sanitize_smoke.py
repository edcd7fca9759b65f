"""Small end-to-end calls of every kernel family (a quick multi-path smoke run): the step (both
Gram engines, both schedules), the comparison solves, the panel kernels, the CG kernels, the
chunked Gram accumulation.  (compute-sanitizer is not available on this pool.)
    python tools/sanitize_smoke.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402
from paper_2510_08430_b200 import parallel  # noqa: E402

dev = torch.device("cuda:0")
w = workloads.CONFIGS[0].with_samples(200)
spins, params = workloads.make_inputs(w)
ij, jj = sr.lattice.for_workload(w)
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
for eng in ("int8", "fp64"):
    for sched in ("batched", "per_block"):
        step = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev, gram_engine=eng, schedule=sched)
        step.run(theta)
b = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev).buf
st = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev)
st.run(theta)
b = st.buf
d = torch.empty_like(b.F)
sr.sr_full_qgt_solve(b.O, b.F, w.lam, d)
sr.sr_ntk_solve(b.O, b.e_tilde, w.lam, d)
parallel.full_qgt_cg(st.ops, parallel.SelfComm(), b.O, b.F, w.lam)
M = torch.eye(130, dtype=torch.complex128, device=dev)
L = torch.empty_like(M)
Li = torch.empty_like(M)
sr.sr_chol_inv(M, 0.1, L, Li)
C = torch.zeros(70, 90, dtype=torch.complex128, device=dev)
sr.sr_gram_tn(b.O[:, :70], b.O[:, :90], C)
sr.sr_gram_nh_sub(b.O[:70, :50].contiguous(), b.O[:90, :50].contiguous(), C)
ch = parallel.ChunkedStep(w.widths, spins, ij, jj, w.lam, dev, chunk=64)
ch.run(theta)
torch.cuda.synchronize()
print("sanitize smoke: ok")
