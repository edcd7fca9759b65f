"""The distributed dense full-QGT solve (parallel.dist_full_qgt) as one rank on one GPU at a
bench workload: S (n_p^2 / 2 complex) formed from the step's centred Jacobian and factorised
panel by panel; timed with CUDA events, compared with the block update and the matrix-free
CG update.   python tools/dist_full_qgt.py [workload] [nb]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_08430_b200 as sr  # noqa: E402
from paper_2510_08430_b200 import parallel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_WORKLOAD
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
eng = sys.argv[3] if len(sys.argv) > 3 else "int8"
w = bench.workload_for(name, 1)
spins, params = bench.workloads.make_inputs(w)
ij, jj = sr.lattice.for_workload(w)
dev = torch.device("cuda:0")
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
step = parallel.LocalStep(w.widths, spins, ij, jj, w.lam, dev)
step.run(theta)
b = step.buf
d_block = b.dtheta.clone()
b.S = None
step.ops.ws = None
torch.cuda.empty_cache()
x_cg, it, res = parallel.full_qgt_cg(step.ops, parallel.SelfComm(), b.O, b.F, w.lam)


class _One(parallel.SelfComm):
    def reduce(self, t, dst, async_op=False):
        return parallel._Done()

    def broadcast(self, t, src):
        pass

    def all_gather(self, out, t):
        out[0].copy_(t)


torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
x = parallel.dist_full_qgt(step.ops, _One(), 0, 1, b.O, b.F, w.lam, nb=nb, engine=eng)
e1.record()
torch.cuda.synchronize()
nrm = lambda v: float(torch.linalg.vector_norm(v).item())  # noqa: E731
n = w.n_params
print(json.dumps({"workload": name, "n_p": n, "n_samples": w.n_samples, "panel_rows": nb, "engine": eng,
                  "ms": e0.elapsed_time(e1), "wall_s": time.perf_counter() - t0,
                  "form_flops": 8.0 * w.n_samples * n * (n + 1) / 2, "chol_flops": 4.0 * n ** 3 / 3,
                  "rel_l2_dense_vs_cg": nrm(x - x_cg) / nrm(x_cg), "rel_l2_block_vs_dense": nrm(d_block - x) / nrm(x),
                  "cg_iterations": it, "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
