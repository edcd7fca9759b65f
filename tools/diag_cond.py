"""Diagnose centring conditioning on a full-size config: per-column |<O>|/std(O) and
GPU-vs-oracle errors of O, A and sampled S entries."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr, workloads
from oracle import estimators, network
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = workloads.CONFIGS[cfg]
spins, params = workloads.make_inputs(w)
dev = torch.device("cuda:0")
theta = torch.from_numpy(sr.model.pack(params)).to(dev)
ns = w.n_samples
lp = torch.empty(ns, dtype=torch.complex128, device=dev)
O = torch.empty(ns, w.n_params, dtype=torch.complex128, device=dev)
sr.sr_jacobian(w.widths, theta, torch.from_numpy(spins).to(dev), lp, O)
offs = sr.block_offsets(w.widths)
rng = np.random.default_rng(0)
cols = np.sort(np.concatenate([rng.choice(np.arange(offs[i], offs[i+1]), 6, replace=False) for i in range(len(offs)-1)]))
O_ref = np.stack([network.log_derivative_row(params, x)[cols] for x in spins])
O_gpu = O[:, torch.as_tensor(cols, device=dev)].cpu().numpy()
cond = np.abs(O_ref.mean(0)) / O_ref.std(0)
print("cond |<O>|/std per sampled col:", np.array2string(cond, precision=1))
print("O colwise rel err:", np.array2string(np.linalg.norm(O_gpu - O_ref, axis=0) / np.linalg.norm(O_ref, axis=0), precision=1))
e = torch.zeros(ns, dtype=torch.complex128, device=dev)
en = torch.empty(1, dtype=torch.complex128, device=dev); et = torch.empty(ns, dtype=torch.complex128, device=dev)
F = torch.empty(w.n_params, dtype=torch.complex128, device=dev)
sr.sr_center_force(O, e, en, et, F)
A_gpu = O[:, torch.as_tensor(cols, device=dev)].cpu().numpy()
A_ref, _ = estimators.scaled_centered(O_ref, np.zeros(ns))
A_gpu_ownO, _ = estimators.scaled_centered(O_gpu, np.zeros(ns))
print("A colwise rel err vs oracle:", np.array2string(np.linalg.norm(A_gpu - A_ref, axis=0) / np.linalg.norm(A_ref, axis=0), precision=1))
print("A colwise err / (|O|/sqrt N):", np.array2string(np.linalg.norm(A_gpu - A_ref, axis=0) / (np.linalg.norm(O_ref, axis=0) / np.sqrt(ns)), precision=1))
print("A(gpu) vs oracle-centring of GPU's own O:", np.array2string(np.linalg.norm(A_gpu - A_gpu_ownO, axis=0) / np.linalg.norm(A_gpu_ownO, axis=0), precision=1))
for i in range(len(offs)-1):
    sel = [c for c in range(len(cols)) if offs[i] <= cols[c] < offs[i+1]]
    Sr = estimators.qgt_full(O_ref[:, sel]); Sg = A_gpu[:, sel].conj().T @ A_gpu[:, sel]
    print(f"block {i}: sampled S rel err {np.linalg.norm(Sg-Sr)/np.linalg.norm(Sr):.2e}")
