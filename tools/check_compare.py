import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2510_08430_b200 as sr
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
ns, n_p = 1000, 700
A = torch.randn(ns, n_p, dtype=torch.complex128, device=dev, generator=g) / ns ** 0.5
F = torch.randn(n_p, dtype=torch.complex128, device=dev, generator=g)
e = torch.randn(ns, dtype=torch.complex128, device=dev, generator=g)
F = (A.conj().T @ e).contiguous()
out = {}
for eng in ("fp64", "int8"):
    sr.sr_set_gram_engine(sr.GRAM_INT8 if eng == "int8" else sr.GRAM_FP64)
    d1 = torch.empty(n_p, dtype=torch.complex128, device=dev); d2 = torch.empty_like(d1)
    S = torch.empty(n_p * n_p, dtype=torch.complex128, device=dev); T = torch.empty(ns * ns, dtype=torch.complex128, device=dev)
    sr.sr_full_qgt_solve(A, F, 1e-3, d1, S_out=S)
    sr.sr_ntk_solve(A, e, 1e-3, d2, T_out=T)
    torch.cuda.synchronize()
    out[eng] = (d1.clone(), d2.clone(), S.clone(), T.clone())
    print(eng, "full vs ntk", (torch.linalg.norm(d1 - d2) / torch.linalg.norm(d1)).item())
for i, nm in enumerate(("d_full", "d_ntk", "S", "T")):
    a, b = out["fp64"][i], out["int8"][i]
    print(nm, "int8 vs fp64", (torch.linalg.norm(a - b) / torch.linalg.norm(a)).item(), "bitwise equal", torch.equal(a, b))
Sref = (A.conj().T @ A).reshape(-1); Tref = (A @ A.conj().T).reshape(-1)
print("S vs torch", (torch.linalg.norm(out["int8"][2] - Sref) / torch.linalg.norm(Sref)).item(), "T vs torch", (torch.linalg.norm(out["int8"][3] - Tref) / torch.linalg.norm(Tref)).item())
