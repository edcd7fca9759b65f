"""Stage-by-stage GPU-vs-oracle diagnostics (prints relative errors; used while developing)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08430_b200 as sr  # noqa: E402
import workloads  # noqa: E402
from oracle import estimators, hamiltonian, network, solvers  # noqa: E402

dev = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def run(w, ns):
    t0 = time.time()
    spins, params = workloads.make_inputs(w, ns)
    ij, jj = sr.lattice.for_workload(w)
    theta = T(sr.model.pack(params))
    sp = T(spins)
    n_p = w.n_params
    lp = torch.empty(ns, dtype=torch.complex128, device=dev)
    O = torch.empty(ns, n_p, dtype=torch.complex128, device=dev)
    sr.sr_jacobian(w.widths, theta, sp, lp, O)
    el = torch.empty(ns, dtype=torch.complex128, device=dev)
    sr.sr_local_energy(w.widths, theta, T(ij), T(jj), sp, lp, el)
    torch.cuda.synchronize()
    O_ref = network.jacobian(params, spins)
    lp_ref = network.log_psi(params, spins)
    el_ref = hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))
    print(f"[{w.name} ns={ns}] log_psi {rel(np.exp(lp.cpu().numpy()), np.exp(lp_ref)):.2e}  "
          f"O {rel(O.cpu().numpy(), O_ref):.2e}  e_loc {rel(el.cpu().numpy(), el_ref):.2e}", flush=True)
    O2 = T(O_ref)
    el2 = T(el_ref)
    energy = torch.empty(1, dtype=torch.complex128, device=dev)
    et = torch.empty(ns, dtype=torch.complex128, device=dev)
    F = torch.empty(n_p, dtype=torch.complex128, device=dev)
    sr.sr_center_force(O2, el2, energy, et, F)
    A_ref, e_ref = estimators.scaled_centered(O_ref, el_ref)
    F_ref = estimators.force(O_ref, el_ref)
    torch.cuda.synchronize()
    print(f"   A {rel(O2.cpu().numpy(), A_ref):.2e}  e~ {rel(et.cpu().numpy(), e_ref):.2e}  "
          f"F {rel(F.cpu().numpy(), F_ref):.2e}  E {abs(energy.item() - estimators.energy(el_ref)):.2e}", flush=True)
    off = network.layer_offsets(params)
    S = torch.empty(sum((off[b + 1] - off[b]) ** 2 for b in range(len(off) - 1)), dtype=torch.complex128, device=dev)
    sr.sr_block_qgt(O2, off, S)
    blocks = estimators.qgt_blocks(O_ref, off)
    Sc = S.cpu().numpy()
    pos = 0
    errs = []
    for b, B in enumerate(blocks):
        n = B.shape[0]
        errs.append(rel(Sc[pos:pos + n * n].reshape(n, n), B))
        pos += n * n
    print("   S_b " + " ".join(f"{e:.2e}" for e in errs), flush=True)
    d = torch.empty(n_p, dtype=torch.complex128, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    sr.sr_block_solve(off, S, F, w.lam, d, info)
    d_ref = solvers.block_solve(blocks, F_ref, off, w.lam)
    torch.cuda.synchronize()
    print(f"   dtheta(block) {rel(d.cpu().numpy(), d_ref):.2e} info {info.item()}", flush=True)
    if n_p <= 20000:
        df = torch.empty(n_p, dtype=torch.complex128, device=dev)
        sr.sr_full_qgt_solve(O2, F, w.lam, df, info=info)
        dn = torch.empty(n_p, dtype=torch.complex128, device=dev)
        sr.sr_ntk_solve(O2, et, w.lam, dn, info=info)
        torch.cuda.synchronize()
        if n_p <= 2000:
            d_full = solvers.full_solve(estimators.qgt_full(O_ref), F_ref, w.lam)
            print(f"   dtheta(full) {rel(df.cpu().numpy(), d_full):.2e}  dtheta(ntk) {rel(dn.cpu().numpy(), d_full):.2e}")
        print(f"   full vs ntk (push-through) {rel(df.cpu().numpy(), dn.cpu().numpy()):.2e}", flush=True)
    print(f"   ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    run(workloads.CONFIGS[0], 512)
    run(workloads.CONFIGS[0], 37)
    run(workloads.CONFIGS[1], 200)
    run(workloads.Workload("wide", "square", (4, 4), 1.0, 0.5, (16, 200, 256), 33), 33)
