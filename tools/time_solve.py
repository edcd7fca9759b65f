"""Time sr_block_solve (CUDA events) for block partitions with each engine.
Usage: python tools/time_solve.py [n1 n2 ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_08430_b200 as sr  # noqa: E402

dev = torch.device("cuda:0")


def run(sizes, reps=3):
    offs = [0] + [int(x) for x in np.cumsum(sizes)]
    n_p = offs[-1]
    ns = 4096
    g = torch.Generator(dev).manual_seed(1)
    A = (torch.randn(ns, n_p, dtype=torch.float64, device=dev, generator=g)
         + 1j * torch.randn(ns, n_p, dtype=torch.float64, device=dev, generator=g)).contiguous() / ns ** 0.5
    S = torch.empty(sum(n * n for n in sizes), dtype=torch.complex128, device=dev)
    sr.sr_block_qgt(A, offs, S)
    F = (A.conj().T @ torch.randn(ns, dtype=torch.complex128, device=dev, generator=g)).contiguous()
    out = {}
    for eng in ("fp64", "int8"):
        sr.sr_set_gram_engine(sr.GRAM_INT8 if eng == "int8" else sr.GRAM_FP64)
        d = torch.empty(n_p, dtype=torch.complex128, device=dev)
        ws = torch.empty(sr._lib.load().sr_block_solve_workspace_bytes(len(sizes), sr._lib._offsets(offs)),
                         dtype=torch.uint8, device=dev)
        sr.sr_block_solve(offs, S, F, 1e-3, d, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            sr.sr_block_solve(offs, S, F, 1e-3, d, workspace=ws)
        graph.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1) / 10
        plain = []
        for _ in range(5):   # without the kernel timer's events
            e0.record()
            sr.sr_block_solve(offs, S, F, 1e-3, d, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            plain.append(e0.elapsed_time(e1))
        names = ("trail_i8", "trail_dmma", "chol_diag", "chol_trsm", "chol_rhs", "chol_inner", "chol_back", "chol_back_rest")
        for k in names:
            sr.sr_kernel_time_ms(k)
        sr.sr_kernel_timer(True)
        e0.record()
        for _ in range(reps):
            sr.sr_block_solve(offs, S, F, 1e-3, d, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        sr.sr_kernel_timer(False)
        ms = e0.elapsed_time(e1) / reps
        parts = []
        for k in names:
            tk, nk = sr.sr_kernel_time_ms(k)
            if nk:
                parts.append(f"{k} {tk / reps:.2f} ms/{nk // reps} ({1e3 * tk / nk:.1f} us each)")
        out[eng] = d.clone()
        fl = sum(4.0 * n ** 3 / 3 for n in sizes)
        print(f"sizes={sizes} {eng}: {ms:.2f} ms/solve with timer, untimed min/median "
              f"{min(plain):.2f}/{sorted(plain)[2]:.2f} ms, graph {gms:.2f} ms ({fl / ms / 1e9:.1f} TFLOP/s ZPOTRF-equivalent)"
              + "\n    " + "; ".join(parts), flush=True)
    r = torch.linalg.vector_norm(out["int8"] - out["fp64"]) / torch.linalg.vector_norm(out["fp64"])
    res = []
    pos = 0
    for b, n in enumerate(sizes):
        Sb = S[pos:pos + n * n].reshape(n, n)
        x = out["int8"][offs[b]:offs[b + 1]]
        rr = Sb @ x + 1e-3 * x + F[offs[b]:offs[b + 1]]
        res.append((torch.linalg.vector_norm(rr) / torch.linalg.vector_norm(F[offs[b]:offs[b + 1]])).item())
        pos += n * n
    print(f"  rel(int8, fp64) = {r.item():.2e}; int8 residuals {['%.1e' % x for x in res]}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run([int(x) for x in sys.argv[1:]])
    else:
        run([6480], reps=1)
        run([3280, 6480, 6480], reps=1)
