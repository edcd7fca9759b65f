"""Quick check of the int8 tcgen05 Gram (sr_block_qgt_i8) against the FP64 DMMA Gram and
numpy; prints errors and CUDA-event timings.  Usage: python tools/check_ozaki.py [ns n...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_08430_b200 as sr  # noqa: E402

dev = torch.device("cuda:0")


def run(ns, sizes, reps=3):
    offs = [0] + [int(x) for x in np.cumsum(sizes)]
    n_p = offs[-1]
    g = torch.Generator(dev).manual_seed(ns)
    A = (torch.randn(ns, n_p, dtype=torch.float64, device=dev, generator=g)
         + 1j * torch.randn(ns, n_p, dtype=torch.float64, device=dev, generator=g)).contiguous()
    n_s = sum(n * n for n in sizes)
    S8 = torch.full((n_s,), complex(np.nan, np.nan), dtype=torch.complex128, device=dev)
    S64 = torch.empty(n_s, dtype=torch.complex128, device=dev)
    t0 = time.time()
    sr.sr_block_qgt_i8(A, offs, S8)
    torch.cuda.synchronize()
    print(f"ns={ns} sizes={sizes}: first i8 call {time.time() - t0:.3f}s", flush=True)
    sr.sr_block_qgt(A, offs, S64)
    torch.cuda.synchronize()
    nan = torch.isnan(S8.real).sum().item() + torch.isnan(S8.imag).sum().item()
    d = torch.linalg.vector_norm(S8 - S64) / torch.linalg.vector_norm(S64)
    print(f"  nan={nan} rel(i8, fp64)={d.item():.3e}", flush=True)
    if n_p <= 2000:
        An = A.cpu().numpy()
        pos = 0
        for b, n in enumerate(sizes):
            ref = An[:, offs[b]:offs[b + 1]].conj().T @ An[:, offs[b]:offs[b + 1]]
            got = S8[pos:pos + n * n].reshape(n, n).cpu().numpy()
            e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            bad = np.argwhere(np.abs(got - ref) > 1e-8 * np.abs(ref).max())
            print(f"  block {b} n={n}: rel(i8, numpy)={e:.3e} bad={len(bad)} first={bad[:4].tolist()}", flush=True)
            pos += n * n
    ws = torch.empty(sr._lib.load().sr_block_qgt_i8_workspace_bytes(ns, len(sizes), sr._lib._offsets(offs)),
                     dtype=torch.uint8, device=dev)
    for name, fn in (("i8", lambda: sr.sr_block_qgt_i8(A, offs, S8, workspace=ws)),
                     ("fp64", lambda: sr.sr_block_qgt(A, offs, S64))):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        fl = sum(4.0 * ns * n * (n + 1) for n in sizes)
        print(f"  {name}: {ms:.3f} ms  {fl / ms / 1e9:.2f} FP64-equivalent TFLOP/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(int(sys.argv[1]), [int(x) for x in sys.argv[2:]])
    else:
        run(64, [128])
        run(37, [64, 18, 130])
        run(512, [220, 420])
        run(9000, [70, 131])
        run(4096, [3280, 6480, 6480])
