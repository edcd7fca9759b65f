"""Single-block (and batched) shifted solves timed as CUDA-graph replays: the owner's solve of
the sharded step.   python tools/solve_graph_time.py [n ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_08430_b200 as sr  # noqa: E402

dev = torch.device("cuda:0")
sizes_list = [[int(x) for x in a.split(",")] for a in sys.argv[1:]] or [[6480], [16512], [3280, 6480, 6480]]
for sizes in sizes_list:
    n_p = sum(sizes)
    offs = [0]
    for n in sizes:
        offs.append(offs[-1] + n)
    g = torch.Generator(device=dev).manual_seed(0)
    ns = 4096
    S = torch.empty(sum(n * n for n in sizes), dtype=torch.complex128, device=dev)
    A = torch.complex(torch.randn(ns, n_p, dtype=torch.float64, device=dev, generator=g),
                      torch.randn(ns, n_p, dtype=torch.float64, device=dev, generator=g)) / ns ** 0.5
    sr.sr_block_qgt_i8(A, offs, S)
    del A
    F = torch.randn(n_p, dtype=torch.complex128, device=dev, generator=g)
    d = torch.empty_like(F)
    ws = torch.empty(sr.load().sr_block_solve_workspace_bytes(len(sizes), sr._lib._offsets(offs)), dtype=torch.uint8,
                     device=dev)
    sr.sr_block_solve(offs, S, F, 1e-3, d, workspace=ws)
    torch.cuda.synchronize()
    graph = sr.Graph(dev)
    with graph.capture():
        sr.sr_block_solve(offs, S, F, 1e-3, d, workspace=ws)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"sizes {sizes}: {e0.elapsed_time(e1) / reps:.3f} ms per solve (graph replay)", flush=True)
