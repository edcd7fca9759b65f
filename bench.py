"""Block-SR step benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

A step is one pass of the whole hot path over one batch of synthetic input
(DESIGN.md §8(a)): Jacobian -> local energy -> centring + force -> block QGT (Gram) ->
block solve, each stage one C-ABI call of libsrblock.so.  Default workload: BASELINE.json
configs[1] (1D Heisenberg ring N=40, MLP 40->80->80->80, N_s=4096, lambda=1e-3).

`value` times the device-resident step with CUDA events on the launching stream
(barrier + synchronize on both sides, max over ranks); `e2e` times sr_step_host (host
inputs copied in, dtheta/energy copied out, every step).  `--impl reference` times the
CPU oracle (the reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "block-SR steps/sec (Jacobian->Gram->solve), Gram FP64 TFLOPS vs B200 peak"
DEFAULT_WORKLOAD = workloads.CONFIGS[1].name
FP64_PEAK_TFLOPS = 37.07        # profiles/r01_fp64_peak.json: DMMA.8x8x4 microbenchmark (tools/fp64_peak.cu)
FP64_PEAK_SOURCE = "measured: tools/fp64_peak.cu DMMA microbenchmark on this pool's B200 (profiles/r01_fp64_peak.json)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_source": "fallback (B200_PROFILING.md)"}


def block_sizes(w):
    return w.layer_sizes


INT8_SLICES = 7                 # digit slices of sr_block_qgt_i8 (include/sr_block.h)
INT8_PAIRS = INT8_SLICES * (INT8_SLICES + 1) // 2
INT8_OVER_BF16 = 4.5 / 2.25     # nominal dense int8 : bf16 tensor rate (B200_PROFILING.md table)


def gram_i8_ops(w, ns):
    """Algorithmic int8 tensor ops of the digit-slice Gram: for each unique Hermitian entry
    (i >= j) the real Re and Im dot products over K' = 2 N_s, INT8_PAIRS slice products
    each, 2 ops per multiply-add."""
    return sum(2 * (n * (n + 1) / 2) * (2 * ns) * INT8_PAIRS * 2 for n in block_sizes(w))


def gram_flops(w, ns):
    """Algorithmic FP64 flops of the block QGT: n_b(n_b+1)/2 unique complex entries of each
    Hermitian S_b, N_s complex multiply-adds (8 real flops) each."""
    return sum(8.0 * ns * n * (n + 1) / 2 for n in block_sizes(w))


def energy_flops(w, spins, ij):
    """Algorithmic flops of the local-energy stage: one network evaluation per connected
    configuration (a bond with anti-parallel spins), the first layer updated by the two
    flipped spins (2 w_1 complex MACs), every later layer dense (w_l w_{l+1} complex MACs),
    8 real flops per complex MAC.  The lncosh evaluations are not counted."""
    flips = int(np.sum(spins[:, ij[:, 0]] != spins[:, ij[:, 1]]))
    macs = 2 * w.widths[1] + sum(w.widths[l] * w.widths[l + 1] for l in range(1, len(w.widths) - 1))
    return 8.0 * flips * macs


def chol_flops(w):
    """Algorithmic flops of the Cholesky factorisations: n^3/6 complex multiply-adds
    (8 real flops each) per block, i.e. 4 n^3 / 3 (LAPACK's ZPOTRF count)."""
    return sum(4.0 * n ** 3 / 3 for n in block_sizes(w))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "power_w": float(np.median(pw)) if pw else None, "samples": len(rows)}


# ----------------------------------------------------------------------------- dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), ws, int(os.environ.get("LOCAL_RANK", "0"))


def config_of(w, world, engine, sharded):
    """The workload description shared by both arms' JSON lines."""
    return {"workload": w.name, "lattice": f"{w.lattice}{'x'.join(map(str, w.extent))}",
            "widths": list(w.widths), "n_samples": w.n_samples, "n_params": w.n_params, "blocks": block_sizes(w),
            "lambda": w.lam, "gram_engine": engine,
            "parallelism": f"samples sharded x{world} (NCCL)" if sharded else "single GPU",
            "l2": f"inputs larger than L2 (O = {16.0 * w.n_samples * w.n_params / 1e9:.2f} GB per step vs 126 MB L2); "
                  "no flush"}


def _quiet_fd1(fn):
    """Run fn() with the process-level stdout (fd 1) sent to /dev/null."""
    sys.stdout.flush()
    saved, devnull = os.dup(1), os.open(os.devnull, os.O_WRONLY)
    os.dup2(devnull, 1)
    try:
        return fn()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
        os.close(devnull)


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2510_08430_b200 as sr
    from paper_2510_08430_b200 import parallel

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if sharded:
        # keep stdout to the one JSON line: the NCCL communicator set-up prints a version banner
        # on fd 1, so it runs with fd 1 pointed at /dev/null
        def _init():
            if "RANK" not in os.environ:   # --sharded without torchrun: a one-rank group
                import socket
                with socket.socket() as so:
                    so.bind(("127.0.0.1", 0))
                    port = so.getsockname()[1]
                os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()
        _quiet_fd1(_init)
    w = workloads.BY_NAME[args.workload]
    spins_all, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    theta_h = sr.model.pack(params)
    n_p, ns = w.n_params, w.n_samples
    offs = sr.block_offsets(w.widths)

    engine = args.gram_engine
    sr.sr_set_gram_engine(sr.GRAM_INT8 if engine == "int8" else sr.GRAM_FP64)   # for sr_step_host (e2e)
    if sharded:
        step = parallel.ShardedStep(w.widths, spins_all, ij, jj, w.lam, rank, world, dev, gram_engine=engine)
    else:
        step = parallel.LocalStep(w.widths, spins_all, ij, jj, w.lam, dev, gram_engine=engine)
    theta = torch.from_numpy(theta_h).to(dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        step.run(theta)
    torch.cuda.synchronize(dev)

    # per-stage breakdown: eager launches with CUDA events between the C-ABI stage calls
    n_ev = len(step.STAGES) + 1
    n_stage_runs = max(1, min(args.steps, 3))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(n_stage_runs)]
    gram_kernel = "gram_i8" if engine == "int8" else "gram_tn"
    sr.sr_kernel_time_ms(gram_kernel)
    sr.sr_kernel_timer(True)                 # CUDA events around the Gram kernel's launches
    sr.sr_reset_launch_count()
    for k in range(n_stage_runs):
        step.run(theta, events=evs[k])
    torch.cuda.synchronize(dev)
    sr.sr_kernel_timer(False)
    launches = sr.sr_launch_count() // n_stage_runs
    gk_ms, gk_n = sr.sr_kernel_time_ms(gram_kernel)
    gram_kernel_ms = gk_ms / n_stage_runs        # all launches of one stage-(4) call (block groups)
    gram_launches = gk_n // n_stage_runs
    stage_ms = {name: float(np.mean([evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(n_stage_runs)]))
                for i, name in enumerate(step.STAGES)}

    # One GPU (also --sharded as a 1-rank NCCL group): the step is replayed as one CUDA graph.
    # More than one rank: eager launches unless SR_BENCH_GRAPH_SHARDED=1 -- graph capture of
    # the NCCL collectives is tested here only on a 1-rank group, and a capture failing on
    # some ranks could leave the others waiting inside a collective.
    use_graph = not args.no_graph and (world == 1 or os.environ.get("SR_BENCH_GRAPH_SHARDED") == "1")
    if use_graph:
        try:
            step.capture(theta)              # the whole step (collectives included) as one CUDA graph
        except Exception as exc:             # capture unsupported here: time the eager step instead
            print(f"bench: CUDA-graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            use_graph = False
            torch.cuda.synchronize(dev)
    if use_graph:
        for _ in range(args.warmup):
            step.replay()
    torch.cuda.synchronize(dev)
    if sharded:
        dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize(dev)
    if sharded:
        dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        if use_graph:
            step.replay()
        else:
            step.run(theta)
    stop.record(stream)
    torch.cuda.synchronize(dev)
    if sharded:
        dist.barrier()
    clk = clocks.stop()
    total_ms = start.elapsed_time(stop)
    if sharded:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # e2e: the same step through sr_step_host (host buffers in and out, every step)
    if sharded:
        e2e = run_e2e_sharded(torch, dist, step, theta_h, dev, args, theta if use_graph else None)
    else:
        comparison = None if args.no_compare else compare_solves(sr, torch, step, w, dev)
        del step                      # the e2e run allocates its own sr_step workspace
        torch.cuda.empty_cache()
        e2e = run_e2e(sr, torch, w, theta_h, spins_all, ij, jj, dev, args)

    if rank != 0:
        if sharded:
            dist.destroy_process_group()
        return
    ms_per_step = total_ms / args.steps
    peaks = _peaks()
    gram_ms = stage_ms["block_qgt"]
    gflop = gram_flops(w, ns / world)
    achieved = gflop / (gram_ms * 1e-3) / 1e12
    fp64_eq = gflop / (gram_kernel_ms * 1e-3) / 1e12
    if engine == "int8":
        ops = gram_i8_ops(w, ns / world)
        # The kernel is timed alone (its own CUDA-event pair) and runs near the maximum SM clock
        # (see "clocks"), so the burst figure applies; the sustained one is reported beside it.
        peak = peaks["bf16_tflops"] * INT8_OVER_BF16
        peak_sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * INT8_OVER_BF16
        ach = ops / (gram_kernel_ms * 1e-3) / 1e12
        roofline = {
            "kernel": "sr::oz::gram_i8 (sr_block_qgt_i8: tcgen05.mma kind::i8, TMA, TMEM)", "bound": "tensor",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s", "op_dtype": "int8 (one multiply-add = 2 ops)",
            "frac": ach / peak, "traffic": _ncu_traffic("gram_i8_traffic.json"),
            "kernel_ms": gram_kernel_ms, "kernel_launches": gram_launches,
            "algorithmic": (f"sum_b 2 (Re, Im) x n_b(n_b+1)/2 entries x K'=2 N_s x {INT8_PAIRS} slice pairs x 2 "
                            f"= {ops:.4e} int8 ops per launch"),
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops (burst) x 2, the nominal dense int8 : bf16 "
                            "ratio (4.5 : 2.25 PFLOP/s, B200_PROFILING.md)"),
            "frac_of_sustained": ach / peak_sus, "sustained_peak": peak_sus,
            "frac_of_tcgen05_microbenchmark": ach / 4763.0,
            "fp64_equivalent": {"achieved_tflops": fp64_eq, "fp64_dmma_peak": FP64_PEAK_TFLOPS,
                                "ratio_to_fp64_peak": fp64_eq / FP64_PEAK_TFLOPS,
                                "algorithmic": f"sum_b 4 N_s n_b (n_b+1) = {gflop:.4e} flop"},
        }
    else:
        roofline = {"kernel": "gram::tile_kernel<TN,HERM_STORE> (sr_block_qgt)", "bound": "tensor",
                    "achieved": fp64_eq, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": fp64_eq / FP64_PEAK_TFLOPS, "traffic": _ncu_traffic("gram_traffic.json"),
                    "kernel_ms": gram_kernel_ms,
                    "algorithmic": f"sum_b 4 N_s n_b (n_b+1) = {gflop:.4e} flop per launch",
                    "peak_source": FP64_PEAK_SOURCE}
    O_bytes = 16.0 * ns / world * n_p
    lo, hi = parallel.shard_range(ns, rank, world) if sharded else (0, ns)
    en_flops = energy_flops(w, spins_all[lo:hi], ij)
    jac_ms = stage_ms["jacobian"]
    rec = {
        "metric": METRIC,
        "value": args.steps / (total_ms * 1e-3),
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded uniform S^z=0 spins, complex-normal weights; workloads.py)",
        "config": config_of(w, world, engine, sharded),
        "roofline": roofline,
        "stage_roofline": {
            "block_qgt": {"engine": engine, "fp64_equivalent_tflops": achieved,
                          "fp64_dmma_peak": FP64_PEAK_TFLOPS, "ratio": achieved / FP64_PEAK_TFLOPS,
                          "includes": "column scaling + digit split + Gram" if engine == "int8" else "Gram"},
            "jacobian": {"bound": "hbm", "achieved_gbs": O_bytes / (jac_ms * 1e-3) / 1e9,
                         "peak_gbs": peaks["hbm_gbs"], "frac": O_bytes / (jac_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "algorithmic": "16 B x N_s x n_p written (O)"},
            "center_force": {"bound": "hbm",
                             "achieved_gbs": 3 * O_bytes / (stage_ms["center_force"] * 1e-3) / 1e9,
                             "peak_gbs": peaks["hbm_gbs"],
                             "frac": 3 * O_bytes / (stage_ms["center_force"] * 1e-3) / 1e9 / peaks["hbm_gbs"],
                             "algorithmic": "O read twice, A written once"},
            "local_energy": {"bound": "fp64 tensor (DMMA dense layers) + FP64 ALU (lncosh)",
                             "achieved_tflops": en_flops / (stage_ms["local_energy"] * 1e-3) / 1e12,
                             "peak_tflops": FP64_PEAK_TFLOPS,
                             "frac": en_flops / (stage_ms["local_energy"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                             "algorithmic": "8 x sum over connected configurations of (2 w_1 + sum_{l>=1} w_l w_{l+1}) "
                                            f"= {en_flops:.4e} flop (lncosh not counted)"},
            "block_solve": {"bound": "tensor", "achieved_tflops": chol_flops(w) / (stage_ms["block_solve"] * 1e-3) / 1e12,
                            "peak_tflops": FP64_PEAK_TFLOPS,
                            "frac": chol_flops(w) / (stage_ms["block_solve"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                            "algorithmic": "sum_b 4 n_b^3 / 3 (ZPOTRF)"},
        },
        "stages_ms": stage_ms,
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "cuda_graph": use_graph,
        "clocks": clk,
        "e2e": e2e,
    }
    if not sharded and comparison is not None:
        rec["comparison_solves"] = comparison
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(rec), flush=True)
    if sharded:
        dist.destroy_process_group()


def compare_solves(sr, torch, step, w, dev):
    """The comparison paths of north_star on the step's own centred Jacobian A, force F and
    residuals e: block QGT + block solve (the method), the full-QGT solve and the
    sample-space NTK solve (§1-2), each timed once eagerly with CUDA events after a
    warm call; reports how far the block update is from the full one, and the push-through
    identity (full == NTK) on real data.  A path whose workspace does not fit in the free
    device memory (with the step's buffers still resident) is skipped."""
    b = step.buf
    lib = sr.load()
    ns = b.O.shape[0]
    free = torch.cuda.mem_get_info(dev)[0] - (2 << 30)
    need = {"full_qgt_solve": lib.sr_full_qgt_solve_workspace_bytes(ns, b.n_p) + 16 * b.n_p,
            "ntk_solve": lib.sr_ntk_solve_workspace_bytes(ns, b.n_p) + 16 * b.n_p}
    out_d = {"full_qgt_solve": torch.empty_like(b.dtheta), "ntk_solve": torch.empty_like(b.dtheta)}
    calls = {"block_qgt+block_solve": lambda ws: (step.ops.block_qgt(b.O, b.offs, b.S),
                                                  step.ops.block_solve(b.offs, b.S, b.F, w.lam, b.dtheta)),
             "full_qgt_solve": lambda ws: sr.sr_full_qgt_solve(b.O, b.F, w.lam, out_d["full_qgt_solve"], workspace=ws),
             "ntk_solve": lambda ws: sr.sr_ntk_solve(b.O, b.e_tilde, w.lam, out_d["ntk_solve"], workspace=ws)}
    ms, skipped = {}, {}
    for name, fn in calls.items():
        ws = None
        if name in need:
            if need[name] > free:
                skipped[name] = f"workspace {need[name] / 1e9:.0f} GB > {free / 1e9:.0f} GB free"
                continue
            ws = torch.empty(int(need[name]), dtype=torch.uint8, device=dev)
        fn(ws)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(ws)
        e1.record()
        torch.cuda.synchronize(dev)
        ms[name] = e0.elapsed_time(e1)
        del ws
        torch.cuda.empty_cache()
    nrm = lambda x: float(torch.linalg.vector_norm(x).item())   # noqa: E731
    out = {"ms": ms, "sizes": {"full_qgt": b.n_p, "ntk": int(ns), "blocks": [int(x) for x in block_sizes(w)]},
           "note": "eager, one timed call each after a warm call; A, F, e from the step above"}
    ref = "full_qgt_solve" if "full_qgt_solve" in ms else ("ntk_solve" if "ntk_solve" in ms else None)
    if "full_qgt_solve" in ms and "ntk_solve" in ms:
        out["rel_l2_full_vs_ntk"] = nrm(out_d["full_qgt_solve"] - out_d["ntk_solve"]) / nrm(out_d["full_qgt_solve"])
    if ref:
        out[f"rel_l2_block_vs_{ref.split('_')[0]}"] = nrm(b.dtheta - out_d[ref]) / nrm(out_d[ref])
    if skipped:
        out["skipped"] = skipped
    return out


def run_e2e_sharded(torch, dist, step, theta_h, dev, args, theta_graph=None):
    """e2e of the sharded step through the public Python API: every step copies theta from
    pinned host memory, runs parallel.ShardedStep (C ABI + NCCL; the captured CUDA graph when
    theta_graph, the buffer it was captured on, is given) and reads dtheta back; host clock
    between barriers, max over ranks.  (The spins shard stays resident: the samples are the
    rank's data, not a per-step input.)"""
    th = torch.from_numpy(theta_h).pin_memory()
    dth = torch.empty(theta_h.shape[0], dtype=torch.complex128).pin_memory()
    theta = theta_graph if theta_graph is not None else torch.empty(theta_h.shape[0], dtype=torch.complex128,
                                                                     device=dev)

    def one():
        theta.copy_(th, non_blocking=True)
        d, _ = step.replay() if theta_graph is not None else step.run(theta)
        dth.copy_(d, non_blocking=True)
        torch.cuda.synchronize(dev)

    for _ in range(max(1, args.warmup)):
        one()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    return {"value": args.steps / float(dt.item()), "unit": "steps/s", "h2d_bytes_per_step": int(th.numel() * 16),
            "d2h_bytes_per_step": int(dth.numel() * 16),
            "api": ("parallel.ShardedStep " + ("graph replay" if theta_graph is not None else "run") +
                    " (C ABI + NCCL), pinned theta in, dtheta out, host-clock timed")}


def run_e2e(sr, torch, w, theta_h, spins, ij, jj, dev, args):
    nb = len(jj)
    th = torch.from_numpy(theta_h).pin_memory()
    sp = torch.from_numpy(spins).pin_memory()
    bij = torch.from_numpy(ij).pin_memory()
    bj = torch.from_numpy(jj).pin_memory()
    dth = torch.empty(w.n_params, dtype=torch.complex128).pin_memory()
    en = torch.empty(1, dtype=torch.complex128).pin_memory()
    nbytes = sr.sr_step_workspace_bytes(w.widths, w.n_samples, nb) + sr.sr_step_host_extra_bytes(
        w.widths, w.n_samples, nb)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(max(1, args.warmup)):
        sr.sr_step_host(w.widths, th, sp, bij, bj, w.lam, dth, en, ws)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sr.sr_step_host(w.widths, th, sp, bij, bj, w.lam, dth, en, ws)
    dt = time.perf_counter() - t0
    del ws
    return {"value": args.steps / dt, "unit": "steps/s",
            "h2d_bytes_per_step": int(th.numel() * 16 + sp.numel() + bij.numel() * 4 + bj.numel() * 8),
            "d2h_bytes_per_step": int(dth.numel() * 16 + en.numel() * 16),
            "api": "sr_step_host (C ABI, pinned host buffers, host-clock timed, stream synchronised per step)"}


def _ncu_traffic(name):
    """dram bytes per launch of the Gram kernel from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- oracle arm
def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_step_estimate(w, n_sub):
    """Time the oracle on a bounded sample of workload w and scale it to one full step.

    Sample: Jacobian, local energies and centring/force on n_sub samples, the block Gram
    on the same n_sub samples, the Cholesky-equivalent solve of the smallest block; each
    part is scaled linearly (samples) or by sum_b n_b^3 / n_min^3 (solve)."""
    from oracle import estimators, hamiltonian, network, solvers
    spins, params = workloads.make_inputs(w, n_sub)
    bonds = hamiltonian.bonds_for(w)
    off = network.layer_offsets(params)
    t0 = time.perf_counter()
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, bonds)
    estimators.force(O, e)
    t1 = time.perf_counter()
    blocks = estimators.qgt_blocks(O, off)
    t2 = time.perf_counter()
    sizes = block_sizes(w)
    b0 = int(np.argmin(sizes))
    S0 = blocks[b0]
    F0 = np.ones(S0.shape[0], dtype=np.complex128)
    solvers.shifted_solve(S0, F0, w.lam)
    t3 = time.perf_counter()
    scale = w.n_samples / n_sub
    solve_scale = sum(n ** 3 for n in sizes) / sizes[b0] ** 3
    est = (t1 - t0) * scale + (t2 - t1) * scale + (t3 - t2) * solve_scale
    sample = (f"{w.name}: Jacobian+E_loc+force and block Gram on {n_sub} of {w.n_samples} samples (x{scale:g}), "
              f"shifted solve of the {sizes[b0]}-block (x{solve_scale:.2f} by sum n_b^3); measured "
              f"{t3 - t0:.1f} s of CPU work")
    return est, sample


def cpu_baseline(w, quick=False):
    est, sample = oracle_step_estimate(w, 64 if quick else 256)
    return {"value": 1.0 / est, "unit": "steps/s", "cores": _threads(), "kind": "oracle", "sample": sample}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = workloads.BY_NAME[args.workload]
    for _ in range(args.warmup):
        oracle_step_estimate(w, 32)
    ests = []
    sample = ""
    for _ in range(args.steps):
        est, sample = oracle_step_estimate(w, 64)
        ests.append(est)
    total = float(np.sum(ests))
    rec = {"metric": METRIC, "value": args.steps / total, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": config_of(w, world, args.gram_engine, world > 1),
           "cpu_baseline": {"value": args.steps / total, "unit": "steps/s", "cores": _threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": args.steps / total, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=list(workloads.BY_NAME))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compare", action="store_true", help="skip the full-QGT / NTK comparison solves")
    ap.add_argument("--no-graph", action="store_true", help="launch stage by stage instead of one CUDA graph")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sample-sharded NCCL step even on one rank (tests the multi-GPU path)")
    ap.add_argument("--gram-engine", default="int8", choices=["int8", "fp64"],
                    help="stage (4) engine: int8 tcgen05 digit slices (default) or FP64 DMMA")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
