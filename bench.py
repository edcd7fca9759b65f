"""Block-SR step benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

A step is one pass of the whole hot path over one batch of synthetic input
(DESIGN.md §8(a)): Jacobian -> local energy -> centring + force -> block QGT (Gram) ->
block solve, each stage one C-ABI call of libsrblock.so.  Default workload: BASELINE.json
configs[3], the largest configuration that fits one GPU (J1-J2 10x10, MLP 100->128 + five
128->128, 6 blocks, N_s=32768, lambda=1e-3), strong scaling over N GPUs.  configs[4]
(--workload j1j2_10x10_w160) is the weak-scaling configuration: 8192 samples per GPU,
N_s = 8192 N, one block owner per GPU at N=8; at N=1 it runs the per-block schedule
(sr_set_step_schedule) so that all eight blocks fit one GPU.

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
DEFAULT_WORKLOAD = workloads.CONFIGS[3].name
WEAK_WORKLOADS = {workloads.CONFIGS[4].name: 8192}     # samples per GPU (BASELINE configs[4])
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
        if not rows:   # a timed region shorter than the sampling interval: one query now
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                rows = [[p.strip() for p in line.split(",")] for line in out.stdout.splitlines()
                        if len(line.split(",")) >= 8]
            except (OSError, subprocess.SubprocessError):
                rows = []
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


def workload_for(name, world):
    """The BASELINE.json configuration a run of `world` GPUs measures: the strong-scaling
    workloads as listed; configs[4] with 8192 samples per GPU (weak scaling)."""
    w = workloads.BY_NAME[name]
    if name in WEAK_WORKLOADS:
        w = w.with_samples(WEAK_WORKLOADS[name] * world)
    return w


def config_of(w, world, engine, sharded, schedule="batched", chunk=0):
    """The workload description shared by both arms' JSON lines."""
    weak = w.name in WEAK_WORKLOADS and w.n_samples == WEAK_WORKLOADS[w.name] * world
    rows = min(chunk, w.n_samples) if chunk else w.n_samples // world
    return {"workload": w.name, "lattice": f"{w.lattice}{'x'.join(map(str, w.extent))}",
            "widths": list(w.widths), "n_samples": w.n_samples, "n_params": w.n_params, "blocks": block_sizes(w),
            "lambda": w.lam, "gram_engine": engine, "step_schedule": schedule,
            "samples_per_gpu": w.n_samples // world,
            "parallelism": f"samples sharded x{world} (NCCL)" if sharded else "single GPU",
            "scaling": ("weak (8192 samples per GPU)" if weak else "strong (fixed N_s)"),
            "l2": f"inputs larger than L2 (O = {16.0 * rows * w.n_params / 1e9:.2f} GB resident per GPU"
                  + (f", {16.0 * w.n_samples * w.n_params / 1e9:.0f} GB over the chunks" if chunk else "")
                  + " vs 126 MB L2); no flush"}


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
def choose_schedule(sr, torch, w, n_local, nb, dev, want):
    """Stage (4)-(5) schedule: as asked, or (auto) batched when its step workspace fits the
    free device memory with room for the comparison solves, else per-block."""
    if want != "auto":
        return want
    free = torch.cuda.mem_get_info(dev)[0]
    need = sr.sr_step_workspace_bytes(w.widths, n_local, nb)
    return "batched" if need < 0.7 * free else "per_block"


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
    w = workloads.BY_NAME[args.workload] if args.full_samples else workload_for(args.workload, world)
    spins_all, params = workloads.make_inputs(w)
    ij, jj = sr.lattice.for_workload(w)
    theta_h = sr.model.pack(params)
    n_p, ns = w.n_params, w.n_samples
    n_local = ns // world

    engine = args.gram_engine
    sr.sr_set_gram_engine(sr.GRAM_INT8 if engine == "int8" else sr.GRAM_FP64)   # for sr_step_host (e2e)
    schedule = "sharded" if sharded else choose_schedule(sr, torch, w, ns, len(jj), dev, args.schedule)
    if args.chunk and not sharded:
        schedule = f"chunked ({args.chunk} samples per pass; parallel.ChunkedStep)"
    if sharded:
        step = parallel.ShardedStep(w.widths, spins_all, ij, jj, w.lam, rank, world, dev, gram_engine=engine)
    elif args.chunk:
        step = parallel.ChunkedStep(w.widths, spins_all, ij, jj, w.lam, dev, chunk=args.chunk)
    else:
        step = parallel.LocalStep(w.widths, spins_all, ij, jj, w.lam, dev, gram_engine=engine, schedule=schedule)
    theta = torch.from_numpy(theta_h).to(dev)
    stream = torch.cuda.current_stream(dev)

    t_warm = time.perf_counter()
    for _ in range(args.warmup):
        step.run(theta)
    torch.cuda.synchronize(dev)
    est_step_s = (time.perf_counter() - t_warm) / max(1, args.warmup)

    # per-stage breakdown: eager launches with CUDA events between the C-ABI stage calls, and
    # the library's CUDA-event timer around every launch of the Gram kernel
    n_ev = len(step.STAGES) + 1
    n_stage_runs = max(1, min(args.steps, 3 if est_step_s < 1.0 else 2))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(n_stage_runs)]
    gram_kernel = "gram_i8" if engine == "int8" else "gram_tn"
    sr.sr_kernel_time_ms(gram_kernel)
    sr.sr_kernel_timer(True)
    sr.sr_reset_launch_count()
    for k in range(n_stage_runs):
        step.run(theta, events=evs[k])
    torch.cuda.synchronize(dev)
    sr.sr_kernel_timer(False)
    launches = sr.sr_launch_count() // n_stage_runs
    gk_ms, gk_n = sr.sr_kernel_time_ms(gram_kernel)
    gram_kernel_ms = gk_ms / n_stage_runs        # all launches of one step's Grams
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
        for _ in range(min(args.warmup, 3 if est_step_s < 1.0 else 1)):
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
    ms_per_step = total_ms / args.steps
    # e2e: at most ~60 s of it
    e2e_steps = max(1, min(args.steps, int(60e3 / max(ms_per_step, 1e-3))))

    fp64 = comparison = None
    if sharded:
        e2e = run_e2e_sharded(torch, dist, step, theta_h, dev, args, theta if use_graph else None, e2e_steps)
    elif args.chunk:
        e2e = run_e2e_api(torch, step, theta_h, dev, theta if use_graph else None, e2e_steps)
    else:
        if engine == "int8" and not args.no_fp64_engine and not args.chunk:
            fp64 = fp64_engine_record(sr, torch, step, theta, w, dev)
        comparison = None if (args.no_compare or args.chunk) else compare_solves(sr, torch, step, w, dev)
        del step                      # the e2e run allocates its own sr_step workspace
        torch.cuda.empty_cache()
        e2e = run_e2e(sr, torch, w, theta_h, spins_all, ij, jj, dev, args, schedule, e2e_steps)

    if rank != 0:
        if sharded:
            dist.destroy_process_group()
        return
    peaks = _peaks()
    gflop = gram_flops(w, n_local)
    fp64_eq = gflop / (gram_kernel_ms * 1e-3) / 1e12
    long_step = ms_per_step > 1000.0
    if engine == "int8":
        ops = gram_i8_ops(w, n_local)
        # The burst figure applies to a kernel timed alone near the maximum clock; a kernel timed
        # inside a multi-second step runs at the sustained (power-capped) clock: B200_PROFILING.md.
        peak_burst = peaks["bf16_tflops"] * INT8_OVER_BF16
        peak_sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * INT8_OVER_BF16
        peak = peak_sus if long_step else peak_burst
        ach = ops / (gram_kernel_ms * 1e-3) / 1e12
        roofline = {
            "kernel": "sr::oz::gram_i8 (sr_block_qgt_i8: tcgen05.mma kind::i8, TMA, TMEM)", "bound": "tensor",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s", "op_dtype": "int8 (one multiply-add = 2 ops)",
            "frac": ach / peak, "traffic": _ncu_traffic("gram_i8", w.name, n_local),
            "kernel_ms": gram_kernel_ms, "kernel_launches": gram_launches,
            "algorithmic": (f"sum_b 2 (Re, Im) x n_b(n_b+1)/2 entries x K'=2 N_s x {INT8_PAIRS} slice pairs x 2 "
                            f"= {ops:.4e} int8 ops per step (all launches)"),
            "peak_source": ("MEASURED_PEAKS.json " + ("bf16_tflops_sustained" if long_step else "bf16_tflops (burst)")
                            + " x 2, the nominal dense int8 : bf16 ratio (4.5 : 2.25 PFLOP/s, B200_PROFILING.md); "
                            + ("sustained: the kernel runs inside a multi-second step" if long_step else
                               "burst: the step is shorter than a second")),
            "frac_of_burst": ach / peak_burst, "frac_of_sustained": ach / peak_sus,
            "frac_of_tcgen05_microbenchmark": ach / 4763.0,
            "fp64_equivalent": {"achieved_tflops": fp64_eq, "fp64_dmma_peak": FP64_PEAK_TFLOPS,
                                "ratio_to_fp64_peak": fp64_eq / FP64_PEAK_TFLOPS,
                                "algorithmic": f"sum_b 4 N_s n_b (n_b+1) = {gflop:.4e} flop"},
        }
    else:
        tma = os.environ.get("SR_FP64_TMA", "1") != "0"
        roofline = {"kernel": ("gram::tn_tma_kernel<HERM_STORE>" if tma else "gram::tile_kernel<TN,HERM_STORE>")
                              + " (sr_block_qgt: FP64 DMMA)", "bound": "tensor",
                    "achieved": fp64_eq, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": fp64_eq / FP64_PEAK_TFLOPS, "traffic": _ncu_traffic("gram_tn", w.name, n_local),
                    "kernel_ms": gram_kernel_ms,
                    "algorithmic": f"sum_b 4 N_s n_b (n_b+1) = {gflop:.4e} flop per step",
                    "peak_source": FP64_PEAK_SOURCE}
    O_bytes = 16.0 * n_local * n_p
    lo, hi = parallel.shard_range(ns, rank, world) if sharded else (0, ns)
    en_flops = energy_flops(w, spins_all[lo:hi], ij)
    jac_ms = stage_ms.get("jacobian")
    qgt_ms = stage_ms.get("block_qgt", gram_kernel_ms)
    solve_ms = stage_ms.get("block_solve", stage_ms.get("block_qgt_solve", 0.0) - gram_kernel_ms)
    chunked = jac_ms is None    # the chunked step times passes, not stages
    if chunked:
        jac_ms = 1.0
    stage_roofline = {
        "block_qgt": {"engine": engine, "fp64_equivalent_tflops": gflop / (qgt_ms * 1e-3) / 1e12,
                      "fp64_dmma_peak": FP64_PEAK_TFLOPS, "ratio": gflop / (qgt_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                      "includes": ("column scaling + digit split + Gram" if engine == "int8" else "Gram")
                      if "block_qgt" in stage_ms else "Gram kernel only (per-block schedule)"},
        "jacobian": {"bound": "hbm", "achieved_gbs": O_bytes / (jac_ms * 1e-3) / 1e9,
                     "peak_gbs": peaks["hbm_gbs"], "frac": O_bytes / (jac_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                     "algorithmic": "16 B x N_s x n_p written (O)"},
        "center_force": {"bound": "hbm",
                         "achieved_gbs": 3 * O_bytes / (stage_ms.get("center_force", 1.0) * 1e-3) / 1e9,
                         "peak_gbs": peaks["hbm_gbs"],
                         "frac": 3 * O_bytes / (stage_ms.get("center_force", 1.0) * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "algorithmic": "O read twice, A written once"},
        "local_energy": {"bound": "fp64 tensor (DMMA dense layers) + FP64 ALU (lncosh)",
                         "achieved_tflops": en_flops / (stage_ms.get("local_energy", 1.0) * 1e-3) / 1e12,
                         "peak_tflops": FP64_PEAK_TFLOPS,
                         "frac": en_flops / (stage_ms.get("local_energy", 1.0) * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                         "algorithmic": "8 x sum over connected configurations of (2 w_1 + sum_{l>=1} w_l w_{l+1}) "
                                        f"= {en_flops:.4e} flop (lncosh not counted)"},
    }
    if chunked:
        stage_roofline = {"block_qgt": stage_roofline["block_qgt"],
                          "note": "chunked step: stages_ms are the two passes over the sample chunks and the solves"}
    if not sharded:
        cf = chol_flops(w)
        stage_roofline["block_solve"] = {
            "bound": "tensor", "ms": solve_ms,
            "fp64_equivalent_tflops": cf / (solve_ms * 1e-3) / 1e12, "fp64_dmma_peak": FP64_PEAK_TFLOPS,
            "ratio_to_fp64_peak": cf / (solve_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
            "algorithmic": "sum_b 4 n_b^3 / 3 (ZPOTRF count)",
            "note": ("FP64-EQUIVALENT rate: the trailing updates run on the int8 engine (exact digit slices), "
                     "chol_diag/TRSM/in-strip updates on FP64 DMMA" if engine == "int8" else "all FP64 DMMA")}
    rec = {
        "metric": METRIC,
        "value": args.steps / (total_ms * 1e-3),
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak" if (world == 1 or w.name in WEAK_WORKLOADS) else "strong",
        "vs_baseline": None,
        "dtype": "f64 (int8 Ozaki-7 emulation: exact int8 digit products, FP64 recombination)" if engine == "int8"
                 else "f64 (DMMA)",
        "data": "synthetic (seeded uniform S^z=0 spins, complex-normal weights; workloads.py)",
        "config": config_of(w, world, engine, sharded, schedule, args.chunk),
        "roofline": roofline,
        "stage_roofline": stage_roofline,
        "stages_ms": stage_ms,
        "stages_note": "eager launches with CUDA events between the C-ABI calls (the timed step is a graph replay)",
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "cuda_graph": use_graph,
        "clocks": clk,
        "e2e": e2e,
    }
    if fp64 is not None:
        rec["fp64_engine"] = fp64
    if comparison is not None:
        rec["comparison_solves"] = comparison
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(rec), flush=True)
    if sharded:
        dist.destroy_process_group()


def fp64_engine_record(sr, torch, step, theta, w, dev):
    """north_star's engine: one eager step with the FP64 DMMA Gram (TMA-staged K-slabs) and
    FP64 DMMA trailing updates, timed with CUDA events; the Gram kernel against the measured
    DMMA peak."""
    prev_eng = step.ops.gram_engine
    step.ops.gram_engine = "fp64"
    prev = sr.sr_set_gram_engine(sr.GRAM_FP64)
    try:
        step.run(theta)                          # warm (FP64-engine attributes, side streams)
        torch.cuda.synchronize(dev)
        sr.sr_kernel_time_ms("gram_tn")
        sr.sr_kernel_timer(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step.run(theta)
        e1.record()
        torch.cuda.synchronize(dev)
        sr.sr_kernel_timer(False)
        gms, n = sr.sr_kernel_time_ms("gram_tn")
    finally:
        sr.sr_set_gram_engine(prev)
        step.ops.gram_engine = prev_eng
    gflop = gram_flops(w, w.n_samples)
    return {"step_ms": e0.elapsed_time(e1), "gram_kernel_ms": gms, "gram_launches": n,
            "gram_tflops": gflop / (gms * 1e-3) / 1e12, "fp64_dmma_peak": FP64_PEAK_TFLOPS,
            "gram_frac_of_dmma_peak": gflop / (gms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
            "kernel": "gram::tn_tma_kernel<HERM_STORE> (FP64 DMMA.8x8x4, TMA 2-D boxes, 3 mbarrier stages)",
            "note": "one eager step after a warm step; Gram and Cholesky trailing updates on FP64 DMMA"}


def compare_solves(sr, torch, step, w, dev):
    """The comparison paths of north_star on the step's own centred Jacobian A, force F and
    residuals e: block QGT + block solve (the method), the full-QGT solve and the
    sample-space NTK solve (§1-2), each timed once eagerly with CUDA events after a
    warm call; reports how far the block update is from the full one, and the push-through
    identity (full == NTK) on real data.  The block path runs first on the step's buffers;
    then the step's S blocks and stage workspace are released so the comparison paths get
    the memory.  A path whose workspace still does not fit is skipped and says why."""
    b = step.buf
    lib = sr.load()
    ns = b.O.shape[0]
    out_d = {}
    if step.schedule == "per_block":
        block_call = lambda ws: step.ops.block_qgt_solve(b.O, b.offs, b.F, w.lam, b.dtheta)  # noqa: E731
    else:
        block_call = lambda ws: (step.ops.block_qgt(b.O, b.offs, b.S),  # noqa: E731
                                 step.ops.block_solve(b.offs, b.S, b.F, w.lam, b.dtheta))
    cg_info = {}

    def full_cg(ws):
        from paper_2510_08430_b200 import parallel
        x, it, res = parallel.full_qgt_cg(step.ops, parallel.SelfComm(), b.O, b.F, w.lam)
        out_d["full_qgt_cg"] = x
        cg_info.update(iterations=it, rel_residual=res)

    def full_dist(ws):
        from paper_2510_08430_b200 import parallel

        class _One(parallel.SelfComm):     # the distributed dense path as one rank
            def reduce(self, t, dst, async_op=False):
                return parallel._Done()

            def broadcast(self, t, src):
                pass

            def all_gather(self, out, t):
                out[0].copy_(t)
        out_d["full_qgt_dist"] = parallel.dist_full_qgt(step.ops, _One(), 0, 1, b.O, b.F, w.lam)

    calls = {"block_qgt+block_solve": block_call,
             "full_qgt_solve": lambda ws: sr.sr_full_qgt_solve(b.O, b.F, w.lam, out_d["full_qgt_solve"], workspace=ws),
             "full_qgt_cg": full_cg,
             "ntk_solve": lambda ws: sr.sr_ntk_solve(b.O, b.e_tilde, w.lam, out_d["ntk_solve"], workspace=ws)}
    # the formed-and-factorised distributed path, as one rank (configs[3]: ~29 s on the int8
    # engine; timed once, without the warm call, above 40000 parameters)
    calls["full_qgt_dist"] = full_dist
    once = {"full_qgt_dist"} if b.n_p > 40000 else set()
    need = {"full_qgt_solve": lib.sr_full_qgt_solve_workspace_bytes(ns, b.n_p) + 16 * b.n_p,
            "ntk_solve": lib.sr_ntk_solve_workspace_bytes(ns, b.n_p) + 16 * b.n_p}
    ms, skipped = {}, {}
    for name, fn in calls.items():
        ws = None
        if name in need:
            if name == "full_qgt_solve":          # the block path is done: free its buffers
                b.S = None
                step.ops.ws = None
                torch.cuda.empty_cache()
            free = torch.cuda.mem_get_info(dev)[0] - (2 << 30)
            if need[name] > free:
                skipped[name] = f"workspace {need[name] / 1e9:.0f} GB > {free / 1e9:.0f} GB free on one B200"
                continue
            ws = torch.empty(int(need[name]), dtype=torch.uint8, device=dev)
            out_d[name] = torch.empty_like(b.dtheta)
        if name not in once:
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
           "note": ("eager, one timed call each after a warm call (full_qgt_dist above 40000 parameters: one "
                    "call, no warm call); A, F, e from the step above; full_qgt_dist = parallel.dist_full_qgt as "
                    "one rank: the full QGT formed and factorised by panels")}
    ref = next((k for k in ("full_qgt_solve", "full_qgt_dist", "full_qgt_cg", "ntk_solve") if k in ms), None)
    if "full_qgt_dist" in ms and "full_qgt_cg" in ms:
        out["rel_l2_full_dist_vs_cg"] = (nrm(out_d["full_qgt_dist"] - out_d["full_qgt_cg"])
                                         / nrm(out_d["full_qgt_cg"]))
    if "full_qgt_solve" in ms and "ntk_solve" in ms:
        out["rel_l2_full_vs_ntk"] = nrm(out_d["full_qgt_solve"] - out_d["ntk_solve"]) / nrm(out_d["full_qgt_solve"])
    if "full_qgt_dist" in ms and "full_qgt_solve" in ms:
        out["rel_l2_full_dist_vs_full"] = (nrm(out_d["full_qgt_dist"] - out_d["full_qgt_solve"])
                                           / nrm(out_d["full_qgt_solve"]))
    if "full_qgt_cg" in ms and "ntk_solve" in ms:
        out["rel_l2_full_cg_vs_ntk"] = nrm(out_d["full_qgt_cg"] - out_d["ntk_solve"]) / nrm(out_d["ntk_solve"])
    if cg_info:
        out["full_qgt_cg"] = dict(cg_info, note="matrix-free: S p = A^H (A p), S never formed (parallel.full_qgt_cg)")
    if ref:
        out["rel_l2_block_vs_full"] = nrm(b.dtheta - out_d[ref]) / nrm(out_d[ref])
        out["block_vs_full_reference"] = ref
    if skipped:
        out["skipped"] = skipped
    return out


def run_e2e_sharded(torch, dist, step, theta_h, dev, args, theta_graph, steps):
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

    one()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    return {"value": steps / float(dt.item()), "unit": "steps/s", "steps": steps,
            "h2d_bytes_per_step": int(th.numel() * 16), "d2h_bytes_per_step": int(dth.numel() * 16),
            "api": ("parallel.ShardedStep " + ("graph replay" if theta_graph is not None else "run") +
                    " (C ABI + NCCL), pinned theta in, dtheta out, host-clock timed")}


def run_e2e_api(torch, step, theta_h, dev, theta_graph, steps):
    """e2e of a one-GPU step object through the public Python API (ChunkedStep): theta copied
    from pinned host memory, the step (its CUDA graph when captured), dtheta read back; host
    clock, synchronised per step."""
    th = torch.from_numpy(theta_h).pin_memory()
    dth = torch.empty(theta_h.shape[0], dtype=torch.complex128).pin_memory()
    theta = theta_graph if theta_graph is not None else torch.empty(theta_h.shape[0], dtype=torch.complex128,
                                                                     device=dev)

    def one():
        theta.copy_(th, non_blocking=True)
        d, _ = step.replay() if theta_graph is not None else step.run(theta)
        dth.copy_(d, non_blocking=True)
        torch.cuda.synchronize(dev)

    one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = time.perf_counter() - t0
    return {"value": steps / dt, "unit": "steps/s", "steps": steps, "h2d_bytes_per_step": int(th.numel() * 16),
            "d2h_bytes_per_step": int(dth.numel() * 16),
            "api": "parallel.ChunkedStep (C ABI) " + ("graph replay" if theta_graph is not None else "run")
                   + ", pinned theta in, dtheta out, host-clock timed"}


def run_e2e(sr, torch, w, theta_h, spins, ij, jj, dev, args, schedule, steps):
    """e2e through sr_step_host (host buffers in and out every step), one warm call (it
    captures the step's CUDA graph) then `steps` timed calls on the host clock."""
    nb = len(jj)
    th = torch.from_numpy(theta_h).pin_memory()
    sp = torch.from_numpy(spins).pin_memory()
    bij = torch.from_numpy(ij).pin_memory()
    bj = torch.from_numpy(jj).pin_memory()
    dth = torch.empty(w.n_params, dtype=torch.complex128).pin_memory()
    en = torch.empty(1, dtype=torch.complex128).pin_memory()
    prev = sr.sr_set_step_schedule(sr.SCHED_PER_BLOCK if schedule == "per_block" else sr.SCHED_BATCHED)
    try:
        nbytes = sr.sr_step_workspace_bytes(w.widths, w.n_samples, nb) + sr.sr_step_host_extra_bytes(
            w.widths, w.n_samples, nb)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        sr.sr_step_host(w.widths, th, sp, bij, bj, w.lam, dth, en, ws)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(steps):
            sr.sr_step_host(w.widths, th, sp, bij, bj, w.lam, dth, en, ws)
        dt = time.perf_counter() - t0
        del ws
    finally:
        sr.sr_set_step_schedule(prev)
    return {"value": steps / dt, "unit": "steps/s", "steps": steps,
            "h2d_bytes_per_step": int(th.numel() * 16 + sp.numel() + bij.numel() * 4 + bj.numel() * 8),
            "d2h_bytes_per_step": int(dth.numel() * 16 + en.numel() * 16),
            "api": "sr_step_host (C ABI, pinned host buffers, host-clock timed, stream synchronised per step)"}


def _ncu_traffic(kernel, workload, n_local):
    """DRAM bytes per step of the Gram kernel from the committed `ncu --set full` capture of
    THIS workload (profiles/traffic_<kernel>_<workload>.json, which names the workload and the
    samples per GPU it was captured at); None when no capture of this workload exists."""
    path = os.path.join(ROOT, "profiles", f"traffic_{kernel}_{workload}.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    if d.get("workload") != workload or int(d.get("n_samples_per_gpu", -1)) != int(n_local):
        return None
    return d.get("dram_bytes_per_step")


# ----------------------------------------------------------------------------- oracle arm
def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return os.cpu_count() or 1


ORACLE_MAX_COLS = 1024    # columns of each block the oracle's Gram and solve sample


def oracle_step_estimate(w, n_sub, max_cols=ORACLE_MAX_COLS):
    """Time the oracle on a bounded sample of workload w and scale it to one full step.

    Sample (bounded in rows AND columns, so that configs[3]/[4] stay within seconds and a few
    GB of host memory): Jacobian, local energies and centring/force on n_sub samples (scaled
    by N_s / n_sub); the block Gram of the first min(n_b, max_cols) columns of every block on
    the same samples (scaled by N_s / n_sub x (n_b / cols)^2 per block); the shifted solve of
    one min(n_min, max_cols) leading sub-block (scaled by sum_b n_b^3 / cols^3)."""
    from oracle import estimators, hamiltonian, network, solvers
    spins, params = workloads.make_inputs(w, n_sub)
    bonds = hamiltonian.bonds_for(w)
    off = network.layer_offsets(params)
    sizes = block_sizes(w)
    t0 = time.perf_counter()
    O = network.jacobian(params, spins)
    e = hamiltonian.local_energies(params, spins, bonds)
    estimators.force(O, e)
    t1 = time.perf_counter()
    t_gram = 0.0          # measured, each block's time scaled by (n_b / cols)^2
    for b, n in enumerate(sizes):
        c = min(n, max_cols)
        tb = time.perf_counter()
        estimators.qgt_blocks(O[:, off[b]:off[b] + c], [0, c])
        t_gram += (time.perf_counter() - tb) * (n / c) ** 2
    b0 = int(np.argmin(sizes))
    c0 = min(sizes[b0], max_cols)
    S0 = estimators.qgt_blocks(O[:, off[b0]:off[b0] + c0], [0, c0])[0]
    F0 = np.ones(c0, dtype=np.complex128)
    t2 = time.perf_counter()
    solvers.shifted_solve(S0, F0, w.lam)
    t3 = time.perf_counter()
    scale = w.n_samples / n_sub
    solve_scale = sum(n ** 3 for n in sizes) / c0 ** 3
    est = (t1 - t0) * scale + t_gram * scale + (t3 - t2) * solve_scale
    sample = (f"{w.name}: Jacobian+E_loc+force on {n_sub} of {w.n_samples} samples (x{scale:g}); block Gram of the "
              f"first {min(max(sizes), max_cols)} columns of each block on those samples (x{scale:g} x (n_b/cols)^2); "
              f"shifted solve of a {c0}-column sub-block (x{solve_scale:.4g} by sum n_b^3); measured "
              f"{t3 - t0:.1f} s of CPU work, extrapolated to {est:.0f} s per full step")
    return est, sample


def cpu_baseline(w, quick=False):
    est, sample = oracle_step_estimate(w, 64 if quick else 256)
    return {"value": 1.0 / est, "unit": "steps/s", "cores": _threads(), "kind": "oracle", "sample": sample,
            "extrapolated": True}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = workload_for(args.workload, world)
    t_run = time.perf_counter()
    for _ in range(args.warmup):
        oracle_step_estimate(w, 16)
    ests = []
    sample = ""
    for _ in range(args.steps):
        est, sample = oracle_step_estimate(w, 32)
        ests.append(est)
    total = float(np.sum(ests))
    wall = time.perf_counter() - t_run
    rec = {"metric": METRIC, "value": args.steps / total, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": config_of(w, world, args.gram_engine, world > 1),
           "extrapolated": True,
           "measured_wall_s": wall,
           "note": ("each step times the CPU oracle on a bounded sample of the workload and scales it to one full "
                    "step (see cpu_baseline.sample); ms_per_step is that extrapolated full-step time, not wall time"),
           "cpu_baseline": {"value": args.steps / total, "unit": "steps/s", "cores": _threads(), "kind": "oracle",
                            "sample": sample, "extrapolated": True},
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
    ap.add_argument("--schedule", default="auto", choices=["auto", "batched", "per_block"],
                    help="stages (4)-(5): all Grams then all solves, or block by block (one block's memory)")
    ap.add_argument("--no-fp64-engine", action="store_true", help="skip the FP64-engine sub-record")
    ap.add_argument("--chunk", type=int, default=0,
                    help="process the samples in chunks of this many (parallel.ChunkedStep; one GPU, int8 engine)")
    ap.add_argument("--full-samples", action="store_true",
                    help="configs[4]: all 65536 samples on this run's GPUs instead of 8192 per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
