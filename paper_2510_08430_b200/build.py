"""Build libsrblock.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsrblock.so")
SOURCES = ["mlp.cu", "center.cu", "chol.cu", "ozaki.cu", "cg.cu", "panel.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-Xptxas", "-v", "--expt-relaxed-constexpr",
]


def _inputs():
    names = SOURCES + [f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    paths = [os.path.join(CSRC, n) for n in names]
    paths.append(os.path.join(os.path.dirname(HERE), "include", "sr_block.h"))
    return paths


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _inputs())


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """Compile every translation unit to an object file in parallel (one nvcc each), then
    link the shared library (static cudart).  defines/out: a measurement variant (extra -D
    macros, written to `out` with its own object directory) -- tools only."""
    if out is None and not force and up_to_date():
        return LIB
    target = out or LIB
    objdir = os.path.join(HERE, "build" if out is None else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]
    jobs = []
    for s in SOURCES:
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [NVCC, *cflags, "-c", os.path.join(CSRC, s), "-o", obj]
        jobs.append((cmd, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log_txt, failed = "", False
    for cmd, obj, p in jobs:
        so, se = p.communicate()
        log_txt += " ".join(cmd) + "\n" + so + se
        failed |= p.returncode != 0
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
            *[o for _, o, _ in jobs], "-o", target + ".tmp"]
    if not failed:
        r = subprocess.run(link, capture_output=True, text=True)
        log_txt += " ".join(link) + "\n" + r.stdout + r.stderr
        failed = r.returncode != 0
    log = os.path.join(HERE, "build.log" if out is None else "build_variant.log")
    with open(log, "w") as f:
        f.write(log_txt)
    if failed:
        sys.stderr.write(log_txt[-6000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(target + ".tmp", target)
    if verbose:
        sys.stderr.write(log_txt)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
