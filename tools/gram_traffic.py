"""DRAM traffic of the block-QGT Gram kernel (gram_i8) for one step of a bench workload.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:gram_i8 --csv --log-file gpurun_out/traffic_<w>.csv \
        python tools/gram_traffic.py run <workload>
    python tools/gram_traffic.py summarise <workload> gpurun_out/traffic_<w>.csv

`run` performs exactly one stage-(4) call (sr_block_qgt_i8, the step's grouping and K-split
launches) on a centred random A of the workload's shape (samples per GPU at N=1);
`summarise` sums the launches of that call and writes profiles/traffic_gram_i8_<workload>.json,
which bench.py attaches as roofline.traffic when it runs that workload."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def run(name):
    import torch
    import paper_2510_08430_b200 as sr
    w = bench.workload_for(name, 1)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.complex(torch.randn(w.n_samples, w.n_params, dtype=torch.float64, device=dev, generator=g),
                      torch.randn(w.n_samples, w.n_params, dtype=torch.float64, device=dev, generator=g))
    offs = sr.block_offsets(w.widths)
    if bench.choose_schedule(sr, torch, w, w.n_samples, 1, dev, "auto") == "per_block":
        n_max = max(offs[b + 1] - offs[b] for b in range(len(offs) - 1))
        S = torch.empty(n_max * n_max, dtype=torch.complex128, device=dev)
        for b in range(len(offs) - 1):
            n = offs[b + 1] - offs[b]
            sr.sr_block_qgt_i8(A[:, offs[b]:offs[b + 1]], [0, n], S[:n * n])
    else:
        S = torch.empty(sum((offs[b + 1] - offs[b]) ** 2 for b in range(len(offs) - 1)), dtype=torch.complex128,
                        device=dev)
        sr.sr_block_qgt_i8(A, offs, S)
    torch.cuda.synchronize()


def summarise(name, path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "msecond": 1e-3, "usecond": 1e-6,
             "nsecond": 1e-9, "second": 1.0}
    tot = {}
    launches = set()
    for r in rows[1:]:
        if "gram_i8" not in r[ki]:
            continue
        launches.add(r[0])
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        tot[r[mi]] = tot.get(r[mi], 0.0) + v
    w = bench.workload_for(name, 1)
    out = {"workload": name, "n_samples_per_gpu": w.n_samples, "kernel": "sr::oz::gram_i8<MODE_HERM>",
           "launches": len(launches), "dram_bytes_read": tot.get("dram__bytes_read.sum"),
           "dram_bytes_write": tot.get("dram__bytes_write.sum"),
           "dram_bytes_per_step": tot.get("dram__bytes_read.sum", 0) + tot.get("dram__bytes_write.sum", 0),
           "kernel_seconds_under_ncu": tot.get("gpu__time_duration.sum"),
           "algorithmic_bytes": sum(21 * bench.workloads.BY_NAME[name].with_samples(w.n_samples).n_samples
                                    * n for n in w.layer_sizes) + 16 * sum(n * n for n in w.layer_sizes),
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/gram_traffic.py run {name})"}
    dst = os.path.join(ROOT, "profiles", f"traffic_gram_i8_{name}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        summarise(sys.argv[2], sys.argv[3])
