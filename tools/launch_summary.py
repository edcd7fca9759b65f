"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: time share per kernel."""
import collections
import csv
import sys


def summarise(path, steps=1):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        k = r[ki]
        name = k.split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
        if "tile_kernel" in k:
            name = "gram::tile_kernel" + k[k.find("<"):k.find(">") + 1]
        tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
        cnt[name] += 1
    s = sum(tot.values())
    out = [f"{len(data)} launches, {s / 1e3:.2f} ms total (cold-cache, serialised)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k:55s} {cnt[k]:6d} launches {v / 1e3 / steps:10.3f} ms/step {100 * v / s:6.2f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1))
