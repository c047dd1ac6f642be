"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) by
kernel: total time, share, launches.  Usage: python tools/ncu_summary.py file.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    data = [r for r in data if mi is None or r[mi] == "gpu__time_duration.sum"]
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][0] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        agg[name][1] += 1
    tot = sum(a[0] for a in agg.values())
    print(f"# {path}: {len(data)} launches, {tot:.3f} ms total (cold-cache, serialised)")
    for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{t:9.3f} ms {100 * t / tot:5.1f}%  n={n:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
