"""Per-kernel DRAM traffic of one step from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum:
mean bytes per launch for each conv kind (fprop / dgrad / wgrad main kernels),
written as JSON for bench.py's roofline "traffic" field.
Usage: python tools/ncu_traffic.py launches.csv out.json"""
import collections
import csv
import json
import re
import sys

KIND = {0: "conv_fwd", 1: "conv_dgrad", 2: "conv_wgrad"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                           h.index("Metric Unit"), h.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        names[r[idi]] = r[ki]
    agg = collections.defaultdict(lambda: [0.0, 0])
    for lid, m in per.items():
        mt = re.search(r"conv_t(?:ma|c)_kernel<\(int\)(\d)", names[lid]) or re.search(r"conv_t(?:ma|c)_kernel<(\d)",
                                                                                     names[lid])
        if not mt:
            continue
        k = KIND[int(mt.group(1))]
        agg[k][0] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        agg[k][1] += 1
    res = {k: {"bytes_per_launch": t / n, "launches": n, "source": path} for k, (t, n) in agg.items()}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
