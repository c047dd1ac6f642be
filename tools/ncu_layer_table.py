"""Per-layer-kind ncu table of the contraction kernels of one in-core ResNet
step (round-1 review item 5): for each (op, C, K, R, stride, H) kind —
launches, ncu time, TFLOP/s (algorithmic FLOPs / ncu time), DRAM bytes per
launch against the algorithmic bytes (one read of every operand + one write of
the output; dgrad accumulation reads the old output too), and tensor-pipe
active % of elapsed cycles.

Input: an ncu CSV (`--csv --log-file`) of `tools/profile_step.py --incore`
taken with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
            sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
The contraction launches (conv_tma_kernel / stem kernels) are matched to the
graph's conv functions in issue order (one launch per fprop / wgrad — or per
image slice for the 3-channel stem — and one per dgrad output phase that a
filter tap reaches); the script checks the counts agree.  The launch list
holds the first instrumented step only when --steps 1.  Not part of the product.

Usage: python tools/ncu_layer_table.py launches.csv [--depth 50 --batch 256] > table.md"""
import argparse
import collections
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "%": 1}
CONTRACTION = re.compile(r"conv_tma_kernel|stem_kernel|stem_wgrad_kernel|conv_simt|conv_tc_kernel")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                           h.index("Metric Unit"), h.index("ID"))
    per = collections.OrderedDict()
    for r in data:
        d = per.setdefault(r[idi], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    return [d for d in per.values() if CONTRACTION.search(d["name"])]


def expected(doc):
    """(function id, kind, attrs) per contraction launch, in issue order."""
    out = []
    for f in json.loads(doc)["functions"]:
        op = f["op"]
        k, a = op["kind"], op.get("attrs", {})
        if k not in ("conv_fwd", "conv_dgrad", "conv_wgrad"):
            continue
        n = 1
        if a["C"] % 8 and k in ("conv_fwd", "conv_wgrad"):      # narrow input: image slices
            per = (a["H"] // 2) * (a["W"] // 2) * 16 * 2 if a["stride"] == 2 else a["H"] * a["W"] * 8 * 2
            sl = max(1, (32 << 20) // per)
            n = -(-a["N"] // sl)
        if k == "conv_dgrad":
            st = a["stride"]
            n = sum(1 for ph in range(st) for pw in range(st)
                    if (ph + a["pad"]) % st < a["R"] and (pw + a["pad"]) % st < a["S"])
        out += [(f["id"], k, a)] * n
    return out


def algo(kind, a):
    N, H, W, C, K, R, S, P, Q = a["N"], a["H"], a["W"], a["C"], a["K"], a["R"], a["S"], a["P"], a["Q"]
    flops = 2.0 * N * P * Q * K * R * S * C
    x, y, w = N * H * W * C * 2, N * P * Q * K * 2, K * R * S * C * 2
    if kind == "conv_fwd":
        b = x + w + y
    elif kind == "conv_dgrad":
        b = y + w + x * (2 if a.get("accumulate") else 1)
    else:
        b = x + y + K * R * S * C * 4
    return flops, b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--depth", type=int, default=50)
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args()
    from paper_2010_14109_b200 import graphs
    from synth import nets
    doc, _ = graphs.build(nets.resnet(a.depth, batch=a.batch), params="persistent")
    L = launches(a.csv)
    E = expected(doc)
    if len(L) < len(E):
        print(f"# launch list has {len(L)} contraction launches, the step issues {len(E)}: truncated list")
        E = E[:len(L)]
    L = L[:len(E)]
    agg = collections.OrderedDict()
    for (fid, kind, at), m in zip(E, L):
        key = (kind, at["C"], at["K"], at["R"], at["stride"], at["H"], bool(at.get("accumulate")))
        g = agg.setdefault(key, {"n": 0, "t": 0.0, "fl": 0.0, "dram": 0.0, "algo": 0.0, "tp": [], "fns": set()})
        fl, b = algo(kind, at)
        g["fns"].add(fid)
        g["n"] += 1
        g["t"] += m.get("gpu__time_duration.sum", 0.0)
        g["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        g["tp"].append(m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", float("nan")))
        # algorithmic work is per function: split evenly over its launches (phases / slices)
        g["fl"] += fl
        g["algo"] += b
    # per-function totals were added once per launch: divide by launches per function
    print(f"# ResNet-{a.depth} b={a.batch} in-core, ncu (cold cache, serialised launches); "
          f"{len(L)} contraction launches matched to {len({e[0] for e in E})} conv functions")
    print("| op | C | K | R | stride | H | acc | functions | launches | ncu ms | TFLOP/s | DRAM MB/fn | algorithmic MB/fn | tensor pipe % (mean) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for key, g in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        nf = len(g["fns"])
        per_fn = g["n"] / nf
        fl = g["fl"] / per_fn
        alg = g["algo"] / per_fn
        tp = [v for v in g["tp"] if v == v]
        print(f"| {key[0]} | {key[1]} | {key[2]} | {key[3]} | {key[4]} | {key[5]} | {'y' if key[6] else ''} | {nf} | "
              f"{g['n']} | {g['t'] * 1e3:.3f} | {fl / g['t'] / 1e12:.0f} | {g['dram'] / nf / 1e6:.1f} | "
              f"{alg / nf / 1e6:.1f} | {sum(tp) / len(tp) if tp else float('nan'):.0f} |")


if __name__ == "__main__":
    main()
