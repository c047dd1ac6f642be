"""Time the attention core (attn_fwd / attn_bwd, bf16) at the BigGAN step's
shapes through the C-ABI, one function per step, and print ms per sample and
the algorithmic HBM bytes rate (S or dP written + read as fp32, P written /
read as bf16).  Run under ncu for the per-kernel split.
Not part of the product.

Usage: python tools/attn_probe.py [--n 4 --L 4096 --dq 24 --dv 96 --reps 5]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--dq", type=int, default=24)
    ap.add_argument("--dv", type=int, default=96)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    N, L, dq, dv = a.n, a.L, a.dq, a.dv
    sizes = {"q": N * L * dq, "k": N * L * dq, "v": N * L * dv, "p": N * L * L, "o": N * L * dv, "do": N * L * dv,
             "dq": N * L * dq, "dk": N * L * dq, "dv": N * L * dv}
    out = {}
    for kind in ("attn_fwd", "attn_bwd"):
        names = ["q", "k", "v", "p", "o"] + (["do", "dq", "dk", "dv"] if kind == "attn_bwd" else [])
        outs = ["p", "o"] if kind == "attn_fwd" else ["dq", "dk", "dv"]
        vars_ = [{"id": n, "bytes": sizes[n] * 2, "persistent": True} for n in names]
        fn = {"id": "f", "in": [n for n in names if n not in outs], "out": outs,
              "op": {"kind": kind, "args": {n: n for n in names},
                     "attrs": {"dtype": "bf16", "N": N, "L": L, "dq": dq, "dv": dv, "n0": 0, "nb": N}}}
        doc = json.dumps({"variables": vars_, "functions": [fn]})
        total = sum(v["bytes"] for v in vars_) + (1 << 30)
        st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=total)
        rng = np.random.default_rng(0)
        for n in names:
            if n not in outs:
                st.write(n, torch.from_numpy(rng.standard_normal(sizes[n]).astype(np.float32) * 0.3)
                         .to(torch.bfloat16).view(torch.int16).numpy())
        st.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            st.step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        st.close()
        LL = N * L * L
        byt = LL * 4 * 2 + LL * 2 * 2 if kind == "attn_fwd" else LL * 4 * 6 + LL * 2 * 2
        out[kind] = {"ms": round(ms, 3), "ms_per_sample": round(ms / N, 4), "algo_GBs": round(byt / ms / 1e6, 1)}
    print(json.dumps({"N": N, "L": L, "dq": dq, "dv": dv, **out}))


if __name__ == "__main__":
    main()
