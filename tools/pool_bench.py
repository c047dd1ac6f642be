"""Per-kernel timing of the stem BN-ReLU-maxpool ops (bn_relu_pool_fwd with
fused statistics, pool_bn_bwd_reduce, pool_bn_bwd_apply) at the ResNet stem
shape (112×112×64 bf16, 3×3/2 pool): one-function graphs through the C-ABI
executor, device-resident operands, CUDA events around each step; GB/s of
ALGORITHMIC bytes (each operand read or written once) against the measured HBM
peak.  Used with ncu for the kernel roofline.  Not part of the product."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graph(kind, N, H=112, W=112, C=64):
    P, Q = H // 2, W // 2
    at = {"dtype": "bf16", "N": N, "H": H, "W": W, "C": C, "r": 3, "stride": 2, "pad": 1, "P": P, "Q": Q}
    ys, ps, ix = N * H * W * C * 2, N * P * Q * C * 2, N * P * Q * C
    v = lambda n, b: {"id": n, "bytes": int(b), "pinned": True}
    prm = [v("gamma", C * 4), v("beta", C * 4), v("stat", 2 * C * 4)]
    if kind == "fwd":
        vs = [v("y", ys), v("out", ps), v("idx", ix)] + prm
        args = {"y": "y", "stat": "stat", "gamma": "gamma", "beta": "beta", "out": "out", "idx": "idx"}
        fn = {"id": "f", "in": ["y", "gamma", "beta", "stat"], "out": ["out", "idx"],
              "op": {"kind": "bn_relu_pool_fwd", "args": args, "attrs": dict(at, stat_in=True)}}
        alg = ys + ps + ix
    else:
        vs = [v("y", ys), v("g", ps), v("idx", ix), v("dgamma", C * 4), v("dbeta", C * 4)] + prm
        args = {"g": "g", "idx": "idx", "y": "y", "stat": "stat", "gamma": "gamma", "beta": "beta",
                "dgamma": "dgamma", "dbeta": "dbeta"}
        if kind == "reduce":
            fn = {"id": "f", "in": ["g", "idx", "y", "stat", "gamma", "beta"], "out": ["dgamma", "dbeta"],
                  "op": {"kind": "pool_bn_bwd_reduce", "args": args, "attrs": at}}
            alg = ys + ps + ix
        else:
            fn = {"id": "f", "in": ["g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta"], "out": ["y"],
                  "op": {"kind": "pool_bn_bwd_apply", "args": args, "attrs": at}}
            alg = 2 * ys + ps + ix
    doc = json.dumps({"variables": vs, "functions": [fn]})
    return doc, sum(x["bytes"] for x in vs), alg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--kinds", default="fwd,reduce,apply")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs", 6549.8)
    for kind in a.kinds.split(","):
        doc, total, alg = graph(kind, a.batch)
        st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
        rng = np.random.default_rng(0)
        for vname, t in st.dev.items():
            if vname == "stat":
                s = np.concatenate([rng.standard_normal(64) * 0.1, 1.0 + rng.random(64)]).astype(np.float32)
                t.view(torch.float32).copy_(torch.from_numpy(s))
            elif vname in ("gamma", "beta", "dgamma", "dbeta"):
                t.view(torch.float32).copy_(torch.from_numpy(rng.standard_normal(64).astype(np.float32)))
            elif vname == "idx":
                t.copy_(torch.from_numpy(rng.integers(0, 9, t.numel(), dtype=np.uint8)))
            else:
                t.view(torch.bfloat16).copy_(torch.from_numpy(rng.standard_normal(t.numel() // 2).astype(np.float32)))
        st.step()
        ms = float(np.median([st.step()["step_ms"] for _ in range(a.reps)]))
        print(json.dumps({"kind": kind, "batch": a.batch, "ms": ms, "alg_bytes": alg, "gbs": alg / ms / 1e6,
                          "frac_of_hbm": alg / ms / 1e6 / hbm}), flush=True)
        st.close()


if __name__ == "__main__":
    main()
