"""Per-kernel timing of the convolution ops at the ResNet-18 b=256 layer
shapes (one-function graphs through the C-ABI executor, device-resident
operands, CUDA events around each step): TFLOP/s and fraction of the measured
bf16 peak per (shape, pass).  Used with ncu for the kernel roofline.  Not part
of the product."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {  # name: N, H, W, C, K, R, stride, pad
    "stem7x7s2": (256, 224, 224, 3, 64, 7, 2, 3),
    "l1_3x3": (256, 56, 56, 64, 64, 3, 1, 1),
    "l2_3x3s2": (256, 56, 56, 64, 128, 3, 2, 1),
    "l2_3x3": (256, 28, 28, 128, 128, 3, 1, 1),
    "l2_1x1s2": (256, 56, 56, 64, 128, 1, 2, 0),
    "l3_3x3": (256, 14, 14, 256, 256, 3, 1, 1),
    "l4_3x3": (256, 7, 7, 512, 512, 3, 1, 1),
}
# ResNet-50 bottleneck 1x1 shapes (b = 256): short reductions, wide outputs
R50 = {
    "r50_1x1_64_256": (256, 56, 56, 64, 256, 1, 1, 0),
    "r50_1x1_256_64": (256, 56, 56, 256, 64, 1, 1, 0),
    "r50_1x1_1024_256": (256, 14, 14, 1024, 256, 1, 1, 0),
    "r50_1x1_512_2048": (256, 7, 7, 512, 2048, 1, 1, 0),
    "r50_3x3_128": (256, 28, 28, 128, 128, 3, 1, 1),
}
SHAPES_ALL = {**SHAPES, **R50}


def graph(kind, s):
    N, H, W, C, K, R, st, pad = s
    P = (H + 2 * pad - R) // st + 1
    Q = (W + 2 * pad - R) // st + 1
    at = {"dtype": "bf16", "N": N, "H": H, "W": W, "C": C, "K": K, "R": R, "S": R, "stride": st, "pad": pad,
          "P": P, "Q": Q}
    xs, ys, ws = N * H * W * C * 2, N * P * Q * K * 2, K * R * R * C * 4
    v = lambda n, b: {"id": n, "bytes": int(b), "pinned": True}
    if kind == "fprop":
        vs, args, ins, outs = [v("x", xs), v("w", ws), v("y", ys)], {"x": "x", "w": "w", "y": "y"}, ["x", "w"], ["y"]
        op = "conv_fwd"
    elif kind == "dgrad":
        vs, args, ins, outs = [v("dy", ys), v("w", ws), v("dx", xs)], {"dy": "dy", "w": "w", "dx": "dx"}, ["dy", "w"], ["dx"]
        op = "conv_dgrad"
    elif kind == "dgrad_acc":   # dx = rnd(dx + dgrad): the residual-gradient accumulation of a bottleneck
        vs, args, ins, outs = [v("dy", ys), v("w", ws), v("dx", xs)], {"dy": "dy", "w": "w", "dx": "dx"}, ["dy", "w", "dx"], ["dx"]
        op = "conv_dgrad"
        at = dict(at, accumulate=True)
    else:
        vs, args, ins, outs = [v("dy", ys), v("x", xs), v("dw", ws)], {"dy": "dy", "x": "x", "dw": "dw"}, ["dy", "x"], ["dw"]
        op = "conv_wgrad"
    doc = json.dumps({"variables": vs, "functions": [{"id": "f", "in": ins, "out": outs,
                                                       "op": {"kind": op, "args": args, "attrs": at}}]})
    return doc, sum(x["bytes"] for x in vs), 2.0 * N * P * Q * K * R * R * C


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=",".join(SHAPES))
    ap.add_argument("--passes", default="fprop,dgrad,wgrad")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = peaks.get("bf16_tflops", 1642.7)
    for name in a.shapes.split(","):
        for kind in a.passes.split(","):
            if name.startswith("stem") and kind.startswith("dgrad"):
                continue
            doc, total, flops = graph(kind, SHAPES_ALL[name])
            st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
            rng = np.random.default_rng(0)
            for vname, t in st.dev.items():
                if vname in ("w",):
                    t.view(torch.float32).copy_(torch.from_numpy(rng.standard_normal(t.numel() // 4).astype(np.float32) * 0.05))
                elif vname in ("x", "dy", "dx"):
                    t.view(torch.bfloat16).copy_(torch.from_numpy(rng.standard_normal(t.numel() // 2).astype(np.float32)))
            st.step()
            ms = float(np.median([st.step()["step_ms"] for _ in range(a.reps)]))
            print(json.dumps({"shape": name, "pass": kind, "ms": ms, "tflops": flops / ms / 1e9,
                              "frac_of_burst_peak": flops / ms / 1e9 / peak}), flush=True)
            st.close()


if __name__ == "__main__":
    main()
