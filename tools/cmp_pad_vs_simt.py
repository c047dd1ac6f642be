import json, numpy as np, torch, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_conv import _graph, _run, bf, _bits, _from_bits
shapes = [(4, 4, 4, 16, 16, 3, 1, 1), (4, 4, 4, 16, 32, 3, 2, 1), (4, 4, 4, 16, 32, 1, 2, 0), (4, 2, 2, 32, 32, 3, 1, 1),
          (4, 8, 8, 16, 16, 3, 1, 1)]
for g in shapes:
    N, H, W, C, K, R, st, pad = g
    rng = np.random.default_rng(5)
    for kind in ("conv_fwd", "conv_dgrad", "conv_wgrad"):
        for acc in ((False, True) if kind == "conv_dgrad" else (False,)):
            doc, (P, Q), total = _graph(kind, g, acc)
            outs = []
            for impl in ("tc", "simt"):
                d = json.loads(doc)
                if impl == "simt":
                    d["functions"][0]["op"]["attrs"]["impl"] = "simt"
                rng = np.random.default_rng(5)
                w = rng.standard_normal((K, R, R, C)).astype(np.float32) * 0.1
                x = bf(rng.standard_normal((N, H, W, C)))
                dy = bf(rng.standard_normal((N, P, Q, K)))
                old = bf(rng.standard_normal((N, H, W, C)))
                if kind == "conv_fwd":
                    r = _run(json.dumps(d), total, {"x": _bits(x), "w": w}, "y", np.uint16); shp = (N, P, Q, K)
                elif kind == "conv_dgrad":
                    r = _run(json.dumps(d), total, {"dy": _bits(dy), "w": w, "dx": _bits(old)}, "dx", np.uint16); shp = (N, H, W, C)
                else:
                    r = _run(json.dumps(d), total, {"dy": _bits(dy), "x": _bits(x)}, "dw", np.float32); shp = (K, R, R, C)
                outs.append(_from_bits(r, shp) if r.dtype == np.uint16 else r.reshape(shp).astype(np.float64))
            a, b = outs
            diff = np.abs(a - b); rel = diff.max() / (np.abs(b).max() + 1e-12)
            print(g, kind, acc, "maxrel", float(rel), "frac_diff", float((diff > 0).mean()))
