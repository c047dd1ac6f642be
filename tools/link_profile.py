"""Per-transfer copy rates of one instrumented out-of-core ResNet-18 step
(bench config: b=256, 25 % budget, W=0, VA 2 MiB): bytes and busy time per
size bucket, and the gaps on each copy stream.  Not part of the product."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from synth import nets
    spec = nets.resnet(18, batch=256)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    budget = G.in_core_peak() // 4
    st, W, phys = bench.setup_step(spec, info, doc, budget, "va", 2 << 20, timeline=True, window=0)
    for _ in range(3):
        m = st.step()
    tl = st.timeline()
    size = {v["id"]: v["bytes"] for v in json.loads(doc)["variables"]}
    for stream in ("h2d", "d2h"):
        ev = sorted((e for e in tl if e["stream"] == stream), key=lambda e: e["t0"])
        buckets = {}
        for e in ev:
            b = size.get(e["id"], 0)
            k = "<1MB" if b < 1e6 else "1-10MB" if b < 1e7 else "10-100MB" if b < 1e8 else ">100MB"
            a = buckets.setdefault(k, [0, 0.0, 0])
            a[0] += b
            a[1] += e["t1"] - e["t0"]
            a[2] += 1
        gaps = [ev[i + 1]["t0"] - ev[i]["t1"] for i in range(len(ev) - 1)]
        print(stream, "copies", len(ev), "span ms %.2f" % (ev[-1]["t1"] - ev[0]["t0"]),
              "busy ms %.2f" % sum(e["t1"] - e["t0"] for e in ev), "gaps>0 ms %.2f" % sum(g for g in gaps if g > 0))
        for k, (b, t, n) in sorted(buckets.items()):
            print("   %-9s n=%4d  %8.1f MB  %7.2f ms  %6.1f GB/s" % (k, n, b / 1e6, t, b / t / 1e6 if t else 0))
    print("step ms", m["step_ms"], "compute busy", m["compute_busy_ms"])
    st.close()


if __name__ == "__main__":
    main()
