"""Per-function / per-op-kind time breakdown of one out-of-core step from the
executor's CUDA-event timeline (not part of the product)."""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="r18", help="r18 | r50 | any bench.py --config")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--budget-frac", type=float, default=0.25)
    ap.add_argument("--mode", default="va")
    ap.add_argument("--incore", action="store_true")
    a = ap.parse_args()
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from synth import nets
    if a.config in ("r18", "r50"):
        spec = nets.resnet(18 if a.config == "r18" else 50, batch=a.batch)
    else:
        class _A:
            config, batch = a.config, a.batch
        spec = bench.spec_for(_A())
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    F = G.in_core_peak()
    budget = F if a.incore else int(F * a.budget_frac)
    st, W, phys = bench.setup_step(spec, info, doc, budget, a.mode, 2 << 20, timeline=True,
                                   window=0 if a.incore else None)
    for _ in range(3):
        m = st.step()
    tl = st.timeline()
    kind = {f["id"]: f["op"]["kind"] for f in json.loads(doc)["functions"]}
    per = defaultdict(float)
    cnt = defaultdict(int)
    fns = []
    for ev in tl:
        if ev["stream"] == "compute":
            d = ev["t1"] - ev["t0"]
            per[kind[ev["id"]]] += d
            cnt[kind[ev["id"]]] += 1
            fns.append((d, ev["id"]))
    print(json.dumps({"step_ms": m["step_ms"], "compute_busy_ms": m["compute_busy_ms"], "overlap": m["overlap_frac"],
                      "h2d_busy": m["h2d_busy_ms"], "d2h_busy": m["d2h_busy_ms"]}))
    for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
        print(f"{k:22s} {v:8.2f} ms  n={cnt[k]}")
    for d, f in sorted(fns, reverse=True)[:25]:
        print(f"  {d:7.3f} ms  {f}")
    st.close()


if __name__ == "__main__":
    main()
