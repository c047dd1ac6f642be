"""In-step vs isolated durations of the same contraction launches (round-1
review item: conv kernels ran ~1.8x longer inside the out-of-core step than in
isolation).  Runs one config's graph twice with per-launch probes
(oc_exec_timeline k_span_ms = in-kernel %globaltimer span, k_mhz = SM clock
from clock64 over the same span):
  ooc     the bench's out-of-core step (swaps on the copy engines and the pack
          kernels running next to compute)
  incore  the same batch in-core (no transfers at all)
and prints, per contraction kind, Σ algorithmic FLOPs / Σ spans in each, the
SM clock, and the event-timed durations (k_ms) beside the in-kernel spans.
Writes one JSON line (and per-function rows with --rows).  Not part of the
product."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

MiB = 1 << 20


def collect(st, steps=3):
    st.step()
    for _ in range(steps):
        st.step()
    return st.timeline()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="r18", choices=["r18", "r50"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--frac", type=float, default=0.27)
    ap.add_argument("--rows", action="store_true")
    ap.add_argument("--pack", type=int, default=64 << 10)
    a = ap.parse_args()
    import numpy as np
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from synth import nets
    depth = 18 if a.config == "r18" else 50
    spec = nets.resnet(depth, batch=a.batch or (256 if depth == 18 else 512))
    pin = MiB if depth == 18 else 0
    doc, info = graphs.build(spec, params="persistent", pin_below=pin)
    G = B.Graph(doc)
    budget = max(G.min_feasible_budget(0), int(G.in_core_peak() * a.frac))
    fl = bench.conv_flops(doc)
    st, W, phys = bench.setup_step(spec, info, doc, budget, "va", 2 * MiB, timeline=True, window=0, pack=a.pack)
    tl_o = collect(st)
    met_o = st.step()
    st.close()
    doc_p, info_p = graphs.build(spec, params="pinned")
    Gp = B.Graph(doc_p)
    Fp = Gp.in_core_peak()
    slab = Gp.plan(Fp, 0, B.OC_ALLOC_ARENA_BEST, chunk_bytes=2 * MiB, phys_bytes=1 << 50,
                   allow_oom=True).stats()["peak_phys"]
    st2 = bench.new_step(spec, info_p, doc_p, Fp, "best", 2 * MiB, slab, 0, timeline=True)
    tl_i = collect(st2)
    met_i = st2.step()
    st2.close()

    def per_fn(tl):
        return {e["id"]: e for e in tl if e["stream"] == "compute" and e["id"] in fl}
    po, pi = per_fn(tl_o), per_fn(tl_i)
    kinds = {}
    rows = []
    for fid, (kind, flops) in fl.items():
        if fid not in po or fid not in pi:
            continue
        o, i = po[fid], pi[fid]
        k = kinds.setdefault(kind, {"flops": 0.0, "ooc_span": 0.0, "inc_span": 0.0, "ooc_ev": 0.0, "inc_ev": 0.0,
                                    "ooc_clk": [], "inc_clk": []})
        k["flops"] += flops
        k["ooc_span"] += o.get("k_span_ms", 0.0)
        k["inc_span"] += i.get("k_span_ms", 0.0)
        k["ooc_ev"] += o.get("k_ms", 0.0)
        k["inc_ev"] += i.get("k_ms", 0.0)
        if o.get("k_mhz"):
            k["ooc_clk"].append(o["k_mhz"])
        if i.get("k_mhz"):
            k["inc_clk"].append(i["k_mhz"])
        rows.append({"fn": fid, "kind": kind, "ooc_span_ms": o.get("k_span_ms"), "inc_span_ms": i.get("k_span_ms"),
                     "ooc_ev_ms": o.get("k_ms"), "inc_ev_ms": i.get("k_ms"), "ooc_mhz": o.get("k_mhz"),
                     "inc_mhz": i.get("k_mhz")})
    out = {"config": a.config, "batch": spec["batch"], "budget": budget, "ooc_step_ms": met_o["step_ms"],
           "incore_step_ms": met_i["step_ms"], "kinds": {}}
    for kind, k in kinds.items():
        out["kinds"][kind] = {
            "tflops_ooc_span": k["flops"] / (k["ooc_span"] / 1e3) / 1e12 if k["ooc_span"] else None,
            "tflops_incore_span": k["flops"] / (k["inc_span"] / 1e3) / 1e12 if k["inc_span"] else None,
            "tflops_ooc_events": k["flops"] / (k["ooc_ev"] / 1e3) / 1e12 if k["ooc_ev"] else None,
            "tflops_incore_events": k["flops"] / (k["inc_ev"] / 1e3) / 1e12 if k["inc_ev"] else None,
            "span_ratio_ooc_over_incore": k["ooc_span"] / k["inc_span"] if k["inc_span"] else None,
            "sm_mhz_ooc_median": float(np.median(k["ooc_clk"])) if k["ooc_clk"] else None,
            "sm_mhz_incore_median": float(np.median(k["inc_clk"])) if k["inc_clk"] else None,
        }
    print(json.dumps(out), flush=True)
    if a.rows:
        for r in rows:
            print(json.dumps(r))


if __name__ == "__main__":
    main()
