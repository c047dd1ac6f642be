"""Knob sweeps of the out-of-core step on one GPU: schedule
window W, allocator mode (VA chunk size / best-fit arena) and budget fraction.
Prints one JSON line per point.  Not part of the product."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="r18")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--fracs", default="0.25")
    ap.add_argument("--wfracs", default="0,0.25,0.5,0.75,1.0")
    ap.add_argument("--modes", default="va")
    ap.add_argument("--chunks", default="2")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--packs", default="65536", help="pack/unpack thresholds in bytes (0 = copy engines only)")
    ap.add_argument("--pin-below", type=int, default=0, help="pin variables smaller than this (bytes, Z26)")
    ap.add_argument("--distances", default="", help="also run the prior-art function-distance windows (F1), e.g. 1,2,4")
    ap.add_argument("--triggers", default="0", help="arrival triggers: 0 = at memory release (executor), "
                                                     "1 = the paper's f_{i-1} boundary (P:91); e.g. 0,1")
    a = ap.parse_args()
    import numpy as np
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from synth import nets
    if a.config == "r1001":
        spec = nets.preact_resnet(1001, batch=a.batch)
    else:
        spec = nets.resnet(18 if a.config == "r18" else 50, batch=a.batch)
    doc, info = graphs.build(spec, params="persistent", pin_below=a.pin_below)
    G = B.Graph(doc)
    F = G.in_core_peak()
    for frac in [float(x) for x in a.fracs.split(",")]:
        budget = int(F * frac)
        try:
            wmax = G.max_feasible_window(budget)
        except B.OcError as e:
            print(json.dumps({"frac": frac, "infeasible": str(e)}), flush=True)
            continue
        for mode in a.modes.split(","):
            for ch in [int(c) for c in a.chunks.split(",")]:
                runs = [(float(x), int(p), 0) for x in a.wfracs.split(",") for p in a.packs.split(",")]
                runs += [(0.0, int(a.packs.split(",")[0]), int(d)) for d in a.distances.split(",") if d]
                runs = [r + (int(t),) for r in runs for t in a.triggers.split(",")]
                for wf, pk, dd, trg in runs:
                    W = int(wmax * wf)
                    try:
                        st, W, phys = bench.setup_step(spec, info, doc, budget, mode, ch << 20, timeline=True,
                                                       window=W, pack=pk, distance=dd, trigger=trg)
                    except Exception as e:  # noqa: BLE001
                        print(json.dumps({"frac": frac, "mode": mode, "chunk_mib": ch, "wfrac": wf, "distance": dd,
                                          "error": str(e)[:200]}), flush=True)
                        continue
                    st.step()
                    ms = [st.step() for _ in range(a.steps)]
                    m = {k: float(np.mean([x[k] for x in ms])) for k in ("step_ms", "compute_busy_ms", "h2d_busy_ms",
                                                                         "d2h_busy_ms", "overlap_frac", "bytes_h2d",
                                                                         "bytes_d2h", "n_h2d", "n_d2h")}
                    mem = st.mem_stats()
                    # F4: the makespan model on this schedule with this run's per-function times
                    fid = [f["id"] for f in json.loads(doc)["functions"]]
                    dur = {}
                    for ev in st.timeline():
                        if ev["stream"] == "compute":
                            dur[ev["id"]] = dur.get(ev["id"], 0.0) + (ev["t1"] - ev["t0"])
                    fm = [dur.get(f, 0.0) for f in fid]
                    bh = m["bytes_h2d"] / max(m["h2d_busy_ms"], 1e-9) / 1e6 or 55.6
                    bd = m["bytes_d2h"] / max(m["d2h_busy_ms"], 1e-9) / 1e6 or 57.3
                    m["predicted_ms"] = st.sched.simulate(fm, bh, bd, 0.0, 0.0, True, model=1)["makespan_ms"]
                    m["predicted_boundary_ms"] = st.sched.simulate(fm, bh, bd, 0.0, 0.0, True)["makespan_ms"]
                    print(json.dumps({"frac": frac, "budget": budget, "mode": mode, "chunk_mib": ch, "wfrac": wf,
                                      "pack": pk, "policy": "paper" if not dd else f"distance {dd}",
                                      "trigger": ("release", "paper")[trg],
                                      "window": W, "phys": phys, "samples_per_s": a.batch / m["step_ms"] * 1e3,
                                      **m, "peak_phys": st.stats["peak_phys"], "if_peak": st.stats["if_peak"],
                                      "map_us_total": mem["map_us"]}), flush=True)
                    st.close()


if __name__ == "__main__":
    main()
