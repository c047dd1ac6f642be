"""Table-1 / Fig.3-shaped sweep on B200 (Table 1 P:127-143,
Fig.3; --net densenet|deeplab|pix2pix: the Fig.4/5 families): ResNet-50 224², batch swept at Table 1's batch/190 ratios
around the in-core maximum b0 under a fixed physical memory B_p, three rows:
  in-core      (no swapping; only batches whose in-core footprint fits B_p)
  schedule     window schedule + caching best-fit arena (the frameworks' default)
  schedule+VA  window schedule + VA chunk pool
For the swapping rows the scheduler budget B_s is the largest one whose
allocator replay fits B_p ("maximum defined memory budget", Fig.3 blue line),
found by bisection with the C-ABI planner; 'x' marks batches no budget fits.
One JSON line per (batch, row).  Not part of the product."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

RATIOS = [64 / 190, 128 / 190, 1.0, 256 / 190, 512 / 190, 928 / 190, 1120 / 190, 1248 / 190, 1440 / 190]


def max_budget(G, phys, mode, chunk, W=0):
    """Largest scheduler budget whose allocator replay fits `phys` (Fig.3 blue line)."""
    from paper_2010_14109_b200 import binding as B
    m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST}[mode]
    lo = G.min_feasible_budget(W)
    if lo > phys:
        return None, None
    def fits(b):
        s = G.plan(b, W, m, chunk_bytes=chunk, phys_bytes=phys, allow_oom=True)
        st = s.stats()
        return st["oom_fn"] < 0, st
    ok, st = fits(lo)
    if not ok:
        return None, None
    hi = phys
    best = (lo, st)
    while hi - lo > (1 << 24):
        mid = (lo + hi) // 2
        ok, st = fits(mid)
        if ok:
            lo, best = mid, (mid, st)
        else:
            hi = mid
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=50)
    ap.add_argument("--net", default="resnet", choices=["resnet", "densenet", "deeplab", "pix2pix"],
                    help="resnet (Table 1) or the paper's Fig.4/5 families (SURVEY F3)")
    ap.add_argument("--phys-gib", type=float, default=8.0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--chunk-mib", type=int, default=40)
    ap.add_argument("--ratios", default="")
    ap.add_argument("--rows", default="incore,best,va")
    a = ap.parse_args()
    import torch
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from synth import nets
    phys = int(a.phys_gib * (1 << 30))
    chunk = a.chunk_mib << 20
    make = {"resnet": lambda b: nets.resnet(a.depth, batch=b), "densenet": lambda b: nets.densenet(batch=b),
            "deeplab": lambda b: nets.deeplabv3plus(batch=b), "pix2pix": lambda b: nets.pix2pixhd(batch=b)}[a.net]
    b0 = bench.trainable_batch(make, phys)
    print(json.dumps({"b0_in_core_max": b0, "phys_bytes": phys, "chunk_bytes": chunk}), flush=True)
    ratios = [float(r) for r in a.ratios.split(",")] if a.ratios else RATIOS
    for r in ratios:
        b = max(1, int(round(b0 * r)))
        spec = make(b)
        doc, info = graphs.build(spec, params="persistent")
        G = B.Graph(doc)
        F = G.in_core_peak()
        for row in a.rows.split(","):
            rec = {"batch": b, "ratio": round(r, 3), "row": row, "F_peak": F}
            if row == "incore":
                # no swapping: parameters/gradients/momentum device-resident
                doc_i, info_i = graphs.build(spec, params="pinned")
                Fi = B.Graph(doc_i).in_core_peak()
                rec["F_peak"] = Fi
                if Fi > phys:
                    rec["result"] = "x"
                    print(json.dumps(rec), flush=True)
                    continue
                budget, W, mode, ph = Fi, 0, "best", Fi
            else:
                mode = row
                budget, st = max_budget(G, phys, mode, chunk)
                if budget is None:
                    rec["result"] = "x"
                    print(json.dumps(rec), flush=True)
                    continue
                W, ph = 0, phys
                rec.update(budget_sched=budget, peak_phys_replay=st["peak_phys"], if_peak=st["if_peak"])
            try:
                t0 = time.time()
                d_, i_ = (doc_i, info_i) if row == "incore" else (doc, info)
                stp, W, phys_used = bench.setup_step(spec, i_, d_, budget, "va" if mode == "va" else "best", chunk,
                                                     timeline=False, window=W)
                stp.step()
                ms = [stp.step()["step_ms"] for _ in range(a.steps)]
                rec.update(result="ok", samples_per_s=b / (sum(ms) / len(ms)) * 1e3, step_ms=sum(ms) / len(ms),
                           phys_pool=phys_used, bytes_h2d=stp.stats["bytes_h2d"], bytes_d2h=stp.stats["bytes_d2h_dirty"],
                           setup_s=time.time() - t0)
                stp.close()
            except Exception as e:  # noqa: BLE001
                rec.update(result="error", error=str(e)[:300])
            torch.cuda.empty_cache()
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
