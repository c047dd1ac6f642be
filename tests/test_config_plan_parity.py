"""Schedule and allocator-replay bit-exactness, C-ABI planner vs CPU oracle, on
the ACTUAL config graphs the bench and the Table-1 sweep run (north_star:
"the schedule bit-exact to the CPU oracle"): canonical schedule bytes
(SHA-256), window ends, F_peak and the replay integers (peak_phys, IF_peak,
N_max, or the OOM point) of the VA pool and the best-/first-fit arenas.

  configs[1]  ResNet-18 224^2 b=256, tensors < 1 MiB pinned, 25 % of F_peak
  configs[2]  ResNet-50 224^2 at Table 1's batches (b0 = 202 under 8 GiB) at
              the scheduler budget the sweep bisects for B_p = 8 GiB
  configs[3]  U-Net 1024^2 b=8 at F_peak/8
  configs[4]  pre-activation ResNet-1001 b=256 (tensors < 2 MiB pinned) and
              the BigGAN-style GAN step b=32, F_peak/4
Windows: 0, half the largest feasible, the largest feasible.
"""
import hashlib

import pytest

from oracle import allocators, graph, scheduler
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20
GiB = 1 << 30
MODES = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST, "first": B.OC_ALLOC_ARENA_FIRST}


def _check(doc, budget, windows, allocs, phys):
    g = graph.load_graph(doc)
    seq = graph.build_sequence(g)
    G = B.Graph(doc)
    assert G.in_core_peak() == graph.in_core_peak(g)
    assert G.footprint() == graph.footprint_stats(g)
    n = 0
    for W in windows:
        o = scheduler.build_schedule(g, seq, budget, W)
        ref = scheduler.canonical_json(o)
        for mode, chunk in allocs:
            s = G.plan(budget, W, MODES[mode], chunk_bytes=chunk, phys_bytes=phys, align=512, allow_oom=True)
            got = s.json()
            assert hashlib.sha256(got.encode()).hexdigest() == hashlib.sha256(ref.encode()).hexdigest(), (W, mode)
            assert s.window_ends() == o.r
            st, _ = allocators.replay(g, o, mode, chunk_bytes=chunk, phys_bytes=phys, align=512)
            cs = s.stats()
            if st["oom"] is None:
                assert cs["oom_fn"] < 0
                assert cs["peak_phys"] == st["peak_phys"]
                if mode == "va":
                    assert (cs["if_peak"], cs["n_max"]) == (st["if_peak"], st["n_max"])
                else:
                    assert cs["peak_alloc"] == st["peak_alloc"]
            else:
                assert (cs["oom_fn"], cs["oom_var"], cs["oom_request"], cs["oom_free_bytes"]) == \
                       (st["oom"]["fn"], st["oom"]["var"], st["oom"]["request"], st["oom"]["free_bytes"])
            n += 1
    return n


def _windows(G, budget):
    wmax = G.max_feasible_window(budget)
    return [0, wmax // 2, wmax]


def test_r18_bench_graph():
    doc, _ = graphs.build(nets.resnet(18, batch=256), params="persistent", inputs="host", pin_below=MiB)
    G = B.Graph(doc)
    budget = G.in_core_peak() // 4
    allocs = [("va", 2 * MiB), ("va", 40 * MiB), ("best", 2 * MiB), ("first", 2 * MiB)]
    assert _check(doc, budget, _windows(G, budget), allocs, phys=budget) == 12


def _max_budget(G, phys, mode, chunk):
    """Largest scheduler budget whose replay fits phys (the sweep's bisection)."""
    lo, hi = G.min_feasible_budget(0), phys
    while hi - lo > (1 << 24):
        mid = (lo + hi) // 2
        if G.plan(mid, 0, MODES[mode], chunk_bytes=chunk, phys_bytes=phys, allow_oom=True).stats()["oom_fn"] < 0:
            lo = mid
        else:
            hi = mid
    return lo


@pytest.mark.parametrize("batch", [68, 202, 544, 987, 1191, 1531])
def test_r50_table1_graphs(batch):
    doc, _ = graphs.build(nets.resnet(50, batch=batch), params="persistent")
    G = B.Graph(doc)
    phys = 8 * GiB
    for mode, chunk in (("va", 2 * MiB), ("best", 2 * MiB)):
        budget = _max_budget(G, phys, mode, chunk)
        _check(doc, budget, [0], [(mode, chunk), ("first", chunk), ("va", 40 * MiB)], phys)


def test_unet_1024_graph():
    doc, _ = graphs.build(nets.unet(batch=8, image=1024), params="persistent")
    G = B.Graph(doc)
    budget = G.in_core_peak() // 8
    _check(doc, budget, _windows(G, budget), [("va", 2 * MiB), ("best", 2 * MiB)], phys=budget)


def test_r1001_graph():
    doc, _ = graphs.build(nets.preact_resnet(1001, batch=256), params="persistent", pin_below=2 * MiB)
    G = B.Graph(doc)
    budget = G.in_core_peak() // 4
    _check(doc, budget, [0, G.max_feasible_window(budget)], [("va", 2 * MiB), ("best", 2 * MiB)], phys=budget)


def test_biggan_graph():
    doc, _ = graphs.build(nets.biggan(batch=32), params="persistent")
    G = B.Graph(doc)
    budget = G.in_core_peak() // 4
    _check(doc, budget, _windows(G, budget), [("va", 2 * MiB), ("va", 40 * MiB), ("best", 2 * MiB)], phys=budget)
