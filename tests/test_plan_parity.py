"""Parity of the C-ABI planner (liboocore.so: oc_plan_schedule and helpers)
with the CPU oracle — bit-exact canonical schedule bytes, window ends,
feasibility boundaries and allocator-replay integers — on the golden
examples, >= 1000 seeded random graphs and the model graphs.  Also checks that
the library loads without a GPU and exports every symbol of include/oocore.h."""
import hashlib
import json
import os
import re

import pytest

from oracle import allocators, graph, scheduler
from paper_2010_14109_b200 import binding as B
from synth import graphs as sg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "schedule_examples.json")


def test_library_loads_and_exports_header_symbols():
    L = B.lib()
    assert L.oc_abi_version() == 1
    hdr = open(os.path.join(ROOT, "include", "oocore.h")).read()
    declared = set(re.findall(r"\b(oc_[a-z_0-9]+)\s*\(", hdr))
    declared = {d for d in declared if not d.endswith("_t")}
    for name in declared:
        assert hasattr(L, name), name
    assert set(B.exported_symbols()) == declared


def _both(doc, budget, window, mode="va", chunk=4, phys=None, align=1, distance=0):
    g = graph.load_graph(doc)
    seq = graph.build_sequence(g)
    G = B.Graph(doc)
    try:
        o = scheduler.build_schedule(g, seq, budget, window, distance=distance)
    except scheduler.InfeasibleBudget as e:
        with pytest.raises(B.OcError) as ei:
            G.plan(budget, window, B.OC_ALLOC_VA, chunk_bytes=1, phys_bytes=max(1, budget), distance=distance)
        assert ei.value.code == B.OC_E_INFEASIBLE_BUDGET
        assert ei.value.fn == e.fn and ei.value.needed == e.needed
        return None
    modes = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST, "first": B.OC_ALLOC_ARENA_FIRST}
    phys = phys if phys is not None else max(1, budget)
    s = G.plan(budget, window, modes[mode], chunk_bytes=chunk, phys_bytes=phys, align=align, allow_oom=True,
               distance=distance)
    assert s.json() == scheduler.canonical_json(o)
    assert s.window_ends() == o.r
    st, _ = allocators.replay(g, o, mode, chunk_bytes=chunk, phys_bytes=phys, align=align)
    cs = s.stats()
    if st["oom"] is None:
        assert s.oom is None
        assert cs["peak_phys"] == st["peak_phys"]
        if mode == "va":
            assert cs["if_peak"] == st["if_peak"] and cs["n_max"] == st["n_max"]
        else:
            assert cs["peak_alloc"] == st["peak_alloc"]
    else:
        assert s.oom is not None
        assert (cs["oom_fn"], cs["oom_var"], cs["oom_request"], cs["oom_free_bytes"]) == \
               (st["oom"]["fn"], st["oom"]["var"], st["oom"]["request"], st["oom"]["free_bytes"])
    return s


def test_golden_examples_parity():
    gold = json.load(open(GOLD))
    for ex in gold["examples"]:
        doc = json.dumps(ex["graph"])
        wins = ex.get("windows") or [{"window": ex["window"], "cases": ex["cases"]}]
        for w in wins:
            for c in w["cases"]:
                _both(doc, c["budget"], w["window"])
    ex = gold["examples"][1]
    a = ex["alloc"]
    for mode in ("best", "first"):
        _both(json.dumps(ex["graph"]), a["budget"], a["window"], mode=mode, phys=16, align=1)


def test_random_graphs_bit_exact():
    hashes = []
    for seed in range(1000):
        doc = sg.random_graph(seed, p_pinned=0.05)
        g = graph.load_graph(doc)
        total = sum(g.var_bytes)
        budget = max(1, total // (1 + seed % 4))
        window = (seed * 7919) % (total + 1)
        mode = ("va", "best", "first")[seed % 3]
        s = _both(doc, budget, window, mode=mode, chunk=1 + seed % 16, phys=budget + (seed % 7) * 8)
        if s is not None:
            hashes.append(hashlib.sha256(s.json().encode()).hexdigest())
    assert len(hashes) > 300


def test_prior_art_distance_windows_bit_exact():
    """F1 policies (vDNN d = 1, LMS-style fixed distance): canonical schedule
    bytes, window ends, replay integers and infeasibility identical to the
    oracle on 300 random graphs; min-feasible budgets identical."""
    n_ok = 0
    for seed in range(300):
        doc = sg.random_graph(seed, p_pinned=0.05)
        g = graph.load_graph(doc)
        total = sum(g.var_bytes)
        budget = max(1, total // (1 + seed % 4))
        d = 1 + seed % 4
        mode = ("va", "best", "first")[seed % 3]
        s = _both(doc, budget, 0, mode=mode, chunk=1 + seed % 16, phys=budget + (seed % 7) * 8, distance=d)
        n_ok += s is not None
        seq = graph.build_sequence(g)
        assert B.Graph(doc).min_feasible_budget(0, distance=d) == scheduler.min_feasible_budget(g, seq, 0,
                                                                                               distance=d)
    assert n_ok > 100


def test_feasibility_helpers_match_oracle():
    for seed in range(60):
        doc = sg.random_graph(seed, n_fns=20, n_vars=30, max_bytes=50, p_pinned=0.1)
        g = graph.load_graph(doc)
        seq = graph.build_sequence(g)
        G = B.Graph(doc)
        for W in (0, 17, 100, 10 ** 9):
            assert G.min_feasible_budget(W) == scheduler.min_feasible_budget(g, seq, W)
        B_ = max(scheduler.min_feasible_budget(g, seq, 0), sum(g.var_bytes) // 3)
        assert G.max_feasible_window(B_) == scheduler.max_feasible_window(g, seq, B_)
        assert G.in_core_peak() == graph.in_core_peak(g)
        assert G.footprint() == graph.footprint_stats(g)


def test_error_classification_matches_oracle():
    docs = ['{"variables": [', '[]',
            json.dumps({"variables": [{"id": "a", "bytes": 0}], "functions": [{"id": "f", "out": ["a"]}]}),
            json.dumps({"variables": [{"id": "a", "bytes": 1.5}], "functions": []}),
            json.dumps({"variables": [{"id": "a", "bytes": 1}], "functions": [{"id": "f", "in": ["a"]}]}),
            json.dumps({"variables": [{"id": "a", "bytes": 1}, {"id": "b", "bytes": 1}],
                        "functions": [{"id": "f", "in": ["b"], "out": ["a"]}, {"id": "g", "in": ["a"], "out": ["b"]}]}),
            json.dumps({"variables": [{"id": "a", "bytes": 1}], "functions": [{"id": "f", "in": [], "out": []}]})]
    for d in docs:
        with pytest.raises(graph.GraphError) as eo:
            graph.load_graph(d)
        with pytest.raises(B.OcError) as ec:
            B.Graph(d)
        assert ec.value.code == {"parse": B.OC_E_PARSE, "invalid": B.OC_E_INVALID}[eo.value.kind], d


def test_makespan_model_bit_exact():
    """oc_simulate reproduces oracle/simulator.py exactly: makespan
    and per-function stalls on 300 random graphs with random compute times and
    link parameters, copies of clean variables elided or not."""
    import numpy as np
    from oracle import simulator
    rng = np.random.default_rng(3)
    n_ok = 0
    for seed in range(300):
        doc = sg.random_graph(seed, p_pinned=0.05)
        g = graph.load_graph(doc)
        seq = graph.build_sequence(g)
        total = sum(g.var_bytes)
        budget = max(1, total // (1 + seed % 3))
        window = (seed * 31) % (total + 1)
        try:
            o = scheduler.build_schedule(g, seq, budget, window)
        except scheduler.InfeasibleBudget:
            continue
        s = B.Graph(doc).plan(budget, window, B.OC_ALLOC_ARENA_BEST, chunk_bytes=1, phys_bytes=budget * 8,
                              allow_oom=True)
        fn_ms = [float(x) for x in rng.uniform(0.0, 3.0, g.n_fns)]
        h2d, d2h = float(rng.uniform(1e-7, 1e-5)), float(rng.uniform(1e-7, 1e-5))
        hu, du = float(rng.uniform(0, 5)), float(rng.uniform(0, 5))
        elide = bool(seed % 2)
        ref = simulator.simulate(g, seq, o, fn_ms, h2d, d2h, hu, du, elide)
        got = s.simulate(fn_ms, h2d, d2h, hu, du, elide)
        assert got["makespan_ms"] == ref["makespan_ms"], seed
        assert got["stall_per_fn_ms"] == ref["stall_ms"], seed
        n_ok += 1
    assert n_ok > 100


def test_executor_makespan_model_bit_exact():
    """oc_simulate model 1 (placement-aware executor ordering) reproduces
    oracle/simulator.simulate_exec exactly, with the allocator placements of
    the VA and best-fit replays."""
    import numpy as np
    from oracle import simulator
    rng = np.random.default_rng(4)
    n_ok = 0
    for seed in range(300):
        doc = sg.random_graph(seed, p_pinned=0.05)
        g = graph.load_graph(doc)
        seq = graph.build_sequence(g)
        total = sum(g.var_bytes)
        budget = max(1, total // (1 + seed % 3))
        window = (seed * 17) % (total + 1)
        try:
            o = scheduler.build_schedule(g, seq, budget, window)
        except scheduler.InfeasibleBudget:
            continue
        mode = ("va", "best")[seed % 2]
        chunk, phys = 1 + seed % 5, total * 4
        st, pl = allocators.replay(g, o, mode, chunk_bytes=chunk, phys_bytes=phys, align=1)
        if st["oom"] is not None:
            continue
        s = B.Graph(doc).plan(budget, window, B.OC_ALLOC_VA if mode == "va" else B.OC_ALLOC_ARENA_BEST,
                              chunk_bytes=chunk, phys_bytes=phys, align=1)
        fn_ms = [float(x) for x in rng.uniform(0.0, 3.0, g.n_fns)]
        h2d, d2h = float(rng.uniform(1e-7, 1e-5)), float(rng.uniform(1e-7, 1e-5))
        elide = bool(seed % 3)
        ref = simulator.simulate_exec(g, seq, o, pl, mode, fn_ms, h2d, d2h, 1.0, 2.0, elide, align=1)
        got = s.simulate(fn_ms, h2d, d2h, 1.0, 2.0, elide, model=1)
        assert got["makespan_ms"] == ref["makespan_ms"], seed
        assert got["stall_per_fn_ms"] == ref["stall_ms"], seed
        n_ok += 1
    assert n_ok > 100
