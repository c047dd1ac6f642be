"""Pins of the makespan model (oracle/simulator.py):
closed-form single-function and perfect-overlap cases, the lower
bounds and the causality / channel-exclusivity audit of the event timeline on
random graphs, and the no-transfer case (W = budget = footprint)."""
import json

import numpy as np

from oracle import graph, scheduler, simulator
from synth import graphs as sg


def _load(doc):
    g = graph.load_graph(doc if isinstance(doc, str) else json.dumps(doc))
    seq = graph.build_sequence(g)
    scheduler.attach_bytes(g, seq)
    return g, seq


def test_single_function_serial_lower_bound():
    """One function reading one 8-byte persistent variable: load + compute."""
    g, seq = _load({"variables": [{"id": "a", "bytes": 8, "persistent": True}],
                    "functions": [{"id": "f", "in": ["a"], "out": []}]})
    sch = scheduler.build_schedule(g, seq, 8, 0)
    r = simulator.simulate(g, seq, sch, [8e-6], h2d_gbs=1.0, d2h_gbs=1.0)   # 1 GB/s: 1 B per 1e-6 ms
    assert np.isclose(r["makespan_ms"], 8e-6 + 8e-6)


def test_prefetch_hides_the_transfer():
    """f1 computes 8 units while f2's 8-byte input arrives (window covers it):
    f2 does not stall."""
    doc = {"variables": [{"id": "a", "bytes": 1, "persistent": True}, {"id": "b", "bytes": 8, "persistent": True}],
           "functions": [{"id": "f1", "in": ["a"], "out": []}, {"id": "f2", "in": ["b"], "out": []}]}
    g, seq = _load(doc)
    sch = scheduler.build_schedule(g, seq, 9, 100)       # everything arrives at f1
    r = simulator.simulate(g, seq, sch, [9e-6, 1e-6], h2d_gbs=1.0, d2h_gbs=1.0)
    assert r["stall_ms"][1] == 0.0
    assert np.isclose(r["makespan_ms"], 1e-6 + 9e-6 + 1e-6)   # a's load, f1, f2


def test_bounds_causality_and_channel_exclusivity():
    """On 300 random graphs: makespan >= every lower bound; every event starts
    after its dependencies; the intervals on each copy channel are disjoint."""
    rng = np.random.default_rng(0)
    for seed in range(300):
        g, seq = _load(sg.random_graph(seed, p_pinned=0.05))
        total = sum(g.var_bytes)
        try:
            sch = scheduler.build_schedule(g, seq, max(1, total // 2), (seed * 13) % (total + 1))
        except scheduler.InfeasibleBudget:
            continue
        fn_ms = list(rng.uniform(0.0, 2.0, g.n_fns))
        r = simulator.simulate(g, seq, sch, fn_ms, h2d_gbs=1e-6, d2h_gbs=2e-6, h2d_us=0.1, d2h_us=0.2)
        lb = simulator.lower_bounds(g, sch, fn_ms, 1e-6, 2e-6)
        assert r["makespan_ms"] >= max(lb["compute"], lb["h2d"], lb["d2h"]) - 1e-9
        for ch in ("h2d", "d2h", "compute"):
            iv = sorted((s, e) for s, e, c, _ in r["events"] if c == ch)
            assert all(iv[k][1] <= iv[k + 1][0] + 1e-12 for k in range(len(iv) - 1)), (seed, ch)
        comp = {i: (s, e) for s, e, c, i in r["events"] if c == "compute"}
        h2d = iter([(e, v) for s, e, c, v in r["events"] if c == "h2d"])
        last = {}                 # var -> completion of its latest arrival so far
        for i in range(g.n_fns):
            for v, kind in sch.ins[i]:
                if kind == "h2d":
                    e, v2 = next(h2d)
                    assert v2 == v
                    last[v] = e
            for v in set(seq.occ[seq.l[i]:seq.e[i] + 1]):   # every input of f_i has arrived
                if v in last:
                    assert last[v] <= comp[i][0] + 1e-12, (seed, i, v)
            if i:
                assert comp[i - 1][1] <= comp[i][0]


def test_everything_resident_no_transfer_stalls():
    """Budget = window = footprint: only initial loads; with zero-cost links
    the makespan is the sum of compute times."""
    for seed in range(50):
        g, seq = _load(sg.random_graph(seed))
        total = sum(g.var_bytes)
        sch = scheduler.build_schedule(g, seq, total, 10 ** 12)
        fn_ms = [1.0] * g.n_fns
        r = simulator.simulate(g, seq, sch, fn_ms, h2d_gbs=1e12, d2h_gbs=1e12)
        assert abs(r["makespan_ms"] - g.n_fns) < 1e-6


def test_executor_model_bounded_by_boundary_model_and_lower_bounds():
    """The placement-aware (executor) model only removes the function-boundary
    gate of the arrivals — the memory it waits for was released no later
    than that boundary — so its makespan is never above the paper-semantics
    model's, and never below the lower bounds (300 random graphs, VA and
    best-fit placements)."""
    from oracle import allocators
    rng = np.random.default_rng(1)
    n_ok = 0
    for seed in range(300):
        g, seq = _load(sg.random_graph(seed, p_pinned=0.05))
        total = sum(g.var_bytes)
        budget = max(1, total // (1 + seed % 3))
        try:
            sch = scheduler.build_schedule(g, seq, budget, (seed * 7) % (total + 1))
        except scheduler.InfeasibleBudget:
            continue
        mode = ("va", "best")[seed % 2]
        st, pl = allocators.replay(g, sch, mode, chunk_bytes=2, phys_bytes=total * 4, align=1)
        if st["oom"] is not None:
            continue
        fn_ms = list(rng.uniform(0.0, 2.0, g.n_fns))
        args = (fn_ms, 1e-6, 2e-6, 0.1, 0.2, bool(seed % 3))
        a = simulator.simulate(g, seq, sch, *args)
        e = simulator.simulate_exec(g, seq, sch, pl, mode, *args, align=1)
        lb = simulator.lower_bounds(g, sch, fn_ms, 1e-6, 2e-6)
        assert e["makespan_ms"] <= a["makespan_ms"] + 1e-9, seed
        assert e["makespan_ms"] >= max(lb["compute"], lb["h2d"]) - 1e-9, seed
        n_ok += 1
    assert n_ok > 100


def test_greedy_makespan_never_beats_the_exhaustive_optimum():
    """on tiny graphs (<= 4 functions, <= 5 variables)
    the greedy's simulated makespan at every window is >= the minimum over
    all resident-set sequences, which itself is >= the lower bounds;
    the brute force finds a schedule exactly when the greedy does (Z11 at
    W = 0).  The gap is measured, not bounded (the paper claims no
    optimality)."""
    from oracle import bruteforce
    rng = np.random.default_rng(2)
    gaps = []
    for seed in range(60):
        g, seq = _load(sg.random_graph(seed, n_fns=4, n_vars=5, max_bytes=6, p_pinned=0.0))
        if sum(1 for v in range(g.n_vars) if not g.pinned[v]) > 5 or g.n_fns > 4:
            continue
        total = sum(g.var_bytes)
        fn_ms = list(rng.uniform(0.5, 2.0, g.n_fns))
        for B in (total // 2, total):
            opt = bruteforce.optimal_makespan(g, seq, B, fn_ms, 1e-6, 1e-6)
            try:
                g0 = scheduler.build_schedule(g, seq, B, 0)
            except scheduler.InfeasibleBudget:
                assert opt is None, (seed, B)
                continue
            assert opt is not None
            for W in (0, 3, 10 ** 9):
                try:
                    sch = scheduler.build_schedule(g, seq, B, W)
                except scheduler.InfeasibleBudget:
                    continue
                m = simulator.simulate(g, seq, sch, fn_ms, 1e-6, 1e-6)["makespan_ms"]
                assert m >= opt - 1e-9, (seed, B, W, m, opt)
                gaps.append(m / opt - 1.0)
            del g0
    assert gaps and min(gaps) >= -1e-9
