"""Pins of the scheduler oracle (oracle/graph.py, oracle/scheduler.py,
oracle/validate.py) against things other than itself: the hand-derived
worked examples (tests/golden), the closed-form feasibility condition
max_i B_i(W) <= B (proof in DESIGN.md §4), special cases
(W = 0, W = ∞), brute force over all schedules (P:62 search space), and the
Fig.1 distance identity."""
import json
import os

import pytest

from oracle import bruteforce, graph, scheduler, validate
from synth import graphs as sg

GOLD = os.path.join(os.path.dirname(__file__), "golden", "schedule_examples.json")


def _load(doc):
    g = graph.load_graph(doc if isinstance(doc, str) else json.dumps(doc))
    return g, graph.build_sequence(g)


def _named(g, sch):
    n = g.var_names
    return [{"in": [[n[v], k] for v, k in sch.ins[i]],
             "wait_out": [n[v] for v in sch.wait_out[i]],
             "reserve_out": [n[v] for v in sch.reserve_out[i]],
             "free": [n[v] for v in sch.free[i]]} for i in range(g.n_fns)]


def _cases():
    gold = json.load(open(GOLD))
    for ex in gold["examples"]:
        wins = ex.get("windows") or [{"window": ex["window"], "r": ex["r"], "B_i": ex["B_i"],
                                      "cases": ex["cases"]}]
        for w in wins:
            for c in w["cases"]:
                yield ex["name"], ex["graph"], w, c


@pytest.mark.parametrize("name,gdoc,w,case", list(_cases()),
                         ids=lambda x: x if isinstance(x, str) else None)
def test_golden_examples(name, gdoc, w, case):
    g, seq = _load(gdoc)
    scheduler.attach_bytes(g, seq)
    assert scheduler.window_ends(seq, w["window"]) == w["r"]
    assert scheduler.window_bytes(g, seq, w["window"]) == w["B_i"]
    if "infeasible" in case:
        with pytest.raises(scheduler.InfeasibleBudget) as ei:
            scheduler.build_schedule(g, seq, case["budget"], w["window"])
        assert g.fn_names[ei.value.fn] == case["infeasible"]["fn"]
        assert ei.value.needed == case["infeasible"]["needed"]
        return
    sch = scheduler.build_schedule(g, seq, case["budget"], w["window"])
    assert _named(g, sch) == case["fn"]
    assert [g.var_names[v] for v in sch.end_wait] == case["end_wait"]
    assert sch.stats == case["stats"]
    ok, err = validate.validate(g, seq, sch, case["budget"])
    assert ok, err


def test_fig1_distance_identity():
    """the distance between f_i and f_{i+3} is the bytes of
    {V_{i+1}, V_{i+2}} — the occurrences strictly between the two spans."""
    for seed in range(50):
        g, seq = _load(sg.random_graph(seed, n_fns=12, n_vars=20))
        for i in range(g.n_fns - 3):
            between = sum(g.var_bytes[v] for v in seq.occ[seq.e[i] + 1:seq.l[i + 3]])
            direct = sum(g.var_bytes[v] for j in (i + 1, i + 2) for v in g.uses(j) if not g.pinned[v])
            assert between == direct


def test_next_use_brute_force_and_length():
    """S:70 quadratic next_use scan; S:84 Σ|V̂_i| = len(v)."""
    for seed in range(50):
        g, seq = _load(sg.random_graph(seed, p_pinned=0.1))
        assert len(seq.occ) == sum(len([v for v in g.uses(i) if not g.pinned[v]]) for i in range(g.n_fns))
        for k in range(len(seq.occ)):
            nxt = None
            for k2 in range(k + 1, len(seq.occ)):
                if seq.occ[k2] == seq.occ[k]:
                    nxt = k2
                    break
            assert seq.next_use[k] == nxt


def test_closed_form_feasibility_scan():
    """Greedy succeeds at (B, W) iff max_i B_i(W) + pinned <= B, scanned over
    every budget."""
    for seed in range(40):
        g, seq = _load(sg.random_graph(seed, n_fns=10, n_vars=12, max_bytes=9, p_pinned=0.1))
        scheduler.attach_bytes(g, seq)
        pinned = scheduler.pinned_bytes(g)
        total = sum(g.var_bytes)
        for W in (0, 5, 13, 10 ** 9):
            need = max(scheduler.window_bytes(g, seq, W)) + pinned
            for B in range(pinned, total + 2):
                try:
                    scheduler.build_schedule(g, seq, B, W)
                    ok = True
                except scheduler.InfeasibleBudget:
                    ok = False
                assert ok == (need <= B), (seed, W, B, need)
            assert scheduler.min_feasible_budget(g, seq, W) == need


def test_distance_window_closed_form_and_special_cases():
    """F1 prior-art policies (vDNN d = 1, LMS fixed distance d):
    the window of f_i is V̂_i ∪ ... ∪ V̂_{i+d}, so greedy feasibility is
    B >= max_i bytes(∪_{j=i..i+d} V̂_j) + pinned — computed here from the
    functions' variable lists, not from the oracle's window ends; d >= n
    gives the same events as an infinite byte window; every schedule passes
    the replay validator."""
    for seed in range(30):
        g, seq = _load(sg.random_graph(seed, n_fns=9, n_vars=11, max_bytes=9, p_pinned=0.1))
        scheduler.attach_bytes(g, seq)
        pinned = scheduler.pinned_bytes(g)
        total = sum(g.var_bytes)
        n = g.n_fns
        fvars = [set(seq.occ[seq.l[i]:seq.e[i] + 1]) for i in range(n)]
        for d in (1, 2, 4):
            need = max(sum(g.var_bytes[v] for v in set().union(*fvars[i:min(i + d, n - 1) + 1]))
                       for i in range(n)) + pinned
            for B in range(pinned, total + 2):
                try:
                    sch = scheduler.build_schedule(g, seq, B, 0, distance=d)
                    ok = True
                except scheduler.InfeasibleBudget:
                    ok = False
                assert ok == (need <= B), (seed, d, B, need)
                if ok:
                    validate.validate(g, seq, sch, B)
            assert scheduler.min_feasible_budget(g, seq, 0, distance=d) == need
        a = scheduler.build_schedule(g, seq, total, 0, distance=n)
        b = scheduler.build_schedule(g, seq, total, 10 ** 12)
        assert (a.ins, a.wait_out, a.reserve_out, a.free) == (b.ins, b.wait_out, b.reserve_out, b.free)
        assert '"distance":%d' % n in scheduler.canonical_json(a)


def test_window_infinite_special_case():
    """window and budget >= footprint -> only initial swap-ins and
    terminal frees (plus write-backs of modified persistent variables)."""
    for seed in range(30):
        g, seq = _load(sg.random_graph(seed))
        total = sum(g.var_bytes)
        sch = scheduler.build_schedule(g, seq, total, 10 ** 12)
        assert all(sch.ins[i] == [] for i in range(1, g.n_fns))
        assert all(sch.wait_out[i] == [] for i in range(g.n_fns))
        for i in range(g.n_fns):
            for v in sch.reserve_out[i]:
                assert g.persistent[v]
        assert sch.stats["bytes_h2d"] == sum(g.var_bytes[v] for v in range(g.n_vars)
                                             if g.persistent[v] and not g.pinned[v])


def test_replay_safety_1000_graphs():
    """on >= 1000 seeded random graphs the greedy either raises
    InfeasibleBudget or returns a schedule that passes the replay validator."""
    n_ok = 0
    for seed in range(1000):
        g, seq = _load(sg.random_graph(seed, p_pinned=0.05))
        scheduler.attach_bytes(g, seq)
        total = sum(g.var_bytes)
        B = max(1, total // (1 + seed % 4))
        W = (seed * 7919) % (total + 1)
        try:
            sch = scheduler.build_schedule(g, seq, B, W)
        except scheduler.InfeasibleBudget:
            continue
        ok, err = validate.validate(g, seq, sch, B)
        assert ok, (seed, err)
        n_ok += 1
    assert n_ok > 300


def test_validator_mutations():
    """the validator rejects a schedule with a swap-in removed or a
    swap-out of a dead variable added."""
    g, seq = _load(json.load(open(GOLD))["examples"][1]["graph"])
    sch = scheduler.build_schedule(g, seq, 12, 8)
    assert validate.validate(g, seq, sch, 12)[0]
    sch.ins[4] = sch.ins[4][1:]                     # drop a1's swap-in at f5
    ok, err = validate.validate(g, seq, sch, 12)
    assert not ok and "not resident" in err
    sch = scheduler.build_schedule(g, seq, 12, 8)
    sch.reserve_out[3].append(2)                     # a2 is dead after f4
    ok, err = validate.validate(g, seq, sch, 12)
    assert not ok
    sch = scheduler.build_schedule(g, seq, 12, 8)
    assert not validate.validate(g, seq, sch, 11)[0]  # budget violated


def test_w0_budget_equals_optimum_over_all_schedules():
    """the minimum budget over ALL schedules (exhaustive DP
    over resident sets) equals the greedy's at W = 0, which equals
    max_i bytes(distinct V̂_i)."""
    for seed in range(25):
        g, seq = _load(sg.random_graph(seed, n_fns=5, n_vars=6, max_bytes=6))
        brute = bruteforce.min_budget_all_schedules(g)
        assert scheduler.min_feasible_budget(g, seq, 0) == brute
        fp = graph.footprint_stats(g)
        assert brute == fp["max_function_bytes"]


def test_greedy_transfer_bytes_vs_optimum():
    """greedy transfer bytes (h2d + dirty d2h) >= the exhaustive
    optimum at the same budget; equality when everything fits (W = ∞)."""
    gaps = []
    for seed in range(25):
        g, seq = _load(sg.random_graph(seed, n_fns=6, n_vars=6, max_bytes=6, p_persistent=0.4))
        scheduler.attach_bytes(g, seq)
        total = sum(g.var_bytes)
        for B in range(1, total + 1):
            for W in (0, 4, 10 ** 6):
                try:
                    sch = scheduler.build_schedule(g, seq, B, W)
                except scheduler.InfeasibleBudget:
                    continue
                opt = bruteforce.optimal_cost(g, B)
                assert opt is not None
                cost = sch.stats["bytes_h2d"] + sch.stats["bytes_d2h_clean_elided"]
                assert cost >= opt, (seed, B, W)
                gaps.append(cost - opt)
        sch = scheduler.build_schedule(g, seq, total, 10 ** 6)
        assert sch.stats["bytes_h2d"] + sch.stats["bytes_d2h_clean_elided"] == bruteforce.optimal_cost(g, total)
    assert gaps


def test_graph_validation_errors():
    bad = [
        '{"variables": [}',                                              # parse
        {"variables": [{"id": "a", "bytes": 0}], "functions": [{"id": "f", "in": [], "out": ["a"]}]},
        {"variables": [{"id": "a", "bytes": 1}, {"id": "a", "bytes": 1}], "functions": []},
        {"variables": [{"id": "a", "bytes": 1}], "functions": [{"id": "f", "in": ["b"], "out": []}]},
        {"variables": [{"id": "a", "bytes": 1}, {"id": "b", "bytes": 1}],   # cycle
         "functions": [{"id": "f", "in": ["b"], "out": ["a"]}, {"id": "g", "in": ["a"], "out": ["b"]}]},
        {"variables": [{"id": "a", "bytes": 1}], "functions": [{"id": "f", "in": ["a"], "out": []}]},
    ]
    for d in bad:
        with pytest.raises(graph.GraphError):
            graph.load_graph(d if isinstance(d, str) else json.dumps(d))


def test_topological_order_tie_break():
    """a diamond listed out of order is re-ordered by Kahn with the
    smallest listed index first."""
    d = {"variables": [{"id": "x", "bytes": 1}, {"id": "y", "bytes": 1}, {"id": "z", "bytes": 1},
                       {"id": "w", "bytes": 1}],
         "functions": [{"id": "f4", "in": ["y", "z"], "out": ["w"]}, {"id": "f2", "in": ["x"], "out": ["y"]},
                       {"id": "f3", "in": ["x"], "out": ["z"]}, {"id": "f1", "in": [], "out": ["x"]}]}
    g = graph.load_graph(json.dumps(d))
    assert g.fn_names == ["f1", "f2", "f3", "f4"]
