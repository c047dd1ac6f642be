"""Pins of the oracle parts the round-1 review found checked only against the
C++ planner (VERDICT r1 "unpinned oracle parts"):

  * canonical schedule bytes — the hand-typed canonical strings of the worked
    examples E0/E1 (tests/golden/canonical_schedules.json, from the
    hand-derived event lists of SURVEY §8(c));
  * graph.in_core_peak (F_peak, reading Z21: the denominator of the 25 % and
    1/8 budgets) — hand-derived goldens for E0/E1, and a brute-force scan that
    decides liveness of every variable at every function straight from the
    definition (v is live at f_i iff some f_j, j <= i, and some f_k, k >= i,
    use it), plus its bounds max_i bytes(V̂_i) <= F_peak <= Σ bytes;
  * scheduler.max_feasible_window (reading Z12, a binary search that assumes
    feasibility is monotone in W) — an exhaustive scan of every window W in
    [0, Σ occurrence bytes] on tiny graphs: the feasible windows form a
    prefix and its last element is the binary search's answer.
The C-ABI is compared with the same goldens."""
import json
import os

from oracle import graph, scheduler
from paper_2010_14109_b200 import binding as B
from synth import graphs as sg

HERE = os.path.dirname(__file__)
CANON = json.load(open(os.path.join(HERE, "golden", "canonical_schedules.json")))
EXAMPLES = {e["name"]: e for e in json.load(open(os.path.join(HERE, "golden", "schedule_examples.json")))["examples"]}


def test_canonical_bytes_of_worked_examples():
    for c in CANON["cases"]:
        doc = json.dumps(EXAMPLES[c["example"]]["graph"])
        g = graph.load_graph(doc)
        o = scheduler.build_schedule(g, graph.build_sequence(g), c["budget"], c["window"])
        assert scheduler.canonical_json(o) == c["canonical"], c["example"]
        s = B.Graph(doc).plan(c["budget"], c["window"], B.OC_ALLOC_VA, chunk_bytes=1, phys_bytes=c["budget"])
        assert s.json() == c["canonical"], c["example"]


def _brute_peak(g):
    pinned = sum(b for v, b in enumerate(g.var_bytes) if g.pinned[v])
    users = [set(g.uses(i)) for i in range(g.n_fns)]
    best = 0
    for i in range(g.n_fns):
        live = 0
        for v in range(g.n_vars):
            if g.pinned[v]:
                continue
            before = any(v in users[j] for j in range(0, i + 1))
            after = any(v in users[k] for k in range(i, g.n_fns))
            if before and after:
                live += g.var_bytes[v]
        best = max(best, live + pinned)
    return best


def test_in_core_peak_goldens():
    for name, want in CANON["in_core_peak"].items():
        doc = json.dumps(EXAMPLES[name]["graph"])
        assert graph.in_core_peak(graph.load_graph(doc)) == want
        assert B.Graph(doc).in_core_peak() == want


def test_in_core_peak_brute_force_and_bounds():
    for seed in range(300):
        doc = sg.random_graph(seed, n_fns=12, n_vars=16, max_bytes=40, p_pinned=0.1)
        g = graph.load_graph(doc)
        peak = graph.in_core_peak(g)
        assert peak == _brute_peak(g), seed
        fp = graph.footprint_stats(g)
        pinned = sum(b for v, b in enumerate(g.var_bytes) if g.pinned[v])
        per_fn = max(sum(g.var_bytes[v] for v in set(g.uses(i)) if not g.pinned[v]) for i in range(g.n_fns))
        assert per_fn + pinned <= peak <= fp["total_bytes"]


def _feasible(g, seq, budget, W):
    try:
        scheduler.build_schedule(g, seq, budget, W)
        return True
    except scheduler.InfeasibleBudget:
        return False


def test_max_feasible_window_exhaustive_scan():
    n_checked = 0
    for seed in range(80):
        doc = sg.random_graph(seed, n_fns=6, n_vars=8, max_bytes=12, p_pinned=0.1)
        g = graph.load_graph(doc)
        seq = graph.build_sequence(g)
        scheduler.attach_bytes(g, seq)
        top = sum(seq.occ_bytes)
        lo = scheduler.min_feasible_budget(g, seq, 0)
        for budget in sorted({lo, lo + 3, (lo + sum(g.var_bytes)) // 2, sum(g.var_bytes)}):
            ok = [_feasible(g, seq, budget, W) for W in range(top + 2)]
            k = ok.index(False) if False in ok else len(ok)
            assert not any(ok[k:]), (seed, budget)          # feasible windows are a prefix
            want = None if k == 0 else min(k - 1, top)
            assert scheduler.max_feasible_window(g, seq, budget) == want, (seed, budget)
            if want is not None:
                assert B.Graph(doc).max_feasible_window(budget) == want
            n_checked += 1
    assert n_checked > 200
