"""The timeline audit (tests/timeline_audit.py) itself, on CPU: the executor
model of the makespan simulator (oracle/simulator.simulate_exec, which orders
every transfer on exactly the release points the executor waits for) yields
timelines that pass R1-R4 on random graphs under the VA and best-fit
replays, and each rule catches a mutation that breaks it.  The same audit
runs on real GPU timelines in tests/test_gpu_timeline_audit.py."""
import copy

import numpy as np

import timeline_audit as TA
from oracle import allocators, graph, scheduler, simulator
from synth import graphs as sg


def _case(seed):
    doc = sg.random_graph(seed, p_pinned=0.05)
    g = graph.load_graph(doc)
    seq = graph.build_sequence(g)
    total = sum(g.var_bytes)
    W = (seed * 13) % (total + 1)
    budget = max(scheduler.min_feasible_budget(g, seq, W), total // (2 + seed % 3))
    o = scheduler.build_schedule(g, seq, budget, W)
    mode = ("va", "best")[seed % 2]
    st, pl = allocators.replay(g, o, mode, chunk_bytes=1 + seed % 4, phys_bytes=total * 4, align=1)
    if st["oom"] is not None:
        return None
    rng = np.random.default_rng(seed)
    ev = simulator.simulate_exec(g, seq, o, pl, mode, [float(x) for x in rng.uniform(0.1, 2.0, g.n_fns)],
                                 1e-3, 1e-3, 0.5, 0.5, True, align=1)["events"]
    return g, o, pl, mode, ev


def test_model_timelines_pass():
    n = 0
    for seed in range(400):
        c = _case(seed)
        if c is None:
            continue
        g, o, pl, mode, ev = c
        assert TA.audit(g, o, pl, mode, ev, align=1) == [], seed
        n += 1
    assert n > 150


def test_mutations_are_caught():
    caught = {"R1": 0, "R2": 0, "R3": 0}
    for seed in range(400):
        c = _case(seed)
        if c is None:
            continue
        g, o, pl, mode, ev = c
        h2d = [e for e in ev if e["stream"] == "h2d"]
        d2h = [e for e in ev if e["stream"] == "d2h"]
        comp = {e["fn"]: e for e in ev if e["stream"] == "compute"}
        if h2d:   # R1: an arrival that lands after its consumer started
            e = h2d[0]
            first = min(j for j in range(e["fn"], g.n_fns) if e["var"] in g.uses(j))
            ev2 = copy.deepcopy(ev)
            for x in ev2:
                if x["stream"] == "h2d" and x["slot"] == e["slot"]:
                    x["t1"] = comp[first]["t0"] + 1.0
            caught["R1"] += any(b.startswith("R1") for b in TA.audit(g, o, pl, mode, ev2, align=1))
        if d2h:   # R3: a swap-out that starts before its producer ended
            e = d2h[0]
            ev2 = copy.deepcopy(ev)
            for x in ev2:
                if x["stream"] == "d2h" and x["dep"] == e["dep"]:
                    x["t0"] = comp[e["fn"]]["t1"] - 0.5
            caught["R3"] += any(b.startswith("R3") for b in TA.audit(g, o, pl, mode, ev2, align=1))
        # R2: pull a reusing H2D back to time 0 (before its previous occupant's readers)
        for e in h2d:
            ev2 = copy.deepcopy(ev)
            for x in ev2:
                if x["stream"] == "h2d" and x["slot"] == e["slot"]:
                    x["t0"] = -1.0
            bad = TA.audit(g, o, pl, mode, ev2, align=1)
            if any(b.startswith("R2") for b in bad):
                caught["R2"] += 1
                break
    assert all(v > 20 for v in caught.values()), caught
