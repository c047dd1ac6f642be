"""configs[0]: 6-layer MLP (width 256, batch 8, fp32) under a 4 MiB budget
that forces swaps.  GPU parity through the C-ABI against the CPU oracle
(1e-5 relative L2 in fp32 mode), and swap transparency: the out-of-core step
is bitwise equal to the in-core step."""
import json

import numpy as np
import pytest

from oracle import graph as og
from oracle import numerics as nm
from oracle import scheduler as osch
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20


def _setup():
    spec = nets.mlp6()
    doc, info = graphs.build(spec, params="persistent", inputs="host")
    return spec, doc, info


def test_mlp_graph_forces_swaps_at_4mib():
    """CPU: the 4 MiB budget is feasible and forces swap traffic; the oracle
    and the C-ABI planner agree bit for bit on the schedule."""
    spec, doc, info = _setup()
    g = og.load_graph(doc)
    seq = og.build_sequence(g)
    total = sum(g.var_bytes)
    assert total > 4 * MiB
    W = osch.max_feasible_window(g, seq, 4 * MiB)
    assert W is not None
    sch = osch.build_schedule(g, seq, 4 * MiB, W)
    assert sch.stats["bytes_d2h"] > 0 and sch.stats["peak_sched"] <= 4 * MiB
    G = B.Graph(doc)
    s = G.plan(4 * MiB, B.OC_WINDOW_MAX_FEASIBLE, B.OC_ALLOC_ARENA_BEST, phys_bytes=8 * MiB)
    assert s.json() == osch.canonical_json(sch)


def _run(spec, doc, info, budget, window, mode, phys, chunk=2 * MiB, pack=64 << 10):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    st = OutOfCoreStep(doc, budget, window, mode=mode, chunk_bytes=chunk, phys_bytes=phys, pack_threshold=pack)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], x)
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    met = st.step()
    out = {"loss": float(st.read(info["loss"])[0]), "metrics": met}
    for k in p:
        out["p." + k] = st.read(info["params"][k]).reshape(p[k].shape)
        out["m." + k] = st.read(info["momentum"][k]).reshape(p[k].shape)
    st.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mode,phys", [("best", 8 * MiB), ("first", 8 * MiB), ("va", 512 * MiB)])
def test_mlp_parity_and_swap_transparency(mode, phys):
    spec, doc, info = _setup()
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    ooc = _run(spec, doc, info, 4 * MiB, B.OC_WINDOW_MAX_FEASIBLE, mode, phys)
    assert ooc["metrics"]["bytes_d2h"] > 0          # swaps really happened
    assert abs(ooc["loss"] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    for k in p:
        assert nm.rel_l2(ooc["m." + k], ref["grads"][k]) <= 1e-5, k      # v = g after one step
        assert nm.rel_l2(ooc["p." + k], ref["params"][k]) <= 1e-5, k
    g = og.load_graph(doc)
    inc = _run(spec, doc, info, og.in_core_peak(g), 0, "best", og.in_core_peak(g) * 2)
    for k in p:
        assert np.array_equal(inc["m." + k], ooc["m." + k]), k          # bitwise swap transparency
        assert np.array_equal(inc["p." + k], ooc["p." + k]), k
    # every swap through the SM pack/unpack kernel (A7) vs none through it
    allpack = _run(spec, doc, info, 4 * MiB, B.OC_WINDOW_MAX_FEASIBLE, mode, phys, pack=1 << 30)
    nopack = _run(spec, doc, info, 4 * MiB, B.OC_WINDOW_MAX_FEASIBLE, mode, phys, pack=0)
    assert allpack["metrics"]["n_h2d"] < nopack["metrics"]["n_h2d"]
    assert allpack["metrics"]["bytes_d2h"] == nopack["metrics"]["bytes_d2h"]
    for k in p:
        assert np.array_equal(allpack["p." + k], ooc["p." + k]) and np.array_equal(nopack["p." + k], ooc["p." + k])
