"""Audit of REAL executed timelines (oc_exec_timeline, CUDA events on the
compute / H2D / D2H streams) against the paper's execution semantics — rules
R1-R4 of tests/timeline_audit.py: every swapped-in tensor is resident before
the function that reads it starts, no write into recycled memory
(VA chunks or arena bytes) starts before the previous occupant's last reader
and its swap-out ended (Fig.2(b): the wait before f_i), every swap-out
starts after the function it follows, and every re-read host copy is
complete.  Placements come from the oracle's allocator replay, which is
bit-exact with the executor's (test_plan_parity.py)."""
import numpy as np
import pytest
import torch

import timeline_audit as TA
from oracle import allocators, graph as og, scheduler as osch
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20


def _run_and_audit(spec, budget, mode, phys, chunk=2 * MiB, pack=64 << 10, pin_below=0, steps=2, trigger=0):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    doc, info = graphs.build(spec, params="persistent", inputs="host", pin_below=pin_below)
    st = OutOfCoreStep(doc, budget, B.OC_WINDOW_MAX_FEASIBLE, mode=mode, chunk_bytes=chunk, phys_bytes=phys,
                       timeline=True, pack_threshold=pack, trigger=trigger)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], x.astype(np.float32) if spec["mode"] == "fp32"
             else torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy())
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    for _ in range(steps):
        met = st.step()
    tl = st.timeline()
    W = st.stats["window"]
    st.close()
    g = og.load_graph(doc)
    o = osch.build_schedule(g, og.build_sequence(g), budget, W)
    rs, pl = allocators.replay(g, o, mode, chunk_bytes=chunk, phys_bytes=phys, align=512)
    assert rs["oom"] is None
    assert met["bytes_d2h"] > 0 and met["bytes_h2d"] > 0
    n_h2d = sum(1 for e in tl if e["stream"] == "h2d")
    assert n_h2d == sum(1 for i in range(g.n_fns) for _, k in o.ins[i] if k == "h2d")
    return TA.audit(g, o, pl, mode, tl, align=512, paper_trigger=trigger == 1)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,phys", [("best", 8 * MiB), ("first", 8 * MiB), ("va", 512 * MiB)])
@pytest.mark.parametrize("pack", [0, 64 << 10])
def test_mlp_timeline(mode, phys, pack):
    bad = _run_and_audit(nets.mlp6(), 4 * MiB, mode, phys, pack=pack)
    assert bad == [], bad[:10]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_mlp_timeline_paper_trigger(mode):
    bad = _run_and_audit(nets.mlp6(), 4 * MiB, mode, 8 * MiB if mode == "best" else 512 * MiB, trigger=1)
    assert bad == [], bad[:10]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_resnet_timelines(mode):
    for spec in (nets.tiny_resnet(batch=4, image=16, classes=10),
                 nets.resnet(18, batch=8, image=64, classes=10, mode="fp32")):
        doc, _ = graphs.build(spec, params="persistent")
        G = B.Graph(doc)
        budget = max(G.min_feasible_budget(0), G.in_core_peak() // 4)
        probe = G.plan(budget, B.OC_WINDOW_MAX_FEASIBLE, B.OC_ALLOC_VA if mode == "va" else B.OC_ALLOC_ARENA_BEST,
                       chunk_bytes=2 * MiB, phys_bytes=1 << 40, allow_oom=True).stats()
        for trigger in (0, 1):
            bad = _run_and_audit(spec, budget, mode, probe["peak_phys"] + 2 * MiB, trigger=trigger)
            assert bad == [], (trigger, bad[:10])
