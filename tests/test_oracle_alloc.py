"""Pins of the allocator oracle (oracle/allocators.py): Eq.1 and Eq.2 of the
paper as closed forms and as invariants on long random traces,
the best-fit worked example of S:258, the E1-alloc example (golden), the VA
no-external-fragmentation property and a counting oracle."""
import json
import os

import numpy as np
import pytest

from oracle import allocators as al
from oracle import graph, scheduler

MiB = 1 << 20
GOLD = os.path.join(os.path.dirname(__file__), "golden", "schedule_examples.json")


def test_eq1_examples():
    """m_r = 100 MiB at m_c = 40 MiB -> m_a = 120 MiB, IF = 20 MiB;
    m_r = 3 m_c -> IF = 0."""
    p = al.VAPool(40 * MiB, 400 * MiB)
    h = p.alloc(100 * MiB)
    assert len(p.chunks_of(h)) * p.m_c == 120 * MiB
    assert p.internal_frag() == 20 * MiB
    p.free(h)
    h = p.alloc(120 * MiB)
    assert p.internal_frag() == 0


def test_best_fit_worked_example():
    """capacity 10: A=10, free A, B=6 reuses A's region leaving 4
    cached; C=5 -> DeviceOOM despite 4 cached bytes."""
    a = al.Arena(10, align=1)
    ha = a.alloc(10)
    a.free(ha)
    hb = a.alloc(6)
    assert a.offset_of(hb) == 0
    assert a.free_bytes() == 4
    assert a.alloc(5) is None


def test_double_free_and_unknown():
    for A in (al.VAPool(2, 10), al.Arena(10, align=1)):
        h = A.alloc(1)
        A.free(h)
        with pytest.raises(al.AllocError, match="DoubleFree"):
            A.free(h)
        with pytest.raises(al.AllocError, match="UnknownHandle"):
            A.free(12345)


def test_eq2_and_no_external_fragmentation_long_trace():
    """on 10^5 random alloc/free steps every live VA allocation has
    0 <= m_a - m_r < m_c (Eq.1); total live IF < live count * m_c <= N_max m_c
    (Eq.2); an allocation succeeds iff free chunks >= k (no external
    fragmentation); the free-chunk count equals capacity - Σ live k
    (S:267 counting oracle)."""
    rng = np.random.default_rng(7)
    m_c = 40
    p = al.VAPool(m_c, 40 * 64)
    live = {}
    for step in range(100000):
        if live and (rng.random() < 0.5 or len(p.free_q) == 0):
            h = list(live)[int(rng.integers(0, len(live)))]
            p.free(h)
            del live[h]
        else:
            m_r = int(rng.integers(1, 300))
            k = -(-m_r // m_c)
            free_before = len(p.free_q)
            h = p.alloc(m_r)
            assert (h is not None) == (free_before >= k)
            if h is not None:
                live[h] = m_r
        for h, m_r in live.items():
            m_a = len(p.chunks_of(h)) * m_c
            assert 0 <= m_a - m_r < m_c
        if step % 97 == 0:
            assert p.internal_frag() < max(1, len(live)) * m_c or not live
            assert p.internal_frag() <= p.n_max * m_c
            assert len(p.free_q) == p.n_chunks - sum(len(p.chunks_of(h)) for h in live)


def test_best_fit_adversarial_trace_fragments():
    """an alternating-size best-fit trace hits DeviceOOM with free
    bytes >= the request (external fragmentation); VA on the same trace
    never does."""
    cap = 1000
    a = al.Arena(cap, align=1)
    hs = [a.alloc(100) for _ in range(10)]
    for h in hs[::2]:
        a.free(h)                     # five 100-byte holes, none adjacent
    assert a.alloc(150) is None and a.free_bytes() >= 150
    v = al.VAPool(50, cap)
    hv = [v.alloc(100) for _ in range(10)]
    for h in hv[::2]:
        v.free(h)
    assert v.alloc(150) is not None


def test_first_vs_best_fit_choice():
    a = al.Arena(100, align=1, policy="best")
    f = al.Arena(100, align=1, policy="first")
    for A in (a, f):
        h1 = A.alloc(30)
        A.alloc(1)
        h2 = A.alloc(10)
        A.alloc(1)
        A.free(h1)
        A.free(h2)
    assert a.offset_of(a.alloc(8)) == 31      # smallest hole that fits
    assert f.offset_of(f.alloc(8)) == 0       # lowest address that fits


def test_segment_local_coalescing():
    """adjacent free blocks merge only inside the same carved segment."""
    a = al.Arena(100, align=1)
    h1 = a.alloc(10)
    h2 = a.alloc(10)
    a.free(h1)
    a.free(h2)
    assert a.alloc(20) is not None          # not satisfied by [0,20): two segments
    assert a.tail == 40


def test_e1_alloc_golden():
    gold = json.load(open(GOLD))["examples"][1]
    ga = gold["alloc"]
    g = graph.load_graph(json.dumps(gold["graph"]))
    seq = graph.build_sequence(g)
    sch = scheduler.build_schedule(g, seq, ga["budget"], ga["window"])
    st, _ = al.replay(g, sch, "va", chunk_bytes=ga["va"]["chunk_bytes"], phys_bytes=ga["va"]["phys_bytes"])
    assert st["peak_phys"] == ga["va"]["peak_phys"]
    assert st["if_peak"] == ga["va"]["if_peak"]
    assert st["n_max"] == ga["va"]["n_max"]
    assert st["oom"] is None
    for mode in ("best", "first"):
        st, _ = al.replay(g, sch, mode, phys_bytes=ga[mode]["phys_bytes"], align=ga[mode]["align"])
        exp = dict(ga[mode]["oom"])
        exp["fn"] = g.fn_names.index(exp["fn"])
        exp["var"] = g.var_names.index(exp["var"])
        assert st["oom"] == exp
