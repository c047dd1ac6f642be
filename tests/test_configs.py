"""Plan-level checks of the benchmark configurations (CPU only): the budget
fractions named in BASELINE.json are feasible for the scheduler and the
allocator replay, and the VA chunk-size effect of Eq.1 shows on
the ResNet-1001 configuration."""
import pytest

from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20


@pytest.fixture(scope="module")
def r1001():
    spec = nets.preact_resnet(1001, batch=256)
    doc, info = graphs.build(spec, params="persistent", pin_below=2 * MiB)
    return B.Graph(doc)


def test_r1001_quarter_budget_feasible_with_2mib_chunks(r1001):
    """configs[4]: at F_peak/4, with tensors below one chunk pinned (Z26), the
    schedule fits and the VA replay needs no more physical memory than the
    budget (every swapped activation is a whole number of 2 MiB chunks)."""
    budget = r1001.in_core_peak() // 4
    assert r1001.min_feasible_budget(0) <= budget
    s = r1001.plan(budget, 0, B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=budget + 64 * MiB)
    st = s.stats()
    assert st["peak_sched"] <= budget
    assert st["peak_phys"] <= budget + 64 * MiB


def test_r1001_40mib_chunks_blow_up_internal_fragmentation(r1001):
    """The same schedule with the paper's 40 MiB chunk: activations of
    2-32 MiB each round up to a 40 MiB chunk, so the replay OOMs at the
    2 MiB pool size — Eq.1 internal fragmentation, the reason m_c must be
    matched to the tensor sizes."""
    budget = r1001.in_core_peak() // 4
    with pytest.raises(B.OcError):
        r1001.plan(budget, 0, B.OC_ALLOC_VA, chunk_bytes=40 * MiB, phys_bytes=budget + 64 * MiB)
    s = r1001.plan(budget, 0, B.OC_ALLOC_VA, chunk_bytes=40 * MiB, phys_bytes=budget * 8, allow_oom=True)
    assert s.stats()["if_peak"] > budget // 2


def test_biggan_config_feasible_and_tiny_gan_schedule_matches_oracle():
    """configs[4] BigGAN-style step: the per-chunk attention maps keep every
    function's working set small enough for a quarter of F_peak; the tiny
    GAN's canonical schedule bytes equal the oracle's."""
    import json
    from oracle import graph as og, scheduler as osch
    spec = nets.biggan(batch=32)
    doc, _ = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    assert G.min_feasible_budget(0) <= G.in_core_peak() // 4
    tdoc, _ = graphs.build(nets.tiny_biggan(batch=4), params="persistent")
    g = og.load_graph(tdoc)
    seq = og.build_sequence(g)
    Gt = B.Graph(tdoc)
    budget = max(Gt.min_feasible_budget(0), Gt.in_core_peak() // 3)
    o = osch.build_schedule(g, seq, budget, 0)
    s = Gt.plan(budget, 0, B.OC_ALLOC_ARENA_BEST, chunk_bytes=1, phys_bytes=budget * 4, allow_oom=True)
    assert s.json() == osch.canonical_json(o)
    assert json.loads(s.json())["stats"]["bytes_d2h"] > 0
