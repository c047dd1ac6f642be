"""DenseNet-BC (the paper's Fig.4/5 family) through the
C-ABI: every gradient within 1e-5 of the oracle in fp32 mode under a swap-
forcing budget (channel concatenation, BN inputs with two consumers, average-
pool transitions), and bitwise swap transparency in bf16."""
import numpy as np
import pytest

from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

from test_gpu_resnet import run_step


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_tiny_densenet_parity_fp32(mode):
    spec = nets.tiny_densenet(batch=4, image=16, classes=10, mode="fp32")
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    budget = max(G.min_feasible_budget(0), G.in_core_peak() // 3)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    out = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE, mode, None, fp32_input=True)
    assert out["metrics"]["bytes_d2h"] > 0
    assert abs(out["loss"] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    # conditioning: the oracle's own response to a 1e-7 relative input
    # perturbation (fp32 rounding size); the stem BN's γ gradient here is a
    # near-total cancellation (norm 3e-6 against 3e-3 for β) that moves 0.8 %
    # (Z24), so its bound is 10x that response instead of 1e-5
    xp = (x * (1 + 1e-7 * np.random.default_rng(9).standard_normal(x.shape))).astype(np.float32)
    ref_p = nm.train_step(spec, p, xp, y)
    for k in p:
        tol = max(1e-5, 10 * nm.rel_l2(ref_p["grads"][k], ref["grads"][k]))
        e = nm.rel_l2(out["m." + k], ref["grads"][k])
        assert e <= tol, (k, e, tol)


@pytest.mark.gpu
def test_densenet_bf16_transparency():
    """DenseNet-BC with 3 blocks of 2 layers on 32² images, bf16: out-of-core (1/4
    budget, VA) == in-core, bitwise."""
    spec = nets.densenet(batch=16, image=32, classes=10, growth=16, blocks=(2, 2, 2), bn_size=2, init=32)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    ooc = run_step(spec, doc, info, max(G.min_feasible_budget(0), peak // 4), B.OC_WINDOW_MAX_FEASIBLE, "va", None)
    inc = run_step(spec, doc, info, peak, 0, "best", None)
    assert ooc["metrics"]["bytes_d2h"] > 0
    for k in nets.make_params(spec):
        assert np.array_equal(ooc["m." + k], inc["m." + k]), k
