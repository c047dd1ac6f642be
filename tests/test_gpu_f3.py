"""The paper's other two families on the GPU (PAPER.md P:206,
Fig.4/5): DeepLabv3+ (513² in the paper) and Pix2PixHD (512×1024), through
the C-ABI out-of-core executor.

  * atrous (dilated) convolutions on the tcgen05 / TMA kernels — fprop,
    stride-1 dgrad and wgrad with dilated im2col offsets, persistent regime
    included — element-wise against the oracle's definition (bf16 outputs
    within 1e-3 relative L2, fp32 weight gradients within 1e-5), and on the
    CUDA cores (fp32 mode);
  * fp32 mode: miniature networks end to end against numerics.train_step —
    loss and every parameter gradient within 1e-5 (north_star fp32);
  * bf16: every function of the step layer-locally within 1e-3
    (tests/layerwise_harness.py) — the miniature nets and the full-size
    DeepLabv3+ 513² and Pix2PixHD 512×1024 steps — and bitwise swap
    transparency (out-of-core == in-core)."""
import json

import numpy as np
import pytest
import torch

from layerwise_harness import run_layerwise
from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20


def bf(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


def bits(t):
    return t.view(torch.int16).numpy()


def from_bits(a, shape):
    return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).float().numpy().reshape(shape).astype(np.float64)


def _conv_graph(kind, N, H, W, C, K, R, pad, dil, dtype="bf16", accumulate=False):
    P = H + 2 * pad - dil * (R - 1)
    attrs = {"dtype": dtype, "N": N, "H": H, "W": W, "C": C, "K": K, "R": R, "S": R, "stride": 1, "pad": pad,
             "P": P, "Q": W + 2 * pad - dil * (R - 1), "dil": dil, "accumulate": accumulate}
    Q = attrs["Q"]
    es = 2 if dtype == "bf16" else 4
    v = lambda n, b: {"id": n, "bytes": int(b), "pinned": True}
    xs, ys, ws = N * H * W * C * es, N * P * Q * K * es, K * R * R * C * 4
    if kind == "conv_fwd":
        vars_, io = [v("x", xs), v("w", ws), v("y", ys)], ({"x": "x", "w": "w", "y": "y"}, ["x", "w"], ["y"])
    elif kind == "conv_dgrad":
        vars_ = [v("dy", ys), v("w", ws), v("dx", xs)]
        io = ({"dy": "dy", "w": "w", "dx": "dx"}, ["dy", "w"] + (["dx"] if accumulate else []), ["dx"])
    else:
        vars_, io = [v("dy", ys), v("x", xs), v("dw", ws)], ({"dy": "dy", "x": "x", "dw": "dw"}, ["dy", "x"], ["dw"])
    fn = {"id": "f", "in": io[1], "out": io[2], "op": {"kind": kind, "args": io[0], "attrs": attrs}}
    return json.dumps({"variables": vars_, "functions": [fn]}), (P, Q), sum(x["bytes"] for x in vars_)


def _run(doc, total, inputs, out, dtype):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in inputs.items():
        st.write(k, a)
    st.step()
    r = st.read(out, dtype)
    st.close()
    return r


ATROUS = [  # N, H, W, C, K, R, pad, dil
    (2, 17, 15, 64, 64, 3, 2, 2),
    (2, 21, 19, 128, 64, 3, 6, 6),
    (2, 33, 33, 512, 512, 3, 2, 2),       # DeepLabv3+ layer4 (output stride 16)
    (2, 33, 33, 2048, 256, 3, 12, 12),    # ASPP rate 12
    (1, 33, 33, 2048, 256, 3, 18, 18),    # ASPP rate 18: most taps in the zero padding
]


@pytest.mark.gpu
@pytest.mark.parametrize("g", ATROUS)
@pytest.mark.parametrize("cap", ["", "3"])
def test_atrous_conv_tensor_cores(g, cap, monkeypatch):
    if cap:   # persistent regime: a 3-CTA grid loops over every unit
        monkeypatch.setenv("OC_CONV_MAX_CTAS", cap)
    N, H, W, C, K, R, pad, dil = g
    rng = np.random.default_rng(31)
    x = bf(rng.standard_normal((N, H, W, C)))
    w = (rng.standard_normal((K, R, R, C)) / np.sqrt(R * R * C)).astype(np.float32)
    doc, (P, Q), total = _conv_graph("conv_fwd", N, H, W, C, K, R, pad, dil)
    y = from_bits(_run(doc, total, {"x": bits(x), "w": w}, "y", np.uint16), (N, P, Q, K))
    xf = x.float().numpy().astype(np.float64)
    wr = nm.round_bf16(w.astype(np.float64))
    ref = nm.round_bf16(nm.conv2d(xf, wr, 1, pad, dil))
    assert nm.rel_l2(y, ref) < 1e-3
    dy = bf(rng.standard_normal((N, P, Q, K)))
    old = bf(rng.standard_normal((N, H, W, C)))
    doc, _, total = _conv_graph("conv_dgrad", N, H, W, C, K, R, pad, dil, accumulate=True)
    dx = from_bits(_run(doc, total, {"dy": bits(dy), "w": w, "dx": bits(old)}, "dx", np.uint16), (N, H, W, C))
    dyf = dy.float().numpy().astype(np.float64)
    rdx, _ = nm.conv2d_backward(np.zeros((N, H, W, C)), wr, dyf, 1, pad, dil)
    assert nm.rel_l2(dx, nm.round_bf16(rdx + old.float().numpy())) < 1e-3
    doc, _, total = _conv_graph("conv_wgrad", N, H, W, C, K, R, pad, dil)
    dw = _run(doc, total, {"dy": bits(dy), "x": bits(x)}, "dw", np.float32).reshape(K, R, R, C)
    _, rdw = nm.conv2d_backward(xf, np.zeros((K, R, R, C)), dyf, 1, pad, dil)
    assert nm.rel_l2(dw, rdw) < 1e-5


@pytest.mark.gpu
def test_atrous_conv_cuda_cores_fp32():
    N, H, W, C, K, R, pad, dil = 2, 13, 11, 16, 8, 3, 4, 4
    rng = np.random.default_rng(32)
    x = rng.standard_normal((N, H, W, C)).astype(np.float32)
    w = rng.standard_normal((K, R, R, C)).astype(np.float32)
    doc, (P, Q), total = _conv_graph("conv_fwd", N, H, W, C, K, R, pad, dil, dtype="f32")
    y = _run(doc, total, {"x": x, "w": w}, "y", np.float32).reshape(N, P, Q, K)
    assert nm.rel_l2(y, nm.conv2d(x.astype(np.float64), w.astype(np.float64), 1, pad, dil)) < 1e-6
    dy = rng.standard_normal((N, P, Q, K)).astype(np.float32)
    doc, _, total = _conv_graph("conv_dgrad", N, H, W, C, K, R, pad, dil, dtype="f32")
    dx = _run(doc, total, {"dy": dy, "w": w, "dx": np.zeros((N, H, W, C), np.float32)}, "dx", np.float32)
    rdx, rdw = nm.conv2d_backward(x.astype(np.float64), w.astype(np.float64), dy.astype(np.float64), 1, pad, dil)
    assert nm.rel_l2(dx.reshape(N, H, W, C), rdx) < 1e-6
    doc, _, total = _conv_graph("conv_wgrad", N, H, W, C, K, R, pad, dil, dtype="f32")
    dw = _run(doc, total, {"dy": dy, "x": x}, "dw", np.float32)
    assert nm.rel_l2(dw.reshape(K, R, R, C), rdw) < 1e-6


def _mini(family, mode):
    if family == "deeplab":
        # batch 8 in fp32: at batch 4 the oracle's own fp32-vs-fp64 difference reaches 4e-6 on a BN
        # gamma gradient (near-total cancellation), too close to the 1e-5 bound (measured: 1.8e-6 at 8)
        return nets.deeplabv3plus(batch=8 if mode == "fp32" else 4, image=33, classes=3, width=8, rates=(2, 3, 4),
                                  aspp=8, low=8, blocks=(1, 1, 1, 1), mode=mode)
    return nets.pix2pixhd(batch=2, image=(16, 32), ngf=8, n_down=2, n_blocks=1, mode=mode)


def _step(spec, budget_frac, mode):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    out = {}
    for name, budget, W, m in (("ooc", max(G.min_feasible_budget(0), int(peak * budget_frac)),
                                B.OC_WINDOW_MAX_FEASIBLE, mode), ("inc", peak, 0, "best")):
        mm = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST}[m]
        phys = G.plan(budget, W, mm, chunk_bytes=2 * MiB, phys_bytes=1 << 40, allow_oom=True).stats()["peak_phys"]
        st = OutOfCoreStep(doc, budget, W, mode=m, chunk_bytes=2 * MiB, phys_bytes=phys + 2 * MiB)
        x, y = nets.make_inputs(spec)
        p = nets.make_params(spec)
        cv = (lambda a: a.astype(np.float32)) if spec["mode"] == "fp32" else (lambda a: bits(bf(a)))
        st.write(info["x"], cv(x))
        st.write(info["labels"], cv(y) if spec["loss"]["type"] == "l1" else y)
        for k, v in p.items():
            st.write(info["params"][k], v)
            st.write(info["momentum"][k], np.zeros_like(v))
        met = st.step()
        out[name] = {"loss": float(st.read(info["loss"])[0]), "met": met,
                     "m": {k: st.read(info["momentum"][k]).reshape(p[k].shape) for k in p}}
        st.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["deeplab", "pix2pix"])
@pytest.mark.parametrize("mode", ["va", "best"])
def test_f3_fp32_parity_and_transparency(family, mode):
    spec = _mini(family, "fp32")
    out = _step(spec, 0.3, mode)
    assert out["ooc"]["met"]["bytes_d2h"] > 0
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    assert abs(out["ooc"]["loss"] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    for k in p:
        assert nm.rel_l2(out["ooc"]["m"][k], ref["grads"][k]) <= 1e-5, k
        assert np.array_equal(out["ooc"]["m"][k], out["inc"]["m"][k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["deeplab", "pix2pix"])
def test_f3_bf16_layerwise_and_transparency(family):
    spec = _mini(family, "bf16")
    lw = run_layerwise(spec, budget_frac=0.3, pin_below=0)
    assert lw["checked"] == lw["functions"] and not lw["failures"], lw["failures"][:10]
    out = _step(spec, 0.3, "va")
    assert out["ooc"]["met"]["bytes_d2h"] > 0
    for k in out["ooc"]["m"]:
        assert np.array_equal(out["ooc"]["m"][k], out["inc"]["m"][k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name,spec", [
    ("deeplabv3plus_513_b2", nets.deeplabv3plus(batch=2)),
    ("pix2pixhd_512x1024_b1", nets.pix2pixhd(batch=1)),
])
def test_f3_full_size_layerwise(name, spec):
    """The paper's image sizes, every function of the bf16 step."""
    lw = run_layerwise(spec, budget_frac=0.25, pin_below=0)
    print(json.dumps({"case": name, "functions": lw["functions"],
                      "worst": {k: float(f"{v:.3e}") for k, v in sorted(lw["worst"].items())}}))
    assert lw["checked"] == lw["functions"] and not lw["failures"], lw["failures"][:10]
