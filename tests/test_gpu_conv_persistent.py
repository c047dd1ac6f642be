"""Element-wise parity of the tcgen05 / TMA convolution kernels with the
oracle's direct-definition convolution (oracle/numerics.py conv2d,
conv2d_backward) in the PERSISTENT regime the full-size step runs them in:
every CTA (or CTA pair) loops over many work units, so the mbarrier phases wrap
past the stage ring, the two TMEM accumulators alternate, staging buffers are
reused and the fused BN-statistics slots sum over several units.

Two ways to get there at sizes the oracle finishes in seconds:
  * shapes whose unit count is far above 148 CTAs / 74 pairs (ResNet-18
    layer-1 and stride-2 layer shapes at batch 16, the 224^2 stem in four
    image slices, the 1x1 64->256 ResNet-50 shape, wgrad at its maximum
    split count = 2 units per SM);
  * the small shapes of test_gpu_conv.py with the grid capped to 3 CTAs
    (OC_CONV_MAX_CTAS, read at every launch: 3 single CTAs or 1 pair).

Tolerance: north_star's 1e-3 relative L2 for bf16 outputs (the oracle rounds
to bf16 where the kernel stores bf16, so only accumulation-order rounding
flips differ), 1e-5 for the fp32 weight gradients."""
import json

import numpy as np
import pytest
import torch

from oracle import numerics as nm
import test_gpu_conv as T

TOL_BF16 = 1e-3


def _geom(g):
    N, H, W, C, K, R, st, pad = g[:8]
    return N, H, W, C, K, R, st, pad, (H + 2 * pad - R) // st + 1, (W + 2 * pad - R) // st + 1


def fprop(g, seed=11):
    N, H, W, C, K, R, st, pad, P, Q = _geom(g)
    rng = np.random.default_rng(seed)
    x = T.bf(rng.standard_normal((N, H, W, C)))
    w = (rng.standard_normal((K, R, R, C)) / np.sqrt(R * R * C)).astype(np.float32)
    doc, _, total = T._graph("conv_fwd", g)
    y = T._from_bits(T._run(doc, total, {"x": T._bits(x), "w": w}, "y", np.uint16), (N, P, Q, K))
    ref = nm.round_bf16(nm.conv2d(x.float().numpy().astype(np.float64), nm.round_bf16(w.astype(np.float64)), st, pad))
    return y, ref


def dgrad(g, accumulate, seed=12):
    N, H, W, C, K, R, st, pad, P, Q = _geom(g)
    rng = np.random.default_rng(seed)
    doc, _, total = T._graph("conv_dgrad", g, accumulate)
    dy = T.bf(rng.standard_normal((N, P, Q, K)))
    w = (rng.standard_normal((K, R, R, C)) / np.sqrt(R * R * K)).astype(np.float32)
    old = T.bf(rng.standard_normal((N, H, W, C)) if accumulate else np.zeros((N, H, W, C)))
    dx = T._from_bits(T._run(doc, total, {"dy": T._bits(dy), "w": w, "dx": T._bits(old)}, "dx", np.uint16),
                      (N, H, W, C))
    ref, _ = nm.conv2d_backward(np.zeros((N, H, W, C)), nm.round_bf16(w.astype(np.float64)),
                                dy.float().numpy().astype(np.float64), st, pad)
    if accumulate:
        ref = ref + old.float().numpy()
    return dx, nm.round_bf16(ref)


def wgrad(g, seed=13):
    N, H, W, C, K, R, st, pad, P, Q = _geom(g)
    rng = np.random.default_rng(seed)
    doc, _, total = T._graph("conv_wgrad", g)
    dy = T.bf(rng.standard_normal((N, P, Q, K)))
    x = T.bf(rng.standard_normal((N, H, W, C)))
    dw = T._run(doc, total, {"dy": T._bits(dy), "x": T._bits(x)}, "dw", np.float32).reshape(K, R, R, C)
    _, ref = nm.conv2d_backward(x.float().numpy().astype(np.float64), np.zeros((K, R, R, C)),
                                dy.float().numpy().astype(np.float64), st, pad)
    return dw, ref


def rows(g):
    N, H, W, C, K, R, st, pad, P, Q = _geom(g)
    return N * P * Q


# bench-scale shapes: units far above 148 CTAs / 74 pairs
SCALE = [  # N, H, W, C, K, R, stride, pad[, images per stem slice]
    (16, 56, 56, 64, 64, 3, 1, 1),        # ResNet-18 layer1 3x3 (M = 50176)
    (192, 28, 28, 128, 256, 3, 2, 1),     # ResNet-18 layer3 entry, stride 2: dgrad over 4 output phases
    (16, 56, 56, 64, 256, 1, 1, 0),       # ResNet-50 1x1 64 -> 256 (short reduction: single-CTA tiles)
    (32, 56, 56, 256, 512, 1, 2, 0),      # ResNet-50 1x1 stride-2 downsample (tap-less dgrad phases)
    (8, 224, 224, 3, 64, 7, 2, 3, 2),     # the 224^2 stem, four slices of 2 images (halo-tile kernels)
]


@pytest.mark.gpu
@pytest.mark.parametrize("g", SCALE)
def test_fprop_bench_scale(g):
    assert rows(g) >= 148 * 128      # at least one 128-row tile per SM: several units per CTA
    y, ref = fprop(g)
    assert nm.rel_l2(y, ref) < TOL_BF16
    assert np.max(np.abs(y - ref)) <= 2 ** -7 * np.max(np.abs(ref))


@pytest.mark.gpu
@pytest.mark.parametrize("g", SCALE[:4])
@pytest.mark.parametrize("accumulate", [False, True])
def test_dgrad_bench_scale(g, accumulate):
    dx, ref = dgrad(g, accumulate)
    assert nm.rel_l2(dx, ref) < TOL_BF16


@pytest.mark.gpu
@pytest.mark.parametrize("g", SCALE + [
    (16, 56, 56, 64, 64, 1, 1, 0),        # one 64 x 64 tile: split-K at its maximum (296 splits, 2 units per SM)
    (32, 14, 14, 256, 256, 3, 1, 1),      # 256-column CTA pairs
])
def test_wgrad_bench_scale(g):
    dw, ref = wgrad(g)
    assert nm.rel_l2(dw, ref) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("g", [SCALE[0], SCALE[2], SCALE[4]])
def test_fused_bn_stats_bench_scale(g, monkeypatch):
    """BN statistics summed by the epilogue across many units per CTA."""
    T.test_conv_fused_bn_stats(g, "", monkeypatch)


# ----------------------------------------------------------------- grid cap
CAP = "3"   # 3 single CTAs or 1 CTA pair


@pytest.mark.gpu
@pytest.mark.parametrize("g", T.SHAPES + T.PAD)
def test_capped_fprop(g, monkeypatch):
    monkeypatch.setenv("OC_CONV_MAX_CTAS", CAP)
    y, ref = fprop(g)
    assert nm.rel_l2(y, ref) < TOL_BF16


@pytest.mark.gpu
@pytest.mark.parametrize("g", T.SHAPES[:5] + T.PAD)
@pytest.mark.parametrize("accumulate", [False, True])
def test_capped_dgrad(g, accumulate, monkeypatch):
    monkeypatch.setenv("OC_CONV_MAX_CTAS", CAP)
    dx, ref = dgrad(g, accumulate)
    assert nm.rel_l2(dx, ref) < TOL_BF16


@pytest.mark.gpu
@pytest.mark.parametrize("g", T.SHAPES + T.PAD + T.WGRAD_PAIR_SHAPES + T.STEM_SHAPES)
def test_capped_wgrad(g, monkeypatch):
    monkeypatch.setenv("OC_CONV_MAX_CTAS", CAP)
    dw, ref = wgrad(g)
    assert nm.rel_l2(dw, ref) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("tile", T.TILES)
@pytest.mark.parametrize("g", T.TILE_SHAPES)
def test_capped_tiles(g, tile, monkeypatch):
    """Every forced fprop / dgrad tile kind, one CTA pair or three CTAs."""
    monkeypatch.setenv("OC_CONV_MAX_CTAS", CAP)
    monkeypatch.setenv("OC_CONV_TILE", tile)
    bn = int(tile.split(",")[0])
    if g[4] % bn == 0:
        y, ref = fprop(g)
        assert nm.rel_l2(y, ref) < TOL_BF16
    if g[3] % bn == 0:
        dx, ref = dgrad(g, True)
        assert nm.rel_l2(dx, ref) < TOL_BF16


@pytest.mark.gpu
@pytest.mark.parametrize("g,tile", T.STAT_CASES[:-1])
def test_capped_fused_bn_stats(g, tile, monkeypatch):
    monkeypatch.setenv("OC_CONV_MAX_CTAS", CAP)
    T.test_conv_fused_bn_stats(g, tile, monkeypatch)


@pytest.mark.gpu
@pytest.mark.parametrize("g", T.STEM_SHAPES)
def test_capped_stem(g, monkeypatch):
    monkeypatch.setenv("OC_CONV_MAX_CTAS", "2")
    y, ref = fprop(g)
    assert nm.rel_l2(y, ref) < TOL_BF16
    dw, ref = wgrad(g)
    assert nm.rel_l2(dw, ref) < 1e-5


# -------------------------------------------------- stem BN-ReLU-maxpool (tiled)
def _pool_graph(N, H, W, C):
    P, Q = (H + 2 - 3) // 2 + 1, (W + 2 - 3) // 2 + 1
    v = lambda n, b: {"id": n, "bytes": int(b), "pinned": True}
    vars_ = [v("y", N * H * W * C * 2), v("stat", 2 * C * 4), v("gamma", C * 4), v("beta", C * 4),
             v("out", N * P * Q * C * 2), v("idx", N * P * Q * C)]
    attrs = {"dtype": "bf16", "N": N, "H": H, "W": W, "C": C, "r": 3, "stride": 2, "pad": 1, "P": P, "Q": Q,
             "stat_in": True}
    fn = {"id": "f", "in": ["y", "stat", "gamma", "beta"], "out": ["out", "idx"],
          "op": {"kind": "bn_relu_pool_fwd", "args": {"y": "y", "stat": "stat", "gamma": "gamma", "beta": "beta",
                                                     "out": "out", "idx": "idx"}, "attrs": attrs}}
    return json.dumps({"variables": vars_, "functions": [fn]}), (P, Q), sum(x["bytes"] for x in vars_)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(16, 112, 112, 64), (3, 37, 23, 64)])
def test_bn_relu_pool_tiled(shape):
    """The stem's fused BN-apply + ReLU + 3x3/2 max pool (bn_relu_pool_rows,
    the row-staged hot-path kernel, for the even 112^2 map; the generic kernel
    for the odd one) against the definition: BN with the given
    batch statistics (fp32 [mu; rstd]), ReLU, bf16 storage rounding, max over
    the window, first maximum in row-major tap order (oracle maxpool).  The
    kernel evaluates gamma*(y-mu)*rstd+beta in fp32, the oracle in fp64, so a
    value within rounding of a bf16 boundary may round one ulp apart and move
    an argmax between near-equal taps: pooled values must agree within one
    ulp everywhere and to 1e-3 relative L2, and every argmax the kernel stores
    must point at a tap whose value is within one ulp of the window maximum;
    disagreements with the oracle's argmax must be rare (< 1e-3)."""
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    N, H, W, C = shape
    rng = np.random.default_rng(21)
    y = T.bf(rng.standard_normal((N, H, W, C)) * 1.5 + 0.3)
    yf = y.float().numpy().astype(np.float64)
    mu = yf.reshape(-1, C).mean(0)
    rstd = 1.0 / np.sqrt(yf.reshape(-1, C).var(0) + nm.BN_EPS)
    stat = np.stack([mu, rstd]).astype(np.float32)
    gamma = (1.0 + 0.1 * rng.standard_normal(C)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(C)).astype(np.float32)
    doc, (P, Q), total = _pool_graph(N, H, W, C)
    s = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in (("y", T._bits(y)), ("stat", stat), ("gamma", gamma), ("beta", beta)):
        s.write(k, a)
    s.step()
    out = T._from_bits(s.read("out", np.uint16), (N, P, Q, C))
    idx = s.read("idx", np.uint8).reshape(N, P, Q, C).astype(np.int64)
    s.close()
    st64 = stat.astype(np.float64)
    z = nm.round_bf16(np.maximum(gamma * (yf - st64[0]) * st64[1] + beta, 0.0))
    ref, arg = nm.maxpool(z, 3, 2, 1)
    # one bf16 ulp (upper bound), floored at the fp32 evaluation error of z
    ulp = np.maximum(np.abs(ref) * 2.0 ** -7, 1e-6)
    assert np.all(np.abs(out - ref) <= ulp)
    assert nm.rel_l2(out, ref) < TOL_BF16
    zp = np.full((N, H + 2, W + 2, C), -np.inf)
    zp[:, 1:H + 1, 1:W + 1] = z
    nn, pp, qq, cc = np.indices((N, P, Q, C))
    at = zp[nn, 2 * pp + idx // 3, 2 * qq + idx % 3, cc]
    assert np.all(np.abs(at - ref) <= ulp)
    assert np.mean(idx != arg) < 1e-3


@pytest.mark.gpu
def test_stem_at_the_r50_bench_batch_sampled():
    """The 7x7/2 stem at the R50 bench batch (1523 images: the whole input
    exceeds 2^31 elements once padded to 64 channels, so the per-slice
    tensor-core path must take it): sampled images against the oracle."""
    N, H, C, K = 1523, 224, 3, 64
    g = (N, H, H, C, K, 7, 2, 3)
    rng = np.random.default_rng(41)
    xs = rng.standard_normal((N, H, H, C)).astype(np.float32)
    x = T.bf(xs)
    w = (rng.standard_normal((K, 7, 7, C)) / np.sqrt(49 * C)).astype(np.float32)
    doc, (P, Q), total = T._graph("conv_fwd", g)
    y = T._run(doc, total, {"x": T._bits(x), "w": w}, "y", np.uint16).reshape(N, P * Q * K)
    wr = nm.round_bf16(w.astype(np.float64))
    for n in (0, 761, N - 1):
        ref = nm.round_bf16(nm.conv2d(x[n:n + 1].float().numpy().astype(np.float64), wr, 2, 3))
        got = T._from_bits(y[n], (1, P, Q, K))
        assert nm.rel_l2(got, ref) < TOL_BF16, n


# -------------------------------------------------- stem BN-ReLU-maxpool backward (row-staged kernels)
def _pool_bwd_graph(kind, N, H, W, C):
    P, Q = (H + 2 - 3) // 2 + 1, (W + 2 - 3) // 2 + 1
    v = lambda n, b: {"id": n, "bytes": int(b), "pinned": True}
    vars_ = [v("g", N * P * Q * C * 2), v("idx", N * P * Q * C), v("y", N * H * W * C * 2), v("stat", 2 * C * 4),
             v("gamma", C * 4), v("beta", C * 4), v("dgamma", C * 4), v("dbeta", C * 4)]
    attrs = {"dtype": "bf16", "N": N, "H": H, "W": W, "C": C, "r": 3, "stride": 2, "pad": 1, "P": P, "Q": Q}
    args = {k: k for k in ("g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta")}
    if kind == "reduce":
        fn = {"id": "f", "in": ["g", "idx", "y", "stat", "gamma", "beta"], "out": ["dgamma", "dbeta"],
              "op": {"kind": "pool_bn_bwd_reduce", "args": args, "attrs": attrs}}
    else:
        fn = {"id": "f", "in": ["g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta"], "out": ["y"],
              "op": {"kind": "pool_bn_bwd_apply", "args": args, "attrs": attrs}}
    return json.dumps({"variables": vars_, "functions": [fn]}), (P, Q), sum(x["bytes"] for x in vars_), attrs


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(32, 112, 112, 64), (3, 20, 36, 64), (2, 21, 23, 64)])
def test_pool_bn_backward(shape):
    """The stem's BN-ReLU-maxpool backward (pool_bn_bwd_reduce: dgamma, dbeta;
    pool_bn_bwd_apply: dy over y) against oracle/layerwise.py's definitions on
    the same bf16 inputs, argmax taps from the oracle's own forward pool.  The
    even stem shapes run the row-staged kernels (bulk-copied row pairs through
    a two-stage ring; 32 × 112² gives every persistent block several row pairs,
    so the ring's phases wrap), the odd shape the generic kernels.  bf16
    tolerance 1e-3 relative L2 (north_star)."""
    from oracle import layerwise as LW
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    N, H, W, C = shape
    rng = np.random.default_rng(23)
    y = T.bf(rng.standard_normal((N, H, W, C)) * 1.5 + 0.3)
    yf = y.float().numpy().astype(np.float64)
    mu = yf.reshape(-1, C).mean(0)
    rstd = 1.0 / np.sqrt(yf.reshape(-1, C).var(0) + nm.BN_EPS)
    stat = np.stack([mu, rstd]).astype(np.float32)
    gamma = (1.0 + 0.1 * rng.standard_normal(C)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(C)).astype(np.float32)
    st64 = stat.astype(np.float64)
    z = nm.round_bf16(np.maximum(gamma * (yf - st64[0]) * st64[1] + beta, 0.0))
    _, arg = nm.maxpool(z, 3, 2, 1)
    P, Q = arg.shape[1:3]
    g = T.bf(rng.standard_normal((N, P, Q, C)))
    gf = g.float().numpy().astype(np.float64)
    ins = {"g": gf, "idx": arg.astype(np.uint8), "y": yf, "stat": st64, "gamma": gamma.astype(np.float64),
           "beta": beta.astype(np.float64)}
    doc, _, total, attrs = _pool_bwd_graph("reduce", N, H, W, C)
    ref = LW.apply("pool_bn_bwd_reduce", attrs, ins)
    s = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in (("g", T._bits(g)), ("idx", arg.astype(np.uint8)), ("y", T._bits(y)), ("stat", stat),
                 ("gamma", gamma), ("beta", beta)):
        s.write(k, a)
    s.step()
    dgamma, dbeta = s.read("dgamma", np.float32), s.read("dbeta", np.float32)
    s.close()
    assert nm.rel_l2(dgamma, ref["dgamma"]) < TOL_BF16
    assert nm.rel_l2(dbeta, ref["dbeta"]) < TOL_BF16
    # apply, from the oracle's dgamma / dbeta (the kernel is tested on its own)
    dg32, db32 = ref["dgamma"].astype(np.float32), ref["dbeta"].astype(np.float32)
    doc, _, total, attrs = _pool_bwd_graph("apply", N, H, W, C)
    ref_dy = LW.apply("pool_bn_bwd_apply", attrs, dict(ins, dgamma=dg32.astype(np.float64),
                                                         dbeta=db32.astype(np.float64)))["y"]
    s = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in (("g", T._bits(g)), ("idx", arg.astype(np.uint8)), ("y", T._bits(y)), ("stat", stat),
                 ("gamma", gamma), ("beta", beta), ("dgamma", dg32), ("dbeta", db32)):
        s.write(k, a)
    s.step()
    dy = T._from_bits(s.read("y", np.uint16), (N, H, W, C))
    s.close()
    assert nm.rel_l2(dy, ref_dy.reshape(N, H, W, C)) < TOL_BF16
