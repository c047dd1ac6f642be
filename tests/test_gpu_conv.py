"""Kernel-level parity of the convolution ops (tcgen05 implicit GEMM and the
CUDA-core fallback) with the oracle's direct-definition convolution, through
the C-ABI executor on one-function graphs: several tiles, ragged M tails,
stride 1 and 2, 1×1 and 3×3 filters, 64- and 128-wide N tiles, dgrad
accumulation and the deterministic split-K wgrad.  bf16 outputs within
north_star's 1e-3 relative L2, fp32 weight gradients within 1e-5."""
import json

import numpy as np
import pytest
import torch

from oracle import numerics as nm

SHAPES = [  # N, H, W, C, K, R, stride, pad
    (2, 9, 7, 64, 64, 3, 1, 1),
    (3, 11, 10, 64, 128, 3, 2, 1),
    (2, 12, 9, 64, 128, 1, 2, 0),
    (1, 8, 8, 128, 128, 3, 1, 1),
    (2, 7, 7, 128, 64, 3, 1, 1),
    (2, 15, 13, 3, 64, 7, 2, 3),      # stem: 3 channels zero-padded to 8, one tap per 16-byte chunk
    (3, 17, 16, 3, 64, 7, 2, 3, 2),   # ... in slices of 2 images (ragged last slice)
    (2, 9, 11, 16, 64, 3, 1, 1),      # 16 channels: 4 taps per K-block
    (3, 10, 9, 5, 128, 3, 2, 1, 1),   # 5 channels, BN = 128, one image per slice
    (2, 16, 14, 3, 64, 7, 2, 3),      # stride-2 stem, even H, W: space-to-depth 4x4 conv over 16 channels
    (3, 18, 12, 3, 128, 7, 2, 3, 2),  # ... BN = 128, slices of 2 images
    (2, 10, 12, 3, 64, 3, 2, 1),      # 3x3 stride 2 -> 2x2 space-to-depth taps
]
# channel counts the 64-wide tiles do not divide: operands zero-padded to 64 in
# workspace copies, weights padded, only the real channels stored
PAD = [
    (2, 9, 7, 32, 16, 3, 1, 1),       # ResNet-1001-like 32 -> 16
    (3, 8, 8, 16, 32, 1, 1, 0),       # 16 -> 32, 1x1 (fprop gathers 16-ch pixels)
    (2, 10, 9, 96, 96, 3, 2, 1),      # BigGAN-like 96 channels, stride 2 (dgrad phases): X and dY read in
                                      # place, the TMA engine zero-fills channels 96..127
    (2, 9, 8, 160, 96, 3, 1, 1),      # DenseNet-like 160 -> 96, both operands read in place
    (3, 8, 7, 224, 128, 1, 1, 0),     # DenseNet bottleneck 1x1 224 -> 128
    (2, 6, 6, 64, 24, 1, 1, 0),       # attention-like 64 -> 24
    (2, 8, 8, 24, 64, 3, 1, 1),       # 24 -> 64
    # output channels not a multiple of 8: fprop stores through a padded
    # workspace output, dgrad / wgrad read a padded dY copy
    (2, 9, 8, 64, 3, 7, 1, 3),        # Pix2PixHD image head 64 -> 3, 7x7
    (2, 6, 7, 64, 21, 1, 1, 0),       # DeepLabv3+ class head -> 21
    (2, 10, 9, 32, 3, 3, 2, 1),       # K = 3, stride 2 (dgrad phases)
]


def bf(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


def _graph(kind, g, accumulate=False):
    N, H, W, C, K, R, st, pad = g[:8]
    P = (H + 2 * pad - R) // st + 1
    Q = (W + 2 * pad - R) // st + 1
    attrs = {"N": N, "H": H, "W": W, "C": C, "K": K, "R": R, "S": R, "stride": st, "pad": pad, "P": P, "Q": Q,
             "accumulate": accumulate}
    if len(g) > 8:
        attrs["pad_slice"] = g[8]
    v = lambda n, b: {"id": n, "bytes": int(b), "pinned": True}
    xs, ys, ws = N * H * W * C * 2, N * P * Q * K * 2, K * R * R * C * 4
    if kind == "conv_fwd":
        vars_ = [v("x", xs), v("w", ws), v("y", ys)]
        fn = {"id": "f", "in": ["x", "w"], "out": ["y"], "op": {"kind": kind, "args": {"x": "x", "w": "w", "y": "y"},
                                                             "attrs": attrs}}
    elif kind == "conv_dgrad":
        vars_ = [v("dy", ys), v("w", ws), v("dx", xs)]
        fn = {"id": "f", "in": ["dy", "w"] + (["dx"] if accumulate else []), "out": ["dx"],
              "op": {"kind": kind, "args": {"dy": "dy", "w": "w", "dx": "dx"}, "attrs": attrs}}
    else:
        vars_ = [v("dy", ys), v("x", xs), v("dw", ws)]
        fn = {"id": "f", "in": ["dy", "x"], "out": ["dw"], "op": {"kind": kind, "args": {"dy": "dy", "x": "x", "dw": "dw"},
                                                               "attrs": attrs}}
    doc = json.dumps({"variables": vars_, "functions": [fn]})
    return doc, (P, Q), sum(x["bytes"] for x in vars_)


def _run(doc, total, inputs, out_name, out_dtype):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in inputs.items():
        st.write(k, a)
    st.step()
    r = st.read(out_name, out_dtype)
    st.close()
    return r


def _bits(t):
    return t.view(torch.int16).numpy()


def _from_bits(a, shape):
    return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).float().numpy().reshape(shape).astype(np.float64)


# narrow inputs (an image) whose output width is not a multiple of 64: the
# forward runs 64-multiple weight rows and stores the real columns; the data gradient through a
# 64-channel padded workspace output (real channels copied or added out), the
# weight gradient through a 16-channel padded copy of X when K needs padding
NARROW_BWD = [
    (2, 12, 10, 3, 96, 3, 1, 1),      # BigGAN discriminator input conv 3 -> 96
    (2, 9, 8, 3, 96, 1, 1, 0),        # ... and its 1x1 shortcut
    (3, 10, 9, 5, 64, 3, 2, 1),       # 5 channels, stride 2 (dgrad phases)
    (2, 11, 7, 3, 16, 3, 1, 1),       # ResNet-1001 input conv 3 -> 16
]


@pytest.mark.gpu
@pytest.mark.parametrize("g", SHAPES + PAD + NARROW_BWD)
def test_conv_fwd(g):
    N, H, W, C, K, R, st, pad = g[:8]
    rng = np.random.default_rng(1)
    x = bf(rng.standard_normal((N, H, W, C)))
    w = rng.standard_normal((K, R, R, C)).astype(np.float32) * 0.1
    doc, (P, Q), total = _graph("conv_fwd", g)
    y = _run(doc, total, {"x": _bits(x), "w": w}, "y", np.uint16)
    y = _from_bits(y, (N, P, Q, K))
    ref = nm.round_bf16(nm.conv2d(x.float().numpy().astype(np.float64), nm.round_bf16(w.astype(np.float64)), st, pad))
    assert nm.rel_l2(y, ref) < 1e-3
    assert np.max(np.abs(y - ref)) <= 2 ** -7 * np.max(np.abs(ref)) + 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("g", SHAPES[:5] + PAD + NARROW_BWD)
@pytest.mark.parametrize("accumulate", [False, True])
def test_conv_dgrad(g, accumulate):
    N, H, W, C, K, R, st, pad = g[:8]
    rng = np.random.default_rng(2)
    doc, (P, Q), total = _graph("conv_dgrad", g, accumulate)
    dy = bf(rng.standard_normal((N, P, Q, K)))
    w = rng.standard_normal((K, R, R, C)).astype(np.float32) * 0.1
    old = bf(rng.standard_normal((N, H, W, C))) if accumulate else bf(np.zeros((N, H, W, C)))
    dx = _run(doc, total, {"dy": _bits(dy), "w": w, "dx": _bits(old)}, "dx", np.uint16)
    dx = _from_bits(dx, (N, H, W, C))
    x0 = np.zeros((N, H, W, C))
    ref, _ = nm.conv2d_backward(x0, nm.round_bf16(w.astype(np.float64)), dy.float().numpy().astype(np.float64), st, pad)
    if accumulate:
        ref = ref + old.float().numpy()
    ref = nm.round_bf16(ref)
    assert nm.rel_l2(dx, ref) < 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("g", SHAPES + PAD + NARROW_BWD)
def test_conv_wgrad(g):
    N, H, W, C, K, R, st, pad = g[:8]
    rng = np.random.default_rng(3)
    doc, (P, Q), total = _graph("conv_wgrad", g)
    dy = bf(rng.standard_normal((N, P, Q, K)))
    x = bf(rng.standard_normal((N, H, W, C)))
    dw = _run(doc, total, {"dy": _bits(dy), "x": _bits(x)}, "dw", np.float32).reshape(K, R, R, C)
    _, ref = nm.conv2d_backward(x.float().numpy().astype(np.float64), np.zeros((K, R, R, C)),
                                dy.float().numpy().astype(np.float64), st, pad)
    assert nm.rel_l2(dw, ref) < 1e-5


# CTA-pair (cta_group::2) tiles and the single-CTA ones, forced per launch
# (OC_CONV_TILE = "N-tile,tiles per unit,CTAs"): ragged M tails that leave the
# second CTA of a pair, or the second tile of a unit, past the last row
TILES = ["256,1,2", "128,2,2", "64,2,2", "128,2,1", "64,1,1"]
TILE_SHAPES = [  # N, H, W, C, K, R, stride, pad
    (2, 9, 7, 64, 256, 3, 1, 1),      # M = 126: one pair, the second CTA's rows all past M
    (3, 11, 10, 256, 256, 3, 2, 1),   # stride 2 (dgrad: 4 phases)
    (2, 12, 9, 128, 256, 1, 2, 0),    # 1x1 stride 2 (dgrad: tap-less phases)
    (5, 13, 13, 128, 128, 3, 1, 1),   # M = 845: several pairs and a ragged tail
    (4, 9, 9, 256, 64, 3, 1, 1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("g", TILE_SHAPES)
def test_conv_tiles_fwd(g, tile, monkeypatch):
    if g[4] % int(tile.split(",")[0]):
        pytest.skip("N tile does not divide K")
    monkeypatch.setenv("OC_CONV_TILE", tile)
    test_conv_fwd(g)


@pytest.mark.gpu
@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("g", TILE_SHAPES)
def test_conv_tiles_dgrad(g, tile, monkeypatch):
    if g[3] % int(tile.split(",")[0]):
        pytest.skip("N tile does not divide C")
    monkeypatch.setenv("OC_CONV_TILE", tile)
    test_conv_dgrad(g, True)


# weight gradient on CTA pairs (K divisible by 128: 256 (r,s,c) rows × 128 / 256
# columns per pair) against single CTAs (OC_WGRAD_CG=1)
WGRAD_PAIR_SHAPES = [
    (2, 9, 7, 64, 256, 3, 1, 1),      # M = 576: the second CTA of the last pair holds 64 rows
    (3, 11, 10, 128, 128, 3, 2, 1),
    (2, 12, 9, 256, 512, 1, 2, 0),    # M = 256: one pair
    (2, 7, 7, 192, 256, 3, 1, 1),     # M = 1728
]


@pytest.mark.gpu
@pytest.mark.parametrize("cg", ["2", "1"])
@pytest.mark.parametrize("g", WGRAD_PAIR_SHAPES)
def test_conv_wgrad_pairs(g, cg, monkeypatch):
    monkeypatch.setenv("OC_WGRAD_CG", cg)
    test_conv_wgrad(g)


# conv_fwd with attrs.bn_stat: the batch statistics [μ; rstd] of the stored y
# for the BN that consumes it — from the tensor-core epilogue's per-channel
# partial sums (pairs, single CTAs, narrow stem slices) or, on the CUDA-core
# path, the BN reduction over y — against the definition over the stored
# bf16 values (biased variance, eps 1e-5; oracle/numerics.py)
STAT_CASES = [
    ((2, 9, 7, 64, 256, 3, 1, 1), "256,1,2"),
    ((5, 13, 13, 128, 128, 3, 1, 1), "128,2,2"),
    ((5, 13, 13, 128, 128, 3, 1, 1), "128,2,1"),
    ((4, 9, 9, 256, 64, 3, 1, 1), "64,2,2"),
    ((3, 11, 10, 64, 128, 3, 2, 1), ""),
    ((3, 17, 16, 3, 64, 7, 2, 3, 2), ""),      # stem: space-to-depth slices of 2 images
    ((2, 15, 13, 3, 64, 7, 2, 3), ""),         # 8-channel pixels
    ((2, 12, 10, 3, 96, 3, 1, 1), ""),         # narrow input, K = 96 (padded weight rows; statistics pass)
    ((2, 9, 7, 64, 64, 3, 1, 1), "simt"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("g,tile", STAT_CASES)
def test_conv_fused_bn_stats(g, tile, monkeypatch):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    N, H, W, C, K, R, st, pad = g[:8]
    if tile and tile != "simt":
        monkeypatch.setenv("OC_CONV_TILE", tile)
    doc, (P, Q), total = _graph("conv_fwd", g)
    d = json.loads(doc)
    d["variables"].append({"id": "stat", "bytes": 2 * K * 4, "pinned": True})
    f = d["functions"][0]
    f["out"].append("stat")
    f["op"]["args"]["stat"] = "stat"
    f["op"]["attrs"]["bn_stat"] = True
    if tile == "simt":
        f["op"]["attrs"]["impl"] = "simt"
    doc = json.dumps(d)
    rng = np.random.default_rng(5)
    x = bf(rng.standard_normal((N, H, W, C)))
    w = rng.standard_normal((K, R, R, C)).astype(np.float32) * 0.1 + 0.02
    s = OutOfCoreStep(doc, total + 2 * K * 4, 0, mode="best", phys_bytes=4096)
    s.write("x", _bits(x))
    s.write("w", w)
    s.step()
    y = _from_bits(s.read("y", np.uint16), (N * P * Q, K))
    stat = s.read("stat", np.float32).reshape(2, K)
    s.close()
    mu = y.mean(0)
    var = np.maximum((y * y).mean(0) - mu * mu, 0)
    rstd = 1 / np.sqrt(var + 1e-5)
    sd = np.sqrt(var)
    assert np.all(np.abs(stat[0] - mu) <= 2e-5 * (np.abs(mu) + sd) + 1e-7)
    assert np.max(np.abs(stat[1] / rstd - 1)) < 2e-5


# the halo-tile stem kernel (space-to-depth 4x4 conv, 64 outputs, output map
# tiled by 16 x 8 blocks): exact tilings, image slices, zero padding at every
# border; and the same shapes on the im2col kernel (OC_CONV_STEM=0)
STEM_SHAPES = [(2, 32, 32, 3, 64, 7, 2, 3), (3, 32, 48, 3, 64, 7, 2, 3, 2), (1, 64, 16, 3, 64, 7, 2, 3)]


@pytest.mark.gpu
@pytest.mark.parametrize("stem", ["1", "0"])
@pytest.mark.parametrize("g", STEM_SHAPES)
def test_conv_stem_halo(g, stem, monkeypatch):
    monkeypatch.setenv("OC_CONV_STEM", stem)
    test_conv_fwd(g)
    test_conv_wgrad(g)


@pytest.mark.gpu
@pytest.mark.parametrize("g", STEM_SHAPES[:2])
def test_conv_stem_halo_fused_bn_stats(g, monkeypatch):
    test_conv_fused_bn_stats(g, "", monkeypatch)
