"""Pins of the numerics oracle (oracle/numerics.py) against things other
than itself: library routines (torch's bf16 conversion, scipy's correlate and
logsumexp, numpy matmul), central finite differences in float64, closed forms
(BN output moments, one SGD step from zero momentum) and brute-force loops."""
import copy

import numpy as np
import pytest
import scipy.signal
import scipy.special
import torch

from oracle import numerics as nm
from synth import nets


def test_round_bf16_matches_library_conversion():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000) * 10.0 ** rng.integers(-6, 6, 100000),
                        [0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.0e38, -2.5]]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    got = nm.round_bf16(x.astype(np.float64))
    assert np.array_equal(ref, got)


def test_conv2d_matches_correlate_and_matmul():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 9, 11, 1))
    w = rng.standard_normal((1, 3, 3, 1))
    y = nm.conv2d(x, w, 1, 1)
    ref = scipy.signal.correlate(np.pad(x[0, :, :, 0], 1), w[0, :, :, 0], mode="valid")
    assert np.allclose(y[0, :, :, 0], ref)
    # stride 2: every other output of the stride-1 result
    y2 = nm.conv2d(x, w, 2, 1)
    assert np.allclose(y2[0, :, :, 0], ref[::2, ::2])
    # 1x1 conv == matmul over channels
    x = rng.standard_normal((2, 5, 4, 6))
    w = rng.standard_normal((3, 1, 1, 6))
    assert np.allclose(nm.conv2d(x, w, 1, 0), x @ w[:, 0, 0, :].T)


def _fd(f, arr, idx, eps=1e-6):
    old = arr[idx]
    arr[idx] = old + eps
    fp = f()
    arr[idx] = old - eps
    fm = f()
    arr[idx] = old
    return (fp - fm) / (2 * eps)


def test_conv2d_backward_finite_differences():
    rng = np.random.default_rng(2)
    for stride, pad, R in ((1, 1, 3), (2, 1, 3), (2, 3, 7), (2, 0, 1)):
        x = rng.standard_normal((2, 9, 8, 3))
        w = rng.standard_normal((4, R, R, 3))
        y = nm.conv2d(x, w, stride, pad)
        G = rng.standard_normal(y.shape)
        dx, dw = nm.conv2d_backward(x, w, G, stride, pad)
        f = lambda: float((nm.conv2d(x, w, stride, pad) * G).sum())
        for _ in range(6):
            i = tuple(int(rng.integers(0, s)) for s in x.shape)
            assert abs(_fd(f, x, i) - dx[i]) < 1e-5 * (1 + abs(dx[i]))
            j = tuple(int(rng.integers(0, s)) for s in w.shape)
            assert abs(_fd(f, w, j) - dw[j]) < 1e-5 * (1 + abs(dw[j]))


def test_maxpool_brute_force_and_first_max():
    rng = np.random.default_rng(3)
    x = np.round(rng.standard_normal((2, 7, 6, 3)), 1)   # many ties
    out, arg = nm.maxpool(x, 3, 2, 1)
    N, H, W, C = x.shape
    for n in range(N):
        for p in range(out.shape[1]):
            for q in range(out.shape[2]):
                for c in range(C):
                    best, bi = -np.inf, None
                    for i in range(3):
                        for j in range(3):
                            h, w_ = p * 2 - 1 + i, q * 2 - 1 + j
                            if 0 <= h < H and 0 <= w_ < W and x[n, h, w_, c] > best:
                                best, bi = x[n, h, w_, c], i * 3 + j
                    assert out[n, p, q, c] == best and arg[n, p, q, c] == bi
    G = rng.standard_normal(out.shape)
    dx = nm.maxpool_backward(G, arg, x.shape, 3, 2, 1)
    assert np.isclose(dx.sum(), G.sum())


def test_softmax_ce_closed_form_and_fd():
    rng = np.random.default_rng(4)
    z = rng.standard_normal((5, 7)) * 3
    y = rng.integers(0, 7, 5)
    loss, dz = nm.softmax_ce(z, y)
    ref = np.mean(scipy.special.logsumexp(z, axis=1) - z[np.arange(5), y])
    assert np.isclose(loss, ref)
    for _ in range(5):
        i = (int(rng.integers(0, 5)), int(rng.integers(0, 7)))
        assert abs(_fd(lambda: nm.softmax_ce(z, y)[0], z, i) - dz[i]) < 1e-7
    assert np.allclose(dz.sum(axis=1), 0.0)


def _fd_check_spec(spec, n_checks=12, tol=2e-5, seed=5):
    spec = copy.deepcopy(spec)
    spec["mode"] = "fp64"
    x, y = nets.make_inputs(spec)
    params = {k: v.astype(np.float64) for k, v in nets.make_params(spec).items()}
    res = nm.train_step(spec, params, x, y)
    rng = np.random.default_rng(seed)
    names = sorted(params)
    for _ in range(n_checks):
        k = names[int(rng.integers(0, len(names)))]
        idx = tuple(int(rng.integers(0, s)) for s in params[k].shape)
        f = lambda: nm.train_step(spec, params, x, y)["loss"]
        num = _fd(f, params[k], idx, eps=1e-6)
        ana = res["grads"][k][idx]
        assert abs(num - ana) <= tol * (abs(ana) + 1e-3), (k, idx, num, ana)


def test_mlp_gradients_finite_differences():
    _fd_check_spec(nets.mlp6(batch=4, width=16, classes=10), n_checks=20)


def test_tiny_resnet_gradients_finite_differences():
    spec = nets.tiny_resnet(batch=2, image=16, classes=5)
    _fd_check_spec(spec, n_checks=16, tol=5e-5)


def test_conv_transpose_is_adjoint_of_strided_conv():
    """<convT(x, W), y> = <x, conv(y, W')> with W'[c, i, j, k] -> KRSC [c][i][j][k]
    as the 2×2 stride-2 conv from the K-channel map to the C-channel map: the
    transposed conv is the adjoint (textbook definition)."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((2, 3, 4, 5))
    w = rng.standard_normal((5, 2, 2, 6))          # [C_in, 2, 2, K_out]
    y = rng.standard_normal((2, 6, 8, 6))
    lhs = np.sum(nm.conv_transpose2x2(x, w) * y)
    rhs = np.sum(x * nm.conv2d(y, w, 2, 0))        # w as KRSC with K=C_in, C=K_out
    assert np.isclose(lhs, rhs)
    G = rng.standard_normal((2, 6, 8, 6))
    dx, dw = nm.conv_transpose2x2_backward(x, w, G)
    f = lambda: float(np.sum(nm.conv_transpose2x2(x, w) * G))
    for _ in range(5):
        i = tuple(int(rng.integers(0, s)) for s in x.shape)
        assert abs(_fd(f, x, i) - dx[i]) < 1e-6 * (1 + abs(dx[i]))
        j = tuple(int(rng.integers(0, s)) for s in w.shape)
        assert abs(_fd(f, w, j) - dw[j]) < 1e-6 * (1 + abs(dw[j]))


def test_unet_gradients_finite_differences():
    """U-Net pieces: concat-conv (two inputs), 2×2 max-pool with a skip consumer,
    transposed conv, per-pixel softmax cross-entropy."""
    spec = nets.unet(batch=2, image=8, base=4, depth=2, classes=3)
    _fd_check_spec(spec, n_checks=24, tol=5e-5)


def test_preact_resnet_gradients_finite_differences():
    """Pre-activation bottleneck blocks (add layer, BN on a tensor with two
    consumers, projection shortcuts): depth 11 = one block per stage."""
    spec = nets.preact_resnet(depth=11, batch=4, image=8, classes=5)
    _fd_check_spec(spec, n_checks=20, tol=5e-5)


def test_bn_output_moments_and_sgd_closed_form():
    spec = nets.mlp6(batch=8, width=32, classes=10)
    spec["mode"] = "fp64"
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    r = nm.train_step(spec, p, x, y)
    for k in p:   # v = g, w' = w - lr g from zero momentum
        assert np.allclose(r["momentum"][k], r["grads"][k])
        assert np.allclose(r["params"][k], p[k] - spec["sgd"]["lr"] * r["grads"][k])
    # BN without ReLU: per-channel output mean = beta, var = gamma^2 var/(var+eps)
    rng = np.random.default_rng(6)
    xin = rng.standard_normal((4, 5, 5, 3)) * 2 + 1
    sp = {"mode": "fp64", "layers": [{"type": "bn", "name": "b", "in": "x", "out": "o", "relu": False,
                                      "residual": None},
                                     {"type": "gap", "name": "g", "in": "o", "out": "f"},
                                     {"type": "linear", "name": "fc", "in": "f", "out": "logits",
                                      "features": 2, "relu": False}],
          "loss": {"type": "softmax_ce", "in": "logits"}, "sgd": {"lr": 0.1, "momentum": 0.9}}
    prm = {"b.gamma": np.array([1.5, 2.0, 0.5]), "b.beta": np.array([0.1, -0.2, 0.3]),
           "fc.W": np.zeros((2, 3)), "fc.b": np.zeros(2)}
    out = nm.train_step(sp, prm, xin, np.array([0, 1, 0, 1]))["acts"]["o"]
    var = xin.var(axis=(0, 1, 2))
    assert np.allclose(out.mean(axis=(0, 1, 2)), prm["b.beta"])
    assert np.allclose(out.var(axis=(0, 1, 2)), prm["b.gamma"] ** 2 * var / (var + nm.BN_EPS))


def test_bf16_mode_close_to_fp64_where_well_conditioned():
    """The bf16 storage contract perturbs the fp64 step by O(bf16 eps) where
    the computation is well conditioned: the loss and the last layer's
    gradients.  (Deeper gradients pass through BN backward, whose mean and
    projection subtractions cancel most of dz after a global average pool, so
    bf16 storage moves them by ~10-20% at these tiny batch sizes — a property
    of bf16 training, which is why GPU parity compares against the oracle at
    the SAME rounding points, Z23.)"""
    spec = nets.tiny_resnet(batch=8, image=32, classes=5)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    r16 = nm.train_step(spec, p, x, y)
    s64 = copy.deepcopy(spec)
    s64["mode"] = "fp64"
    r64 = nm.train_step(s64, p, x, y)
    assert abs(r16["loss"] - r64["loss"]) < 1e-3 * abs(r64["loss"])
    assert nm.rel_l2(r16["grads"]["fc.W"], r64["grads"]["fc.W"]) < 2e-2
    assert nm.rel_l2(r16["grads"]["fc.b"], r64["grads"]["fc.b"]) < 2e-2
    assert nm.rel_l2(r16["acts"]["feat"], r64["acts"]["feat"]) < 2e-2


def test_bf16_deep_net_gradients_are_chaotic():
    """Why the deep bf16 GPU-vs-oracle comparison is made on the loss, per
    kernel and in fp32: perturbing ONE conv output of ResNet-18
    by 1e-6 relative noise — the size of fp32 accumulation-order differences —
    moves the oracle's own bf16-mode parameter gradients by >10%, because bf16
    rounding turns sub-ulp differences into ulp jumps that grow layer by layer;
    in fp32 mode the same perturbation moves them by <1e-4."""
    spec = nets.resnet(18, batch=8, image=64)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    shape = p["conv1.W"].shape
    orig = nm.conv2d
    out = {}
    for mode in ("bf16", "fp32"):
        spec["mode"] = mode
        r0 = nm.train_step(spec, p, x, y)
        rng = np.random.default_rng(0)

        def noisy(xx, w, st, pad, dil=1):
            yy = orig(xx, w, st, pad, dil)
            return yy * (1 + 1e-6 * rng.standard_normal(yy.shape)) if w.shape == shape else yy
        nm.conv2d = noisy
        try:
            r1 = nm.train_step(spec, p, x, y)
        finally:
            nm.conv2d = orig
        out[mode] = np.median([nm.rel_l2(r1["grads"][k], r0["grads"][k]) for k in p])
    assert out["bf16"] > 1e-1 and out["fp32"] < 1e-4, out


# ---------------------------------------------------------------- GAN step (configs[4])


def test_upsample_avgpool_loops_and_adjoints():
    """upsample2 / avgpool2 against explicit loops, and each backward is the
    adjoint of its forward (<f(x), y> = <x, f*(y)>)."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 4, 5))
    up = nm.upsample2(x)
    for i in range(6):
        for j in range(8):
            assert np.array_equal(up[:, i, j], x[:, i // 2, j // 2])
    y = rng.standard_normal(up.shape)
    assert np.isclose((up * y).sum(), (x * nm.upsample2_backward(y)).sum())
    x2 = rng.standard_normal((2, 6, 4, 3))
    ap = nm.avgpool2(x2)
    for i in range(3):
        for j in range(2):
            assert np.allclose(ap[:, i, j], x2[:, 2 * i:2 * i + 2, 2 * j:2 * j + 2].mean(axis=(1, 2)))
    y2 = rng.standard_normal(ap.shape)
    assert np.isclose((ap * y2).sum(), (x2 * nm.avgpool2_backward(y2)).sum())


def test_attention_definition_and_finite_differences():
    """SAGAN attention: per-position loops of the definition, rows of P sum to
    one, and the backward against central differences (fp64)."""
    rng = np.random.default_rng(1)
    N, L, dq, dv = 2, 5, 3, 4
    q, k = rng.standard_normal((N, L, dq)), rng.standard_normal((N, L, dq))
    v = rng.standard_normal((N, L, dv))
    ident = nm.rounder("fp64")
    P, o = nm.attention(q, k, v, ident)
    for n in range(N):
        for i in range(L):
            s = np.array([q[n, i] @ k[n, j] for j in range(L)])
            p = np.exp(s - s.max()) / np.exp(s - s.max()).sum()
            assert np.allclose(P[n, i], p) and np.allclose(o[n, i], p @ v[n])
    assert np.allclose(P.sum(axis=2), 1.0)
    R = rng.standard_normal(o.shape)
    dq_, dk_, dv_ = nm.attention_backward(q, k, v, P, o, R)
    f = lambda: (nm.attention(q, k, v, ident)[1] * R).sum()
    for arr, grad in ((q, dq_), (k, dk_), (v, dv_)):
        for idx in [(0, 1, 2), (1, 4, 0), (1, 0, 1)]:
            assert abs(_fd(f, arr, idx) - grad[idx]) < 1e-7 * (1 + abs(grad[idx]))


def test_hinge_loss_closed_form():
    s = np.array([2.0, 0.5, -0.5, -2.0])     # two real, two fake
    loss, ds = nm.hinge_d(s, 2)
    assert np.isclose(loss, (0 + 0.5) / 2 + (0.5 + 0) / 2)
    assert np.allclose(ds, [0.0, -0.5, 0.5, 0.0])


def test_gan_step_gradients_finite_differences():
    """tiny BigGAN (every layer kind: linear->reshape, BN-ReLU, nearest
    upsampling, convs, residual adds, attention, tanh, ReLU, average pooling,
    GAP, linear score) in fp64: the D-step gradients against central
    differences of the hinge loss; the G-step gradients against central
    differences of −mean D'(G(z2)) with D' the updated discriminator held fixed."""
    spec = nets.tiny_biggan(batch=3, mode="fp64")
    pG, pD = nets.make_gan_params(spec)
    pG = {k: v.astype(np.float64) for k, v in pG.items()}
    pD = {k: v.astype(np.float64) for k, v in pD.items()}
    z1, z2, x = nets.make_gan_inputs(spec)
    res = nm.gan_step(spec, pG, pD, z1, z2, x)
    G_, D_ = spec["G"], spec["D"]

    def d_loss():
        a = {"z": z1.astype(np.float64)}
        nm._Net(G_["layers"], pG, "fp64").forward(a)
        ad = {"x": np.concatenate([x.astype(np.float64), a[G_["out"]]])}
        nm._Net(D_["layers"], pD, "fp64").forward(ad, fp32_out=(D_["out"],))
        return nm.hinge_d(ad[D_["out"]].reshape(-1), 3)[0]

    pD_new = res["pD"]

    def g_loss():
        a = {"z": z2.astype(np.float64)}
        nm._Net(G_["layers"], pG, "fp64").forward(a)
        ad = {"x": a[G_["out"]]}
        nm._Net(D_["layers"], pD_new, "fp64").forward(ad, fp32_out=(D_["out"],))
        return float(-ad[D_["out"]].mean())

    assert np.isclose(d_loss(), res["loss_d"]) and np.isclose(g_loss(), res["loss_g"])
    rng = np.random.default_rng(7)
    for params, grads, f in ((pD, res["gradsD"], d_loss), (pG, res["gradsG"], g_loss)):
        names = sorted(params)
        for _ in range(16):
            k = names[int(rng.integers(0, len(names)))]
            idx = tuple(int(rng.integers(0, s)) for s in params[k].shape)
            num = _fd(f, params[k], idx, eps=1e-6)
            ana = grads[k][idx]
            assert abs(num - ana) <= 2e-5 * (abs(ana) + 1e-3), (k, idx, num, ana)
    for k in pG:     # every G parameter, attention included, receives a gradient
        assert np.abs(res["gradsG"][k]).max() > 0, k


def test_densenet_gradients_finite_differences():
    """tiny DenseNet-BC: concatenation, average-pool transitions,
    BN inputs with two consumers — every parameter kind against central
    differences (fp64)."""
    _fd_check_spec(nets.tiny_densenet(batch=3, image=16, classes=5), n_checks=20)
