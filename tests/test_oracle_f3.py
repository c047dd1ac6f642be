"""Pins of the oracle pieces added for the paper's other two families (SURVEY
§8(f) F3; Pix2PixHD on 512×1024, DeepLabv3+ on 513×513)
against things other than the oracle itself: library routines (scipy's
correlate with a zero-dilated kernel, torch's bilinear interpolation and
transposed convolution, numpy's reflect padding — all in float64), adjoint
identities, closed forms, and central finite differences through whole
miniature networks."""
import numpy as np
import scipy.signal
import torch
import torch.nn.functional as F

from oracle import numerics as nm
from synth import nets

from test_oracle_numerics import _fd, _fd_check_spec


def test_dilated_conv_matches_correlate_with_dilated_kernel():
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 13, 12, 1))
    w = rng.standard_normal((1, 3, 3, 1))
    for d in (1, 2, 3):
        wd = np.zeros((2 * d + 1, 2 * d + 1))
        wd[::d, ::d] = w[0, :, :, 0]
        ref = scipy.signal.correlate(np.pad(x[0, :, :, 0], d), wd, mode="valid")
        y = nm.conv2d(x, w, 1, d, d)
        assert np.allclose(y[0, :, :, 0], ref)


def test_dilated_conv_backward_finite_differences():
    rng = np.random.default_rng(12)
    for st, pad, d in ((1, 2, 2), (1, 6, 6), (2, 2, 2)):
        x = rng.standard_normal((2, 11, 10, 3))
        w = rng.standard_normal((4, 3, 3, 3))
        G = rng.standard_normal(nm.conv2d(x, w, st, pad, d).shape)
        dx, dw = nm.conv2d_backward(x, w, G, st, pad, d)
        f = lambda: float((nm.conv2d(x, w, st, pad, d) * G).sum())
        for _ in range(6):
            i = tuple(int(rng.integers(0, s)) for s in x.shape)
            assert abs(_fd(f, x, i) - dx[i]) < 1e-5 * (1 + abs(dx[i]))
            j = tuple(int(rng.integers(0, s)) for s in w.shape)
            assert abs(_fd(f, w, j) - dw[j]) < 1e-5 * (1 + abs(dw[j]))


def test_bilinear_matches_torch_and_is_adjoint():
    rng = np.random.default_rng(13)
    for (h, w), (ho, wo) in (((3, 3), (9, 9)), ((33, 33), (129, 129)), ((9, 7), (33, 20)), ((1, 1), (5, 4)),
                             ((129, 129), (513, 513))):
        x = rng.standard_normal((2, h, w, 3))
        ref = F.interpolate(torch.from_numpy(x).permute(0, 3, 1, 2), size=(ho, wo), mode="bilinear",
                            align_corners=False).permute(0, 2, 3, 1).numpy()
        assert np.allclose(nm.upsample_bilinear(x, (ho, wo)), ref, atol=1e-12)
        g = rng.standard_normal((2, ho, wo, 3))
        lhs = np.sum(nm.upsample_bilinear(x, (ho, wo)) * g)
        rhs = np.sum(x * nm.upsample_bilinear_backward(g, (h, w)))
        assert np.isclose(lhs, rhs, rtol=1e-12)


def test_reflect_pad_matches_numpy_and_is_adjoint():
    rng = np.random.default_rng(14)
    x = rng.standard_normal((2, 6, 9, 3))
    for p in (1, 3):
        ref = np.pad(x, ((0, 0), (p, p), (p, p), (0, 0)), mode="reflect")
        assert np.array_equal(nm.reflect_pad(x, p), ref)
        g = rng.standard_normal(ref.shape)
        assert np.isclose(np.sum(ref * g), np.sum(x * nm.reflect_pad_backward(g, p)), rtol=1e-12)


def test_transposed_conv_matches_torch():
    rng = np.random.default_rng(15)
    x = rng.standard_normal((2, 5, 7, 4))
    w = rng.standard_normal((4, 3, 3, 6))               # [C_in, R, S, K_out]
    y = nm.conv_transpose2d(x, w, 2, 1, (10, 14))
    ref = F.conv_transpose2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w).permute(0, 3, 1, 2),
                             stride=2, padding=1, output_padding=1).permute(0, 2, 3, 1).numpy()
    assert np.allclose(y, ref, atol=1e-12)
    G = rng.standard_normal(y.shape)
    dx, dw = nm.conv_transpose2d_backward(x, w, G, 2, 1)
    f = lambda: float(np.sum(nm.conv_transpose2d(x, w, 2, 1, (10, 14)) * G))
    for _ in range(5):
        i = tuple(int(rng.integers(0, s)) for s in x.shape)
        assert abs(_fd(f, x, i) - dx[i]) < 1e-6 * (1 + abs(dx[i]))
        j = tuple(int(rng.integers(0, s)) for s in w.shape)
        assert abs(_fd(f, w, j) - dw[j]) < 1e-6 * (1 + abs(dw[j]))


def test_instance_norm_moments_and_backward():
    rng = np.random.default_rng(16)
    x = rng.standard_normal((3, 5, 6, 4)) * 2.0 + 0.7
    xh, rstd = nm.instance_norm(x)
    assert np.allclose(xh.mean(axis=(1, 2)), 0, atol=1e-12)
    var = x.var(axis=(1, 2))
    assert np.allclose(xh.var(axis=(1, 2)), var / (var + nm.BN_EPS), rtol=1e-12)
    G = rng.standard_normal(x.shape)
    f = lambda: float(np.sum(nm.instance_norm(x)[0] * G))
    dx = nm.instance_norm_backward(xh, rstd, G)
    for _ in range(8):
        i = tuple(int(rng.integers(0, s)) for s in x.shape)
        assert abs(_fd(f, x, i) - dx[i]) < 1e-6 * (1 + abs(dx[i]))


def test_l1_loss_closed_form():
    y = np.array([[1.0, -2.0], [0.5, 3.0]])
    t = np.array([[0.0, -2.0], [1.5, 1.0]])
    loss, g = nm.l1_loss(y, t)
    assert loss == (1.0 + 0.0 + 1.0 + 2.0) / 4
    assert np.array_equal(g, np.array([[0.25, 0.0], [-0.25, 0.25]]))


def test_deeplabv3plus_gradients_finite_differences():
    """Atrous convs, ASPP (image pooling branch, 4-way concat), bilinear
    decoder, per-pixel CE — through a miniature DeepLabv3+."""
    spec = nets.deeplabv3plus(batch=2, image=33, classes=3, width=4, rates=(2, 3, 4), aspp=8, low=4,
                              blocks=(1, 1, 1, 1))
    _fd_check_spec(spec, n_checks=24, tol=5e-5)


def test_pix2pixhd_gradients_finite_differences():
    """Reflection padding, instance norm, residual blocks, stride-2 transposed
    convs, tanh and the L1 loss — through a miniature Pix2PixHD generator."""
    spec = nets.pix2pixhd(batch=2, image=(16, 32), ngf=4, n_down=2, n_blocks=1)
    _fd_check_spec(spec, n_checks=24, tol=5e-5)
