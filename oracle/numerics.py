"""Oracle: reference training step (forward, backward, SGD-momentum update).

The method is exact for the numerics: swapping is a byte copy, so the
out-of-core step must produce the gradients of the ordinary step (SURVEY
§8(c) C6).  This module is that ordinary step, written from the textbook
definitions in float64 with the storage roundings of the GPU contract:

  rounding points (DESIGN.md §3 "numerics contract"):
    * every layer output tensor is stored in the activation dtype
      (bf16 in "bf16" mode, fp32 in "fp32" mode); logits and the loss are fp32;
    * conv / linear weights are used as act-dtype copies of fp32 masters;
    * the gradient of every activation tensor is stored in the act dtype;
      a tensor read by several layers accumulates the contributions in
      reverse layer order: G = rnd(c_first), then G = rnd(G + c) (c unrounded);
    * parameter gradients, BN statistics, momentum and masters are fp32.
  ReLU'(0) = 0; maxpool takes the first maximum in row-major window order,
  compared on the stored (rounded) values; BN uses batch statistics with the
  biased variance and eps = 1e-5 (training mode).

Definitions used (standard):
  linear      y = x Wᵀ + b
  conv2d      y[n,p,q,k] = Σ_{r,s,c} x[n, p·st−pad+r, q·st−pad+s, c] · W[k,r,s,c]
  batch norm  x̂ = (y − μ)/√(σ²+eps), out = γ x̂ + β (+ residual), then ReLU
              dy = γ/√(σ²+eps) · (dz − mean(dz) − x̂ · mean(dz · x̂))
  softmax-CE  L = mean_n(−log softmax(z_n)[y_n]);  dz = (softmax(z) − onehot)/N
  SGD-mom.    v ← μ v + g;  w ← w − lr · v
  GAN layers (configs[4] BigGAN-style step):
  upsample2   y[n,2i+a,2j+b,c] = x[n,i,j,c]          (nearest, ×2)
  avgpool2    y[n,i,j,c] = ¼ Σ_{a,b} x[n,2i+a,2j+b,c]
  tanh, relu  elementwise; tanh' = 1 − y², relu'(0) = 0
  attention   SAGAN self-attention over the H·W positions of one sample:
              q = x Wqᵀ, k = x Wkᵀ, v = x Wvᵀ (1×1 convs), P = softmax_rows(q kᵀ),
              o = P v, out = o Woᵀ, y = x + γ·out  (γ a learned scalar, ".gain")
  concat      y = [a, b] along channels (DenseNet); gradient split
  hinge       D: L = mean(relu(1 − D(x_real))) + mean(relu(1 + D(G(z))));
              G: L = −mean(D(G(z)))
"""
import numpy as np

BN_EPS = 1e-5


def round_bf16(a):
    """Round float64 values to the nearest bfloat16 (round-half-to-even),
    returned as float64.  bf16 keeps the top 16 bits of the fp32 format: 1 sign,
    8 exponent, 7 mantissa bits; from float64 that means dropping the low 45
    bits of the 52-bit mantissa with RNE.  Values here stay in the normal fp32
    exponent range."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    bits = a.view(np.uint64)
    lsb = (bits >> np.uint64(45)) & np.uint64(1)
    bits = (bits + np.uint64((1 << 44) - 1) + lsb) & ~np.uint64((1 << 45) - 1)
    return bits.view(np.float64)


def round_fp32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def _identity(a):
    return np.asarray(a, dtype=np.float64)


def rounder(mode):
    """Storage rounding of activations: bf16, fp32, or none ("fp64", used by
    the finite-difference pins)."""
    return {"bf16": round_bf16, "fp32": round_fp32, "fp64": _identity}[mode]


# ------------------------------------------------------------------ layers


def conv2d(x, w, stride, pad, dil=1):
    """x [N,H,W,C], w [K,R,S,C] -> y [N,P,Q,K] (definition above; dilation d:
    tap (r, s) reads x[n, p·st − pad + d·r, q·st − pad + d·s, c], the atrous
    convolution of DeepLab)."""
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    P = (H + 2 * pad - dil * (R - 1) - 1) // stride + 1
    Q = (W + 2 * pad - dil * (S - 1) - 1) // stride + 1
    xp = np.zeros((N, H + 2 * pad, W + 2 * pad, C))
    xp[:, pad:pad + H, pad:pad + W, :] = x
    y = np.zeros((N, P, Q, K))
    for r in range(R):
        for s in range(S):
            patch = xp[:, dil * r:dil * r + stride * P:stride, dil * s:dil * s + stride * Q:stride, :]
            y += patch @ w[:, r, s, :].T
    return y


def conv2d_backward(x, w, dy, stride, pad, dil=1):
    """Returns (dx, dw) for conv2d."""
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    _, P, Q, _ = dy.shape
    xp = np.zeros((N, H + 2 * pad, W + 2 * pad, C))
    xp[:, pad:pad + H, pad:pad + W, :] = x
    dxp = np.zeros_like(xp)
    dw = np.zeros_like(w, dtype=np.float64)
    dy2 = dy.reshape(-1, K)
    for r in range(R):
        for s in range(S):
            sl = (slice(None), slice(dil * r, dil * r + stride * P, stride), slice(dil * s, dil * s + stride * Q, stride))
            patch = xp[sl]
            dw[:, r, s, :] = dy2.T @ patch.reshape(-1, C)
            dxp[sl] += dy @ w[:, r, s, :]
    return dxp[:, pad:pad + H, pad:pad + W, :], dw


def conv_transpose2d(x, w, stride, pad, out_hw):
    """Transposed convolution (Pix2PixHD's upsampling layers): the adjoint of
    the conv2d that maps an out_hw map to x's map, x [N,H,W,C_in],
    w [C_in,R,S,K_out] read as that conv's KRSC weight (K = C_in)."""
    N = x.shape[0]
    dx, _ = conv2d_backward(np.zeros((N, out_hw[0], out_hw[1], w.shape[3])), w, x, stride, pad)
    return dx


def conv_transpose2d_backward(x, w, g, stride, pad):
    """(dx, dw) of conv_transpose2d: dx = conv2d(g, w) (the forward conv),
    dw = that conv's weight gradient with x in the role of its dy."""
    dx = conv2d(g, w, stride, pad)
    _, dw = conv2d_backward(g, w, x, stride, pad)
    return dx, dw


def bilinear_coeffs(n_in, n_out):
    """1-D bilinear interpolation weights, half-pixel centres (PyTorch
    align_corners=False): output i samples input coordinate
    src = max((i + 0.5)·n_in/n_out − 0.5, 0); i0 = floor(src),
    i1 = min(i0 + 1, n_in − 1), weights (1 − λ, λ), λ = src − i0."""
    src = np.maximum((np.arange(n_out) + 0.5) * (n_in / n_out) - 0.5, 0.0)
    i0 = np.minimum(np.floor(src).astype(np.int64), n_in - 1)
    i1 = np.minimum(i0 + 1, n_in - 1)
    lam = src - i0
    return i0, i1, lam


def upsample_bilinear(x, out_hw):
    """x [N,H,W,C] -> [N,Ho,Wo,C]: separable bilinear interpolation (rows, then columns)."""
    r0, r1, a = bilinear_coeffs(x.shape[1], out_hw[0])
    c0, c1, b = bilinear_coeffs(x.shape[2], out_hw[1])
    rows = x[:, r0] * (1 - a)[None, :, None, None] + x[:, r1] * a[None, :, None, None]
    return rows[:, :, c0] * (1 - b)[None, None, :, None] + rows[:, :, c1] * b[None, None, :, None]


def upsample_bilinear_backward(g, in_hw):
    """Adjoint of upsample_bilinear: each output's gradient scattered to its
    four source pixels with the same weights."""
    N, Ho, Wo, C = g.shape
    r0, r1, a = bilinear_coeffs(in_hw[0], Ho)
    c0, c1, b = bilinear_coeffs(in_hw[1], Wo)
    rows = np.zeros((N, Ho, in_hw[1], C))
    np.add.at(rows, (slice(None), slice(None), c0), g * (1 - b)[None, None, :, None])
    np.add.at(rows, (slice(None), slice(None), c1), g * b[None, None, :, None])
    dx = np.zeros((N, in_hw[0], in_hw[1], C))
    np.add.at(dx, (slice(None), r0), rows * (1 - a)[None, :, None, None])
    np.add.at(dx, (slice(None), r1), rows * a[None, :, None, None])
    return dx


def reflect_index(n, p):
    """Source index of each padded position of a length-n axis padded by p on
    both sides with reflection (the edge value not repeated: ... 2 1 | 0 1 2 ...)."""
    k = np.arange(-p, n + p)
    k = np.where(k < 0, -k, k)
    return np.where(k >= n, 2 * (n - 1) - k, k)


def reflect_pad(x, p):
    """[N,H,W,C] -> [N,H+2p,W+2p,C] (Pix2PixHD's ReflectionPad2d)."""
    return x[:, reflect_index(x.shape[1], p)][:, :, reflect_index(x.shape[2], p)]


def reflect_pad_backward(g, p):
    N, Hp, Wp, C = g.shape
    H, W = Hp - 2 * p, Wp - 2 * p
    rows = np.zeros((N, Hp, W, C))
    np.add.at(rows, (slice(None), slice(None), reflect_index(W, p)), g)
    dx = np.zeros((N, H, W, C))
    np.add.at(dx, (slice(None), reflect_index(H, p)), rows)
    return dx


def instance_norm(x):
    """Per sample and channel over the H·W positions (Pix2PixHD's
    InstanceNorm2d, no affine): x̂ = (x − μ_nc)/√(σ²_nc + eps), biased variance.
    Returns (x̂, rstd [N,1,1,C])."""
    mu = x.mean(axis=(1, 2), keepdims=True)
    var = ((x - mu) ** 2).mean(axis=(1, 2), keepdims=True)
    rstd = 1.0 / np.sqrt(var + BN_EPS)
    return (x - mu) * rstd, rstd


def instance_norm_backward(xhat, rstd, dz):
    """dx = rstd·(dz − mean_hw(dz) − x̂·mean_hw(dz·x̂))."""
    return rstd * (dz - dz.mean(axis=(1, 2), keepdims=True) - xhat * (dz * xhat).mean(axis=(1, 2), keepdims=True))


def l1_loss(y, t):
    """L = mean |y − t|; dL/dy = sign(y − t)/count (sign(0) = 0)."""
    d = y - t
    return float(np.abs(d).mean()), np.sign(d) / d.size


def conv_transpose2x2(x, w):
    """2×2 stride-2 transposed convolution, x [N,H,W,C], w [C,2,2,K]:
    y[n, 2p+i, 2q+j, k] = Σ_c x[n,p,q,c] · w[c,i,j,k]."""
    N, H, W, C = x.shape
    K = w.shape[3]
    y = np.zeros((N, 2 * H, 2 * W, K))
    for i in range(2):
        for j in range(2):
            y[:, i::2, j::2, :] = x @ w[:, i, j, :]
    return y


def conv_transpose2x2_backward(x, w, g):
    """Returns (dx, dw) for conv_transpose2x2."""
    N, H, W, C = x.shape
    dx = np.zeros((N, H, W, C))
    dw = np.zeros(w.shape)
    for i in range(2):
        for j in range(2):
            gij = g[:, i::2, j::2, :]
            dx += gij @ w[:, i, j, :].T
            dw[:, i, j, :] = x.reshape(-1, C).T @ gij.reshape(-1, w.shape[3])
    return dx, dw


def maxpool(x, r, stride, pad):
    """Returns (out, argmax index into the r×r window, row-major, first max)."""
    N, H, W, C = x.shape
    P = (H + 2 * pad - r) // stride + 1
    Q = (W + 2 * pad - r) // stride + 1
    xp = np.full((N, H + 2 * pad, W + 2 * pad, C), -np.inf)
    xp[:, pad:pad + H, pad:pad + W, :] = x
    out = np.full((N, P, Q, C), -np.inf)
    arg = np.zeros((N, P, Q, C), dtype=np.int64)
    for i in range(r):
        for j in range(r):
            cand = xp[:, i:i + stride * P:stride, j:j + stride * Q:stride, :]
            better = cand > out          # strict: the first maximum wins
            out = np.where(better, cand, out)
            arg = np.where(better, i * r + j, arg)
    return out, arg


def maxpool_backward(dout, arg, x_shape, r, stride, pad):
    N, H, W, C = x_shape
    _, P, Q, _ = dout.shape
    dxp = np.zeros((N, H + 2 * pad, W + 2 * pad, C))
    for i in range(r):
        for j in range(r):
            sel = (arg == i * r + j)
            dxp[:, i:i + stride * P:stride, j:j + stride * Q:stride, :] += np.where(sel, dout, 0.0)
    return dxp[:, pad:pad + H, pad:pad + W, :]


def softmax_ce(z, labels):
    """Mean cross-entropy and its gradient wrt the logits."""
    N = z.shape[0]
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    p = e / e.sum(axis=1, keepdims=True)
    loss = -np.mean(np.log(p[np.arange(N), labels]))
    dz = p.copy()
    dz[np.arange(N), labels] -= 1.0
    return loss, dz / N


def upsample2(x):
    return np.repeat(np.repeat(x, 2, axis=1), 2, axis=2)


def upsample2_backward(g):
    """Σ over each 2×2 block, summed in the order (0,0), (0,1), (1,0), (1,1)."""
    return ((g[:, 0::2, 0::2] + g[:, 0::2, 1::2]) + g[:, 1::2, 0::2]) + g[:, 1::2, 1::2]


def avgpool2(x):
    return 0.25 * (((x[:, 0::2, 0::2] + x[:, 0::2, 1::2]) + x[:, 1::2, 0::2]) + x[:, 1::2, 1::2])


def avgpool2_backward(g):
    return upsample2(0.25 * g)


def attention(q, k, v, rnd):
    """Per sample n: P = softmax over keys of q kᵀ (rows = query positions),
    stored in the act dtype; o = P v.  q, k [N, L, dq], v [N, L, dv]."""
    S = np.einsum("nid,njd->nij", q, k)
    S = S - S.max(axis=2, keepdims=True)
    e = np.exp(S)
    P = rnd(e / e.sum(axis=2, keepdims=True))
    return P, rnd(np.einsum("nij,njd->nid", P, v))


def attention_backward(q, k, v, P, o, do):
    """Gradients of o = softmax(q kᵀ) v wrt q, k, v (P the stored softmax):
    dv = Pᵀ do; dP = do vᵀ; dS = P ⊙ (dP − rowsum(dP ⊙ P)), rowsum(dP ⊙ P)_i
    = do_i · o_i; dq = dS k; dk = dSᵀ q."""
    dv = np.einsum("nij,nid->njd", P, do)
    dP = np.einsum("nid,njd->nij", do, v)
    rs = np.einsum("nid,nid->ni", do, o)[:, :, None]
    dS = P * (dP - rs)
    return np.einsum("nij,njd->nid", dS, k), np.einsum("nij,nid->njd", dS, q), dv


# --------------------------------------------------------------- training step


class _Net:
    """Forward / backward interpreter of a layer list (the definitions above,
    with the storage roundings of the numerics contract)."""

    def __init__(self, layers, params, mode):
        self.layers = layers
        self.mode = mode
        self.rnd = rounder(mode)
        self.r32 = _identity if mode == "fp64" else round_fp32
        self.f64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
        self.wcopy = {k: self.rnd(v) for k, v in self.f64.items()
                      if k.endswith((".W", ".W2", ".Wq", ".Wk", ".Wv", ".Wo"))}

    def forward(self, acts, fp32_out=()):
        rnd, f64, wcopy = self.rnd, self.f64, self.wcopy
        saved = {}
        for lay in self.layers:
            t, nm = lay["type"], lay["name"]
            xin = acts[lay["in"]]
            if t == "linear":
                xi = xin.reshape(xin.shape[0], -1)
                y = xi @ wcopy[nm + ".W"].T + f64[nm + ".b"]
                if lay["relu"]:
                    y = np.maximum(y, 0.0)
                # logits / scores (a linear feeding a loss) are fp32
                out = self.r32(y) if lay["out"] in fp32_out else rnd(y)
                if lay.get("reshape"):
                    out = out.reshape([xin.shape[0]] + list(lay["reshape"]))
            elif t == "conv":
                out = rnd(conv2d(xin, wcopy[nm + ".W"], lay["stride"], lay["pad"], lay.get("dil", 1)))
                if lay.get("in2"):
                    # conv over the concatenation [in, in2] = conv(in, W) + conv(in2, W2);
                    # contributions to one stored tensor accumulate in order with a
                    # rounding after each (Z23)
                    out = rnd(out + conv2d(acts[lay["in2"]], wcopy[nm + ".W2"], lay["stride"], lay["pad"]))
            elif t == "convT":
                out = rnd(conv_transpose2x2(xin, wcopy[nm + ".W"]))
            elif t == "tconv":
                out = rnd(conv_transpose2d(xin, wcopy[nm + ".W"], lay["stride"], lay["pad"], lay["_out_hw"]))
            elif t == "in":
                xhat, rstd = instance_norm(xin)
                z = np.maximum(xhat, 0.0) if lay["relu"] else xhat
                out = rnd(z)
                saved[nm] = (xhat, rstd)
            elif t == "reflect_pad":
                out = reflect_pad(xin, lay["pad"])
            elif t == "upsample_bilinear":
                out = rnd(upsample_bilinear(xin, lay["size"]))
            elif t == "bn":
                axes = tuple(range(xin.ndim - 1))
                mu = xin.mean(axis=axes)
                var = ((xin - mu) ** 2).mean(axis=axes)
                rstd = 1.0 / np.sqrt(var + BN_EPS)
                xhat = (xin - mu) * rstd
                z = f64[nm + ".gamma"] * xhat + f64[nm + ".beta"]
                if lay.get("residual"):
                    z = z + acts[lay["residual"]]
                if lay["relu"]:
                    z = np.maximum(z, 0.0)
                out = rnd(z)
                saved[nm] = (xhat, rstd)
            elif t == "maxpool":
                out, arg = maxpool(xin, lay["r"], lay["stride"], lay["pad"])
                saved[nm] = arg
            elif t == "gap":
                out = rnd(xin.mean(axis=(1, 2), keepdims=bool(lay.get("keepdims"))))
            elif t == "add":                      # residual sum
                out = rnd(xin + acts[lay["in2"]])
            elif t == "relu":
                out = np.maximum(xin, 0.0)
            elif t == "tanh":
                out = rnd(np.tanh(xin))
            elif t == "concat":                    # channels [in, in2] (a copy: no rounding)
                out = np.concatenate([xin, acts[lay["in2"]]], axis=-1)
            elif t == "upsample2":
                out = upsample2(xin)
            elif t == "avgpool2":
                out = rnd(avgpool2(xin))
            elif t == "attn":
                N, H, W, C = xin.shape
                x2 = xin.reshape(N, H * W, C)
                q = rnd(x2 @ wcopy[nm + ".Wq"].reshape(-1, C).T)
                k = rnd(x2 @ wcopy[nm + ".Wk"].reshape(-1, C).T)
                v = rnd(x2 @ wcopy[nm + ".Wv"].reshape(-1, C).T)
                P, o = attention(q, k, v, rnd)
                ao = rnd(o @ wcopy[nm + ".Wo"].reshape(C, -1).T)
                out = rnd(x2 + f64[nm + ".gain"][0] * ao).reshape(xin.shape)
                saved[nm] = (q, k, v, P, o, ao)
            else:
                raise ValueError(t)
            acts[lay["out"]] = out
        return saved

    def backward(self, acts, saved, G, grads=None, input_names=()):
        """Reverse-order backward from the gradients in G (tensor -> grad).
        grads: dict to fill with parameter gradients, or None (data gradients
        only).  input_names: graph inputs whose gradient is wanted."""
        rnd, f64, wcopy, r32 = self.rnd, self.f64, self.wcopy, self.r32

        def acc(name, c):
            G[name] = rnd(c) if name not in G else rnd(G[name] + c)

        def pg(key, val):
            if grads is not None:
                grads[key] = r32(val)

        produced = {lay["out"] for lay in self.layers}
        for lay in reversed(self.layers):
            t, nm = lay["type"], lay["name"]
            if lay["out"] not in G:
                continue
            g = G[lay["out"]]
            xin = acts[lay["in"]]
            need_dx = lay["in"] in produced or lay["in"] in input_names
            if t == "linear":
                out = acts[lay["out"]]
                g2 = g.reshape(g.shape[0], -1)
                out2 = out.reshape(out.shape[0], -1)
                dz = g2 * (out2 > 0) if lay["relu"] else g2
                xi = xin.reshape(xin.shape[0], -1)
                pg(nm + ".W", dz.T @ xi)
                pg(nm + ".b", dz.sum(axis=0))
                if need_dx:
                    acc(lay["in"], (dz @ wcopy[nm + ".W"]).reshape(xin.shape))
            elif t == "conv":
                dx, dw = conv2d_backward(xin, wcopy[nm + ".W"], g, lay["stride"], lay["pad"], lay.get("dil", 1))
                pg(nm + ".W", dw)
                if need_dx:
                    acc(lay["in"], dx)
                if lay.get("in2"):
                    dx2, dw2 = conv2d_backward(acts[lay["in2"]], wcopy[nm + ".W2"], g, lay["stride"], lay["pad"])
                    pg(nm + ".W2", dw2)
                    acc(lay["in2"], dx2)
            elif t == "convT":
                dx, dw = conv_transpose2x2_backward(xin, wcopy[nm + ".W"], g)
                pg(nm + ".W", dw)
                acc(lay["in"], dx)
            elif t == "tconv":
                dx, dw = conv_transpose2d_backward(xin, wcopy[nm + ".W"], g, lay["stride"], lay["pad"])
                pg(nm + ".W", dw)
                if need_dx:
                    acc(lay["in"], dx)
            elif t == "in":
                xhat, rstd = saved[nm]
                dz = g * (acts[lay["out"]] > 0) if lay["relu"] else g
                if need_dx:
                    acc(lay["in"], instance_norm_backward(xhat, rstd, dz))
            elif t == "reflect_pad":
                if need_dx:
                    acc(lay["in"], reflect_pad_backward(g, lay["pad"]))
            elif t == "upsample_bilinear":
                if need_dx:
                    acc(lay["in"], upsample_bilinear_backward(g, xin.shape[1:3]))
            elif t == "bn":
                xhat, rstd = saved[nm]
                out = acts[lay["out"]]
                dz = g * (out > 0) if lay["relu"] else g
                axes = tuple(range(xin.ndim - 1))
                pg(nm + ".gamma", (dz * xhat).sum(axis=axes))
                pg(nm + ".beta", dz.sum(axis=axes))
                if lay.get("residual"):
                    acc(lay["residual"], dz)
                dy = f64[nm + ".gamma"] * rstd * (dz - dz.mean(axis=axes) - xhat * (dz * xhat).mean(axis=axes))
                acc(lay["in"], dy)
            elif t == "maxpool":
                acc(lay["in"], maxpool_backward(g, saved[nm], xin.shape, lay["r"], lay["stride"], lay["pad"]))
            elif t == "gap":
                H, W = xin.shape[1], xin.shape[2]
                g4 = g.reshape(g.shape[0], 1, 1, -1)
                acc(lay["in"], np.broadcast_to(g4 / (H * W), xin.shape))
            elif t == "add":
                acc(lay["in"], g)
                acc(lay["in2"], g)
            elif t == "relu":
                if need_dx:
                    acc(lay["in"], g * (xin > 0))
            elif t == "tanh":
                y = acts[lay["out"]]
                if need_dx:
                    acc(lay["in"], g * (1.0 - y * y))
            elif t == "concat":
                ca = xin.shape[-1]
                if need_dx:
                    acc(lay["in"], g[..., :ca])
                acc(lay["in2"], g[..., ca:])
            elif t == "upsample2":
                if need_dx:
                    acc(lay["in"], upsample2_backward(g))
            elif t == "avgpool2":
                if need_dx:
                    acc(lay["in"], avgpool2_backward(g))
            elif t == "attn":
                q, k, v, P, o, ao = saved[nm]
                N, H, W, C = xin.shape
                x2 = xin.reshape(N, H * W, C)
                g2 = g.reshape(N, H * W, C)
                gam = f64[nm + ".gain"][0]
                pg(nm + ".gain", np.array([(g2 * ao).sum()]))
                dao = rnd(gam * g2)
                Wo = wcopy[nm + ".Wo"].reshape(C, -1)
                pg(nm + ".Wo", (dao.reshape(-1, C).T @ o.reshape(-1, o.shape[-1])).reshape(C, 1, 1, -1))
                do = rnd(dao @ Wo)
                dq, dk, dv = attention_backward(q, k, v, P, o, do)
                dq, dk, dv = rnd(dq), rnd(dk), rnd(dv)
                # x feeds the residual, then q, k, v (contributions in that order)
                parts = [g2]
                for d, wn in ((dq, ".Wq"), (dk, ".Wk"), (dv, ".Wv")):
                    Wm = wcopy[nm + wn].reshape(-1, C)
                    pg(nm + wn, (d.reshape(-1, d.shape[-1]).T @ x2.reshape(-1, C)).reshape(-1, 1, 1, C))
                    parts.append(d @ Wm)
                if need_dx:
                    for c in parts:
                        acc(lay["in"], c.reshape(xin.shape))
        return G


def _sgd(spec, params, grads, momentum, r32):
    lr, mu = spec["sgd"]["lr"], spec["sgd"]["momentum"]
    new_p, new_m = {}, {}
    for k in params:
        m0 = np.zeros_like(np.asarray(params[k], np.float64)) if momentum is None else np.asarray(momentum[k],
                                                                                                  np.float64)
        v = r32(mu * m0 + grads[k])
        new_m[k] = v
        new_p[k] = r32(np.asarray(params[k], np.float64) - lr * v)
    return new_p, new_m


def train_step(spec, params, x, labels, momentum=None):
    """One step.  `params`: dict name -> fp32 array (masters); `momentum`:
    dict or None (zeros).  Returns dict with loss, grads, new params, new
    momentum and the stored activations (for inspection)."""
    _attach_out_hw(spec)
    net = _Net(spec["layers"], params, spec["mode"])
    rnd, r32 = net.rnd, net.r32
    acts = {"x": rnd(np.asarray(x, np.float64))}
    pix = spec["loss"]["type"] in ("softmax_ce_pix", "l1")
    saved = net.forward(acts, fp32_out=() if pix else (spec["loss"]["in"],))
    if spec["loss"]["type"] == "l1":
        # L1 to a target image (the synthetic stand-in for Pix2PixHD's losses);
        # the output and its gradient are act-dtype tensors, the target is
        # stored in the act dtype
        z = acts[spec["loss"]["in"]]
        loss, dz = l1_loss(z, rnd(np.asarray(labels, np.float64)).reshape(z.shape))
        G = {spec["loss"]["in"]: rnd(dz)}
    elif pix:
        # per-pixel cross-entropy over the channel axis, mean over all pixels;
        # the logits are a conv output (act dtype) and so is their gradient
        z = acts[spec["loss"]["in"]]
        K = z.shape[-1]
        loss, dlogits = softmax_ce(z.reshape(-1, K), np.asarray(labels).reshape(-1))
        G = {spec["loss"]["in"]: rnd(dlogits.reshape(z.shape))}
    else:
        loss, dlogits = softmax_ce(acts[spec["loss"]["in"]], labels)
        G = {spec["loss"]["in"]: r32(dlogits)}   # dlogits stored fp32
    grads = {}
    net.backward(acts, saved, G, grads)
    new_p, new_m = _sgd(spec, params, grads, momentum, r32)
    return {"loss": float(loss), "grads": grads, "params": new_p, "momentum": new_m, "acts": acts}


def _attach_out_hw(spec):
    """Output sizes of the transposed convs (from the layer list's shapes)."""
    if not any(l["type"] == "tconv" for l in spec["layers"]):
        return
    from synth import nets
    shapes, _ = nets.tensor_shapes(spec)
    for lay in spec["layers"]:
        if lay["type"] == "tconv":
            lay["_out_hw"] = tuple(shapes[lay["out"]][:2])


def hinge_d(s, n_real):
    """D hinge loss over scores s [2N] (real first) and its gradient."""
    real, fake = s[:n_real], s[n_real:]
    loss = np.maximum(0.0, 1.0 - real).mean() + np.maximum(0.0, 1.0 + fake).mean()
    ds = np.concatenate([-(real < 1.0).astype(np.float64) / len(real), (fake > -1.0).astype(np.float64) / len(fake)])
    return float(loss), ds


def gan_step(spec, pG, pD, z1, z2, x_real, momG=None, momD=None):
    """One BigGAN-style step: a D-step on [x_real; G(z1)]
    with the hinge loss and an SGD-momentum update of D, then a G-step on
    G(z2) through the updated D (D's parameters fixed) with L = −mean D(G(z2))
    and an SGD-momentum update of G."""
    mode = spec["mode"]
    N = z1.shape[0]
    G_, D_ = spec["G"], spec["D"]
    g_net = _Net(G_["layers"], pG, mode)
    rnd, r32 = g_net.rnd, g_net.r32
    # ---- D-step
    a1 = {"z": rnd(np.asarray(z1, np.float64))}      # z stored in the act dtype
    g_net.forward(a1)
    xd = np.concatenate([rnd(np.asarray(x_real, np.float64)), a1[G_["out"]]])
    d_net = _Net(D_["layers"], pD, mode)
    ad = {"x": xd}
    sd = d_net.forward(ad, fp32_out=(D_["out"],))
    score = ad[D_["out"]].reshape(-1)
    loss_d, ds = hinge_d(score, N)
    gradsD = {}
    d_net.backward(ad, sd, {D_["out"]: r32(ds.reshape(-1, 1))}, gradsD)
    pD_new, momD_new = _sgd(spec, pD, gradsD, momD, r32)
    # ---- G-step through the updated D
    a2 = {"z": rnd(np.asarray(z2, np.float64))}
    sg = g_net.forward(a2)
    d2 = _Net(D_["layers"], pD_new, mode)
    ad2 = {"x": a2[G_["out"]]}
    sd2 = d2.forward(ad2, fp32_out=(D_["out"],))
    score2 = ad2[D_["out"]].reshape(-1)
    loss_g = float(-score2.mean())
    Gd = d2.backward(ad2, sd2, {D_["out"]: r32(np.full((N, 1), -1.0 / N))}, None, input_names=("x",))
    gradsG = {}
    g_net.backward(a2, sg, {G_["out"]: Gd["x"]}, gradsG)
    pG_new, momG_new = _sgd(spec, pG, gradsG, momG, r32)
    return {"loss_d": loss_d, "loss_g": loss_g, "gradsD": gradsD, "gradsG": gradsG, "pD": pD_new, "pG": pG_new,
            "momD": momD_new, "momG": momG_new, "score_d": score, "score_g": score2}


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0))
