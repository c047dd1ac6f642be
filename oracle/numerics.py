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


def conv2d(x, w, stride, pad):
    """x [N,H,W,C], w [K,R,S,C] -> y [N,P,Q,K] (definition above)."""
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    xp = np.zeros((N, H + 2 * pad, W + 2 * pad, C))
    xp[:, pad:pad + H, pad:pad + W, :] = x
    y = np.zeros((N, P, Q, K))
    for r in range(R):
        for s in range(S):
            patch = xp[:, r:r + stride * P:stride, s:s + stride * Q:stride, :]
            y += patch @ w[:, r, s, :].T
    return y


def conv2d_backward(x, w, dy, stride, pad):
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
            patch = xp[:, r:r + stride * P:stride, s:s + stride * Q:stride, :]
            dw[:, r, s, :] = dy2.T @ patch.reshape(-1, C)
            dxp[:, r:r + stride * P:stride, s:s + stride * Q:stride, :] += dy @ w[:, r, s, :]
    return dxp[:, pad:pad + H, pad:pad + W, :], dw


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


# --------------------------------------------------------------- training step


def train_step(spec, params, x, labels, momentum=None):
    """One step.  `params`: dict name -> fp32 array (masters); `momentum`:
    dict or None (zeros).  Returns dict with loss, grads, new params, new
    momentum and the stored activations (for inspection)."""
    mode = spec["mode"]
    rnd = rounder(mode)
    round_fp32 = _identity if mode == "fp64" else globals()["round_fp32"]
    f64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    wcopy = {}                                # act-dtype copies of weights
    for k, v in f64.items():
        if k.endswith(".W") or k.endswith(".W2"):
            wcopy[k] = rnd(v)
    acts = {"x": rnd(np.asarray(x, np.float64))}
    saved = {}
    # ---------------- forward
    for lay in spec["layers"]:
        t, nm = lay["type"], lay["name"]
        xin = acts[lay["in"]]
        if t == "linear":
            xi = xin.reshape(xin.shape[0], -1)
            y = xi @ wcopy[nm + ".W"].T + f64[nm + ".b"]
            if lay["relu"]:
                y = np.maximum(y, 0.0)
            # logits (a linear without ReLU feeding the loss) are fp32
            out = round_fp32(y) if lay["out"] == spec["loss"]["in"] else rnd(y)
        elif t == "conv":
            out = rnd(conv2d(xin, wcopy[nm + ".W"], lay["stride"], lay["pad"]))
            if lay.get("in2"):
                # conv over the concatenation [in, in2] = conv(in, W) + conv(in2, W2);
                # contributions to one stored tensor accumulate in order with a
                # rounding after each (Z23)
                out = rnd(out + conv2d(acts[lay["in2"]], wcopy[nm + ".W2"], lay["stride"], lay["pad"]))
        elif t == "convT":
            out = rnd(conv_transpose2x2(xin, wcopy[nm + ".W"]))
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
            out = rnd(xin.mean(axis=(1, 2)))
        elif t == "add":                      # residual sum of a pre-activation block
            out = rnd(xin + acts[lay["in2"]])
        else:
            raise ValueError(t)
        acts[lay["out"]] = out
    grads = {}
    if spec["loss"]["type"] == "softmax_ce_pix":
        # per-pixel cross-entropy over the channel axis, mean over all pixels;
        # the logits are a conv output (act dtype) and so is their gradient
        z = acts[spec["loss"]["in"]]
        K = z.shape[-1]
        loss, dlogits = softmax_ce(z.reshape(-1, K), np.asarray(labels).reshape(-1))
        G = {spec["loss"]["in"]: rnd(dlogits.reshape(z.shape))}
    else:
        loss, dlogits = softmax_ce(acts[spec["loss"]["in"]], labels)
        G = {spec["loss"]["in"]: round_fp32(dlogits)}   # dlogits stored fp32
    # ---------------- backward (reverse layer order)

    def acc(name, c):
        G[name] = rnd(c) if name not in G else rnd(G[name] + c)

    for lay in reversed(spec["layers"]):
        t, nm = lay["type"], lay["name"]
        if lay["out"] not in G:
            continue
        g = G[lay["out"]]
        xin = acts[lay["in"]]
        need_dx = lay["in"] != "x"
        if t == "linear":
            out = acts[lay["out"]]
            dz = g * (out > 0) if lay["relu"] else g
            xi = xin.reshape(xin.shape[0], -1)
            grads[nm + ".W"] = round_fp32(dz.T @ xi)
            grads[nm + ".b"] = round_fp32(dz.sum(axis=0))
            if need_dx:
                acc(lay["in"], (dz @ wcopy[nm + ".W"]).reshape(xin.shape))
        elif t == "conv":
            dx, dw = conv2d_backward(xin, wcopy[nm + ".W"], g, lay["stride"], lay["pad"])
            grads[nm + ".W"] = round_fp32(dw)
            if need_dx:
                acc(lay["in"], dx)
            if lay.get("in2"):
                dx2, dw2 = conv2d_backward(acts[lay["in2"]], wcopy[nm + ".W2"], g, lay["stride"], lay["pad"])
                grads[nm + ".W2"] = round_fp32(dw2)
                acc(lay["in2"], dx2)
        elif t == "convT":
            dx, dw = conv_transpose2x2_backward(xin, wcopy[nm + ".W"], g)
            grads[nm + ".W"] = round_fp32(dw)
            acc(lay["in"], dx)
        elif t == "bn":
            xhat, rstd = saved[nm]
            out = acts[lay["out"]]
            dz = g * (out > 0) if lay["relu"] else g
            axes = tuple(range(xin.ndim - 1))
            grads[nm + ".gamma"] = round_fp32((dz * xhat).sum(axis=axes))
            grads[nm + ".beta"] = round_fp32(dz.sum(axis=axes))
            if lay.get("residual"):
                acc(lay["residual"], dz)
            dy = f64[nm + ".gamma"] * rstd * (dz - dz.mean(axis=axes) - xhat * (dz * xhat).mean(axis=axes))
            acc(lay["in"], dy)
        elif t == "maxpool":
            acc(lay["in"], maxpool_backward(g, saved[nm], xin.shape, lay["r"], lay["stride"], lay["pad"]))
        elif t == "gap":
            H, W = xin.shape[1], xin.shape[2]
            acc(lay["in"], np.broadcast_to(g[:, None, None, :] / (H * W), xin.shape))
        elif t == "add":
            acc(lay["in"], g)
            acc(lay["in2"], g)
    # ---------------- SGD with momentum (fp32 state)
    lr, mu = spec["sgd"]["lr"], spec["sgd"]["momentum"]
    new_p, new_m = {}, {}
    for k in params:
        m0 = np.zeros_like(f64[k]) if momentum is None else np.asarray(momentum[k], np.float64)
        v = round_fp32(mu * m0 + grads[k])
        new_m[k] = v
        new_p[k] = round_fp32(f64[k] - lr * v)
    return {"loss": float(loss), "grads": grads, "params": new_p, "momentum": new_m, "acts": acts}


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0))
