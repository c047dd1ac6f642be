"""Oracle: the definition of every function f_i of the conv-net training-step
graph, one function at a time (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The paper's step is the ordinary training step — forward, backward and update
functions executed in sequence — and swapping moves bytes without
changing them, so every function of the out-of-core step must compute exactly
what its definition says from the values it reads.  This module states that
definition per op kind of the graph document (paper_2010_14109_b200/graphs_conv.py
emits them), in float64 with the storage roundings of the numerics contract
(oracle/numerics.py header; Z23):

  apply(kind, attrs, ins) -> outs
    ins   role -> float64 array of the values the function READS (bf16 / fp32
          stored values decoded exactly; u8 / i32 as integers)
    outs  role -> the values the function must WRITE (float64, already rounded
          to the storage dtype — bf16 activations and their gradients, fp32
          BN statistics [mu; rstd], parameter gradients, loss, logits and
          optimizer state; u8 argmax taps as integers)

Two uses:
  * layer-local parity (tests/test_gpu_layerwise.py): each GPU function is
    fed its own stored inputs, captured from the GPU before it runs, and its
    outputs are compared with apply(...) — the comparison is then well posed
    at north_star's 1e-3 for every function of a deep bf16 net, where the
    end-to-end comparison is not (Z24: sub-ulp differences compound
    through bf16 rounding layer by layer);
  * run_graph(doc, values): the whole step executed function by function with
    these definitions.  It is pinned to numerics.train_step (itself pinned by
    finite differences and library routines) in tests/test_oracle_layerwise.py.

Op definitions (roles as in the graph document; rnd = storage rounding):
  conv_fwd        y = rnd(conv2d(x, rnd(W)))  [accumulate: rnd(y + conv2d)]
                  bn_stat: stat = [mean(y), 1/sqrt(var(y) + eps)] over the
                  stored y (biased variance)
  conv_dgrad      dx = rnd(conv2d_backward_x(dy, rnd(W)))  [accumulate: rnd(dx + c)]
  conv_wgrad      dw = conv2d_backward_w(x, dy)            (fp32 gradient)
  bn_fwd          stat as above unless attrs.stat_in;
                  out = rnd(relu?(gamma (y - mu) rstd + beta (+ res)))
  bn_bwd_reduce   x^ = (y - mu) rstd; dz = g * mask, mask = 1 (no ReLU),
                  [out > 0] (stored output given), [gamma x^ + beta > 0];
                  dbeta = sum dz, dgamma = sum dz x^
  bn_bwd_apply    dy = gamma rstd (dz - dbeta/n - x^ dgamma/n) with the
                  dgamma, dbeta the function reads; written over y
                  (rnd(dy)) or accumulated into acc (rnd(acc + dy)); with a
                  residual, dz written over g
  bn_relu_pool_fwd  z = rnd(relu(gamma (y - mu) rstd + beta)); out, idx =
                  maxpool(z) (first maximum, row-major taps); stat unless stat_in
  pool_bn_bwd_reduce  ga = rnd(maxpool_backward(g, idx)); dz = ga [gamma x^ + beta > 0];
                  dbeta = sum dz, dgamma = sum dz x^
  pool_bn_bwd_apply   y := rnd(gamma rstd (dz - dbeta/n - x^ dgamma/n))
  gap_fwd / gap_bwd   out = rnd(mean_hw x);  dx = rnd(g / HW) broadcast
  linear_fwd      y = x rnd(W)^T + b (relu?), stored fp32 if out_f32 else rnd
  linear_bwd      dz = dy (ReLU-masked by y > 0); dw = dz^T x; db = sum_m dz;
                  dx = rnd(dz rnd(W))
  softmax_ce      loss = mean_m(logsumexp(z_m) - z_m[y_m]); dlogits = (p - onehot)/M
  allreduce       one replica: the identity (the DP mean of C7 is tested elsewhere)
  sgd             v = mu v + g; w = w - lr v  (fp32 state)
"""
import json

import numpy as np

from . import numerics as nm


r32 = nm.round_fp32


def _stat(y2):
    """[mu; rstd] of rows y2 [rows, C] (training-mode batch statistics,
    biased variance), stored fp32."""
    mu = y2.mean(axis=0)
    var = ((y2 - mu) ** 2).mean(axis=0)
    return r32(np.stack([mu, 1.0 / np.sqrt(var + nm.BN_EPS)]))


def _rnd(attrs):
    return nm.round_bf16 if attrs.get("dtype", "bf16") == "bf16" else nm.round_fp32


def _geom(a):
    return a["N"], a["H"], a["W"], a["C"], a["K"], a["R"], a["S"], a["stride"], a["pad"], a["P"], a["Q"]


def conv_fwd(a, ins):
    N, H, W, C, K, R, S, st, pad, P, Q = _geom(a)
    rnd = _rnd(a)
    x = ins["x"].reshape(N, H, W, C)
    w = ins["w"].reshape(K, R, S, C)
    c = nm.conv2d(x, rnd(w), st, pad, a.get("dil", 1))
    y = rnd(ins["y"].reshape(N, P, Q, K) + c) if a.get("accumulate") else rnd(c)
    out = {"y": y}
    if a.get("bn_stat"):
        out["stat"] = _stat(y.reshape(-1, K))
    return out


def conv_dgrad(a, ins):
    N, H, W, C, K, R, S, st, pad, P, Q = _geom(a)
    rnd = _rnd(a)
    dy = ins["dy"].reshape(N, P, Q, K)
    w = ins["w"].reshape(K, R, S, C)
    dx, _ = nm.conv2d_backward(np.zeros((N, H, W, C)), rnd(w), dy, st, pad, a.get("dil", 1))
    if a.get("accumulate"):
        return {"dx": rnd(ins["dx"].reshape(N, H, W, C) + dx)}
    return {"dx": rnd(dx)}


def conv_wgrad(a, ins):
    N, H, W, C, K, R, S, st, pad, P, Q = _geom(a)
    x = ins["x"].reshape(N, H, W, C)
    dy = ins["dy"].reshape(N, P, Q, K)
    _, dw = nm.conv2d_backward(x, np.zeros((K, R, S, C)), dy, st, pad, a.get("dil", 1))
    return {"dw": r32(dw)}


# transposed convs: attrs describe the conv g they invert (g's input = the
# big map, its output = the small map, its KRSC weight = the convT weight)
def convT_fwd(a, ins):
    return {"y": conv_dgrad(a, {"dy": ins["x"], "w": ins["w"]})["dx"]}


def convT_dgrad(a, ins):
    out = conv_fwd(dict(a, bn_stat=False), {"x": ins["dy"], "w": ins["w"], "y": ins.get("dx")})
    return {"dx": out["y"]}


def convT_wgrad(a, ins):
    return conv_wgrad(a, {"x": ins["dy"], "dy": ins["x"]})


def _bn_out(a, y2, stat, gamma, beta, res):
    z = gamma * (y2 - stat[0]) * stat[1] + beta
    if res is not None:
        z = z + res
    if a.get("relu"):
        z = np.maximum(z, 0.0)
    return _rnd(a)(z)


def bn_fwd(a, ins):
    C = a["C"]
    y2 = ins["y"].reshape(-1, C)
    out = {}
    stat = ins["stat"].reshape(2, C) if a.get("stat_in") else _stat(y2)
    if not a.get("stat_in"):
        out["stat"] = stat
    res = ins["res"].reshape(-1, C) if a.get("has_res") else None
    out["out"] = _bn_out(a, y2, stat, ins["gamma"], ins["beta"], res)
    return out


def _dz_mask(a, ins, y2, stat, C):
    g = ins["g"].reshape(-1, C)
    xh = (y2 - stat[0]) * stat[1]
    if not a.get("relu"):
        return g, xh
    if "out" in ins:
        return g * (ins["out"].reshape(-1, C) > 0), xh
    return g * (ins["gamma"] * xh + ins["beta"] > 0), xh


def bn_bwd_reduce(a, ins):
    C = a["C"]
    y2 = ins["y"].reshape(-1, C)
    stat = ins["stat"].reshape(2, C)
    dz, xh = _dz_mask(a, ins, y2, stat, C)
    return {"dgamma": r32((dz * xh).sum(axis=0)), "dbeta": r32(dz.sum(axis=0))}


def _bn_dy(gamma, stat, dz, xh, dgamma, dbeta, n):
    return gamma * stat[1] * (dz - dbeta / n - xh * (dgamma / n))


def bn_bwd_apply(a, ins):
    C = a["C"]
    rnd = _rnd(a)
    y2 = ins["y"].reshape(-1, C)
    stat = ins["stat"].reshape(2, C)
    dz, xh = _dz_mask(a, ins, y2, stat, C)
    dy = _bn_dy(ins["gamma"], stat, dz, xh, ins["dgamma"], ins["dbeta"], y2.shape[0])
    out = {}
    if a.get("accumulate"):
        out["acc"] = rnd(ins["acc"].reshape(-1, C) + dy)
    else:
        out["y"] = rnd(dy)
    if a.get("has_res"):
        out["g"] = dz
    return out


def _pool_geom(a):
    return a["N"], a["H"], a["W"], a["C"], a["r"], a["stride"], a["pad"], a["P"], a["Q"]


def bn_relu_pool_fwd(a, ins):
    N, H, W, C, r, st, pad, P, Q = _pool_geom(a)
    y2 = ins["y"].reshape(-1, C)
    out = {}
    stat = ins["stat"].reshape(2, C) if a.get("stat_in") else _stat(y2)
    if not a.get("stat_in"):
        out["stat"] = stat
    z = _bn_out(dict(a, relu=True), y2, stat, ins["gamma"], ins["beta"], None).reshape(N, H, W, C)
    out["out"], out["idx"] = nm.maxpool(z, r, st, pad)
    return out


def _pool_dz(a, ins):
    N, H, W, C, r, st, pad, P, Q = _pool_geom(a)
    ga = _rnd(a)(nm.maxpool_backward(ins["g"].reshape(N, P, Q, C), ins["idx"].reshape(N, P, Q, C).astype(np.int64),
                                     (N, H, W, C), r, st, pad)).reshape(-1, C)
    y2 = ins["y"].reshape(-1, C)
    stat = ins["stat"].reshape(2, C)
    xh = (y2 - stat[0]) * stat[1]
    return ga * (ins["gamma"] * xh + ins["beta"] > 0), xh, stat


def pool_bn_bwd_reduce(a, ins):
    dz, xh, _ = _pool_dz(a, ins)
    return {"dgamma": r32((dz * xh).sum(axis=0)), "dbeta": r32(dz.sum(axis=0))}


def pool_bn_bwd_apply(a, ins):
    dz, xh, stat = _pool_dz(a, ins)
    return {"y": _rnd(a)(_bn_dy(ins["gamma"], stat, dz, xh, ins["dgamma"], ins["dbeta"], dz.shape[0]))}


def gap_fwd(a, ins):
    N, HW, C = a["N"], a["HW"], a["C"]
    return {"out": _rnd(a)(ins["x"].reshape(N, HW, C).mean(axis=1))}


def gap_bwd(a, ins):
    N, HW, C = a["N"], a["HW"], a["C"]
    g = ins["g"].reshape(N, 1, C)
    return {"dx": _rnd(a)(np.broadcast_to(g / HW, (N, HW, C)))}


def linear_fwd(a, ins):
    M, N, K = a["M"], a["N"], a["K"]
    rnd = _rnd(a)
    w = ins["w"].reshape(N, K)
    wc = rnd(w) if a.get("dtype", "f32") != "f32" else w
    y = ins["x"].reshape(M, K) @ wc.T + ins["b"]
    if a.get("relu"):
        y = np.maximum(y, 0.0)
    return {"y": r32(y) if (a.get("out_f32") or a.get("dtype", "f32") == "f32") else rnd(y)}


def linear_bwd(a, ins):
    M, N, K = a["M"], a["N"], a["K"]
    rnd = _rnd(a)
    dz = ins["dy"].reshape(M, N)
    if a.get("relu"):
        dz = dz * (ins["y"].reshape(M, N) > 0)
    w = ins["w"].reshape(N, K)
    wc = rnd(w) if a.get("dtype", "f32") != "f32" else w
    out = {"dw": r32(dz.T @ ins["x"].reshape(M, K)), "db": r32(dz.sum(axis=0))}
    dx = dz @ wc
    out["dx"] = rnd(dx) if a.get("dtype", "f32") != "f32" else r32(dx)
    return out


def softmax_ce(a, ins):
    M, N = a["M"], a["N"]
    loss, dz = nm.softmax_ce(ins["logits"].reshape(M, N), ins["labels"].astype(np.int64).reshape(M))
    return {"loss": r32(np.array([loss])), "dlogits": r32(dz)}


def sgd(a, ins):
    lr, mu = a["lr"], a["momentum"]
    outs_w, outs_m = [], []
    for w, g, m in zip(ins["w"], ins["g"], ins["m"]):
        v = r32(mu * m + g)
        outs_m.append(v)
        outs_w.append(r32(w - lr * v))
    return {"w": outs_w, "m": outs_m}


def allreduce(a, ins):
    return {"bufs": list(ins["bufs"])}


def _acc(a, ins, role, val, shape):
    rnd = _rnd(a)
    if a.get("accumulate"):
        return rnd(ins[role].reshape(shape) + val)
    return rnd(val)


def upsample_bilinear_fwd(a, ins):
    x = ins["x"].reshape(a["N"], a["H"], a["W"], a["C"])
    return {"y": _rnd(a)(nm.upsample_bilinear(x, (a["Ho"], a["Wo"])))}


def upsample_bilinear_bwd(a, ins):
    g = ins["g"].reshape(a["N"], a["Ho"], a["Wo"], a["C"])
    shape = (a["N"], a["H"], a["W"], a["C"])
    return {"dx": _acc(a, ins, "dx", nm.upsample_bilinear_backward(g, (a["H"], a["W"])), shape)}


def reflect_pad_fwd(a, ins):
    return {"y": nm.reflect_pad(ins["x"].reshape(a["N"], a["H"], a["W"], a["C"]), a["pad"])}


def reflect_pad_bwd(a, ins):
    p = a["pad"]
    g = ins["g"].reshape(a["N"], a["H"] + 2 * p, a["W"] + 2 * p, a["C"])
    return {"dx": _acc(a, ins, "dx", nm.reflect_pad_backward(g, p), (a["N"], a["H"], a["W"], a["C"]))}


def _in_stat(x):
    mu = x.mean(axis=1)
    var = ((x - mu[:, None, :]) ** 2).mean(axis=1)
    return r32(np.stack([mu, 1.0 / np.sqrt(var + nm.BN_EPS)], axis=1))   # [N, 2, C]


def instnorm_fwd(a, ins):
    N, HW, C = a["N"], a["HW"], a["C"]
    x = ins["x"].reshape(N, HW, C)
    st = _in_stat(x)
    xh = (x - st[:, 0:1, :]) * st[:, 1:2, :]
    return {"stat": st, "out": _rnd(a)(np.maximum(xh, 0.0) if a.get("relu") else xh)}


def instnorm_bwd(a, ins):
    N, HW, C = a["N"], a["HW"], a["C"]
    x = ins["x"].reshape(N, HW, C)
    st = ins["stat"].reshape(N, 2, C)
    xh = (x - st[:, 0:1, :]) * st[:, 1:2, :]
    g = ins["g"].reshape(N, HW, C)
    dz = g * (xh > 0) if a.get("relu") else g
    dx = st[:, 1:2, :] * (dz - dz.mean(axis=1, keepdims=True) - xh * (dz * xh).mean(axis=1, keepdims=True))
    return {"dx": _acc(a, ins, "dx", dx, (N, HW, C))}


def tanh_fwd(a, ins):
    return {"y": _rnd(a)(np.tanh(ins["x"]))}


def tanh_bwd(a, ins):
    return {"dx": _acc(a, ins, "dx", ins["g"] * (1.0 - ins["y"] * ins["y"]), ins["g"].shape)}


def add_fwd(a, ins):
    return {"out": _rnd(a)(ins["a"] + ins["b"])}


def concat_ch_fwd(a, ins):
    rows, Ca, Cb = a["rows"], a["Ca"], a["Cb"]
    return {"out": np.concatenate([ins["a"].reshape(rows, Ca), ins["b"].reshape(rows, Cb)], axis=1)}


def concat_ch_bwd(a, ins):
    rows, Ca, Cb = a["rows"], a["Ca"], a["Cb"]
    g = ins["g"].reshape(rows, Ca + Cb)
    rnd = _rnd(a)
    da = rnd(ins["da"].reshape(rows, Ca) + g[:, :Ca]) if a.get("acc_a") else g[:, :Ca]
    db = rnd(ins["db"].reshape(rows, Cb) + g[:, Ca:]) if a.get("acc_b") else g[:, Ca:]
    return {"da": da, "db": db}


def softmax_ce_pix(a, ins):
    rows, K = a["rows"], a["K"]
    loss, dz = nm.softmax_ce(ins["logits"].reshape(rows, K), ins["labels"].astype(np.int64).reshape(rows))
    return {"loss": r32(np.array([loss])), "dlogits": _rnd(a)(dz)}


def l1_loss(a, ins):
    loss, dy = nm.l1_loss(ins["y"], ins["target"])
    return {"loss": r32(np.array([loss])), "dy": _rnd(a)(dy)}


OPS = {f.__name__: f for f in (conv_fwd, conv_dgrad, conv_wgrad, bn_fwd, bn_bwd_reduce, bn_bwd_apply,
                               bn_relu_pool_fwd, pool_bn_bwd_reduce, pool_bn_bwd_apply, gap_fwd, gap_bwd,
                               linear_fwd, linear_bwd, softmax_ce, sgd, allreduce, convT_fwd, convT_dgrad,
                               convT_wgrad, upsample_bilinear_fwd, upsample_bilinear_bwd, reflect_pad_fwd,
                               reflect_pad_bwd, instnorm_fwd, instnorm_bwd, tanh_fwd, tanh_bwd, add_fwd,
                               concat_ch_fwd, concat_ch_bwd, softmax_ce_pix, l1_loss)}
LIST_ROLES = {"sgd": ("w", "g", "m"), "allreduce": ("bufs",)}


def apply(kind, attrs, ins):
    if kind not in OPS:
        raise KeyError(f"no layer-local definition for op kind {kind!r}")
    return OPS[kind](attrs, ins)


def run_graph(doc, values):
    """Execute the graph document function by function (its declared order,
    which graphs.build emits topologically) with the definitions above.
    values: var name -> float64 array (inputs, parameters, momentum); filled
    in place with every variable's final value.  Returns values."""
    d = json.loads(doc)
    for f in d["functions"]:
        op = f["op"]
        kind, attrs, args = op["kind"], op.get("attrs", {}), op["args"]
        ins = {}
        for role, var in args.items():
            if isinstance(var, list):
                ins[role] = [values[v] for v in var if v in values]
            elif var in values:
                ins[role] = values[var]
        outs = apply(kind, attrs, ins)
        for role, val in outs.items():
            var = args[role]
            if isinstance(var, list):
                for v, x in zip(var, val):
                    values[v] = x
            else:
                values[var] = val
    return values
