"""Conv-net (ResNet-shaped) training-step graph builder.

Function granularity is chosen so every function's working set stays small
(the budget floor is max_i bytes(V̂_i)):
  conv          conv_fwd            [x, W] -> [y]
  bn(+res,relu) bn_fwd              [y, γ, β, res] -> [out, stat]
  stem bn+pool  bn_relu_pool_fwd    [y, γ, β] -> [pooled, stat, idx]   (the BN
                output is never stored; idx = u8 argmax tap)
  backward, reverse layer order (oracle/numerics.py contract):
  bn            bn_bwd_reduce       [g, out, y, stat, γ] -> [dγ, dβ]
                bn_bwd_apply        [g, out, y, stat, γ, dγ, dβ] -> [y := dy, g := dz]
                (in place: y holds dy afterwards; with a residual, g holds dz,
                which is the residual's first gradient contribution)
  stem          pool_bn_bwd_reduce / pool_bn_bwd_apply (y := dy in place)
  conv          conv_wgrad [dy, x] -> [dW];  conv_dgrad [dy, W, (G)] -> [G]
                (G accumulates: first contribution rnd(c), later rnd(G + c))
  per layer     allreduce [grads] -> [grads]; sgd [W, g, m] -> [W, m]
  DenseNet      concat_ch_fwd [a, b] -> [out]; concat_ch_bwd [g] -> [da, db]
                (each slice stored or accumulated); avgpool2 transitions
"""
import numpy as np

from synth import nets

from .graphs import BF16, F32, I32, U8, Builder, _pvars, _update


def build_convnet(spec, params="pinned", inputs="host", dp_bucket_bytes=0):
    # bf16 storage (tcgen05 convs) or the fp32 parity mode (CUDA-core convs, no TF32)
    ACT, DT = (BF16, "bf16") if spec["mode"] == "bf16" else (F32, "f32")
    b = Builder(dp_bucket_bytes)
    Nb = spec["batch"]
    shapes, pshapes = nets.tensor_shapes(spec)
    pin_in = inputs == "pinned"
    x = b.var("x", Nb * int(np.prod(spec["input"])) * ACT, persistent=not pin_in, pinned=pin_in,
              shape=[Nb] + spec["input"], dtype=DT)
    if spec["loss"]["type"] == "l1":   # the target image (act dtype) of the L1 loss
        tshape = shapes[spec["loss"]["in"]]
        y = b.var("labels", Nb * int(np.prod(tshape)) * ACT, persistent=not pin_in, pinned=pin_in,
                  shape=[Nb] + tshape, dtype=DT)
    else:
        ylen = Nb * (int(np.prod(spec["input"][:2])) if spec["loss"]["type"] == "softmax_ce_pix" else 1)
        y = b.var("labels", ylen * I32, persistent=not pin_in, pinned=pin_in, shape=[ylen], dtype="i32")
    P, Mo, G = _pvars(b, spec, pshapes, params)
    layers = spec["layers"]

    def nbytes(t, dt=ACT):
        return Nb * int(np.prod(shapes[t])) * dt

    # fuse a bn(relu) immediately consumed only by a maxpool (the stem)
    consumers = {}
    for lay in layers:
        for t in [lay["in"]] + [lay[k] for k in ("residual", "in2") if lay.get(k)]:
            consumers.setdefault(t, []).append(lay["name"])
    fused_pool = {}
    for i, lay in enumerate(layers[:-1]):
        nxt = layers[i + 1]
        if lay["type"] == "bn" and lay["relu"] and not lay.get("residual") and nxt["type"] == "maxpool" \
                and nxt["in"] == lay["out"] and consumers[lay["out"]] == [nxt["name"]]:
            fused_pool[lay["name"]] = nxt
    skip = {p["name"] for p in fused_pool.values()}
    # a bn whose input is a plain conv's output gets its batch statistics from
    # that conv (conv_fwd attrs.bn_stat: the tensor-core epilogue sums Σy, Σy²
    # of the stored values per channel, so the bn skips its reduction pass)
    conv_out = {lay["out"]: lay["name"] for lay in layers if lay["type"] == "conv" and not lay.get("in2")}
    bn_of_conv = {}
    if DT == "bf16" and spec.get("fused_bn_stats", True):
        for lay in layers:
            if lay["type"] == "bn" and lay["in"] in conv_out:
                bn_of_conv[conv_out[lay["in"]]] = lay["name"]

    t = {"x": x}       # tensor -> variable holding it
    stat, idx, saved_out = {}, {}, {}
    for lay in layers:
        nm, ty = lay["name"], lay["type"]
        if nm in skip:
            continue
        if ty == "conv":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            Pq, Qq, K = shapes[lay["out"]]
            attrs = {"dtype": DT, "N": Nb, "H": H, "W": W, "C": C, "K": K, "R": lay["r"], "S": lay["s"],
                     "stride": lay["stride"],
                     "pad": lay["pad"], "P": Pq, "Q": Qq}
            if lay.get("dil", 1) > 1:
                attrs["dil"] = lay["dil"]
            lay["_attrs"] = attrs
            if nm in bn_of_conv:
                bnm = bn_of_conv[nm]
                stat[bnm] = b.var(f"stat.{bnm}", 2 * K * F32, shape=[2, K], dtype="f32")
                b.fn(f"fwd.{nm}", "conv_fwd",
                     {"x": t[lay["in"]], "w": P[nm + ".W"], "y": t[lay["out"]], "stat": stat[bnm]},
                     dict(attrs, bn_stat=True), [t[lay["in"]], P[nm + ".W"]], [t[lay["out"]], stat[bnm]])
            else:
                b.fn(f"fwd.{nm}", "conv_fwd", {"x": t[lay["in"]], "w": P[nm + ".W"], "y": t[lay["out"]]}, attrs,
                     [t[lay["in"]], P[nm + ".W"]], [t[lay["out"]]])
            if lay.get("in2"):
                # conv over [in, in2] without materialising the concat: a second conv
                # accumulates into y (y = rnd(y + conv(in2, W2)), Z23)
                C2 = shapes[lay["in2"]][-1]
                lay["_attrs2"] = dict(attrs, C=C2, accumulate=True)
                b.fn(f"fwd.{nm}.2", "conv_fwd", {"x": t[lay["in2"]], "w": P[nm + ".W2"], "y": t[lay["out"]]},
                     lay["_attrs2"], [t[lay["in2"]], P[nm + ".W2"], t[lay["out"]]], [t[lay["out"]]])
        elif ty == "convT":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            # the 2×2 stride-2 conv whose data gradient this is: input = the big map
            # (C_g = K_out), output = the small map (K_g = C_in), weight [C_in][2][2][K_out]
            attrs = {"dtype": DT, "N": Nb, "H": 2 * H, "W": 2 * W, "C": lay["k"], "K": C, "R": 2, "S": 2,
                     "stride": 2, "pad": 0, "P": H, "Q": W}
            lay["_attrs"] = attrs
            b.fn(f"fwd.{nm}", "convT_fwd", {"x": t[lay["in"]], "w": P[nm + ".W"], "y": t[lay["out"]]}, attrs,
                 [t[lay["in"]], P[nm + ".W"]], [t[lay["out"]]])
        elif ty == "tconv":
            # transposed conv (Pix2PixHD): the data gradient of the conv from the
            # output map to the input map (convT_* ops, virtual conv attrs)
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            Ho, Wo, Ko = shapes[lay["out"]]
            attrs = {"dtype": DT, "N": Nb, "H": Ho, "W": Wo, "C": Ko, "K": C, "R": lay["r"], "S": lay["r"],
                     "stride": lay["stride"], "pad": lay["pad"], "P": H, "Q": W}
            lay["_attrs"] = attrs
            b.fn(f"fwd.{nm}", "convT_fwd", {"x": t[lay["in"]], "w": P[nm + ".W"], "y": t[lay["out"]]}, attrs,
                 [t[lay["in"]], P[nm + ".W"]], [t[lay["out"]]])
        elif ty == "in":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            stat[nm] = b.var(f"stat.{nm}", Nb * 2 * C * F32, shape=[Nb, 2, C], dtype="f32")
            lay["_attrs"] = {"dtype": DT, "N": Nb, "HW": H * W, "C": C, "relu": lay["relu"]}
            b.fn(f"fwd.{nm}", "instnorm_fwd", {"x": t[lay["in"]], "out": t[lay["out"]], "stat": stat[nm]},
                 lay["_attrs"], [t[lay["in"]]], [t[lay["out"]], stat[nm]])
        elif ty in ("reflect_pad", "upsample_bilinear"):
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            Ho, Wo, _ = shapes[lay["out"]]
            lay["_attrs"] = {"dtype": DT, "N": Nb, "H": H, "W": W, "C": C, "pad": lay.get("pad", 0), "Ho": Ho,
                             "Wo": Wo}
            b.fn(f"fwd.{nm}", ty + "_fwd", {"x": t[lay["in"]], "y": t[lay["out"]]}, lay["_attrs"], [t[lay["in"]]],
                 [t[lay["out"]]])
        elif ty == "tanh":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            lay["_attrs"] = {"dtype": DT, "n": Nb * int(np.prod(shapes[lay["out"]]))}
            b.fn(f"fwd.{nm}", "tanh_fwd", {"x": t[lay["in"]], "y": t[lay["out"]]}, lay["_attrs"], [t[lay["in"]]],
                 [t[lay["out"]]])
        elif ty == "maxpool":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            idx[nm] = b.var(f"idx.{nm}", nbytes(lay["out"], U8), shape=[Nb] + shapes[lay["out"]], dtype="u8")
            H, W, C = shapes[lay["in"]]
            Pq, Qq, _ = shapes[lay["out"]]
            lay["_attrs"] = {"dtype": DT, "N": Nb, "H": H, "W": W, "C": C, "r": lay["r"], "stride": lay["stride"],
                             "pad": lay["pad"], "P": Pq, "Q": Qq}
            b.fn(f"fwd.{nm}", "maxpool_fwd", {"x": t[lay["in"]], "out": t[lay["out"]], "idx": idx[nm]},
                 lay["_attrs"], [t[lay["in"]]], [t[lay["out"]], idx[nm]])
        elif ty == "bn":
            C = shapes[lay["in"]][-1]
            stat_in = nm in stat   # produced by the conv (bn_stat)
            if not stat_in:
                stat[nm] = b.var(f"stat.{nm}", 2 * C * F32, shape=[2, C], dtype="f32")
            sin = [stat[nm]] if stat_in else []
            sout = [] if stat_in else [stat[nm]]
            if nm in fused_pool:
                pool = fused_pool[nm]
                H, W, _ = shapes[lay["in"]]
                Pq, Qq, _ = shapes[pool["out"]]
                t[pool["out"]] = b.var(pool["out"], nbytes(pool["out"]), shape=[Nb] + shapes[pool["out"]],
                                       dtype=DT)
                idx[nm] = b.var(f"idx.{nm}", nbytes(pool["out"], U8), shape=[Nb] + shapes[pool["out"]], dtype="u8")
                attrs = {"dtype": DT, "N": Nb, "H": H, "W": W, "C": C, "r": pool["r"], "stride": pool["stride"],
                         "pad": pool["pad"],
                         "P": Pq, "Q": Qq}
                lay["_attrs"] = attrs
                ins = [t[lay["in"]], P[nm + ".gamma"], P[nm + ".beta"]] + sin
                b.fn(f"fwd.{nm}+{pool['name']}", "bn_relu_pool_fwd",
                     {"y": t[lay["in"]], "stat": stat[nm], "gamma": P[nm + ".gamma"], "beta": P[nm + ".beta"],
                      "out": t[pool["out"]], "idx": idx[nm]}, dict(attrs, stat_in=stat_in), ins,
                     sout + [t[pool["out"]], idx[nm]])
            else:
                t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
                rows = Nb * int(np.prod(shapes[lay["in"]][:-1]))
                res = t[lay["residual"]] if lay.get("residual") else None
                attrs = {"dtype": DT, "rows": rows, "C": C, "relu": lay["relu"], "has_res": res is not None}
                lay["_attrs"] = attrs
                b.fn(f"fwd.{nm}", "bn_fwd",
                     {"y": t[lay["in"]], "stat": stat[nm], "gamma": P[nm + ".gamma"], "beta": P[nm + ".beta"],
                      "res": res, "out": t[lay["out"]]}, dict(attrs, stat_in=stat_in),
                     [t[lay["in"]], P[nm + ".gamma"], P[nm + ".beta"], res] + sin, sout + [t[lay["out"]]])
        elif ty == "avgpool2":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            lay["_attrs"] = {"dtype": DT, "N": Nb, "H": H, "W": W, "C": C}
            b.fn(f"fwd.{nm}", "avgpool2_fwd", {"x": t[lay["in"]], "y": t[lay["out"]]}, lay["_attrs"],
                 [t[lay["in"]]], [t[lay["out"]]])
        elif ty == "concat":
            # DenseNet: the layer's features appended to the running map (a copy)
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, Ca = shapes[lay["in"]]
            lay["_attrs"] = {"dtype": DT, "rows": Nb * H * W, "Ca": Ca, "Cb": shapes[lay["in2"]][-1]}
            b.fn(f"fwd.{nm}", "concat_ch_fwd", {"a": t[lay["in"]], "b": t[lay["in2"]], "out": t[lay["out"]]},
                 lay["_attrs"], [t[lay["in"]], t[lay["in2"]]], [t[lay["out"]]])
        elif ty == "gap":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            H, W, C = shapes[lay["in"]]
            lay["_attrs"] = {"dtype": DT, "N": Nb, "HW": H * W, "C": C}
            b.fn(f"fwd.{nm}", "gap_fwd", {"x": t[lay["in"]], "out": t[lay["out"]]}, lay["_attrs"], [t[lay["in"]]],
                 [t[lay["out"]]])
        elif ty == "add":
            t[lay["out"]] = b.var(lay["out"], nbytes(lay["out"]), shape=[Nb] + shapes[lay["out"]], dtype=DT)
            lay["_attrs"] = {"dtype": DT, "n": Nb * int(np.prod(shapes[lay["out"]]))}
            b.fn(f"fwd.{nm}", "add_fwd", {"a": t[lay["in"]], "b": t[lay["in2"]], "out": t[lay["out"]]},
                 lay["_attrs"], [t[lay["in"]], t[lay["in2"]]], [t[lay["out"]]])
        elif ty == "linear":
            t[lay["out"]] = b.var(lay["out"], Nb * lay["features"] * F32, shape=[Nb, lay["features"]], dtype="f32")
            K = int(np.prod(shapes[lay["in"]]))
            lay["_attrs"] = {"M": Nb, "N": lay["features"], "K": K, "relu": False, "dtype": DT, "out_f32": True}
            b.fn(f"fwd.{nm}", "linear_fwd", {"x": t[lay["in"]], "w": P[nm + ".W"], "b": P[nm + ".b"],
                                             "y": t[lay["out"]]}, lay["_attrs"],
                 [t[lay["in"]], P[nm + ".W"], P[nm + ".b"]], [t[lay["out"]]])
        else:
            raise ValueError(f"unsupported layer {ty}")
    loss = b.var("loss", F32, persistent=True, shape=[], dtype="f32")
    logits = t[spec["loss"]["in"]]
    g = {}   # tensor -> variable holding its gradient
    if spec["loss"]["type"] == "l1":
        lt = spec["loss"]["in"]
        g[lt] = b.var("grad." + lt, nbytes(lt), shape=[Nb] + shapes[lt], dtype=DT)
        b.fn("loss", "l1_loss", {"y": logits, "target": y, "loss": loss, "dy": g[lt]},
             {"dtype": DT, "n": Nb * int(np.prod(shapes[lt]))}, [logits, y], [loss, g[lt]])
    elif spec["loss"]["type"] == "softmax_ce_pix":
        # per-pixel CE over the channel axis of a conv output (act dtype in and out)
        lt = spec["loss"]["in"]
        g[lt] = b.var("grad.logits", nbytes(lt), shape=[Nb] + shapes[lt], dtype=DT)
        rows = Nb * int(np.prod(shapes[lt][:-1]))
        b.fn("loss", "softmax_ce_pix", {"logits": logits, "labels": y, "loss": loss, "dlogits": g[lt]},
             {"dtype": DT, "rows": rows, "K": spec["classes"]}, [logits, y], [loss, g[lt]])
    else:
        g[spec["loss"]["in"]] = b.var("grad.logits", Nb * spec["classes"] * F32, shape=[Nb, spec["classes"]],
                                      dtype="f32")
        b.fn("loss", "softmax_ce", {"logits": logits, "labels": y, "loss": loss, "dlogits": g[spec["loss"]["in"]]},
             {"M": Nb, "N": spec["classes"]}, [logits, y], [loss, g[spec["loss"]["in"]]])

    # tensors that carry no gradient: the input image and whatever parameter-free
    # single-input layers derive from it alone (Pix2PixHD's reflection-padded
    # input) — the conv reading one needs its weight gradient but no dgrad
    nograd = {"x"}
    for lay in layers:
        if lay["type"] in ("reflect_pad", "upsample_bilinear", "tanh", "avgpool2", "in") and lay["in"] in nograd:
            nograd.add(lay["out"])

    for lay in reversed(layers):
        nm, ty = lay["name"], lay["type"]
        if nm in skip:
            continue
        out_t = fused_pool[nm]["out"] if nm in fused_pool else lay["out"]
        if out_t not in g:
            continue
        gv = g[out_t]
        if ty == "linear":
            dx = b.var(f"grad.{lay['in']}", nbytes(lay["in"]), shape=[Nb] + shapes[lay["in"]], dtype=DT)
            at = dict(lay["_attrs"], dy_f32=True)
            b.fn(f"bwd.{nm}", "linear_bwd", {"dy": gv, "x": t[lay["in"]], "w": P[nm + ".W"], "dw": G[nm + ".W"],
                                             "db": G[nm + ".b"], "dx": dx}, at,
                 [gv, t[lay["in"]], P[nm + ".W"]], [G[nm + ".W"], G[nm + ".b"], dx])
            g[lay["in"]] = dx
            _update(b, spec, nm, P, Mo, G, [nm + ".W", nm + ".b"])
        elif ty == "gap":
            assert lay["in"] not in g
            dx = b.var(f"grad.{lay['in']}", nbytes(lay["in"]), shape=[Nb] + shapes[lay["in"]], dtype=DT)
            b.fn(f"bwd.{nm}", "gap_bwd", {"g": gv, "dx": dx}, lay["_attrs"], [gv], [dx])
            g[lay["in"]] = dx
        elif ty == "bn" and nm in fused_pool:
            yv = t[lay["in"]]
            args = {"g": gv, "idx": idx[nm], "y": yv, "stat": stat[nm], "gamma": P[nm + ".gamma"],
                    "beta": P[nm + ".beta"], "dgamma": G[nm + ".gamma"], "dbeta": G[nm + ".beta"]}
            b.fn(f"bwd.{nm}.reduce", "pool_bn_bwd_reduce", args, lay["_attrs"],
                 [gv, idx[nm], yv, stat[nm], P[nm + ".gamma"], P[nm + ".beta"]], [G[nm + ".gamma"], G[nm + ".beta"]])
            b.fn(f"bwd.{nm}.apply", "pool_bn_bwd_apply", args, lay["_attrs"],
                 [gv, idx[nm], yv, stat[nm], P[nm + ".gamma"], P[nm + ".beta"], G[nm + ".gamma"], G[nm + ".beta"]],
                 [yv])
            g[lay["in"]] = yv                    # y now holds dy
            _update(b, spec, nm, P, Mo, G, [nm + ".gamma", nm + ".beta"])
        elif ty == "bn":
            yv, ov = t[lay["in"]], t[lay["out"]]
            res = lay.get("residual")
            # ReLU mask: from the stored output only when a residual entered the sum;
            # otherwise recomputed from y, γ, β — the backward then touches g and y only
            use_out = lay["relu"] and bool(res)
            args = {"g": gv, "out": ov if use_out else None, "y": yv, "stat": stat[nm], "gamma": P[nm + ".gamma"],
                    "beta": P[nm + ".beta"] if (lay["relu"] and not use_out) else None,
                    "dgamma": G[nm + ".gamma"], "dbeta": G[nm + ".beta"]}
            ins = [gv, ov if use_out else None, yv, stat[nm], P[nm + ".gamma"], args["beta"]]
            b.fn(f"bwd.{nm}.reduce", "bn_bwd_reduce", args, lay["_attrs"], ins, [G[nm + ".gamma"], G[nm + ".beta"]])
            if lay["in"] in g:
                # the BN input has another consumer whose gradient arrived first (a
                # pre-activation block's shortcut): accumulate dy into it, G = rnd(G + dy)
                acc_v = g[lay["in"]]
                b.fn(f"bwd.{nm}.apply", "bn_bwd_apply", dict(args, acc=acc_v), dict(lay["_attrs"], accumulate=True),
                     ins + [G[nm + ".gamma"], G[nm + ".beta"], acc_v], [acc_v] + ([gv] if res else []))
            else:
                b.fn(f"bwd.{nm}.apply", "bn_bwd_apply", args, lay["_attrs"],
                     ins + [G[nm + ".gamma"], G[nm + ".beta"]], [yv] + ([gv] if res else []))
                g[lay["in"]] = yv
            if res:
                assert res not in g, "residual must receive its first gradient here"
                g[res] = gv                      # gv now holds dz
            _update(b, spec, nm, P, Mo, G, [nm + ".gamma", nm + ".beta"])
        elif ty == "add":
            # out = a + b: both inputs receive g.  No kernel: the gradient variable
            # is shared; in a pre-activation block every reader of g[a] (the last
            # conv's backward) runs before any accumulation into g[b] (the shortcut's
            # other consumer), so the aliasing is safe in the reverse layer order.
            for src in (lay["in"], lay["in2"]):
                assert src not in g, "add: input already has a gradient contribution"
                g[src] = gv
        elif ty == "conv":
            dy = gv
            parts = [(lay["in"], nm + ".W", lay["_attrs"], "")]
            if lay.get("in2"):
                parts.append((lay["in2"], nm + ".W2", lay["_attrs2"], "2"))
            for src, wname, at, sfx in parts:
                at = {k: v for k, v in at.items() if k != "accumulate"}
                b.fn(f"bwd.{nm}.wgrad{sfx}", "conv_wgrad", {"dy": dy, "x": t[src], "dw": G[wname]}, at,
                     [dy, t[src]], [G[wname]])
                if src not in nograd:
                    acc = src in g
                    if acc:
                        dx = g[src]
                        ins = [dy, P[wname], dx]
                    else:
                        dx = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                        ins = [dy, P[wname]]
                        g[src] = dx
                    b.fn(f"bwd.{nm}.dgrad{sfx}", "conv_dgrad", {"dy": dy, "w": P[wname], "dx": dx},
                         dict(at, accumulate=acc), ins, [dx])
            _update(b, spec, nm, P, Mo, G, [p[1] for p in parts])
        elif ty == "convT":
            # dW via the virtual conv's wgrad with the roles of its input/output-gradient swapped
            src = lay["in"]
            b.fn(f"bwd.{nm}.wgrad", "convT_wgrad", {"dy": gv, "x": t[src], "dw": G[nm + ".W"]}, lay["_attrs"],
                 [gv, t[src]], [G[nm + ".W"]])
            if src in nograd:
                _update(b, spec, nm, P, Mo, G, [nm + ".W"])
                continue
            acc = src in g
            if acc:
                dx = g[src]
                ins = [gv, P[nm + ".W"], dx]
            else:
                dx = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                ins = [gv, P[nm + ".W"]]
                g[src] = dx
            b.fn(f"bwd.{nm}.dgrad", "convT_dgrad", {"dy": gv, "w": P[nm + ".W"], "dx": dx},
                 dict(lay["_attrs"], accumulate=acc), ins, [dx])
            _update(b, spec, nm, P, Mo, G, [nm + ".W"])
        elif ty == "tconv":
            src = lay["in"]
            b.fn(f"bwd.{nm}.wgrad", "convT_wgrad", {"dy": gv, "x": t[src], "dw": G[nm + ".W"]}, lay["_attrs"],
                 [gv, t[src]], [G[nm + ".W"]])
            if src in nograd:
                _update(b, spec, nm, P, Mo, G, [nm + ".W"])
                continue
            acc = src in g
            if acc:
                dx = g[src]
                ins = [gv, P[nm + ".W"], dx]
            else:
                dx = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                ins = [gv, P[nm + ".W"]]
                g[src] = dx
            b.fn(f"bwd.{nm}.dgrad", "convT_dgrad", {"dy": gv, "w": P[nm + ".W"], "dx": dx},
                 dict(lay["_attrs"], accumulate=acc), ins, [dx])
            _update(b, spec, nm, P, Mo, G, [nm + ".W"])
        elif ty in ("in", "reflect_pad", "upsample_bilinear", "tanh"):
            src = lay["in"]
            if src in nograd:
                continue
            acc = src in g
            if acc:
                dx = g[src]
            else:
                dx = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                g[src] = dx
            at = dict(lay["_attrs"], accumulate=acc)
            if ty == "in":
                args = {"g": gv, "x": t[src], "stat": stat[nm], "dx": dx}
                ins = [gv, t[src], stat[nm]]
            elif ty == "tanh":
                args = {"g": gv, "y": t[lay["out"]], "dx": dx}
                ins = [gv, t[lay["out"]]]
            else:
                args = {"g": gv, "dx": dx}
                ins = [gv]
            b.fn(f"bwd.{nm}", {"in": "instnorm", "tanh": "tanh"}.get(ty, ty) + "_bwd", args, at,
                 ins + ([dx] if acc else []), [dx])
        elif ty == "avgpool2":
            src = lay["in"]
            acc = src in g
            if acc:
                dx = g[src]
                ins = [gv, dx]
            else:
                dx = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                ins = [gv]
                g[src] = dx
            b.fn(f"bwd.{nm}", "avgpool2_bwd", {"g": gv, "dx": dx}, dict(lay["_attrs"], accumulate=acc), ins, [dx])
        elif ty == "concat":
            outs, ins, accs = [], [gv], []
            for src in (lay["in"], lay["in2"]):
                acc = src in g
                if acc:
                    ins.append(g[src])
                else:
                    g[src] = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                outs.append(g[src])
                accs.append(acc)
            b.fn(f"bwd.{nm}", "concat_ch_bwd", {"g": gv, "da": outs[0], "db": outs[1]},
                 dict(lay["_attrs"], acc_a=accs[0], acc_b=accs[1]), ins, outs)
        elif ty == "maxpool":
            src = lay["in"]
            acc = src in g
            if acc:
                dx = g[src]
                ins = [gv, idx[nm], dx]
            else:
                dx = b.var(f"grad.{src}", nbytes(src), shape=[Nb] + shapes[src], dtype=DT)
                ins = [gv, idx[nm]]
                g[src] = dx
            b.fn(f"bwd.{nm}", "maxpool_bwd", {"g": gv, "idx": idx[nm], "dx": dx},
                 dict(lay["_attrs"], accumulate=acc), ins, [dx])
        else:
            raise ValueError(ty)
    info = {"params": P, "momentum": Mo, "grads": G, "x": x, "labels": y, "loss": loss, "meta": b.meta}
    return b.doc(), info
