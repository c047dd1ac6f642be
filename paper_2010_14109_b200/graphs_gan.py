"""GAN training-step graph builder (configs[4], BigGAN-style).

One step, as the oracle's gan_step (oracle/numerics.py):
  D-step   g1.* = G(z1) (forward only)          x_d = concat(x_real, g1.img)
           d1.* = D(x_d), hinge_d, D backward with parameter gradients,
           per-layer all-reduce + SGD of D right after each layer's backward
  G-step   g2.* = G(z2), d2.* = D'(g2.img) through the updated D,
           hinge_g, D backward for data gradients only, then G backward with
           parameter gradients and the per-layer G update.
Functions touch a few whole tensors each, so the schedule's working sets stay
small; the L×L attention map P is an ordinary (large) swappable activation.

Gradient accumulation follows the numerics contract: contributions to one
tensor arrive in reverse layer order, the first stored rounded, later ones
accumulated rnd(G + c) by the consuming op's accumulate mode; a residual add
or the attention residual passes its output gradient on by aliasing the
variable (no kernel).
"""
from synth import nets

from .graphs import BF16, F32, Builder, _pvars, _update


def _chunks(N, L, act, cap=128 << 20):
    """Sample chunks of the attention maps: at most `cap` bytes of P each."""
    nb = max(1, min(N, cap // (L * L * act)))
    return [(n0, min(nb, N - n0)) for n0 in range(0, N, nb)]


class _Pass:
    """One forward (and optionally backward) pass of a layer list."""

    def __init__(self, b, spec, layers, shapes, batch, prefix, P, Mo, G, ACT, DT):
        self.b, self.spec, self.layers, self.shapes = b, spec, layers, shapes
        self.N, self.px = batch, prefix
        self.P, self.Mo, self.G = P, Mo, G
        self.ACT, self.DT = ACT, DT
        self.t = {}           # tensor -> variable
        self.aux = {}         # layer -> saved variables (BN stats, attention q/k/v/P/o)

    def nbytes(self, tensor, dt=None):
        n = self.N
        for d in self.shapes[tensor]:
            n *= d
        return n * (dt or self.ACT)

    def var(self, tensor, dt=None, dtype=None):
        return self.b.var(self.px + tensor, self.nbytes(tensor, dt), shape=[self.N] + self.shapes[tensor],
                          dtype=dtype or self.DT)

    def gvar(self, tensor):
        return self.b.var(self.px + "grad." + tensor, self.nbytes(tensor), shape=[self.N] + self.shapes[tensor],
                          dtype=self.DT)

    def conv_attrs(self, lay, src=None):
        H, W, C = self.shapes[src or lay["in"]]
        Pq, Qq, K = self.shapes[lay["out"]]
        return {"dtype": self.DT, "N": self.N, "H": H, "W": W, "C": C, "K": K, "R": lay["r"], "S": lay["s"],
                "stride": lay["stride"], "pad": lay["pad"], "P": Pq, "Q": Qq}

    # ------------------------------------------------------------ forward
    def forward(self, inputs, fp32_out=()):
        b, t, P = self.b, self.t, self.P
        t.update(inputs)
        for lay in self.layers:
            nm, ty, src = lay["name"], lay["type"], lay["in"]
            x = t[src]
            n_el = self.nbytes(src) // self.ACT
            if ty == "linear":
                f32o = lay["out"] in fp32_out
                y = self.var(lay["out"], F32 if f32o else None, "f32" if f32o else None)
                K = self.nbytes(src) // self.ACT // self.N
                at = {"M": self.N, "N": lay["features"], "K": K, "relu": lay["relu"], "dtype": self.DT,
                      "out_f32": f32o}
                lay["_attrs"] = at
                b.fn(f"{self.px}fwd.{nm}", "linear_fwd", {"x": x, "w": P[nm + ".W"], "b": P[nm + ".b"], "y": y}, at,
                     [x, P[nm + ".W"], P[nm + ".b"]], [y])
            elif ty == "conv":
                y = self.var(lay["out"])
                at = self.conv_attrs(lay)
                b.fn(f"{self.px}fwd.{nm}", "conv_fwd", {"x": x, "w": P[nm + ".W"], "y": y}, at, [x, P[nm + ".W"]], [y])
            elif ty == "bn":
                C = self.shapes[src][-1]
                st = b.var(f"{self.px}stat.{nm}", 2 * C * F32, shape=[2, C], dtype="f32")
                y = self.var(lay["out"])
                at = {"dtype": self.DT, "rows": n_el // C, "C": C, "relu": lay["relu"], "has_res": False}
                self.aux[nm] = (st, at)
                b.fn(f"{self.px}fwd.{nm}", "bn_fwd", {"y": x, "stat": st, "gamma": P[nm + ".gamma"],
                                                      "beta": P[nm + ".beta"], "out": y}, at,
                     [x, P[nm + ".gamma"], P[nm + ".beta"]], [st, y])
            elif ty in ("upsample2", "avgpool2"):
                y = self.var(lay["out"])
                H, W, C = self.shapes[src]
                at = {"dtype": self.DT, "N": self.N, "H": H, "W": W, "C": C}
                b.fn(f"{self.px}fwd.{nm}", ty + "_fwd", {"x": x, "y": y}, at, [x], [y])
            elif ty in ("relu", "tanh"):
                y = self.var(lay["out"])
                b.fn(f"{self.px}fwd.{nm}", ty + "_fwd", {"x": x, "y": y}, {"dtype": self.DT, "n": n_el}, [x], [y])
            elif ty == "add":
                y = self.var(lay["out"])
                b.fn(f"{self.px}fwd.{nm}", "add_fwd", {"a": x, "b": t[lay["in2"]], "out": y},
                     {"dtype": self.DT, "n": n_el}, [x, t[lay["in2"]]], [y])
            elif ty == "gap":
                y = self.var(lay["out"])
                H, W, C = self.shapes[src]
                b.fn(f"{self.px}fwd.{nm}", "gap_fwd", {"x": x, "out": y}, {"dtype": self.DT, "N": self.N,
                                                                         "HW": H * W, "C": C}, [x], [y])
            elif ty == "attn":
                y = self.attn_forward(lay, x)
            else:
                raise ValueError(ty)
            t[lay["out"]] = y
        return t

    def attn_forward(self, lay, x):
        b, P, nm = self.b, self.P, lay["name"]
        H, W, C = self.shapes[lay["in"]]
        L, dq, dv = H * W, lay["dq"], lay["dv"]
        N = self.N

        def v(name, ch, dt=None):
            return b.var(f"{self.px}{nm}.{name}", N * L * ch * (dt or self.ACT), shape=[N, H, W, ch],
                         dtype=self.DT)
        q, k, vv, o, ao = v("q", dq), v("k", dq), v("v", dv), v("o", dv), v("ao", C)
        y = self.var(lay["out"])
        base = {"dtype": self.DT, "N": N, "H": H, "W": W, "C": C, "R": 1, "S": 1, "stride": 1, "pad": 0, "P": H,
                "Q": W}
        for w, out, kk in ((".Wq", q, dq), (".Wk", k, dq), (".Wv", vv, dv)):
            b.fn(f"{self.px}fwd.{nm}{w}", "conv_fwd", {"x": x, "w": P[nm + w], "y": out}, dict(base, K=kk),
                 [x, P[nm + w]], [out])
        # the L×L map in per-chunk variables, one function per chunk of samples,
        # so no function's working set holds the whole batch's maps
        pms, at = [], {"dtype": self.DT, "N": N, "L": L, "dq": dq, "dv": dv}
        for n0, nb in _chunks(N, L, self.ACT):
            pc = b.var(f"{self.px}{nm}.P{n0}", nb * L * L * self.ACT, shape=[nb, L, L], dtype=self.DT)
            atc = dict(at, n0=n0, nb=nb)
            b.fn(f"{self.px}fwd.{nm}.core{n0}", "attn_fwd", {"q": q, "k": k, "v": vv, "p": pc, "o": o}, atc,
                 [q, k, vv] + ([o] if n0 else []), [pc, o])
            pms.append((pc, atc))
        ato = dict(base, C=dv, K=C)
        b.fn(f"{self.px}fwd.{nm}.Wo", "conv_fwd", {"x": o, "w": P[nm + ".Wo"], "y": ao}, ato, [o, P[nm + ".Wo"]],
             [ao])
        b.fn(f"{self.px}fwd.{nm}.res", "scale_add_fwd", {"x": x, "a": ao, "gain": P[nm + ".gain"], "y": y},
             {"dtype": self.DT, "n": N * L * C}, [x, ao, P[nm + ".gain"]], [y])
        self.aux[nm] = {"q": q, "k": k, "v": vv, "P": pms, "o": o, "ao": ao, "base": base, "ato": ato}
        return y

    # ------------------------------------------------------------ backward
    def backward(self, g, params=True, want=()):
        """g: tensor -> gradient variable (seeded with the output's gradient).
        params: emit parameter gradients and the per-layer update; want:
        graph inputs whose gradient is needed."""
        b, t, P, G = self.b, self.t, self.P, self.G
        produced = {lay["out"] for lay in self.layers}

        def need(src):
            return src in produced or src in want

        def into(src):
            """(variable, accumulate) for a gradient contribution to src"""
            if src in g:
                return g[src], True
            g[src] = self.gvar(src)
            return g[src], False

        for lay in reversed(self.layers):
            nm, ty, src = lay["name"], lay["type"], lay["in"]
            if lay["out"] not in g:
                continue
            gv = g[lay["out"]]
            x = t[src]
            pnames = []
            if ty == "linear":
                at = dict(lay["_attrs"], dy_f32=lay["_attrs"]["out_f32"])
                dx = None
                if need(src):
                    dx, acc = into(src)
                    assert not acc, "linear: input gradient accumulation not supported"
                args = {"dy": gv, "x": x, "w": P[nm + ".W"], "dw": G[nm + ".W"] if params else None,
                        "db": G[nm + ".b"] if params else None, "dx": dx}
                outs = [G[nm + ".W"], G[nm + ".b"]] if params else []
                b.fn(f"{self.px}bwd.{nm}", "linear_bwd", args, at, [gv, x, P[nm + ".W"]], outs + ([dx] if dx else []))
                pnames = [nm + ".W", nm + ".b"]
            elif ty == "conv":
                at = self.conv_attrs(lay)
                if params:
                    b.fn(f"{self.px}bwd.{nm}.wgrad", "conv_wgrad", {"dy": gv, "x": x, "dw": G[nm + ".W"]}, at,
                         [gv, x], [G[nm + ".W"]])
                    pnames = [nm + ".W"]
                if need(src):
                    dx, acc = into(src)
                    b.fn(f"{self.px}bwd.{nm}.dgrad", "conv_dgrad", {"dy": gv, "w": P[nm + ".W"], "dx": dx},
                         dict(at, accumulate=acc), [gv, P[nm + ".W"]] + ([dx] if acc else []), [dx])
            elif ty == "bn":
                assert params, "BN backward without parameter gradients is not needed by the GAN step"
                st, at = self.aux[nm]
                yv = x
                dg, db = G[nm + ".gamma"], G[nm + ".beta"]
                args = {"g": gv, "y": yv, "stat": st, "gamma": P[nm + ".gamma"],
                        "beta": P[nm + ".beta"] if lay["relu"] else None, "dgamma": dg, "dbeta": db}
                ins = [gv, yv, st, P[nm + ".gamma"], args["beta"]]
                b.fn(f"{self.px}bwd.{nm}.reduce", "bn_bwd_reduce", args, at, ins, [dg, db])
                if src in g:
                    acc_v = g[src]
                    b.fn(f"{self.px}bwd.{nm}.apply", "bn_bwd_apply", dict(args, acc=acc_v), dict(at, accumulate=True),
                         ins + [dg, db, acc_v], [acc_v])
                else:
                    # in place: y holds dy afterwards (y is not read again in this backward)
                    b.fn(f"{self.px}bwd.{nm}.apply", "bn_bwd_apply", args, at, ins + [dg, db], [yv])
                    g[src] = yv
                pnames = [nm + ".gamma", nm + ".beta"]
            elif ty in ("upsample2", "avgpool2"):
                if need(src):
                    dx, acc = into(src)
                    H, W, C = self.shapes[src]
                    at = {"dtype": self.DT, "N": self.N, "H": H, "W": W, "C": C, "accumulate": acc}
                    b.fn(f"{self.px}bwd.{nm}", ty + "_bwd", {"g": gv, "dx": dx}, at, [gv] + ([dx] if acc else []),
                         [dx])
            elif ty in ("relu", "tanh"):
                if need(src):
                    dx, acc = into(src)
                    ref = x if ty == "relu" else t[lay["out"]]
                    n_el = self.nbytes(src) // self.ACT
                    args = {"g": gv, ("x" if ty == "relu" else "y"): ref, "dx": dx}
                    b.fn(f"{self.px}bwd.{nm}", ty + "_bwd", args, {"dtype": self.DT, "n": n_el, "accumulate": acc},
                         [gv, ref] + ([dx] if acc else []), [dx])
            elif ty == "add":
                for s2 in (src, lay["in2"]):
                    assert s2 not in g, "add: input already has a gradient contribution"
                    g[s2] = gv
            elif ty == "gap":
                dx, acc = into(src)
                assert not acc
                H, W, C = self.shapes[src]
                b.fn(f"{self.px}bwd.{nm}", "gap_bwd", {"g": gv, "dx": dx}, {"dtype": self.DT, "N": self.N,
                                                                          "HW": H * W, "C": C}, [gv], [dx])
            elif ty == "attn":
                pnames = self.attn_backward(lay, gv, g, params)
            if params and pnames:
                _update(b, self.spec, f"{self.px}{nm}", P, self.Mo, G, pnames)
        return g

    def attn_backward(self, lay, gv, g, params):
        b, P, G, nm = self.b, self.P, self.G, lay["name"]
        a = self.aux[nm]
        x = self.t[lay["in"]]
        N, H, W, C = self.N, *self.shapes[lay["in"]]
        dq_, dv_ = lay["dq"], lay["dv"]

        def v(name, ch):
            return b.var(f"{self.px}{nm}.grad.{name}", N * H * W * ch * self.ACT, shape=[N, H, W, ch], dtype=self.DT)
        dao = v("ao", C)
        dgain = G[nm + ".gain"] if params else b.var(f"{self.px}scratch.{nm}.dgain", F32, dtype="f32")
        b.fn(f"{self.px}bwd.{nm}.res", "scale_add_bwd", {"g": gv, "a": a["ao"], "gain": P[nm + ".gain"],
                                                        "dgain": dgain, "da": dao},
             {"dtype": self.DT, "n": N * H * W * C}, [gv, a["ao"], P[nm + ".gain"]], [dgain, dao])
        do = v("o", dv_)
        if params:
            b.fn(f"{self.px}bwd.{nm}.Wo.wgrad", "conv_wgrad", {"dy": dao, "x": a["o"], "dw": G[nm + ".Wo"]},
                 a["ato"], [dao, a["o"]], [G[nm + ".Wo"]])
        b.fn(f"{self.px}bwd.{nm}.Wo.dgrad", "conv_dgrad", {"dy": dao, "w": P[nm + ".Wo"], "dx": do},
             dict(a["ato"], accumulate=False), [dao, P[nm + ".Wo"]], [do])
        dq, dk, dvv = v("q", dq_), v("k", dq_), v("v", dv_)
        for i, (pc, atc) in enumerate(a["P"]):
            b.fn(f"{self.px}bwd.{nm}.core{atc['n0']}", "attn_bwd",
                 {"q": a["q"], "k": a["k"], "v": a["v"], "p": pc, "o": a["o"], "do": do, "dq": dq, "dk": dk,
                  "dv": dvv}, atc, [a["q"], a["k"], a["v"], pc, a["o"], do] + ([dq, dk, dvv] if i else []),
                 [dq, dk, dvv])
        # x's gradient: the residual (aliased, first), then the q, k, v contributions
        assert lay["in"] not in g
        g[lay["in"]] = gv
        for w, d, kk in ((".Wq", dq, dq_), (".Wk", dk, dq_), (".Wv", dvv, dv_)):
            at = dict(a["base"], K=kk)
            if params:
                b.fn(f"{self.px}bwd.{nm}{w}.wgrad", "conv_wgrad", {"dy": d, "x": x, "dw": G[nm + w]}, at, [d, x],
                     [G[nm + w]])
            b.fn(f"{self.px}bwd.{nm}{w}.dgrad", "conv_dgrad", {"dy": d, "w": P[nm + w], "dx": gv},
                 dict(at, accumulate=True), [d, P[nm + w], gv], [gv])
        return [nm + s for s in (".gain", ".Wo", ".Wq", ".Wk", ".Wv")] if params else []


def build_gan(spec, params="persistent", inputs="host"):
    ACT, DT = (BF16, "bf16") if spec["mode"] == "bf16" else (F32, "f32")
    b = Builder()
    N, I, Z = spec["batch"], spec["image"], spec["z_dim"]
    gs, gp, ds, dp = nets.gan_shapes(spec)
    pin_in = inputs == "pinned"
    z1 = b.var("z1", N * Z * ACT, persistent=not pin_in, pinned=pin_in, shape=[N, Z], dtype=DT)
    z2 = b.var("z2", N * Z * ACT, persistent=not pin_in, pinned=pin_in, shape=[N, Z], dtype=DT)
    xr = b.var("x_real", N * I * I * 3 * ACT, persistent=not pin_in, pinned=pin_in, shape=[N, I, I, 3], dtype=DT)
    PG, MG, GG = _pvars(b, spec, gp, params)
    PD, MD, GD = _pvars(b, spec, dp, params)
    Gs, Ds = spec["G"], spec["D"]
    loss_d = b.var("loss_d", F32, persistent=True, shape=[], dtype="f32")
    loss_g = b.var("loss_g", F32, persistent=True, shape=[], dtype="f32")

    # ---------------- D-step
    g1 = _Pass(b, spec, Gs["layers"], gs, N, "g1.", PG, MG, GG, ACT, DT)
    g1.forward({"z": z1})
    xd = b.var("d1.x", 2 * N * I * I * 3 * ACT, shape=[2 * N, I, I, 3], dtype=DT)
    b.fn("d1.concat", "concat_batch", {"a": xr, "b": g1.t[Gs["out"]], "out": xd},
         {"dtype": DT, "na": N * I * I * 3, "nb": N * I * I * 3}, [xr, g1.t[Gs["out"]]], [xd])
    d1 = _Pass(b, spec, Ds["layers"], ds, 2 * N, "d1.", PD, MD, GD, ACT, DT)
    d1.forward({"x": xd}, fp32_out=(Ds["out"],))
    ds1 = b.var("d1.grad.score", 2 * N * F32, shape=[2 * N, 1], dtype="f32")
    b.fn("d1.hinge", "hinge_d", {"score": d1.t[Ds["out"]], "loss": loss_d, "dscore": ds1},
         {"n_real": N, "n_fake": N}, [d1.t[Ds["out"]]], [loss_d, ds1])
    d1.backward({Ds["out"]: ds1}, params=True)

    # ---------------- G-step through the updated D
    g2 = _Pass(b, spec, Gs["layers"], gs, N, "g2.", PG, MG, GG, ACT, DT)
    g2.forward({"z": z2})
    d2 = _Pass(b, spec, Ds["layers"], ds, N, "d2.", PD, MD, GD, ACT, DT)
    d2.forward({"x": g2.t[Gs["out"]]}, fp32_out=(Ds["out"],))
    ds2 = b.var("d2.grad.score", N * F32, shape=[N, 1], dtype="f32")
    b.fn("d2.hinge", "hinge_g", {"score": d2.t[Ds["out"]], "loss": loss_g, "dscore": ds2}, {"n": N},
         [d2.t[Ds["out"]]], [loss_g, ds2])
    gd = d2.backward({Ds["out"]: ds2}, params=False, want=("x",))
    g2.backward({Gs["out"]: gd["x"]}, params=True)
    info = {"G": {"params": PG, "momentum": MG, "grads": GG}, "D": {"params": PD, "momentum": MD, "grads": GD},
            "z1": z1, "z2": z2, "x_real": xr, "loss_d": loss_d, "loss_g": loss_g, "meta": b.meta}
    return b.doc(), info
