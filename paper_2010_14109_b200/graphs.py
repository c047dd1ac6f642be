"""Training-step graph builder: unrolls a network spec (synth/nets.py) into
the function-sequence the paper schedules — forward, loss, backward and
update functions over sized variables ("including forward, backward,
and update") — with an op descriptor per function for the executor.

This is workload construction, not the method: it decides which variables
exist, their byte sizes and which functions use them.  The planner
(oc_plan_schedule) and the executor (oc_run_step) are in liboocore.

Variable classes (reading Z10):
  params / momentum   persistent (host-authoritative, swappable) for the MLP
                      config; pinned (device-resident) for the conv nets
  grads               swappable for the MLP; pinned for the conv nets
  activations, their gradients, BN statistics, pool indices: swappable
  x, labels           persistent inputs (host) — or pinned when the bench
                      measures with inputs resident in HBM
  loss                persistent (written back to the host every step)
"""
import json

import numpy as np

from synth import nets

F32, BF16, I32, U8 = 4, 2, 4, 1


class Builder:
    def __init__(self, dp_bucket_bytes=0):
        self.vars = []
        self.fns = []
        self.meta = {}
        self._names = set()
        self._bytes = {}
        # data-parallel gradient buckets: see _update
        self.dp_bucket = dp_bucket_bytes
        self.dp_pending, self.dp_prev, self.dp_nbytes, self.dp_count, self.dp_spec = [], [], 0, 0, None

    def var(self, name, nbytes, persistent=False, pinned=False, **meta):
        assert name not in self._names, name
        self._names.add(name)
        self.vars.append({"id": name, "bytes": int(max(1, nbytes)), "persistent": bool(persistent),
                          "pinned": bool(pinned)})
        self._bytes[name] = int(max(1, nbytes))
        self.meta[name] = meta
        return name

    def fn(self, name, kind, args, attrs, ins, outs):
        ins = [v for v in dict.fromkeys(ins) if v is not None]
        outs = [v for v in dict.fromkeys(outs) if v is not None]
        self.fns.append({"id": name, "in": ins, "out": outs,
                         "op": {"kind": kind, "args": {k: v for k, v in args.items() if v is not None},
                                "attrs": attrs}})

    def doc(self):
        if self.dp_bucket:
            _dp_flush(self, final=True)
        return json.dumps({"variables": self.vars, "functions": self.fns}, separators=(",", ":"))


def build(spec, params="persistent", inputs="host", pin_below=0, dp_bucket_bytes=0):
    """Returns (graph document JSON, info dict).  info maps roles to variable
    names: params (name -> var), momentum, grads, x, labels, loss, shapes.

    pin_below: variables smaller than this many bytes (other than the step's
    inputs and loss) are pinned — resident for the whole step, charged to the
    budget, never swapped (Z26: the LMS-style size threshold; with VA
    chunks of m_c bytes a tensor far below m_c would otherwise map a whole
    chunk, Eq.1).

    dp_bucket_bytes: data-parallel replicas — gradients are
    averaged in buckets of about this many bytes, one allreduce function per
    bucket placed right after the backward of its last layer, and the bucket's
    SGD update (one multi-tensor function) one bucket later, so that with a
    communicator attached the exchange of bucket k runs on the executor's
    communication stream while the backward of bucket k+1 computes.  0: one
    allreduce + SGD pair per layer right after its backward (single replica)."""
    if "G" in spec:                       # GAN step (configs[4], graphs_gan.py)
        from .graphs_gan import build_gan
        if dp_bucket_bytes:
            raise ValueError("gradient buckets: not for the GAN step (D's update must precede the G-step)")
        return build_gan(spec, params, inputs)
    if any(l["type"] != "linear" for l in spec["layers"]):
        doc, info = _build_convnet(spec, params, inputs, dp_bucket_bytes)
    else:
        doc, info = _build_mlp(spec, params, inputs, dp_bucket_bytes)
    if pin_below:
        d = json.loads(doc)
        keep = {info["x"], info["labels"], info["loss"]}
        for v in d["variables"]:
            if v["bytes"] < pin_below and v["id"] not in keep:
                v["pinned"], v["persistent"] = True, False
        doc = json.dumps(d, separators=(",", ":"))
    return doc, info


def _pvars(b, spec, pshapes, params):
    persistent = params == "persistent"
    pinned = params == "pinned"
    P, Mo, G = {}, {}, {}
    for name, shp in pshapes.items():
        n = int(np.prod(shp))
        P[name] = b.var(f"{name}", n * F32, persistent=persistent, pinned=pinned, shape=shp, dtype="f32")
        Mo[name] = b.var(f"mom.{name}", n * F32, persistent=persistent, pinned=pinned, shape=shp, dtype="f32")
        G[name] = b.var(f"grad.{name}", n * F32, pinned=pinned, shape=shp, dtype="f32")
    return P, Mo, G


def _dp_flush(b, final=False):
    """Emit the pending bucket's allreduce, then the previous bucket's SGD
    (and at the end of the step the last bucket's SGD too)."""
    if b.dp_pending:
        gs = [G[n] for (_, P, Mo, G, names) in b.dp_pending for n in names]
        b.fn(f"allreduce.bucket{b.dp_count}", "allreduce", {"bufs": gs}, {"bucket": b.dp_count}, gs, gs)
        b.dp_count += 1
    groups = [b.dp_prev] + ([b.dp_pending] if final else [])
    for grp in groups:
        if not grp:
            continue
        ws = [P[n] for (_, P, Mo, G, names) in grp for n in names]
        gs = [G[n] for (_, P, Mo, G, names) in grp for n in names]
        ms = [Mo[n] for (_, P, Mo, G, names) in grp for n in names]
        b.fn(f"sgd.{grp[0][0]}..{grp[-1][0]}", "sgd", {"w": ws, "g": gs, "m": ms},
             {"lr": b.dp_spec["sgd"]["lr"], "momentum": b.dp_spec["sgd"]["momentum"]}, ws + gs + ms, ws + ms)
    b.dp_prev = [] if final else b.dp_pending
    b.dp_pending, b.dp_nbytes = [], 0


def _update(b, spec, layer, P, Mo, G, names):
    """Per-layer gradient all-reduce (a no-op on one replica) and SGD update,
    placed right after the layer's backward function — or, with gradient
    buckets (build(dp_bucket_bytes=...)), the layer joins the open bucket."""
    if b.dp_bucket:
        b.dp_spec = spec
        b.dp_pending.append((layer, P, Mo, G, names))
        b.dp_nbytes += sum(b._bytes[G[n]] for n in names)
        if b.dp_nbytes >= b.dp_bucket:
            _dp_flush(b)
        return
    gs = [G[n] for n in names]
    b.fn(f"allreduce.{layer}", "allreduce", {"bufs": gs}, {}, gs, gs)
    ws, ms = [P[n] for n in names], [Mo[n] for n in names]
    b.fn(f"sgd.{layer}", "sgd", {"w": ws, "g": gs, "m": ms},
         {"lr": spec["sgd"]["lr"], "momentum": spec["sgd"]["momentum"]}, ws + gs + ms, ws + ms)


def _build_mlp(spec, params, inputs, dp_bucket_bytes=0):
    b = Builder(dp_bucket_bytes)
    M = spec["batch"]
    act = F32 if spec["mode"] == "fp32" else BF16
    dt = "f32" if spec["mode"] == "fp32" else "bf16"
    shapes, pshapes = nets.tensor_shapes(spec)
    pin_in = inputs == "pinned"
    x = b.var("x", M * int(np.prod(spec["input"])) * act, persistent=not pin_in, pinned=pin_in,
              shape=[M] + spec["input"], dtype=dt)
    y = b.var("labels", M * I32, persistent=not pin_in, pinned=pin_in, shape=[M], dtype="i32")
    P, Mo, G = _pvars(b, spec, pshapes, params)
    layers = spec["layers"]
    t = {"x": x}
    for lay in layers:
        is_logits = lay["out"] == spec["loss"]["in"]
        nb = M * lay["features"] * (F32 if is_logits else act)
        t[lay["out"]] = b.var(lay["out"], nb, shape=[M, lay["features"]], dtype="f32" if is_logits else dt)
    loss = b.var("loss", F32, persistent=True, shape=[], dtype="f32")
    K = int(np.prod(spec["input"]))
    for lay in layers:
        nm = lay["name"]
        is_logits = lay["out"] == spec["loss"]["in"]
        b.fn(f"fwd.{nm}", "linear_fwd", {"x": t[lay["in"]], "w": P[nm + ".W"], "b": P[nm + ".b"], "y": t[lay["out"]]},
             {"M": M, "N": lay["features"], "K": K, "relu": lay["relu"], "dtype": dt, "out_f32": is_logits},
             [t[lay["in"]], P[nm + ".W"], P[nm + ".b"]], [t[lay["out"]]])
        K = lay["features"]
    logits = t[spec["loss"]["in"]]
    grad = {spec["loss"]["in"]: b.var("grad.logits", M * spec["classes"] * F32, shape=[M, spec["classes"]],
                                      dtype="f32")}
    b.fn("loss", "softmax_ce", {"logits": logits, "labels": y, "loss": loss, "dlogits": grad[spec["loss"]["in"]]},
         {"M": M, "N": spec["classes"]}, [logits, y], [loss, grad[spec["loss"]["in"]]])
    for idx in range(len(layers) - 1, -1, -1):
        lay = layers[idx]
        nm = lay["name"]
        fin = shapes[lay["in"]][0]
        dx = None
        if lay["in"] != "x":
            dx = b.var(f"grad.{lay['in']}", M * fin * act, shape=[M, fin], dtype=dt)
            grad[lay["in"]] = dx
        dy = grad[lay["out"]]
        is_logits = lay["out"] == spec["loss"]["in"]
        b.fn(f"bwd.{nm}", "linear_bwd",
             {"dy": dy, "y": t[lay["out"]] if lay["relu"] else None, "x": t[lay["in"]], "w": P[nm + ".W"],
              "dw": G[nm + ".W"], "db": G[nm + ".b"], "dx": dx},
             {"M": M, "N": lay["features"], "K": fin, "relu": lay["relu"], "dtype": dt, "dy_f32": is_logits},
             [dy, t[lay["out"]] if lay["relu"] else None, t[lay["in"]], P[nm + ".W"]],
             [G[nm + ".W"], G[nm + ".b"], dx])
        _update(b, spec, nm, P, Mo, G, [nm + ".W", nm + ".b"])
    info = {"params": P, "momentum": Mo, "grads": G, "x": x, "labels": y, "loss": loss, "meta": b.meta}
    return b.doc(), info


def _build_convnet(spec, params, inputs, dp_bucket_bytes=0):
    from . import graphs_conv
    return graphs_conv.build_convnet(spec, params, inputs, dp_bucket_bytes)
