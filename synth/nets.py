"""Network specifications (layer lists) for the BASELINE.json configs, and
seeded tensors for them.  Pure data: the oracle interprets a spec with its own
numpy definitions; the product's graph builder unrolls the same spec into a
training-step function graph.

Spec format
  {"name", "mode": "fp32"|"bf16", "batch": b, "input": [F] or [H, W, C],
   "classes": K, "sgd": {"lr", "momentum"},
   "layers": [ {"type": "linear", "name", "in", "out", "features", "relu": bool},
               {"type": "conv",   "name", "in", "out", "k", "r", "s", "stride", "pad"},
               {"type": "bn",     "name", "in", "out", "relu": bool, "residual": tensor|None},
               {"type": "maxpool","name", "in", "out", "r", "stride", "pad"},
               {"type": "gap",    "name", "in", "out"} ],
   "loss": {"type": "softmax_ce", "in": logits tensor}}
The network input tensor is named "x"; labels are "y".  Layout: NHWC
activations, KRSC conv weights, [out, in] linear weights.
"""
import numpy as np

BN_EPS = 1e-5


def mlp6(batch=8, width=256, classes=256, mode="fp32"):
    """configs[0]: 6×Linear(256→256), ReLU after 1-5, softmax-CE over 256
    classes, SGD-momentum 0.9, lr 0.01."""
    layers = []
    prev = "x"
    for i in range(1, 7):
        out = f"h{i}" if i < 6 else "logits"
        layers.append({"type": "linear", "name": f"fc{i}", "in": prev, "out": out,
                       "features": width if i < 6 else classes, "relu": i < 6})
        prev = out
    return {"name": "mlp6", "mode": mode, "batch": batch, "input": [width], "classes": classes,
            "sgd": {"lr": 0.01, "momentum": 0.9}, "layers": layers,
            "loss": {"type": "softmax_ce", "in": "logits"}}


def resnet(depth=18, batch=8, image=224, classes=1000, mode="bf16", width=64, in_ch=3):
    """ResNet-18/34 (basic blocks) or ResNet-50 (bottleneck) in NHWC.  The
    image keeps its 3 channels in memory (the stem's working set bounds the
    feasible budget); kernels pad channels internally."""
    cfg = {18: ("basic", [2, 2, 2, 2]), 34: ("basic", [3, 4, 6, 3]),
           50: ("bottleneck", [3, 4, 6, 3])}[depth]
    kind, blocks = cfg
    L = []

    def conv(name, i, o, k, r, st, pad):
        L.append({"type": "conv", "name": name, "in": i, "out": o, "k": k, "r": r, "s": r,
                  "stride": st, "pad": pad})

    def bn(name, i, o, relu, res=None):
        L.append({"type": "bn", "name": name, "in": i, "out": o, "relu": relu, "residual": res})

    conv("conv1", "x", "c1", width, 7, 2, 3)
    bn("bn1", "c1", "a1", True)
    L.append({"type": "maxpool", "name": "pool1", "in": "a1", "out": "p1", "r": 3, "stride": 2, "pad": 1})
    prev, ch = "p1", width
    for si, nb in enumerate(blocks):
        planes = width * (2 ** si)
        for bi in range(nb):
            st = 2 if (bi == 0 and si > 0) else 1
            pre = f"l{si + 1}b{bi}"
            out_ch = planes * (4 if kind == "bottleneck" else 1)
            res = prev
            if st != 1 or ch != out_ch:
                conv(pre + "_dsc", prev, pre + "_dy", out_ch, 1, st, 0)
                bn(pre + "_dsbn", pre + "_dy", pre + "_ds", False)
                res = pre + "_ds"
            if kind == "basic":
                conv(pre + "_c1", prev, pre + "_y1", planes, 3, st, 1)
                bn(pre + "_bn1", pre + "_y1", pre + "_a1", True)
                conv(pre + "_c2", pre + "_a1", pre + "_y2", planes, 3, 1, 1)
                bn(pre + "_bn2", pre + "_y2", pre + "_out", True, res)
            else:
                conv(pre + "_c1", prev, pre + "_y1", planes, 1, 1, 0)
                bn(pre + "_bn1", pre + "_y1", pre + "_a1", True)
                conv(pre + "_c2", pre + "_a1", pre + "_y2", planes, 3, st, 1)
                bn(pre + "_bn2", pre + "_y2", pre + "_a2", True)
                conv(pre + "_c3", pre + "_a2", pre + "_y3", out_ch, 1, 1, 0)
                bn(pre + "_bn3", pre + "_y3", pre + "_out", True, res)
            prev, ch = pre + "_out", out_ch
    L.append({"type": "gap", "name": "gap", "in": prev, "out": "feat"})
    L.append({"type": "linear", "name": "fc", "in": "feat", "out": "logits", "features": classes,
              "relu": False})
    return {"name": f"resnet{depth}", "mode": mode, "batch": batch, "input": [image, image, in_ch],
            "classes": classes, "sgd": {"lr": 0.1, "momentum": 0.9}, "layers": L,
            "loss": {"type": "softmax_ce", "in": "logits"}}


def preact_resnet(depth=1001, batch=8, image=32, classes=10, mode="bf16", widths=(16, 32, 64)):
    """Pre-activation bottleneck ResNet for CIFAR-shaped inputs (He et al.
    2016, "identity mappings"; the paper cites ResNet-1001 as a model that
    needs out-of-core training): depth = 9n + 2, three stages of n
    bottleneck blocks  a = relu(bn(x)); h = conv1x1 -> bn-relu -> conv3x3(stride)
    -> bn-relu -> conv1x1(4w); out = h + shortcut, shortcut = x or conv1x1(a)."""
    assert (depth - 2) % 9 == 0
    n = (depth - 2) // 9
    L = []
    L.append({"type": "conv", "name": "conv1", "in": "x", "out": "s0", "k": widths[0], "r": 3, "s": 3,
              "stride": 1, "pad": 1})
    prev, ch = "s0", widths[0]
    for si, w in enumerate(widths):
        for bi in range(n):
            st = 2 if (bi == 0 and si > 0) else 1
            pre = f"s{si + 1}b{bi}"
            L.append({"type": "bn", "name": pre + "_bn1", "in": prev, "out": pre + "_a", "relu": True,
                      "residual": None})
            if st != 1 or ch != 4 * w:
                L.append({"type": "conv", "name": pre + "_proj", "in": pre + "_a", "out": pre + "_sc",
                          "k": 4 * w, "r": 1, "s": 1, "stride": st, "pad": 0})
                sc = pre + "_sc"
            else:
                sc = prev
            L.append({"type": "conv", "name": pre + "_c1", "in": pre + "_a", "out": pre + "_h1", "k": w, "r": 1,
                      "s": 1, "stride": 1, "pad": 0})
            L.append({"type": "bn", "name": pre + "_bn2", "in": pre + "_h1", "out": pre + "_a1", "relu": True,
                      "residual": None})
            L.append({"type": "conv", "name": pre + "_c2", "in": pre + "_a1", "out": pre + "_h2", "k": w, "r": 3,
                      "s": 3, "stride": st, "pad": 1})
            L.append({"type": "bn", "name": pre + "_bn3", "in": pre + "_h2", "out": pre + "_a2", "relu": True,
                      "residual": None})
            L.append({"type": "conv", "name": pre + "_c3", "in": pre + "_a2", "out": pre + "_h3", "k": 4 * w,
                      "r": 1, "s": 1, "stride": 1, "pad": 0})
            L.append({"type": "add", "name": pre + "_add", "in": pre + "_h3", "in2": sc, "out": pre + "_out"})
            prev, ch = pre + "_out", 4 * w
    L.append({"type": "bn", "name": "bn_final", "in": prev, "out": "a_final", "relu": True, "residual": None})
    L.append({"type": "gap", "name": "gap", "in": "a_final", "out": "feat"})
    L.append({"type": "linear", "name": "fc", "in": "feat", "out": "logits", "features": classes, "relu": False})
    return {"name": f"preact_resnet{depth}", "mode": mode, "batch": batch, "input": [image, image, 3],
            "classes": classes, "sgd": {"lr": 0.1, "momentum": 0.9}, "layers": L,
            "loss": {"type": "softmax_ce", "in": "logits"}}


def unet(batch=8, image=1024, base=64, depth=4, classes=19, mode="bf16"):
    """U-Net for semantic segmentation (configs[3]): per level two
    conv3×3-BN-ReLU, 2×2 max-pool down, 2×2 stride-2 transposed conv up, the
    skip tensor concatenated with the upsampled one — expressed as a conv with
    two inputs (`in2`, weights W and W2 over the two channel groups, no
    materialised concat) — and a 1×1 head to `classes` logits with a
    per-pixel softmax cross-entropy."""
    L = []

    def cbr(name, i, o, k, i2=None):
        c = {"type": "conv", "name": name + "_c", "in": i, "out": name + "_y", "k": k, "r": 3, "s": 3,
             "stride": 1, "pad": 1}
        if i2:
            c["in2"] = i2
        L.append(c)
        L.append({"type": "bn", "name": name + "_bn", "in": name + "_y", "out": o, "relu": True, "residual": None})

    prev = "x"
    skips = []
    for lvl in range(depth):
        w = base * 2 ** lvl
        cbr(f"e{lvl}a", prev, f"e{lvl}a_o", w)
        cbr(f"e{lvl}b", f"e{lvl}a_o", f"e{lvl}", w)
        skips.append(f"e{lvl}")
        L.append({"type": "maxpool", "name": f"pool{lvl}", "in": f"e{lvl}", "out": f"p{lvl}", "r": 2, "stride": 2,
                  "pad": 0})
        prev = f"p{lvl}"
    w = base * 2 ** depth
    cbr("mida", prev, "mida_o", w)
    cbr("midb", "mida_o", "mid", w)
    prev = "mid"
    for lvl in range(depth - 1, -1, -1):
        w = base * 2 ** lvl
        L.append({"type": "convT", "name": f"up{lvl}", "in": prev, "out": f"u{lvl}", "k": w})
        cbr(f"d{lvl}a", f"u{lvl}", f"d{lvl}a_o", w, i2=skips[lvl])
        cbr(f"d{lvl}b", f"d{lvl}a_o", f"d{lvl}", w)
        prev = f"d{lvl}"
    L.append({"type": "conv", "name": "head", "in": prev, "out": "logits", "k": classes, "r": 1, "s": 1,
              "stride": 1, "pad": 0})
    return {"name": "unet", "mode": mode, "batch": batch, "input": [image, image, 3], "classes": classes,
            "sgd": {"lr": 0.01, "momentum": 0.9}, "layers": L,
            "loss": {"type": "softmax_ce_pix", "in": "logits"}}


def tiny_resnet(batch=4, image=16, classes=10, mode="bf16"):
    """A two-stage basic-block ResNet small enough for the fp64 oracle in
    seconds, with every layer kind of ResNet-18 (stem 7×7/2, maxpool,
    identity and downsample blocks, gap, fc)."""
    spec = resnet(18, batch=batch, image=image, classes=classes, mode=mode, width=16)
    keep = []
    for lay in spec["layers"]:
        if lay["name"].startswith(("l3", "l4")):
            continue
        keep.append(lay)
    for lay in keep:
        if lay["type"] == "gap":
            lay["in"] = "l2b1_out"
    spec["layers"] = keep
    spec["name"] = "tiny_resnet"
    return spec


# ----------------------------------------------------------------------------
# shapes and seeded tensors


def tensor_shapes(spec):
    """Shape of every activation tensor (without batch) and every parameter."""
    return net_shapes(spec["layers"], "x", list(spec["input"]))


def net_shapes(layers, in_name, in_shape):
    shapes = {in_name: list(in_shape)}
    params = {}
    for lay in layers:
        t = lay["type"]
        ish = shapes[lay["in"]]
        if t == "linear":
            fin = int(np.prod(ish))
            params[lay["name"] + ".W"] = [lay["features"], fin]
            params[lay["name"] + ".b"] = [lay["features"]]
            shapes[lay["out"]] = list(lay["reshape"]) if lay.get("reshape") else [lay["features"]]
        elif t == "conv":
            H, W, C = ish
            d = lay.get("dil", 1)
            P = (H + 2 * lay["pad"] - d * (lay["r"] - 1) - 1) // lay["stride"] + 1
            Q = (W + 2 * lay["pad"] - d * (lay["s"] - 1) - 1) // lay["stride"] + 1
            params[lay["name"] + ".W"] = [lay["k"], lay["r"], lay["s"], C]
            if lay.get("in2"):          # second input channel group (concat-conv)
                H2, W2, C2 = shapes[lay["in2"]]
                assert (H2, W2) == (H, W)
                params[lay["name"] + ".W2"] = [lay["k"], lay["r"], lay["s"], C2]
            shapes[lay["out"]] = [P, Q, lay["k"]]
        elif t == "convT":              # 2×2 stride-2 transposed conv, weight [C_in, 2, 2, K_out]
            H, W, C = ish
            params[lay["name"] + ".W"] = [C, 2, 2, lay["k"]]
            shapes[lay["out"]] = [2 * H, 2 * W, lay["k"]]
        elif t == "tconv":             # transposed conv, weight [C_in, r, r, K_out]
            H, W, C = ish
            Ho = (H - 1) * lay["stride"] - 2 * lay["pad"] + lay["r"] + lay.get("out_pad", 0)
            Wo = (W - 1) * lay["stride"] - 2 * lay["pad"] + lay["r"] + lay.get("out_pad", 0)
            params[lay["name"] + ".W"] = [C, lay["r"], lay["r"], lay["k"]]
            shapes[lay["out"]] = [Ho, Wo, lay["k"]]
        elif t == "in":                 # instance norm (no affine parameters)
            shapes[lay["out"]] = list(ish)
        elif t == "reflect_pad":
            shapes[lay["out"]] = [ish[0] + 2 * lay["pad"], ish[1] + 2 * lay["pad"], ish[2]]
        elif t == "upsample_bilinear":
            shapes[lay["out"]] = [lay["size"][0], lay["size"][1], ish[2]]
        elif t == "bn":
            C = ish[-1]
            params[lay["name"] + ".gamma"] = [C]
            params[lay["name"] + ".beta"] = [C]
            shapes[lay["out"]] = list(ish)
        elif t == "maxpool":
            H, W, C = ish
            P = (H + 2 * lay["pad"] - lay["r"]) // lay["stride"] + 1
            Q = (W + 2 * lay["pad"] - lay["r"]) // lay["stride"] + 1
            shapes[lay["out"]] = [P, Q, C]
        elif t == "gap":
            shapes[lay["out"]] = [1, 1, ish[-1]] if lay.get("keepdims") else [ish[-1]]
        elif t == "add":
            assert shapes[lay["in2"]] == ish, (lay["name"], shapes[lay["in2"]], ish)
            shapes[lay["out"]] = list(ish)
        elif t in ("relu", "tanh"):
            shapes[lay["out"]] = list(ish)
        elif t == "concat":             # channel concatenation [in, in2]
            H2, W2, C2 = shapes[lay["in2"]]
            assert (H2, W2) == tuple(ish[:2])
            shapes[lay["out"]] = [ish[0], ish[1], ish[2] + C2]
        elif t == "upsample2":
            shapes[lay["out"]] = [2 * ish[0], 2 * ish[1], ish[2]]
        elif t == "avgpool2":
            shapes[lay["out"]] = [ish[0] // 2, ish[1] // 2, ish[2]]
        elif t == "attn":
            C = ish[-1]
            dq, dv = lay["dq"], lay["dv"]
            params[lay["name"] + ".Wq"] = [dq, 1, 1, C]
            params[lay["name"] + ".Wk"] = [dq, 1, 1, C]
            params[lay["name"] + ".Wv"] = [dv, 1, 1, C]
            params[lay["name"] + ".Wo"] = [C, 1, 1, dv]
            params[lay["name"] + ".gain"] = [1]
            shapes[lay["out"]] = list(ish)
        else:
            raise ValueError(t)
    return shapes, params


def make_inputs(spec, seed_x=0, seed_y=1):
    """x ~ N(0,1) (padded stem channels are zero), y ~ U{0..classes-1}; fp32."""
    b = spec["batch"]
    rx = np.random.default_rng(seed_x)
    x = rx.standard_normal([b] + list(spec["input"])).astype(np.float32)
    if len(spec["input"]) == 3 and spec["input"][2] == 8:
        x[..., 3:] = 0.0
    ysize = b
    if spec.get("loss", {}).get("type") == "l1":   # a target image ~ N(0,1) of the output's shape
        shp, _ = tensor_shapes(spec)
        y = np.random.default_rng(seed_y).standard_normal([b] + shp[spec["loss"]["in"]]).astype(np.float32)
        return x, y
    if spec.get("loss", {}).get("type") == "softmax_ce_pix":   # one label per pixel
        ysize = [b] + list(spec["input"][:2])
    y = np.random.default_rng(seed_y).integers(0, spec["classes"], size=ysize).astype(np.int32)
    return x, y


def make_params(spec, seed=2, pshapes=None):
    """Linear: W, b ~ U(±1/sqrt(fan_in)); conv: W ~ N(0, 2/fan_in) (He);
    BN: gamma = 1, beta = 0; attention gain γ = 0.5 (BigGAN starts at 0,
    which would leave the attention weights without gradient in a one-step
    check).  All fp32."""
    rng = np.random.default_rng(seed)
    if pshapes is None:
        _, pshapes = tensor_shapes(spec)
    out = {}
    for name, shp in pshapes.items():
        if name.endswith(".gain"):
            out[name] = np.full(shp, 0.5, np.float32)
        elif name.endswith(".gamma"):
            out[name] = np.ones(shp, np.float32)
        elif name.endswith(".beta"):
            out[name] = np.zeros(shp, np.float32)
        elif len(shp) == 4:
            fan_in = shp[1] * shp[2] * shp[3]
            out[name] = (rng.standard_normal(shp) * np.sqrt(2.0 / fan_in)).astype(np.float32)
        elif len(shp) == 2:
            bound = 1.0 / np.sqrt(shp[1])
            out[name] = rng.uniform(-bound, bound, shp).astype(np.float32)
        else:
            fan_in = pshapes[name[:-2] + ".W"][1]
            bound = 1.0 / np.sqrt(fan_in)
            out[name] = rng.uniform(-bound, bound, shp).astype(np.float32)
    return out


def densenet(batch=64, image=224, classes=1000, mode="bf16", growth=32, blocks=(6, 12, 24, 16), bn_size=4,
             init=64, compression=0.5):
    """DenseNet-BC (Huang et al.; DenseNet-121 by default), the second workload
    family of the paper's Fig.4/5: stem conv7×7/2-BN-ReLU-
    maxpool3/2; dense layers BN-ReLU-conv1×1(4k)-BN-ReLU-conv3×3(k) whose
    output is concatenated to the running feature map (materialised, one
    2-input concatenation per layer — the quadratic memory the family is known
    for); transitions BN-ReLU-conv1×1(θC)-avgpool2; BN-ReLU-GAP-FC."""
    L = []

    def conv(name, i, o, k, r, st, pad):
        L.append({"type": "conv", "name": name, "in": i, "out": o, "k": k, "r": r, "s": r, "stride": st, "pad": pad})

    def bn(name, i, o):
        L.append({"type": "bn", "name": name, "in": i, "out": o, "relu": True, "residual": None})

    conv("conv0", "x", "c0", init, 7, 2, 3)
    bn("bn0", "c0", "a0")
    L.append({"type": "maxpool", "name": "pool0", "in": "a0", "out": "p0", "r": 3, "stride": 2, "pad": 1})
    prev, C = "p0", init
    for bi, nl in enumerate(blocks):
        for li in range(nl):
            p = f"b{bi}l{li}"
            bn(p + ".bn1", prev, p + ".a1")
            conv(p + ".c1", p + ".a1", p + ".y1", bn_size * growth, 1, 1, 0)
            bn(p + ".bn2", p + ".y1", p + ".a2")
            conv(p + ".c2", p + ".a2", p + ".y2", growth, 3, 1, 1)
            L.append({"type": "concat", "name": p + ".cat", "in": prev, "in2": p + ".y2", "out": p + ".cat"})
            prev, C = p + ".cat", C + growth
        if bi < len(blocks) - 1:
            p = f"t{bi}"
            Ct = int(C * compression)
            bn(p + ".bn", prev, p + ".a")
            conv(p + ".c", p + ".a", p + ".y", Ct, 1, 1, 0)
            L.append({"type": "avgpool2", "name": p + ".pool", "in": p + ".y", "out": p + ".o"})
            prev, C = p + ".o", Ct
    bn("bnf", prev, "af")
    L.append({"type": "gap", "name": "gap", "in": "af", "out": "feat"})
    L.append({"type": "linear", "name": "fc", "in": "feat", "out": "logits", "features": classes, "relu": False})
    return {"name": f"densenet{sum(blocks) * 2 + 5}", "mode": mode, "batch": batch, "input": [image, image, 3],
            "classes": classes, "sgd": {"lr": 0.1, "momentum": 0.9}, "layers": L,
            "loss": {"type": "softmax_ce", "in": "logits"}}


def tiny_densenet(batch=4, image=16, classes=10, mode="bf16"):
    """Two dense blocks of two layers, growth 8, every DenseNet layer kind."""
    return densenet(batch=batch, image=image, classes=classes, mode=mode, growth=8, blocks=(2, 2), bn_size=2,
                    init=16)


def biggan(batch=32, image=128, ch=96, z_dim=120, mode="bf16", n_blocks=5, attn_res=64,
           g_mult=(16, 16, 8, 4, 2, 1), d_mult=(1, 2, 4, 8, 16)):
    """configs[4] first half: a BigGAN-style 128² GAN step.
    G: z -> linear -> 4×4×16ch, 5 up-ResBlocks (BN-ReLU-up-conv3×3-BN-ReLU-
    conv3×3 + up-conv1×1 shortcut), self-attention at 64², BN-ReLU-conv3×3-tanh.
    D: 5 down-ResBlocks (ReLU-conv3×3-ReLU-conv3×3-avgpool + conv1×1-avgpool
    shortcut; no pre-ReLU in the first), self-attention at 64², ReLU, global
    average pool, linear -> score.  Hinge loss, a D-step then a G-step.
    Simplified against BigGAN: unconditional (no class
    embedding / conditional BN / projection), no spectral normalisation,
    SGD-momentum instead of Adam."""
    base = image >> n_blocks
    G, D = [], []
    c0 = g_mult[0] * ch
    G.append({"type": "linear", "name": "g.fc", "in": "z", "out": "g.h0", "features": base * base * c0,
              "relu": False, "reshape": [base, base, c0]})
    prev, res, cin = "g.h0", base, c0
    for b in range(n_blocks):
        cout = g_mult[b + 1] * ch
        p = f"g.b{b}"
        G += [{"type": "bn", "name": p + ".bn1", "in": prev, "out": p + ".a1", "relu": True, "residual": None},
              {"type": "upsample2", "name": p + ".up1", "in": p + ".a1", "out": p + ".u1"},
              {"type": "conv", "name": p + ".c1", "in": p + ".u1", "out": p + ".y1", "k": cout, "r": 3, "s": 3,
               "stride": 1, "pad": 1},
              {"type": "bn", "name": p + ".bn2", "in": p + ".y1", "out": p + ".a2", "relu": True, "residual": None},
              {"type": "conv", "name": p + ".c2", "in": p + ".a2", "out": p + ".y2", "k": cout, "r": 3, "s": 3,
               "stride": 1, "pad": 1},
              {"type": "upsample2", "name": p + ".up0", "in": prev, "out": p + ".u0"},
              {"type": "conv", "name": p + ".sc", "in": p + ".u0", "out": p + ".s0", "k": cout, "r": 1, "s": 1,
               "stride": 1, "pad": 0},
              {"type": "add", "name": p + ".add", "in": p + ".y2", "in2": p + ".s0", "out": p + ".o"}]
        prev, res, cin = p + ".o", res * 2, cout
        if res == attn_res:
            G.append({"type": "attn", "name": p + ".attn", "in": prev, "out": p + ".att", "dq": max(1, cin // 8),
                      "dv": max(1, cin // 2)})
            prev = p + ".att"
    G += [{"type": "bn", "name": "g.bnf", "in": prev, "out": "g.af", "relu": True, "residual": None},
          {"type": "conv", "name": "g.cf", "in": "g.af", "out": "g.yf", "k": 3, "r": 3, "s": 3, "stride": 1,
           "pad": 1},
          {"type": "tanh", "name": "g.tanh", "in": "g.yf", "out": "g.img"}]
    prev, res, cin = "x", image, 3
    for b in range(n_blocks):
        cout = d_mult[b] * ch
        p = f"d.b{b}"
        if b == 0:
            first = prev
        else:
            D.append({"type": "relu", "name": p + ".r0", "in": prev, "out": p + ".r0"})
            first = p + ".r0"
        D += [{"type": "conv", "name": p + ".c1", "in": first, "out": p + ".y1", "k": cout, "r": 3, "s": 3,
               "stride": 1, "pad": 1},
              {"type": "relu", "name": p + ".r1", "in": p + ".y1", "out": p + ".a1"},
              {"type": "conv", "name": p + ".c2", "in": p + ".a1", "out": p + ".y2", "k": cout, "r": 3, "s": 3,
               "stride": 1, "pad": 1},
              {"type": "avgpool2", "name": p + ".pool", "in": p + ".y2", "out": p + ".h"},
              {"type": "conv", "name": p + ".sc", "in": prev, "out": p + ".s0", "k": cout, "r": 1, "s": 1,
               "stride": 1, "pad": 0},
              {"type": "avgpool2", "name": p + ".pool0", "in": p + ".s0", "out": p + ".s1"},
              {"type": "add", "name": p + ".add", "in": p + ".h", "in2": p + ".s1", "out": p + ".o"}]
        prev, res, cin = p + ".o", res // 2, cout
        if res == attn_res:
            D.append({"type": "attn", "name": p + ".attn", "in": prev, "out": p + ".att", "dq": max(1, cin // 8),
                      "dv": max(1, cin // 2)})
            prev = p + ".att"
    D += [{"type": "relu", "name": "d.rf", "in": prev, "out": "d.rf"},
          {"type": "gap", "name": "d.gap", "in": "d.rf", "out": "d.feat"},
          {"type": "linear", "name": "d.fc", "in": "d.feat", "out": "d.score", "features": 1, "relu": False}]
    return {"name": "biggan", "mode": mode, "batch": batch, "z_dim": z_dim, "image": image,
            "sgd": {"lr": 0.01, "momentum": 0.9},
            "G": {"layers": G, "in": "z", "out": "g.img"}, "D": {"layers": D, "in": "x", "out": "d.score"}}


def tiny_biggan(batch=4, mode="fp32"):
    """A 16² GAN with every BigGAN layer kind: 2 up / 2 down blocks, attention at 8²."""
    return biggan(batch=batch, image=16, ch=8, z_dim=8, mode=mode, n_blocks=2, attn_res=8, g_mult=(4, 2, 1),
                  d_mult=(1, 2))


def gan_shapes(spec):
    gs, gp = net_shapes(spec["G"]["layers"], "z", [spec["z_dim"]])
    I = spec["image"]
    ds, dp = net_shapes(spec["D"]["layers"], "x", [I, I, 3])
    return gs, gp, ds, dp


def make_gan_inputs(spec, seed=0):
    """z1, z2 ~ N(0,1) [b, z_dim]; x_real ~ U(−1, 1) NHWC (the tanh range)."""
    b, I = spec["batch"], spec["image"]
    r = np.random.default_rng(seed)
    z1 = r.standard_normal((b, spec["z_dim"])).astype(np.float32)
    z2 = r.standard_normal((b, spec["z_dim"])).astype(np.float32)
    x = r.uniform(-1.0, 1.0, (b, I, I, 3)).astype(np.float32)
    return z1, z2, x


def make_gan_params(spec, seed=2):
    _, gp, _, dp = gan_shapes(spec)
    return make_params(spec, seed, gp), make_params(spec, seed + 1, dp)


def deeplabv3plus(batch=4, image=513, classes=21, mode="bf16", width=64, rates=(6, 12, 18), aspp=256, low=48,
                  blocks=(3, 4, 6, 3)):
    """DeepLabv3+ (the paper's third family, PASCAL VOC 513²) on a
    ResNet-50 backbone at output stride 16: layer4 keeps stride 1 and dilates
    its 3×3 convs by 2; ASPP over the stride-16 features (1×1 conv, three 3×3
    atrous convs at `rates`, image pooling: global average → 1×1 conv → BN-ReLU
    → bilinear back to the map), concatenated and projected by a 1×1 conv; the
    decoder upsamples ×4 (bilinear), concatenates the 1×1-reduced stride-4
    features, two 3×3 convs, a 1×1 classifier and a bilinear upsample to the
    input size; per-pixel softmax cross-entropy.  Every conv is followed by
    BN(-ReLU).  Synthetic shapes: the backbone is ResNet-50 rather than the
    paper's (unstated) one."""
    L = []

    def conv(name, i, o, k, r, st, pad, dil=1):
        L.append({"type": "conv", "name": name, "in": i, "out": o, "k": k, "r": r, "s": r, "stride": st, "pad": pad,
                  "dil": dil})

    def bn(name, i, o, relu, res=None):
        L.append({"type": "bn", "name": name, "in": i, "out": o, "relu": relu, "residual": res})

    def cbr(name, i, o, k, r=1, dil=1):
        conv(name + "_c", i, name + "_y", k, r, 1, dil * (r - 1) // 2, dil)
        bn(name + "_bn", name + "_y", o, True)

    conv("conv1", "x", "c1", width, 7, 2, 3)
    bn("bn1", "c1", "a1", True)
    L.append({"type": "maxpool", "name": "pool1", "in": "a1", "out": "p1", "r": 3, "stride": 2, "pad": 1})
    prev, ch = "p1", width
    for si, nb in enumerate(blocks):
        planes = width * (2 ** si)
        for bi in range(nb):
            st = 2 if (bi == 0 and si in (1, 2)) else 1        # output stride 16: layer4 not strided
            dil = 2 if si == 3 else 1
            pre = f"l{si + 1}b{bi}"
            out_ch = planes * 4
            res = prev
            if st != 1 or ch != out_ch:
                conv(pre + "_dsc", prev, pre + "_dy", out_ch, 1, st, 0)
                bn(pre + "_dsbn", pre + "_dy", pre + "_ds", False)
                res = pre + "_ds"
            conv(pre + "_c1", prev, pre + "_y1", planes, 1, 1, 0)
            bn(pre + "_bn1", pre + "_y1", pre + "_a1", True)
            conv(pre + "_c2", pre + "_a1", pre + "_y2", planes, 3, st, dil, dil)
            bn(pre + "_bn2", pre + "_y2", pre + "_a2", True)
            conv(pre + "_c3", pre + "_a2", pre + "_y3", out_ch, 1, 1, 0)
            bn(pre + "_bn3", pre + "_y3", pre + "_out", True, res)
            prev, ch = pre + "_out", out_ch
    low_feat = "l1b%d_out" % (blocks[0] - 1)
    shapes, _ = net_shapes(L, "x", [image, image, 3])
    fh, fw = shapes[prev][:2]
    lh, lw = shapes[low_feat][:2]
    # ASPP
    cbr("aspp0", prev, "aspp0_o", aspp)
    for j, r in enumerate(rates):
        cbr(f"aspp{j + 1}", prev, f"aspp{j + 1}_o", aspp, 3, r)
    L.append({"type": "gap", "name": "aspp_gap", "in": prev, "out": "aspp_g", "keepdims": True})
    cbr("aspp_pool", "aspp_g", "aspp_p", aspp)
    L.append({"type": "upsample_bilinear", "name": "aspp_up", "in": "aspp_p", "out": "aspp4_o", "size": [fh, fw]})
    cat = "aspp0_o"
    for j in range(1, 5):
        L.append({"type": "concat", "name": f"aspp_cat{j}", "in": cat, "in2": f"aspp{j}_o", "out": f"aspp_cat{j}"})
        cat = f"aspp_cat{j}"
    cbr("aspp_proj", cat, "aspp_out", aspp)
    # decoder
    L.append({"type": "upsample_bilinear", "name": "dec_up", "in": "aspp_out", "out": "dec_u", "size": [lh, lw]})
    cbr("dec_low", low_feat, "dec_l", low)
    L.append({"type": "concat", "name": "dec_cat", "in": "dec_u", "in2": "dec_l", "out": "dec_c"})
    cbr("dec1", "dec_c", "dec1_o", aspp, 3)
    cbr("dec2", "dec1_o", "dec2_o", aspp, 3)
    conv("cls", "dec2_o", "cls_o", classes, 1, 1, 0)
    L.append({"type": "upsample_bilinear", "name": "cls_up", "in": "cls_o", "out": "logits", "size": [image, image]})
    return {"name": "deeplabv3plus", "mode": mode, "batch": batch, "input": [image, image, 3], "classes": classes,
            "sgd": {"lr": 0.01, "momentum": 0.9}, "layers": L, "loss": {"type": "softmax_ce_pix", "in": "logits"}}


def pix2pixhd(batch=1, image=(512, 1024), ngf=64, n_down=4, n_blocks=9, in_ch=3, out_ch=3, mode="bf16"):
    """Pix2PixHD's global generator (the paper's second family, Cityscapes
    512×1024): ReflectionPad 3 → conv 7×7 → IN-ReLU; n_down stride-2
    3×3 convs doubling the channels (IN-ReLU); n_blocks residual blocks
    (reflection pad 1, conv 3×3, IN-ReLU, reflection pad 1, conv 3×3, IN, + x);
    n_down transposed 3×3 stride-2 convs (output padding 1) halving the
    channels (IN-ReLU); ReflectionPad 3 → conv 7×7 → tanh.  IN = instance
    norm without affine parameters.  Trained here against an L1 loss to a
    synthetic target image (the multi-scale discriminator, feature-matching and
    VGG losses of Pix2PixHD are not modelled: synthetic shapes of the
    generator's step)."""
    L = []
    H, W = image

    def conv(name, i, o, k, r, st, pad):
        L.append({"type": "conv", "name": name, "in": i, "out": o, "k": k, "r": r, "s": r, "stride": st,
                  "pad": pad})

    L.append({"type": "reflect_pad", "name": "pad0", "in": "x", "out": "x_p", "pad": 3})
    conv("c0", "x_p", "c0_y", ngf, 7, 1, 0)
    L.append({"type": "in", "name": "in0", "in": "c0_y", "out": "a0", "relu": True})
    prev, ch = "a0", ngf
    for i in range(n_down):
        conv(f"down{i}", prev, f"down{i}_y", ch * 2, 3, 2, 1)
        L.append({"type": "in", "name": f"down{i}_in", "in": f"down{i}_y", "out": f"down{i}_o", "relu": True})
        prev, ch = f"down{i}_o", ch * 2
    for b in range(n_blocks):
        pre = f"res{b}"
        L.append({"type": "reflect_pad", "name": pre + "_p1", "in": prev, "out": pre + "_xp1", "pad": 1})
        conv(pre + "_c1", pre + "_xp1", pre + "_y1", ch, 3, 1, 0)
        L.append({"type": "in", "name": pre + "_in1", "in": pre + "_y1", "out": pre + "_a1", "relu": True})
        L.append({"type": "reflect_pad", "name": pre + "_p2", "in": pre + "_a1", "out": pre + "_xp2", "pad": 1})
        conv(pre + "_c2", pre + "_xp2", pre + "_y2", ch, 3, 1, 0)
        L.append({"type": "in", "name": pre + "_in2", "in": pre + "_y2", "out": pre + "_n2", "relu": False})
        L.append({"type": "add", "name": pre + "_add", "in": prev, "in2": pre + "_n2", "out": pre + "_out"})
        prev = pre + "_out"
    for i in range(n_down):
        L.append({"type": "tconv", "name": f"up{i}", "in": prev, "out": f"up{i}_y", "k": ch // 2, "r": 3,
                  "stride": 2, "pad": 1, "out_pad": 1})
        L.append({"type": "in", "name": f"up{i}_in", "in": f"up{i}_y", "out": f"up{i}_o", "relu": True})
        prev, ch = f"up{i}_o", ch // 2
    L.append({"type": "reflect_pad", "name": "padf", "in": prev, "out": "pf", "pad": 3})
    conv("cf", "pf", "cf_y", out_ch, 7, 1, 0)
    L.append({"type": "tanh", "name": "tanh", "in": "cf_y", "out": "out"})
    return {"name": "pix2pixhd", "mode": mode, "batch": batch, "input": [H, W, in_ch], "classes": out_ch,
            "sgd": {"lr": 0.01, "momentum": 0.9}, "layers": L, "loss": {"type": "l1", "in": "out"}}
