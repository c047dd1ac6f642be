"""configs[3] family — U-Net (concat-conv without a materialised concat,
plain max-pool with a skip consumer, 2×2 stride-2 transposed conv through
the conv kernels, per-pixel softmax cross-entropy): GPU parity with the oracle
in fp32 (1e-5), bitwise swap transparency in bf16, transposed-conv kernels
in bf16 against the direct definition, and the 1024² config's feasibility
at 1/8 of its footprint (CPU)."""
import json

import numpy as np
import pytest
import torch

from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

from test_gpu_resnet import run_step  # noqa: E402

MiB = 1 << 20


def test_unet_1024_feasible_at_one_eighth():
    spec = nets.unet(batch=8)
    doc, _ = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    assert G.min_feasible_budget(0) <= peak // 8
    W = G.max_feasible_window(peak // 8)
    s = G.plan(peak // 8, W, B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=peak, allow_oom=True)
    assert s.stats()["peak_sched"] <= peak // 8


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_unet_parity_fp32(mode):
    spec = nets.unet(batch=2, image=32, base=8, depth=2, classes=5, mode="fp32")
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    budget = max(G.min_feasible_budget(0), peak // 3)
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    ref = nm.train_step(spec, p, x, y)
    out = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE, mode, None, fp32_input=True)
    assert out["metrics"]["bytes_d2h"] > 0
    assert abs(out["loss"] - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    errs = {k: nm.rel_l2(out["m." + k], ref["grads"][k]) for k in p}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= 1e-5, (worst, errs[worst])


@pytest.mark.gpu
def test_unet_bf16_transparency_and_loss():
    spec = nets.unet(batch=2, image=64, base=64, depth=2, classes=19)
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    x, y = nets.make_inputs(spec)
    ooc = run_step(spec, doc, info, max(G.min_feasible_budget(0), peak // 6), B.OC_WINDOW_MAX_FEASIBLE, "va", None)
    inc = run_step(spec, doc, info, peak, 0, "best", None)
    assert ooc["metrics"]["bytes_d2h"] > 0
    for k in nets.make_params(spec):
        assert np.array_equal(ooc["m." + k], inc["m." + k]), k
    ref = nm.train_step(spec, nets.make_params(spec), x, y)
    assert abs(ooc["loss"] - ref["loss"]) <= 1e-3 * abs(ref["loss"])


def _bf(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


def _run1(kind, args, vars_, attrs, inputs, out_name, out_dtype):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    v = [{"id": n, "bytes": int(b), "pinned": True} for n, b in vars_]
    ins = [args[k] for k in args if k not in ("y", "dx", "dw")] + ([args["dx"]] if attrs.get("accumulate") else [])
    outs = [args[k] for k in ("y", "dx", "dw") if k in args]
    doc = json.dumps({"variables": v, "functions": [{"id": "f", "in": ins, "out": outs,
                                                      "op": {"kind": kind, "args": args, "attrs": attrs}}]})
    st = OutOfCoreStep(doc, sum(b for _, b in vars_), 0, mode="best", phys_bytes=4096)
    for k, a in inputs.items():
        st.write(k, a)
    st.step()
    r = st.read(out_name, out_dtype)
    st.close()
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(2, 5, 7, 128, 64), (1, 8, 8, 256, 128)])
def test_conv_transpose_kernels_bf16(shape):
    N, H, W, C, K = shape
    rng = np.random.default_rng(4)
    x = _bf(rng.standard_normal((N, H, W, C)))
    w = (rng.standard_normal((C, 2, 2, K)) * 0.1).astype(np.float32)
    g = _bf(rng.standard_normal((N, 2 * H, 2 * W, K)))
    at = {"dtype": "bf16", "N": N, "H": 2 * H, "W": 2 * W, "C": K, "K": C, "R": 2, "S": 2, "stride": 2, "pad": 0,
          "P": H, "Q": W}
    xs, ys, ws = N * H * W * C * 2, N * 4 * H * W * K * 2, C * 4 * K * 4
    bits = lambda t: t.view(torch.int16).numpy()
    unb = lambda a, s: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).float().numpy().reshape(s).astype(
        np.float64)
    w_bf = nm.round_bf16(w.astype(np.float64))
    y = _run1("convT_fwd", {"x": "x", "w": "w", "y": "y"}, [("x", xs), ("w", ws), ("y", ys)], at,
              {"x": bits(x), "w": w}, "y", np.uint16)
    ref = nm.round_bf16(nm.conv_transpose2x2(x.float().numpy().astype(np.float64), w_bf))
    assert nm.rel_l2(unb(y, (N, 2 * H, 2 * W, K)), ref) < 2e-3
    dx_ref, dw_ref = nm.conv_transpose2x2_backward(x.float().numpy().astype(np.float64), w_bf,
                                                   g.float().numpy().astype(np.float64))
    dx = _run1("convT_dgrad", {"dy": "dy", "w": "w", "dx": "dx"}, [("dy", ys), ("w", ws), ("dx", xs)], at,
               {"dy": bits(g), "w": w}, "dx", np.uint16)
    assert nm.rel_l2(unb(dx, (N, H, W, C)), nm.round_bf16(dx_ref)) < 2e-3
    dw = _run1("convT_wgrad", {"dy": "dy", "x": "x", "dw": "dw"}, [("dy", ys), ("x", xs), ("dw", ws)], at,
               {"dy": bits(g), "x": bits(x)}, "dw", np.float32)
    assert nm.rel_l2(dw.reshape(C, 2, 2, K), dw_ref) < 1e-5
