"""bf16 dense layers on the tensor cores (kernels/ops_dense.cu → gemm_tc.cu)
through the C-ABI, element by element against the oracle's per-function
definitions (oracle/layerwise.py linear_fwd / linear_bwd: the fp32 master
weight rounded to bf16, fp32 accumulation, bias, optional ReLU; backward with
an fp32 logits gradient (split into an exact bf16 hi + lo pair on the GPU) or
a bf16 hidden-layer gradient).  Shapes: the ResNet FC (512 → 1000) with a
ragged batch, a 120-wide input (the GAN's z), and a ReLU layer (forward on the
tensor cores; its masked backward stays on the SIMT kernel).  bf16 outputs
within the north_star 1e-3; fp32 outputs (logits, dW, db) within 1e-4."""
import json

import numpy as np
import pytest
import torch

from oracle import layerwise as lw
from oracle import numerics as nm

CASES = [  # M, N, K, relu
    (37, 1000, 512, False),
    (200, 24, 120, False),
    (64, 256, 256, True),
]


def _bits(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).view(torch.int16).numpy()


def _dec(raw):
    return (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _run(kind, roles, attrs, inputs, outs):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    vars_ = [{"id": r, "bytes": int(nb), "pinned": True} for r, nb in roles.items()]
    fn = {"id": "f", "in": [r for r in roles if r in inputs], "out": outs,
          "op": {"kind": kind, "args": {r: r for r in roles}, "attrs": attrs}}
    doc = json.dumps({"variables": vars_, "functions": [fn]})
    total = sum(v["bytes"] for v in vars_)
    st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in inputs.items():
        st.write(k, a)
    st.step()
    r = {o: st.read(o, np.uint8) for o in outs}
    st.close()
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("out_f32", [True, False])
def test_linear_fwd_tc(case, out_f32):
    M, N, K, relu = case
    rng = np.random.default_rng(11)
    x = nm.round_bf16(rng.standard_normal((M, K)))
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    b = (rng.standard_normal(N) * 0.1).astype(np.float32)
    at = {"M": M, "N": N, "K": K, "dtype": "bf16", "out_f32": out_f32, "relu": relu}
    roles = {"x": M * K * 2, "w": N * K * 4, "b": N * 4, "y": M * N * (4 if out_f32 else 2)}
    out = _run("linear_fwd", roles, at, {"x": _bits(x), "w": w, "b": b}, ["y"])
    y = out["y"].view(np.float32).astype(np.float64) if out_f32 else _dec(out["y"])
    ref = lw.linear_fwd(at, {"x": x, "w": w.astype(np.float64), "b": b.astype(np.float64)})["y"]
    assert nm.rel_l2(y, ref.reshape(y.shape)) < (1e-4 if out_f32 else 1e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES[:2])
@pytest.mark.parametrize("dy_f32", [True, False])
def test_linear_bwd_tc(case, dy_f32):
    M, N, K, _ = case
    rng = np.random.default_rng(12)
    x = nm.round_bf16(rng.standard_normal((M, K)))
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    dy = rng.standard_normal((M, N)) / M
    dy = dy.astype(np.float32).astype(np.float64) if dy_f32 else nm.round_bf16(dy)
    at = {"M": M, "N": N, "K": K, "dtype": "bf16", "dy_f32": dy_f32}
    roles = {"dy": M * N * (4 if dy_f32 else 2), "x": M * K * 2, "w": N * K * 4, "dw": N * K * 4, "db": N * 4,
             "dx": M * K * 2}
    ins = {"dy": dy.astype(np.float32) if dy_f32 else _bits(dy), "x": _bits(x), "w": w}
    out = _run("linear_bwd", roles, at, ins, ["dw", "db", "dx"])
    ref = lw.linear_bwd(at, {"dy": dy, "x": x, "w": w.astype(np.float64)})
    assert nm.rel_l2(out["dw"].view(np.float32).astype(np.float64), ref["dw"].reshape(-1)) < 1e-4
    assert nm.rel_l2(out["db"].view(np.float32).astype(np.float64), ref["db"].reshape(-1)) < 1e-4
    assert nm.rel_l2(_dec(out["dx"]), ref["dx"].reshape(-1)) < 1e-3
