"""SAGAN attention core (the BigGAN step's dominant op, configs[4]) through the
C-ABI, element by element against the oracle's definitions
(oracle/numerics.py attention / attention_backward: P = rnd(softmax(q kᵀ)),
o = rnd(P v); dv = rnd(Pᵀ do), dS = P ⊙ (do vᵀ − rowsum), dq = rnd(dS k),
dk = rnd(dSᵀ q)).

bf16 runs the products on the tensor cores (kernels/gemm_tc.cu): K-major and
MN-major operand tiles, zero-filled 12- and 24-wide query dimensions (the
scalar-load path when a row is not 16-byte aligned), the fp32 dS as an exact
bf16 hi + lo pair, ragged tiles (L = 200 against 128-row / 256-column tiles)
and the bench's L = 4096 (64 × 64 feature map).  The backward is checked
layer-locally: it receives the P and o the GPU forward stored, so each output
is compared with its definition on identical inputs at the north_star 1e-3.
fp32 mode keeps the exact SIMT FFMA products (1e-5)."""
import json

import numpy as np
import pytest
import torch

from oracle import numerics as nm

CASES = [  # N, L, dq, dv
    (3, 200, 24, 96),      # ragged L, 16-byte rows
    (2, 200, 12, 48),      # 12-wide q/k rows (24 bytes: scalar loads)
    (2, 64, 8, 16),        # one partial tile
    (3, 512, 24, 96),      # one-pass softmax of 512-wide rows
    (2, 4096, 24, 96),     # the bench's G attention (64 × 64 map)
]


def _bf(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


def _bits(t):
    return t.view(torch.int16).numpy()


def _dec(raw, shape):
    return (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64).reshape(shape)


def _run(kind, N, L, dq, dv, inputs, outs, dtype):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    es = 2 if dtype == "bf16" else 4
    sizes = {"q": N * L * dq, "k": N * L * dq, "v": N * L * dv, "p": N * L * L, "o": N * L * dv, "do": N * L * dv,
             "dq": N * L * dq, "dk": N * L * dq, "dv": N * L * dv}
    names = ["q", "k", "v", "p", "o"] + (["do", "dq", "dk", "dv"] if kind == "attn_bwd" else [])
    vars_ = [{"id": n, "bytes": sizes[n] * es, "pinned": True} for n in names]
    ins = [n for n in names if n in inputs]
    fn = {"id": "f", "in": ins, "out": outs,
          "op": {"kind": kind, "args": {n: n for n in names},
                 "attrs": {"dtype": dtype, "N": N, "L": L, "dq": dq, "dv": dv, "n0": 0, "nb": N}}}
    doc = json.dumps({"variables": vars_, "functions": [fn]})
    total = sum(v["bytes"] for v in vars_)
    st = OutOfCoreStep(doc, total, 0, mode="best", phys_bytes=4096)
    for k, a in inputs.items():
        st.write(k, a)
    st.step()
    r = {o: st.read(o, np.uint16 if dtype == "bf16" else np.float32) for o in outs}
    st.close()
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_attention_bf16_tensor_core(case):
    N, L, dq, dv = case
    rng = np.random.default_rng(7)
    q, k = _bf(rng.standard_normal((N, L, dq)) * 0.5), _bf(rng.standard_normal((N, L, dq)) * 0.5)
    v, do = _bf(rng.standard_normal((N, L, dv))), _bf(rng.standard_normal((N, L, dv)))
    f64 = lambda t: t.float().numpy().astype(np.float64)
    out = _run("attn_fwd", N, L, dq, dv, {"q": _bits(q), "k": _bits(k), "v": _bits(v)}, ["p", "o"], "bf16")
    P, o = _dec(out["p"], (N, L, L)), _dec(out["o"], (N, L, dv))
    Pr, orf = nm.attention(f64(q), f64(k), f64(v), nm.round_bf16)
    assert nm.rel_l2(P, Pr) < 1e-3
    assert nm.rel_l2(o, orf) < 1e-3
    # layer-local backward: the GPU's own P and o
    out = _run("attn_bwd", N, L, dq, dv, {"q": _bits(q), "k": _bits(k), "v": _bits(v), "p": out["p"], "o": out["o"],
                                          "do": _bits(do)}, ["dq", "dk", "dv"], "bf16")
    dqr, dkr, dvr = nm.attention_backward(f64(q), f64(k), f64(v), P, o, f64(do))
    for name, ref, shape in (("dq", dqr, (N, L, dq)), ("dk", dkr, (N, L, dq)), ("dv", dvr, (N, L, dv))):
        got = _dec(out[name], shape)
        assert nm.rel_l2(got, nm.round_bf16(ref)) < 1e-3, name


@pytest.mark.gpu
def test_attention_fp32_simt():
    N, L, dq, dv = 2, 200, 12, 48
    rng = np.random.default_rng(8)
    q, k = rng.standard_normal((N, L, dq)) * 0.5, rng.standard_normal((N, L, dq)) * 0.5
    v, do = rng.standard_normal((N, L, dv)), rng.standard_normal((N, L, dv))
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    q, k, v, do = (f32(a).astype(np.float64) for a in (q, k, v, do))
    out = _run("attn_fwd", N, L, dq, dv, {"q": f32(q), "k": f32(k), "v": f32(v)}, ["p", "o"], "f32")
    P, o = out["p"].astype(np.float64).reshape(N, L, L), out["o"].astype(np.float64).reshape(N, L, dv)
    Pr, orf = nm.attention(q, k, v, lambda a: a.astype(np.float32).astype(np.float64))
    assert nm.rel_l2(P, Pr) < 1e-5 and nm.rel_l2(o, orf) < 1e-5
    out = _run("attn_bwd", N, L, dq, dv, {"q": f32(q), "k": f32(k), "v": f32(v), "p": f32(P), "o": f32(o),
                                          "do": f32(do)}, ["dq", "dk", "dv"], "f32")
    refs = nm.attention_backward(q, k, v, P, o, do)
    for name, ref in zip(("dq", "dk", "dv"), refs):
        assert nm.rel_l2(out[name].astype(np.float64).reshape(ref.shape), ref) < 1e-5, name
