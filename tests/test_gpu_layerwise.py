"""Layer-local parity of the whole out-of-core training step with the oracle,
at north_star's 1e-3, for deep bf16 nets at full 224^2 resolution — including
the bench's own configuration (configs[1]: ResNet-18, batch 256, 25 % of
F_peak, tensors < 1 MiB pinned, VA 2 MiB chunks, window 0).

End to end, a deep bf16 net is chaotic (Z24: a 1e-6 perturbation
of one conv output moves the oracle's own parameter gradients by ~27 %), so
per-gradient 1e-3 parity of the final gradients is ill-posed.  Layer-locally
it is well posed: the step is the ordinary training step executed function
by function, so each function f_i must compute its definition
(oracle/layerwise.py, pinned to numerics.train_step in
tests/test_oracle_layerwise.py) from the values it read.  The executor's
inspection hook (oc_exec_set_hook / oc_exec_read_var) captures, on the GPU,
the bytes of every input of f_i right before its kernels and of every output
right after them, during a real out-of-core step (swaps, VA mappings and the
same kernels and launch configuration as the bench, issued eagerly); the
oracle applies f_i's definition to the captured inputs and every output is
compared element by element:
  * floating-point outputs (bf16 activations and activation gradients, fp32
    BN statistics, parameter gradients, logits, loss, momentum, parameters):
    relative L2 <= 1e-3 (north_star "within 1e-3 relative for bf16");
  * the max-pool argmax (u8): where floating point decides an integer the
    kernel evaluates BN in fp32 and the oracle in fp64, so a window whose two
    best taps round to within one bf16 ulp may pick either — at most 1e-3 of
    the entries may differ, and the pooled values themselves are held to
    1e-3 above.
Every function of the step is checked; the worst error per op kind is
printed (and written to $OC_LAYERWISE_REPORT as JSON when set)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import layerwise
from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20
TOL = 1e-3


def decode(raw, dtype):
    if dtype == "bf16":
        return (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if dtype == "f32":
        return raw.view(np.float32).astype(np.float64)
    if dtype == "i32":
        return raw.view(np.int32).astype(np.int64)
    if dtype == "u8":
        return raw.astype(np.int64)
    raise ValueError(dtype)


def run_layerwise(spec, budget_frac=0.25, pin_below=MiB, mode="va", window=0, chunk=2 * MiB):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    doc, info = graphs.build(spec, params="persistent", inputs="host", pin_below=pin_below)
    meta = info["meta"]
    G = B.Graph(doc)
    budget = max(G.min_feasible_budget(window), int(G.in_core_peak() * budget_frac))
    m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST}[mode]
    probe = G.plan(budget, window, m, chunk_bytes=chunk, phys_bytes=budget * 4, allow_oom=True).stats()
    st = OutOfCoreStep(doc, budget, window, mode=mode, chunk_bytes=chunk,
                       phys_bytes=probe["peak_phys"] + chunk if mode == "va" else probe["peak_phys"])
    assert st.stats["bytes_d2h"] > 0, "the budget must force swap-outs"
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy())
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    fns = json.loads(doc)["functions"]
    by_pos = {int(B.lib().oc_graph_fn_position(G.h, j)): f for j, f in enumerate(fns)}
    state = {"pre": None}
    worst, failures, checked = {}, [], [0]

    def rd(v):
        return decode(st.read_device(v), meta[v]["dtype"])

    def hook(i, phase):
        try:
            f = by_pos[i]
            if phase == 0:
                state["pre"] = {v: rd(v) for v in f["in"]}
                return
            pre, post = state["pre"], {v: rd(v) for v in f["out"]}
            op = f["op"]
            kind, attrs, args = op["kind"], op.get("attrs", {}), op["args"]
            ins = {}
            for role, var in args.items():
                if isinstance(var, list):
                    if all(v in pre for v in var):
                        ins[role] = [pre[v] for v in var]
                elif var in pre:
                    ins[role] = pre[var]
            outs = layerwise.apply(kind, attrs, ins)
            for role, exp in outs.items():
                vs = args[role] if isinstance(args[role], list) else [args[role]]
                es = exp if isinstance(args[role], list) else [exp]
                for v, e in zip(vs, es):
                    got = post[v]
                    e = np.asarray(e, np.float64).reshape(-1)
                    if meta[v]["dtype"] == "u8":
                        err = float(np.mean(got != e))
                    else:
                        err = nm.rel_l2(got, e)
                    key = f"{kind}.{role}"
                    worst[key] = max(worst.get(key, 0.0), err)
                    if not err <= TOL:
                        failures.append((f["id"], role, v, err))
            checked[0] += 1
        except Exception as ex:  # noqa: BLE001 — ctypes swallows exceptions raised in callbacks
            failures.append((by_pos.get(i, {}).get("id"), "exception", repr(ex)[:300], None))

    st.set_hook(hook)
    met = st.step()
    st.set_hook(None)
    st.close()
    return {"functions": len(fns), "checked": checked[0], "worst": worst, "failures": failures,
            "bytes_h2d": met["bytes_h2d"], "bytes_d2h": met["bytes_d2h"]}


def _report(name, r):
    line = {"case": name, "functions": r["functions"], "checked": r["checked"], "bytes_h2d": r["bytes_h2d"],
            "bytes_d2h": r["bytes_d2h"], "worst_by_op_role": {k: float(f"{v:.3e}") for k, v in sorted(r["worst"].items())}}
    print(json.dumps(line))
    path = os.environ.get("OC_LAYERWISE_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(line) + "\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name,spec", [
    ("resnet18_224_b16", nets.resnet(18, batch=16)),
    ("resnet50_224_b8", nets.resnet(50, batch=8)),
])
def test_layerwise_parity(name, spec):
    r = run_layerwise(spec)
    _report(name, r)
    assert r["checked"] == r["functions"]
    assert not r["failures"], r["failures"][:10]


@pytest.mark.gpu
def test_layerwise_parity_bench_config():
    """configs[1] exactly as bench.py times it (batch 256): every function,
    every output element."""
    r = run_layerwise(nets.resnet(18, batch=256))
    _report("resnet18_224_b256_bench", r)
    assert r["checked"] == r["functions"]
    assert not r["failures"], r["failures"][:10]
