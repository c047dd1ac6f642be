"""Layer-local parity harness (test infrastructure; used by
tests/test_gpu_layerwise.py, tests/test_gpu_resnet.py and
__graft_entry__.smoke()): runs ONE real out-of-core step through the C-ABI
executor with its inspection hook (oc_exec_set_hook / oc_exec_read_var),
captures on the GPU the bytes of every input of each function right before
its kernels and of every output right after them, applies the function's
definition (oracle/layerwise.py) to the captured inputs and compares every
output element by element (relative L2; u8 argmax entries: fraction that
differ).  See tests/test_gpu_layerwise.py for the tolerance rationale."""
import json

import numpy as np
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


def run_layerwise(spec, budget_frac=0.25, pin_below=MiB, mode="va", window=0, chunk=2 * MiB, doc_transform=None,
                  tol=TOL):
    """One out-of-core step with every function checked; returns counts, the
    worst error per (op kind, role) and the failures above `tol`."""
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    doc, info = graphs.build(spec, params="persistent", inputs="host", pin_below=pin_below)
    if doc_transform:
        doc = doc_transform(doc)
    meta = info["meta"]
    G = B.Graph(doc)
    budget = max(G.min_feasible_budget(window), int(G.in_core_peak() * budget_frac))
    m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST}[mode]
    probe = G.plan(budget, window, m, chunk_bytes=chunk, phys_bytes=1 << 40, allow_oom=True).stats()
    st = OutOfCoreStep(doc, budget, window, mode=mode, chunk_bytes=chunk,
                       phys_bytes=probe["peak_phys"] + chunk if mode == "va" else probe["peak_phys"])
    assert st.stats["bytes_d2h"] > 0, "the budget must force swap-outs"
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], x.astype(np.float32) if spec["mode"] == "fp32"
             else torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy())
    if spec["loss"]["type"] == "l1":   # the target image, stored in the act dtype
        y = y.astype(np.float32) if spec["mode"] == "fp32" else \
            torch.from_numpy(np.ascontiguousarray(y, np.float32)).to(torch.bfloat16).view(torch.int16).numpy()
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
                    if not err <= tol:
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
