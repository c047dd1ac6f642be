"""Pins of oracle/layerwise.py (per-function definitions of the conv-net graph)
against oracle/numerics.py's whole training step, which is itself pinned by
central finite differences and library routines (test_oracle_numerics.py):
executing the graph document function by function with the layer-local
definitions (layerwise.run_graph) must reproduce numerics.train_step's loss,
every parameter gradient and every updated parameter.

The two are independent formulations: numerics interprets the network's
layer list (forward, then reverse-order backward with the accumulation rules
of its own), layerwise follows the graph document's functions (fused
BN-ReLU-maxpool stem, BN statistics from the conv, in-place BN backward with
the ReLU mask recomputed from y, the gradient accumulation order the graph
builder chose).  They differ only where the GPU contract stores a value in
fp32 that numerics keeps in fp64 (BN statistics, dgamma/dbeta read back by
the BN apply): in fp32 mode that is ~1e-7 relative, so the chain must agree
to 1e-6; in bf16 mode such differences can flip a bf16 rounding, so the
chain must agree to 1e-3 on the shallow nets and bitwise on the loss path
(the forward values feeding the loss are rounded the same way)."""
import numpy as np
import pytest

from oracle import layerwise, numerics as nm
from paper_2010_14109_b200 import graphs
from synth import nets


def _chain(spec):
    doc, info = graphs.build(spec, params="pinned")
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    rnd = nm.rounder(spec["mode"])
    lab = rnd(np.asarray(y, np.float64)) if spec["loss"]["type"] == "l1" else np.asarray(y, np.int64)
    vals = {info["x"]: rnd(np.asarray(x, np.float64)), info["labels"]: lab}
    for k, v in p.items():
        vals[info["params"][k]] = np.asarray(v, np.float64)
        vals[info["momentum"][k]] = np.zeros(np.asarray(v).shape)
    layerwise.run_graph(doc, vals)
    ref = nm.train_step(spec, p, x, y)
    return vals, info, ref, p


@pytest.mark.parametrize("spec,tol", [
    (nets.tiny_resnet(batch=4, image=16, classes=10, mode="fp32"), 1e-6),
    (nets.resnet(18, batch=8, image=64, classes=10, mode="fp32"), 1e-5),
    (nets.tiny_resnet(batch=4, image=16, classes=10, mode="bf16"), 1e-3),
    # F3 families (the paper's Fig.4/5 networks): atrous convs, ASPP, bilinear
    # decoder; reflection padding, instance norm, transposed convs, tanh, L1
    (nets.deeplabv3plus(batch=4, image=33, classes=3, width=8, rates=(2, 3, 4), aspp=8, low=8,
                        blocks=(1, 1, 1, 1), mode="fp32"), 1e-5),
    (nets.pix2pixhd(batch=2, image=(16, 32), ngf=8, n_down=2, n_blocks=1, mode="fp32"), 1e-5),
    (nets.pix2pixhd(batch=2, image=(16, 32), ngf=8, n_down=2, n_blocks=1, mode="bf16"), 1e-3),
])
def test_graph_chain_equals_train_step(spec, tol):
    vals, info, ref, p = _chain(spec)
    assert abs(vals[info["loss"]][0] - ref["loss"]) <= 1e-6 * abs(ref["loss"])
    worst = 0.0
    for k in p:
        g = vals[info["grads"][k]].reshape(p[k].shape)
        e = nm.rel_l2(g, ref["grads"][k])
        worst = max(worst, e)
        assert e <= tol, (k, e)
        assert nm.rel_l2(vals[info["params"][k]].reshape(p[k].shape), ref["params"][k]) <= tol
    print(f"worst gradient rel-L2 chain vs train_step: {worst:.2e}")


def test_every_conv_graph_op_kind_has_a_definition():
    import json
    for spec in (nets.resnet(18, batch=2, image=32), nets.resnet(50, batch=2, image=32), nets.tiny_resnet(),
                 nets.deeplabv3plus(batch=2, image=65), nets.pix2pixhd(batch=1, image=(32, 64), ngf=8)):
        doc, _ = graphs.build(spec, params="pinned")
        kinds = {f["op"]["kind"] for f in json.loads(doc)["functions"]}
        assert kinds <= set(layerwise.OPS), kinds - set(layerwise.OPS)
