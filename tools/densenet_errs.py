import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_resnet import run_step
from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B, graphs
from synth import nets
spec = nets.tiny_densenet(batch=4, image=16, classes=10, mode="fp32")
doc, info = graphs.build(spec, params="persistent")
G = B.Graph(doc)
x, y = nets.make_inputs(spec); p = nets.make_params(spec)
ref = nm.train_step(spec, p, x, y)
for frac in (1.0, 0.34):
    budget = max(G.min_feasible_budget(0), int(G.in_core_peak() * frac))
    out = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE if frac < 1 else 0, "va", None, fp32_input=True)
    print("frac", frac, "loss", out["loss"], ref["loss"])
    for k in p:
        print(" ", k, "%.2e" % nm.rel_l2(out["m." + k], ref["grads"][k]))
