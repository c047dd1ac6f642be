import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_resnet import run_step
from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B, graphs
from synth import nets
spec = nets.tiny_resnet(batch=4, image=16, classes=10)
doc, info = graphs.build(spec, params="persistent")
G = B.Graph(doc); peak = G.in_core_peak()
budget = max(G.min_feasible_budget(0), int(peak * 0.5))
x, y = nets.make_inputs(spec); p = nets.make_params(spec)
ref = nm.train_step(spec, p, x, y)
out = run_step(spec, doc, info, budget, B.OC_WINDOW_MAX_FEASIBLE, "va", 256 << 20)
for k in p:
    print(k, nm.rel_l2(out["m." + k], ref["grads"][k]))
