"""One out-of-core step of a small config, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool racecheck python tools/sanitize_step.py mlp|tiny_resnet|r18_64
Swaps forced by the budget; VA pool (2 MiB chunks) or best-fit arena."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(which, mode="va"):
    import torch
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    from synth import nets
    spec = {"mlp": lambda: nets.mlp6(), "tiny_resnet": lambda: nets.tiny_resnet(batch=4, image=16, classes=10),
            "r18_64": lambda: nets.resnet(18, batch=4, image=64, classes=10)}[which]()
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    budget = 4 << 20 if which == "mlp" else max(G.min_feasible_budget(0), G.in_core_peak() // 4)
    m = B.OC_ALLOC_VA if mode == "va" else B.OC_ALLOC_ARENA_BEST
    probe = G.plan(budget, B.OC_WINDOW_MAX_FEASIBLE, m, chunk_bytes=2 << 20, phys_bytes=1 << 40,
                   allow_oom=True).stats()
    st = OutOfCoreStep(doc, budget, B.OC_WINDOW_MAX_FEASIBLE, mode=mode, chunk_bytes=2 << 20,
                       phys_bytes=probe["peak_phys"] + (2 << 20))
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], x.astype(np.float32) if spec["mode"] == "fp32"
             else torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy())
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    met = st.step()
    met2 = st.step()
    print(which, mode, "loss", float(st.read(info["loss"])[0]), "h2d", met2["bytes_h2d"], "d2h", met2["bytes_d2h"],
          "kernels", met2["n_kernels"])
    st.close()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "va")
