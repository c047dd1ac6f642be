"""BigGAN-style GAN step (configs[4]) through the C-ABI:
parity with the oracle's gan_step on a 16² GAN that has every layer kind
(BN-ReLU, nearest upsampling, convs, residual adds, SAGAN attention, tanh,
ReLU, average pooling, GAP, linear score, hinge losses, D-step then G-step
through the updated D), and swap transparency (out-of-core == in-core,
bitwise) in bf16."""
import numpy as np
import pytest

from oracle import numerics as nm
from paper_2010_14109_b200 import binding as B
from paper_2010_14109_b200 import graphs
from synth import nets

MiB = 1 << 20


def _bits(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).view(torch.int16).numpy()


def run_gan(spec, budget_frac, mode="va"):
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    doc, info = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    F = G.in_core_peak()
    budget = max(G.min_feasible_budget(0), int(F * budget_frac))
    m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST}[mode]
    probe = G.plan(budget, B.OC_WINDOW_MAX_FEASIBLE, m, chunk_bytes=2 * MiB, phys_bytes=8 * budget + (1 << 30),
                   allow_oom=True)
    st = OutOfCoreStep(doc, budget, B.OC_WINDOW_MAX_FEASIBLE, mode=mode, chunk_bytes=2 * MiB,
                       phys_bytes=probe.stats()["peak_phys"] + 2 * MiB)
    pG, pD = nets.make_gan_params(spec)
    z1, z2, x = nets.make_gan_inputs(spec)
    f32 = spec["mode"] == "fp32"
    for name, arr in (("z1", z1), ("z2", z2), ("x_real", x)):
        st.write(info[name], arr if f32 else _bits(arr))
    for net, p in (("G", pG), ("D", pD)):
        for k, v in p.items():
            st.write(info[net]["params"][k], v)
            st.write(info[net]["momentum"][k], np.zeros_like(v))
    met = st.step()
    out = {"loss_d": float(st.read(info["loss_d"])[0]), "loss_g": float(st.read(info["loss_g"])[0]), "met": met}
    for net, p in (("G", pG), ("D", pD)):
        for k in p:
            out[net + ".m." + k] = st.read(info[net]["momentum"][k]).reshape(p[k].shape)
            out[net + ".p." + k] = st.read(info[net]["params"][k]).reshape(p[k].shape)
    st.close()
    return out, (pG, pD, z1, z2, x)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["va", "best"])
def test_tiny_gan_parity_fp32(mode):
    """fp32 mode under a 1/3 budget: both losses, every D and G parameter
    gradient (= the momentum after one step from zero) and the updated
    parameters within 1e-5 of the oracle."""
    spec = nets.tiny_biggan(batch=4, mode="fp32")
    out, (pG, pD, z1, z2, x) = run_gan(spec, 1 / 3, mode)
    assert out["met"]["bytes_d2h"] > 0
    ref = nm.gan_step(spec, pG, pD, z1, z2, x)
    assert abs(out["loss_d"] - ref["loss_d"]) <= 1e-5 * abs(ref["loss_d"])
    assert abs(out["loss_g"] - ref["loss_g"]) <= 1e-5 * max(1e-3, abs(ref["loss_g"]))
    errs = {}
    for net, grads, newp in (("D", ref["gradsD"], ref["pD"]), ("G", ref["gradsG"], ref["pG"])):
        for k in grads:
            errs[net + ".g." + k] = nm.rel_l2(out[net + ".m." + k], grads[k])
            errs[net + ".p." + k] = nm.rel_l2(out[net + ".p." + k], newp[k])
    worst = max(errs, key=errs.get)
    assert errs[worst] <= 1e-5, (worst, errs[worst])


@pytest.mark.gpu
def test_tiny_gan_bf16_transparency_and_loss():
    """bf16: out-of-core (1/3 budget, VA) == in-core bitwise; losses within
    1e-3 of the oracle."""
    spec = nets.tiny_biggan(batch=8, mode="bf16")
    ooc, (pG, pD, z1, z2, x) = run_gan(spec, 1 / 3, "va")
    inc, _ = run_gan(spec, 1.0, "va")
    assert ooc["met"]["bytes_d2h"] > 0
    for k in ooc:
        if k.startswith(("G.", "D.")):
            assert np.array_equal(ooc[k], inc[k]), k
    ref = nm.gan_step(spec, pG, pD, z1, z2, x)
    assert abs(ooc["loss_d"] - ref["loss_d"]) <= 1e-3 * abs(ref["loss_d"])
