"""Benchmark of the out-of-core training step (BASELINE.json metric:
"samples/sec at k× in-budget batch vs in-core; host-link GB/s; overlap %").

Default workload (N=1): configs[2] — ResNet-50, 224×224 synthetic images,
per GPU a fixed PHYSICAL device budget B_p = 8 GiB ("else
B = 8 GiB"; the paper's fixed 16 GB V100) that holds everything the
step puts on the device: pinned variables + the VA swap pool + the
executor's compute workspace.  b0 = the largest batch whose in-core step
(footprint F_peak + workspace) fits B_p; the step runs at the paper's
1440-equivalent batch round(1440/190 · b0) (7.5× over the
in-core maximum).  The scheduler budget B_s is the largest one whose
allocator replay fits the pool B_p − pinned − workspace (Fig.3's "maximum
defined memory budget"), window 0 (the measured best on this
link-bound step), VA allocator with 2 MiB chunks.  One step = forward +
backward + update of the whole network through the C-ABI (oc_run_step),
inputs and parameters swapped in from pinned host memory as part of the
schedule.  Retention = samples/s ÷ in-core samples/s at b0 (the paper's
55 % = 321/581).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config r50|r18|mlp|unet|r1001|biggan|densenet] [--mode va|best|first]

--config r18: configs[1] (ResNet-18 b=256, B_p = 25 % of the in-core footprint).
Multi-GPU: one process per GPU (torchrun; `--gpus N` spawns it when
WORLD_SIZE is unset), each replica with its own budget, pool and host link
(weak scaling); gradients averaged with NCCL inside the step.  Rank 0 prints
ONE JSON line.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MiB = 1 << 20
GiB = 1 << 30
PCIE5_X16_GBS = 63.0          # 32 GT/s × 16 × 128/130 / 8, per direction
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # derived peak for FFMA kernels
PAPER_MULTIPLE = 1440 / 190   # batch 1440 = 7.5× the in-core maximum 190


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="r50",
                    choices=["r50", "r18", "r1001", "mlp", "biggan", "unet", "densenet", "deeplab", "pix2pix"])
    ap.add_argument("--mode", default="va", choices=["va", "best", "first"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--phys-gib", type=float, default=8.0, help="r50: physical device budget per GPU (GiB)")
    ap.add_argument("--multiple", type=float, default=PAPER_MULTIPLE, help="r50: batch = multiple × b0")
    ap.add_argument("--budget-frac", type=float, default=None,
                    help="other configs: physical budget as a fraction of the in-core footprint "
                         "(default 0.125 for configs[3] U-Net, else 0.25)")
    ap.add_argument("--chunk-mib", type=int, default=2)
    ap.add_argument("--bucket-mib", type=int, default=25,
                    help="N > 1: gradient allreduce bucket size (one ncclGroup on the comm stream per bucket)")
    ap.add_argument("--no-incore", action="store_true")
    ap.add_argument("--window", default=None,
                    help="auto (timed probes) | model (makespan model, F4) | max | <bytes>; default 0 for r50, "
                         "auto otherwise")
    ap.add_argument("--no-graph", action="store_true", help="issue every step eagerly (no CUDA graph replay)")
    ap.add_argument("--policy", default="paper", choices=["paper", "vdnn", "lms"],
                    help="swap-timing window: the paper's byte window, or the prior-art function-distance "
                         "window (vdnn = 1 function ahead, lms = --distance functions ahead; SURVEY F1)")
    ap.add_argument("--distance", type=int, default=3, help="lms policy: functions of look-ahead")
    ap.add_argument("--trigger", default="release", choices=["release", "paper"],
                    help="arrival trigger: at the release of the reused memory (executor default) or at the "
                         "end of f_{i-1} as the paper's Fig.2 (P:91)")
    a = ap.parse_args()
    if a.budget_frac is None:
        a.budget_frac = 0.125 if a.config == "unet" else 0.25
    if a.window is None:
        a.window = "0" if a.config == "r50" else "auto"
    return a


# ----------------------------------------------------------------- workloads
def spec_for(args, batch=None):
    from synth import nets
    c = args.config
    if c == "mlp":
        return nets.mlp6()
    if c == "r50":
        return nets.resnet(50, batch=batch or args.batch or 256)
    if c == "densenet":      # the paper's second family (Fig.4/5), DenseNet-121 224²
        return nets.densenet(batch=batch or args.batch or 128)
    if c == "unet":          # configs[3]: U-Net 1024² b=8
        return nets.unet(batch=batch or args.batch or 8, image=1024)
    if c == "biggan":
        return nets.biggan(batch=batch or args.batch or 32)
    if c == "r1001":
        return nets.preact_resnet(1001, batch=batch or args.batch or 256)
    if c == "deeplab":       # DeepLabv3+ on PASCAL-VOC-sized 513² images
        return nets.deeplabv3plus(batch=batch or args.batch or 16)
    if c == "pix2pix":       # Pix2PixHD global generator on Cityscapes-sized 512×1024
        return nets.pix2pixhd(batch=batch or args.batch or 4)
    return nets.resnet(18, batch=batch or args.batch or 256)


def pin_below_for(args):
    # tensors under one threshold (BN parameters, small weights, their optimizer
    # state) stay resident (Z26); R50 keeps the paper-literal
    # all-swappable graph (Table 1)
    return {"r18": MiB, "r1001": args.chunk_mib * MiB}.get(args.config, 0)


def workload_name(args, spec, B_p, b0):
    c = args.config
    if c == "r50":
        return (f"configs[2] ResNet-50 224x224 b={spec['batch']} = {spec['batch'] / b0:.2f} x b0 (b0 = {b0}, the "
                f"in-core maximum under B_p = {B_p / GiB:.2f} GiB physical per GPU)")
    if c == "r18":
        return (f"configs[1] ResNet-18 224x224 b={spec['batch']}, physical budget {args.budget_frac:.2f} x in-core "
                "footprint, tensors < 1 MiB pinned")
    if c == "mlp":
        return "configs[0] 6-layer MLP fp32 b=8, 4 MiB scheduler budget"
    if c == "unet":
        return (f"configs[3] U-Net 1024x1024 base 64 depth 4, 19 classes, b={spec['batch']} at "
                f"{args.budget_frac:.3f} of the in-core footprint")
    if c == "biggan":
        return (f"configs[4] BigGAN-style 128x128 ch=96 GAN step (D-step + G-step) b={spec['batch']} at "
                f"{args.budget_frac:.2f} of the in-core footprint")
    if c == "r1001":
        return (f"configs[4] pre-activation ResNet-1001 32x32 b={spec['batch']} at {args.budget_frac:.2f} of the "
                "in-core footprint, tensors < 1 VA chunk pinned")
    if c == "deeplab":
        return (f"F3 DeepLabv3+ (ResNet-50, output stride 16) 513x513 b={spec['batch']} at {args.budget_frac:.2f} "
                "of the in-core footprint")
    if c == "pix2pix":
        return (f"F3 Pix2PixHD global generator 512x1024 b={spec['batch']} (L1 loss) at {args.budget_frac:.2f} of "
                "the in-core footprint")
    return f"F3 DenseNet-121 224x224 b={spec['batch']} at {args.budget_frac:.2f} of the in-core footprint"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev):
        self.dev = dev
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


class PcieSampler:
    """Counter-backed host-link throughput during the timed region: NVML's PCIe
    throughput counters (nvmlDeviceGetPcieThroughput, KB/s over 20 ms windows;
    TX = device -> host, RX = host -> device), sampled every 25 ms on a thread —
    an independent check of the CUDA-event-derived host-link GB/s."""

    def __init__(self, dev):
        self.dev = dev
        self.tx, self.rx = [], []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.info = {}

    def run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.info = {"link_gen": pynvml.nvmlDeviceGetCurrPcieLinkGeneration(h),
                         "link_width": pynvml.nvmlDeviceGetCurrPcieLinkWidth(h)}
            while not self.stop.is_set():
                self.tx.append(pynvml.nvmlDeviceGetPcieThroughput(h, pynvml.NVML_PCIE_UTIL_TX_BYTES))
                self.rx.append(pynvml.nvmlDeviceGetPcieThroughput(h, pynvml.NVML_PCIE_UTIL_RX_BYTES))
                self.stop.wait(0.025)
        except Exception as e:  # noqa: BLE001
            self.info["error"] = str(e)[:120]

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=5)

    def summary(self):
        if not self.tx:
            return dict(self.info, samples=0)
        kb = 1e3 / 1e9   # KB/s -> GB/s
        return dict(self.info, samples=len(self.tx), d2h_gbs_mean=float(np.mean(self.tx)) * kb,
                    h2d_gbs_mean=float(np.mean(self.rx)) * kb, d2h_gbs_p90=float(np.percentile(self.tx, 90)) * kb,
                    h2d_gbs_p90=float(np.percentile(self.rx, 90)) * kb,
                    source="NVML nvmlDeviceGetPcieThroughput (20 ms windows) during the timed steps")


# ----------------------------------------------------------- memory budgets
def in_core_device_bytes(spec):
    """Device bytes of the IN-CORE step: F_peak with parameters, gradients and
    momentum resident, plus the executor workspace."""
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    doc, _ = graphs.build(spec, params="pinned")
    G = B.Graph(doc)
    return G.in_core_peak() + G.workspace_bytes()


def trainable_batch(spec_fn, phys, lo=1, hi=8192):
    """b0: the largest batch whose in-core step fits `phys` device bytes
    (bisection) — the denominator of the trainable-batch multiple."""
    if in_core_device_bytes(spec_fn(lo)) > phys:
        return 0
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if in_core_device_bytes(spec_fn(mid)) <= phys:
            lo = mid
        else:
            hi = mid - 1
    return lo


def fit_budget(G, pool, mode, chunk, W=0, distance=0):
    """Largest scheduler budget B_s whose allocator replay fits a swap pool of
    `pool` physical bytes (Fig.3 'maximum defined memory budget'); None if
    even the minimum feasible budget does not fit."""
    from paper_2010_14109_b200 import binding as B
    m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST, "first": B.OC_ALLOC_ARENA_FIRST}[mode]
    lo = G.min_feasible_budget(W, distance=distance) if distance else G.min_feasible_budget(W)

    def fits(b):
        return G.plan(b, W, m, chunk_bytes=chunk, phys_bytes=pool, allow_oom=True,
                      distance=distance).stats()["oom_fn"] < 0
    if not fits(lo):
        return None
    pinned = G.plan(lo, W, m, chunk_bytes=chunk, phys_bytes=pool, allow_oom=True, distance=distance).stats()[
        "pinned_bytes"]
    hi = pinned + pool + 1
    if fits(hi):
        return hi
    while hi - lo > MiB:
        mid = (lo + hi) // 2
        if fits(mid):
            lo = mid
        else:
            hi = mid
    return lo


def host_ram_bytes():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def host_copy_bytes(doc, sched_json):
    """Pinned host bytes the executor allocates: persistent swappable
    variables and every variable the schedule ever swaps out."""
    d = json.loads(doc)
    s = json.loads(sched_json)
    need = {i for i, v in enumerate(d["variables"]) if v.get("persistent") and not v.get("pinned")}
    for f in s["fn"]:
        need.update(f["reserve_out"])
    return sum((d["variables"][i]["bytes"] + 255) // 256 * 256 for i in need)


def link_probe(nbytes=256 * MiB):
    """Pinned host <-> device copy bandwidth on this box, per direction and
    duplex (GB/s, CUDA events): the link roofline's denominators."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s1):
                e0.record()
                fn()
                e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = nbytes / (best / 1e3) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    out["duplex"] = 2 * nbytes / (time.perf_counter() - t0) / 1e9
    return out


# ----------------------------------------------------------------- setup
def new_step(spec, info, doc, budget, mode, chunk, phys, window, timeline=False, pack=64 << 10, use_graph=False,
             distance=0, trigger=0):
    import torch
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    from synth import nets
    st = OutOfCoreStep(doc, budget, window, mode=mode, chunk_bytes=chunk, phys_bytes=phys, timeline=timeline,
                       pack_threshold=pack, use_graph=use_graph, distance=distance, trigger=trigger)
    if "G" in spec:          # GAN step: noise, real images, G and D parameters
        pG, pD = nets.make_gan_params(spec)
        z1, z2, xr = nets.make_gan_inputs(spec)
        for name, arr in (("z1", z1), ("z2", z2), ("x_real", xr)):
            st.write(info[name], torch.from_numpy(arr).to(torch.bfloat16).view(torch.int16).numpy()
                     if spec["mode"] == "bf16" else arr)
        for net, pp in (("G", pG), ("D", pD)):
            for k, v in pp.items():
                st.write(info[net]["params"][k], v)
                st.write(info[net]["momentum"][k], np.zeros_like(v))
        return st
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    st.write(info["x"], torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy()
             if spec["mode"] == "bf16" else x)
    if spec["loss"]["type"] == "l1" and spec["mode"] == "bf16":   # the L1 target image, act dtype
        y = torch.from_numpy(y).to(torch.bfloat16).view(torch.int16).numpy()
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    return st


def setup_step(spec, info, doc, budget, mode, chunk, timeline=True, window=None, pack=64 << 10, use_graph=False,
               distance=0, trigger=0):
    """Scheduler budget -> executor with the pool sized to the replay's
    physical peak (tools: sweeps that fix B_s rather than B_p)."""
    from paper_2010_14109_b200 import binding as B
    G = B.Graph(doc)
    W = window if window is not None else G.max_feasible_window(budget)
    probe = G.plan(budget, W, B.OC_ALLOC_VA if mode == "va" else B.OC_ALLOC_ARENA_BEST, chunk_bytes=chunk,
                   phys_bytes=budget * 4, allow_oom=True, distance=distance)
    ps = probe.stats()
    phys = ps["peak_phys"] + chunk if mode == "va" else max(ps["peak_phys"], 1)
    st = new_step(spec, info, doc, budget, mode, chunk, phys, W, timeline, pack, use_graph, distance, trigger)
    return st, W, phys


def conv_flops(doc):
    """Algorithmic FLOPs per function (2·MACs) for the tensor-contraction ops."""
    d = json.loads(doc)
    fl = {}
    for f in d["functions"]:
        op = f.get("op") or {}
        a = op.get("attrs", {})
        k = op.get("kind")
        if k in ("conv_fwd", "conv_dgrad", "conv_wgrad"):
            fl[f["id"]] = (k, 2.0 * a["N"] * a["P"] * a["Q"] * a["K"] * a["R"] * a["S"] * a["C"])
        elif k in ("linear_fwd", "linear_bwd"):
            fl[f["id"]] = (k, 2.0 * a["M"] * a["N"] * a["K"] * (1 if k == "linear_fwd" else 2))
        elif k in ("attn_fwd", "attn_bwd"):
            nb, L = a.get("nb", a["N"]), a["L"]
            per = (a["dq"] + a["dv"]) if k == "attn_fwd" else (2 * a["dv"] + 2 * a["dq"])
            fl[f["id"]] = (k, 2.0 * nb * L * L * per)
    return fl


def _union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def compute_under_transfer(tl):
    """|T ∩ C| / |C| of one instrumented step's timeline: the share of the
    compute time that runs while a transfer is in flight (the executor's
    overlap_frac is the other ratio, |T ∩ C| / |T|)."""
    C = _union([(e["t0"], e["t1"]) for e in tl if e["stream"] == "compute"])
    T = _union([(e["t0"], e["t1"]) for e in tl if e["stream"] in ("h2d", "d2h")])
    inter, j = 0.0, 0
    for a, b in C:
        while j < len(T) and T[j][1] <= a:
            j += 1
        k = j
        while k < len(T) and T[k][0] < b:
            inter += max(0.0, min(b, T[k][1]) - max(a, T[k][0]))
            k += 1
    c = sum(b - a for a, b in C)
    return inter / c if c > 0 else None


def conv_bytes(doc):
    """Algorithmic HBM bytes per convolution function: one read of each
    operand and one write of the result (bf16 activations and weights, fp32
    weight gradient), plus one read of the result when the epilogue
    accumulates into it."""
    d = json.loads(doc)
    out = {}
    for f in d["functions"]:
        op = f.get("op") or {}
        a = op.get("attrs", {})
        k = op.get("kind")
        if k not in ("conv_fwd", "conv_dgrad", "conv_wgrad"):
            continue
        e = 2 if a.get("dtype", "bf16") == "bf16" else 4
        x = a["N"] * a["H"] * a["W"] * a["C"] * e
        y = a["N"] * a["P"] * a["Q"] * a["K"] * e
        w = a["K"] * a["R"] * a["S"] * a["C"]
        acc = 1 if a.get("accumulate") else 0
        if k == "conv_fwd":
            out[f["id"]] = x + w * e + y * (1 + acc)
        elif k == "conv_dgrad":
            out[f["id"]] = y + w * e + x * (1 + acc)
        else:
            out[f["id"]] = y + x + w * 4
    return out


def attn_bytes(doc):
    """Algorithmic HBM bytes per attention function (bf16 tensor-core path,
    DESIGN.md §7): forward P written and read (bf16; the scores are recomputed,
    never stored, when dq ≤ 64) = 4·L² per sample, else S written and read
    (fp32) too = 12·L²; backward P read twice, dS written once and read twice =
    16·L² per sample (the L-wide q, k, v, o tensors are < 2 % and left out)."""
    d = json.loads(doc)
    out = {}
    for f in d["functions"]:
        op = f.get("op") or {}
        a = op.get("attrs", {})
        if op.get("kind") in ("attn_fwd", "attn_bwd"):
            nb, L = a.get("nb", a["N"]), a["L"]
            per = (4 if a["dq"] <= 64 else 12) if op["kind"] == "attn_fwd" else 16
            out[f["id"]] = per * nb * L * L
    return out


def copy_rates(tl, vbytes):
    """Per-copy host-link rates of the instrumented pass: bytes-weighted
    quantiles of bytes / duration per direction, and the share of each
    direction's busy time during which the other direction was also copying
    (a duplex PCIe link shares its bandwidth: ~50 GB/s each way when both run)."""
    out = {}
    iv = {"h2d": [], "d2h": []}
    for ev in tl:
        if ev["stream"] in iv and ev["t1"] > ev["t0"]:
            iv[ev["stream"]].append((ev["t0"], ev["t1"], vbytes.get(ev["id"], 0)))
    for d, lst in iv.items():
        if not lst:
            continue
        rates = sorted(((b / ((t1 - t0) * 1e-3) / 1e9, b) for t0, t1, b in lst), key=lambda x: x[0])
        tot = sum(b for _, b in rates)
        q, acc = {}, 0
        for r, b in rates:
            acc += b
            for k in (0.1, 0.5, 0.9):
                if f"p{int(k * 100)}" not in q and acc >= k * tot:
                    q[f"p{int(k * 100)}"] = round(r, 2)
        other = sorted((t0, t1) for t0, t1, _ in iv["d2h" if d == "h2d" else "h2d"])
        both = 0.0
        for t0, t1, _ in lst:
            for o0, o1 in other:
                if o0 >= t1:
                    break
                both += max(0.0, min(t1, o1) - max(t0, o0))
        busy = sum(t1 - t0 for t0, t1, _ in lst)
        out[d] = {"copies": len(lst), "gbs_bytes_weighted": q, "gbs_sum_of_copies": round(tot / (busy * 1e-3) / 1e9, 2),
                  "share_with_other_direction": round(both / busy, 3) if busy else None}
    return out


def time_steps(st, steps, warmup, world):
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        st.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(st.streams[0])
    mets = [st.step() for _ in range(steps)]
    e1.record(st.streams[0])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    return e0.elapsed_time(e1), (t1 - t0) * 1e3, mets


def max_over_ranks(vals, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64)
    if world > 1:
        t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t = t.cpu()
    return [float(x) for x in t]


def attach(st, rank, world):
    import torch.distributed as dist
    from paper_2010_14109_b200.runtime import nccl_unique_id
    if world <= 1:
        return
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    st.attach_nccl(uid[0], rank, world)


def in_core_rate(args, spec, rank, world, chunk, steps):
    """In-core step at this spec's batch: no swapping at all — parameters,
    gradients and momentum device-resident, budget = F_peak, W = 0, best-fit
    arena; NCCL attached for N > 1 (same exchange as the out-of-core step);
    samples/s over all ranks from the max-over-ranks device time."""
    import torch
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    torch.cuda.empty_cache()
    doc_p, info_p = graphs.build(spec, params="pinned", inputs="host")
    G_p = B.Graph(doc_p)
    F_p = G_p.in_core_peak()
    # the best-fit arena's carved peak (fragmentation included) sizes the slab
    slab = G_p.plan(F_p, 0, B.OC_ALLOC_ARENA_BEST, chunk_bytes=chunk, phys_bytes=1 << 50,
                    allow_oom=True).stats()["peak_phys"]
    st2 = new_step(spec, info_p, doc_p, F_p, "best", chunk, slab, 0, use_graph=not args.no_graph)
    attach(st2, rank, world)
    ms, _, _ = time_steps(st2, max(3, steps // 2), max(1, args.warmup), world)
    st2.close()
    ms = max_over_ranks([ms], world)[0]
    return spec["batch"] * world * max(3, steps // 2) / (ms / 1e3)


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from synth import nets

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    chunk = args.chunk_mib * MiB
    dist_ = {"paper": 0, "vdnn": 1, "lms": args.distance}[args.policy]
    trigger = 1 if args.trigger == "paper" else 0
    mode = args.mode
    ram = host_ram_bytes()
    if world > 1:   # one decision for every replica (they must plan identical schedules)
        r = [ram]
        dist.broadcast_object_list(r, src=0)
        ram = r[0]
    notes = []

    # ---- physical budget, batch, scheduler budget
    b0 = None
    if args.config == "mlp":
        spec = spec_for(args)
        doc, info = graphs.build(spec, params="persistent", inputs="host")
        G = B.Graph(doc)
        F_peak, ws = G.in_core_peak(), G.workspace_bytes()
        W0 = 0
        B_s = 4 * MiB   # configs[0]: the scheduler budget itself (all variables swappable)
        probe = G.plan(B_s, B.OC_WINDOW_MAX_FEASIBLE, B.OC_ALLOC_ARENA_BEST if mode != "va" else B.OC_ALLOC_VA,
                       chunk_bytes=chunk, phys_bytes=B_s * 64, allow_oom=True).stats()
        pinned = probe["pinned_bytes"]
        pool = probe["peak_phys"] + (chunk if mode == "va" else 0)
        B_p = pinned + pool + ws
    else:
        B_p = None
        for attempt in range(6):
            if args.config == "r50":
                B_p = B_p or int(args.phys_gib * GiB)
                b0 = trainable_batch(lambda b: spec_for(args, b), B_p)
                spec = spec_for(args, args.batch or max(1, int(round(args.multiple * b0))))
            else:
                spec = spec_for(args)
            doc, info = graphs.build(spec, params="persistent", inputs="host", pin_below=pin_below_for(args),
                                     dp_bucket_bytes=(args.bucket_mib * MiB if world > 1 and "G" not in spec else 0))
            G = B.Graph(doc)
            F_peak, ws = G.in_core_peak(), G.workspace_bytes()
            if args.config != "r50":
                B_p = B_p or int(args.budget_frac * (F_peak + ws))
                b0 = trainable_batch(lambda b: spec_for(args, b), B_p) if "G" not in spec else None
            probe = G.plan(G.min_feasible_budget(0), 0, B.OC_ALLOC_VA, chunk_bytes=chunk, phys_bytes=1 << 50,
                           allow_oom=True).stats()
            pinned = probe["pinned_bytes"]
            pool = B_p - pinned - ws
            pool = pool // chunk * chunk if mode == "va" else pool
            if pool <= 0:
                raise RuntimeError(f"physical budget {B_p} B cannot hold pinned {pinned} + workspace {ws}")
            if args.config != "r50" and fit_budget(G, pool, mode, chunk, 0) is None:
                # the fraction is below what any schedule can run in once the pinned
                # bytes, the workspace and the allocator's granularity are counted:
                # raise B_p to the smallest physical budget that runs, and say so
                lo, hi = B_p, int(F_peak + ws)
                while hi - lo > MiB:
                    mid = (lo + hi) // 2
                    pm = (mid - pinned - ws) // chunk * chunk if mode == "va" else mid - pinned - ws
                    if pm > 0 and fit_budget(G, pm, mode, chunk, 0) is not None:
                        hi = mid
                    else:
                        lo = mid
                notes.append(f"{args.budget_frac:.3f} x footprint = {B_p} B cannot hold the minimum feasible "
                             f"schedule + pinned + workspace; B_p raised to {hi} B = "
                             f"{hi / (F_peak + ws):.3f} x footprint")
                B_p = hi
                pool = (B_p - pinned - ws) // chunk * chunk if mode == "va" else B_p - pinned - ws
            host_est = sum(v["bytes"] for v in json.loads(doc)["variables"] if not v.get("pinned"))
            if world > 1 and ram and world * host_est > 0.8 * ram and args.config == "r50" and not args.batch:
                # N replicas share the host's RAM — shrink the per-GPU budget until they fit
                B_p = int(B_p * 0.8 * ram / (world * host_est) * 0.95)
                notes.append(f"B_p scaled to {B_p / GiB:.2f} GiB so that {world} x host copies fit host RAM")
                continue
            break
        W0 = 0
    # schedule-window: the paper's single hyperparameter, "decided experimentally"
    window_probe = []
    if args.config == "mlp":
        B_s_of = {}
        W_sel = int(args.window) if args.window.isdigit() else G.max_feasible_window(B_s)
    else:
        B_s0 = fit_budget(G, pool, mode, chunk, 0, dist_)
        if B_s0 is None:
            raise RuntimeError(f"no scheduler budget fits the {pool} B pool (min feasible "
                               f"{G.min_feasible_budget(0)} B)")
        wmax = G.max_feasible_window(B_s0)
        if dist_:
            W_sel = 0
        elif args.window == "auto":
            best = None
            for wf in (0.0, 0.25, 0.5, 1.0):
                Wc = int(wmax * wf)
                Bc = fit_budget(G, pool, mode, chunk, Wc)
                if Bc is None:
                    continue
                stc = new_step(spec, info, doc, Bc, mode, chunk, pool, Wc)
                stc.step()
                ms = float(np.mean([stc.step()["step_ms"] for _ in range(2)]))
                stc.close()
                window_probe.append({"window": Wc, "budget": Bc, "ms": ms})
                if best is None or ms < best[1]:
                    best = (Wc, ms)
            W_sel = best[0]
        elif args.window == "max":
            W_sel = wmax
        else:
            W_sel = int(args.window)
        B_s = fit_budget(G, pool, mode, chunk, W_sel, dist_)
    if world > 1:   # every replica runs the identical schedule
        sel = [W_sel]
        dist.broadcast_object_list(sel, src=0)
        W_sel = sel[0]

    # one executor serves the timed pass (CUDA-graph replay, no per-event
    # timing) and the instrumented pass (timeline events, eager issue)
    st = new_step(spec, info, doc, B_s, mode, chunk, pool, W_sel, timeline=True, use_graph=not args.no_graph,
                  distance=dist_, trigger=trigger)
    host_bytes = host_copy_bytes(doc, st.sched.json())
    host_pool_bytes, host_numa = st.host_info()
    if world > 1:
        import hashlib
        hs = [None] * world
        dist.all_gather_object(hs, hashlib.sha256(st.sched.json().encode()).hexdigest())
        if len(set(hs)) != 1:
            raise RuntimeError(f"ranks planned different schedules: {hs}")
    attach(st, rank, world)
    st.set_timeline(False)
    with Clocks(dev) as clk, PcieSampler(dev) as pcie:
        dev_ms, wall_ms, mets = time_steps(st, args.steps, args.warmup, world)
    loss = float(st.read(info["loss_g" if "G" in spec else "loss"])[0])
    ss = st.stats
    mstat = st.mem_stats()
    n_k = int(sum(m["n_kernels"] for m in mets))
    h2d = float(np.mean([m["bytes_h2d"] for m in mets]))
    d2h = float(np.mean([m["bytes_d2h"] for m in mets]))
    # instrumented pass: same executor, CUDA events around every function and transfer
    st.set_timeline(True)
    st.step()
    mets_i, tls = [], []
    for _ in range(3):
        mets_i.append(st.step())
        tls.append(st.timeline())
    # the step whose summed contraction spans are the median of the three: one
    # step's timeline, consistent as a whole, robust to a one-off stall
    spans = [sum((e.get("k_span_ms") or 0.0) for e in t if e["stream"] == "compute") for t in tls]
    tl = tls[sorted(range(3), key=lambda i: spans[i])[1]]
    st.close()
    fid = [f["id"] for f in json.loads(doc)["functions"]]
    vbytes = {v["id"]: v["bytes"] for v in json.loads(doc)["variables"]}
    dur = {}
    for ev in tl:
        if ev["stream"] == "compute":
            dur[ev["id"]] = dur.get(ev["id"], 0.0) + (ev["t1"] - ev["t0"])
    fn_ms = [dur.get(f, 0.0) for f in fid]
    bw_h = float(np.mean([m["bytes_h2d"] / max(m["h2d_busy_ms"], 1e-9) for m in mets_i])) / 1e6
    bw_d = float(np.mean([m["bytes_d2h"] / max(m["d2h_busy_ms"], 1e-9) for m in mets_i])) / 1e6
    copy_diag = copy_rates(tl, vbytes)
    link = link_probe()
    bw_h = bw_h if bw_h > 1 else link["h2d"]
    bw_d = bw_d if bw_d > 1 else link["d2h"]
    sim = st.sched.simulate(fn_ms, bw_h, bw_d, 0.0, 0.0, True, model=1)
    sim0 = st.sched.simulate(fn_ms, bw_h, bw_d, 0.0, 0.0, True, model=0)
    dev_ms, wall_ms = max_over_ranks([dev_ms, wall_ms], world)
    B_glob = spec["batch"] * world
    value = B_glob * args.steps / (dev_ms / 1e3)
    e2e = B_glob * args.steps / (wall_ms / 1e3)
    step_ms = dev_ms / args.steps
    overlap = float(np.mean([m["overlap_frac"] for m in mets_i]))
    cut = compute_under_transfer(tl)
    h2d_busy = float(np.mean([m["h2d_busy_ms"] for m in mets_i]))
    d2h_busy = float(np.mean([m["d2h_busy_ms"] for m in mets_i]))
    comp_busy = float(np.mean([m["compute_busy_ms"] for m in mets_i]))
    instr_step_ms = float(np.mean([m["step_ms"] for m in mets_i]))
    # transfers by phase (forward = functions up to the loss): the practical
    # link bound of a step whose forward drives D2H and backward drives H2D
    loss_pos = max(i for i, f in enumerate(fid) if f.startswith(("loss", "d1.hinge", "d2.hinge")) or f == "loss")
    ph = {"h2d_fwd": 0, "h2d_bwd": 0, "d2h_fwd": 0, "d2h_bwd": 0}
    for ev in tl:
        if ev["stream"] in ("h2d", "d2h"):
            ph[f"{ev['stream']}_{'fwd' if ev['fn'] <= loss_pos else 'bwd'}"] += vbytes[ev["id"]]
    t_duplex = max(h2d / (link["h2d"] * 1e9), d2h / (link["d2h"] * 1e9))
    t_phase = max(ph["d2h_fwd"] / (link["d2h"] * 1e9), ph["h2d_fwd"] / (link["h2d"] * 1e9)) + \
        max(ph["h2d_bwd"] / (link["h2d"] * 1e9), ph["d2h_bwd"] / (link["d2h"] * 1e9))
    # dominant contraction kernel from the per-function CUDA events of the instrumented pass
    fl = conv_flops(doc)
    abytes = attn_bytes(doc)
    cbytes = conv_bytes(doc)
    per_kind = {}
    per_launch = {}   # kind -> [Σ max(FLOPs/tensor peak, bytes/HBM peak) s, Σ measured s, Σ HBM-bound s]
    per_shape = {}
    fattrs = {f["id"]: (f.get("op") or {}).get("attrs", {}) for f in json.loads(doc)["functions"]}
    pk_ = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    for ev in tl:
        if ev["stream"] != "compute" or ev["id"] not in fl:
            continue
        kind, f = fl[ev["id"]]
        if kind.startswith("attn") and spec["mode"] == "bf16":
            f = abytes[ev["id"]]   # HBM-bound on the tensor-core path: bytes, not FLOPs
        a = per_kind.setdefault(kind, [0.0, 0.0, 0, 0.0, []])
        a[0] += f
        if ev["id"] in cbytes and spec["mode"] == "bf16":
            t_tc_ = f / (pk_.get("bf16_tflops_sustained", 1395.5) * 1e12)
            t_hbm_ = cbytes[ev["id"]] / (pk_.get("hbm_gbs", 6549.8) * 1e9)
            pl = per_launch.setdefault(kind, [0.0, 0.0, 0.0, 0.0, 0])
            pl[3] += cbytes[ev["id"]]
            pl[4] += max(1, ev.get("k_n") or 1)
            pl[0] += max(t_tc_, t_hbm_)
            pl[1] += (ev.get("k_span_ms") or ev.get("k_ms") or (ev["t1"] - ev["t0"])) / 1e3
            pl[2] += t_hbm_ if t_hbm_ > t_tc_ else 0.0
            at_ = fattrs[ev["id"]]
            key_ = f'{at_["C"]}>{at_["K"]} {at_["R"]}x{at_["S"]}/{at_["stride"]} {at_["H"]}x{at_["W"]}' + \
                (" acc" if at_.get("accumulate") else "")
            sh = per_shape.setdefault(kind, {}).setdefault(key_, [0.0, 0.0, 0.0, 0.0, 0])
            sh[0] += (ev.get("k_span_ms") or ev.get("k_ms") or (ev["t1"] - ev["t0"])) / 1e3
            sh[1] += f
            sh[2] += cbytes[ev["id"]]
            sh[3] += max(t_tc_, t_hbm_)
            sh[4] += 1
        if ev.get("k_n"):
            # in-kernel span (%globaltimer, first CTA start to last CTA end) when probed, else the events
            a[1] += (ev.get("k_span_ms") or ev["k_ms"]) / 1e3
            a[2] += ev["k_n"]
            a[3] += ev["k_ms"] / 1e3
            if ev.get("k_mhz"):
                a[4].append(ev["k_mhz"])
        else:
            a[1] += (ev["t1"] - ev["t0"]) / 1e3
            a[2] += 1
            a[3] += (ev["t1"] - ev["t0"]) / 1e3
    # in-core references
    incore_b0 = incore_same = None
    if not args.no_incore and spec["mode"] == "bf16":
        if args.config == "r50" and b0:
            incore_b0 = in_core_rate(args, spec_for(args, b0), rank, world, chunk, args.steps)
            if in_core_device_bytes(spec) < 0.85 * torch.cuda.get_device_properties(dev).total_memory:
                incore_same = in_core_rate(args, spec, rank, world, chunk, args.steps)
        else:
            incore_same = in_core_rate(args, spec, rank, world, chunk, args.steps)
    if rank != 0:
        return None
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
    roof = None
    if per_kind:
        kind, (flops, secs, cnt, ev_secs, mhz) = max(per_kind.items(), key=lambda kv: kv[1][1])
        ach = flops / secs / 1e12
        impl = os.environ.get("OC_CONV_IMPL", "tc")
        if kind.startswith("attn") and spec["mode"] == "bf16":   # tensor-core products, HBM-bound
            gbs = flops / secs / 1e9
            roof = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / peaks["hbm_gbs"], "traffic": None, "kernel": kind, "launches": cnt,
                    "algorithmic_bytes": "12·L² per sample forward, 16·L² backward (bench.attn_bytes)",
                    "timed": "CUDA events around each attention function in the instrumented pass (all its "
                             "kernels: products, softmax, split reductions)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        elif impl == "simt" or kind.startswith("attn"):   # CUDA-core FFMA kernels
            roof = {"bound": "alu", "achieved": ach, "peak": FP32_SIMT_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP32_SIMT_TFLOPS, "traffic": None, "kernel": kind, "launches": cnt,
                    "timed": "CUDA events around each contraction kernel launch in the instrumented pass",
                    "peak_source": "derived: 148 SM x 128 FFMA lanes x 2 x 1.965 GHz"}
        else:
            pk = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
            tpath = os.path.join(ROOT, "profiles", f"r02_conv_traffic_{args.config}.json")
            traffic = None
            if os.path.exists(tpath):
                traffic = json.load(open(tpath)).get(kind, {}).get("bytes_per_launch")
            roof = {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                    "traffic": traffic, "traffic_unit": f"DRAM bytes per launch (ncu --set full, {tpath[len(ROOT) + 1:]})",
                    "kernel": kind, "launches": cnt,
                    "timed": "in-kernel %globaltimer span of each contraction launch (first CTA start to last CTA "
                             "end) in the instrumented pass, operand re-layout kernels excluded",
                    "achieved_event_timed": flops / ev_secs / 1e12 if ev_secs else None,
                    "algorithmic_bytes_per_launch": None if kind not in per_launch else
                    per_launch[kind][3] / per_launch[kind][4],
                    "per_launch_roofline": None if kind not in per_launch else {
                        "frac": per_launch[kind][0] / per_launch[kind][1],
                        "hbm_bound_share_of_bound_time": per_launch[kind][2] / per_launch[kind][0],
                        "definition": "Σ over this kind's launches of max(FLOPs / sustained bf16 peak, algorithmic "
                                      "bytes / HBM peak) ÷ Σ of their measured spans: short-reduction 1x1 "
                                      "convolutions are HBM-bound, so `frac` (FLOP rate ÷ tensor peak) "
                                      "understates how close the kind runs to its roofline"},
                    "by_shape": None if kind not in per_shape else [
                        {"shape": k_, "launches": v_[4], "ms": v_[0] * 1e3, "tflops": v_[1] / v_[0] / 1e12,
                         "gbs": v_[2] / v_[0] / 1e9, "frac_of_roofline": v_[3] / v_[0]}
                        for k_, v_ in sorted(per_shape[kind].items(), key=lambda kv: -kv[1][0])[:12]],
                    "sm_mhz_in_kernels": float(np.median(mhz)) if mhz else None,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step)"}
    total_flops = sum(f for (_, f) in fl.values())
    t_tc = total_flops / (peaks.get("bf16_tflops_sustained", 1395.5) * 1e12)
    incore_ref = incore_b0 or incore_same
    line = {
        "metric": "samples/sec at k x in-budget batch vs in-core; host-link GB/s; overlap %",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if spec["mode"] == "bf16" else "f32", "data": "synthetic (seeded N(0,1) images, U labels)",
        "config": {"workload": workload_name(args, spec, B_p, b0 or 1), "global_batch": B_glob,
                   "per_gpu_batch": spec["batch"], "b0_in_core_max": b0,
                   "physical_budget_bytes": B_p, "pinned_bytes": pinned, "workspace_bytes": ws,
                   "swap_pool_bytes": pool, "scheduler_budget_bytes": B_s,
                   "device_bytes_used": pinned + pool + ws,
                   "in_core_footprint_bytes": F_peak, "window_bytes": W_sel, "window_selection": window_probe or
                   args.window, "allocator": mode, "chunk_bytes": chunk,
                   "swap_policy": args.policy if not dist_ else f"{args.policy} (function distance {dist_})",
                   "arrival_trigger": args.trigger, "host_copy_bytes": host_bytes, "host_ram_bytes": ram,
                   "host_pool_bytes": host_pool_bytes, "host_pool_numa_node": host_numa,
                   "dp_bucket_bytes": args.bucket_mib * MiB if world > 1 else None,
                   "parallelism": f"dp{world}", "cuda_graph_replay": not args.no_graph,
                   "l2_flush": "inputs larger than L2 (activations GBs per step)", "notes": notes},
        "clocks": clk.summary(),
        "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "wall clock around oc_run_step: host inputs/parameters swapped in, loss written back, "
                        "every step"},
        "gpu_launches": n_k,
        "roofline": roof,
        "link_roofline": {"t_duplex_ms": t_duplex * 1e3, "t_phase_separated_ms": t_phase * 1e3,
                          "frac_duplex": t_duplex * 1e3 / step_ms, "frac_phase_separated": t_phase * 1e3 / step_ms,
                          "bytes_by_phase": ph, "measured_gbs": link, "pcie5_x16_gbs_per_dir": PCIE5_X16_GBS,
                          "t_tensor_ms": t_tc * 1e3,
                          "note": "duplex = max(h2d/BW_h2d, d2h/BW_d2h); phase-separated = forward transfers then "
                                  "backward transfers, each direction-limited (SURVEY H1)"},
        "host_link": {"h2d_gbs_step": h2d / (step_ms / 1e3) / 1e9, "d2h_gbs_step": d2h / (step_ms / 1e3) / 1e9,
                      "h2d_gbs_busy": (h2d / (h2d_busy / 1e3) / 1e9) if h2d_busy else None,
                      "d2h_gbs_busy": (d2h / (d2h_busy / 1e3) / 1e9) if d2h_busy else None,
                      "pcie5_x16_gbs_per_dir": PCIE5_X16_GBS, "measured_pinned_gbs": link,
                      "nvml_pcie_counters": pcie.summary(), "per_copy": copy_diag},
        "overlap_pct": 100 * overlap,
        "overlap_definition": "|transfer ∩ compute| / |transfer| (executor timeline unions); the compute side "
                              "is compute_under_transfer_pct",
        "compute_under_transfer_pct": None if cut is None else 100 * cut,
        "makespan_model": {"predicted_ms": sim["makespan_ms"], "predicted_boundary_ms": sim0["makespan_ms"],
                           "compute_ms": sim["compute_ms"], "stall_ms": sim["stall_ms"],
                           "link_gbs": {"h2d": bw_h, "d2h": bw_d, "source": "bytes / busy copy time of the "
                                                                           "instrumented pass"}},
        "instrumented_pass": {"steps": 3, "ms_per_step": instr_step_ms,
                              "note": "overlap, busy times and kernel durations come from this pass (CUDA events "
                                      "around every function and transfer); the timed steps replay a CUDA graph"},
        "compute_busy_ms": comp_busy,
        "in_core_samples_per_s": incore_ref,
        "in_core_same_batch_samples_per_s": incore_same,
        "fraction_of_in_core": (value / incore_ref) if incore_ref else None,
        "trainable_batch_multiple": (spec["batch"] / b0) if b0 else None,
        "schedule": {k: ss[k] for k in ("bytes_h2d", "bytes_alloc", "bytes_d2h", "bytes_d2h_dirty", "peak_sched",
                                        "peak_phys", "if_peak", "n_max")},
        "vmm": {k: mstat[k] for k in ("n_driver_map", "n_map_calls", "n_map_memo_hits", "map_us")},
        "loss": loss,
        "paper_context": "V100 16 GB, fp32: ResNet-50 b=1440 (7.5x the in-core maximum 190) at 321 images/s = "
                         "55% of in-core 581 (PAPER.md P:10, Table 1 P:135-137)",
    }
    if args.config != "mlp":
        line["cpu_baseline"] = cpu_baseline(args)
    return line


# ------------------------------------------------------------ oracle (CPU)
def oracle_sample(args):
    """The oracle's bounded sample of the configured workload: (one-step
    callable, samples per step, time scale to the real sample, description)."""
    from oracle import numerics as nm
    from synth import nets
    if args.config == "biggan":
        spec = nets.biggan(batch=1)
        pG, pD = nets.make_gan_params(spec)
        z1, z2, xr = nets.make_gan_inputs(spec)
        return (lambda: nm.gan_step(spec, pG, pD, z1, z2, xr)), 1, 1.0, \
            "biggan batch 1 per step (numpy float64 oracle with bf16 rounding)"
    if args.config == "unet":
        # b = 1 on a 256² crop, scaled by pixel count (labelled extrapolated)
        spec = nets.unet(batch=1, image=256)
        scale, note = 16.0, "unet batch 1 on a 256x256 crop, time scaled by the 16x pixel count (extrapolated)"
    elif args.config == "mlp":
        spec, scale, note = nets.mlp6(), 1.0, "mlp6 batch 8 per step"
    elif args.config == "densenet":
        spec = nets.densenet(batch=1)
        scale, note = 1.0, "densenet121 batch 1 per step"
    elif args.config == "deeplab":
        spec = nets.deeplabv3plus(batch=2, image=257)
        scale, note = 2.0, ("deeplabv3plus batch 2 on a 257x257 crop, time scaled by the 4x pixel count to one "
                            "513x513 sample pair (extrapolated)")
    elif args.config == "pix2pix":
        spec = nets.pix2pixhd(batch=1, image=(128, 256))
        scale, note = 16.0, "pix2pixhd batch 1 on a 128x256 crop, time scaled by the 16x pixel count (extrapolated)"
    else:
        spec = {"r50": lambda: nets.resnet(50, batch=1), "r1001": lambda: nets.preact_resnet(1001, batch=2)}.get(
            args.config, lambda: nets.resnet(18, batch=2))()
        scale, note = 1.0, f"{spec['name']} batch {spec['batch']} per step"
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    return (lambda: nm.train_step(spec, p, x, y)), spec["batch"], scale, note + " (numpy float64 oracle)"


def oracle_threads():
    """Threads the numpy oracle actually uses (the BLAS pool; torchrun sets
    OMP_NUM_THREADS=1 for its workers)."""
    try:
        from threadpoolctl import threadpool_info
        n = [i["num_threads"] for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:  # noqa: BLE001
        pass
    return len(os.sched_getaffinity(0))


def cpu_baseline(args, min_s=10.0):
    """The oracle on a bounded sample of the same workload, on all host cores
    (repeated steps until ~10 s of CPU work)."""
    cores = oracle_threads()
    fn, batch, scale, note = oracle_sample(args)
    t0 = time.perf_counter()
    steps = 0
    while steps == 0 or (time.perf_counter() - t0 < min_s and steps < 50):
        fn()
        steps += 1
    dt = (time.perf_counter() - t0) * scale
    return {"value": batch * steps / dt, "unit": "samples/s", "cores": cores, "kind": "oracle",
            "sample": f"{note}, {steps} step(s)"}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, bounded sample per step."""
    cores = oracle_threads()
    fn, batch, scale, note = oracle_sample(args)
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    dt = (time.perf_counter() - t0) * scale
    v = batch * args.steps / dt
    return {"impl": "reference", "metric": "samples/sec at k x in-budget batch vs in-core; host-link GB/s; overlap %",
            "value": v, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {note} (bounded CPU sample of the GPU arm's workload)"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle", "sample": note},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def spawn(args):
    """`--gpus N` without a torchrun environment: launch N ranks (one per GPU)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    line = run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
