"""Host logic of bench.py's derived metrics (no GPU): the timeline overlap
ratios, the algorithmic FLOP / byte counts the roofline divides by, and the
link bounds' phase split inputs."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _brute_cut(tl, lo, hi, step=0.25):
    """|T ∩ C| / |C| by sampling the time axis on a fine grid."""
    ts = np.arange(lo, hi, step) + step / 2
    c = np.zeros_like(ts, dtype=bool)
    t = np.zeros_like(ts, dtype=bool)
    for e in tl:
        m = (ts >= e["t0"]) & (ts < e["t1"])
        if e["stream"] == "compute":
            c |= m
        elif e["stream"] in ("h2d", "d2h"):
            t |= m
    return (c & t).sum() / c.sum()


def test_compute_under_transfer_matches_brute_force():
    rng = np.random.default_rng(5)
    for _ in range(50):
        tl = []
        for s in ("compute", "h2d", "d2h"):
            for _ in range(int(rng.integers(1, 8))):
                a = float(rng.integers(0, 80))
                tl.append({"stream": s, "t0": a, "t1": a + float(rng.integers(1, 20))})
        got = bench.compute_under_transfer(tl)
        assert abs(got - _brute_cut(tl, 0, 100)) < 1e-9


def test_compute_under_transfer_edges():
    assert bench.compute_under_transfer([{"stream": "h2d", "t0": 0, "t1": 1}]) is None
    tl = [{"stream": "compute", "t0": 0, "t1": 10}, {"stream": "d2h", "t0": 10, "t1": 20}]
    assert bench.compute_under_transfer(tl) == 0.0
    tl = [{"stream": "compute", "t0": 2, "t1": 4}, {"stream": "h2d", "t0": 0, "t1": 10},
          {"stream": "d2h", "t0": 1, "t1": 3}]
    assert bench.compute_under_transfer(tl) == 1.0


def _conv_doc(kind, acc=False, dtype="bf16"):
    a = {"dtype": dtype, "N": 2, "H": 8, "W": 6, "C": 64, "K": 128, "R": 3, "S": 3, "stride": 2, "pad": 1,
         "P": 4, "Q": 3, "accumulate": acc}
    return json.dumps({"variables": [], "functions": [{"id": "f", "in": [], "out": [],
                                                       "op": {"kind": kind, "args": {}, "attrs": a}}]})


def test_conv_flops_and_bytes():
    x, y, w = 2 * 8 * 6 * 64, 2 * 4 * 3 * 128, 128 * 3 * 3 * 64
    macs = 2 * 4 * 3 * 128 * 9 * 64
    for kind in ("conv_fwd", "conv_dgrad", "conv_wgrad"):
        assert bench.conv_flops(_conv_doc(kind))["f"] == (kind, 2.0 * macs)
    assert bench.conv_bytes(_conv_doc("conv_fwd"))["f"] == 2 * x + 2 * w + 2 * y
    assert bench.conv_bytes(_conv_doc("conv_fwd", acc=True))["f"] == 2 * x + 2 * w + 4 * y
    assert bench.conv_bytes(_conv_doc("conv_dgrad"))["f"] == 2 * y + 2 * w + 2 * x
    assert bench.conv_bytes(_conv_doc("conv_dgrad", acc=True))["f"] == 2 * y + 2 * w + 4 * x
    assert bench.conv_bytes(_conv_doc("conv_wgrad"))["f"] == 2 * y + 2 * x + 4 * w
    assert bench.conv_bytes(_conv_doc("conv_fwd", dtype="f32"))["f"] == 4 * x + 4 * w + 4 * y
