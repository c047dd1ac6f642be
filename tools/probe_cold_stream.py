"""Host-link D2H / H2D rate when copies stream through a large pinned host
region once (as the out-of-core step's swap-outs do: every copy lands on
fresh host pages) against the same copies repeated on one warm region: does
the I/O translation of a cold 4 KiB-page pinned pool (cudaHostAlloc) cost
rate, and does a transparent-huge-page pool (mmap + MADV_HUGEPAGE +
cudaHostRegister) avoid it?  Prints one JSON line.  Not part of the product.

Usage: python tools/probe_cold_stream.py [--pool-gib 48 --copy-mib 256]"""
import argparse
import ctypes
import json
import mmap
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_host_pages import MADV_HUGEPAGE, cudart, libc  # noqa: E402


def stream_rate(rt, dptr, base, size, n, d2h, warm):
    s = torch.cuda.Stream()
    kind = 2 if d2h else 1
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    count = size // n
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(count):
        h = base + (0 if warm else i * n)
        dst, src = (h, dptr) if d2h else (dptr, h)
        rt.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src), n, kind, ctypes.c_void_p(s.cuda_stream))
    e1.record(s)
    torch.cuda.synchronize()
    return round(n * count / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


def measure(rt, dptr, base, size, n):
    out = {}
    for d2h in (True, False):
        k = "d2h" if d2h else "h2d"
        out[k + "_cold_pass1"] = stream_rate(rt, dptr, base, size, n, d2h, warm=False)
        out[k + "_cold_pass2"] = stream_rate(rt, dptr, base, size, n, d2h, warm=False)
        out[k + "_warm_one_region"] = stream_rate(rt, dptr, base, size, n, d2h, warm=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pool-gib", type=int, default=48)
    ap.add_argument("--copy-mib", type=int, default=256)
    a = ap.parse_args()
    size, n = a.pool_gib << 30, a.copy_mib << 20
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    rt = cudart()
    res = {"pool_gib": a.pool_gib, "copy_mib": a.copy_mib,
           "thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()}
    pinned = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    res["cudaHostAlloc"] = measure(rt, dev.data_ptr(), pinned.data_ptr(), size, n)
    del pinned
    p = libc.mmap(None, size, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    libc.madvise(p, size, MADV_HUGEPAGE)
    libc.memset(p, 0, size)
    rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
    rc = rt.cudaHostRegister(p, size, 1 | 2)
    res["AnonHugePages"] = [x for x in open("/proc/meminfo") if x.startswith("AnonHugePages")][0].strip()
    res["mmap_thp_register"] = measure(rt, dev.data_ptr(), p, size, n) if rc == 0 else f"register failed {rc}"
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
