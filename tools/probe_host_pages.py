"""Host-link copy rate into a large page-locked host region allocated three
ways: cudaHostAlloc (4 KiB pages), anonymous mmap + madvise(MADV_HUGEPAGE)
(transparent 2 MiB pages) + cudaHostRegister, and plain mmap +
cudaHostRegister — copies of 1 GiB at offsets spread over the region, D2H and
H2D.  Does the page size of the pinned pool change the per-copy rate (I/O
translation of many 4 KiB pages)?  Prints one JSON line.  Not part of the
product.

Usage: python tools/probe_host_pages.py [--pool-gib 48]"""
import argparse
import ctypes
import json
import mmap

import torch

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
libc.memset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
libc.munmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
MADV_HUGEPAGE = 14


def cudart():
    lib = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    return lib


def rate(dev_ptr, host_ptr, n, d2h, iters=4):
    rt = cudart()
    s = torch.cuda.Stream()
    kind = 2 if d2h else 1   # cudaMemcpyDeviceToHost / HostToDevice
    dst, src = (host_ptr, dev_ptr) if d2h else (dev_ptr, host_ptr)
    rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rt.cudaMemcpyAsync(dst, src, n, kind, ctypes.c_void_p(s.cuda_stream))
    e0.record(s)
    for _ in range(iters):
        rt.cudaMemcpyAsync(dst, src, n, kind, ctypes.c_void_p(s.cuda_stream))
    e1.record(s)
    torch.cuda.synchronize()
    return round(n * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


def sweep(base, size, dev, n):
    out = []
    for frac in (0.0, 0.33, 0.66, 0.97):
        off = min(int(frac * size) & ~((1 << 21) - 1), size - n)
        out.append({"off_gib": round(off / 2**30, 1), "d2h": rate(dev, base + off, n, True),
                    "h2d": rate(dev, base + off, n, False)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pool-gib", type=int, default=48)
    a = ap.parse_args()
    size = a.pool_gib << 30
    n = 1 << 30
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    dptr = dev.data_ptr()
    rt = cudart()
    res = {"thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()}
    pinned = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    res["cudaHostAlloc"] = sweep(pinned.data_ptr(), size, dptr, n)
    del pinned
    for label, huge in (("mmap_thp_register", True), ("mmap_register", False)):
        p = libc.mmap(None, size, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
        if huge:
            libc.madvise(p, size, MADV_HUGEPAGE)
        libc.memset(p, 0, size)
        rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
        rc = rt.cudaHostRegister(p, size, 1 | 2)
        if huge:
            res["AnonHugePages_while_mapped"] = [x for x in open("/proc/meminfo")
                                                 if x.startswith("AnonHugePages")][0].strip()
        if rc != 0:
            res[label] = f"cudaHostRegister failed ({rc})"
        else:
            res[label] = sweep(p, size, dptr, n)
            rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
            rt.cudaHostUnregister(p)
        libc.munmap(p, size)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
