"""Host-link copy rate into different regions of one large pinned host
allocation (the executor's host pool is a single cudaHostAlloc region of
tens of GB): does the rate depend on where in the pool a copy lands (NUMA
placement of the pages), and on the copy size?  Prints one JSON line.
Not part of the product.

Usage: python tools/probe_host_pool.py [--pool-gib 64 --copy-mib 1024]"""
import argparse
import json

import torch


def rate(dev, host, n, d2h, iters=4):
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        (host[:n].copy_(dev[:n], non_blocking=True) if d2h else dev[:n].copy_(host[:n], non_blocking=True))
        e0.record(s)
        for _ in range(iters):
            (host[:n].copy_(dev[:n], non_blocking=True) if d2h else dev[:n].copy_(host[:n], non_blocking=True))
        e1.record(s)
    torch.cuda.synchronize()
    return round(n * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pool-gib", type=int, default=64)
    ap.add_argument("--copy-mib", type=int, default=1024)
    a = ap.parse_args()
    n = a.copy_mib << 20
    pool = torch.empty(a.pool_gib << 30, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {"pool_gib": a.pool_gib, "copy_mib": a.copy_mib, "regions": []}
    for frac in (0.0, 0.25, 0.5, 0.75, 0.98):
        off = int(frac * (a.pool_gib << 30)) & ~((1 << 21) - 1)
        off = min(off, (a.pool_gib << 30) - n)
        h = pool[off:off + n]
        out["regions"].append({"offset_gib": round(off / 2**30, 1), "d2h": rate(dev, h, n, True),
                               "h2d": rate(dev, h, n, False)})
    sizes = {}
    for mib in (1, 4, 16, 64, 256):
        m = mib << 20
        sizes[f"{mib}MiB"] = {"d2h": rate(dev, pool, m, True, iters=16), "h2d": rate(dev, pool, m, False, iters=16)}
    out["sizes_at_offset0"] = sizes
    print(json.dumps(out))


if __name__ == "__main__":
    main()
