"""Host-link copy rate of one 1 GiB copy as a function of the host and device
offsets' alignment (the executor packs host copies at 256-byte alignment).
Prints one JSON line.  Not part of the product."""
import json

import torch


def rate(dst, src, iters=4):
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        dst.copy_(src, non_blocking=True)
        e0.record(s)
        for _ in range(iters):
            dst.copy_(src, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    return round(src.numel() * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


def main():
    n = 1 << 30
    host = torch.empty(n + (1 << 21), dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(n + (1 << 21), dtype=torch.uint8, device="cuda")
    out = {}
    for ho in (0, 256, 4096, 65536 + 256):
        for do in (0, 256):
            out[f"host+{ho}_dev+{do}"] = {"d2h": rate(host[ho:ho + n], dev[do:do + n]),
                                         "h2d": rate(dev[do:do + n], host[ho:ho + n])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
