"""Does splitting one large pinned copy over several copy-engine streams raise
the single-direction host-link rate?  (The out-of-core step is bound by one
direction at a time: forward D2H, backward H2D.)  Prints one JSON line: GB/s
per direction for 1, 2 and 4 concurrent streams each moving an equal share of
the same total, plus pinned-vs-mapped host memory.  Not part of the product."""
import json

import torch


def rate(total, parts, direction, iters=8):
    n = total // parts
    hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(parts)]
    ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(parts)]
    ss = [torch.cuda.Stream() for _ in range(parts)]

    def go():
        for h, d, s in zip(hs, ds, ss):
            with torch.cuda.stream(s):
                if direction == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)

    go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        go()
    e1.record()
    torch.cuda.synchronize()
    return round(n * parts * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)


def main():
    out = {}
    for total_mib in (64, 512):
        total = total_mib << 20
        for parts in (1, 2, 4):
            out[f"{total_mib}MiB_x{parts}"] = {"h2d": rate(total, parts, "h2d"), "d2h": rate(total, parts, "d2h")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
