"""Phase-0 box probe: pinned host<->device copy bandwidth per
direction, alone and duplex, on copy-engine streams.  Not part of the product;
the numbers are recorded in DESIGN.md / profiles/ as the host-link roofline
denominators."""
import json
import os
import torch


def bw(nbytes, fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    out = {"cores": len(os.sched_getaffinity(0))}
    sh = torch.cuda.Stream()
    sd = torch.cuda.Stream()
    for mb in (2, 40, 256, 1024):
        n = mb << 20
        h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
        d_b = torch.empty(n, dtype=torch.uint8, device="cuda")

        def h2d():
            with torch.cuda.stream(sh):
                d_a.copy_(h_in, non_blocking=True)
            torch.cuda.current_stream().wait_stream(sh)

        def d2h():
            with torch.cuda.stream(sd):
                h_out.copy_(d_b, non_blocking=True)
            torch.cuda.current_stream().wait_stream(sd)

        def duplex():
            with torch.cuda.stream(sh):
                d_a.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(sd):
                h_out.copy_(d_b, non_blocking=True)
            torch.cuda.current_stream().wait_stream(sh)
            torch.cuda.current_stream().wait_stream(sd)

        out[f"{mb}MiB"] = {
            "h2d_gbs": round(bw(n, h2d), 2),
            "d2h_gbs": round(bw(n, d2h), 2),
            "duplex_total_gbs": round(bw(2 * n, duplex), 2),
        }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
