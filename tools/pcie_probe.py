#!/usr/bin/env python
"""PCIe ground truth for the e2e (host-buffer) outer step (development tool):
pinned H2D alone, D2H alone, and both at once on two streams, for the 4.4 GB
vectors of the 1.1B workload, in chunks of the size the host path uses."""
import json
import sys
import time

import torch


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_100_000_000
    chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 16 << 20
    dev = torch.device("cuda:0")
    h_src = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_dst = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_src.fill_(1.0)
    d_a = torch.empty(n, dtype=torch.float32, device=dev)
    d_b = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            for o in range(0, n, chunk):
                d_a[o:o + chunk].copy_(h_src[o:o + chunk], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            for o in range(0, n, chunk):
                h_dst[o:o + chunk].copy_(d_b[o:o + chunk], non_blocking=True)

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    gb = n * 4 / 1e9
    t_h2d = timed(h2d)
    t_d2h = timed(d2h)
    t_both = timed(lambda: (h2d(), d2h()))
    print(json.dumps({"bytes_each_gb": gb, "chunk_elems": chunk, "h2d_ms": t_h2d * 1e3, "h2d_gbs": gb / t_h2d,
                      "d2h_ms": t_d2h * 1e3, "d2h_gbs": gb / t_d2h, "both_ms": t_both * 1e3,
                      "both_gbs_aggregate": 2 * gb / t_both}))


if __name__ == "__main__":
    main()
