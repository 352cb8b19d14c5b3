#!/usr/bin/env python
"""NCCL all-reduce bus bandwidth on this box (development tool; run under torchrun).

    NCCL_ALGO=NVLS torchrun --nproc-per-node 4 tools/nccl_probe.py

Times torch.distributed.all_reduce (NCCL) of a flat FP16 / FP32 buffer of the
1.1B-parameter pseudo-gradient with SUM and AVG, CUDA events, max over ranks.
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    dist.init_process_group("nccl")
    r, k = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    n = int(os.environ.get("PROBE_N", 1_100_000_000))
    dtypes = [getattr(torch, d) for d in os.environ.get("PROBE_DTYPES", "float16,float32").split(",")]
    for dtype in dtypes:
        x = torch.randn(n, dtype=dtype, device="cuda") * 1e-3
        for op_name, op in (("sum", dist.ReduceOp.SUM), ("avg", dist.ReduceOp.AVG)):
            for _ in range(2):
                dist.all_reduce(x, op=op)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            steps = 5
            for _ in range(steps):
                dist.all_reduce(x, op=op)
            b.record()
            b.synchronize()
            got = [None] * k  # (object gather: NCCL_ALGO=NVLS has no FP32 all-reduce)
            dist.all_gather_object(got, a.elapsed_time(b) / steps)
            ms = max(got)
            bus = x.numel() * x.element_size() * 2 * (k - 1) / k / (ms * 1e-3) / 1e9
            if r == 0:
                print(json.dumps({"dtype": str(dtype), "op": op_name, "algo": os.environ.get("NCCL_ALGO", "default"),
                                  "ms": ms, "bus_gbs": bus}), flush=True)
        del x
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
