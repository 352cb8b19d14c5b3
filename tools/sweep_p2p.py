#!/usr/bin/env python
"""Sweep the DLC_MODE_P2P tuning in-process (development tool; run under torchrun).

    torchrun --nproc-per-node 4 tools/sweep_p2p.py --params 1100000000 \
        --plans "1,1,2,2,1,1;1,3,3,1" --fold-ctas 0 48 80 --fold-threads 0 256 --repeat 2

Times the outer step (CUDA events on the engine stream, max over ranks) for every
combination of piece plan x fold CTAs x fold threads (dlc_p2p_set_tuning; 0 = the
measured default), interleaving the repeats so box drift spreads over all
configurations, plus the NCCL ordered mode as the baseline.
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2407_07852_b200 as D  # noqa: E402
from paper_2407_07852_b200 import dist as PD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=1_100_000_000)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--plans", default="", help="';'-separated piece plans ('' = default)")
    ap.add_argument("--fold-ctas", type=int, nargs="+", default=[0])
    ap.add_argument("--fold-threads", type=int, nargs="+", default=[0])
    ap.add_argument("--piece-ctas", type=int, nargs="+", default=[0])
    ap.add_argument("--fold-kernel", type=int, nargs="+", default=[0], help="0 single-leader, 1 warp-specialised")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--no-ordered", action="store_true")
    a = ap.parse_args()
    r = PD.init("gloo")
    torch.cuda.set_device(r.local)
    D.lib.dlc_set_device(r.local)
    n, k = a.params, r.world
    colls = {"p2p": PD.make_nccl_collective(r, D.MODE_P2P)}
    if not a.no_ordered:
        colls["ordered"] = PD.make_nccl_collective(r, D.MODE_ORDERED)
    eng = D.DilocoEngine(D.DilocoConfig(1, k, D.FP16, 1 << 40), D.OptimHyperparams(), n, r.local)
    eng.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    xs = [torch.empty(n, dtype=torch.float32, device=f"cuda:{r.local}") for _ in range(2)]
    for i, x in enumerate(xs):
        eng.rng_perturb(4242, "local", r.rank * 16 + i, -1e-3, 1e-3, dst_dev_ptr=x.data_ptr())
    stream = torch.cuda.ExternalStream(eng.stream, device=f"cuda:{r.local}")
    plans = [p for p in a.plans.split(";")] if a.plans else [""]
    configs = [("p2p", p, fc, ft, pc, fk) for p, fc, ft, pc, fk in
               itertools.product(plans, a.fold_ctas, a.fold_threads, a.piece_ctas, a.fold_kernel)]
    if not a.no_ordered:
        configs.insert(0, ("ordered", "", 0, 0, 0, 0))
    results = []
    for mode, plan, fc, ft, pc, fk in configs * a.repeat:
        D.set_p2p_tuning(plan=[int(x) for x in plan.split(",")] if plan else None, fold_ctas=fc, fold_threads=ft,
                         piece_ctas=pc, fold_kernel=fk)
        c = colls[mode]
        for s in range(2):
            eng.outer_step_from(c, xs[s % 2].data_ptr())
        eng.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(a.steps):
            eng.outer_step_from(c, xs[s % 2].data_ptr())
        e1.record(stream)
        e1.synchronize()
        ms = PD.max_over_ranks(e0.elapsed_time(e1) / a.steps, r.world)
        results.append({"mode": mode, "plan": plan or "default", "fold_ctas": fc, "fold_threads": ft,
                        "piece_ctas": pc, "fold_kernel": fk, "ms": ms})
        if r.rank == 0:
            print(json.dumps(results[-1]), flush=True)
    D.set_p2p_tuning()
    eng.close()
    for c in colls.values():
        c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
