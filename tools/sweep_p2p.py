#!/usr/bin/env python
"""Sweep the DLC_MODE_P2P knobs in-process (development tool; run under torchrun).

    torchrun --nproc-per-node 4 tools/sweep_p2p.py --params 1100000000

Times the outer step (CUDA events on the engine stream, max over ranks) for
DLC_P2P_COPY x DLC_P2P_PIECES x DLC_COMM_CTAS, plus the NCCL ordered mode.
"""
import argparse
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
    a = ap.parse_args()
    r = PD.init("gloo")
    torch.cuda.set_device(r.local)
    D.lib.dlc_set_device(r.local)
    n, k = a.params, r.world
    colls = {"p2p": PD.make_nccl_collective(r, D.MODE_P2P), "ordered": PD.make_nccl_collective(r, D.MODE_ORDERED)}
    eng = D.DilocoEngine(D.DilocoConfig(1, k, D.FP16, 1 << 40), D.OptimHyperparams(), n, r.local)
    eng.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    xs = [torch.empty(n, dtype=torch.float32, device=f"cuda:{r.local}") for _ in range(2)]
    for i, x in enumerate(xs):
        eng.rng_perturb(4242, "local", r.rank * 16 + i, -1e-3, 1e-3, dst_dev_ptr=x.data_ptr())
    stream = torch.cuda.ExternalStream(eng.stream, device=f"cuda:{r.local}")
    configs = [("ordered", None, None, None, None, 0, 0, 128, "")]
    movers = os.environ.get("SWEEP_MOVERS", "sm,ce").split(",")
    pieces_l = [int(x) for x in os.environ.get("SWEEP_PIECES", "1,2,4,8").split(",")]
    ctas_l = [int(x) for x in os.environ.get("SWEEP_CTAS", "0,32,64,128,256").split(",")]
    barriers = os.environ.get("SWEEP_BARRIERS", "flag").split(",")
    piece_ctas_l = [int(x) for x in os.environ.get("SWEEP_PIECE_CTAS", "0").split(",")]
    tma_l = [int(x) for x in os.environ.get("SWEEP_TMA_CTAS", "0").split(",")]  # 0: per-thread fold
    tthr_l = [int(x) for x in os.environ.get("SWEEP_TMA_THREADS", "128").split(",")]
    # SWEEP_ENV="A=1,B=2;A=0": extra environment per config; SWEEP_REPEAT: interleaved repeats (A/B)
    env_l = os.environ.get("SWEEP_ENV", "").split(";")
    plans = os.environ.get("SWEEP_PLANS", "").split(";") if os.environ.get("SWEEP_PLANS") else None
    for barrier in barriers:
        for mover in movers:
            for pieces in (plans or pieces_l):
                for ctas in (ctas_l if mover in ("sm", "push", "push2") else (0,)):
                    for pc in piece_ctas_l:
                        for tc in tma_l:
                            for tt in tthr_l:
                                for ev in env_l:
                                    configs.append(("p2p", mover, pieces, ctas, barrier, pc, tc, tt, ev))
    configs = configs * int(os.environ.get("SWEEP_REPEAT", "1"))
    results = []
    for mode, mover, pieces, ctas, barrier, pc, tc, tt, ev in configs:
        for kv in filter(None, ev.split(",")):
            key, val = kv.split("=", 1)
            os.environ[key] = val
        os.environ["DLC_TMA_THREADS"] = str(tt)
        os.environ["DLC_P2P_PIECE_CTAS"] = str(pc)
        os.environ["DLC_FOLD_TMA"] = "1" if tc else "0"  # tc < 0: TMA fold, default CTA count
        if tc > 0:
            os.environ["DLC_TMA_CTAS"] = str(tc)
        else:
            os.environ.pop("DLC_TMA_CTAS", None)
        if mover:
            os.environ["DLC_P2P_COPY"] = mover
            if isinstance(pieces, str):
                os.environ["DLC_P2P_PLAN"] = pieces
            else:
                os.environ.pop("DLC_P2P_PLAN", None)
                os.environ["DLC_P2P_PIECES"] = str(pieces)
            os.environ["DLC_COMM_CTAS"] = str(ctas)
            os.environ["DLC_P2P_BARRIER"] = barrier
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
        results.append({"mode": mode, "mover": mover, "pieces": pieces, "ctas": ctas, "barrier": barrier,
                        "piece_ctas": pc, "tma_ctas": tc, "tma_threads": tt, "env": ev, "ms": ms})
        if r.rank == 0:
            print(json.dumps(results[-1]), flush=True)
    eng.close()
    for c in colls.values():
        c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
