#!/usr/bin/env python
"""Run DLC_MODE_P2P outer steps of a single-process dlc_world (development / ncu tool).

    python tools/world_step.py --ranks 4 --params 1100000000 --steps 2
    ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum \
        -k regex:fold_push python tools/world_step.py --ranks 4

One process drives every rank (rank r on GPU r % ngpu) and the ranks
synchronise through CUDA events, not spinning flag barriers, so ncu's kernel
replay can capture the owner fold while it moves its bytes over NVLink: per
launch, the NVLink bytes the fold pulls (nvlrx) and pushes (nvltx) on its GPU,
and its duration with the links to itself.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_07852_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=0, help="0 = one per GPU")
    ap.add_argument("--params", type=int, default=1_100_000_000)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--precision", choices=["fp16", "fp32"], default="fp16")
    a = ap.parse_args()
    g = D.device_count()
    k = a.ranks or g
    prec = D.FP16 if a.precision == "fp16" else D.FP32
    world = D.World(D.DilocoConfig(1, k, prec, 1 << 30), D.OptimHyperparams(), a.params, [i % g for i in range(k)],
                    mode=D.MODE_P2P)
    for r, e in enumerate(world.engines):
        e.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    times = []
    for s in range(a.steps):
        for r, e in enumerate(world.engines):
            e.rng_perturb(4242, "local", s * 64 + r, -1e-3, 1e-3)  # end-of-window weights
        for e in world.engines:
            e.synchronize()
        t0 = time.perf_counter()
        res = world.outer_step()
        times.append((time.perf_counter() - t0) * 1e3)
        assert res.applied
    world.close()
    w = 2 if prec == D.FP16 else 4
    S = D.slot_elems(a.params, k) if hasattr(D, "slot_elems") else None
    print(json.dumps({"ranks": k, "gpus": g, "params": a.params, "precision": a.precision, "wall_ms": times,
                      "nvlink_bytes_per_direction_per_rank": 2 * (k - 1) * (-(-a.params // k)) * w,
                      "slot": S}))


if __name__ == "__main__":
    main()
