"""One rank of the full-size multi-GPU parity test (tests/test_multigpu.py).

Config 4 at full size: 1.1B parameters per worker, one worker per GPU, FP16
pseudo-gradients, P2P mode (and the NCCL ordered mode), two outer rounds.  Each
rank checks slices at the start, an unaligned middle, the end, every owner-slot
edge q*S and every piece boundary of the P2P plan inside every slot, of its
theta_t / theta_local / momentum, against the oracle's rank-ordered outer round
over every rank's inputs restricted to the slice (all elementwise), bit for bit.
(Every element at full size, K ranks sharing one GPU: tests/test_full_size.py.)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_07852_b200 as D  # noqa: E402
from paper_2407_07852_b200 import dist as PD  # noqa: E402
from oracle import driver as DR  # noqa: E402
from oracle import oracle as O  # noqa: E402

N = int(os.environ.get("MP_FULL_N", 1_100_000_000))
M = 4096
E = 256  # elements on each side of a slot edge / piece boundary


def slice_starts(n, k):
    """Start, middle, end, and [b - E, b + E) around every slot edge and every piece
    boundary of the default plan (1,1,2,2,1,1 eighths of a slot at this size)."""
    S = PD.slot_elems(n, k)
    cum = [1, 2, 4, 6, 7]
    starts = {(0, M), (n // 2 - 777, M), (n - M, M)}
    for q in range(k + 1):
        for b in [0] + [(S // 64) * c // 8 * 64 for c in cum]:
            x = q * S + b
            lo, hi = max(0, x - E), min(n, x + E)
            if lo < hi:
                starts.add((lo, hi - lo))
    return sorted(starts)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def main():
    r = PD.init("gloo")
    D.lib.dlc_set_device(r.local)
    k = r.world
    port = O.port()
    hyper = DR.Hyper()
    out = {"rank": r.rank, "checks": []}
    for mode_name, mode in (("p2p", D.MODE_P2P), ("ordered", D.MODE_ORDERED)):
        coll = PD.make_nccl_collective(r, mode)
        e = D.DilocoEngine(D.DilocoConfig(1, k, D.FP16, 4), D.OptimHyperparams(), N, r.local)
        e.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
        slices = slice_starts(N, k)
        ws = {(lo, m): DR.make_workers(O.rng_fill(4242, "theta", 0, m, -0.05, 0.05, first=lo), k, hyper)
              for lo, m in slices}
        for rnd in range(2):
            # end-of-window weights: theta_t - U(-1e-3, 1e-3) keyed by (round, rank)
            e.rng_perturb(4242, "local", rnd * 64 + r.rank, -1e-3, 1e-3)
            res = e.outer_step(coll, wait=True)
            assert res.applied and res.outer_epoch == rnd + 1
            for lo, m in slices:
                for j, w in enumerate(ws[lo, m]):
                    noise = O.rng_fill(4242, "local", rnd * 64 + j, m, -1e-3, 1e-3, first=lo)
                    w.theta_local = (w.theta_t - noise).astype(np.float32)
                DR.outer_round(port, ws[lo, m], D.FP16, hyper)
                me = ws[lo, m][r.rank]
                for which, want in ((D.THETA_T, me.theta_t), (D.THETA_LOCAL, me.theta_local),
                                    (D.MOMENTUM, me.buf)):
                    got = e.download_range(which, lo, m)
                    assert np.array_equal(bits(got), bits(want)), (mode_name, rnd, lo, which)
            out["checks"].append(f"{mode_name} round {rnd}: {len(slices)} slices (slot edges, piece boundaries) "
                                 f"x 3 vectors bitwise at N={N}")
        e.close()
        coll.close()
    PD.barrier(r.world)
    print("MPRESULT " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
