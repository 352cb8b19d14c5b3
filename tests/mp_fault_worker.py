"""One rank of the membership-change test (launched by tests/test_multigpu.py via torchrun).

Mirrors the reference's "killing one of four peers mid-reduce leaves survivor
mean" (test_collective.cpp:460-531) on the device path:

* DLC_MODE_P2P: every rank runs a full round, then the victim stops arriving
  mid-reduce (dlc_collective_inject_stall, the reference's stage hook).  Every
  rank's round fails with CollectiveError and leaves the engine state exactly
  as it was; the survivors shrink the collective around the victim and retry
  the same epoch: survivor mean, survivor divisor, contributors = K-1,
  attempts = 2, bitwise equal to the oracle's outer round over the survivors
  (reduce_average in survivor order, reduce.cpp:33-89), then one more round on
  the shrunk fleet.  The victim gets "excluded from round" when it tries to
  shrink itself in; a shrink below quorum raises QuorumError.
* DLC_MODE_ORDERED / DLC_MODE_ALLREDUCE: a planned exclusion after a full
  round; survivors run the next round on the shrunk NCCL communicator
  (ordered bitwise, allreduce within SPEC.md:325's tolerance).
* DLC_MODE_ORDERED / DLC_MODE_ALLREDUCE with a stalled peer (round 2): the
  victim never enters the round; NCCL does not time out, so the engine's
  failure detector does (reduce_timeout_ms after the round was enqueued): the
  survivors' outer step raises CollectiveError, they shrink with
  DLC_SHRINK_ABORT (which releases their blocked NCCL work), find the engine
  state unchanged, and retry the same epoch over the survivors (attempts = 2).
"""
import time
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


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def state(e):
    return {w: e.download(w) for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM)}


def want_state(w):
    return {D.THETA_T: w.theta_t, D.THETA_LOCAL: w.theta_local, D.ADAM_M: w.m, D.ADAM_V: w.v, D.MOMENTUM: w.buf}


def same(got, want):
    return all(np.array_equal(bits(got[k]), bits(want[k])) for k in want)


def close(e, w, mode, tag):
    """Bitwise for the rank-ordered modes; NCCL's reduction order within 1e-5 on theta_t."""
    if mode != D.MODE_ALLREDUCE:
        assert same(state(e), want_state(w)), tag
        return
    err = float(np.max(np.abs(e.download(D.THETA_T).astype(np.float64) - w.theta_t.astype(np.float64))))
    assert err <= 1e-5, (tag, err)


def main():
    r = PD.init("gloo")
    D.lib.dlc_set_device(r.local)
    k = r.world
    victim = 2 if k >= 4 else 1
    survivors = [j for j in range(k) if j != victim]
    me_alive = r.rank != victim
    out = {"rank": r.rank, "checks": []}
    port = O.port()
    n, h = 40_009, 2
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(77, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        return O.rng_fill(77, "grad", w * 1000 + t, n, -1e-2, 1e-2)

    cases = [("p2p-stall", D.MODE_P2P, D.FP16), ("p2p-stall", D.MODE_P2P, D.FP32),
             ("ordered-planned", D.MODE_ORDERED, D.FP16), ("allreduce-planned", D.MODE_ALLREDUCE, D.FP32),
             ("ordered-stall", D.MODE_ORDERED, D.FP32), ("allreduce-stall", D.MODE_ALLREDUCE, D.FP16)]
    for name, mode, prec in cases:
        tag = f"{name}/{'fp16' if prec else 'fp32'}"
        coll = PD.make_nccl_collective(r, mode)
        coll.set_reduce_timeout_ms(1500)
        ws = DR.make_workers(theta0, k, hyper)
        e = D.DilocoEngine(D.DilocoConfig(h, k, prec, 3 * h), D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2),
                           n, r.local)
        e.upload(D.THETA_T, theta0)
        e.upload(D.THETA_LOCAL, theta0)
        step = 0

        def inner(workers_idx):
            nonlocal step
            for _t in range(h):
                for j in workers_idx:
                    DR.inner_step(port, ws[j], grad_fn(j, step), hyper)
                if r.rank in workers_idx:
                    e.inner_step_host(grad_fn(r.rank, step), grad_is_scaled=False)
                step += 1

        # round 1: the whole fleet
        inner(list(range(k)))
        res = e.outer_step(coll, wait=True, report=True)
        DR.outer_round(port, ws, prec, hyper)
        assert res.applied and res.report.contributors == k and res.report.attempts == 1, tag
        close(e, ws[r.rank], mode, (tag, "round 1"))
        stall = name.endswith("stall")
        inner(list(range(k)) if stall else survivors)

        if stall and mode != D.MODE_P2P:
            # round 2: the victim never arrives; the survivors' round times out
            if not me_alive:
                time.sleep(4.0)  # past the survivors' 1.5 s deadline: it stopped participating
            else:
                before = state(e)
                epoch0 = e.scalars().outer_epoch
                t0 = time.time()
                try:
                    e.outer_step(coll, wait=True, report=True)
                    raise AssertionError(f"{tag}: the round with a stalled peer succeeded")
                except D.CollectiveError as x:
                    assert "timed out" in str(x), (tag, str(x))
                assert time.time() - t0 < 15.0, tag
                sub = coll.shrink([victim], quorum_min=k - 1, abort=True)  # releases the blocked round
                assert e.scalars().outer_epoch == epoch0, tag
                assert same(state(e), before), (tag, "a failed round changed the engine state")
                out["checks"].append(f"{tag}: timed-out round leaves state unchanged")
                res = e.outer_step(sub, wait=True, report=True)
                sw = [ws[j] for j in survivors]
                DR.outer_round(port, sw, prec, hyper)
                assert res.applied and res.report.contributors == k - 1 and res.report.attempts == 2, (
                    tag, res.report.attempts)
                close(e, ws[r.rank], mode, (tag, "survivor retry"))
                out["checks"].append(f"{tag}: survivors {survivors} after the timeout")
                e.close()
                sub.close()
                coll.close()
                continue
        if mode == D.MODE_P2P:
            # round 2: the victim stops arriving after its first barrier (mid-reduce)
            before = state(e)
            epoch0 = e.scalars().outer_epoch
            if not me_alive:
                coll.inject_stall(1)
            try:
                e.outer_step(coll, wait=True, report=True)
                raise AssertionError(f"{tag}: the round with a stalled peer succeeded")
            except D.CollectiveError:
                pass
            assert e.scalars().outer_epoch == epoch0, tag
            assert same(state(e), before), (tag, "a failed round changed the engine state")
            out["checks"].append(f"{tag}: failed round leaves state unchanged")
        if not me_alive:
            try:
                coll.shrink([victim])
                raise AssertionError("victim shrank itself in")
            except D.CollectiveError as x:
                assert "excluded from round" in str(x)
            out["checks"].append(f"{tag}: victim excluded")
            e.close()
            coll.close()
            continue
        try:
            coll.shrink([victim], quorum_min=k)
            raise AssertionError("quorum not enforced")
        except D.QuorumError:
            pass
        sub = coll.shrink([victim], quorum_min=k - 1)
        assert sub.world_size() == k - 1 and sub.members() == survivors, (tag, sub.members())
        assert sub.rank() == survivors.index(r.rank)
        # retry of the same epoch over the survivors
        res = e.outer_step(sub, wait=True, report=True)
        sw = [ws[j] for j in survivors]
        DR.outer_round(port, sw, prec, hyper)
        assert res.applied and res.report.contributors == k - 1, tag
        assert res.report.attempts == (2 if mode == D.MODE_P2P else 1), (tag, res.report.attempts)
        close(e, ws[r.rank], mode, (tag, "survivor round"))
        # one more round on the shrunk fleet
        inner(survivors)
        res = e.outer_step(sub, wait=True, report=True)
        DR.outer_round(port, sw, prec, hyper)
        assert res.applied and res.report.contributors == k - 1 and res.report.attempts == 1, tag
        close(e, ws[r.rank], mode, (tag, "round 3"))
        out["checks"].append(f"{tag}: survivors {survivors} bitwise" if mode != D.MODE_ALLREDUCE
                             else f"{tag}: survivors {survivors} within 1e-5")
        e.close()
        sub.close()
        coll.close()
    PD.barrier(r.world)
    print("MPRESULT " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
