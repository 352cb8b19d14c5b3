"""One rank of the multi-GPU parity test (launched by tests/test_multigpu.py via torchrun).

Every rank drives one GPU as one DiLoCo worker; the collective is the NCCL
communicator inside libdiloco_cuda.so.  Each rank replays the whole K-worker
run on the CPU oracle and checks its own worker:
  * ordered mode: bit-exact (theta_t, theta_local, m, v, momentum);
  * allreduce mode (NCCL's own reduction order): theta_t within
    lr*(1+mu)*tol(dbar) + 2 ulp, tol(dbar) = K*2^-24*max|delta| (FP32) or
    2^-10*max|delta| + 2^-24 (FP16), SPEC.md:325 / test_engine.cpp:311-323.
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


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def main():
    r = PD.init("gloo")
    D.lib.dlc_set_device(r.local)
    k = r.world
    out = {"rank": r.rank, "checks": []}
    port = O.port()
    n, h, rounds = 50_021, 3, 2
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(4242, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(4242, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == (k - 1, 1):
            g[3] = np.inf  # one overflowed inner step on the last worker
        return g

    # P2P with the measured defaults and with a few tuning overrides (piece
    # plan, a tiny fold grid, 512-thread fold CTAs)
    cases = [("ordered", D.MODE_ORDERED, {}), ("p2p", D.MODE_P2P, {}),
             ("p2p-plan2222", D.MODE_P2P, {"plan": [2, 2, 2, 2]}),
             ("p2p-plan134-tma3", D.MODE_P2P, {"plan": [1, 3, 4], "fold_ctas": 3}),
             ("p2p-tma512", D.MODE_P2P, {"fold_threads": 512, "piece_ctas": 37}),
             ("allreduce", D.MODE_ALLREDUCE, {})]
    for mode_name, mode, tuning in cases:
        D.set_p2p_tuning(**tuning)
        coll = PD.make_nccl_collective(r, mode)
        assert coll.world_size() == k and coll.rank() == r.rank
        for prec in (D.FP32, D.FP16):
            workers, hist = DR.simulate(port, theta0, grad_fn, k, h, rounds, prec, hyper)
            cfg = D.DilocoConfig(h, k, prec, h * rounds)
            hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
            e = D.DilocoEngine(cfg, hp, n, r.local)
            e.upload(D.THETA_T, theta0)
            e.upload(D.THETA_LOCAL, theta0)
            step = 0
            for _ in range(rounds):
                for _t in range(h):
                    e.inner_step_host(grad_fn(r.rank, step), grad_is_scaled=False)
                    step += 1
                res = e.outer_step(coll, wait=True, report=True)
                assert res.applied
                rep = res.report
                # the reference's byte law (reduce.cpp:91-104); wire = the padded slots moved
                assert rep.contributors == k and rep.data_bytes_sent == D.per_peer_reduce_bytes(n, k, r.rank, prec)
                assert rep.wire_bytes_sent == 2 * (k - 1) * PD.slot_elems(n, k) * (2 if prec == D.FP16 else 4)
                assert all_sum(r, rep.data_bytes_sent) == D.fleet_reduce_bytes(n, k, prec)
                assert all_sum(r, rep.data_bytes_received) == D.fleet_reduce_bytes(n, k, prec)
            me = workers[r.rank]
            got = {w: e.download(w) for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM)}
            if mode != D.MODE_ALLREDUCE:
                for w, want in ((D.THETA_T, me.theta_t), (D.THETA_LOCAL, me.theta_local), (D.ADAM_M, me.m),
                                (D.ADAM_V, me.v), (D.MOMENTUM, me.buf)):
                    assert np.array_equal(bits(got[w]), bits(want)), (mode_name, prec, w)
                out["checks"].append(f"{mode_name}/{'fp16' if prec else 'fp32'}: bitwise")
            else:
                # first round only: later rounds compound through AdamW's nonlinearity
                deltas = hist[0][2]
                mx = np.max(np.abs(np.stack(deltas)), axis=0).astype(np.float64)
                tol_d = (k * 2.0 ** -24 * mx) if prec == D.FP32 else (2.0 ** -10 * mx + 2.0 ** -24)
                e1 = D.DilocoEngine(D.DilocoConfig(1, k, prec, 1), hp, n, r.local)
                e1.upload(D.THETA_T, theta0)
                loc = workers_round0_local(port, theta0, grad_fn, k, h, hyper, r.rank)
                e1.upload(D.THETA_LOCAL, loc)
                e1.outer_step(coll, wait=True)
                got_t = e1.download(D.THETA_T).astype(np.float64)
                w0, _ = DR.simulate(port, theta0, grad_fn, k, h, 1, prec, hyper)
                want_t = w0[r.rank].theta_t.astype(np.float64)
                tol = 0.7 * 1.9 * tol_d + 2 * np.spacing(np.abs(want_t).astype(np.float32)).astype(np.float64)
                err = np.abs(got_t - want_t)
                assert np.all(err <= tol), (mode_name, prec, float(np.max(err / tol)))
                out["checks"].append(f"{mode_name}/{'fp16' if prec else 'fp32'}: max err/tol "
                                     f"{float(np.max(err / tol)):.3f}")
                e1.close()
            e.close()
        if mode_name == "p2p":  # run_training (engine.cpp:176-240) over this collective
            workers, _ = DR.simulate(port, theta0, grad_fn, k, h, rounds, D.FP16, hyper)
            e = D.DilocoEngine(D.DilocoConfig(h, k, D.FP16, h * rounds),
                               D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2), n, r.local)
            e.upload(D.THETA_T, theta0)
            e.upload(D.THETA_LOCAL, theta0)
            gptr = e.device_ptr(D.GRAD)

            def producer(step, e=e, gptr=gptr):
                e.upload(D.GRAD, grad_fn(r.rank, step))
                return gptr, False, 1.0

            recs = []
            res = D.run_training(e, coll, producer, sink=recs.append, worker_index=r.rank)
            # ledger (test_harness.cpp:121-133): the fleet's bytes = rounds x fleet_reduce_bytes
            assert res["rounds_done"] == rounds
            assert res["reduce_data_bytes"] == rounds * D.per_peer_reduce_bytes(n, k, r.rank, D.FP16)
            assert all_sum(r, res["reduce_data_bytes"]) == rounds * D.fleet_reduce_bytes(n, k, D.FP16)
            assert sum(1 for x in recs if x["kind"] == "round" and x["contributors"] == k) == rounds
            for w, want in ((D.THETA_T, workers[r.rank].theta_t), (D.MOMENTUM, workers[r.rank].buf)):
                assert np.array_equal(bits(e.download(w)), bits(want)), ("run_training", w)
            e.close()
            out["checks"].append("run_training over p2p: bitwise")
        # e2e host-buffer outer step (dlc_engine_outer_step_host) vs the oracle's outer round
        for prec, n2 in ((D.FP32, 20_011), (D.FP16, 20_011), (D.FP16, 5), (D.FP32, 1)):  # tiny: N < K slots
            th = O.rng_fill(5, "theta", 0, n2, -1, 1)
            locs = [(th - O.rng_fill(5, "local", j, n2, -1e-3, 1e-3)).astype(np.float32) for j in range(k)]
            e2 = D.DilocoEngine(D.DilocoConfig(1, k, prec, 1), D.OptimHyperparams(), n2, r.local)
            e2.upload(D.THETA_T, th)
            out_t = np.empty(n2, np.float32)
            res = e2.outer_step_host(coll, locs[r.rank], out_t)
            assert res.applied
            ws = DR.make_workers(th, k, hyper)
            for j, w in enumerate(ws):
                w.theta_local = locs[j].copy()
            DR.outer_round(port, ws, prec, hyper)
            if mode != D.MODE_ALLREDUCE:
                assert np.array_equal(bits(out_t), bits(ws[r.rank].theta_t)), (mode_name, prec)
            else:
                assert np.max(np.abs(out_t - ws[r.rank].theta_t)) <= 1e-3
            e2.close()
        # e2e host path with a non-finite delta on the last rank: the step is skipped
        # everywhere and the returned theta_t is the unchanged one (engine.cpp:136-144)
        n2 = 30_001
        th = O.rng_fill(6, "theta", 0, n2, -1, 1)
        loc = (th - O.rng_fill(6, "local", r.rank, n2, -1e-3, 1e-3)).astype(np.float32)
        if r.rank == k - 1:
            loc[n2 // 2] = np.inf  # in another owner's slot
            own = (k - 1) * PD.slot_elems(n2, k) + 7  # in this rank's own slot (folded locally)
            if own < n2:
                loc[own] = -np.inf
        e2 = D.DilocoEngine(D.DilocoConfig(1, k, D.FP16, 1), D.OptimHyperparams(), n2, r.local)
        e2.upload(D.THETA_T, th)
        out_t = np.full(n2, np.nan, np.float32)
        res = e2.outer_step_host(coll, loc, out_t)
        assert not res.applied and res.outer_epoch == 1, (mode_name, res)
        assert np.array_equal(bits(out_t), bits(th)), mode_name
        e2.close()
        # host-buffer plugin call (Collective::all_reduce_avg) vs reduce_average in rank order
        for prec in (D.FP32, D.FP16):
            deltas = [O.rng_fill(9, "delta", j, 10_007, -1, 1) for j in range(k)]
            got, rep = coll.all_reduce_avg(deltas[r.rank], prec, outer_epoch=3)
            _, want = port.reduce_average(deltas, prec)
            if mode != D.MODE_ALLREDUCE:
                assert np.array_equal(bits(got), bits(want))
            else:
                assert np.max(np.abs(got - want)) <= (2.0 ** -10 if prec else k * 2.0 ** -23)
            assert rep.contributors == k and rep.outer_epoch == 3
            assert rep.data_bytes_sent == D.per_peer_reduce_bytes(10_007, k, r.rank, prec)
        # linearity (test_collective.cpp:398-419) and the byte law: FP16 halves the bytes (:421-458)
        x = O.rng_fill(10, "x", r.rank, 4099, -1, 1)
        y = O.rng_fill(10, "y", r.rank, 4099, -1, 1)
        ax, rx = coll.all_reduce_avg(x, D.FP32)
        ay, _ = coll.all_reduce_avg(y, D.FP32)
        axy, _ = coll.all_reduce_avg((x + y).astype(np.float32), D.FP32)
        assert np.max(np.abs((ax + ay) - axy)) <= 1e-6 * max(1.0, float(np.max(np.abs(axy))))
        _, r16 = coll.all_reduce_avg(x, D.FP16)
        assert 2 * r16.data_bytes_sent == rx.data_bytes_sent
        coll.close()
    D.set_p2p_tuning()
    PD.barrier(r.world)
    print("MPRESULT " + json.dumps(out), flush=True)


def all_sum(r, x: int) -> int:
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(x)], dtype=torch.int64)
    dist.all_reduce(t)
    return int(t.item())


def workers_round0_local(port, theta0, grad_fn, k, h, hyper, rank):
    ws = DR.make_workers(theta0, k, hyper)
    for t in range(h):
        for wi, w in enumerate(ws):
            DR.inner_step(port, w, grad_fn(wi, t), hyper)
    return ws[rank].theta_local


if __name__ == "__main__":
    main()
