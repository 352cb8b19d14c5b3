"""Single-process world (dlc_world_*): K engines driven by one host thread, every
collective mode, against the oracle's K-worker run (bitwise for P2P / ordered,
the stated tolerance for NCCL's all-reduce).

In DLC_MODE_P2P the ranks synchronise through CUDA events, so they may share a
device: on a one-GPU box every K below runs the whole P2P data plane (piece
pipeline, TMA owner fold with its bulk copies, finish gate) with K ranks on
cuda:0.  This is the K-worker parity of the reference's Fleet tests
(/root/reference/proj/tests/test_collective.cpp:366-396: every peer bitwise equal
to reduce_average in peer order) and of run_simulated's outer round
(/root/reference/proj/src/netsim.cpp:325-357).
"""
import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from oracle import driver as DR
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def gpus():
    try:
        return D.device_count()
    except D.Error:
        return 0


@pytest.fixture(autouse=True)
def default_tuning():
    if gpus() < 1:
        pytest.skip("no CUDA device")
    D.set_p2p_tuning()
    yield
    D.set_p2p_tuning()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def run_world(port, k, prec, mode, devices, n=40_009, h=2, rounds=2, overflow=(None, None), seed=77,
              nonfinite_round=None, fused=True, inner_mode=A.INNER_PINGPONG):
    """K workers, `rounds` windows of H inner steps: the GPU world vs the oracle.
    overflow=(w, t): grad[5] = inf for worker w at global step t (that worker's
    inner step is skipped).  nonfinite_round: a non-finite theta_local on the
    last worker before that round's outer step (every rank skips it).
    fused: K2 fused into each window's last inner step (the default), else the
    outer step's own K2 pieces."""
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(seed, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(seed, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == overflow:
            g[5] = np.inf
        return g

    world = D.World(D.DilocoConfig(h, k, prec, h * rounds), hp, n, devices, mode=mode, inner_mode=inner_mode)
    for e in world.engines:
        e.set_fused_delta(fused)
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, theta0)
    ws = DR.make_workers(theta0, k, hyper)
    step = 0
    for rnd in range(rounds):
        for _ in range(h):
            for wi, e in enumerate(world.engines):
                e.inner_step_host(grad_fn(wi, step))
                DR.inner_step(port, ws[wi], grad_fn(wi, step), hyper)
            step += 1
        if nonfinite_round == rnd:
            bad = world.engines[k - 1].download(A.THETA_LOCAL)
            bad[n - 3] = np.nan
            world.engines[k - 1].upload(A.THETA_LOCAL, bad)
            ws[k - 1].theta_local = bad.copy()
        _, applied, _ = DR.outer_round(port, ws, prec, hyper)
        res = world.outer_step()
        assert res.applied == applied and res.outer_epoch == rnd + 1
    return world, ws


def check_bitwise(world, ws):
    for wi, e in enumerate(world.engines):
        w = ws[wi]
        for which, want in ((A.THETA_T, w.theta_t), (A.THETA_LOCAL, w.theta_local), (A.MOMENTUM, w.buf),
                            (A.ADAM_M, w.m), (A.ADAM_V, w.v)):
            got = e.download(which)
            assert np.array_equal(bits(got), bits(want)), (wi, which, int(np.sum(bits(got) != bits(want))))
        sc = e.scalars()
        assert sc.step_count == w.step_count and sc.outer_epoch == w.outer_epoch


# ---- K ranks sharing cuda:0 (the driver's one-GPU box) -------------------------------------

@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
@pytest.mark.parametrize("k", [2, 3, 4, 5, 8])
def test_world_shared_device_p2p(port, k, prec):
    """K = 2..8 ranks on one GPU: the TMA owner fold at KK = k, ragged N (40,009
    is not a multiple of any slot quantum), an overflowed inner step on the last
    worker, two rounds."""
    world, ws = run_world(port, k, prec, A.MODE_P2P, [0] * k, overflow=(k - 1, 1))
    check_bitwise(world, ws)
    world.close()


@pytest.mark.parametrize("inner_mode", [A.INNER_PINGPONG, A.INNER_INPLACE])
@pytest.mark.parametrize("fused", [True, False, "mixed"])
@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
def test_world_fused_delta(port, prec, fused, inner_mode):
    """K2 fused into the window's last inner step (dlc_engine_set_fused_delta)
    against the unfused outer K2, and a mix of both in one fleet: H = 3, three
    rounds; worker 1 overflows on the last step of round 0 (its fused delta is
    discarded and the gated K2 recomputes it from the unchanged theta_local),
    worker 2 on the first step of round 1, and round 2 replaces worker 0's
    theta_local after its last inner step (the upload drops the fused delta).
    Both inner modes."""
    k, h, n, seed = 4, 3, 30_011, 91
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(seed, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(seed, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) in ((1, 2), (2, 3)):
            g[7] = np.inf
        return g

    world = D.World(D.DilocoConfig(h, k, prec, 3 * h), hp, n, [0] * k, mode=A.MODE_P2P, inner_mode=inner_mode)
    for i, e in enumerate(world.engines):
        e.set_fused_delta(i % 2 == 0 if fused == "mixed" else fused)
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, theta0)
    ws = DR.make_workers(theta0, k, hyper)
    step = 0
    for rnd in range(3):
        for _ in range(h):
            for wi, e in enumerate(world.engines):
                e.inner_step_host(grad_fn(wi, step))
                DR.inner_step(port, ws[wi], grad_fn(wi, step), hyper)
            step += 1
        if rnd == 2:
            moved = world.engines[0].download(A.THETA_LOCAL)
            moved[: n // 2] += np.float32(1e-3)
            world.engines[0].upload(A.THETA_LOCAL, moved)
            ws[0].theta_local = moved.copy()
        _, applied, _ = DR.outer_round(port, ws, prec, hyper)
        res = world.outer_step()
        assert res.applied == applied and res.outer_epoch == rnd + 1
    check_bitwise(world, ws)
    world.close()


@pytest.mark.parametrize("k,exclude", [(4, [2]), (8, [0, 3, 7]), (3, [0, 1])])
@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
def test_world_shrink_survivor_rounds(port, k, exclude, prec):
    """Membership change between rounds: one round over K
    ranks, then the world drops `exclude` and runs two rounds over the
    survivors, bitwise against the oracle's outer round over the survivors in
    order with divisor K' (collective.cpp:1369-1395; test_collective.cpp:460-531
    "survivor mean").  Below-quorum, out-of-range and mid-window shrinks raise
    and change nothing."""
    n, h, seed = 20_011, 2, 13
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(seed, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(seed, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == (k - 1, 5):
            g[3] = np.inf
        return g

    world = D.World(D.DilocoConfig(h, k, prec, 3 * h), hp, n, [0] * k, mode=A.MODE_P2P)
    for e in world.engines:
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, theta0)
    ws = DR.make_workers(theta0, k, hyper)
    alive = list(range(k))
    step = 0
    for rnd in range(3):
        if rnd == 1:
            with pytest.raises(D.QuorumError):
                world.shrink(list(range(k)), quorum_min=1)
            with pytest.raises(D.ConfigError):
                world.shrink([k])
            survivors = [r for r in alive if r not in exclude]
            with pytest.raises(D.QuorumError):
                world.shrink(exclude, quorum_min=len(survivors) + 1)
            world.shrink(exclude)
            alive = survivors
            assert world.members() == alive
        for _ in range(h):
            for idx, w in enumerate(alive):
                world.engines[idx].inner_step_host(grad_fn(w, step))
                DR.inner_step(port, ws[w], grad_fn(w, step), hyper)
            step += 1
            if rnd == 2 and step % h == 1:
                with pytest.raises(D.Error):
                    world.shrink([0])  # mid-window
        _, applied, _ = DR.outer_round(port, [ws[w] for w in alive], prec, hyper)
        res = world.outer_step()
        assert res.applied == applied and res.outer_epoch == rnd + 1
    check_bitwise(world, [ws[w] for w in alive])
    world.close()


@pytest.mark.parametrize("mode", [A.MODE_ORDERED, A.MODE_ALLREDUCE, A.MODE_P2P])
def test_world_shrink_one_rank_per_gpu(port, mode):
    """dlc_world_shrink with one rank per GPU: the NCCL worlds get fresh
    communicators over the survivors' devices, the P2P world re-binds its peer
    tables; one round over 3 ranks, then two over ranks 0 and 2 (ordered and
    P2P bitwise, all-reduce within its tolerance)."""
    if gpus() < 3:
        pytest.skip("needs 3 GPUs")
    n, h, seed, k = 30_011, 2, 19, 3
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(seed, "theta", 0, n, -0.05, 0.05)
    world = D.World(D.DilocoConfig(h, k, A.FP16, 3 * h), hp, n, [0, 1, 2], mode=mode)
    for e in world.engines:
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, theta0)
    ws = DR.make_workers(theta0, k, hyper)
    alive, step = [0, 1, 2], 0
    for rnd in range(3):
        if rnd == 1:
            world.shrink([1])
            alive = [0, 2]
            assert world.members() == alive
        for _ in range(h):
            for idx, w in enumerate(alive):
                g = O.rng_fill(seed, "grad", w * 1000 + step, n, -1e-2, 1e-2)
                world.engines[idx].inner_step_host(g)
                DR.inner_step(port, ws[w], g, hyper)
            step += 1
        DR.outer_round(port, [ws[w] for w in alive], A.FP16, hyper)
        res = world.outer_step()
        assert res.applied and res.outer_epoch == rnd + 1
    if mode != A.MODE_ALLREDUCE:
        check_bitwise(world, [ws[w] for w in alive])
    else:
        for idx, w in enumerate(alive):
            got = world.engines[idx].download(A.THETA_T)
            assert np.max(np.abs(got - ws[w].theta_t)) <= 1e-3
    world.close()


@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
@pytest.mark.parametrize("k", [9, 16])
def test_world_shared_device_p2p_wide(port, k, prec):
    """K > 8: the owner fold without a TMA instance (per-thread loads)."""
    world, ws = run_world(port, k, prec, A.MODE_P2P, [0] * k, n=10_007, overflow=(0, 0))
    check_bitwise(world, ws)
    world.close()


@pytest.mark.parametrize("n", [1, 7, 511, 4 * 512 + 3])
def test_world_shared_device_tiny(port, n):
    """N below the slot quantum: most owner slots are padding (and N < K)."""
    world, ws = run_world(port, 8, A.FP16, A.MODE_P2P, [0] * 8, n=n, h=1, rounds=2)
    check_bitwise(world, ws)
    world.close()


@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
def test_world_shared_device_nonfinite_skip(port, prec):
    """A non-finite pseudo-gradient on one worker: the mean is non-finite, every
    rank skips Nesterov but still refreshes theta_local (engine.cpp:136-144)."""
    world, ws = run_world(port, 4, prec, A.MODE_P2P, [0] * 4, rounds=3, nonfinite_round=1)
    check_bitwise(world, ws)
    world.close()


@pytest.mark.parametrize("tuning", [dict(plan=[2, 2, 2, 2]), dict(plan=[1, 3, 4], fold_ctas=3),
                                    dict(fold_threads=512, piece_ctas=37), dict(plan=[1] * 16, fold_ctas=1),
                                    dict(fold_kernel=1), dict(fold_kernel=1, fold_threads=256, fold_ctas=5)])
def test_world_shared_device_tuning(port, tuning):
    """The tuning overrides change the schedule, never the bits."""
    D.set_p2p_tuning(**tuning)
    world, ws = run_world(port, 4, A.FP16, A.MODE_P2P, [0] * 4, overflow=(2, 0))
    check_bitwise(world, ws)
    world.close()


def test_world_shared_device_nccl_modes_rejected():
    with pytest.raises(D.Error):
        D.World(D.DilocoConfig(1, 2, A.FP16, 1), D.OptimHyperparams(), 1000, [0, 0], mode=A.MODE_ORDERED)


# ---- one rank per GPU (every mode) -----------------------------------------------------------

@pytest.mark.parametrize("mode", [A.MODE_P2P, A.MODE_ORDERED, A.MODE_ALLREDUCE])
@pytest.mark.parametrize("k,prec", [(2, A.FP16), (2, A.FP32), (3, A.FP16), (4, A.FP16)])
def test_world_matches_oracle(port, mode, k, prec):
    if gpus() < k:
        pytest.skip(f"needs {k} GPUs")
    world, ws = run_world(port, k, prec, mode, list(range(k)), overflow=(k - 1, 1))
    if mode != A.MODE_ALLREDUCE:
        check_bitwise(world, ws)
    else:  # NCCL's reduction order: every worker identical, close to the reference
        t0 = world.engines[0].download(A.THETA_T)
        for wi, e in enumerate(world.engines):
            got_t = e.download(A.THETA_T)
            assert np.array_equal(bits(got_t), bits(t0))
            assert np.max(np.abs(got_t - ws[wi].theta_t)) <= 1e-3
    world.close()


@pytest.mark.parametrize("k", [4, 8])
def test_world_mixed_devices_p2p(port, k):
    """Ranks spread over the available GPUs round-robin (several per GPU): event
    dependencies across devices and within one."""
    g = gpus()
    if g < 2:
        pytest.skip("needs 2 GPUs")
    world, ws = run_world(port, k, A.FP16, A.MODE_P2P, [i % g for i in range(k)], overflow=(1, 2))
    check_bitwise(world, ws)
    world.close()
