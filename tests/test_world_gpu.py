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
              nonfinite_round=None):
    """K workers, `rounds` windows of H inner steps: the GPU world vs the oracle.
    overflow=(w, t): grad[5] = inf for worker w at global step t (that worker's
    inner step is skipped).  nonfinite_round: a non-finite theta_local on the
    last worker before that round's outer step (every rank skips it)."""
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(seed, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(seed, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == overflow:
            g[5] = np.inf
        return g

    world = D.World(D.DilocoConfig(h, k, prec, h * rounds), hp, n, devices, mode=mode)
    for e in world.engines:
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


@pytest.mark.parametrize("k", [9, 16])
def test_world_shared_device_p2p_wide(port, k):
    """K > 8: the owner fold without a TMA instance (per-thread loads)."""
    world, ws = run_world(port, k, A.FP16, A.MODE_P2P, [0] * k, n=10_007, overflow=(0, 0))
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
