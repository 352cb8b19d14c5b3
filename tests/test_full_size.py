"""Parity at BASELINE.json's full sizes, on a B200 (configs 2-5), on EVERY element.

The GPU runs the full-size vectors; tests/chunked_oracle.py replays the oracle
chunk by chunk on the host cores and compares every element of theta_t,
theta_local, m, v and momentum of every worker, bit for bit (the reference's
whole-vector comparisons, /root/reference/proj/tests/test_engine.cpp:213-241,
test_collective.cpp:368-396).  The multi-worker cases run K ranks of a
dlc_world on cuda:0 (DLC_MODE_P2P with event synchronisation): the pipelined
pieces, the TMA owner fold and the finish gate at full size on one GPU.
"""
import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from oracle import driver as DR
from chunked_oracle import compare_whole  # tests/chunked_oracle.py

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    try:
        n = D.device_count()
    except D.Error:
        n = 0
    if n < 1:
        pytest.skip("no CUDA device")
    D.lib.dlc_set_device(0)
    D.set_p2p_tuning()


def _hp(hyper):
    return D.OptimHyperparams(inner_lr=hyper.inner_lr, warmup_steps=hyper.warmup_steps,
                              weight_decay=hyper.weight_decay, outer_lr=hyper.outer_lr,
                              outer_momentum=hyper.outer_momentum, scaler_init_scale=hyper.scale,
                              scaler_growth_interval=hyper.growth_interval)


def _oracle_chunk(port, k, h, rounds, prec, hyper, overflow):
    """The oracle's K-worker run restricted to elements [lo, lo + length): inputs
    are the same counter-based streams at element offset lo.  An overflow
    injected at (worker, step) is a global skip of that worker's step, so every
    chunk injects it."""
    from oracle import oracle as O

    def run(lo, length):
        th0 = O.rng_fill(4242, "theta", 0, length, -0.05, 0.05, first=lo)

        def grad_fn(w, t):
            g = O.rng_fill(4242, "grad", w * 1000 + t, length, -1e-2, 1e-2, first=lo)
            if (w, t) == overflow:
                g[-1] = np.inf
            return g
        ws, _ = DR.simulate(port, th0, grad_fn, k, h, rounds, prec, hyper)
        return ws
    return run


def _run_engines(engines, n, h, rounds, overflow, outer):
    for e in engines:
        e.rng_fill(A.THETA_T, 4242, "theta", 0, -0.05, 0.05)
        e.rng_fill(A.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    step = 0
    for rnd in range(rounds):
        for _ in range(h):
            for wi, e in enumerate(engines):
                e.rng_fill(A.GRAD, 4242, "grad", wi * 1000 + step, -1e-2, 1e-2)
                if (wi, step) == overflow:
                    e.upload_range(A.GRAD, n - 1, [np.inf])
                e.inner_step(e.device_ptr(A.GRAD), grad_is_scaled=False)
            step += 1
        res = outer()
        assert res.applied and res.outer_epoch == rnd + 1


@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
def test_full_size_1p1b_window(port, prec):
    """Configs 4/5 on one worker: 1.1B parameters, H = 3 inner steps (the second
    overflows at the last element: a global skip) and the fused outer step;
    all 5 x 1.1B elements compared."""
    n, h = 1_100_000_000, 3
    hyper = DR.Hyper(warmup_steps=5)
    e = D.DilocoEngine(D.DilocoConfig(h, 1, prec, h), _hp(hyper), n)
    _run_engines([e], n, h, 1, (0, 1), lambda: e.outer_step(None, wait=True))
    assert e.scalars().overflow_skips == 1
    done = compare_whole([e], n, 1 << 23, _oracle_chunk(port, 1, h, 1, prec, hyper, (0, 1)))
    assert done == 5 * n
    e.close()


@pytest.mark.parametrize("overflow_step", [1, 2])
def test_full_size_1p1b_fused_boundary(port, overflow_step):
    """One worker's window boundary as ONE pass (DilocoOptimizer::step,
    boundary_solo_kernel) at 1.1B: H = 3 with the overflow mid-window (1) or on
    the window's last step (2: the fused outer values are discarded and the
    gated pass reruns the outer step from the unchanged theta_local); all
    5 x 1.1B elements compared."""
    n, h = 1_100_000_000, 3
    hyper = DR.Hyper(warmup_steps=5)
    e = D.DilocoEngine(D.DilocoConfig(h, 1, A.FP16, h), _hp(hyper), n)
    e.rng_fill(A.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(A.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    opt = D.DilocoOptimizer(e)
    for step in range(h):
        e.rng_fill(A.GRAD, 4242, "grad", step, -1e-2, 1e-2)
        if step == overflow_step:
            e.upload_range(A.GRAD, n - 1, [np.inf])
        opt.step(e.device_ptr(A.GRAD), grad_is_scaled=False)
    assert opt.round_just_completed
    sc = e.scalars()
    assert sc.overflow_skips == 1 and sc.outer_epoch == 1 and sc.last_applied == 1
    done = compare_whole([e], n, 1 << 23, _oracle_chunk(port, 1, h, 1, A.FP16, hyper, (0, overflow_step)))
    assert done == 5 * n
    e.close()


@pytest.mark.parametrize("prec", [A.FP32, A.FP16])
def test_full_size_150m_eight_workers(port, prec):
    """Configs 2 / 3: 150M parameters x 8 workers (8 ranks of a P2P world on one
    GPU), H = 2, two rounds, an overflowed inner step on the last worker; all
    5 x 8 x 150M elements compared."""
    n, k, h, rounds = 150_000_000, 8, 2, 2
    hyper = DR.Hyper(warmup_steps=5)
    world = D.World(D.DilocoConfig(h, k, prec, h * rounds), _hp(hyper), n, [0] * k, mode=A.MODE_P2P)
    _run_engines(world.engines, n, h, rounds, (k - 1, 1), world.outer_step)
    done = compare_whole(world.engines, n, 1 << 20, _oracle_chunk(port, k, h, rounds, prec, hyper, (k - 1, 1)))
    assert done == 5 * k * n
    world.close()


def test_full_size_1p1b_two_workers(port):
    """Config 4 (1.1B, FP16 average, Nesterov 0.7 / 0.9) with two workers of a
    P2P world on one GPU (~100 GB of HBM), one window of H = 1 per round, two
    rounds; all 5 x 2 x 1.1B elements compared."""
    n, k, h, rounds = 1_100_000_000, 2, 1, 2
    hyper = DR.Hyper(warmup_steps=5)
    world = D.World(D.DilocoConfig(h, k, A.FP16, h * rounds), _hp(hyper), n, [0] * k, mode=A.MODE_P2P)
    _run_engines(world.engines, n, h, rounds, (None, None), world.outer_step)
    done = compare_whole(world.engines, n, 1 << 23, _oracle_chunk(port, k, h, rounds, A.FP16, hyper, (None, None)))
    assert done == 5 * k * n
    world.close()
