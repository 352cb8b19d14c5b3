"""Parity at BASELINE.json's full sizes, on a B200 (configs 2-5).

Every operation on the path is elementwise apart from the rank-ordered fold,
which is elementwise across workers, so any slice of a full-size run is
computed exactly by the CPU oracle from the same counter-based inputs restricted
to that slice (rng streams are addressable by element).  These
tests run the full-size vectors on the GPU and check slices at the start,
middle (unaligned) and end of every state vector, bit for bit; the 1.1B
multi-GPU case is tests/mp_full_worker.py via tests/test_multigpu.py.
"""
import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from oracle import driver as DR
from oracle import oracle as O

pytestmark = pytest.mark.gpu
M = 4096  # slice length


@pytest.fixture(scope="module", autouse=True)
def gpu():
    try:
        n = D.device_count()
    except D.Error:
        n = 0
    if n < 1:
        pytest.skip("no CUDA device")
    D.lib.dlc_set_device(0)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def slices(n):
    return [0, n // 2 - 777, n - M]


def _hp(hyper):
    return D.OptimHyperparams(inner_lr=hyper.inner_lr, warmup_steps=hyper.warmup_steps,
                              weight_decay=hyper.weight_decay, outer_lr=hyper.outer_lr,
                              outer_momentum=hyper.outer_momentum, scaler_init_scale=hyper.scale,
                              scaler_growth_interval=hyper.growth_interval)


def _check_slices(e, n, ws, wi=0):
    for lo in slices(n):
        w = ws[lo][wi]
        for which, want in ((A.THETA_T, w.theta_t), (A.THETA_LOCAL, w.theta_local), (A.ADAM_M, w.m),
                            (A.ADAM_V, w.v), (A.MOMENTUM, w.buf)):
            got = e.download_range(which, lo, M)
            assert np.array_equal(bits(got), bits(want)), (lo, which)


@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
def test_full_size_1p1b_window(port, prec):
    """Config 4/5 shape on one worker: 1.1B parameters, H = 3 inner steps (the
    second with an injected overflow at the last element) and the fused outer step."""
    n, h = 1_100_000_000, 3
    hyper = DR.Hyper(warmup_steps=5)
    e = D.DilocoEngine(D.DilocoConfig(h, 1, prec, h), _hp(hyper), n)
    e.rng_fill(A.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(A.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    for t in range(h):
        e.rng_fill(A.GRAD, 4242, "grad", t, -1e-2, 1e-2)
        if t == 1:
            e.upload_range(A.GRAD, n - 1, [np.inf])
        e.inner_step(e.device_ptr(A.GRAD), grad_is_scaled=False)
    assert e.scalars().overflow_skips == 1
    assert e.outer_step(None, wait=True).applied
    ws = {}
    for lo in slices(n):
        th0 = O.rng_fill(4242, "theta", 0, M, -0.05, 0.05, first=lo)

        def grad_fn(w, t, lo=lo):
            g = O.rng_fill(4242, "grad", t, M, -1e-2, 1e-2, first=lo)
            if t == 1:  # the overflow is global: step 1 is skipped in every slice
                g[-1] = np.inf
            return g
        ws[lo], _ = DR.simulate(port, th0, grad_fn, 1, h, 1, prec, hyper)
    _check_slices(e, n, ws)
    e.close()


@pytest.mark.parametrize("prec", [A.FP32, A.FP16])
def test_full_size_150m_eight_workers(port, prec):
    """Configs 2 / 3: 150M parameters, 8 workers (in-process fleet on one GPU),
    H = 2, one outer step with the rank-ordered fold over all 8."""
    n, k, h = 150_000_000, 8, 2
    hyper = DR.Hyper(warmup_steps=5)
    engines = [D.DilocoEngine(D.DilocoConfig(h, k, prec, h), _hp(hyper), n) for _ in range(k)]
    for wi, e in enumerate(engines):
        e.rng_fill(A.THETA_T, 4242, "theta", 0, -0.05, 0.05)
        e.rng_fill(A.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    for t in range(h):
        for wi, e in enumerate(engines):
            e.rng_fill(A.GRAD, 4242, "grad", wi * 1000 + t, -1e-2, 1e-2)
            e.inner_step(e.device_ptr(A.GRAD), grad_is_scaled=False)
    assert D.outer_step_local(engines).applied
    ws = {}
    for lo in slices(n):
        th0 = O.rng_fill(4242, "theta", 0, M, -0.05, 0.05, first=lo)
        grad_fn = lambda w, t, lo=lo: O.rng_fill(4242, "grad", w * 1000 + t, M, -1e-2, 1e-2, first=lo)  # noqa: E731
        ws[lo], _ = DR.simulate(port, th0, grad_fn, k, h, 1, prec, hyper)
    for wi, e in enumerate(engines):
        _check_slices(e, n, ws, wi)
    for e in engines:
        e.close()
