"""Single-process multi-GPU world (dlc_world_*): K engines on K GPUs driven by
one host thread, every collective mode, against the oracle's K-worker run
(bitwise for P2P / ordered, the stated tolerance for NCCL's all-reduce)."""
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


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("mode", [A.MODE_P2P, A.MODE_ORDERED, A.MODE_ALLREDUCE])
@pytest.mark.parametrize("k,prec", [(2, A.FP16), (2, A.FP32), (3, A.FP16), (4, A.FP16)])
def test_world_matches_oracle(port, mode, k, prec):
    if gpus() < k:
        pytest.skip(f"needs {k} GPUs")
    n, h, rounds = 40_009, 2, 2
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(77, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(77, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == (k - 1, 1):
            g[5] = np.inf
        return g

    world = D.World(D.DilocoConfig(h, k, prec, h * rounds), hp, n, list(range(k)), mode=mode)
    for e in world.engines:
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, theta0)
    step = 0
    for rnd in range(rounds):
        for _ in range(h):
            for wi, e in enumerate(world.engines):
                e.inner_step_host(grad_fn(wi, step))
            step += 1
        res = world.outer_step()
        assert res.applied and res.outer_epoch == rnd + 1
    workers, hist = DR.simulate(port, theta0, grad_fn, k, h, rounds, prec, hyper)
    for wi, e in enumerate(world.engines):
        w = workers[wi]
        got_t = e.download(A.THETA_T)
        if mode != A.MODE_ALLREDUCE:
            for which, want in ((A.THETA_T, w.theta_t), (A.THETA_LOCAL, w.theta_local), (A.MOMENTUM, w.buf),
                                (A.ADAM_M, w.m), (A.ADAM_V, w.v)):
                assert np.array_equal(bits(e.download(which)), bits(want)), (wi, which)
        else:  # NCCL's reduction order: every worker identical, close to the reference
            assert np.array_equal(bits(got_t), bits(world.engines[0].download(A.THETA_T)))
            assert np.max(np.abs(got_t - w.theta_t)) <= 1e-3
    world.close()

