"""In-process K-worker DiLoCo driver over an oracle library (TEST INFRASTRUCTURE).

Restates the reference's in-process loop ``run_simulated``
(/root/reference/proj/src/netsim.cpp:242-388: K x H inner steps, K pseudo-
gradients, one ``reduce_average``, K outer steps) and ``apply_inner_step``
(engine.cpp:50-69) with the gradient producer replaced by synthetic gradients
(the task/model is out of scope).  Every arithmetic call
goes to the chosen library (reference build or C restatement), so this file
only sequences calls; it holds no math of its own.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import oracle as O


@dataclass
class Hyper:
    """OptimHyperparams defaults, engine.hpp:34-46."""
    inner_lr: float = 4e-4
    warmup_steps: int = 1000
    total_steps: int = 0
    cosine: bool = False
    weight_decay: float = 0.1
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    outer_lr: float = 0.7
    outer_momentum: float = 0.9
    scale: float = 65536.0
    growth_interval: int = 2000


@dataclass
class Worker:
    """EngineState, engine.hpp:48-56 (task cursor omitted)."""
    theta_t: np.ndarray
    theta_local: np.ndarray
    m: np.ndarray
    v: np.ndarray
    buf: np.ndarray
    step_count: int = 0
    scale: float = 65536.0
    good: int = 0
    outer_epoch: int = 0
    skipped: list = field(default_factory=list)


def make_workers(theta0: np.ndarray, k: int, hyper: Hyper):
    """Replicas start identical (engine.cpp:80-81)."""
    z = lambda: np.zeros_like(theta0)  # noqa: E731
    return [Worker(theta0.copy(), theta0.copy(), z(), z(), z(), scale=hyper.scale) for _ in range(k)]


def inner_step(lib, w: Worker, grad: np.ndarray, hyper: Hyper) -> bool:
    """apply_inner_step (engine.cpp:50-69) given the raw gradient.

    Returns True when the step was skipped for overflow."""
    scaled = (grad.astype(np.float32) * np.float32(w.scale)).astype(np.float32)  # engine.cpp:24
    unscaled, overflow = lib.scaler_unscale_and_check(w.scale, scaled)
    if not overflow:
        lr = lib.lr_at(hyper.warmup_steps, hyper.total_steps, hyper.inner_lr, hyper.cosine,
                       w.step_count + 1)
        st, p, w.step_count = lib.adamw_step(w.theta_local, unscaled, w.m, w.v, w.step_count, lr,
                                             hyper.beta1, hyper.beta2, hyper.eps, hyper.weight_decay)
        assert st == O.OK, st
        w.theta_local = p
    w.scale, w.good = lib.scaler_update(w.scale, w.good, hyper.growth_interval, overflow)
    w.skipped.append(bool(overflow))
    return bool(overflow)


def outer_round(lib, workers, precision: int, hyper: Hyper):
    """Pseudo-gradients -> reduce_average -> outer_step on every worker
    (netsim.cpp:325-357; engine.cpp:115-146).  Returns (dbar, applied)."""
    deltas = [lib.axpy(-1.0, w.theta_local, w.theta_t) for w in workers]  # engine.cpp:122
    st, dbar = lib.reduce_average(deltas, precision)
    assert st == O.OK, st
    applied = lib.all_finite(dbar)  # engine.cpp:136
    for w in workers:
        if applied:
            st, w.theta_t = lib.nesterov_step(w.theta_t, dbar, w.buf, hyper.outer_lr,
                                              hyper.outer_momentum)
            assert st == O.OK
        w.theta_local = w.theta_t.copy()  # engine.cpp:143
        w.outer_epoch += 1
    return dbar, applied, deltas


def simulate(lib, theta0, grad_fn, k: int, h: int, rounds: int, precision: int, hyper: Hyper):
    """grad_fn(worker, global_inner_step) -> raw FP32 gradient."""
    workers = make_workers(theta0, k, hyper)
    history = []
    step = 0
    for _ in range(rounds):
        for _t in range(h):
            for wi, w in enumerate(workers):
                inner_step(lib, w, grad_fn(wi, step), hyper)
            step += 1
        history.append(outer_round(lib, workers, precision, hyper))
    return workers, history
