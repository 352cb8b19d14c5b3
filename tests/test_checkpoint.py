"""Checkpoint / resume in the reference's ODLCKPT1 format.

CPU: the committed fixture tests/golden/engine.ckpt (written by the reference's
save_checkpoint) reads back through the reference's load_checkpoint.
GPU: device engines load that file, write byte-identical files, and resume
bit-for-bit (test_harness.cpp:197-222 style).
"""
import os

import numpy as np
import pytest

from oracle import driver as DR
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_reference_reads_golden_checkpoint(ref):
    z = np.load(os.path.join(GOLD, "engine_ckpt.npz"))
    got = ref.checkpoint_read(os.path.join(GOLD, "engine.ckpt"), 0, z["theta_t"].size)
    for k in ("theta_t", "theta_local", "m", "v", "buf"):
        assert np.array_equal(bits(got[k]), bits(z[k]))
    for k in ("step_count", "inner_step", "outer_epoch", "consecutive_good", "config_hash", "completed_rounds"):
        assert got[k] == int(z[k])
    assert got["scale"] == float(z["scale"]) and got["engines"] == 1


@pytest.fixture
def gpu():
    import paper_2407_07852_b200 as D
    try:
        n = D.device_count()
    except D.Error:
        n = 0
    if n < 1:
        pytest.skip("no CUDA device")
    D.lib.dlc_set_device(0)
    return D


@pytest.mark.gpu
def test_engine_loads_and_rewrites_reference_checkpoint(gpu, tmp_path):
    D = gpu
    z = np.load(os.path.join(GOLD, "engine_ckpt.npz"))
    n = z["theta_t"].size
    e = D.DilocoEngine(D.DilocoConfig(10, 1, D.FP16, 100), D.OptimHyperparams(), n)
    meta = D.checkpoint_load([e], os.path.join(GOLD, "engine.ckpt"))
    assert meta["config_hash"] == 0xC0FFEE and meta["completed_rounds"] == 3
    for which, k in ((D.THETA_T, "theta_t"), (D.THETA_LOCAL, "theta_local"), (D.ADAM_M, "m"), (D.ADAM_V, "v"),
                     (D.MOMENTUM, "buf")):
        assert np.array_equal(bits(e.download(which)), bits(z[k]))
    s = e.scalars()
    assert (s.step_count, s.inner_step, s.outer_epoch, s.consecutive_good) == (17, 20, 4, 5)
    assert s.scale == 32768.0
    out = str(tmp_path / "rewrite.ckpt")
    D.checkpoint_save([e], out, config_hash=0xC0FFEE, completed_rounds=3, clock_seconds=1.25,
                      reduce_data_bytes=123456)
    with open(out, "rb") as a, open(os.path.join(GOLD, "engine.ckpt"), "rb") as b:
        assert a.read() == b.read()  # byte-identical to the reference's writer
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("segments", [None, [("w", 60_000), ("b", 5_011)]])
def test_resume_is_bitwise(gpu, tmp_path, segments):
    """Save mid-run, restore into a fresh engine, continue both: identical trajectories,
    and the reference's load_checkpoint reads the engine's file."""
    D = gpu
    n = 65_011
    hyper = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=3)
    cfg = D.DilocoConfig(2, 1, D.FP16, 12)
    a = D.DilocoEngine(cfg, hyper, n)
    th = O.rng_fill(1, "theta", 0, n, -0.1, 0.1)
    a.upload(D.THETA_T, th)
    a.upload(D.THETA_LOCAL, th)
    grads = [O.rng_fill(1, "grad", t, n, -1e-2, 1e-2) for t in range(12)]
    for t in range(6):
        a.inner_step_host(grads[t])
        if (t + 1) % 2 == 0:
            a.outer_step(None)
    path = str(tmp_path / "mid.ckpt")
    D.checkpoint_save([a], path, completed_rounds=3, segments=segments)
    b = D.DilocoEngine(cfg, hyper, n)
    D.checkpoint_load([b], path)
    for t in range(6, 12):
        for e in (a, b):
            e.inner_step_host(grads[t])
            if (t + 1) % 2 == 0:
                e.outer_step(None)
    for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM):
        assert np.array_equal(bits(a.download(w)), bits(b.download(w)))
    r = O.reference()
    if r is not None:
        got = r.checkpoint_read(path, 0, n)
        assert got["step_count"] == 6 and got["outer_epoch"] == 3 and got["inner_step"] == 6
    with pytest.raises(D.ShapeError):
        D.checkpoint_load([D.DilocoEngine(cfg, hyper, n + 1)], path)
    # SerializationError like checkpoint.cpp:45,60,170: truncated file, bad magic
    raw = open(path, "rb").read()
    bad = path + ".bad"
    for blob in (raw[: len(raw) // 2], b"XXXXXXXX" + raw[8:]):
        with open(bad, "wb") as f:
            f.write(blob)
        with pytest.raises(D.SerializationError):
            D.checkpoint_load([D.DilocoEngine(cfg, hyper, n)], bad)
    a.close()
    b.close()


@pytest.mark.gpu
def test_failed_load_changes_nothing(gpu, tmp_path):
    """load is all or nothing (the reference parses the whole file before any
    restore_state, checkpoint.cpp:162-198): a file whose SECOND engine is
    truncated, one with a bad number in a header, and one whose layout differs
    from the caller's all fail, and both engines keep their state, counters
    and hyperparameters bit for bit (checked by continuing them against twins
    that never saw the failed loads)."""
    D = gpu
    n = 30_011
    hyper = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=3)
    cfg = D.DilocoConfig(2, 1, D.FP16, 8)

    def make(seed):
        e = D.DilocoEngine(cfg, hyper, n)
        th = O.rng_fill(seed, "theta", 0, n, -0.1, 0.1)
        e.upload(D.THETA_T, th)
        e.upload(D.THETA_LOCAL, th)
        for t in range(2):
            e.inner_step_host(O.rng_fill(seed, "grad", t, n, -1e-2, 1e-2))
        e.outer_step(None)
        return e

    # a valid 2-engine file with other state and other hyperparameters
    other = [D.DilocoEngine(cfg, D.OptimHyperparams(outer_lr=0.3, weight_decay=0.0), n) for _ in range(2)]
    for j, e in enumerate(other):
        e.upload(D.THETA_T, O.rng_fill(50 + j, "theta", 0, n, -1, 1))
    good = str(tmp_path / "two.ckpt")
    D.checkpoint_save(other, good, segments=[("w", n - 11), ("b", 11)])
    raw = open(good, "rb").read()
    bad_files = {"truncated_second": raw[: len(raw) - 4 * n // 2]}
    txt = raw.replace(b"scale=", b"scale=x", 1)
    bad_files["bad_number"] = txt
    engines, twins = [make(1), make(2)], [make(1), make(2)]
    for name, blob in bad_files.items():
        p = str(tmp_path / name)
        with open(p, "wb") as f:
            f.write(blob)
        with pytest.raises(D.SerializationError):
            D.checkpoint_load(engines, p)
    with pytest.raises(D.ShapeError):  # restore_state's layout check against the caller's Layout
        D.checkpoint_load(engines, good, segments=[("w", n - 12), ("b", 12)])
    for e, t in zip(engines, twins):
        for step in range(2, 4):
            for x in (e, t):
                x.inner_step_host(O.rng_fill(9, "grad", step, n, -1e-2, 1e-2))
        for x in (e, t):
            x.outer_step(None)
        for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM):
            assert np.array_equal(bits(e.download(w)), bits(t.download(w))), w
        a, b = e.scalars(), t.scalars()
        assert (a.step_count, a.inner_step, a.outer_epoch, a.scale) == (b.step_count, b.inner_step, b.outer_epoch,
                                                                          b.scale)
    # and the good file with the right layout restores both engines
    D.checkpoint_load(engines, good, segments=[("w", n - 11), ("b", 11)])
    for e, o in zip(engines, other):
        for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM):
            assert np.array_equal(bits(e.download(w)), bits(o.download(w))), w
    for e in engines + twins + other:
        e.close()


@pytest.mark.gpu
def test_checkpoint_hook_after_fused_boundary(gpu, tmp_path):
    """run_training's on_round hook (the reference's checkpoint hook,
    engine.hpp:154) after one worker's FUSED window boundary: the file holds
    the boundary's state (theta_local following theta_t, the new moments), and
    an engine resumed from it continues bit-identically to the uninterrupted
    run and to the two-step path."""
    D = gpu
    n, h, rounds = 40_009, 3, 4
    hyper = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    th = O.rng_fill(3, "theta", 0, n, -0.1, 0.1)
    grads = [O.rng_fill(3, "grad", t, n, -1e-2, 1e-2) for t in range(h * rounds)]
    grads[5][7] = np.inf  # an overflow on a window's last step (the gated rerun)

    def engine(fused):
        e = D.DilocoEngine(D.DilocoConfig(h, 1, D.FP16, h * rounds), hyper, n)
        e.set_fused_delta(fused)
        e.upload(D.THETA_T, th)
        e.upload(D.THETA_LOCAL, th)
        return e

    paths = []

    def run(e, hook):
        gptr = e.device_ptr(D.GRAD)

        def producer(step):
            e.upload(D.GRAD, grads[step])
            return gptr, False, 0.0
        return D.run_training(e, None, producer, on_round=hook)

    a = engine(True)

    def save(rounds_done):
        if rounds_done == 2:
            p = str(tmp_path / "r2.ckpt")
            D.checkpoint_save([a], p, completed_rounds=rounds_done)
            paths.append(p)
    run(a, save)
    twostep = engine(False)
    run(twostep, None)
    for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM):
        assert np.array_equal(bits(a.download(w)), bits(twostep.download(w))), w
    b = engine(True)
    D.checkpoint_load([b], paths[0])
    assert b.scalars().inner_step == 2 * h and b.scalars().outer_epoch == 2
    gptr = b.device_ptr(D.GRAD)
    opt = D.DilocoOptimizer(b)
    for t in range(2 * h, h * rounds):
        b.upload(D.GRAD, grads[t])
        opt.step(gptr, grad_is_scaled=False)
    for w in (D.THETA_T, D.THETA_LOCAL, D.ADAM_M, D.ADAM_V, D.MOMENTUM):
        assert np.array_equal(bits(a.download(w)), bits(b.download(w))), w
    for e in (a, b, twostep):
        e.close()
