"""Parity of the CUDA path (through the C ABI) with the oracle — run on a B200.

Bar: FP32 path and the FP16 ordered path are bit-exact against
the reference CPU functions on identical inputs; NaNs compare by class.  The
oracle is the C restatement (pinned to the reference build by
tests/test_oracle.py) and the committed golden fixtures produced by the
reference itself.
"""
import ctypes as C
import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from oracle import driver as DR
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def same(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    nan = np.isnan(a) & np.isnan(b)
    return np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(bits(a)[~nan], bits(b)[~nan])


@pytest.fixture(scope="module", autouse=True)
def gpu():
    try:
        n = D.device_count()
    except D.Error:
        n = 0
    if n < 1:
        pytest.skip("no CUDA device")
    D.lib.dlc_set_device(0)


# ---- FP16 codec (fp16.cpp:25-85; test_tensor.cpp:28-99) ---------------------------------

def test_fp16_encode_exhaustive(port):
    """Every one of the 2^32 FP32 bit patterns encodes to the reference's code."""
    chunk = 1 << 26
    for start in range(0, 1 << 32, chunk):
        got = D.fp16_encode_bits(start, chunk)
        x = np.arange(start, start + chunk, dtype=np.uint64).astype(np.uint32).view(np.float32)
        want, _ = port.encode_fp16(x)
        if not np.array_equal(got, want):
            bad = np.nonzero(got != want)[0][:5]
            raise AssertionError(f"mismatch at bit patterns {[hex(start + int(i)) for i in bad]}: "
                                 f"got {got[bad]}, want {want[bad]}")


def test_fp16_decode_every_code(port, golden):
    codes = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    got = D.decode_fp16(codes)
    assert same(got, port.decode_fp16(codes))
    assert same(got, golden("fp16_codec.npz")["decoded_all"])
    # exact round trip for every finite code (test_tensor.cpp:68-76)
    fin = codes[(codes & 0x7C00) != 0x7C00]
    back, ov = D.encode_fp16(D.decode_fp16(fin))
    assert not ov and np.array_equal(back, fin)


def test_fp16_codec_golden(golden):
    z = golden("fp16_codec.npz")
    got, ov = D.encode_fp16(z["x"])
    assert np.array_equal(got, z["codes"])
    assert ov  # the fixture holds inf / overflow values


def test_fp16_scalar_goldens():
    enc = lambda x: int(D.encode_fp16([x])[0][0])  # noqa: E731
    assert enc(1.0) == 0x3C00 and enc(-0.0) == 0x8000 and enc(0.0) == 0
    assert enc(65520.0) == 0x7C00 and enc(-65520.0) == 0xFC00 and enc(65519.0) == 0x7BFF
    assert enc(1e30) == 0x7C00 and enc(float("nan")) == 0x7E00 and enc(1e-9) == 0
    assert D.decode_fp16([enc(2049.0)])[0] == 2048.0
    assert D.decode_fp16([0x7BFF])[0] == 65504.0
    _, ov = D.encode_fp16([1.5, -2.0, 0.25])
    assert not ov
    codes, ov = D.encode_fp16([1e9, 1.0])
    assert ov and codes[0] == 0x7C00
    codes, ov = D.encode_fp16(np.zeros(0, np.float32))
    assert codes.size == 0 and not ov


# ---- host-buffer reference functions ------------------------------------------------------

def test_adamw_golden_trajectory(golden):
    z = golden("adamw.npz")
    st = D.AdamWState.init(z["p0"].size)
    p = z["p0"].copy()
    for t in range(5):
        p = D.adamw_step(st, p, z["grads"][t], float(z["lrs"][t]))
        assert np.array_equal(bits(p), bits(z["traj"][t])), t
    assert np.array_equal(bits(st.m), bits(z["m"])) and np.array_equal(bits(st.v), bits(z["v"]))
    assert st.step_count == int(z["step_count"])


def test_adamw_goldens_and_errors():
    st = D.AdamWState.init(1, weight_decay=0.1)
    p = D.adamw_step(st, [1.0], [0.1], 4e-4)
    assert abs(float(p[0]) - 0.99956) <= 1e-6 * 0.99956 and st.step_count == 1
    st = D.AdamWState.init(3, weight_decay=0.0)
    assert np.array_equal(D.adamw_step(st, [1, -2, 0.5], [0, 0, 0], 4e-4), np.float32([1, -2, 0.5]))
    st = D.AdamWState.init(1, weight_decay=0.0)
    with pytest.raises(D.NumericError):
        D.adamw_step(st, [1.0], [np.inf], 1e-3)
    assert st.step_count == 0 and st.m[0] == 0 and st.v[0] == 0
    with pytest.raises(D.ConfigError):
        D.adamw_step(st, [1.0], [0.1], -1e-3)
    with pytest.raises(D.ShapeError):
        D.adamw_step(st, [1.0, 2.0], [0.1], 1e-3)


def test_adamw_random_vs_oracle(port):
    rng = np.random.default_rng(5)
    n = 100_003  # ragged: exercises the scalar tail
    for trial in range(3):
        p = rng.uniform(-2, 2, n).astype(np.float32)
        st = D.AdamWState.init(n, weight_decay=0.05 * trial)
        m, v, sc = np.zeros(n, np.float32), np.zeros(n, np.float32), 0
        for s in range(4):
            g = (rng.uniform(-1, 1, n) * 10.0 ** (trial - 2)).astype(np.float32)
            g[:3] = [0.0, 1e-40, -3e-39]
            out = D.adamw_step(st, p, g, 1e-3 * (s + 1))
            _, want, sc = port.adamw_step(p, g, m, v, sc, 1e-3 * (s + 1), wd=0.05 * trial)
            assert np.array_equal(bits(out), bits(want))
            assert np.array_equal(bits(st.m), bits(m)) and np.array_equal(bits(st.v), bits(v))
            p = out


def test_nesterov_golden(golden):
    z = golden("nesterov.npz")
    st = D.NesterovState.init(z["theta0"].size, 0.7, 0.9)
    th = z["theta0"].copy()
    for t in range(4):
        th = D.nesterov_step(st, th, z["grads"][t])
        assert np.array_equal(bits(th), bits(z["traj"][t]))
    assert np.array_equal(bits(st.momentum_buf), bits(z["buf"]))
    st = D.NesterovState.init(1, 0.7, 0.9)
    out = D.nesterov_step(st, [10.0], [1.0])
    assert st.momentum_buf[0] == 1.0 and abs(float(out[0]) - 8.67) <= 1e-6 * 8.67
    st = D.NesterovState.init(2, 1.0, 0.0)
    assert np.array_equal(D.nesterov_step(st, [1.25, -3.5], [0.25, 0.5]), np.float32([1.0, -4.0]))
    with pytest.raises(D.NumericError):
        D.nesterov_step(D.NesterovState.init(1), [1.0], [np.nan])


def test_reduce_average_golden(golden):
    z = golden("reduce.npz")
    for k in (1, 2, 3, 5, 8):
        for prec in (0, 1):
            got = D.reduce_average(list(z[f"in_k{k}"]), prec)
            assert same(got, z[f"out_k{k}_p{prec}"]), (k, prec)
    assert np.array_equal(D.reduce_average([[2, 4], [4, 8]], 0), np.float32([3, 6]))
    with pytest.raises(D.CollectiveError):
        D.reduce_average([], 0)
    with pytest.raises(D.ShapeError):
        D.reduce_average([[1.0], [1.0, 2.0]], 0)


def test_reduce_average_many_contributors(port):
    rng = np.random.default_rng(3)
    cs = [rng.uniform(-1, 1, 999).astype(np.float32) * np.float32(2.0 ** (j % 7)) for j in range(40)]
    for prec in (0, 1):
        assert same(D.reduce_average(cs, prec), port.reduce_average(cs, prec)[1])


def test_unscale_axpy_all_finite(port):
    rng = np.random.default_rng(9)
    x = np.ldexp(rng.uniform(-2, 2, 50001), rng.integers(-40, 40, 50001)).astype(np.float32)
    x[7] = np.inf
    for scale in (65536.0, 2.0 ** -20, 1.0):
        u, ov = D.scaler_unscale_and_check(D.LossScaler(scale), x)
        u2, ov2 = port.scaler_unscale_and_check(scale, x)
        assert ov == ov2 and same(u, u2)
    y = rng.uniform(-1, 1, 50001).astype(np.float32)
    assert np.array_equal(bits(D.axpy(-1.0, x, y)), bits(port.axpy(-1.0, x, y)))
    assert np.array_equal(D.axpy(-1.0, [0.5, 2.5], [1.0, 2.0]), np.float32([0.5, -0.5]))
    assert not D.all_finite(x) and D.all_finite(y) and D.all_finite(np.zeros(0, np.float32))


# ---- device-resident engine: full DiLoCo trajectories -------------------------------------

def run_engines(k, h, rounds, prec, n, hyper, grad_fn, theta0, inner_mode=A.INNER_PINGPONG):
    cfg = D.DilocoConfig(h, k, prec, h * rounds)
    hp = D.OptimHyperparams(inner_lr=hyper.inner_lr, warmup_steps=hyper.warmup_steps,
                            weight_decay=hyper.weight_decay, outer_lr=hyper.outer_lr,
                            outer_momentum=hyper.outer_momentum, scaler_init_scale=hyper.scale,
                            scaler_growth_interval=hyper.growth_interval)
    engines = [D.DilocoEngine(cfg, hp, n, 0, inner_mode) for _ in range(k)]
    for e in engines:
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, theta0)
    step = 0
    results = []
    for _ in range(rounds):
        for _t in range(h):
            for wi, e in enumerate(engines):
                e.inner_step_host(grad_fn(wi, step), grad_is_scaled=False)
            step += 1
        results.append(D.outer_step_local(engines))
    return engines


@pytest.mark.parametrize("inner_mode", [A.INNER_PINGPONG, A.INNER_INPLACE])
@pytest.mark.parametrize("prec", [0, 1])
def test_engine_matches_reference_golden_trajectory(golden, prec, inner_mode):
    """K=2, H=5, 2 rounds, injected overflow at (worker 1, step 3) — bitwise vs the reference."""
    z = golden("diloco_k2_h5.npz")
    theta0 = z["theta0"]
    n = theta0.size

    def grad_fn(w, t):
        g = O.rng_fill(4242, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == (1, 3):
            g[17] = np.inf
        return g

    hyper = DR.Hyper(inner_lr=4e-4, warmup_steps=5)
    engines = run_engines(2, 5, 2, prec, n, hyper, grad_fn, theta0, inner_mode)
    for wi, e in enumerate(engines):
        for which, name in ((A.THETA_T, "theta_t"), (A.THETA_LOCAL, "theta_local"), (A.ADAM_M, "m"),
                            (A.ADAM_V, "v"), (A.MOMENTUM, "buf")):
            assert np.array_equal(bits(e.download(which)), bits(z[f"p{prec}_w{wi}_{name}"])), (wi, name)
        s = e.scalars()
        assert s.step_count == int(z[f"p{prec}_w{wi}_step_count"])
        assert s.scale == float(z[f"p{prec}_w{wi}_scale"])
        assert s.outer_epoch == 2 and s.inner_step == 10
        assert s.overflow_skips == (1 if wi == 1 else 0)
        e.close()


@pytest.mark.parametrize("k,prec", [(2, 0), (3, 1), (8, 1), (8, 0)])
def test_engine_config1_shape_vs_oracle(port, k, prec):
    """Config-1 shape (N = 2^20 ragged to 2^20 + 5, H = 50, 1 outer step) at K = 2, and K up to 8."""
    n = (1 << 20) + 5 if k == 2 else 40_000 + 3
    h = 50 if k == 2 else 4
    hyper = DR.Hyper(inner_lr=4e-4, warmup_steps=20)
    theta0 = O.rng_fill(4242, "theta", 0, n, -0.05, 0.05)
    grads = {}

    def grad_fn(w, t):
        key = (w, t)
        if key not in grads:
            grads[key] = O.rng_fill(4242, "grad", w * 100_000 + t, n, -1e-2, 1e-2)
        return grads[key]

    workers, hist = DR.simulate(port, theta0, grad_fn, k, h, 1, prec, hyper)
    engines = run_engines(k, h, 1, prec, n, hyper, grad_fn, theta0)
    for wi, e in enumerate(engines):
        assert np.array_equal(bits(e.download(A.THETA_T)), bits(workers[wi].theta_t))
        assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(workers[wi].theta_local))
        assert np.array_equal(bits(e.download(A.MOMENTUM)), bits(workers[wi].buf))
        assert np.array_equal(bits(e.download(A.ADAM_M)), bits(workers[wi].m))
        assert np.array_equal(bits(e.download(A.ADAM_V)), bits(workers[wi].v))
        e.close()


def test_outer_nonfinite_skip_and_resnapshot():
    """engine.cpp:136-144 / test_engine.cpp:179-191: a non-finite mean skips Nesterov, resets local."""
    n = 1000
    theta0 = O.rng_fill(1, "theta", 0, n, -1, 1)
    cfg = D.DilocoConfig(1, 2, A.FP16, 2)
    engines = [D.DilocoEngine(cfg, D.OptimHyperparams(), n) for _ in range(2)]
    for wi, e in enumerate(engines):
        e.upload(A.THETA_T, theta0)
        local = theta0 - np.float32(0.01)
        if wi == 1:
            local[5] = -7e4  # delta = 7e4 encodes to +inf in FP16
        e.upload(A.THETA_LOCAL, local)
    res = D.outer_step_local(engines)
    assert not res.applied and res.outer_epoch == 1
    for e in engines:
        assert np.array_equal(e.download(A.THETA_T), theta0)
        assert np.array_equal(e.download(A.THETA_LOCAL), theta0)
        assert not e.download(A.MOMENTUM).any()
        assert e.scalars().outer_skips == 1
    # solo engine, FP32: NaN in theta_local skips too
    e = D.DilocoEngine(D.DilocoConfig(1, 1, A.FP32, 1), D.OptimHyperparams(), n)
    e.upload(A.THETA_T, theta0)
    bad = theta0.copy()
    bad[999] = np.nan
    e.upload(A.THETA_LOCAL, bad)
    r = e.outer_step(None, wait=True)
    assert not r.applied
    assert np.array_equal(e.download(A.THETA_LOCAL), theta0)


def test_outer_identity_transport():
    """test_engine.cpp:156-169: K=1, lr=1, mu=0 transports theta_local exactly (FP32)."""
    n = 4099
    theta0 = O.rng_fill(2, "theta", 0, n, -1, 1)
    local = O.rng_fill(2, "local", 0, n, -1, 1)
    hp = D.OptimHyperparams(outer_lr=1.0, outer_momentum=0.0)
    e = D.DilocoEngine(D.DilocoConfig(3, 1, A.FP32, 3), hp, n)
    e.upload(A.THETA_T, theta0)
    e.upload(A.THETA_LOCAL, local)
    r = e.outer_step(None, wait=True)
    assert r.applied
    # theta - 1*(delta + 0) with delta = theta - local is local up to one rounding; the
    # reference's arithmetic is reproduced bit for bit:
    port = O.port()
    tt, tl, buf = theta0.copy(), local.copy(), np.zeros(n, np.float32)
    d = port.axpy(-1.0, tl, tt)
    _, want = port.nesterov_step(tt, d, buf, 1.0, 0.0)
    assert np.array_equal(bits(e.download(A.THETA_T)), bits(want))


def test_engine_errors():
    e = D.DilocoEngine(D.DilocoConfig(5, 1, A.FP32, 5), D.OptimHyperparams(), 64)
    g = np.zeros(64, np.float32)
    e.inner_step_host(g)
    with pytest.raises(D.Error):  # engine.cpp:116-120, mid-window
        e.outer_step(None)
    for _ in range(4):
        e.inner_step_host(g)
    e.outer_step(None)
    with pytest.raises(D.Error):  # engine.cpp:98-100, past total_inner_steps
        e.inner_step_host(g)
    with pytest.raises(D.CollectiveError):  # K mismatch
        D.DilocoEngine(D.DilocoConfig(1, 2, A.FP32, 1), D.OptimHyperparams(), 64).outer_step(None)
    with pytest.raises(D.ShapeError):
        e.upload(A.THETA_T, np.zeros(63, np.float32))


def test_inner_overflow_skip_semantics():
    """engine.cpp:50-69: overflow leaves p/m/v/step_count, halves the scale, cursor advances."""
    n = 513
    for mode in (A.INNER_PINGPONG, A.INNER_INPLACE):
        e = D.DilocoEngine(D.DilocoConfig(10, 1, A.FP32, 10), D.OptimHyperparams(warmup_steps=2), n, 0, mode)
        th = O.rng_fill(3, "theta", 0, n, -1, 1)
        e.upload(A.THETA_LOCAL, th)
        g = O.rng_fill(3, "grad", 0, n, -1e-2, 1e-2)
        r = e.inner_step_host(g)
        assert not r.overflow_skipped and r.lr == np.float32(2e-4)
        before = {w: e.download(w) for w in (A.THETA_LOCAL, A.ADAM_M, A.ADAM_V)}
        bad = g.copy()
        bad[512] = np.inf  # lands in the scalar tail
        r = e.inner_step_host(bad)
        assert r.overflow_skipped and r.lr == 0.0
        for w, arr in before.items():
            assert np.array_equal(bits(e.download(w)), bits(arr))
        s = e.scalars()
        assert s.step_count == 1 and s.inner_step == 2 and s.scale == 32768.0 and s.overflow_skips == 1
        r = e.inner_step_host(g)  # lr index continues from the applied-step count (engine.cpp:64)
        assert not r.overflow_skipped and r.lr == np.float32(4e-4)


@pytest.mark.parametrize("inner_mode", [A.INNER_PINGPONG, A.INNER_INPLACE])
@pytest.mark.parametrize("k", [1, 2])
def test_theta_local_follows_theta_t(port, tmp_path, k, inner_mode):
    """theta_local := theta_t after every outer step (engine.cpp:141-143) is recorded,
    not stored, in PINGPONG engines (Pair::follow).  Overflows on the first inner step
    of a window (the step that would read the followed buffer), writes through
    upload / device_ptr, and checkpoints taken right after an outer step must all
    behave as if the copy had been made."""
    n, h, rounds = 3001, 2, 3
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=1)
    theta0 = O.rng_fill(11, "theta", 0, n, -0.5, 0.5)

    def grad_fn(w, t):
        g = O.rng_fill(11, "grad", w * 100 + t, n, -1e-2, 1e-2)
        if t in (h, 2 * h) and w == k - 1:  # first step of rounds 2 and 3
            g[n - 1] = np.inf
        return g

    workers, _ = DR.simulate(port, theta0, grad_fn, k, h, rounds, 0, hyper)
    engines = run_engines(k, h, rounds, 0, n, hyper, grad_fn, theta0, inner_mode)
    for wi, e in enumerate(engines):
        assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(workers[wi].theta_t))
        assert np.array_equal(bits(e.download(A.THETA_T)), bits(workers[wi].theta_t))
        assert np.array_equal(bits(e.download(A.ADAM_M)), bits(workers[wi].m))
        assert e.scalars().overflow_skips == (2 if wi == k - 1 else 0)
    e = engines[0]
    want_t = workers[0].theta_t
    # checkpoint right after an outer step round-trips theta_local
    path = str(tmp_path / "follow.ckpt")
    D.checkpoint_save(engines, path)
    fresh = [D.DilocoEngine(e.config, D.OptimHyperparams(), n, 0, inner_mode) for _ in range(k)]
    D.checkpoint_load(fresh, path)
    for wi, x in enumerate(fresh):
        assert np.array_equal(bits(x.download(A.THETA_LOCAL)), bits(workers[wi].theta_t))
        assert np.array_equal(bits(x.download(A.THETA_T)), bits(workers[wi].theta_t))
        x.close()
    # writing theta_t leaves theta_local alone, and vice versa
    other = O.rng_fill(12, "theta", 0, n, -1, 1)
    e.upload(A.THETA_T, other)
    assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(want_t))
    e.upload(A.THETA_T, want_t)
    e.rng_fill(A.THETA_LOCAL, 12, "theta", 0, -1, 1)  # device-side write through the live pointer
    assert np.array_equal(bits(e.download(A.THETA_T)), bits(want_t))
    assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(other))
    for x in engines:
        x.close()


def test_large_n_slices_vs_oracle(port):
    """150M-parameter buffers (configs 2-3): elementwise path, so oracle slices are exact."""
    n = 150_000_000
    hyper = DR.Hyper(inner_lr=4e-4, warmup_steps=5)
    hp = D.OptimHyperparams(inner_lr=4e-4, warmup_steps=5)
    e = D.DilocoEngine(D.DilocoConfig(2, 1, A.FP16, 2), hp, n)
    e.rng_fill(A.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(A.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    for t in range(2):
        e.rng_fill(A.GRAD, 4242, "grad", t, -1e-2, 1e-2)
        e.inner_step(e.device_ptr(A.GRAD), grad_is_scaled=False)
    r = e.outer_step(None, wait=True)
    assert r.applied
    out = {w: e.download(w) for w in (A.THETA_T, A.THETA_LOCAL, A.ADAM_M, A.ADAM_V, A.MOMENTUM)}
    for lo in (0, n // 2 - 777, n - 4096):
        sl = slice(lo, lo + 4096)
        th0 = O.rng_fill(4242, "theta", 0, 4096, -0.05, 0.05, first=lo)
        w = DR.make_workers(th0, 1, hyper)[0]
        for t in range(2):
            DR.inner_step(port, w, O.rng_fill(4242, "grad", t, 4096, -1e-2, 1e-2, first=lo), hyper)
        DR.outer_round(port, [w], 1, hyper)
        for which, arr in ((A.THETA_T, w.theta_t), (A.THETA_LOCAL, w.theta_local), (A.ADAM_M, w.m),
                           (A.ADAM_V, w.v), (A.MOMENTUM, w.buf)):
            assert np.array_equal(bits(out[which][sl]), bits(arr)), (lo, which)
    e.close()


def test_optimizer_facade_rounds():
    """DilocoOptimizer::step (engine.cpp:162-174): outer round after every H-th inner step."""
    n = 1024
    e = D.DilocoEngine(D.DilocoConfig(3, 1, A.FP32, 9), D.OptimHyperparams(), n)
    opt = D.DilocoOptimizer(e, D.SoloCollective(0))
    e.rng_fill(A.GRAD, 1, "g", 0, -1e-2, 1e-2)
    g = e.device_ptr(A.GRAD)
    flags = []
    for _ in range(9):
        opt.step(g, grad_is_scaled=False)
        flags.append(opt.round_just_completed)
    assert flags == [False, False, True] * 3
    assert e.scalars().outer_epoch == 3


def test_solo_collective_host_plugin(golden):
    z = golden("reduce.npz")
    c = D.SoloCollective(0)
    assert c.world_size() == 1
    for prec in (0, 1):
        out, rep = c.all_reduce_avg(z["in_k1"][0], prec, outer_epoch=4)
        assert same(out, z[f"out_k1_p{prec}"])
        assert rep.contributors == 1 and rep.outer_epoch == 4 and rep.data_bytes_sent == 0


@pytest.mark.parametrize("prec", [0, 1])
def test_outer_step_host_buffers_chunked(port, prec):
    """dlc_engine_outer_step_host (the e2e path): chunked H2D / fused solo step / D2H,
    bitwise vs the oracle's outer round, including a skipped (non-finite) step."""
    n = 3 * (16 << 20) + 1001  # several 64 MB chunks plus a ragged tail
    hyper = DR.Hyper()
    e = D.DilocoEngine(D.DilocoConfig(1, 1, prec, 1), D.OptimHyperparams(), n)
    e.rng_fill(A.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    theta0 = e.download(A.THETA_T)
    loc = (theta0 - O.rng_fill(4242, "local", 0, n, -1e-3, 1e-3)).astype(np.float32)
    out = np.empty(n, np.float32)
    r = e.outer_step_host(None, loc, out)
    assert r.applied
    w = DR.make_workers(theta0, 1, hyper)[0]
    w.theta_local = loc.copy()
    DR.outer_round(port, [w], prec, hyper)
    assert np.array_equal(bits(out), bits(w.theta_t))
    assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(w.theta_t))
    assert np.array_equal(bits(e.download(A.MOMENTUM)), bits(w.buf))
    # second step, non-finite in the last chunk: skipped, theta_t returned unchanged
    bad = loc.copy()
    bad[n - 7] = np.nan
    r = e.outer_step_host(None, bad, out)
    assert not r.applied and r.outer_epoch == 2
    assert np.array_equal(bits(out), bits(w.theta_t))
    assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(w.theta_t))
    assert np.array_equal(bits(e.download(A.THETA_T)), bits(w.theta_t))
    e.close()


@pytest.mark.parametrize("prec", [0, 1])
def test_external_collective_outer_step(port, prec):
    """compute_pseudo_gradient -> any host collective (here reduce_average) -> apply_outer_step:
    the split the reference's SocketCollective needs between boxes."""
    n, k = 30_011, 3
    hyper = DR.Hyper()
    theta0 = O.rng_fill(6, "theta", 0, n, -1, 1)
    locs = [(theta0 - O.rng_fill(6, "local", j, n, -1e-3, 1e-3)).astype(np.float32) for j in range(k)]
    engines = [D.DilocoEngine(D.DilocoConfig(1, k, prec, 1), D.OptimHyperparams(), n) for _ in range(k)]
    deltas = []
    for e, loc in zip(engines, locs):
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, loc)
        d, ep = e.compute_pseudo_gradient()
        assert ep == 0
        deltas.append(d)
    _, mean = port.reduce_average(deltas, prec)
    ws = DR.make_workers(theta0, k, hyper)
    for w, loc in zip(ws, locs):
        w.theta_local = loc.copy()
    dbar, applied, ref_deltas = DR.outer_round(port, ws, prec, hyper)
    for d, rd in zip(deltas, ref_deltas):
        assert np.array_equal(bits(d), bits(rd))
    for e, w in zip(engines, ws):
        r = e.apply_outer_step(mean, 0)
        assert r.applied and r.outer_epoch == 1
        assert np.array_equal(bits(e.download(A.THETA_T)), bits(w.theta_t))
        assert np.array_equal(bits(e.download(A.THETA_LOCAL)), bits(w.theta_t))
        with pytest.raises(D.CollectiveError):
            e.apply_outer_step(mean, 0)  # stale epoch (engine.cpp:129-134)
        e.close()


# ---- engine properties mirrored from the reference's own tests ----------------------------

def test_identity_transport_equals_bare_adamw(port):
    """test_engine.cpp:213-241: K=1, H=1, outer lr=1, mu=0 DiLoCo == bare AdamW, bitwise, 60 steps."""
    n = 4099
    # weights in [0.5, 1] and small steps keep theta_t and theta_local within a factor of
    # two, so theta_t - (theta_t - theta_local) is exact (Sterbenz) as in the reference test
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=5, weight_decay=0.0)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=5, weight_decay=0.0, outer_lr=1.0, outer_momentum=0.0)
    e = D.DilocoEngine(D.DilocoConfig(1, 1, A.FP32, 60), hp, n)
    theta0 = O.rng_fill(11, "theta", 0, n, 0.5, 1.0)
    e.upload(A.THETA_T, theta0)
    e.upload(A.THETA_LOCAL, theta0)
    bare = DR.make_workers(theta0, 1, hyper)[0]
    opt = D.DilocoOptimizer(e, None)
    for t in range(60):
        g = O.rng_fill(11, "grad", t, n, -1e-1, 1e-1)
        e.upload(A.GRAD, g)
        opt.step(e.device_ptr(A.GRAD), grad_is_scaled=False)
        assert opt.round_just_completed
        DR.inner_step(port, bare, g, hyper)
        assert np.array_equal(bits(e.download(A.THETA_T)), bits(bare.theta_local)), t
    e.close()


def test_averaging_equivalence_local_fleet():
    """test_engine.cpp:243-294: outer lr=1, mu=0 makes theta_t the mean of the workers' theta_local
    (<= 1e-6 relative), identical on every worker."""
    n, k = 20_011, 3
    hp = D.OptimHyperparams(outer_lr=1.0, outer_momentum=0.0)
    theta0 = O.rng_fill(12, "theta", 0, n, -1, 1)
    engines = [D.DilocoEngine(D.DilocoConfig(1, k, A.FP32, 1), hp, n) for _ in range(k)]
    locs = []
    for j, e in enumerate(engines):
        e.upload(A.THETA_T, theta0)
        loc = (theta0 + O.rng_fill(12, "move", j, n, -1e-2, 1e-2)).astype(np.float32)
        e.upload(A.THETA_LOCAL, loc)
        locs.append(loc.astype(np.float64))
    assert D.outer_step_local(engines).applied
    mean = np.mean(np.stack(locs), axis=0)
    t0 = engines[0].download(A.THETA_T)
    # relative to the operands' scale: where the mean cancels to ~0 the error is
    # one rounding of the deltas (|theta0 - local_j| <= 1e-2), not of the mean
    scale = np.maximum(np.abs(mean), np.max(np.abs(np.stack(locs) - theta0.astype(np.float64)), axis=0))
    assert np.all(np.abs(t0 - mean) / np.maximum(scale, 1e-12) <= 1e-6)
    # and bit for bit the reference's outer round
    hyper = DR.Hyper(outer_lr=1.0, outer_momentum=0.0)
    ws = DR.make_workers(theta0, k, hyper)
    for j, w in enumerate(ws):
        w.theta_local = locs[j].astype(np.float32)
    DR.outer_round(O.port(), ws, A.FP32, hyper)
    assert np.array_equal(bits(t0), bits(ws[0].theta_t))
    for e in engines[1:]:
        assert np.array_equal(bits(e.download(A.THETA_T)), bits(t0))
    for e in engines:
        e.close()


def test_reruns_are_bitwise_deterministic():
    """test_harness.cpp:135-146: identical inputs, identical bits on a second run."""
    n = 1 << 18

    def run():
        e = D.DilocoEngine(D.DilocoConfig(3, 1, A.FP16, 9), D.OptimHyperparams(warmup_steps=2), n)
        e.rng_fill(A.THETA_T, 13, "theta", 0, -1, 1)
        e.rng_fill(A.THETA_LOCAL, 13, "theta", 0, -1, 1)
        opt = D.DilocoOptimizer(e, None)
        for t in range(9):
            e.rng_fill(A.GRAD, 13, "grad", t, -1e-2, 1e-2)
            opt.step(e.device_ptr(A.GRAD), grad_is_scaled=False)
        out = [e.download(w) for w in (A.THETA_T, A.THETA_LOCAL, A.ADAM_M, A.ADAM_V, A.MOMENTUM)]
        e.close()
        return out

    a, b = run(), run()
    for x, y in zip(a, b):
        assert np.array_equal(bits(x), bits(y))


@pytest.mark.parametrize("n", [0, 1, 3, 7, 513])
@pytest.mark.parametrize("prec", [0, 1])
def test_tiny_and_empty_vectors(port, n, prec):
    """Degenerate sizes through every engine path: solo (fused K2+K4) and an
    in-process fleet of 3 (K2 -> fold -> K4), against the oracle."""
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=1)
    theta0 = O.rng_fill(31, "theta", 0, n, -1, 1)
    grad_fn = lambda w, t: O.rng_fill(31, "grad", w * 10 + t, n, -1e-2, 1e-2)  # noqa: E731
    for k in (1, 3):
        workers, _ = DR.simulate(port, theta0, grad_fn, k, 2, 2, prec, hyper)
        engines = run_engines(k, 2, 2, prec, n, hyper, grad_fn, theta0)
        for wi, e in enumerate(engines):
            for which, want in ((A.THETA_T, workers[wi].theta_t), (A.THETA_LOCAL, workers[wi].theta_local),
                                (A.MOMENTUM, workers[wi].buf), (A.ADAM_M, workers[wi].m)):
                got = e.download(which)
                assert got.size == n and np.array_equal(bits(got), bits(want)), (k, wi, which)
            assert e.scalars().outer_epoch == 2
            e.close()


@pytest.mark.parametrize("tma", [1, 2, 0])
@pytest.mark.parametrize("prec", [0, 1])
def test_fold_push_kernels_every_world_size(port, prec, tma):
    """The P2P owner fold for K = 1..9 and 16 (the compile-time-K TMA kernels,
    single-leader and warp-specialised, the per-thread kernels and the generic
    one), bit for bit against reduce_average in rank order, with the non-finite
    mark."""
    n = 64 * 301
    rng = np.random.default_rng(prec * 10 + tma)
    for k in list(range(1, 10)) + [16]:
        xs = [(rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-12, 12, n)).astype(np.float32) for _ in range(k)]
        if k == 5:
            xs[3][77] = np.inf
        if prec:
            codes = [port.encode_fp16(x)[0] for x in xs]
            ins = [port.decode_fp16(c) for c in codes]
            raw = codes
        else:
            ins = raw = xs
        arr = (C.c_void_p * k)(*[c.ctypes.data for c in raw])
        out = np.empty(n, np.uint16 if prec else np.float32)
        bad = C.c_int(0)
        assert A.lib.dlc_fold_push_probe(arr, k, n, prec, tma, out.ctypes.data, C.byref(bad)) == 0
        _, want = port.reduce_average(ins, prec)
        got = port.decode_fp16(out) if prec else out
        assert same(got, want), (k, prec, tma)
        assert bool(bad.value) == (not np.all(np.isfinite(want))), k


@pytest.mark.parametrize("k", [2, 8, 9])
def test_p2p_kernels_probe_runs(k):
    """The single-device probe of the K > 1 kernels (tools/p2p_kernels_probe.py)
    launches K2, the owner fold (TMA for k <= 8, per-thread above) and K4 on a
    ragged size and reports a positive time for each."""
    ms = (C.c_float * 3)()
    assert A.lib.dlc_p2p_kernels_probe(k, 1_000_003, 1, 2, ms) == 0, A.lib.dlc_last_error()
    assert all(t > 0 for t in ms)
    assert A.lib.dlc_p2p_kernels_probe(1, 1024, 1, 1, ms) == A.EINVAL


def test_fp16_reduction_bounds(port):
    """test_engine.cpp:296-324 on the device: the FP16 average stays within
    2^-10 of the FP32 one, relative to the result for same-sign contributions
    and to the largest contribution for mixed signs."""
    rng = np.random.default_rng(21)
    n = 50_000
    for k in (2, 3, 8):
        same_sign = [rng.uniform(0.5, 2.0, n).astype(np.float32) * np.float32(2.0 ** -j) for j in range(k)]
        f32 = D.reduce_average(same_sign, A.FP32)
        f16 = D.reduce_average(same_sign, A.FP16)
        assert np.all(np.abs(f16 - f32) / np.abs(f32) <= 2.0 ** -10)
        mixed = [rng.uniform(-1, 1, n).astype(np.float32) for _ in range(k)]
        m32 = D.reduce_average(mixed, A.FP32)
        m16 = D.reduce_average(mixed, A.FP16)
        scale = np.max(np.abs(np.stack(mixed)), axis=0)
        assert np.all(np.abs(m16 - m32) / scale <= 2.0 ** -10)


def test_run_training_records_and_state(port):
    """run_training (engine.cpp:176-240): the record stream (step / round /
    event kinds, skip events), the round hook, RunResult, and the final state
    bitwise against the oracle's K=1 run with the same gradients."""
    n, h, total = 5003, 3, 9
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(41, "theta", 0, n, -0.5, 0.5)

    def grad_np(t):
        g = O.rng_fill(41, "grad", t, n, -1e-2, 1e-2)
        if t == 4:
            g[n - 1] = np.inf
        return g

    e = D.DilocoEngine(D.DilocoConfig(h, 1, A.FP16, total), hp, n)
    e.upload(A.THETA_T, theta0)
    e.upload(A.THETA_LOCAL, theta0)
    gptr = e.device_ptr(A.GRAD)

    def producer(step):
        e.upload(A.GRAD, grad_np(step))
        return gptr, False, 0.25 * step

    records, rounds = [], []
    res = D.run_training(e, None, producer, sink=records.append, on_round=rounds.append)
    assert res["steps_done"] == total and res["rounds_done"] == total // h
    assert res["final_train_loss"] == np.float32(0.25 * (total - 1)) and res["reduce_data_bytes"] == 0
    kinds = [r["kind"] for r in records]
    assert kinds.count("step") == total and kinds.count("round") == total // h
    assert [r["event"] for r in records if r["kind"] == "event"] == ["inner_overflow_skip"]
    assert rounds == [1, 2, 3]
    steps = [r for r in records if r["kind"] == "step"]
    assert [r["inner_step"] for r in steps] == list(range(1, total + 1))
    assert [r["outer_epoch"] for r in steps] == [0, 0, 1, 1, 1, 2, 2, 2, 3]
    assert steps[4]["lr"] == 0.0 and abs(steps[1]["perplexity"] - np.exp(0.25)) < 1e-6
    workers, _ = DR.simulate(port, theta0, lambda w, t: grad_np(t), 1, h, total // h, A.FP16, hyper)
    for which, want in ((A.THETA_T, workers[0].theta_t), (A.THETA_LOCAL, workers[0].theta_local),
                        (A.ADAM_M, workers[0].m), (A.MOMENTUM, workers[0].buf)):
        assert np.array_equal(bits(e.download(which)), bits(want)), which
    with pytest.raises(ZeroDivisionError):  # a failing producer aborts the loop with its own error
        e2 = D.DilocoEngine(D.DilocoConfig(h, 1, A.FP16, total), hp, n)
        D.run_training(e2, None, lambda step: 1 / 0)
    e.close()


@pytest.mark.parametrize("inner_mode", [A.INNER_PINGPONG, A.INNER_INPLACE])
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("prec", [A.FP16, A.FP32])
def test_optimizer_step_fused_solo_boundary(port, prec, fused, inner_mode):
    """DilocoOptimizer::step (engine.cpp:162-174) for one worker: the window's
    last inner step and the SoloCollective outer step as ONE pass
    (launch_boundary_solo, the default) or as two steps, bitwise against the
    oracle over four windows of H = 3: an overflow on a window's last step
    (round 0: the outer step reruns from the unchanged theta_local), one
    mid-window (round 1), a non-finite delta (round 2: theta_t / theta_local
    uploaded at +-3e38 so the delta overflows; the outer step is skipped and
    theta_local := theta_t), and an ordinary round last.  Ragged N."""
    n, h, rounds, seed = 70_003, 3, 4, 57
    hyper = DR.Hyper(inner_lr=1e-3, warmup_steps=2)
    hp = D.OptimHyperparams(inner_lr=1e-3, warmup_steps=2)
    theta0 = O.rng_fill(seed, "theta", 0, n, -0.05, 0.05)

    def grad_np(t):
        g = O.rng_fill(seed, "grad", t, n, -1e-2, 1e-2)
        if t in (2, 4):
            g[n - 2] = np.inf
        return g

    e = D.DilocoEngine(D.DilocoConfig(h, 1, prec, h * rounds), hp, n, 0, inner_mode)
    e.set_fused_delta(fused)
    e.upload(A.THETA_T, theta0)
    e.upload(A.THETA_LOCAL, theta0)
    gptr = e.device_ptr(A.GRAD)
    opt = D.DilocoOptimizer(e)
    (w,) = DR.make_workers(theta0, 1, hyper)
    t = 0
    for rnd in range(rounds):
        if rnd == 2:  # a non-finite delta at this window's end
            tt = e.download(A.THETA_T)
            tt[11] = np.float32(3e38)
            e.upload(A.THETA_T, tt)
            tl = e.download(A.THETA_LOCAL)
            tl[11] = np.float32(-3e38)
            e.upload(A.THETA_LOCAL, tl)
            w.theta_t, w.theta_local = tt.copy(), tl.copy()
        if rnd == 3:  # back to an ordinary element
            tt = e.download(A.THETA_T)
            tt[11] = np.float32(0.01)
            e.upload(A.THETA_T, tt)
            e.upload(A.THETA_LOCAL, tt)
            w.theta_t, w.theta_local = tt.copy(), tt.copy()
        for _ in range(h):
            e.upload(A.GRAD, grad_np(t))
            opt.step(gptr, grad_is_scaled=False)
            DR.inner_step(port, w, grad_np(t), hyper)
            t += 1
        assert opt.round_just_completed
        _, applied, _ = DR.outer_round(port, [w], prec, hyper)
        sc = e.scalars()
        assert sc.outer_epoch == rnd + 1 and bool(sc.last_applied) == applied, (rnd, applied)
        assert applied == (rnd != 2)
        for which, want in ((A.THETA_T, w.theta_t), (A.THETA_LOCAL, w.theta_local), (A.ADAM_M, w.m),
                            (A.ADAM_V, w.v), (A.MOMENTUM, w.buf)):
            assert np.array_equal(bits(e.download(which)), bits(want)), (rnd, which)
        assert sc.step_count == w.step_count
    e.close()
