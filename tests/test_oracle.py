"""Pin the CPU oracle (C restatement) before trusting it.

* the reference's own test goldens (test_optim.cpp, test_tensor.cpp,
  test_engine.cpp, test_collective.cpp) against the restatement AND the
  reference build;
* the restatement bit-for-bit against the reference build on random inputs;
* the restatement against the committed golden fixtures (tests/golden/,
  produced by the reference build via tests/golden/make_golden.py).
"""
import math

import numpy as np
import pytest

from oracle import driver as D
from oracle import oracle as O


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def same_bits_or_both_nan(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    nan = np.isnan(a) & np.isnan(b)
    return np.array_equal(bits(a)[~nan], bits(b)[~nan]) and np.array_equal(np.isnan(a), np.isnan(b))


@pytest.fixture(params=["port", "reference"])
def lib(request):
    if request.param == "port":
        return O.port()
    r = O.reference()
    if r is None:
        pytest.skip("reference build absent")
    return r


# ---- fp16 codec: test_tensor.cpp:28-99 ---------------------------------------------

def test_fp16_scalar_examples(lib):
    assert lib.fp16_encode_scalar(1.0) == 0x3C00
    assert lib.fp16_decode_scalar(lib.fp16_encode_scalar(2049.0)) == 2048.0
    assert lib.fp16_encode_scalar(0.0) == 0x0000
    assert lib.fp16_encode_scalar(-0.0) == 0x8000
    assert lib.fp16_decode_scalar(lib.fp16_encode_scalar(1.5)) == 1.5
    assert lib.fp16_decode_scalar(lib.fp16_encode_scalar(1e-9)) == 0.0


def test_fp16_overflow_is_infinity(lib):
    assert lib.fp16_encode_scalar(65520.0) == 0x7C00
    assert lib.fp16_encode_scalar(-65520.0) == 0xFC00
    assert lib.fp16_encode_scalar(65519.0) == 0x7BFF
    assert lib.fp16_decode_scalar(0x7BFF) == 65504.0
    assert lib.fp16_encode_scalar(1e30) == 0x7C00
    assert math.isinf(lib.fp16_decode_scalar(lib.fp16_encode_scalar(math.inf)))
    assert lib.fp16_encode_scalar(math.nan) == 0x7E00
    assert math.isnan(lib.fp16_decode_scalar(lib.fp16_encode_scalar(math.nan)))


def test_fp16_decode_every_code(lib):
    codes = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    got = lib.decode_fp16(codes)
    want = codes.view(np.float16).astype(np.float32)  # IEEE definition
    assert same_bits_or_both_nan(got, want)


def test_fp16_round_trip_every_finite_code(lib):
    codes = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = codes[(codes & 0x7C00) != 0x7C00]
    back, ov = lib.encode_fp16(lib.decode_fp16(finite))
    assert not ov
    assert np.array_equal(back, finite)


def test_fp16_encode_fuzz_matches_ieee_rne(lib):
    # test_tensor.cpp:78-87: exponent-spread values vs a bit-independent converter.
    rng = np.random.default_rng(2024)
    x = np.ldexp(rng.uniform(-2, 2, 200000).astype(np.float32), rng.integers(-32, 32, 200000))
    x = x.astype(np.float32)
    got, _ = lib.encode_fp16(x)
    want = x.astype(np.float16).view(np.uint16)  # numpy: IEEE RNE, overflow -> inf
    assert np.array_equal(got, want)


def test_fp16_relative_error_up_to_2048(lib):
    rng = np.random.default_rng(7)
    x = rng.uniform(-2048, 2048, 100000).astype(np.float32)
    x = x[np.abs(x) >= 2.0 ** -14]
    back = lib.decode_fp16(lib.encode_fp16(x)[0])
    assert np.all(np.abs(back.astype(np.float64) - x) <= np.ldexp(np.abs(x.astype(np.float64)), -11))


def test_encode_overflow_flag(lib):
    _, ov = lib.encode_fp16(np.float32([1.5, -2.0, 0.25]))
    assert not ov
    codes, ov = lib.encode_fp16(np.float32([1e9, 1.0]))
    assert ov and codes[0] == 0x7C00
    codes, ov = lib.encode_fp16(np.zeros(0, np.float32))
    assert codes.size == 0 and not ov


# ---- axpy / pseudo-gradient: test_tensor.cpp:109-121, test_engine.cpp:77-97 ----------

def test_axpy_examples(lib):
    assert np.array_equal(lib.axpy(1.0, [1, 2], [0, 0]), np.float32([1, 2]))
    assert np.array_equal(lib.axpy(0.0, [9, 9], [3, 4]), np.float32([3, 4]))
    assert np.array_equal(lib.axpy(-1.0, [0.5, 2.5], [1.0, 2.0]), np.float32([0.5, -0.5]))


# ---- optim: test_optim.cpp ------------------------------------------------------------

def test_adamw_null_gradient_identity(lib):
    m = np.zeros(3, np.float32)
    v = np.zeros(3, np.float32)
    st, p, sc = lib.adamw_step(np.float32([1, -2, 0.5]), np.zeros(3, np.float32), m, v, 0, 4e-4,
                               wd=0.0)
    assert st == 0 and sc == 1
    assert np.array_equal(p, np.float32([1, -2, 0.5]))


def test_adamw_first_step_golden(lib):
    m = np.zeros(1, np.float32)
    v = np.zeros(1, np.float32)
    st, p, sc = lib.adamw_step(np.float32([1.0]), np.float32([0.1]), m, v, 0, 4e-4, wd=0.1)
    assert st == 0
    assert abs(float(p[0]) - 0.99956) <= 1e-6 * 0.99956
    # ScalarAdamW recurrence (tests/support/optim_oracle.hpp:14-33) in float32:
    f = np.float32
    mm = f(0.9) * f(0) + (f(1) - f(0.9)) * f(0.1)
    vv = f(0.95) * f(0) + (f(1) - f(0.95)) * f(0.1) * f(0.1)
    mh = mm / (f(1) - f(0.9))
    vh = vv / (f(1) - f(0.95))
    want = f(1) - f(4e-4) * (mh / (np.sqrt(vh) + f(1e-8)) + f(0.1) * f(1))
    assert p[0] == want


def test_adamw_rejects_nonfinite(lib):
    m = np.zeros(1, np.float32)
    v = np.zeros(1, np.float32)
    st, _, sc = lib.adamw_step(np.float32([1.0]), np.float32([np.inf]), m, v, 0, 1e-3, wd=0.0)
    assert st == O.ENUMERIC and sc == 0
    st, _, sc = lib.adamw_step(np.float32([1.0]), np.float32([0.1]), m, v, 0, -1e-3, wd=0.0)
    assert st == O.ECONFIG and sc == 0


def test_nesterov_goldens(lib):
    buf = np.zeros(1, np.float32)
    st, p = lib.nesterov_step(np.float32([10.0]), np.float32([1.0]), buf, 0.7, 0.9)
    assert st == 0 and buf[0] == 1.0
    assert abs(float(p[0]) - 8.67) <= 1e-6 * 8.67
    buf = np.zeros(2, np.float32)
    _, p = lib.nesterov_step(np.float32([1.25, -3.5]), np.float32([0.25, 0.5]), buf, 1.0, 0.0)
    assert np.array_equal(p, np.float32([1.0, -4.0]))
    buf = np.zeros(1, np.float32)
    th = np.float32([0.0])
    for want in (1.0, 1.9, 2.71):
        _, th = lib.nesterov_step(th, np.float32([1.0]), buf, 0.7, 0.9)
        assert abs(float(buf[0]) - want) <= 1e-6 * want
    st, _ = lib.nesterov_step(np.float32([1.0]), np.float32([np.nan]), np.zeros(1, np.float32), 0.7, 0.9)
    assert st == O.ENUMERIC


def test_lr_schedule(lib):
    lr = lambda s, cos: lib.lr_at(1000, 10000, 4e-4, cos, s)  # noqa: E731
    assert abs(lr(500, False) - 2e-4) <= 1e-7 * 2e-4
    assert lr(1000, False) == np.float32(4e-4)
    assert lr(5000, False) == np.float32(4e-4)
    assert lr(1000, True) == np.float32(4e-4)
    assert abs(lr(10000, True) - 4e-5) <= 1e-6 * 4e-5
    assert abs(lr(20000, True) - 4e-5) <= 1e-6 * 4e-5
    assert lr(0, True) == 0.0
    vals = [lr(s, True) for s in range(0, 1001)]
    assert all(b >= a for a, b in zip(vals, vals[1:]))


def test_scaler(lib):
    _, ov = lib.scaler_unscale_and_check(65536.0, np.float32([np.inf, 1.0]))
    assert ov
    s, g = lib.scaler_update(65536.0, 0, 2000, ov)
    assert s == 32768.0 and g == 0
    for _ in range(2000):
        s, g = lib.scaler_update(s, g, 2000, False)
    assert s == 65536.0 and g == 0
    g0 = np.float32([1e-4, -3.7, 42.0])
    back, ov = lib.scaler_unscale_and_check(65536.0, g0 * np.float32(65536.0))
    assert not ov and np.array_equal(back, g0)
    s = 1.0
    for _ in range(200):
        s, _ = lib.scaler_update(s, 0, 2000, True)
        assert s > 0 and math.log2(s) == math.floor(math.log2(s))


# ---- reduce: test_collective.cpp:355-366, test_engine.cpp:296-324 ----------------------

def test_two_peer_average(lib):
    st, out = lib.reduce_average([np.float32([2, 4]), np.float32([4, 8])], 0)
    assert st == 0 and np.array_equal(out, np.float32([3, 6]))


def test_fp16_reduction_within_one_encode(lib):
    a = np.float32([0.5, 1024.0, 2.0 ** -13, 3.1415])
    b = np.float32([0.25, 512.0, 2.0 ** -12, 2.5])
    f32 = lib.reduce_average([a, b], 0)[1].astype(np.float64)
    f16 = lib.reduce_average([a, b], 1)[1].astype(np.float64)
    assert np.all(np.abs(f16 - f32) / np.abs(f32) <= 2.0 ** -10)
    c = np.float32([0.5, -1024.0, 2.0 ** -13, 3.1415])
    d = np.float32([0.25, 512.0, 2.0 ** -12, -2.5])
    m32 = lib.reduce_average([c, d], 0)[1].astype(np.float64)
    m16 = lib.reduce_average([c, d], 1)[1].astype(np.float64)
    scale = np.maximum(np.maximum(np.abs(c), np.abs(d)), 2.0 ** -14)
    assert np.all(np.abs(m16 - m32) / scale <= 2.0 ** -10)


def test_reduce_empty_is_error(lib):
    st, _ = lib.reduce_average([], 0)
    assert st == O.ECOLLECTIVE


def test_partition_and_byte_law(lib):
    assert lib.partition_ranges(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert lib.partition_ranges(2, 4) == [(0, 1), (1, 1), (2, 0), (2, 0)]
    n = 24 * 50
    for k in (2, 3, 4, 8):
        for r in range(k):
            b = lib.per_peer_reduce_bytes(n, k, r, 0)
            assert b == 2 * (k - 1) * n * 4 // k
        assert lib.fleet_reduce_bytes(n, k, 1) == 2 * (k - 1) * n * 2
    assert lib.per_peer_reduce_bytes(n, 1, 0, 0) == 0


# ---- restatement == reference, bit for bit ---------------------------------------------

def test_port_matches_reference_bitwise(ref):
    P = O.port()
    rng = np.random.default_rng(99)
    n = 50000
    x = np.ldexp(rng.uniform(-2, 2, n), rng.integers(-40, 40, n)).astype(np.float32)
    x[:5] = [np.nan, np.inf, -np.inf, -0.0, 1e-45]
    assert np.array_equal(P.encode_fp16(x)[0], ref.encode_fp16(x)[0])
    for t in range(3):
        p = rng.uniform(-2, 2, n).astype(np.float32)
        g = rng.uniform(-1, 1, n).astype(np.float32) * np.float32(10.0 ** (t - 2))
        m1, v1 = np.zeros(n, np.float32), np.zeros(n, np.float32)
        m2, v2 = m1.copy(), v1.copy()
        sc1 = sc2 = 0
        for s in range(4):
            _, p1, sc1 = P.adamw_step(p, g, m1, v1, sc1, 1e-3 * (s + 1), wd=0.05 * t)
            _, p2, sc2 = ref.adamw_step(p, g, m2, v2, sc2, 1e-3 * (s + 1), wd=0.05 * t)
            assert np.array_equal(bits(p1), bits(p2)) and sc1 == sc2
            assert np.array_equal(bits(m1), bits(m2)) and np.array_equal(bits(v1), bits(v2))
            p = p1
        b1, b2 = np.zeros(n, np.float32), np.zeros(n, np.float32)
        _, o1 = P.nesterov_step(p, g, b1, 0.7, 0.9)
        _, o2 = ref.nesterov_step(p, g, b2, 0.7, 0.9)
        assert np.array_equal(bits(o1), bits(o2)) and np.array_equal(bits(b1), bits(b2))
        cs = [rng.uniform(-1, 1, n).astype(np.float32) * np.float32(4 ** j) for j in range(5)]
        for prec in (0, 1):
            assert same_bits_or_both_nan(P.reduce_average(cs, prec)[1], ref.reduce_average(cs, prec)[1])
        u1, ov1 = P.scaler_unscale_and_check(2.0 ** -3, x)
        u2, ov2 = ref.scaler_unscale_and_check(2.0 ** -3, x)
        assert ov1 == ov2 and same_bits_or_both_nan(u1, u2)
    for s in (0, 1, 3, 999, 1000, 1001, 5000, 9999, 10000, 12000):
        for cos in (False, True):
            assert P.lr_at(1000, 10000, 4e-4, cos, s) == ref.lr_at(1000, 10000, 4e-4, cos, s)


# ---- restatement == committed fixtures (works without the reference) -------------------

def test_port_matches_golden_codec(port, golden):
    z = golden("fp16_codec.npz")
    assert np.array_equal(port.encode_fp16(z["x"])[0], z["codes"])
    codes = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    assert same_bits_or_both_nan(port.decode_fp16(codes), z["decoded_all"])


def test_port_matches_golden_adamw_nesterov(port, golden):
    z = golden("adamw.npz")
    p, sc = z["p0"].copy(), 0
    m, v = np.zeros_like(p), np.zeros_like(p)
    for t in range(5):
        st, p, sc = port.adamw_step(p, z["grads"][t], m, v, sc, float(z["lrs"][t]))
        assert st == 0 and np.array_equal(bits(p), bits(z["traj"][t]))
    assert np.array_equal(bits(m), bits(z["m"])) and np.array_equal(bits(v), bits(z["v"]))
    assert sc == int(z["step_count"])
    z = golden("nesterov.npz")
    th, buf = z["theta0"].copy(), np.zeros_like(z["theta0"])
    for t in range(4):
        _, th = port.nesterov_step(th, z["grads"][t], buf, 0.7, 0.9)
        assert np.array_equal(bits(th), bits(z["traj"][t]))
    assert np.array_equal(bits(buf), bits(z["buf"]))


def test_port_matches_golden_reduce(port, golden):
    z = golden("reduce.npz")
    for k in (1, 2, 3, 5, 8):
        for prec in (0, 1):
            _, out = port.reduce_average(list(z[f"in_k{k}"]), prec)
            assert same_bits_or_both_nan(out, z[f"out_k{k}_p{prec}"]), (k, prec)


def test_port_matches_golden_diloco_trajectory(port, golden):
    z = golden("diloco_k2_h5.npz")
    theta0 = z["theta0"]
    n = theta0.size
    assert np.array_equal(O.rng_fill(4242, "theta", 0, n, -0.05, 0.05), theta0)

    def grad_fn(w, t):
        g = O.rng_fill(4242, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == (1, 3):
            g[17] = np.inf
        return g

    assert np.array_equal(grad_fn(1, 3), z["grad_w1_t3"], equal_nan=True)
    hyper = D.Hyper(inner_lr=4e-4, warmup_steps=5)
    for prec in (0, 1):
        workers, hist = D.simulate(port, theta0, grad_fn, 2, 5, 2, prec, hyper)
        for wi, w in enumerate(workers):
            for name in ("theta_t", "theta_local", "m", "v", "buf"):
                assert np.array_equal(bits(getattr(w, name)), bits(z[f"p{prec}_w{wi}_{name}"])), name
            assert w.step_count == int(z[f"p{prec}_w{wi}_step_count"])
            assert w.scale == float(z[f"p{prec}_w{wi}_scale"])
        assert workers[1].skipped[3] and not workers[0].skipped[3]
        for r, (dbar, applied, _) in enumerate(hist):
            assert np.array_equal(bits(dbar), bits(z[f"p{prec}_r{r}_dbar"]))
            assert applied == bool(z[f"p{prec}_r{r}_applied"])
