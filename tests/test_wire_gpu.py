"""Wire framing from / into device memory and full cross-box rounds (SURVEY.md
§8f row f2), on a B200: frames byte-identical to the reference's framing of the
same scalars, decode round trips, and K-worker all-reduce rounds whose only
exchange is those bytes ending bit-identical to the reference's outer round."""
import ctypes as C
import socket
import threading

import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from paper_2407_07852_b200 import wire as W
from oracle import driver as DR
from oracle import oracle as O

pytestmark = pytest.mark.gpu

PEERS = [(0x1111 * (j + 1), 0xABCDEF0123456789 ^ j) for j in range(8)]


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


def _torch_dev(arr):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr)).to("cuda:0")


def _encode(dev, offset, n, tags):
    size = C.c_size_t(0)
    assert A.lib.dlc_wire_frames_size(n, C.byref(tags), C.byref(size), None) == 0
    out = np.empty(max(size.value, 1), np.uint8)
    used = C.c_size_t(0)
    st = A.lib.dlc_wire_encode(C.c_void_p(dev.data_ptr()), offset, n, C.byref(tags), C.c_void_p(out.ctypes.data),
                               out.nbytes, C.byref(used), None)
    assert st == 0, A.lib.dlc_last_error()
    return out[:used.value].tobytes()


@pytest.mark.parametrize("prec,chunk,n,off", [(1, 1 << 20, 1_000_003, 0), (1, 1000, 10_007, 5), (0, 4096, 10_007, 9),
                                               (0, 3, 301, 0), (1, 2, 257, 1 << 40)])
def test_encode_matches_reference_framing(port, prec, chunk, n, off):
    rng = np.random.default_rng(n)
    vals = rng.integers(0, 65536, n, dtype=np.uint16) if prec else rng.standard_normal(n).astype(np.float32)
    tags = W.make_tags(A.MSG_REDUCE_CHUNK, prec, 42, 1, 6, PEERS[3], chunk)
    got = _encode(_torch_dev(vals.view(np.int16) if prec else vals), off, n, tags)
    name = port.chunk_name(1, 6, *PEERS[3])
    want = port.send_chunk_span(A.MSG_REDUCE_CHUNK, 42, name, prec, off, vals, chunk)
    assert got == want


def test_decode_round_trip_and_split_feeds(port):
    import torch
    n, chunk = 50_001, 6000
    vals = np.random.default_rng(1).integers(0, 65536, n, dtype=np.uint16)
    name = port.chunk_name(0, 0, *PEERS[0])
    stream = port.send_chunk_span(A.MSG_REDUCE_RESULT, 7, name, 1, 1000, vals, chunk)
    out = torch.zeros(n + 10, dtype=torch.int16, device="cuda:0")
    chunks = (A.WireChunk * 256)()
    nc, used = C.c_size_t(0), C.c_size_t(0)
    # arrive in ragged pieces: decode what is complete, keep the rest
    pending = b""
    got_chunks = 0
    rng = np.random.default_rng(2)
    at = 0
    while at < len(stream):
        take = int(rng.integers(1, 20_000))
        pending += stream[at:at + take]
        at += take
        buf = np.frombuffer(pending, np.uint8)
        st = A.lib.dlc_wire_decode(C.c_void_p(buf.ctypes.data), len(pending), 1, 1000, n + 10,
                                   C.c_void_p(out.data_ptr()), chunks, 256, C.byref(nc), C.byref(used), None)
        assert st == 0
        assert all(chunks[i].accepted for i in range(nc.value))
        got_chunks += nc.value
        pending = pending[used.value:]
    assert pending == b"" and got_chunks == -(-n // (chunk // 2))
    back = out.cpu().numpy().view(np.uint16)
    assert np.array_equal(back[:n], vals) and not back[n:].any()


def _engines(k, n, prec, theta0, locs, hp=None):
    hp = hp or D.OptimHyperparams()
    es = []
    for j in range(k):
        e = D.DilocoEngine(D.DilocoConfig(1, k, prec, 4), hp, n)
        e.upload(A.THETA_T, theta0)
        e.upload(A.THETA_LOCAL, locs[j])
        es.append(e)
    return es


@pytest.mark.parametrize("k,prec,n,chunk", [(3, 1, 10_007, 4096), (3, 0, 10_007, 1 << 20), (4, 1, 7, 2),
                                             (2, 0, 200_003, 100_000)])
def test_wire_round_matches_reference_outer_round(port, k, prec, n, chunk):
    theta0 = O.rng_fill(21, "theta", 0, n, -1, 1)
    locs = [(theta0 - O.rng_fill(21, "local", j, n, -1e-2, 1e-2)).astype(np.float32) for j in range(k)]
    engines = _engines(k, n, prec, theta0, locs)
    # the frames one worker puts on the wire are the reference's frames of its encoded delta
    rd = W.WireRound(engines[1], 1, PEERS[:k], attempt=2, chunk_size_bytes=chunk)
    delta = port.axpy(-1.0, locs[1], theta0)
    scal = port.encode_fp16(delta)[0] if prec else delta
    for p in range(k):
        off, ln = rd.ranges[p]
        want = port.send_chunk_span(A.MSG_REDUCE_CHUNK, 0, port.chunk_name(2, p, *PEERS[1]), prec, off,
                                    scal[off:off + ln], chunk)
        assert rd.scatter_frames(p).tobytes() == want
    # full rounds (twice: momentum carries over), bytes only between workers
    hyper = DR.Hyper()
    ws = DR.make_workers(theta0, k, hyper)
    for rnd in range(2):
        for j, w in enumerate(ws):
            w.theta_local = locs[j].copy() if rnd == 0 else (w.theta_t - O.rng_fill(22, "l", j, n, -1e-2, 1e-2))
        if rnd == 1:
            for j, e in enumerate(engines):
                e.upload(A.THETA_LOCAL, ws[j].theta_local)
        res = W.all_reduce_local(engines, PEERS[:k], attempt=rnd, chunk_size_bytes=chunk)
        DR.outer_round(port, ws, prec, hyper)
        assert all(r.applied for r in res) and all(r.outer_epoch == rnd + 1 for r in res)
        for j, e in enumerate(engines):
            for which, want in ((A.THETA_T, ws[j].theta_t), (A.THETA_LOCAL, ws[j].theta_local),
                                (A.MOMENTUM, ws[j].buf)):
                assert np.array_equal(bits(e.download(which)), bits(want)), (rnd, j, which)
    for e in engines:
        e.close()


def test_wire_round_over_sockets_and_nonfinite_skip(port):
    """A real byte transport (socket pairs) between the workers; an FP16
    overflow in one delta makes every worker skip the outer step."""
    k, n = 3, 30_011
    theta0 = O.rng_fill(23, "theta", 0, n, -1, 1)
    locs = [(theta0 - O.rng_fill(23, "local", j, n, -1e-2, 1e-2)).astype(np.float32) for j in range(k)]
    locs[2][n - 1] = -7e4  # delta 7e4 + theta encodes to +inf
    engines = _engines(k, n, A.FP16, theta0, locs)

    def deliver(src, dst, frames):
        a, b = socket.socketpair()
        data = frames.tobytes()
        t = threading.Thread(target=lambda: (a.sendall(data), a.close()))
        t.start()
        got = bytearray()
        while True:
            part = b.recv(1 << 16)
            if not part:
                break
            got += part
        t.join()
        b.close()
        return bytes(got)

    res = W.all_reduce_local(engines, PEERS[:k], chunk_size_bytes=8192, deliver=deliver)
    assert not any(r.applied for r in res)
    for e in engines:
        assert np.array_equal(e.download(A.THETA_T), theta0)
        assert np.array_equal(e.download(A.THETA_LOCAL), theta0)
        assert e.scalars().outer_skips == 1
        e.close()


def test_wire_epoch_guard_and_mid_window():
    n = 1000
    e = D.DilocoEngine(D.DilocoConfig(2, 2, A.FP16, 4), D.OptimHyperparams(), n)
    e.inner_step_host(np.zeros(n, np.float32))
    with pytest.raises(D.Error):  # engine.cpp:116-120
        e.wire_begin()
    e.inner_step_host(np.zeros(n, np.float32))
    ep = e.wire_begin()
    with pytest.raises(D.CollectiveError):  # engine.cpp:129-134
        e.wire_finish(ep + 1)
    e.close()
