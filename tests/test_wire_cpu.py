"""Wire framing on the CPU: the oracle restatement pinned
to the reference's own wire.cpp and its tests, and the host-only parts of the
C ABI (frame sizes, frame validation and drop rules that never touch the GPU)."""
import ctypes as C

import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from paper_2407_07852_b200 import wire as W
from oracle import oracle as O

PEER = (0x0123456789ABCDEF, 0xFEDCBA9876543210)


def test_frame_goldens_from_reference_tests(port, ref):
    """test_collective.cpp:134-186: heartbeat frame bytes, reduce payload prefix layout."""
    for lib in (port, ref):
        f = lib.encode_frame(3, bytes([0xAA, 0xBB]))
        assert len(f) == 16 and f[:4] == b"ODLC" and f[4] == 1 and f[5] == 3 and f[6] == 2
        assert f[7:14] == bytes(7) and f[14:] == bytes([0xAA, 0xBB])
        p = lib.encode_reduce_payload(7, 3, 1, bytes([1, 2, 3]))
        assert len(p) == 16 and p[0] == 7 and p[8] == 3 and p[12] == 1 and p[13:] == bytes([1, 2, 3])
    bad = bytearray(port.encode_frame(3, b"\xaa\xbb"))
    bad[0] = ord("X")
    with pytest.raises(ValueError):
        ref.parse_frames(bytes(bad))


def test_port_framing_matches_reference_encoders(port, ref):
    rng = np.random.default_rng(0)
    for trial in range(20):
        payload = rng.integers(0, 256, int(rng.integers(0, 3000)), dtype=np.uint8).tobytes()
        ty = int(rng.integers(1, 10))
        assert port.encode_frame(ty, payload) == ref.encode_frame(ty, payload)
        ep, ci, pr = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 2 ** 32)), int(rng.integers(0, 2))
        assert port.encode_reduce_payload(ep, ci, pr, payload) == ref.encode_reduce_payload(ep, ci, pr, payload)


@pytest.mark.parametrize("prec,chunk", [(1, 1 << 20), (1, 1000), (0, 4096), (0, 3), (1, 2)])
def test_send_chunk_span_stream_parses_with_reference_parser(port, ref, prec, chunk):
    """The restated send_chunk_span stream, fed to the reference's FrameParser in
    odd-sized pieces, yields the chunk sequence collective.cpp:1318-1345 defines."""
    n = 2501
    vals = np.arange(n, dtype=np.uint16) if prec else np.arange(n, dtype=np.float32) * 0.5
    name = port.chunk_name(3, 2, *PEER)
    assert name == "a3.p2.f0123456789abcdeffedcba9876543210"
    stream = port.send_chunk_span(5, 11, name, prec, 777, vals, chunk)
    w = 2 if prec else 4
    per = max(1, chunk // w)
    frames = ref.parse_frames(stream, feed=97)
    assert len(frames) == -(-n // per)
    for i, fr in enumerate(frames):
        assert fr["type"] == 5 and fr["ok"] and fr["epoch"] == 11 and fr["chunk_index"] == i
        assert fr["precision"] == prec
    mine, used = port.parse_chunk_frames(stream)
    assert used == len(stream) and len(mine) == len(frames)
    got = b"".join(m["scalars"] for m in mine)
    assert got == vals.tobytes()
    assert [m["offset"] for m in mine] == [777 + i * per for i in range(len(mine))]
    assert all(m["name"] == name for m in mine)


def test_frames_size_matches_restatement(port):
    for prec in (0, 1):
        for chunk in (1, 2, 5, 4096, 1 << 20):
            for n in (0, 1, 2, 999, 100_003):
                t = W.make_tags(A.MSG_REDUCE_CHUNK, prec, 5, 12, 345, PEER, chunk)
                size, frames = C.c_size_t(0), C.c_uint64(0)
                assert A.lib.dlc_wire_frames_size(n, C.byref(t), C.byref(size), C.byref(frames)) == 0
                vals = np.zeros(n, np.uint16 if prec else np.float32)
                name = port.chunk_name(12, 345, *PEER)
                assert size.value == len(port.send_chunk_span(5, 5, name, prec, 0, vals, chunk))


def _decode(data: bytes, prec=1, base=0, cap=1 << 20):
    buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
    chunks = (A.WireChunk * 64)()
    nc, used = C.c_size_t(0), C.c_size_t(0)
    st = A.lib.dlc_wire_decode(C.c_void_p(buf.ctypes.data), len(data), prec, base, cap, None, chunks, 64,
                               C.byref(nc), C.byref(used), None)
    return st, [chunks[i] for i in range(nc.value)], used.value


def test_decode_validation_and_drops_without_gpu(port):
    """Frames the device decoder rejects before any copy: FrameParser errors
    (SerializationError), incomplete tails, and the drop rules of
    handle_reduce_chunk (collective.cpp:1017-1047)."""
    name = port.chunk_name(0, 1, *PEER)
    good = port.send_chunk_span(5, 9, name, 1, 0, np.arange(10, dtype=np.uint16), 8)  # 4-element chunks
    # wrong precision for this buffer: every chunk parsed, none accepted (no device touched)
    st, chunks, used = _decode(good, prec=0)
    assert st == 0 and used == len(good) and len(chunks) == 3
    assert [c.accepted for c in chunks] == [0, 0, 0]
    assert [(c.offset, c.length, c.chunk_index) for c in chunks] == [(0, 4, 0), (4, 4, 1), (8, 2, 2)]
    assert chunks[0].partition == 1 and (chunks[0].from_hi, chunks[0].from_lo) == PEER
    # incomplete tail: only whole frames are consumed
    st, chunks, used = _decode(good[:-3], prec=0)
    assert st == 0 and len(chunks) == 2 and used == chunks[1].frame_offset + chunks[1].frame_bytes
    # other message types pass through unaccepted
    hb = port.encode_frame(3, b"\x01\x02")
    st, chunks, used = _decode(hb + good, prec=0)
    assert st == 0 and chunks[0].msg_type == 3 and not chunks[0].accepted and used == len(hb) + len(good)
    # out-of-range and unparsable names are dropped
    st, chunks, _ = _decode(good, prec=1, base=100, cap=5)
    assert st == 0 and not any(c.accepted for c in chunks)
    bad_name = port.send_chunk_span(5, 9, "zzz", 1, 0, np.arange(3, dtype=np.uint16), 64)
    st, chunks, _ = _decode(bad_name, prec=1)
    assert st == 0 and len(chunks) == 1 and not chunks[0].accepted
    # malformed frames raise SerializationError (status DLC_ESERIAL) and stop there
    for mutate in (lambda b: b.__setitem__(0, ord("X")), lambda b: b.__setitem__(4, 2),
                   lambda b: b.__setitem__(5, 42), lambda b: b.__setitem__(27, 2)):
        b = bytearray(good)
        mutate(b)
        st, _, used = _decode(bytes(b), prec=0)
        assert st == A.ESERIAL and used == 0
    # truncated reduce payload inside a complete frame
    st, _, _ = _decode(port.encode_frame(5, b"\x00" * 12), prec=0)
    assert st == A.ESERIAL


def test_serialization_error_maps_to_python_exception():
    assert D.SerializationError is not None
    from paper_2407_07852_b200.diloco import _check
    with pytest.raises(D.SerializationError):
        _check(A.ESERIAL)
