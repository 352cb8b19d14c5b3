"""ctypes front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Two libraries are exposed with one numpy-level API:

* ``port()`` — ``oracle/_build/liboracle.so``, the C restatement in
  ``diloco_oracle.c`` (cites /root/reference/proj file:line per function).
* ``reference()`` — ``oracle/_ref/libdiloco_ref.so``, the reference's own
  ``fp16.cpp tensor.cpp optim.cpp reduce.cpp`` compiled by ``oracle/Makefile``
  and wrapped by ``ref_shim.cpp``.  Present when it was built in the build
  container (it travels to the GPU box with the snapshot); ``None`` otherwise.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` arm may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdiloco_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u64 = C.c_uint64

OK, ESHAPE, ECONFIG, ENUMERIC, ECOLLECTIVE, ESERIAL, EAGAIN = 0, 1, 2, 3, 4, 5, 6
_u8p = C.POINTER(C.c_uint8)


def build(ref: bool | None = None) -> None:
    """Compile the restatement (always) and the reference (when present)."""
    targets = [PORT_SO]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        targets.append("ref")
        lib = os.path.join(os.path.dirname(HERE), "paper_2407_07852_b200", "libdiloco_cuda.so")
        if os.path.exists(lib):
            targets.append("dropin")  # C++ drop-in layer vs the reference (tests/cpp)
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class _Lib:
    """Common numpy API over either library (prefix 'orc_' or 'ref_')."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.kind = "port" if prefix == "orc_" else "reference"
        L = C.CDLL(path)
        self._L = L
        p = prefix

        def fn(name, res, *args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = list(args)
            return f

        self._enc1 = fn("fp16_encode", C.c_uint16, C.c_float)
        self._dec1 = fn("fp16_decode", C.c_float, C.c_uint16)
        self._enc = fn("encode_fp16", C.c_int, _f32p, _sz, _u16p)
        self._dec = fn("decode_fp16", None if p == "orc_" else C.c_int, _u16p, _sz, _f32p)
        self._all_finite = fn("all_finite", C.c_int, _f32p, _sz)
        self._axpy = fn("axpy", None if p == "orc_" else C.c_int, C.c_float, _f32p, _f32p, _sz, _f32p)
        self._lr_at = fn("lr_at", C.c_float, _u64, _u64, C.c_float, C.c_int, _u64)
        self._adamw = fn("adamw_step", C.c_int, _f32p, _f32p, _f32p, _f32p, _sz, C.c_float,
                         C.c_float, C.c_float, C.c_float, C.POINTER(_u64), C.c_float, _f32p)
        self._nest = fn("nesterov_step", C.c_int, _f32p, _f32p, _f32p, _sz, C.c_float, C.c_float, _f32p)
        self._unscale = fn("scaler_unscale_and_check", C.c_int, C.c_float, _f32p, _sz, _f32p)
        self._scaler_update = fn("scaler_update", None, C.POINTER(C.c_float), C.POINTER(_u64), _u64, C.c_int)
        self._part = fn("partition_ranges", None, _sz, _sz, C.POINTER(_sz), C.POINTER(_sz))
        self._ppb = fn("per_peer_reduce_bytes", _u64, _sz, _sz, _sz, C.c_int)
        self._fleet = fn("fleet_reduce_bytes", _u64, _sz, _sz, C.c_int)
        if p == "orc_":
            self._reduce = fn("reduce_average", C.c_int, C.POINTER(C.c_void_p), _sz, _sz, C.c_int,
                              C.c_void_p, _f32p)
            self._key = fn("rng_key", _u64, _u64, C.c_char_p, _u64)
            self._fill = fn("rng_fill", None, _u64, _u64, _sz, C.c_float, C.c_float, _f32p)
            vp = C.c_void_p
            self._frame = fn("encode_frame", _sz, C.c_uint8, vp, _sz, vp)
            self._rpayload = fn("encode_reduce_payload", _sz, _u64, C.c_uint32, C.c_uint8, vp, _sz, vp)
            self._segment = fn("encode_chunk_segment", _sz, C.c_char_p, _sz, _u64, _u64, vp, _sz, vp)
            self._cname = fn("chunk_name", _sz, C.c_uint32, C.c_uint32, _u64, _u64, C.c_char_p)
            self._span = fn("send_chunk_span", _sz, C.c_uint8, _u64, C.c_char_p, _sz, C.c_int, _u64, vp, _u64,
                            _u64, vp)
            P = C.POINTER
            self._parse = fn("parse_chunk_frame", C.c_int, vp, _sz, P(_sz), P(C.c_uint8), P(_u64), P(C.c_uint32),
                             P(C.c_uint8), P(_sz), P(_sz), P(_u64), P(_u64), P(_sz), P(_sz))
        else:
            self._reduce = fn("reduce_average", C.c_int, C.POINTER(C.c_void_p), _sz, _sz, C.c_int, _f32p)
            _dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
            self._bench_outer = fn("bench_outer", C.c_int, C.c_int, _sz, _sz, C.c_int, C.c_int, C.c_int,
                                   C.c_float, C.c_float, _dp)
            self._bench_inner = fn("bench_inner", C.c_int, C.c_int, _sz, C.c_int, C.c_int, _dp)
            vp = C.c_void_p
            self._ck_read = fn("checkpoint_read", C.c_int, C.c_char_p, _sz, _sz, vp, vp, vp, vp, vp,
                               C.POINTER(_u64), C.POINTER(C.c_double), C.POINTER(_u64))
            self._ck_write = fn("checkpoint_write", C.c_int, C.c_char_p, _sz, vp, vp, vp, vp, vp,
                                C.POINTER(_u64), C.POINTER(C.c_double), C.POINTER(_u64))
            P = C.POINTER
            self._frame = fn("encode_frame", C.c_int, C.c_uint8, vp, _sz, vp, P(_sz))
            self._rpayload = fn("encode_reduce_payload", C.c_int, _u64, C.c_uint32, C.c_uint8, vp, _sz, vp, P(_sz))
            self._parse_frames = fn("parse_frames", C.c_int, vp, _sz, _sz, vp, vp, vp, vp, vp, vp, _sz, P(_sz))
            self._bench_wire = fn("bench_wire", C.c_int, C.c_int, _sz, C.c_int, _sz, C.c_int, P(C.c_double), P(_u64))

    # -- checkpoints through the reference's save/load_checkpoint (reference only) --------
    _CK_U = ("step_count", "growth_interval", "consecutive_good", "inner_step", "outer_epoch", "engines")
    _CK_D = ("beta1", "beta2", "eps", "weight_decay", "outer_lr", "outer_momentum", "scale", "clock_seconds")
    _CK_H = ("config_hash", "completed_rounds", "reduce_data_bytes")
    _CK_V = ("theta_t", "theta_local", "m", "v", "buf")

    def checkpoint_read(self, path, idx, n):
        vec = {k: np.empty(n, np.float32) for k in self._CK_V}
        u, d, h = (_u64 * 6)(), (C.c_double * 8)(), (_u64 * 3)()
        st = self._ck_read(path.encode(), idx, n, *[vec[k].ctypes.data for k in self._CK_V], u, d, h)
        if st:
            raise RuntimeError(f"ref_checkpoint_read failed with status {st}")
        out = dict(vec)
        out.update({k: int(u[i]) for i, k in enumerate(self._CK_U)})
        out.update({k: float(d[i]) for i, k in enumerate(self._CK_D)})
        out.update({k: int(h[i]) for i, k in enumerate(self._CK_H)})
        return out

    def checkpoint_write(self, path, state):
        vec = [np.ascontiguousarray(state[k], np.float32) for k in self._CK_V]
        u = (_u64 * 6)(*[int(state.get(k, 0)) for k in self._CK_U])
        d = (C.c_double * 8)(*[float(state.get(k, 0.0)) for k in self._CK_D])
        h = (_u64 * 3)(*[int(state.get(k, 0)) for k in self._CK_H])
        st = self._ck_write(path.encode(), vec[0].size, *[x.ctypes.data for x in vec], u, d, h)
        if st:
            raise RuntimeError(f"ref_checkpoint_write failed with status {st}")

    # -- codec ---------------------------------------------------------------
    def fp16_encode_scalar(self, x: float) -> int:
        return int(self._enc1(float(x)))

    def fp16_decode_scalar(self, b: int) -> float:
        return float(self._dec1(int(b)))

    def encode_fp16(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.empty(v.size, np.uint16)
        ov = self._enc(v, v.size, out)
        return out, bool(ov)

    def decode_fp16(self, b):
        b = np.ascontiguousarray(b, np.uint16)
        out = np.empty(b.size, np.float32)
        self._dec(b, b.size, out)
        return out

    # -- tensor ----------------------------------------------------------------
    def all_finite(self, v) -> bool:
        v = np.ascontiguousarray(v, np.float32)
        return bool(self._all_finite(v, v.size))

    def axpy(self, alpha, x, y):
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        out = np.empty_like(y)
        self._axpy(alpha, x, y, x.size, out)
        return out

    # -- optim -----------------------------------------------------------------
    def lr_at(self, warmup, total, base_lr, cosine, step) -> float:
        return float(self._lr_at(warmup, total, base_lr, int(cosine), step))

    def adamw_step(self, p, g, m, v, step_count, lr, b1=0.9, b2=0.95, eps=1e-8, wd=0.1):
        """Returns (status, p_new, step_count); m and v are updated in place."""
        p = np.ascontiguousarray(p, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        assert m.dtype == np.float32 and v.dtype == np.float32
        sc = _u64(step_count)
        out = np.empty_like(p)
        st = self._adamw(p, g, m, v, p.size, b1, b2, eps, wd, C.byref(sc), lr, out)
        return st, out, int(sc.value)

    def nesterov_step(self, p, g, buf, lr, mu):
        p = np.ascontiguousarray(p, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        out = np.empty_like(p)
        st = self._nest(p, g, buf, p.size, lr, mu, out)
        return st, out

    def scaler_unscale_and_check(self, scale, g):
        g = np.ascontiguousarray(g, np.float32)
        out = np.empty_like(g)
        ov = self._unscale(scale, g, g.size, out)
        return out, bool(ov)

    def scaler_update(self, scale, good, growth, overflow):
        s = C.c_float(scale)
        gd = _u64(good)
        self._scaler_update(C.byref(s), C.byref(gd), growth, int(overflow))
        return float(s.value), int(gd.value)

    # -- reduce ----------------------------------------------------------------
    def reduce_average(self, contribs, precision: int):
        cs = [np.ascontiguousarray(c, np.float32) for c in contribs]
        k, n = len(cs), (cs[0].size if cs else 0)
        arr = (C.c_void_p * max(k, 1))(*[c.ctypes.data for c in cs])
        out = np.empty(n, np.float32)
        if self.kind == "port":
            scratch = np.empty(max(k * n, 1), np.float32)
            st = self._reduce(arr, k, n, precision, scratch.ctypes.data, out)
        else:
            st = self._reduce(arr, k, n, precision, out)
        return st, out

    def partition_ranges(self, n, k):
        off = (_sz * k)()
        ln = (_sz * k)()
        self._part(n, k, off, ln)
        return [(off[i], ln[i]) for i in range(k)]

    def per_peer_reduce_bytes(self, n, k, rank, precision):
        return int(self._ppb(n, k, rank, precision))

    def fleet_reduce_bytes(self, n, k, precision):
        return int(self._fleet(n, k, precision))

    # -- wire codec (wire.cpp:10-104; collective.cpp:63-152, 1318-1345) ----------
    def encode_frame(self, msg_type: int, payload: bytes) -> bytes:
        pl = np.frombuffer(bytes(payload), np.uint8) if payload else np.zeros(1, np.uint8)
        out = np.empty(14 + len(payload), np.uint8)
        if self.kind == "port":
            self._frame(msg_type, pl.ctypes.data, len(payload), out.ctypes.data)
        else:
            used = _sz(0)
            st = self._frame(msg_type, pl.ctypes.data, len(payload), out.ctypes.data, C.byref(used))
            assert st == 0 and used.value == out.size
        return out.tobytes()

    def encode_reduce_payload(self, epoch: int, chunk_index: int, precision: int, segment: bytes) -> bytes:
        sg = np.frombuffer(bytes(segment), np.uint8) if segment else np.zeros(1, np.uint8)
        out = np.empty(13 + len(segment), np.uint8)
        if self.kind == "port":
            self._rpayload(epoch, chunk_index, precision, sg.ctypes.data, len(segment), out.ctypes.data)
        else:
            used = _sz(0)
            st = self._rpayload(epoch, chunk_index, precision, sg.ctypes.data, len(segment), out.ctypes.data,
                                C.byref(used))
            assert st == 0 and used.value == out.size
        return out.tobytes()

    # (restatement only: the reference keeps these in collective.cpp's anonymous namespace)
    def encode_chunk_segment(self, name: str, offset: int, length: int, scalars: bytes) -> bytes:
        sc = np.frombuffer(bytes(scalars), np.uint8) if scalars else np.zeros(1, np.uint8)
        out = np.empty(32 + len(name) + len(scalars), np.uint8)
        self._segment(name.encode(), len(name), offset, length, sc.ctypes.data, len(scalars), out.ctypes.data)
        return out.tobytes()

    def chunk_name(self, attempt: int, partition: int, hi: int, lo: int) -> str:
        buf = C.create_string_buffer(96)
        n = self._cname(attempt, partition, hi, lo, buf)
        return buf.raw[:n].decode()

    def send_chunk_span(self, msg_type, epoch, name, precision, global_offset, scalars, chunk_size_bytes) -> bytes:
        """The bytes send_chunk_span writes to one connection; `scalars` is an array of
        uint16 codes (FP16) or float32 values (FP32)."""
        sc = np.ascontiguousarray(scalars)
        elems = sc.size
        nm = name.encode()
        size = self._span(msg_type, epoch, nm, len(nm), precision, global_offset, sc.ctypes.data, elems,
                          chunk_size_bytes, None)
        out = np.empty(max(size, 1), np.uint8)
        self._span(msg_type, epoch, nm, len(nm), precision, global_offset, sc.ctypes.data, elems, chunk_size_bytes,
                   out.ctypes.data)
        return out[:size].tobytes()

    def parse_chunk_frames(self, data: bytes):
        """Every complete frame of `data` as a dict; stops at an incomplete tail.
        Raises ValueError (SerializationError) on a malformed frame."""
        buf = np.frombuffer(bytes(data), np.uint8) if data else np.zeros(1, np.uint8)
        out, at = [], 0
        while True:
            v = [_sz(0), C.c_uint8(0), _u64(0), C.c_uint32(0), C.c_uint8(0), _sz(0), _sz(0), _u64(0), _u64(0),
                 _sz(0), _sz(0)]
            st = self._parse(buf.ctypes.data + at, len(data) - at, *[C.byref(x) for x in v])
            if st == EAGAIN:
                return out, at
            if st != OK:
                raise ValueError(f"SerializationError at byte {at}")
            fb, ty, ep, ci, pr, no, nl, off, ln, so, sb = [x.value for x in v]
            out.append({"type": ty, "epoch": ep, "chunk_index": ci, "precision": pr,
                        "name": bytes(data[at + no:at + no + nl]).decode(errors="replace"),
                        "offset": off, "length": ln, "scalars": bytes(data[at + so:at + so + sb]),
                        "frame_offset": at, "frame_bytes": fb})
            at += fb

    def parse_frames(self, data: bytes, feed: int = 0, max_frames: int = 1 << 16):
        """Reference only: FrameParser fed in `feed`-byte pieces + decode_reduce_payload."""
        buf = np.frombuffer(bytes(data), np.uint8) if data else np.zeros(1, np.uint8)
        ty = np.zeros(max_frames, np.uint8)
        pl = np.zeros(max_frames, np.uint64)
        ep = np.zeros(max_frames, np.uint64)
        ci = np.zeros(max_frames, np.uint32)
        pr = np.zeros(max_frames, np.uint8)
        ok = np.zeros(max_frames, np.int32)
        nf = _sz(0)
        st = self._parse_frames(buf.ctypes.data, len(data), feed, ty.ctypes.data, pl.ctypes.data, ep.ctypes.data,
                                ci.ctypes.data, pr.ctypes.data, ok.ctypes.data, max_frames, C.byref(nf))
        if st == ESERIAL:
            raise ValueError("SerializationError")
        assert st == OK, st
        k = nf.value
        return [{"type": int(ty[i]), "payload_len": int(pl[i]), "epoch": int(ep[i]), "chunk_index": int(ci[i]),
                 "precision": int(pr[i]), "ok": bool(ok[i])} for i in range(k)]

    # -- CPU baseline harness (reference only) -----------------------------------
    def bench_outer(self, threads, n, k, precision, warmup, iters, lr=0.7, mu=0.9):
        """Wall seconds of each timed iteration of run_simulated's outer round over
        n parameters x k workers, split across `threads` host threads."""
        t = np.zeros(iters, np.float64)
        st = self._bench_outer(threads, n, k, precision, warmup, iters, lr, mu, t)
        if st:
            raise RuntimeError(f"ref_bench_outer failed with status {st}")
        return [float(x) for x in t]

    def bench_wire(self, threads, slice_len, precision, chunk_bytes, iters):
        """(seconds per iteration, frame bytes per iteration) of the reference's scatter-side framing."""
        t, b = C.c_double(0), _u64(0)
        st = self._bench_wire(threads, slice_len, precision, chunk_bytes, iters, C.byref(t), C.byref(b))
        if st:
            raise RuntimeError(f"ref_bench_wire failed with status {st}")
        return float(t.value), int(b.value)

    def bench_inner(self, threads, n, warmup, iters):
        """Wall seconds of each timed apply_inner_step over n parameters."""
        t = np.zeros(iters, np.float64)
        st = self._bench_inner(threads, n, warmup, iters, t)
        if st:
            raise RuntimeError(f"ref_bench_inner failed with status {st}")
        return [float(x) for x in t]


_port = None
_ref = None


def port() -> _Lib:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        _port = _Lib(PORT_SO, "orc_")
    return _port


def reference():
    """The compiled reference, or None when oracle/_ref was never built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = _Lib(REF_SO, "ref_")
    return _ref


# -- synthetic inputs, generated identically on CPU and GPU --------

def rng_key(seed: int, purpose: str, index: int) -> int:
    return int(port()._key(seed, purpose.encode(), index))


def rng_fill(seed: int, purpose: str, index: int, n: int, lo: float, hi: float, first: int = 0):
    out = np.empty(n, np.float32)
    port()._fill(rng_key(seed, purpose, index), first, n, lo, hi, out)
    return out
