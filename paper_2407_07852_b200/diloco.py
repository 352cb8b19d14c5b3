"""Python mirror of the reference DiLoCo API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/diloco/{optim,tensor,reduce,engine}.hpp): the
free functions take and return host vectors (numpy float32), optimizer state
is mutated in place, overflow is a signal and bad inputs raise the reference's
exception classes.  All arithmetic runs in libdiloco_cuda.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi as A
from ._capi import lib


# ---- errors, errors.hpp:12-51 ----------------------------------------------------------

class Error(A.DiLoCoError):
    pass


class ShapeError(Error):
    pass


class ConfigError(Error):
    pass


class NumericError(Error):
    pass


class CollectiveError(Error):
    pass


class SerializationError(Error):
    pass


class QuorumError(Error):
    """errors.hpp:42: a membership change left fewer than quorum_min workers."""


_EXC = {A.ESHAPE: ShapeError, A.ECONFIG: ConfigError, A.ENUMERIC: NumericError,
        A.ECOLLECTIVE: CollectiveError, A.ENCCL: CollectiveError, A.ESERIAL: SerializationError,
        A.EQUORUM: QuorumError}


def _check(status: int) -> None:
    if status != A.OK:
        raise _EXC.get(status, Error)(status, lib.dlc_last_error().decode(errors="replace"))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a.size else None


# ---- state types, optim.hpp:17-56 ------------------------------------------------------

@dataclass
class AdamWState:
    m: np.ndarray
    v: np.ndarray
    step_count: int = 0
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1

    @staticmethod
    def init(n: int, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1) -> "AdamWState":
        return AdamWState(np.zeros(n, np.float32), np.zeros(n, np.float32), 0, beta1, beta2, eps, weight_decay)


@dataclass
class NesterovState:
    momentum_buf: np.ndarray
    lr: float = 0.7
    momentum: float = 0.9

    @staticmethod
    def init(n: int, lr=0.7, momentum=0.9) -> "NesterovState":
        return NesterovState(np.zeros(n, np.float32), lr, momentum)


@dataclass
class LrSchedule:
    warmup_steps: int = 1000
    total_steps: int = 0
    base_lr: float = 4e-4
    decay: int = A.LR_NONE


@dataclass
class LossScaler:
    scale: float = 65536.0
    growth_interval: int = 2000
    consecutive_good: int = 0


# ---- free functions --------------------------------------------------------------------

def axpy(alpha: float, x, y) -> np.ndarray:
    """tensor.hpp:108 — y + alpha * x."""
    x, y = _f32(x), _f32(y)
    if x.shape != y.shape:
        raise ShapeError(A.ESHAPE, "axpy: layout mismatch")
    out = np.empty_like(y)
    _check(lib.dlc_axpy(alpha, _ptr(x), _ptr(y), x.size, _ptr(out)))
    return out


def encode_fp16(v):
    """tensor.hpp:111 — (codes uint16, overflow flag)."""
    v = _f32(v)
    out = np.empty(v.size, np.uint16)
    ov = C.c_int(0)
    _check(lib.dlc_encode_fp16(_ptr(v), v.size, _ptr(out), C.byref(ov)))
    return out, bool(ov.value)


def decode_fp16(bits) -> np.ndarray:
    """tensor.hpp:115."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty(b.size, np.float32)
    _check(lib.dlc_decode_fp16(_ptr(b), b.size, _ptr(out)))
    return out


def all_finite(v) -> bool:
    v = _f32(v)
    r = C.c_int(1)
    _check(lib.dlc_all_finite(_ptr(v), v.size, C.byref(r)))
    return bool(r.value)


def lr_at(schedule: LrSchedule, step: int) -> float:
    """optim.hpp:49."""
    s = A.LrSchedule(schedule.warmup_steps, schedule.total_steps, schedule.base_lr, schedule.decay)
    return float(lib.dlc_lr_at(C.byref(s), step))


def adamw_step(state: AdamWState, params, grad, lr: float) -> np.ndarray:
    """optim.hpp:61-62 — returns new params; state.m/v/step_count updated in place."""
    p, g = _f32(params), _f32(grad)
    if p.shape != g.shape or p.shape != state.m.shape:
        raise ShapeError(A.ESHAPE, "adamw_step: layout mismatch")
    st = A.AdamWState(state.m.ctypes.data, state.v.ctypes.data, state.step_count, state.beta1, state.beta2,
                      state.eps, state.weight_decay)
    out = np.empty_like(p)
    _check(lib.dlc_adamw_step(C.byref(st), _ptr(p), _ptr(g), p.size, lr, _ptr(out)))
    state.step_count = int(st.step_count)
    return out


def nesterov_step(state: NesterovState, params, pseudo_grad) -> np.ndarray:
    """optim.hpp:65-66."""
    p, g = _f32(params), _f32(pseudo_grad)
    if p.shape != g.shape or p.shape != state.momentum_buf.shape:
        raise ShapeError(A.ESHAPE, "nesterov_step: layout mismatch")
    st = A.NesterovState(state.momentum_buf.ctypes.data, state.lr, state.momentum)
    out = np.empty_like(p)
    _check(lib.dlc_nesterov_step(C.byref(st), _ptr(p), _ptr(g), p.size, _ptr(out)))
    return out


def scaler_unscale_and_check(scaler: LossScaler, grad):
    """optim.hpp:76-77 — (unscaled grad, overflow)."""
    g = _f32(grad)
    s = A.LossScaler(scaler.scale, scaler.growth_interval, scaler.consecutive_good)
    out = np.empty_like(g)
    ov = C.c_int(0)
    _check(lib.dlc_scaler_unscale_and_check(C.byref(s), _ptr(g), g.size, _ptr(out), C.byref(ov)))
    return out, bool(ov.value)


def scaler_update(scaler: LossScaler, overflow: bool) -> None:
    """optim.hpp:80."""
    s = A.LossScaler(scaler.scale, scaler.growth_interval, scaler.consecutive_good)
    lib.dlc_scaler_update(C.byref(s), int(bool(overflow)))
    scaler.scale, scaler.consecutive_good = float(s.scale), int(s.consecutive_good)


def reduce_average(contributions, precision: int) -> np.ndarray:
    """reduce.hpp:65-66."""
    cs = [_f32(c) for c in contributions]
    if any(c.shape != cs[0].shape for c in cs):
        raise ShapeError(A.ESHAPE, "reduce_average: contribution layout mismatch")
    n = cs[0].size if cs else 0
    arr = (C.c_void_p * max(len(cs), 1))(*[c.ctypes.data for c in cs])
    out = np.empty(n, np.float32)
    _check(lib.dlc_reduce_average(arr, len(cs), n, precision, _ptr(out)))
    return out


def partition_ranges(n: int, k: int):
    off, ln = (C.c_size_t * k)(), (C.c_size_t * k)()
    lib.dlc_partition_ranges(n, k, off, ln)
    return [(off[i], ln[i]) for i in range(k)]


def per_peer_reduce_bytes(n, k, rank, precision) -> int:
    return int(lib.dlc_per_peer_reduce_bytes(n, k, rank, precision))


def fleet_reduce_bytes(n, k, precision) -> int:
    return int(lib.dlc_fleet_reduce_bytes(n, k, precision))


def rng_key(seed: int, purpose: str, index: int) -> int:
    return int(lib.dlc_rng_key(seed, purpose.encode(), index))


def device_count() -> int:
    c = C.c_int(0)
    _check(lib.dlc_device_count(C.byref(c)))
    return c.value


# ---- collective plugin, reduce.hpp:86-106 ----------------------------------------------

class Collective:
    handle: C.c_void_p

    def world_size(self) -> int:
        return int(lib.dlc_collective_world_size(self.handle))

    def rank(self) -> int:
        return int(lib.dlc_collective_rank(self.handle))

    def all_reduce_avg(self, delta, precision: int, outer_epoch: int = 0):
        """Collective::all_reduce_avg on a host pseudo-gradient -> (mean, ReduceReport)."""
        d = _f32(delta)
        out = np.empty_like(d)
        rep = A.ReduceReport()
        _check(lib.dlc_collective_all_reduce_avg(self.handle, _ptr(d), d.size, precision, outer_epoch,
                                                 _ptr(out), C.byref(rep)))
        return out, rep

    def close(self):
        if getattr(self, "handle", None):
            _check(lib.dlc_collective_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SoloCollective(Collective):
    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.dlc_collective_create_solo(device, C.byref(h)))
        self.handle = h


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.dlc_nccl_unique_id(buf))
    return buf.raw


class NcclCollective(Collective):
    """One rank per process and GPU over NCCL (NVLink / NVSwitch)."""

    def __init__(self, rank: int, world: int, unique_id: bytes, device: int, mode: int = A.MODE_ORDERED):
        h = C.c_void_p()
        _check(lib.dlc_collective_create_nccl(rank, world, unique_id, device, mode, C.byref(h)))
        self.handle = h
        self.mode = mode

    def shrink(self, exclude, quorum_min: int = 1, abort: bool = False) -> "NcclCollective":
        """Survivors-only membership change (collective.cpp:1369-1395): a new collective
        over this world minus `exclude` (ranks of this collective).  Raises
        CollectiveError("excluded from round") on an excluded caller and QuorumError
        below quorum_min."""
        ex = (C.c_int * max(len(exclude), 1))(*exclude)
        h = C.c_void_p()
        _check(lib.dlc_collective_shrink(self.handle, ex, len(exclude), quorum_min,
                                         A.SHRINK_ABORT if abort else A.SHRINK_DEFAULT, C.byref(h)))
        n = NcclCollective.__new__(NcclCollective)
        n.handle = h
        n.mode = self.mode
        return n

    def members(self):
        """Original ranks of the current members, sorted (the round's contributors)."""
        buf = (C.c_int * 32)()
        k = int(lib.dlc_collective_members(self.handle, buf, 32))
        return [int(buf[i]) for i in range(k)]

    def set_reduce_timeout_ms(self, ms: int) -> None:
        """NodeOptions::reduce_timeout_ms: the P2P barriers' failure detector."""
        _check(lib.dlc_collective_set_reduce_timeout_ms(self.handle, ms))

    def inject_stall(self, barrier_index: int) -> None:
        """Fault injection (set_stage_hook): stop arriving from the n-th P2P barrier on."""
        _check(lib.dlc_collective_inject_stall(self.handle, barrier_index))


# ---- device-resident engine, engine.hpp:76-157 ------------------------------------------

@dataclass
class DilocoConfig:
    """engine.hpp:22-32."""
    local_steps_h: int = 500
    num_workers_k: int = 1
    reduce_precision: int = A.FP32
    total_inner_steps: int = 500


@dataclass
class OptimHyperparams:
    """engine.hpp:34-46."""
    inner_lr: float = 4e-4
    warmup_steps: int = 1000
    lr_decay: int = A.LR_NONE
    weight_decay: float = 0.1
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    outer_lr: float = 0.7
    outer_momentum: float = 0.9
    scaler_init_scale: float = 65536.0
    scaler_growth_interval: int = 2000


@dataclass
class InnerStepResult:
    lr: float
    overflow_skipped: bool


@dataclass
class OuterStepResult:
    applied: bool
    outer_epoch: int
    report: object = field(default=None)


class DilocoEngine:
    """Device-resident DilocoEngine: all state in HBM on `device`."""

    def __init__(self, config: DilocoConfig, hyper: OptimHyperparams, n_params: int, device: int = 0,
                 inner_mode: int = A.INNER_PINGPONG):
        cfg = A.Config(config.local_steps_h, config.num_workers_k, config.reduce_precision,
                       config.total_inner_steps)
        hp = A.Hyperparams(hyper.inner_lr, hyper.warmup_steps, hyper.lr_decay, hyper.weight_decay, hyper.beta1,
                           hyper.beta2, hyper.adam_eps, hyper.outer_lr, hyper.outer_momentum,
                           hyper.scaler_init_scale, hyper.scaler_growth_interval)
        h = C.c_void_p()
        _check(lib.dlc_engine_create(C.byref(cfg), C.byref(hp), n_params, device, inner_mode, C.byref(h)))
        self.handle = h
        self.n = n_params
        self.device = device
        self.config = config
        self.hyper = hyper

    # buffers
    def upload(self, which: int, host) -> None:
        a = _f32(host)
        _check(lib.dlc_engine_upload(self.handle, which, _ptr(a), a.size))

    def download(self, which: int) -> np.ndarray:
        out = np.empty(self.n, np.float32)
        _check(lib.dlc_engine_download(self.handle, which, _ptr(out), self.n))
        return out

    def download_range(self, which: int, offset: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float32)
        _check(lib.dlc_engine_download_range(self.handle, which, offset, _ptr(out), count))
        return out

    def upload_range(self, which: int, offset: int, host) -> None:
        a = _f32(host)
        _check(lib.dlc_engine_upload_range(self.handle, which, offset, _ptr(a), a.size))

    def device_ptr(self, which: int) -> int:
        p = C.c_void_p()
        _check(lib.dlc_engine_device_ptr(self.handle, which, C.byref(p)))
        return int(p.value or 0)

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib.dlc_engine_stream(self.handle, C.byref(s)))
        return int(s.value or 0)

    def scalars(self) -> A.EngineScalars:
        s = A.EngineScalars()
        _check(lib.dlc_engine_get_scalars(self.handle, C.byref(s)))
        return s

    def set_scalars(self, s: A.EngineScalars) -> None:
        _check(lib.dlc_engine_set_scalars(self.handle, C.byref(s)))

    def synchronize(self) -> None:
        _check(lib.dlc_engine_synchronize(self.handle))

    # steps
    def inner_step(self, grad_dev_ptr: int, grad_is_scaled: bool = True, wait: bool = False):
        res = A.InnerResult() if wait else None
        _check(lib.dlc_engine_inner_step(self.handle, C.c_void_p(grad_dev_ptr), int(grad_is_scaled),
                                         C.byref(res) if wait else None))
        return InnerStepResult(float(res.lr), bool(res.overflow_skipped)) if wait else None

    def inner_step_host(self, grad, grad_is_scaled: bool = False) -> InnerStepResult:
        g = _f32(grad)
        res = A.InnerResult()
        _check(lib.dlc_engine_inner_step_host(self.handle, _ptr(g), int(grad_is_scaled), C.byref(res)))
        return InnerStepResult(float(res.lr), bool(res.overflow_skipped))

    def outer_step(self, collective: Collective | None = None, wait: bool = False, report: bool = False):
        res = A.OuterResult()
        rep = A.ReduceReport() if report else None
        _check(lib.dlc_engine_outer_step(self.handle, collective.handle if collective else None,
                                         C.byref(res) if (wait or report) else None,
                                         C.byref(rep) if report else None))
        if wait or report:
            return OuterStepResult(bool(res.applied), int(res.outer_epoch), rep)
        return None

    def outer_step_host(self, collective, theta_local, theta_t_out) -> OuterStepResult:
        """theta_local / theta_t_out: host arrays (pinned for async copies) or raw pointers."""
        src = theta_local if isinstance(theta_local, int) else _f32(theta_local).ctypes.data
        dst = theta_t_out if isinstance(theta_t_out, int) else theta_t_out.ctypes.data
        res = A.OuterResult()
        _check(lib.dlc_engine_outer_step_host(self.handle, collective.handle if collective else None,
                                              C.c_void_p(src), C.c_void_p(dst), C.byref(res)))
        return OuterStepResult(bool(res.applied), int(res.outer_epoch))

    def outer_step_from(self, collective, theta_local_dev_ptr: int, wait: bool = False):
        res = A.OuterResult()
        _check(lib.dlc_engine_outer_step_from(self.handle, collective.handle if collective else None,
                                              C.c_void_p(theta_local_dev_ptr), C.byref(res) if wait else None,
                                              None))
        return OuterStepResult(bool(res.applied), int(res.outer_epoch)) if wait else None

    def compute_pseudo_gradient(self):
        """DilocoEngine::compute_pseudo_gradient (engine.cpp:115-126): (FP32 delta on the host, outer epoch)."""
        out = np.empty(self.n, np.float32)
        ep = C.c_uint64(0)
        _check(lib.dlc_engine_compute_pseudo_gradient(self.handle, _ptr(out), C.byref(ep)))
        return out, int(ep.value)

    def apply_outer_step(self, mean, outer_epoch: int) -> OuterStepResult:
        """DilocoEngine::outer_step (engine.cpp:128-146) on a host FP32 mean from any collective."""
        m = _f32(mean)
        if m.size != self.n:
            raise ShapeError(A.ESHAPE, "apply_outer_step: length mismatch")
        res = A.OuterResult()
        _check(lib.dlc_engine_apply_outer_step(self.handle, _ptr(m), outer_epoch, C.byref(res)))
        return OuterStepResult(bool(res.applied), int(res.outer_epoch))

    # -- wire rounds (include/diloco_cuda.h section 5; paper_2407_07852_b200/wire.py) --
    def wire_begin(self) -> int:
        ep = C.c_uint64(0)
        _check(lib.dlc_engine_wire_begin(self.handle, C.byref(ep)))
        return int(ep.value)

    def wire_encode(self, which: int, offset: int, length: int, tags: A.WireTags, out=None) -> np.ndarray:
        """Frames of DELTA / MEAN [offset, offset + length) as a uint8 array (or into `out`)."""
        size = C.c_size_t(0)
        _check(lib.dlc_wire_frames_size(length, C.byref(tags), C.byref(size), None))
        if out is None:
            out = np.empty(max(size.value, 1), np.uint8)
        used = C.c_size_t(0)
        _check(lib.dlc_engine_wire_encode(self.handle, which, offset, length, C.byref(tags),
                                          C.c_void_p(out.ctypes.data), out.nbytes, C.byref(used)))
        return out[:used.value]

    def wire_decode(self, which: int, row: int, base_offset: int, capacity: int, data, max_chunks: int = 4096):
        """Returns (list of WireChunk, bytes consumed)."""
        buf = np.frombuffer(data, np.uint8) if not isinstance(data, np.ndarray) else data
        chunks = (A.WireChunk * max_chunks)()
        nc, used = C.c_size_t(0), C.c_size_t(0)
        _check(lib.dlc_engine_wire_decode(self.handle, which, row, base_offset, capacity,
                                          C.c_void_p(buf.ctypes.data) if buf.size else None, buf.nbytes, chunks,
                                          max_chunks, C.byref(nc), C.byref(used)))
        return [chunks[i] for i in range(min(nc.value, max_chunks))], int(used.value)

    def wire_fold(self, rank: int, k: int, offset: int, length: int) -> None:
        _check(lib.dlc_engine_wire_fold(self.handle, rank, k, offset, length))

    def wire_finish(self, outer_epoch: int) -> OuterStepResult:
        res = A.OuterResult()
        _check(lib.dlc_engine_wire_finish(self.handle, outer_epoch, C.byref(res)))
        return OuterStepResult(bool(res.applied), int(res.outer_epoch))

    def set_fused_delta(self, on: bool) -> None:
        """K2 fused into the window's last inner step (opt-in; K > 1)."""
        _check(lib.dlc_engine_set_fused_delta(self.handle, int(on)))

    def set_timing(self, on: bool) -> None:
        _check(lib.dlc_engine_set_timing(self.handle, int(on)))

    def phase_times(self):
        """(ms[4], count[4]) per phase: inner AdamW, pseudo-grad, collective, outer Nesterov."""
        ms = (C.c_double * 4)()
        cnt = (C.c_uint64 * 4)()
        _check(lib.dlc_engine_phase_times(self.handle, ms, cnt))
        return list(ms), list(cnt)

    def rng_fill(self, which: int, seed: int, purpose: str, index: int, lo: float, hi: float, first: int = 0):
        _check(lib.dlc_rng_fill_device(self.handle, which, rng_key(seed, purpose, index), first, lo, hi))

    def rng_perturb(self, seed: int, purpose: str, index: int, lo: float, hi: float, dst_dev_ptr: int = 0):
        """dst (default: the engine's theta_local) = theta_t - U(lo, hi)."""
        _check(lib.dlc_rng_perturb(self.handle, C.c_void_p(dst_dev_ptr or None), rng_key(seed, purpose, index),
                                   lo, hi))

    def close(self):
        if getattr(self, "handle", None):
            if getattr(self, "_owned", True):
                _check(lib.dlc_engine_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class World:
    """Single-process world (include/diloco_cuda.h): K engines driven by one host
    thread, the device analogue of run_simulated's K workers (netsim.cpp:325-357).
    In DLC_MODE_P2P several ranks may share a device (``devices=[0] * k``): the
    ranks then synchronise through CUDA events, and the whole P2P data plane
    (piece pipeline, TMA owner fold, finish gate) runs on one GPU."""

    def __init__(self, config: DilocoConfig, hyper: OptimHyperparams, n_params: int, devices,
                 inner_mode: int = A.INNER_PINGPONG, mode: int = A.MODE_P2P):
        cfg = A.Config(config.local_steps_h, config.num_workers_k, config.reduce_precision,
                       config.total_inner_steps)
        hp = A.Hyperparams(hyper.inner_lr, hyper.warmup_steps, hyper.lr_decay, hyper.weight_decay, hyper.beta1,
                           hyper.beta2, hyper.adam_eps, hyper.outer_lr, hyper.outer_momentum,
                           hyper.scaler_init_scale, hyper.scaler_growth_interval)
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(lib.dlc_world_create(C.byref(cfg), C.byref(hp), n_params, devs, inner_mode, mode, C.byref(h)))
        self.handle = h
        self.engines = []
        for r, d in enumerate(devices):
            eh = C.c_void_p()
            _check(lib.dlc_world_engine(h, r, C.byref(eh)))
            e = DilocoEngine.__new__(DilocoEngine)
            e.handle, e.n, e.device, e.config, e.hyper, e._owned = eh, n_params, d, config, hyper, False
            self.engines.append(e)

    def outer_step(self, wait: bool = True):
        if not wait:
            _check(lib.dlc_world_outer_step(self.handle, None))
            return None
        res = A.OuterResult()
        _check(lib.dlc_world_outer_step(self.handle, C.byref(res)))
        return OuterStepResult(bool(res.applied), int(res.outer_epoch))

    def shrink(self, exclude, quorum_min: int = 0) -> None:
        """dlc_world_shrink: the next rounds run over the ranks not in `exclude`
        (survivor order and divisor, collective.cpp:1369-1395); the excluded
        engines are destroyed."""
        ex = list(exclude)
        arr = (C.c_int * max(len(ex), 1))(*ex)
        _check(lib.dlc_world_shrink(self.handle, arr, len(ex), quorum_min))
        dropped = set(ex)
        for r, e in enumerate(self.engines):
            if r in dropped:
                e.handle = None
        self.engines = [e for r, e in enumerate(self.engines) if r not in dropped]

    def members(self) -> list:
        """Original ranks of the current members."""
        buf = (C.c_int * 32)()
        n = lib.dlc_world_members(self.handle, buf, 32)
        return [buf[i] for i in range(n)]

    def close(self):
        if getattr(self, "handle", None):
            for e in self.engines:
                e.handle = None
            _check(lib.dlc_world_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def set_p2p_tuning(plan=None, fold_ctas: int = 0, fold_threads: int = 0, piece_ctas: int = 0,
                   fold_kernel: int = 0) -> None:
    """dlc_p2p_set_tuning: override the measured DLC_MODE_P2P defaults (sweeps);
    no arguments restores them."""
    if plan is None and not (fold_ctas or fold_threads or piece_ctas or fold_kernel):
        _check(lib.dlc_p2p_set_tuning(None))
        return
    t = A.P2PTuning()
    plan = list(plan or [])
    t.plan_len = len(plan)
    for i, v in enumerate(plan):
        t.plan[i] = int(v)
    t.fold_ctas, t.fold_threads, t.piece_ctas, t.fold_kernel = fold_ctas, fold_threads, piece_ctas, fold_kernel
    _check(lib.dlc_p2p_set_tuning(C.byref(t)))


def outer_step_local(engines) -> OuterStepResult:
    """K in-process engines on one device: run_simulated's outer round (netsim.cpp:325-357)."""
    arr = (C.c_void_p * len(engines))(*[e.handle.value for e in engines])
    res = A.OuterResult()
    _check(lib.dlc_engines_outer_step_local(arr, len(engines), C.byref(res)))
    return OuterStepResult(bool(res.applied), int(res.outer_epoch))


def checkpoint_save(engines, path: str, config_hash: int = 0, completed_rounds: int = 0,
                    clock_seconds: float = 0.0, reduce_data_bytes: int = 0, ledger=None, segments=None) -> None:
    """save_checkpoint (checkpoint.cpp:131-160) of device engines in the ODLCKPT1 format.

    ledger: optional [(compute_s, comm_s, idle_s), ...]; segments: optional
    [(name, length), ...] Layout (default one segment "p")."""
    arr = (C.c_void_p * len(engines))(*[e.handle.value for e in engines])
    led = np.ascontiguousarray(ledger if ledger is not None else np.zeros((0, 3)), np.float64).reshape(-1)
    meta = A.CheckpointMeta(config_hash, completed_rounds, clock_seconds, reduce_data_bytes, led.size // 3,
                            led.ctypes.data_as(C.POINTER(C.c_double)) if led.size else None)
    names = lens = None
    nseg = 0
    if segments:
        nseg = len(segments)
        names = (C.c_char_p * nseg)(*[s[0].encode() for s in segments])
        lens = (C.c_uint64 * nseg)(*[int(s[1]) for s in segments])
    _check(lib.dlc_checkpoint_save(arr, len(engines), path.encode(), C.byref(meta), names, lens, nseg))


def checkpoint_load(engines, path: str, segments=None) -> dict:
    """load_checkpoint (checkpoint.cpp:162-198) into device engines, all or nothing;
    returns the header fields.  segments: optional [(name, length), ...] Layout
    every vector must carry (restore_state, engine.cpp:148-155)."""
    arr = (C.c_void_p * len(engines))(*[e.handle.value for e in engines])
    meta = A.CheckpointMeta()
    if segments:
        nseg = len(segments)
        names = (C.c_char_p * nseg)(*[s[0].encode() for s in segments])
        lens = (C.c_uint64 * nseg)(*[int(s[1]) for s in segments])
        _check(lib.dlc_checkpoint_load_layout(arr, len(engines), path.encode(), names, lens, nseg, C.byref(meta)))
    else:
        _check(lib.dlc_checkpoint_load(arr, len(engines), path.encode(), C.byref(meta)))
    return {"config_hash": int(meta.config_hash), "completed_rounds": int(meta.completed_rounds),
            "clock_seconds": float(meta.clock_seconds), "reduce_data_bytes": int(meta.reduce_data_bytes),
            "ledger_workers": int(meta.ledger_workers)}


def run_training(engine: "DilocoEngine", collective=None, producer=None, sink=None, on_round=None,
                 worker_index: int = 0) -> dict:
    """run_training (engine.cpp:176-240) on a device engine.

    producer(inner_step) -> (grad_device_ptr, grad_is_scaled, loss): the
    gradient producer (task.cpp, out of scope).  sink(record: dict) receives the
    MetricsRecord stream; on_round(rounds_done) fires after every outer round.
    Returns the RunResult fields as a dict."""
    errors = []

    def _producer(_user, step, grad_out, scaled_out, loss_out):
        try:
            g, scaled, loss = producer(int(step))
            grad_out[0] = C.c_void_p(int(g))
            scaled_out[0] = int(bool(scaled))
            loss_out[0] = float(loss)
            return 0
        except Exception as e:  # reported after the call
            errors.append(e)
            return 1

    def _sink(_user, rec):
        r = rec.contents
        sink({"kind": ("step", "round", "event")[r.kind], "worker": r.worker, "inner_step": r.inner_step,
              "outer_epoch": r.outer_epoch, "loss": r.loss, "perplexity": r.perplexity, "lr": r.lr,
              "compute_ms": r.compute_ms, "comm_ms": r.comm_ms, "bytes_sent": r.bytes_sent,
              "contributors": r.contributors, "event": r.event.decode() if r.event else ""})

    def _round(_user, n):
        on_round(int(n))

    cb_p = A.GRAD_PRODUCER(_producer)
    cb_s = A.METRICS_SINK(_sink) if sink else A.METRICS_SINK()
    cb_r = A.ROUND_HOOK(_round) if on_round else A.ROUND_HOOK()
    res = A.RunResult()
    st = lib.dlc_run_training(engine.handle, collective.handle if collective is not None else None, cb_p, cb_s, cb_r,
                              None, worker_index, C.byref(res))
    if errors:
        raise errors[0]
    _check(st)
    return {f: getattr(res, f) for f, _ in A.RunResult._fields_}


class DilocoOptimizer:
    """Single-optimizer facade (engine.hpp:122-140; paper Fig. 2)."""

    def __init__(self, engine: DilocoEngine, collective: Collective | None = None):
        self.engine = engine
        self.collective = collective
        self.round_just_completed = False

    def step(self, grad_dev_ptr: int, grad_is_scaled: bool = True) -> None:
        done = C.c_int(0)
        _check(lib.dlc_optimizer_step(self.engine.handle, self.collective.handle if self.collective else None,
                                      C.c_void_p(grad_dev_ptr), int(grad_is_scaled), C.byref(done)))
        self.round_just_completed = bool(done.value)

    def zero_grad(self) -> None:
        pass


def fp16_encode_bits(start: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint16)
    _check(lib.dlc_fp16_encode_bits(start, n, _ptr(out)))
    return out
