"""ctypes binding of include/diloco_cuda.h (libdiloco_cuda.so, built in-tree).

This is the reference-side binding a Python integrator would write; the C++
reference binds the same symbols directly.  There is no
fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdiloco_cuda.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "diloco_cuda.h")

OK, ESHAPE, ECONFIG, ENUMERIC, ECOLLECTIVE, ECUDA, ENCCL, EINVAL, ESERIAL, EQUORUM = range(10)
SHRINK_DEFAULT, SHRINK_ABORT = 0, 1
FP32, FP16 = 0, 1
LR_NONE, LR_COSINE = 0, 1
MODE_ORDERED, MODE_ALLREDUCE, MODE_P2P = 0, 1, 2
INNER_PINGPONG, INNER_INPLACE = 0, 1
THETA_T, THETA_LOCAL, ADAM_M, ADAM_V, MOMENTUM, GRAD = range(6)
MSG_REDUCE_CHUNK, MSG_REDUCE_RESULT = 5, 6
WIRE_DELTA, WIRE_MEAN, WIRE_ROW = range(3)


class AdamWState(C.Structure):
    _fields_ = [("m", C.c_void_p), ("v", C.c_void_p), ("step_count", C.c_uint64), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float)]


class NesterovState(C.Structure):
    _fields_ = [("momentum_buf", C.c_void_p), ("lr", C.c_float), ("momentum", C.c_float)]


class LrSchedule(C.Structure):
    _fields_ = [("warmup_steps", C.c_uint64), ("total_steps", C.c_uint64), ("base_lr", C.c_float),
                ("decay", C.c_int)]


class LossScaler(C.Structure):
    _fields_ = [("scale", C.c_float), ("growth_interval", C.c_uint64), ("consecutive_good", C.c_uint64)]


class ReduceReport(C.Structure):
    _fields_ = [("outer_epoch", C.c_uint64), ("contributors", C.c_size_t), ("data_bytes_sent", C.c_uint64),
                ("data_bytes_received", C.c_uint64), ("wire_bytes_sent", C.c_uint64),
                ("wire_bytes_received", C.c_uint64), ("wall_ms", C.c_double), ("attempts", C.c_uint32)]


class P2PTuning(C.Structure):
    _fields_ = [("plan", C.c_uint32 * 32), ("plan_len", C.c_uint32), ("fold_ctas", C.c_int32),
                ("fold_threads", C.c_int32), ("piece_ctas", C.c_int32), ("fold_kernel", C.c_int32)]


class WireTags(C.Structure):
    _fields_ = [("msg_type", C.c_uint8), ("precision", C.c_int), ("outer_epoch", C.c_uint64),
                ("attempt", C.c_uint32), ("partition", C.c_uint32), ("from_hi", C.c_uint64),
                ("from_lo", C.c_uint64), ("chunk_size_bytes", C.c_uint64)]


class WireChunk(C.Structure):
    _fields_ = [("msg_type", C.c_uint8), ("precision", C.c_uint8), ("accepted", C.c_int),
                ("chunk_index", C.c_uint32), ("attempt", C.c_uint32), ("partition", C.c_uint32),
                ("outer_epoch", C.c_uint64), ("from_hi", C.c_uint64), ("from_lo", C.c_uint64),
                ("offset", C.c_uint64), ("length", C.c_uint64), ("frame_offset", C.c_uint64),
                ("frame_bytes", C.c_uint64)]


class MetricsRecord(C.Structure):
    _fields_ = [("kind", C.c_int), ("worker", C.c_int), ("inner_step", C.c_uint64), ("outer_epoch", C.c_uint64),
                ("loss", C.c_float), ("perplexity", C.c_float), ("lr", C.c_float), ("compute_ms", C.c_double),
                ("comm_ms", C.c_double), ("bytes_sent", C.c_uint64), ("contributors", C.c_size_t),
                ("event", C.c_char_p)]


class RunResult(C.Structure):
    _fields_ = [("steps_done", C.c_uint64), ("rounds_done", C.c_uint64), ("final_train_loss", C.c_float),
                ("reduce_data_bytes", C.c_uint64), ("reduce_wire_bytes", C.c_uint64), ("comm_ms", C.c_double),
                ("compute_ms", C.c_double)]


GRAD_PRODUCER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                            C.POINTER(C.c_float))
METRICS_SINK = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(MetricsRecord))
ROUND_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64)
RECORD_STEP, RECORD_ROUND, RECORD_EVENT = 0, 1, 2


class Config(C.Structure):
    _fields_ = [("local_steps_h", C.c_uint64), ("num_workers_k", C.c_size_t), ("reduce_precision", C.c_int),
                ("total_inner_steps", C.c_uint64)]


class Hyperparams(C.Structure):
    _fields_ = [("inner_lr", C.c_float), ("warmup_steps", C.c_uint64), ("lr_decay", C.c_int),
                ("weight_decay", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
                ("outer_lr", C.c_float), ("outer_momentum", C.c_float), ("scaler_init_scale", C.c_float),
                ("scaler_growth_interval", C.c_uint64)]


class EngineScalars(C.Structure):
    _fields_ = [("step_count", C.c_uint64), ("inner_step", C.c_uint64), ("outer_epoch", C.c_uint64),
                ("scale", C.c_float), ("consecutive_good", C.c_uint64), ("overflow_skips", C.c_uint64),
                ("outer_skips", C.c_uint64), ("last_lr", C.c_float), ("last_overflow", C.c_int),
                ("last_applied", C.c_int)]


class CheckpointMeta(C.Structure):
    _fields_ = [("config_hash", C.c_uint64), ("completed_rounds", C.c_uint64), ("clock_seconds", C.c_double),
                ("reduce_data_bytes", C.c_uint64), ("ledger_workers", C.c_size_t),
                ("ledger", C.POINTER(C.c_double))]


class InnerResult(C.Structure):
    _fields_ = [("lr", C.c_float), ("overflow_skipped", C.c_int)]


class OuterResult(C.Structure):
    _fields_ = [("applied", C.c_int), ("outer_epoch", C.c_uint64)]


P = C.c_void_p
SZ = C.c_size_t
I = C.c_int
F = C.c_float
U64 = C.c_uint64
PP = C.POINTER(C.c_void_p)

_SIGS = {
    "dlc_abi_version": (I, []),
    "dlc_last_error": (C.c_char_p, []),
    "dlc_device_count": (I, [C.POINTER(I)]),
    "dlc_set_device": (I, [I]),
    "dlc_axpy": (I, [F, P, P, SZ, P]),
    "dlc_encode_fp16": (I, [P, SZ, P, C.POINTER(I)]),
    "dlc_decode_fp16": (I, [P, SZ, P]),
    "dlc_all_finite": (I, [P, SZ, C.POINTER(I)]),
    "dlc_lr_at": (F, [C.POINTER(LrSchedule), U64]),
    "dlc_adamw_step": (I, [C.POINTER(AdamWState), P, P, SZ, F, P]),
    "dlc_nesterov_step": (I, [C.POINTER(NesterovState), P, P, SZ, P]),
    "dlc_scaler_scale_loss": (F, [C.POINTER(LossScaler), F]),
    "dlc_scaler_unscale_and_check": (I, [C.POINTER(LossScaler), P, SZ, P, C.POINTER(I)]),
    "dlc_scaler_update": (None, [C.POINTER(LossScaler), I]),
    "dlc_reduce_average": (I, [PP, SZ, SZ, I, P]),
    "dlc_partition_ranges": (None, [SZ, SZ, C.POINTER(SZ), C.POINTER(SZ)]),
    "dlc_per_peer_reduce_bytes": (U64, [SZ, SZ, SZ, I]),
    "dlc_fleet_reduce_bytes": (U64, [SZ, SZ, I]),
    "dlc_nccl_unique_id": (I, [C.c_char_p]),
    "dlc_collective_create_nccl": (I, [I, I, C.c_char_p, I, I, C.POINTER(P)]),
    "dlc_collective_create_solo": (I, [I, C.POINTER(P)]),
    "dlc_collective_destroy": (I, [P]),
    "dlc_collective_world_size": (SZ, [P]),
    "dlc_collective_rank": (I, [P]),
    "dlc_collective_all_reduce_avg": (I, [P, P, SZ, I, U64, P, C.POINTER(ReduceReport)]),
    "dlc_collective_shrink": (I, [P, C.POINTER(I), SZ, SZ, I, C.POINTER(P)]),
    "dlc_collective_members": (SZ, [P, C.POINTER(I), SZ]),
    "dlc_collective_set_reduce_timeout_ms": (I, [P, U64]),
    "dlc_collective_inject_stall": (I, [P, C.c_int64]),
    "dlc_hyperparams_default": (None, [C.POINTER(Hyperparams)]),
    "dlc_engine_create": (I, [C.POINTER(Config), C.POINTER(Hyperparams), SZ, I, I, C.POINTER(P)]),
    "dlc_engine_destroy": (I, [P]),
    "dlc_engine_size": (SZ, [P]),
    "dlc_engine_stream": (I, [P, C.POINTER(P)]),
    "dlc_engine_upload": (I, [P, I, P, SZ]),
    "dlc_engine_download": (I, [P, I, P, SZ]),
    "dlc_engine_download_range": (I, [P, I, SZ, P, SZ]),
    "dlc_engine_upload_range": (I, [P, I, SZ, P, SZ]),
    "dlc_engine_device_ptr": (I, [P, I, C.POINTER(P)]),
    "dlc_engine_get_scalars": (I, [P, C.POINTER(EngineScalars)]),
    "dlc_engine_set_scalars": (I, [P, C.POINTER(EngineScalars)]),
    "dlc_engine_synchronize": (I, [P]),
    "dlc_engine_inner_step": (I, [P, P, I, C.POINTER(InnerResult)]),
    "dlc_engine_inner_step_host": (I, [P, P, I, C.POINTER(InnerResult)]),
    "dlc_engine_outer_step": (I, [P, P, C.POINTER(OuterResult), C.POINTER(ReduceReport)]),
    "dlc_engine_outer_step_host": (I, [P, P, P, P, C.POINTER(OuterResult)]),
    "dlc_engine_outer_step_from": (I, [P, P, P, C.POINTER(OuterResult), C.POINTER(ReduceReport)]),
    "dlc_engine_compute_pseudo_gradient": (I, [P, P, C.POINTER(C.c_uint64)]),
    "dlc_engine_apply_outer_step": (I, [P, P, C.c_uint64, C.POINTER(OuterResult)]),
    "dlc_engine_set_timing": (I, [P, I]),
    "dlc_engine_set_fused_delta": (I, [P, I]),
    "dlc_engine_phase_times": (I, [P, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "dlc_engines_outer_step_local": (I, [PP, SZ, C.POINTER(OuterResult)]),
    "dlc_checkpoint_save": (I, [PP, SZ, C.c_char_p, C.POINTER(CheckpointMeta), C.POINTER(C.c_char_p),
                                C.POINTER(C.c_uint64), SZ]),
    "dlc_checkpoint_load": (I, [PP, SZ, C.c_char_p, C.POINTER(CheckpointMeta)]),
    "dlc_checkpoint_load_layout": (I, [PP, SZ, C.c_char_p, C.POINTER(C.c_char_p), C.POINTER(C.c_uint64), SZ,
                                       C.POINTER(CheckpointMeta)]),
    "dlc_optimizer_step": (I, [P, P, P, I, C.POINTER(I)]),
    "dlc_rng_key": (U64, [U64, C.c_char_p, U64]),
    "dlc_rng_fill_device": (I, [P, I, U64, U64, F, F]),
    "dlc_rng_perturb": (I, [P, P, U64, F, F]),
    "dlc_fp16_encode_bits": (I, [C.c_uint32, SZ, P]),
    "dlc_fold_push_probe": (I, [PP, I, SZ, I, I, P, C.POINTER(I)]),
    "dlc_p2p_kernels_probe": (I, [I, SZ, I, I, C.POINTER(C.c_float)]),
    "dlc_p2p_overlap_probe": (I, [I, SZ, I, I, I, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "dlc_run_training": (I, [P, P, GRAD_PRODUCER, METRICS_SINK, ROUND_HOOK, P, I, C.POINTER(RunResult)]),
    "dlc_p2p_set_tuning": (I, [C.POINTER(P2PTuning)]),
    "dlc_p2p_get_tuning": (I, [C.POINTER(P2PTuning)]),
    "dlc_world_create": (I, [C.POINTER(Config), C.POINTER(Hyperparams), SZ, P, I, I, C.POINTER(P)]),
    "dlc_world_destroy": (I, [P]),
    "dlc_world_engine": (I, [P, I, C.POINTER(P)]),
    "dlc_world_outer_step": (I, [P, C.POINTER(OuterResult)]),
    "dlc_world_shrink": (I, [P, C.POINTER(C.c_int), SZ, SZ]),
    "dlc_world_members": (SZ, [P, C.POINTER(C.c_int), SZ]),
    "dlc_wire_frames_size": (I, [U64, C.POINTER(WireTags), C.POINTER(SZ), C.POINTER(C.c_uint64)]),
    "dlc_wire_encode": (I, [P, U64, U64, C.POINTER(WireTags), P, SZ, C.POINTER(SZ), P]),
    "dlc_wire_decode": (I, [P, SZ, I, U64, U64, P, C.POINTER(WireChunk), SZ, C.POINTER(SZ), C.POINTER(SZ), P]),
    "dlc_engine_wire_begin": (I, [P, C.POINTER(C.c_uint64)]),
    "dlc_engine_wire_encode": (I, [P, I, U64, U64, C.POINTER(WireTags), P, SZ, C.POINTER(SZ)]),
    "dlc_engine_wire_decode": (I, [P, I, I, U64, U64, P, SZ, C.POINTER(WireChunk), SZ, C.POINTER(SZ),
                                   C.POINTER(SZ)]),
    "dlc_engine_wire_fold": (I, [P, I, I, U64, U64]),
    "dlc_engine_wire_finish": (I, [P, C.c_uint64, C.POINTER(OuterResult)]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/diloco_cuda.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^DLC_API [^(]*?\b(dlc_\w+)\s*\(", text, re.M)))


class DiLoCoError(RuntimeError):
    """Status != DLC_OK; .status holds the code (see include/diloco_cuda.h)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run __graft_entry__.build() "
                          "(there is no CPU fallback for the DiLoCo hot path)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


def check(status: int) -> None:
    if status != OK:
        raise DiLoCoError(status, lib.dlc_last_error().decode(errors="replace"))
