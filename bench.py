#!/usr/bin/env python
"""bench.py — DiLoCo outer-sync throughput on B200 (one worker per GPU).

Metric (BASELINE.json): outer-sync params/sec & ms/outer-step at 1/2/4/8 B200;
inner AdamW HBM GB/s vs peak.

Workload (configs[3]/[4] of BASELINE.json, one DiLoCo worker per GPU): a 1.1B
flat FP32 parameter vector per worker, FP16 pseudo-gradient cast + FP16
average (ordered NCCL scatter / rank-order fold / all-gather), outer Nesterov
lr=0.7 momentum=0.9.  One timed *step* = one outer step: K2 pseudo-grad ->
C1 cross-worker average -> K4 Nesterov + theta_local refresh, on that step's
synthetic end-of-window weights (two device-resident variants alternate, so
every step sees a fresh, non-zero delta).  `value` = workers x params /
outer-step time (weak scaling: every GPU holds a full replica).  The inner
AdamW step (K1: unscale + overflow check + AdamW, one HBM pass) is timed in the
same run and reported under "inner_adamw".

Arms: default = this repo's CUDA path; `--impl reference` = the reference's own
CPU implementation (oracle/_ref, compiled from /root/reference/proj/src) on the
host cores.  Under torchrun (N>1) one process drives one GPU; timings are CUDA
events on the engine stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "outer-sync params/sec & ms/outer-step at 1/2/4/8 B200; inner AdamW HBM GB/s vs peak"
PEAK_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--params", type=int, default=1_100_000_000)
    ap.add_argument("--precision", choices=["fp16", "fp32"], default="fp16")
    ap.add_argument("--mode", choices=["p2p", "ordered", "allreduce"], default="p2p")
    ap.add_argument("--inner-mode", choices=["pingpong", "inplace"], default="pingpong")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-wire", action="store_true")
    ap.add_argument("--no-training", action="store_true")
    ap.add_argument("--no-boundary", action="store_true")
    ap.add_argument("--plan", default=None, help="P2P piece plan override, e.g. 1,2,3,2,1 (dlc_p2p_set_tuning)")
    ap.add_argument("--fold-ctas", type=int, default=0)
    ap.add_argument("--fold-threads", type=int, default=0)
    return ap.parse_args()


def plan_of(args, n):
    """The piece plan of the P2P / pipelined all-reduce step (engine_util.cu piece_plan)."""
    if args.plan:
        return [int(x) for x in args.plan.split(",")]
    return [1, 2, 2, 1] if n < 400_000_000 else [1, 2, 3, 2, 1]


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def ncu_traffic(kernel_prefix: str, n: int, launches: int = 1):
    """DRAM read+write bytes of the kernel per step from the committed ncu capture
    (profiles/ncu_traffic.json, tools/ncu_summary.py), when it was taken at the same size."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    if int(d.get("params", -1)) != n:
        return None
    for k, v in d.get("bytes_per_launch", {}).items():
        if k.startswith(kernel_prefix):
            return v * launches
    return None


def nvlink_from_profile(k, n, fp16):
    """The owner fold's NVLink bytes per step from the committed ncu capture of a
    one-process world (profiles/r2_ncu_nvlink_fold_world.json: every fold launch
    with nvl{rx,tx}__bytes{,_data_user}.sum, the kernels serialised by ncu), when
    it was taken at this K and size: per GPU and step, its own fold's pulls and
    pushes, counted twice for the peers' folds that read from and write into it."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_nvlink_fold_world.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    launches = d.get(f"k{k}")
    if not launches or n != 1_100_000_000 or not fp16:
        return None
    dev0 = [x for x in launches if x["device"] == 0]
    w = [1, 1, 2, 2, 1, 1]  # the piece plan of that capture: one step's fold launches per GPU
    step = dev0[:len(w)]
    if not step:
        return None
    scale = sum(w) / sum(w[:len(step)])  # a capture cut short (ncu -c) covers the first pieces only
    user_rx = scale * sum(x["nvl_rx_user_bytes"] for x in step)
    user_tx = scale * sum(x["nvl_tx_user_bytes"] for x in step)
    link_tx = scale * sum(x["nvl_tx_bytes"] for x in step)
    alone_ms = scale * sum(x["ms"] for x in step)
    return {"source": "profiles/r2_ncu_nvlink_fold_world.json (ncu, fold launches of GPU 0, one step)",
            "pieces_captured": len(step),
            "own_fold_user_bytes_rx": user_rx, "own_fold_user_bytes_tx": user_tx,
            "user_bytes_per_direction_per_step": user_rx + user_tx,
            "algorithmic_bytes_per_direction": 2 * (k - 1) * (-(-n // k)) * 2,
            "own_fold_link_bytes_tx": link_tx, "fold_alone_ms": alone_ms,
            "fold_alone_user_gbs_per_direction": user_rx / (alone_ms * 1e-3) / 1e9,
            "fold_alone_link_tx_gbs": link_tx / (alone_ms * 1e-3) / 1e9,
            "fold_alone_link_frac_of_900": link_tx / (alone_ms * 1e-3) / 1e9 / 900.0,
            "note": "the fold's bound is NVLink, not HBM: kernels_alone.fold_push runs it over local rows on one "
                    "GPU (no links), this is the same kernel moving its bytes over NVLink"}


def pcie_probe():
    try:
        with open(os.path.join(ROOT, "profiles", "r2_pcie_probe_1gpu.json")) as f:
            return json.load(f)
    except Exception:
        return None


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback"


# ---- clocks sampler (B200_PROFILING.md "clocks DURING the timed region") -----------------

class Clocks:
    """Samples SM clock, power and clock-event reasons through NVML every 2 ms
    (the same counters `nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.*`
    reads) on a background thread for the duration of the timed region."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int, enabled: bool = True):
        import threading
        self.samples = []
        self.err = None
        self.stop_evt = threading.Event()
        self.thread = None
        if not enabled:
            self.err = "disabled"
            return
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[device]) if vis and vis.split(",")[device].isdigit() else device
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(phys)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # NVML missing: report, do not guess
            self.err = f"nvml unavailable: {e}"
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        N = self.N
        while not self.stop_evt.is_set():
            try:
                self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetPowerUsage(self.h) / 1000.0,
                                     N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception as e:
                self.err = str(e)
                return
            time.sleep(0.002)

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "unavailable"]}
        self.stop_evt.set()
        self.thread.join(timeout=5)
        N = self.N
        reasons = sorted({name for _, _, mask in self.samples for name, attr in self.REASONS
                          if mask & getattr(N, attr, 0)})
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_sm,
                "sm_mhz_min": min(sm) if sm else None, "reasons": reasons, "samples": len(sm),
                "power_w_max": max(s[1] for s in self.samples) if sm else None, "source": "nvml"}


class NvlinkCounters:
    """NVML's cumulative NVLink data counters of this GPU (all links), read before
    and after the timed region: NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX
    (fields 138 / 139, aggregate scope), in KiB (calibrated with a known peer
    copy by tools/nvlink_probe.py, profiles/r2_nvlink_probe_*.json)."""

    TX, RX, ALL = 138, 139, 0xFFFFFFFF

    def __init__(self, device: int):
        self.err = None
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[device]) if vis and vis.split(",")[device].isdigit() else device
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(phys)
            self.t0 = self._read()
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"

    def _read(self):
        vals = self.N.nvmlDeviceGetFieldValues(self.h, [(self.TX, self.ALL), (self.RX, self.ALL)])
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError(f"field {v.fieldId}: nvml status {v.nvmlReturn}")
        return [int(v.value.ullVal) for v in vals]

    def stop(self, seconds: float, expected_bytes_per_direction: float):
        if self.err:
            return {"source": self.err}
        try:
            t1 = self._read()
        except Exception as e:  # noqa: BLE001
            return {"source": f"nvml read failed: {e}"}
        tx, rx = ((b - a) * 1024 for a, b in zip(self.t0, t1))
        return {"source": "nvml NVLINK_THROUGHPUT_DATA_TX/RX (KiB, all links)", "tx_bytes": tx, "rx_bytes": rx,
                "tx_gbs": tx / seconds / 1e9, "rx_gbs": rx / seconds / 1e9, "peak_gbs_per_direction": 900.0,
                "tx_frac_of_900": tx / seconds / 900e9, "rx_frac_of_900": rx / seconds / 900e9,
                "expected_bytes_per_direction": expected_bytes_per_direction,
                "tx_over_expected": tx / expected_bytes_per_direction if expected_bytes_per_direction else None}


# ---- CPU baseline: the reference's own functions on host threads --------------------------

def host_mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 0


def cpu_reference_outer(n: int, k: int, prec: int, iters: int, warmup: int = 0, full_ok: bool = True):
    """The reference's own outer round (oracle/_ref, run_simulated's K x axpy +
    reduce_average + K x outer_step, netsim.cpp:325-357) on every host core, each
    thread on a disjoint slice.  At the full workload (n params x k workers) when
    it fits in half the host's available memory (~4 (5k + 3) B/param live),
    else on a bounded sample whose per-step time is extrapolated linearly in
    params (the work is elementwise) and labelled so.
    Returns (params_per_s, per-step seconds, dict describing the run)."""
    from oracle import oracle as O
    lib = O.reference()
    if lib is None:
        return None
    threads = os.cpu_count() or 1
    need = 4 * (5 * k + 3) * n
    full = full_ok and need <= 0.5 * host_mem_available()
    sample = n if full else max(threads << 16, min(n, (16 << 20) * threads // k))
    secs = lib.bench_outer(threads, sample, k, prec, warmup, iters)
    units = k * sample
    desc = {"kind": "reference", "cores": threads,
            "sample": (f"{'the full workload' if full else 'a bounded sample'}: {sample} params x {k} workers "
                       f"({'fp16' if prec else 'fp32'}) split over {threads} threads, per step K x axpy + "
                       f"reduce_average + K x (all_finite, nesterov_step, theta_local = theta_t) "
                       f"(netsim.cpp:325-357); the reference's math is single-threaded per call, "
                       f"here every core takes a slice (reduce_average included), {iters} steps"),
            "sample_params_per_worker": sample, "sample_ms_per_step": statistics.mean(secs) * 1e3,
            "extrapolated": not full}
    if not full:
        desc["full_step_ms_extrapolated"] = statistics.mean(secs) * 1e3 * n / sample
    return units / statistics.mean(secs), secs, desc


def cpu_reference_inner(n: int, iters: int = 3):
    """The reference's apply_inner_step (engine.cpp:50-69: scale_gradient,
    scaler_unscale_and_check, lr_at, adamw_step, scaler_update) on every host
    core over a bounded sample of the parameter vector."""
    from oracle import oracle as O
    lib = O.reference()
    if lib is None:
        return None
    threads = os.cpu_count() or 1
    sample = max(threads << 16, min(n, (16 << 20) * threads))
    secs = lib.bench_inner(threads, sample, 1, iters)
    v = sample / statistics.mean(secs)
    return {"value": v, "unit": "params/s", "cores": threads, "kind": "reference",
            "sample": f"a bounded sample: {sample} params split over {threads} threads, apply_inner_step "
                      f"(scale + unscale/check + AdamW + scaler update), {iters} steps",
            "sample_ms_per_step": statistics.mean(secs) * 1e3,
            "full_step_ms_extrapolated": statistics.mean(secs) * 1e3 * n / sample, "extrapolated": sample != n,
            "hbm_equivalent_gbs": 28 * v / 1e9}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    k = args.gpus if world == 1 else world
    prec = 1 if args.precision == "fp16" else 0
    res = cpu_reference_outer(args.params, k, prec, args.steps, args.warmup)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    value, secs, desc = res
    # ms_per_step is the measured step: the full workload, or the bounded sample
    # (then desc carries the extrapolated full-size step time, labelled)
    ms = statistics.mean(secs) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "params/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, k),
            "cpu_baseline": dict(desc, value=value, unit="params/s"),
            "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def workload_config(args, k):
    return {"workload": f"DiLoCo outer step, {args.params / 1e9:.3g}B flat params per worker, {k} worker(s) "
                        f"(1 per GPU), {args.precision} pseudo-grad + {args.precision} average "
                        f"({args.mode}), Nesterov lr=0.7 mu=0.9",
            "params_per_worker": args.params, "workers": k, "precision": args.precision, "reduce_mode": args.mode,
            "inner_mode": args.inner_mode, "parallelism": f"diloco-dp{k}",
            "theta_local_refresh": "follows theta_t until the next applied inner step (no store)"
            if args.inner_mode == "pingpong" else "stored by K4",
            "l2": "inputs larger than L2 (every vector >= 126 MB)" if args.params * 2 > 126e6 else "L2-resident"}


# ---- wire codec ------------------------------------------------------

def measure_wire(D, eng, n, prec, steps=3, cpu=True):
    """Frames of the whole pseudo-gradient (the scatter side of a cross-box round)
    produced from HBM into a pinned host buffer, and decoded back into the
    device mean buffer: wall time through the public API, PCIe-bound.  Beside it
    the reference's own framing of the same vector on the host cores."""
    import torch

    from paper_2407_07852_b200 import _capi as A
    from paper_2407_07852_b200 import wire as W
    tags = W.make_tags(A.MSG_REDUCE_CHUNK, prec, 0, 0, 1, (0x0123456789ABCDEF, 0xFEDCBA9876543210))
    import ctypes as C
    size = C.c_size_t(0)
    A.lib.dlc_wire_frames_size(n, C.byref(tags), C.byref(size), None)
    host = torch.empty(size.value, dtype=torch.uint8, pin_memory=True)
    arr = host.numpy()
    eng.wire_begin()
    eng.wire_encode(A.WIRE_DELTA, 0, n, tags, out=arr)  # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.wire_encode(A.WIRE_DELTA, 0, n, tags, out=arr)
    enc = (time.perf_counter() - t0) / steps
    eng.wire_decode(A.WIRE_MEAN, 0, 0, n, arr)
    t0 = time.perf_counter()
    for _ in range(steps):
        _, used = eng.wire_decode(A.WIRE_MEAN, 0, 0, n, arr)
    dec = (time.perf_counter() - t0) / steps
    assert used == size.value
    out = {"frame_bytes": size.value, "chunk_size_bytes": int(tags.chunk_size_bytes),
           "encode_ms": enc * 1e3, "encode_gbs": size.value / enc / 1e9, "encode_params_per_s": n / enc,
           "decode_ms": dec * 1e3, "decode_gbs": size.value / dec / 1e9, "decode_params_per_s": n / dec,
           "host_buffer": "pinned", "note": "device -> frames in host memory over PCIe (copy engine, strided)"}
    del host, arr
    if cpu:
        from oracle import oracle as O
        lib = O.reference()
        if lib is not None:
            threads = os.cpu_count() or 1
            slice_len = max(1 << 16, min(1 << 24, n // threads))
            sec, fbytes = lib.bench_wire(threads, slice_len, prec, int(tags.chunk_size_bytes), 2)
            out["cpu_reference"] = {"params_per_s": threads * slice_len / sec, "gbs": fbytes / sec / 1e9,
                                    "cores": threads, "kind": "reference",
                                    "sample": f"{threads} threads x {slice_len} params: axpy + encode_fp16 + "
                                              f"send_chunk_span framing (collective.cpp:1318-1345)"}
    return out


# ---- run_training (engine.cpp:176-240) through the C ABI -------------------------------------

def measure_training_loop(D, coll, n, k, prec, local, max_over_ranks, barrier, h=4, rounds=8):
    """dlc_run_training for `rounds` windows of H inner steps with a device-side
    gradient producer (a resident loss-scaled gradient): host wall time per step
    against the device time of the steps themselves (CUDA events inside the
    loop).  The loop enqueues each step without waiting for the previous one, so
    `gpu_busy` near 1 means the host never starves the GPU."""
    cfg = D.DilocoConfig(local_steps_h=h, num_workers_k=k, reduce_precision=prec, total_inner_steps=h * rounds)
    e = D.DilocoEngine(cfg, D.OptimHyperparams(), n, local)
    e.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.GRAD, 4242, "grad", 0, -1e-2 * 65536.0, 1e-2 * 65536.0)
    gptr = e.device_ptr(D.GRAD)
    e.synchronize()
    recs = []
    barrier()
    t0 = time.perf_counter()
    res = D.run_training(e, coll, lambda step: (gptr, True, 0.0), sink=recs.append)
    wall = time.perf_counter() - t0
    dev_ms = res["compute_ms"] + res["comm_ms"]
    e.close()
    steps = int(res["steps_done"])
    return {"steps": steps, "local_steps_h": h, "rounds": int(res["rounds_done"]),
            "wall_ms_per_step": max_over_ranks(wall * 1e3 / steps), "device_ms_per_step": dev_ms / steps,
            "gpu_busy": dev_ms / (wall * 1e3), "records": len(recs),
            "producer": "device-resident loss-scaled gradient (no host copy)",
            "note": "dlc_run_training: steps enqueued back to back, records emitted two steps behind"}


# ---- the window boundary: K2 fused into the last inner step vs the outer step's own K2 -------

def measure_window_boundary(D, coll, n, k, prec, local, max_over_ranks, barrier, windows=4, warmup=1,
                            inner_mode=0):
    """The last inner step of a window plus the outer step that follows it
    (DilocoOptimizer::step at inner_step % H == 0, engine.cpp:162-174), timed
    with CUDA events on the engine stream around exactly those two calls, H = 2
    so theta_local != theta_t when the fused K1 runs (it reads theta_t).
    Variants, interleaved window by window on one engine: "unfused" (inner
    step, then the outer step with its own K2) and "fused": at K = 1
    DilocoOptimizer::step's single pass (K1 + K2 + K4, launch_boundary_solo,
    the default there), at K > 1 the opt-in K1 that also writes the delta
    (dlc_engine_set_fused_delta).  Per variant: the boundary's mean time and
    the K1 / K2 / K4 phase times (max over ranks)."""
    import torch
    h = 2
    variants = [("unfused", False), ("fused", True)]
    total = h * len(variants) * (warmup + windows)
    cfg = D.DilocoConfig(local_steps_h=h, num_workers_k=k, reduce_precision=prec, total_inner_steps=total)
    e = D.DilocoEngine(cfg, D.OptimHyperparams(), n, local, inner_mode)
    opt = D.DilocoOptimizer(e, coll)
    e.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.GRAD, 4242, "grad", k * 100 + 7, -1e-2 * 65536.0, 1e-2 * 65536.0)
    gptr = e.device_ptr(D.GRAD)
    e.synchronize()
    stream = torch.cuda.ExternalStream(e.stream, device=f"cuda:{local}")
    rec = {name: {"ms": [], "k1": [], "k2": [], "k4": []} for name, _ in variants}
    e.set_timing(True)
    for wi in range(warmup + windows):
        for name, fused in variants:
            e.set_fused_delta(fused)
            e.inner_step(gptr, grad_is_scaled=True)
            barrier()
            e.synchronize()
            e.phase_times()  # reset
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if fused and k == 1:
                opt.step(gptr, grad_is_scaled=True)
            else:
                e.inner_step(gptr, grad_is_scaled=True)
                e.outer_step(coll)
            b.record(stream)
            b.synchronize()
            e.synchronize()
            ph, _ = e.phase_times()
            if wi >= warmup:
                r = rec[name]
                r["ms"].append(a.elapsed_time(b))
                r["k1"].append(ph[0])
                r["k2"].append(ph[1])
                r["k4"].append(ph[3])
    e.set_timing(False)
    e.close()
    out = {}
    for name, _ in variants:
        r = rec[name]
        out[name] = {key + "_ms": max_over_ranks(statistics.mean(v)) for key, v in
                     (("boundary", r["ms"]), ("k1", r["k1"]), ("k2", r["k2"]), ("k4", r["k4"]))}
    out["fused_saves_ms"] = out["unfused"]["boundary_ms"] - out["fused"]["boundary_ms"]
    if k == 1:  # the fused pass: 40 B/param (theta_local, g, m, v, theta_t, momentum in; m, v, theta_t, momentum out);
        # INPLACE engines: + the 4 B/param overflow pre-pass and the theta_local store = 48
        peak, kind = measured_peak()
        bpp = 40 if inner_mode == 0 else 48
        ach = bpp * n / (out["fused"]["k1_ms"] * 1e-3) / 1e9
        out["fused"]["roofline"] = {"kernel": "boundary_solo_kernel (K1+K2+K4)" if inner_mode == 0 else
                                    "unscale_check + boundary_solo_inplace_kernel (K1+K2+K4)", "bytes_per_param": bpp,
                                    "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                                    "peak_source": kind, "traffic": ncu_traffic("boundary_solo_kernel", n) if inner_mode == 0 else None}
    out.update({"windows_each": windows, "local_steps_h": h,
                "what": "last inner step (K1) + outer step, CUDA events on the engine stream, variants interleaved; "
                        "k1 / k2 / k4 = summed event-timed phases of that boundary (k4: busy time of the pieces)"})
    return out


# ---- our arm -----------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2407_07852_b200 as D

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    D.lib.dlc_set_device(local)
    if args.plan or args.fold_ctas or args.fold_threads:
        D.set_p2p_tuning(plan=plan_of(args, args.params) if args.plan else None, fold_ctas=args.fold_ctas,
                         fold_threads=args.fold_threads)
    k = world
    n = args.params
    prec = D.FP16 if args.precision == "fp16" else D.FP32
    mode = {"p2p": D.MODE_P2P, "ordered": D.MODE_ORDERED, "allreduce": D.MODE_ALLREDUCE}[args.mode]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    coll = None
    if k > 1:
        uid = [D.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        coll = D.NcclCollective(rank, world, uid[0], local, mode)

    cfg = D.DilocoConfig(local_steps_h=1, num_workers_k=k, reduce_precision=prec, total_inner_steps=1 << 40)
    hp = D.OptimHyperparams()
    inner_mode = D.INNER_PINGPONG if args.inner_mode == "pingpong" else D.INNER_INPLACE
    eng = D.DilocoEngine(cfg, hp, n, local, inner_mode)
    eng.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    # two synthetic end-of-window weight sets per worker (theta_t - U(-1e-3, 1e-3))
    xs = [torch.empty(n, dtype=torch.float32, device=f"cuda:{local}") for _ in range(2)]
    for i, x in enumerate(xs):
        eng.rng_perturb(4242, "local", rank * 16 + i, -1e-3, 1e-3, dst_dev_ptr=x.data_ptr())
    eng.rng_fill(D.GRAD, 4242, "grad", rank, -1e-2 * 65536.0, 1e-2 * 65536.0)  # loss-scaled grads
    gptr = eng.device_ptr(D.GRAD)
    eng.synchronize()
    stream = torch.cuda.ExternalStream(eng.stream, device=f"cuda:{local}")

    def timed(fn, steps):
        barrier()
        eng.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s in range(steps):
            fn(s)
        b.record(stream)
        b.synchronize()
        eng.synchronize()
        barrier()
        return max_over_ranks(a.elapsed_time(b))

    outer = lambda s: eng.outer_step_from(coll, xs[s % 2].data_ptr())  # noqa: E731
    inner = lambda s: eng.inner_step(gptr, grad_is_scaled=True)  # noqa: E731
    for s in range(args.warmup):
        outer(s)
        inner(s)
    eng.synchronize()

    clocks = Clocks(local, enabled=not args.no_clocks)
    eng.set_timing(True)
    eng.phase_times()
    nvl = NvlinkCounters(local) if k > 1 else None
    outer_ms = timed(outer, args.steps)
    nvl_res = nvl.stop(outer_ms * 1e-3, 2 * (k - 1) * (-(-n // k)) * (2 if prec == D.FP16 else 4) * args.steps) \
        if nvl else None
    if world > 1:  # every rank's own counters
        allv = [None] * world
        dist.all_gather_object(allv, nvl_res)
        nvl_res = allv
    ph_ms, ph_n = eng.phase_times()
    inner_total = timed(inner, args.steps)
    ph2_ms, ph2_n = eng.phase_times()
    clk = clocks.stop()
    eng.set_timing(False)

    ms_step = outer_ms / args.steps
    inner_ms = inner_total / args.steps
    peak, peak_kind = measured_peak()
    wire = 2 if prec == D.FP16 else 4
    # algorithmic bytes per parameter
    # PINGPONG engines do not store theta_local' (it follows theta_t', Pair::follow
    # in kernels.cuh): K4 = theta_t, momentum, mean in; theta_t', momentum' out
    follow = args.inner_mode == "pingpong"
    b_solo = 20 if follow else 24
    b_k1, b_k2, b_k4 = 28, 8 + wire, (16 if follow else 20) + wire
    # per step: the summed intervals (K > 1 P2P times every K4 piece launch and the
    # finish gate on their own, so this is K4's busy time, not its waits for means)
    k4_ms = max_over_ranks(ph_ms[3] / args.steps)
    k2_ms = max_over_ranks(ph_ms[1] / max(ph_n[1], 1))
    coll_ms = max_over_ranks(ph_ms[2] / max(ph_n[2], 1)) if ph_n[2] else 0.0
    k1_ms = max_over_ranks(ph2_ms[0] / max(ph2_n[0], 1))

    def roof(bpp, ms):
        ach = bpp * n / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": peak_kind, "bytes_per_param": bpp, "kernel_ms": ms}

    line = {"metric": METRIC, "value": k * n / (ms_step * 1e-3), "unit": "params/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, k)}
    if k == 1:
        # one worker: K2 and K4 fused into one pass (theta_t, theta_local, momentum in;
        # theta_t', momentum' (+ theta_local' in place mode) out) = 20 (24) B/param
        rl = roof(b_solo, k4_ms)
        rl["kernel"] = "outer_solo_kernel (K2+K4 fused)"
        line["phases_ms"] = {"outer_solo_K2K4": k4_ms}
        line["phase_roofline"] = {"outer_solo_K2K4": rl["frac"]}
        rl["traffic"] = ncu_traffic("outer_solo_kernel", n)
    else:
        rl = roof(b_k4, k4_ms)
        rl["kernel"] = ("nesterov_p2p_piece_kernel (K4)" if mode == D.MODE_P2P else "nesterov_outer_kernel (K4)")
        line["phases_ms"] = {"pseudo_grad_K2": k2_ms, "collective_C1_K3": coll_ms, "nesterov_K4": k4_ms}
        line["phase_roofline"] = {"pseudo_grad_K2": roof(b_k2, k2_ms)["frac"], "nesterov_K4": rl["frac"]}
        rl["traffic"] = None
        if mode == D.MODE_P2P:
            # multi-rank runs cannot be profiled: the capture is the same kernel over all N
            # params on one GPU (tools/p2p_kernels_probe.py), i.e. one step's pieces
            rl["traffic"] = ncu_traffic("nesterov_p2p_piece_kernel<%d>" % (1 if prec == D.FP16 else 0), n)
            rl["traffic_source"] = "ncu of the kernel alone on one GPU (tools/p2p_kernels_probe.py)"
    line["roofline"] = rl
    if k > 1 and mode == D.MODE_P2P and rank == 0:
        # the same kernels alone on this GPU (no exchange traffic sharing HBM): each
        # kernel's own ceiling, against which the in-step phase_roofline is read
        import ctypes
        ms3 = (ctypes.c_float * 3)()
        if D.lib.dlc_p2p_kernels_probe(k, n, prec, 3, ms3) == 0:
            line["kernels_alone"] = {
                name: {"ms": t, "bytes_per_param": bpp, "frac": roof(bpp, t)["frac"]}
                for name, bpp, t in (("pseudo_grad_K2", b_k2, ms3[0]), ("fold_push", 2 * wire, ms3[1]),
                                     ("nesterov_K4", 16 + wire, ms3[2]))}
            # the warp-specialised fold alone too (the step uses the single-leader one:
            # tied inside the step, where the fold is NVLink-bound; see nvlink_ncu)
            from paper_2407_07852_b200 import _capi as A
            t0 = A.P2PTuning()
            D.lib.dlc_p2p_get_tuning(ctypes.byref(t0))
            t1 = A.P2PTuning()
            ctypes.memmove(ctypes.byref(t1), ctypes.byref(t0), ctypes.sizeof(t0))
            t1.fold_kernel = 1
            D.lib.dlc_p2p_set_tuning(ctypes.byref(t1))
            if D.lib.dlc_p2p_kernels_probe(k, n, prec, 3, ms3) == 0:
                line["kernels_alone"]["fold_push_warp_specialised"] = {
                    "ms": ms3[1], "bytes_per_param": 2 * wire, "frac": roof(2 * wire, ms3[1])["frac"]}
            D.lib.dlc_p2p_set_tuning(ctypes.byref(t0))
            line["kernels_alone"]["note"] = ("each kernel alone on one GPU over local rows (no NVLink); the fold's "
                                             "bound in the step is NVLink (nvlink_ncu)")
    # whole-step roofline: HBM bytes at the measured copy peak and
    # NVLink bytes per direction at the pool's measured 770 GB/s peer copy
    # (B200_PROFILING.md); serial = sum, bound = max (perfect overlap).
    nvlink_peak = 770.0
    hbm_bpp = b_solo if k == 1 else (b_k2 + b_k4)
    wire_bytes = 2 * (k - 1) * (-(-n // k)) * wire if k > 1 else 0
    hbm_ms = hbm_bpp * n / (peak * 1e9) * 1e3
    nvl_ms = wire_bytes / (nvlink_peak * 1e9) * 1e3
    # the exchange itself also streams through HBM: every delta is read once
    # (by its owner, locally or over NVLink) and every mean written once
    hbm_coll = 2 * wire * n if k > 1 else 0
    hbm_all_ms = (hbm_bpp * n + hbm_coll) / (peak * 1e9) * 1e3
    line["step_roofline"] = {"hbm_bytes": hbm_bpp * n, "nvlink_bytes_per_direction": wire_bytes,
                             "hbm_ms": hbm_ms, "nvlink_ms": nvl_ms, "serial_ms": hbm_ms + nvl_ms,
                             "bound_ms": max(hbm_ms, nvl_ms), "frac_of_serial": (hbm_ms + nvl_ms) / ms_step,
                             "frac_of_bound": max(hbm_ms, nvl_ms) / ms_step, "nvlink_peak_gbs": nvlink_peak,
                             "hbm_peak_gbs": peak, "hbm_bytes_incl_exchange": hbm_bpp * n + hbm_coll,
                             "frac_of_bound_incl_exchange": max(hbm_all_ms, nvl_ms) / ms_step}
    if k > 1:
        # weak-scaling ceiling: one worker's outer step needs b_solo B/param and no
        # exchange; K workers each need (K2 + K4 + exchange) HBM bytes or the NVLink
        # time, whichever is longer, so value(K) / (K value(1)) cannot exceed this
        solo_ms = b_solo * n / (peak * 1e9) * 1e3
        line["step_roofline"]["weak_scaling_ceiling"] = solo_ms / max(hbm_all_ms, nvl_ms)
    if k > 1:
        # algorithmic NVLink bytes per direction (the padded owner slots each GPU
        # serves and receives) over the whole step and over the exchange's busy time
        line["exchange_gbs_per_direction_over_step"] = wire_bytes / (ms_step * 1e-3) / 1e9
        key = "exchange_gbs_per_direction_over_collective" if mode == D.MODE_P2P else "nccl_bus_gbs"
        line[key] = wire_bytes / (coll_ms * 1e-3) / 1e9 if coll_ms else None
        line["nvlink_counters"] = nvl_res  # per rank, measured by each GPU itself
        if mode == D.MODE_P2P:
            line["nvlink_ncu"] = nvlink_from_profile(k, n, prec == D.FP16)
    ir = roof(b_k1, k1_ms)
    ir["kernel"] = "adamw_kernel (K1, %s)" % args.inner_mode
    ir["traffic"] = ncu_traffic("adamw_kernel", n)
    line["inner_adamw"] = {"ms_per_step": inner_ms, "kernel_ms": k1_ms, "roofline": ir,
                           "vs_8TBs_spec": ir["achieved"] / 8000.0}
    # outer: fused solo + recovery (K=1) or K2 + fold/check + K4; inner: K1 (+ pre-pass in place)
    if k == 1:
        per_outer = 2  # outer_solo + finish
    elif mode == D.MODE_P2P:
        pieces = len(plan_of(args, n))
        # K2, fold_push, K4 per piece, the finish gate; flag barriers A_0, B_p, commit
        per_outer = 3 * pieces + 1 + (pieces + 2)
    elif mode == D.MODE_ALLREDUCE:
        pieces = len(plan_of(args, n))
        per_outer = 3 * pieces + 1  # K2, non-finite check, K4 pieces, finish (NCCL's own kernels not counted)
    else:
        per_outer = 3  # K2, fold / non-finite check, K4
    per_inner = 2 if args.inner_mode == "pingpong" else 3  # (pre-pass,) AdamW, finalize
    line["gpu_launches"] = args.steps * (per_outer + per_inner)
    line["clocks"] = clk

    # e2e through the public C ABI with host buffers: H2D theta_local, outer step, D2H theta_t.
    if not args.no_e2e:
        e2e_steps = args.e2e_steps or max(3, min(args.steps, 5))
        from paper_2407_07852_b200 import dist as PD
        with PD.gpu_local_memory(local) as local_cpus:  # pinned pages on the GPU's own NUMA node
            hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
            ht = torch.empty(n, dtype=torch.float32, pin_memory=True)
            hx.copy_(xs[0])
        eng.outer_step_host(coll, hx.data_ptr(), ht.data_ptr())  # warm
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            eng.outer_step_host(coll, hx.data_ptr(), ht.data_ptr())
        dt = max_over_ranks(time.perf_counter() - t0)
        line["e2e"] = {"value": k * n * e2e_steps / dt, "unit": "params/s", "h2d_bytes_per_step": 4 * n,
                       "d2h_bytes_per_step": 4 * n, "ms_per_step": dt * 1e3 / e2e_steps, "steps": e2e_steps,
                       "host_buffers": "pinned, " + (f"GPU-local NUMA node ({len(local_cpus)} CPUs)"
                                                      if local_cpus else "default NUMA placement")}
        probe = pcie_probe()
        if probe and world == 1 and n == 1_100_000_000:
            # the same bytes H2D and D2H at once on two streams, no kernel (tools/pcie_probe.py)
            line["e2e"]["copy_ceiling_ms"] = probe["both_ms"]
            line["e2e"]["frac_of_copy_ceiling"] = probe["both_ms"] / (dt * 1e3 / e2e_steps)
            line["e2e"]["copy_ceiling_source"] = "profiles/r2_pcie_probe_1gpu.json (pinned H2D + D2H concurrently)"
        del hx, ht

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # a bounded sample (~10 s of CPU work); the --impl reference arm times the full workload
        res = cpu_reference_outer(n, k, 1 if prec == D.FP16 else 0, iters=2, full_ok=False)
        if res is not None:
            v, secs, desc = res
            line["cpu_baseline"] = dict(desc, value=v, unit="params/s")
        ci = cpu_reference_inner(n)
        if ci is not None:
            line["inner_adamw"]["cpu_baseline"] = ci
    if world == 1 and not args.no_wire:
        line["wire"] = measure_wire(D, eng, n, prec, cpu=not args.no_cpu_baseline)
    eng.close()
    if not args.no_boundary:
        line["window_boundary"] = measure_window_boundary(D, coll, n, k, prec, local, max_over_ranks, barrier,
                                                          inner_mode=inner_mode)
    if not args.no_training:
        line["training_loop"] = measure_training_loop(D, coll, n, k, prec, local, max_over_ranks, barrier)
        if n > 150_000_000:  # the paper's Llama-150M size (configs 2-3): ~0.6 ms inner steps
            line["training_loop_150m"] = measure_training_loop(D, coll, 150_000_000, k, prec, local,
                                                               max_over_ranks, barrier, rounds=32)
    if rank == 0:
        print(json.dumps(line))
    if coll:
        coll.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _json_stdout():
    """Keep stdout for the one JSON line: native libraries (NCCL's version banner
    under NCCL_DEBUG, CUDA) write to fd 1 directly, so fd 1 becomes stderr and the
    result line goes to the saved stdout."""
    global print
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    out = os.fdopen(saved, "w", buffering=1)
    import builtins

    def print(*a, **kw):  # noqa: A001
        kw.setdefault("file", out)
        kw.setdefault("flush", True)
        builtins.print(*a, **kw)


def main():
    args = parse()
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        _json_stdout()
    rank, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not launched by torchrun: relaunch one process per GPU
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29533")] + sys.argv
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
