"""CPU-side checks of the C ABI (no GPU needed).

* libdiloco_cuda.so loads and exports every symbol include/diloco_cuda.h declares;
* host-scalar entry points (lr_at, scaler_update, partition/byte law, rng key)
  match the oracle;
* compute entry points fail loudly without a GPU (no CPU fallback).
"""
import ctypes as C
import subprocess

import numpy as np
import pytest

import paper_2407_07852_b200 as D
from paper_2407_07852_b200 import _capi as A
from oracle import oracle as O


def test_library_exports_every_header_symbol():
    declared = A.header_symbols()
    assert len(declared) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(A.lib, s)
    assert A.lib.dlc_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", A.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_lr_at_matches_oracle(port):
    for cos in (0, 1):
        for step in (0, 1, 5, 500, 999, 1000, 1001, 5000, 9999, 10000, 20000):
            s = D.LrSchedule(1000, 10000, 4e-4, cos)
            assert D.lr_at(s, step) == port.lr_at(1000, 10000, 4e-4, cos, step)


def test_scaler_update_matches_oracle(port):
    sc = D.LossScaler(65536.0, 3, 0)
    s, g = 65536.0, 0
    rng = np.random.default_rng(1)
    for ov in rng.random(300) < 0.3:
        D.scaler_update(sc, ov)
        s, g = port.scaler_update(s, g, 3, ov)
        assert (sc.scale, sc.consecutive_good) == (s, g)
    sc = D.LossScaler(1.0, 2000, 0)
    for _ in range(100):
        D.scaler_update(sc, True)
    assert sc.scale == 2.0 ** -20


def test_partition_and_bytes_match_oracle(port):
    for n in (0, 1, 7, 1000, 24 * 50, 1_000_003):
        for k in (1, 2, 3, 4, 8):
            assert D.partition_ranges(n, k) == port.partition_ranges(n, k)
            for r in range(k):
                for p in (0, 1):
                    assert D.per_peer_reduce_bytes(n, k, r, p) == port.per_peer_reduce_bytes(n, k, r, p)
            assert D.fleet_reduce_bytes(n, k, 1) == port.fleet_reduce_bytes(n, k, 1)


def test_rng_key_matches_counter_rng():
    for seed, purpose, idx in ((4242, "theta", 0), (17, "adamw-oracle", 0), (4242, "grad", 1003)):
        assert D.rng_key(seed, purpose, idx) == O.rng_key(seed, purpose, idx)


def test_compute_fails_loudly_without_gpu():
    try:
        n = D.device_count()
    except D.Error:
        n = 0
    if n > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(D.Error) as ei:
        D.axpy(1.0, [1.0, 2.0], [3.0, 4.0])
    assert ei.value.status == A.ECUDA
    with pytest.raises(D.Error):
        D.DilocoEngine(D.DilocoConfig(1, 1, A.FP32, 1), D.OptimHyperparams(), 16)


def test_config_validation_precedes_device():
    # DilocoConfig::validate (engine.cpp:31-48) errors are ConfigError even without a GPU.
    for cfg in (D.DilocoConfig(0, 1, A.FP32, 10), D.DilocoConfig(5, 0, A.FP32, 10),
                D.DilocoConfig(50, 1, A.FP32, 120), D.DilocoConfig(5, 1, 7, 10)):
        with pytest.raises(D.ConfigError):
            D.DilocoEngine(cfg, D.OptimHyperparams(), 16)


def test_null_arguments_are_einval():
    assert A.lib.dlc_engine_create(None, None, 0, 0, 0, None) == A.EINVAL
    assert b"null" in A.lib.dlc_last_error()
    assert A.lib.dlc_reduce_average(None, 0, 4, 0, None) == A.ECOLLECTIVE
    assert A.lib.dlc_engine_destroy(None) == A.OK
    assert A.lib.dlc_collective_world_size(None) == 1
    assert A.lib.dlc_engine_size(C.c_void_p()) == 0


def test_round2_entry_points_validate_without_gpu():
    # round-2 entry points: argument checks come before any device work
    assert A.lib.dlc_world_shrink(None, None, 0, 0) == A.EINVAL
    assert A.lib.dlc_world_members(None, None, 0) == 0
    assert A.lib.dlc_engine_set_fused_delta(None, 1) == A.EINVAL
    assert b"null" in A.lib.dlc_last_error()
    t = A.P2PTuning()
    t.fold_kernel = 2
    assert A.lib.dlc_p2p_set_tuning(C.byref(t)) == A.ECONFIG
    assert A.lib.dlc_p2p_set_tuning(None) == A.OK
