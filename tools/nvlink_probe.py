#!/usr/bin/env python
"""Calibrate NVML's NVLink traffic counters on this box (development tool).

    python tools/nvlink_probe.py

Copies a known number of bytes from GPU 0 to GPU 1 (torch peer copy) and prints,
for each GPU, the change of every candidate NVML field: the throughput counters
(NVML_FI_DEV_NVLINK_THROUGHPUT_{DATA,RAW}_{TX,RX}, aggregate scope 0xFFFFFFFF and
per link) and the per-link byte counters (NVML_FI_DEV_NVLINK_COUNT_{XMIT,RCV}_BYTES).
The field whose delta matches the copied bytes (after its unit) is the one
bench.py samples around the timed region.
"""
import json

import pynvml as N
import torch

FIELDS = {"DATA_TX": 138, "DATA_RX": 139, "RAW_TX": 140, "RAW_RX": 141, "XMIT_BYTES": 202, "RCV_BYTES": 204}


STATUS = {}


def read(h, fid, scope):
    try:
        v = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
        if v.nvmlReturn != 0:
            STATUS[(fid, scope)] = int(v.nvmlReturn)
            return None
        return int(v.value.ullVal)
    except Exception as e:  # noqa: BLE001
        return f"err {e}"


def snapshot(handles):
    out = {}
    for g, h in enumerate(handles):
        for name, fid in FIELDS.items():
            out[(g, name, "all")] = read(h, fid, 0xFFFFFFFF)
            for link in range(18):
                out[(g, name, link)] = read(h, fid, link)
    return out


def main():
    N.nvmlInit()
    ng = torch.cuda.device_count()
    handles = [N.nvmlDeviceGetHandleByIndex(i) for i in range(min(ng, 2))]
    nbytes = 4 << 30
    a = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda:0").fill_(1.0)
    b = torch.empty_like(a, device="cuda:1")
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    s0 = snapshot(handles)
    reps = 4
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    s1 = snapshot(handles)
    moved = reps * nbytes
    res = {"bytes_copied_gpu0_to_gpu1": moved, "deltas": {}}
    for key, v0 in s0.items():
        v1 = s1[key]
        if isinstance(v0, int) and isinstance(v1, int) and v1 != v0:
            res["deltas"][f"gpu{key[0]}.{key[1]}.{key[2]}"] = {"delta": v1 - v0, "ratio_to_bytes": (v1 - v0) / moved}
    res["unsupported"] = sorted({f"{k[1]}.{k[2]}" for k, v in s0.items() if v is None})
    res["nvml_status"] = {f"{fid}.{sc}": st for (fid, sc), st in list(STATUS.items())[:16]}
    links = {}
    for link in range(18):
        try:
            links[link] = int(N.nvmlDeviceGetNvLinkState(handles[0], link))
        except Exception as e:  # noqa: BLE001
            links[link] = str(e)[:40]
    res["nvlink_state_gpu0"] = links
    import subprocess
    for cmd in (["nvidia-smi", "nvlink", "-s", "-i", "0"], ["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"]):
        try:
            res[" ".join(cmd)] = subprocess.run(cmd, capture_output=True, text=True, timeout=30).stdout[-1500:]
        except Exception as e:  # noqa: BLE001
            res[" ".join(cmd)] = str(e)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
