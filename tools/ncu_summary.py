#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (development tool).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/rN_ncu_full_summary.csv \
        [--traffic profiles/ncu_traffic.json --params 1100000000]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/rN_launches.csv

The traffic JSON maps kernel name -> DRAM bytes (read + write) per launch at
--params parameters; bench.py reports it as roofline.traffic when its own
parameter count matches.
"""
import argparse
import csv
import io
import json
import re
import subprocess

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def full(rep, out, traffic, params):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    idx = [h.index(k) for k in KEYS if k in h]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([h[i] for i in idx])
        w.writerow([units[i] for i in idx])
        for r in rows[2:]:
            w.writerow([r[i] for i in idx])
    if traffic:
        rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        res = {}
        for r in rows[2:]:
            b = float(r[rd]) * UNIT.get(units[rd], 1) + float(r[wr]) * UNIT.get(units[wr], 1)
            res.setdefault(short(r[h.index("Kernel Name")]), []).append(b)
        data = {"params": params, "source": rep, "bytes_per_launch": {k: sum(v) / len(v) for k, v in res.items()}}
        with open(traffic, "w") as f:
            json.dump(data, f, indent=1)


def launches(src, out):
    rows = [ln for ln in open(src) if not ln.startswith("==")]
    rd = list(csv.reader(io.StringIO("".join(rows))))
    h = rd[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "duration", "unit"])
        for r in rd[1:]:
            w.writerow([short(r[ki]), r[vi], r[ui]])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--traffic")
    ap.add_argument("--params", type=int, default=0)
    a = ap.parse_args()
    if a.launches:
        launches(a.src, a.out)
    else:
        full(a.src, a.out, a.traffic, a.params)
