"""Time the K > 1 outer-step kernels on ONE GPU (development / ncu tool).

    python tools/p2p_kernels_probe.py [--params N] [--k 2 4 8] [--precision fp16]

For each worker count k: K2 (pseudo_grad_piece over a whole owner-slot range),
the owner fold + mean push (fold_push_tma_kernel for k <= 8) over k local rows,
and K4 (nesterov_p2p_piece), each alone on an idle GPU, with CUDA events.
In the real step these kernels share HBM with each other and with the NVLink
exchange; alone they show each kernel's own ceiling, and `ncu` can capture them
in one process (a multi-rank run cannot be profiled).  Algorithmic bytes per
parameter: K2 8 + w, fold 2w (the w-byte rows one GPU serves to the owners plus
the w-byte means it receives), K4 16 + w  (w = 2 FP16, 4 FP32).
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_07852_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=1_100_000_000)
    ap.add_argument("--k", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--precision", choices=["fp16", "fp32"], default="fp16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--fold-kernel", type=int, nargs="+", default=[0], help="0 single-leader, 1 warp-specialised")
    ap.add_argument("--fold-threads", type=int, nargs="+", default=[0], help="0 = default by K")
    ap.add_argument("--fold-ctas", type=int, nargs="+", default=[0], help="0 = default max(16, 320 / K)")
    ap.add_argument("--overlap", action="store_true",
                    help="also time K4 while the fold (320/k CTAs, as in the step) runs on a second stream")
    a = ap.parse_args()
    D.lib.dlc_set_device(0)
    prec = D.FP16 if a.precision == "fp16" else D.FP32
    w = 2 if prec == D.FP16 else 4
    n = a.params
    import itertools
    for k, fk, ft, fc in itertools.product(a.k, a.fold_kernel, a.fold_threads, a.fold_ctas):
        D.set_p2p_tuning(fold_kernel=fk, fold_threads=ft, fold_ctas=fc)
        ms = (C.c_float * 3)()
        ov = (C.c_float * 2)()
        st = D.lib.dlc_p2p_overlap_probe(k, n, prec, a.reps, 0, ms, ov if a.overlap else None)
        if st != 0:
            raise RuntimeError(D.lib.dlc_last_error().decode())
        out = {"k": k, "params": n, "precision": a.precision, "fold_kernel": fk, "fold_threads": ft,
               "fold_ctas": fc}
        for name, bpp, t in (("K2_pseudo_grad_piece", 8 + w, ms[0]), ("fold_push", 2 * w, ms[1]),
                             ("K4_nesterov_p2p_piece", 16 + w, ms[2])):
            out[name] = {"ms": round(t, 4), "bytes_per_param": bpp, "gbs": round(bpp * n / (t * 1e-3) / 1e9, 1)}
        if a.overlap:
            out["K4_while_fold_runs"] = {"ms": round(ov[0], 4), "gbs": round((16 + w) * n / (ov[0] * 1e-3) / 1e9, 1),
                                         "fold_ms": round(ov[1], 4)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
