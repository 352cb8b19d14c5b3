#!/usr/bin/env python
"""The fused single-worker window boundary (boundary_solo_kernel) at 1.1B params
through DilocoOptimizer::step, for an ncu capture of that kernel
(development tool):

    python tools/boundary_probe.py && ncu --set full -k regex:boundary_solo_kernel -c 2 ... python tools/boundary_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_07852_b200 as D  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_100_000_000
    D.lib.dlc_set_device(0)
    h, windows = 2, 3
    e = D.DilocoEngine(D.DilocoConfig(h, 1, D.FP16, h * windows), D.OptimHyperparams(), n, 0)
    e.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.THETA_LOCAL, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.GRAD, 4242, "grad", 0, -1e-2 * 65536.0, 1e-2 * 65536.0)
    g = e.device_ptr(D.GRAD)
    opt = D.DilocoOptimizer(e)
    for _ in range(h * windows):
        opt.step(g, grad_is_scaled=True)
    e.synchronize()
    print("boundary_probe ok:", e.scalars().outer_epoch, "rounds")
    e.close()


if __name__ == "__main__":
    main()
