#!/usr/bin/env python
"""K1 (the inner AdamW step) alone at 1.1B params: CUDA events on the engine
stream over 20 steps after 3 warm-up steps (development tool, A/B builds)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2407_07852_b200 as D  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_100_000_000
    steps = 20
    D.lib.dlc_set_device(0)
    e = D.DilocoEngine(D.DilocoConfig(1 << 20, 1, D.FP16, 1 << 30), D.OptimHyperparams(), n, 0)
    e.rng_fill(D.THETA_T, 4242, "theta", 0, -0.05, 0.05)
    e.rng_fill(D.GRAD, 4242, "grad", 0, -1e-2 * 65536.0, 1e-2 * 65536.0)
    g = e.device_ptr(D.GRAD)
    s = torch.cuda.ExternalStream(e.stream, device="cuda:0")
    for _ in range(3):
        e.inner_step(g, grad_is_scaled=True)
    e.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        e.inner_step(g, grad_is_scaled=True)
    b.record(s)
    b.synchronize()
    ms = a.elapsed_time(b) / steps
    print(json.dumps({"n": n, "k1_ms": ms, "gbs": 28 * n / (ms * 1e-3) / 1e9}))
    e.close()


if __name__ == "__main__":
    main()
