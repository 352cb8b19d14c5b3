#!/usr/bin/env python
"""Small single-GPU workload touching every kernel family, for
`compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_case.py`
(development tool).  Ragged sizes exercise the scalar tails."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_07852_b200 as D  # noqa: E402


def main():
    D.lib.dlc_set_device(0)
    rng = np.random.default_rng(0)
    n = 10_007
    for prec in (D.FP32, D.FP16):
        for mode in (D.INNER_PINGPONG, D.INNER_INPLACE):
            cfg = D.DilocoConfig(2, 3, prec, 4)
            engines = [D.DilocoEngine(cfg, D.OptimHyperparams(warmup_steps=2), n, 0, mode) for _ in range(3)]
            th = rng.uniform(-1, 1, n).astype(np.float32)
            for e in engines:
                e.upload(D.THETA_T, th)
                e.upload(D.THETA_LOCAL, th)
            for t in range(4):
                for e in engines:
                    g = rng.uniform(-1e-2, 1e-2, n).astype(np.float32)
                    if t == 1:
                        g[n - 1] = np.inf
                    e.inner_step_host(g)
                if t % 2 == 1:
                    D.outer_step_local(engines)
            for e in engines:
                e.close()
        # solo: fused outer step, host-buffer chunked path, external split, checkpoint
        e = D.DilocoEngine(D.DilocoConfig(1, 1, prec, 3), D.OptimHyperparams(), n)
        e.upload(D.THETA_T, th)
        out = np.empty(n, np.float32)
        e.outer_step_host(None, th - 1e-3, out)
        d, ep = e.compute_pseudo_gradient()
        e.apply_outer_step(d, ep)
        e.outer_step(None, wait=True)
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "c.ckpt")
            D.checkpoint_save([e], path)
            D.checkpoint_load([e], path)
        e.close()
    # host-buffer reference functions
    x = rng.uniform(-1, 1, n).astype(np.float32)
    st = D.AdamWState.init(n)
    D.adamw_step(st, x, x * 1e-2, 1e-3)
    D.nesterov_step(D.NesterovState.init(n), x, x)
    D.reduce_average([x, x, x], 1)
    D.encode_fp16(x)
    D.decode_fp16(D.encode_fp16(x)[0])
    D.scaler_unscale_and_check(D.LossScaler(), x)
    D.fp16_encode_bits(0x7F000000, 1 << 16)
    print("sanitize case done")


if __name__ == "__main__":
    main()
