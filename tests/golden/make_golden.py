"""Generate the committed golden fixtures from the REFERENCE build.

Run in the build container (needs /root/reference to build oracle/_ref):

    python tests/golden/make_golden.py

Every output below is produced by the reference's own functions
(oracle/_ref/libdiloco_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  The fixtures pin the C restatement (tests/test_oracle.py)
and the CUDA path (tests/test_gpu_parity.py) on the GPU box, where
/root/reference does not exist.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import driver as D  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def edge_floats():
    """Values that exercise every codec branch (fp16.cpp:25-63)."""
    specials = np.array([0.0, -0.0, 1.0, 2049.0, 65504.0, 65519.0, 65520.0, -65520.0, 1e30, -1e30,
                         np.inf, -np.inf, np.nan, 1e-9, 2.0 ** -25, 2.0 ** -24, 1.5 * 2.0 ** -25,
                         2.0 ** -14, 2.0 ** -14 * (1 - 2.0 ** -11), 5.960464477539063e-08,
                         3.0517578125e-05, 6.1035156e-05, 1e-40, -1e-45], np.float32)
    return specials


def main():
    O.build(ref=True)
    R = O.reference()
    assert R is not None, "reference build missing"
    rng = np.random.default_rng(20240710)

    # --- fp16 codec fuzz: exponent-spread values like test_tensor.cpp:78-87 ---
    mant = rng.uniform(-2, 2, 60000).astype(np.float32)
    ex = rng.integers(-32, 32, 60000)
    fuzz = np.concatenate([edge_floats(), np.ldexp(mant, ex).astype(np.float32)])
    # ties: exact midpoints between adjacent halves (normal and subnormal)
    codes = rng.integers(0, 0x7BFF, 4000).astype(np.uint16)
    lo = codes.view(np.float16).astype(np.float64)
    hi = (codes + 1).view(np.float16).astype(np.float64)
    ties = ((lo + hi) / 2).astype(np.float32)
    fuzz = np.concatenate([fuzz, ties, -ties])
    enc, ov = R.encode_fp16(fuzz)
    np.savez_compressed(os.path.join(OUT, "fp16_codec.npz"), x=fuzz, codes=enc,
                        decoded_all=R.decode_fp16(np.arange(65536, dtype=np.uint32).astype(np.uint16)))

    # --- AdamW: 5-step trajectories, test_optim.cpp:64-82 style ---
    n = 2048
    p0 = rng.uniform(-2, 2, n).astype(np.float32)
    grads = rng.uniform(-1, 1, (5, n)).astype(np.float32)
    grads[:, :8] = np.float32([0, 1e-30, -1e-30, 1e-3, 30.0, -7.5, 1e-38, 3e-39])
    lrs = np.float32([4e-4, 1e-3, 0.0, 7e-3, 2.5e-4])
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    p, sc, traj = p0.copy(), 0, []
    for t in range(5):
        st, p, sc = R.adamw_step(p, grads[t], m, v, sc, float(lrs[t]), 0.9, 0.95, 1e-8, 0.1)
        assert st == 0
        traj.append(p.copy())
    np.savez_compressed(os.path.join(OUT, "adamw.npz"), p0=p0, grads=grads, lrs=lrs,
                        traj=np.stack(traj), m=m, v=v, step_count=sc)

    # --- Nesterov: 4 steps, test_optim.cpp:122-139 style ---
    th0 = rng.uniform(-5, 5, n).astype(np.float32)
    gs = rng.uniform(-1, 1, (4, n)).astype(np.float32)
    buf = np.zeros(n, np.float32)
    th, tr = th0.copy(), []
    for t in range(4):
        st, th = R.nesterov_step(th, gs[t], buf, 0.7, 0.9)
        assert st == 0
        tr.append(th.copy())
    np.savez_compressed(os.path.join(OUT, "nesterov.npz"), theta0=th0, grads=gs, traj=np.stack(tr),
                        buf=buf)

    # --- reduce_average, K = 1..8, FP32 and FP16 (reduce.cpp:46-89) ---
    red = {}
    for k in (1, 2, 3, 5, 8):
        cs = rng.uniform(-1e-2, 1e-2, (k, n)).astype(np.float32)
        cs[:, 0] = 6e4  # fp16: each decodes to 60000, sum exceeds 65504 before the mean
        cs[:, 1] = np.float32(2.0 ** -20)  # fp16 subnormal contributions
        cs[0, 2] = 7e4  # fp16 overflow -> inf in one contribution
        for prec in (0, 1):
            st, out = R.reduce_average(list(cs), prec)
            assert st == 0
            red[f"in_k{k}"] = cs
            red[f"out_k{k}_p{prec}"] = out
    np.savez_compressed(os.path.join(OUT, "reduce.npz"), **red)

    # --- full DiLoCo trajectory (config-1 shape at small N): K=2, H=5, 2 rounds,
    #     with an injected overflow at (worker 1, step 3) and both precisions ---
    hyper = D.Hyper(inner_lr=4e-4, warmup_steps=5)
    n = 4096
    theta0 = O.rng_fill(4242, "theta", 0, n, -0.05, 0.05)

    def grad_fn(w, t):
        g = O.rng_fill(4242, "grad", w * 1000 + t, n, -1e-2, 1e-2)
        if (w, t) == (1, 3):
            g[17] = np.inf
        return g

    traj = {"theta0": theta0}
    for prec in (0, 1):
        workers, hist = D.simulate(R, theta0, grad_fn, 2, 5, 2, prec, hyper)
        for wi, w in enumerate(workers):
            for name in ("theta_t", "theta_local", "m", "v", "buf"):
                traj[f"p{prec}_w{wi}_{name}"] = getattr(w, name)
            traj[f"p{prec}_w{wi}_step_count"] = w.step_count
            traj[f"p{prec}_w{wi}_scale"] = w.scale
            traj[f"p{prec}_w{wi}_skipped"] = np.array(w.skipped)
        for r, (dbar, applied, _) in enumerate(hist):
            traj[f"p{prec}_r{r}_dbar"] = dbar
            traj[f"p{prec}_r{r}_applied"] = applied
    for k, g in ((0, 0), (1, 0), (0, 3), (1, 3)):
        traj[f"grad_w{k}_t{g}"] = grad_fn(k, g)
    np.savez_compressed(os.path.join(OUT, "diloco_k2_h5.npz"), **traj)
    # --- ODLCKPT1 checkpoint written by the reference's save_checkpoint ---
    n = 1031
    ck = {name: rng.uniform(-1, 1, n).astype(np.float32) for name in ("theta_t", "theta_local", "m", "buf")}
    ck["v"] = rng.uniform(0, 1e-3, n).astype(np.float32)
    ck.update(step_count=17, growth_interval=2000, consecutive_good=5, inner_step=20, outer_epoch=4,
              beta1=np.float32(0.9), beta2=np.float32(0.95), eps=np.float32(1e-8), weight_decay=np.float32(0.1),
              outer_lr=np.float32(0.7), outer_momentum=np.float32(0.9), scale=32768.0, clock_seconds=1.25,
              config_hash=0xC0FFEE, completed_rounds=3, reduce_data_bytes=123456)
    R.checkpoint_write(os.path.join(OUT, "engine.ckpt"), ck)
    np.savez_compressed(os.path.join(OUT, "engine_ckpt.npz"), **{k: np.asarray(v) for k, v in ck.items()})
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
