# 1-GPU: the fused single-worker window boundary (K1+K2+K4) — smoke, GPU suite, bench (development script)
O=gpurun_out/r2l
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rs -x -k "fused_solo or run_training" > $O/pytest_fused.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-wire > $O/bench_1gpu.json 2> $O/bench_1gpu.err
echo done
