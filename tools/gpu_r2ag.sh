# 1-GPU: the fused single-worker boundary for INPLACE engines — parity, bench with --inner-mode inplace (development script)
O=gpurun_out/r2ag
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_checkpoint.py -q -rs -x > $O/pytest.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1
timeout 300 python bench.py --inner-mode inplace --no-e2e --no-cpu-baseline --no-wire --no-training > $O/bench_inplace.json 2> $O/bench_inplace.err
echo done
