# 1-GPU: final validation at HEAD — smoke, the GPU suite, bench (development script)
O=gpurun_out/r2aj
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err
echo done
