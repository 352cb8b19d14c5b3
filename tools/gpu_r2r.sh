# 1-GPU: the GPU suite (incl. the C++ drop-in test) and the bench with the e2e copy ceiling (development script)
O=gpurun_out/r2r
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err
echo done
