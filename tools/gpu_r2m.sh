# 1-GPU: bench with the fused single-worker boundary, then its launch list (development script)
O=gpurun_out/r2m
mkdir -p $O
timeout 400 python bench.py --no-cpu-baseline --no-wire > $O/bench_1gpu.json 2> $O/bench_1gpu.err
echo done
