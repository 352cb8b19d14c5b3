# 2/4-GPU: window boundary A/B with the bulk-copy push in K1; world + multi-GPU parity (development script)
O=gpurun_out/r2j
mkdir -p $O
timeout 900 python -m pytest tests/test_world_gpu.py -q -rs -x > $O/pytest_world.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --no-e2e --no-training --no-cpu-baseline --no-wire --steps 5 > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
echo done
timeout 900 python -m pytest tests/test_multigpu.py -q -rs -x > $O/pytest_multi.log 2>&1
