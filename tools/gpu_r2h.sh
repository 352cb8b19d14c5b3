# 4-GPU: fused K2 with the rows pushed into the owners (scatter inside the last inner step) — smoke, GPU suite, bench at 2 / 4 GPUs (development script)
O=gpurun_out/r2h
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_world_gpu.py tests/test_multigpu.py -q -rs -x > $O/pytest_world_multi.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --no-e2e --no-training > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
timeout 1500 python -m pytest tests -m gpu -q -rs -x --deselect tests/test_world_gpu.py --deselect tests/test_multigpu.py > $O/pytest_rest.log 2>&1
echo done
