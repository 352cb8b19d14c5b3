# 4-GPU check of the multi-process P2P path after the restructure (development script)
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_world_gpu.py -q -rs --durations=10 > $O/multigpu.log 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --no-cpu-baseline > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
echo done
