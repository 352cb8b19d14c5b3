# 4-GPU: bench lines at HEAD (1 / 2 / 4 GPUs) (development script)
O=gpurun_out/r2ao
mkdir -p $O
timeout 600 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
echo done
