# 4-GPU: 150M configs (BASELINE 2-3) at 1 / 2 / 4 GPUs, FP16 and FP32, final code (development script)
O=gpurun_out/r2ar
mkdir -p $O
F="--params 150000000 --no-e2e --no-cpu-baseline --no-wire --no-training --no-boundary"
for p in fp16 fp32; do
  timeout 300 python bench.py $F --precision $p > $O/bench_150m_${p}_1gpu.json 2> $O/err_${p}_1
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n $F --precision $p > $O/bench_150m_${p}_${n}gpu.json 2> $O/err_${p}_${n}
  done
done
echo done
