# 2/4-GPU: window boundary A/B (unfused / fused local / fused push / push without fence) + trace of one fused-push boundary (development script)
O=gpurun_out/r2i
mkdir -p $O
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --no-e2e --no-training --no-cpu-baseline --no-wire --steps 5 > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
echo done
