# 4-GPU: K2 fused into the window's last inner step — smoke, the whole GPU suite, bench at 1 / 2 / 4 GPUs (development script)
O=gpurun_out/r2g
mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs -x --durations=10 > $O/pytest_gpu.log 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
timeout 300 python bench.py --no-cpu-baseline > $O/bench_1gpu.json 2> $O/bench_1gpu.err
echo done
