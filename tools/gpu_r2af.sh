# 4-GPU snapshot: smoke, the whole GPU suite, bench and the reference arm at 1 / 2 / 4 GPUs (development script)
O=gpurun_out/r2af
mkdir -p $O
nvidia-smi -L > $O/gpus.txt; nproc >> $O/gpus.txt; free -g >> $O/gpus.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err
timeout 600 python bench.py --impl reference > $O/ref_1gpu.json 2> $O/ref_1gpu.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --impl reference --gpus $n > $O/ref_${n}gpu.json 2> $O/ref_${n}gpu.err
done
echo done
