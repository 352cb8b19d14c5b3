# One 4-GPU gpurun call: smoke, the GPU suite, bench at 1 / 2 / 4 GPUs and the reference arm (development script)
O=gpurun_out/final
mkdir -p $O
head -3 /proc/meminfo > $O/meminfo.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
done
python bench.py --impl reference > $O/ref_1gpu.json 2> $O/ref_1gpu.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29560 bench.py --impl reference --gpus 4 > $O/ref_4gpu.json 2> $O/ref_4gpu.err
