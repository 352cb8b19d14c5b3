timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "parity" > gpurun_out/c150_pytest.log 2>&1
for p in fp16 fp32; do for n in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n --params 150000000 --precision $p > gpurun_out/c150b_${p}_${n}gpu.json 2>/dev/null
done; done
