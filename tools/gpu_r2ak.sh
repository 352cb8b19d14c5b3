# 2-GPU: multi-GPU suite at HEAD and the 2-GPU bench line (development script)
O=gpurun_out/r2ak
mkdir -p $O
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_world_gpu.py -q -rs > $O/pytest_multi.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 > $O/bench_2gpu.json 2> $O/bench_2gpu.err
echo done
