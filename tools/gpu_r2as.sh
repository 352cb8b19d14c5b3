# 4-GPU: DLC_TRACE timeline of the 150M P2P step (development script)
O=gpurun_out/r2as
mkdir -p $O
DLC_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 4 --params 150000000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-wire --no-training --no-boundary > $O/bench.json 2> $O/trace.log
echo done
