# 4-GPU: in-step A/B of the fold kernels and their thread / CTA counts (development script)
O=gpurun_out/r2d
mkdir -p $O
for n in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n tools/sweep_p2p.py --no-ordered --steps 8 --repeat 2 --fold-kernel 0 --fold-threads 128 256 512 --fold-ctas 0 40 120 > $O/sweep_${n}gpu.log 2> $O/sweep_${n}gpu.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n tools/sweep_p2p.py --no-ordered --steps 8 --repeat 2 --fold-kernel 1 > $O/sweep_${n}gpu_leader.log 2>> $O/sweep_${n}gpu.err
done
timeout 300 python tools/nvlink_probe.py > $O/nvlink_probe.json 2> $O/nvlink_probe.err
echo done
