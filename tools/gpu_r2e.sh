# 4-GPU: checkpoint tests; longer interleaved in-step A/B of the fold kernels; NVLink counter probe (development script)
O=gpurun_out/r2e
mkdir -p $O
timeout 600 python -m pytest tests/test_checkpoint.py -q -rs > $O/pytest_ckpt.log 2>&1
timeout 300 python tools/nvlink_probe.py > $O/nvlink_probe.json 2> $O/nvlink_probe.err
for n in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n tools/sweep_p2p.py --no-ordered --steps 10 --repeat 4 --fold-kernel 0 1 --fold-threads 128 256 > $O/sweep_${n}gpu.log 2> $O/sweep_${n}gpu.err
done
echo done
