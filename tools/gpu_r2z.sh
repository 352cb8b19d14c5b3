# 2/4-GPU: piece-plan sweep at 1.1B params per worker (development script)
O=gpurun_out/r2z2
mkdir -p $O
for n in 4 2; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/sweep_p2p.py --no-ordered --steps 10 --repeat 8 --plans "1,1,2,2,1,1;1,2,3,2,1" > $O/sweep_1p1b_${n}gpu.log 2> $O/sweep_1p1b_${n}gpu.err
done
echo done
