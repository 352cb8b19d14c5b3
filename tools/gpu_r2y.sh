# 2/4-GPU: piece-plan sweep at 150M params per worker (BASELINE configs 2-3) (development script)
O=gpurun_out/r2y
mkdir -p $O
for n in 4 2; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/sweep_p2p.py --params 150000000 --no-ordered --steps 20 --repeat 3 --plans "1,3,3,1;1,1;1,2,1;1;1,2,2,1;1,4,4,1;1,1,1,1,1,1" > $O/sweep_150m_${n}gpu.log 2> $O/sweep_150m_${n}gpu.err
done
echo done
