# 2/4-GPU: second piece-plan sweep at 150M (uneven plans) (development script)
O=gpurun_out/r2at
mkdir -p $O
for n in 4 2; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/sweep_p2p.py --params 150000000 --no-ordered --steps 30 --repeat 4 --plans "1,2,2,1;1,3,1;1,2,3,2,1;1,3,3,2;1,2,3,1;1,4,2;1,3,3,3,1" > $O/sweep_150m_${n}gpu.log 2> $O/sweep_150m_${n}gpu.err
done
echo done
