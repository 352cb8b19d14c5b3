# 4-GPU: NVLink bytes of the owner fold (ncu on a one-process dlc_world), and the in-step A/B of the two TMA fold kernels at 2 and 4 GPUs (development script)
O=gpurun_out/r2o
mkdir -p $O
M=nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((k-1))) timeout 300 python tools/world_step.py --ranks $k > $O/world_step_${k}.json 2> $O/world_step_${k}.err && \
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((k-1))) timeout 900 ncu --metrics $M --clock-control none -k regex:fold_push -c $((6*k)) --csv --log-file $O/ncu_nvlink_fold_${k}.csv python tools/world_step.py --ranks $k > $O/ncu_world_${k}.log 2>&1
done
for n in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n tools/sweep_p2p.py --no-ordered --steps 10 --repeat 6 --fold-kernel 0 1 > $O/ab_fold_kernel_${n}gpu.log 2> $O/ab_fold_kernel_${n}gpu.err
done
echo done
