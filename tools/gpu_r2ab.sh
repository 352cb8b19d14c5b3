# 2/4-GPU: fold CTA sweep with the 1,2,3,2,1 plan (development script)
O=gpurun_out/r2ab
mkdir -p $O
CUDA_VISIBLE_DEVICES=0,1,2,3 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 tools/sweep_p2p.py --no-ordered --steps 10 --repeat 4 --fold-ctas 0 60 100 120 > $O/sweep_ctas_4gpu.log 2> $O/sweep_ctas_4gpu.err
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 tools/sweep_p2p.py --no-ordered --steps 10 --repeat 4 --fold-ctas 0 100 130 200 --fold-threads 0 256 > $O/sweep_ctas_2gpu.log 2> $O/sweep_ctas_2gpu.err
echo done
