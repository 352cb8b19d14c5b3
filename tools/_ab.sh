run() { timeout 600 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --mode allreduce --steps 6 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],3), d.get('phases_ms'))"; }
run X=0
run NCCL_MAX_NCHANNELS=8
run NCCL_MAX_NCHANNELS=16
run NCCL_MAX_NCHANNELS=4
run NCCL_PROTO=Simple
run DLC_AR_SERIAL=1
run X=0
