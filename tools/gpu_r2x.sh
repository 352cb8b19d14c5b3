# 1-GPU: launch list of the K = 8 world parity test (TMA fold at KK = 8 on one GPU) (development script)
O=gpurun_out/r2x
mkdir -p $O
timeout 300 python -m pytest tests/test_world_gpu.py -q -k "test_world_shared_device_p2p and 8" > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fold_push|flag_barrier|pseudo_grad_piece|nesterov_p2p_piece|p2p_finish" --csv --log-file $O/launches_k8.csv python -m pytest tests/test_world_gpu.py -q -k "test_world_shared_device_p2p and 8" > $O/ncu.log 2>&1
echo done
