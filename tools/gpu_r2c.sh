# 1-GPU: fold kernel A/B alone (probe), GPU tests of the fold and the world, ncu of both folds (development script)
O=gpurun_out/r2c
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "fold or probe" tests/test_world_gpu.py -q -rs > $O/pytest.log 2>&1
timeout 600 python tools/p2p_kernels_probe.py --k 2 4 8 --fold-kernel 0 1 --fold-threads 0 128 256 512 --reps 5 > $O/probe.jsonl 2> $O/probe.err
timeout 300 python tools/p2p_kernels_probe.py --k 4 --fold-kernel 0 1 --fold-ctas 0 80 148 --fold-threads 128 256 --reps 5 > $O/probe_ctas.jsonl 2>> $O/probe.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fold_push -c 2 -o $O/fold_ws_vs_leader_k4 python tools/p2p_kernels_probe.py --k 4 --fold-kernel 0 1 --reps 1 > $O/ncu.log 2>&1
echo done
