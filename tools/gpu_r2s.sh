# 4-GPU: world tests (shrink in every mode with one rank per GPU) (development script)
O=gpurun_out/r2s
mkdir -p $O
timeout 900 python -m pytest tests/test_world_gpu.py -q -rs > $O/pytest_world.log 2>&1
echo done
