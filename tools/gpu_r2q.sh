# 4-GPU: membership / failure-detector tests, then the multi-GPU parity (development script)
O=gpurun_out/r2q
mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -q -rs > $O/pytest_multigpu.log 2>&1
echo done
