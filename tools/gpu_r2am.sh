# 4-GPU: the whole GPU suite and smoke at HEAD (development script)
O=gpurun_out/r2am
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=5 > $O/pytest_gpu.log 2>&1
echo done
