# 4-GPU: NCCL-mode failure detector (membership tests), the GPU suite, PCIe probe (development script)
O=gpurun_out/r2p
mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -q -rs -x -k membership > $O/pytest_membership.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1
timeout 300 python tools/pcie_probe.py > $O/pcie.json 2> $O/pcie.err
timeout 300 python tools/pcie_probe.py 1100000000 67108864 > $O/pcie_256mb.json 2>> $O/pcie.err
echo done
