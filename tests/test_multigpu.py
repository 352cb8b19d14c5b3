"""Multi-GPU parity (NCCL over NVLink): one process per GPU via torchrun.

Runs tests/mp_gpu_worker.py on 2, 3 and 4 ranks (3 = a non-power-of-two fleet
with ragged owner slots); each case is skipped when the box has fewer GPUs.
"""
import os
import subprocess
import sys

import pytest

import paper_2407_07852_b200 as D

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpus():
    try:
        return D.device_count()
    except D.Error:
        return 0


@pytest.mark.parametrize("nproc", [2, 3, 4])
def test_multigpu_parity(nproc):
    if gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc),
           os.path.join(ROOT, "tests", "mp_gpu_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    # ranks share stdout, so their result lines may interleave: count markers
    assert p.returncode == 0 and p.stdout.count("MPRESULT") == nproc, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("nproc", [2, 4])
def test_multigpu_full_size(nproc):
    """Config 4 at its full size (1.1B parameters per worker), slices checked bitwise."""
    if gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29620 + nproc),
           os.path.join(ROOT, "tests", "mp_full_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0 and p.stdout.count("MPRESULT") == nproc, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("nproc", [2, 3, 4])
def test_multigpu_membership_change(nproc):
    """A peer stalls mid-reduce (P2P) or leaves (ordered / allreduce): survivors shrink
    the collective and finish the round with the survivor mean (test_collective.cpp:460-531)."""
    if gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + nproc),
           os.path.join(ROOT, "tests", "mp_fault_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0 and p.stdout.count("MPRESULT") == nproc, p.stdout[-3000:] + p.stderr[-3000:]
