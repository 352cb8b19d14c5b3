"""B200-native DiLoCo optimizer hot path (arXiv 2407.07852, OpenDiLoCo).

The product is libdiloco_cuda.so (sm_100a kernels + NCCL behind the C ABI in
include/diloco_cuda.h).  This package is its Python mirror of the reference
API; importing it fails loudly when the library is not built.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build_library() -> str:
    """Compile libdiloco_cuda.so in-tree for sm_100a (nvcc cross-compiles, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc"), "-j4"], check=True)
    return os.path.join(HERE, "libdiloco_cuda.so")


from . import _capi  # noqa: E402  (raises ImportError when the .so is missing)
from .diloco import *  # noqa: E402,F401,F403
from ._capi import (FP16, FP32, INNER_INPLACE, INNER_PINGPONG, MODE_ALLREDUCE,  # noqa: E402,F401
                    MODE_ORDERED, MODE_P2P, THETA_T, THETA_LOCAL, ADAM_M, ADAM_V, MOMENTUM, GRAD, LR_NONE, LR_COSINE)
