"""Multi-process plumbing for one DiLoCo worker per GPU (host side only).

torch.distributed (gloo) is the control plane: rendezvous, the 128-byte
ncclUniqueId broadcast, barriers and max-over-ranks timing.  The data plane is
the NCCL communicator inside libdiloco_cuda.so (dlc_collective_create_nccl);
no tensor data ever goes through torch.distributed.
"""
from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass


@dataclass
class Rank:
    rank: int
    world: int
    local: int


def env_rank() -> Rank:
    return Rank(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "gloo") -> Rank:
    """Join the torchrun rendezvous (MASTER_ADDR/PORT from the environment)."""
    import torch.distributed as dist
    r = env_rank()
    if r.world > 1 and not dist.is_initialized():
        dist.init_process_group(backend)
    return r


def broadcast_unique_id(make_id, rank: int, world: int) -> bytes:
    """Rank 0 creates the id with make_id(); every rank returns the same 128 bytes."""
    if world == 1:
        return make_id()
    import torch.distributed as dist
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad ncclUniqueId broadcast")
    return bytes(uid)


def gpu_local_cpus(device: int) -> list | None:
    """Host CPUs NVML reports as closest to `device` (None without NVML)."""
    try:
        import pynvml as N
        N.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        ids = vis.split(",") if vis else None
        phys = int(ids[device]) if ids and ids[device].strip().isdigit() else device
        h = N.nvmlDeviceGetHandleByIndex(phys)
        words = N.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        allowed = os.sched_getaffinity(0)
        cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
        return [c for c in cpus if c in allowed] or None
    except Exception:
        return None


@contextlib.contextmanager
def gpu_local_memory(device: int):
    """Allocate host buffers on `device`'s own NUMA node.

    Runs the body pinned to the GPU-local CPUs, so pinned buffers allocated in it
    (cudaHostAlloc first-touches in the calling thread) land on the GPU's node and
    the e2e path's H2D / D2H copies do not cross the socket interconnect when
    several ranks stream at once.  The previous affinity is restored on exit (the
    pages stay where they are).  Yields the CPU list, or None when NVML is
    unavailable or DLC_NUMA_BIND=0 (nothing changes then)."""
    cpus = None if os.environ.get("DLC_NUMA_BIND", "1") == "0" else gpu_local_cpus(device)
    if not cpus:
        yield None
        return
    prev = os.sched_getaffinity(0)
    os.sched_setaffinity(0, cpus)
    try:
        yield cpus
    finally:
        os.sched_setaffinity(0, prev)


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


SLOT_QUANTUM = 64 * 8  # engine.cu: 64 elements x kMaxPieces


def slot_elems(n: int, k: int) -> int:
    """Owner slot size S used by the engine (engine.cu): ceil(n / k) rounded up to SLOT_QUANTUM."""
    return ((-(-n // k)) + SLOT_QUANTUM - 1) // SLOT_QUANTUM * SLOT_QUANTUM


def make_nccl_collective(rank: Rank, mode: int):
    """NcclCollective for this rank (needs the built library and a GPU)."""
    from . import diloco as D
    uid = broadcast_unique_id(D.nccl_unique_id, rank.rank, rank.world)
    return D.NcclCollective(rank.rank, rank.world, uid, rank.local, mode)
