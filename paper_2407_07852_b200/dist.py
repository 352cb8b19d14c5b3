"""Multi-process plumbing for one DiLoCo worker per GPU (host side only).

torch.distributed (gloo) is the control plane: rendezvous, the 128-byte
ncclUniqueId broadcast, barriers and max-over-ranks timing.  The data plane is
the NCCL communicator inside libdiloco_cuda.so (dlc_collective_create_nccl);
no tensor data ever goes through torch.distributed.
"""
from __future__ import annotations

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
