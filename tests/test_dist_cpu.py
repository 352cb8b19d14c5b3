"""World-size-2 gloo tests of the multi-process host logic (CPU, no GPU).

* the ncclUniqueId made by libdiloco_cuda.so on rank 0 reaches every rank intact;
* max-over-ranks timing;
* a CPU model of the engine's ordered collective plan (pad to K*S, owner r holds
  slot r, scatter, rank-order fold, all-gather) reproduces reduce_average on the
  full vectors bit for bit, for ragged N — the property the NCCL path relies on
  (reduce.cpp:20-89; collective.cpp:1400-1531).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        from oracle import oracle as O
        from paper_2407_07852_b200 import dist as PD
        import paper_2407_07852_b200 as D

        r = PD.init("gloo")
        assert (r.rank, r.world) == (rank, world)
        uid = PD.broadcast_unique_id(D.nccl_unique_id, r.rank, r.world)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(i == ids[0] for i in ids) and len(uid) == 128
        assert PD.max_over_ranks(float(rank) * 3.5, world) == 3.5 * (world - 1)

        port_lib = O.port()
        for n in (1000, 4099, 64 * world + 1):
            S = PD.slot_elems(n, world)
            full = [O.rng_fill(7, "delta", j, n, -1.0, 1.0) * np.float32(2.0 ** j) for j in range(world)]
            mine = np.zeros(world * S, np.float32)
            mine[:n] = full[rank]
            for prec in (0, 1):
                # scatter: slot j of my delta to owner j (grouped send/recv in the engine)
                recv = [None] * world
                reqs = []
                for j in range(world):
                    if j == rank:
                        recv[j] = torch.from_numpy(mine[j * S:(j + 1) * S].copy())
                        continue
                    recv[j] = torch.empty(S)
                    reqs.append(dist.isend(torch.from_numpy(mine[j * S:(j + 1) * S].copy()), j))
                    reqs.append(dist.irecv(recv[j], j))
                for q_ in reqs:
                    q_.wait()
                # owner fold in rank order (K3)
                st, slot = port_lib.reduce_average([t.numpy() for t in recv], prec)
                assert st == 0
                gathered = [torch.empty(S) for _ in range(world)]
                dist.all_gather(gathered, torch.from_numpy(slot))
                dbar = torch.cat(gathered).numpy()[:n]
                _, want = port_lib.reduce_average(full, prec)
                assert np.array_equal(dbar.view(np.uint32), want.view(np.uint32)), (n, prec)
        dist.barrier()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results


def test_gpu_local_memory_is_a_noop_without_nvml_or_when_disabled(monkeypatch):
    """dist.gpu_local_memory: with DLC_NUMA_BIND=0, or where NVML cannot answer (this
    container has no driver), the body runs with the caller's affinity untouched."""
    from paper_2407_07852_b200 import dist as PD
    before = os.sched_getaffinity(0)
    monkeypatch.setenv("DLC_NUMA_BIND", "0")
    with PD.gpu_local_memory(0) as cpus:
        assert cpus is None and os.sched_getaffinity(0) == before
    monkeypatch.delenv("DLC_NUMA_BIND")
    with PD.gpu_local_memory(0) as cpus:
        if cpus is None:
            assert os.sched_getaffinity(0) == before
        else:  # a GPU host: pinned to the GPU-local CPUs inside, restored after
            assert os.sched_getaffinity(0) == set(cpus)
    assert os.sched_getaffinity(0) == before
