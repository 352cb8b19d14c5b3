"""Whole-vector parity at full size (TEST INFRASTRUCTURE).

Every operation on the DiLoCo path is elementwise across parameters (the fold
is elementwise across workers), and the synthetic inputs come from counter-
based streams addressable by element.  So the oracle's run over
any chunk [lo, lo + L) of the vector is exactly the chunk of the full run, and a
full-size GPU run can be checked on EVERY element by running the oracle chunk
by chunk on the host cores (ctypes releases the GIL, so chunks run in parallel)
and comparing each chunk with the same range downloaded from the engines.
"""
from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_2407_07852_b200 import _capi as A

BUFFERS = ((A.THETA_T, "theta_t"), (A.THETA_LOCAL, "theta_local"), (A.ADAM_M, "m"), (A.ADAM_V, "v"),
           (A.MOMENTUM, "buf"))


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def compare_whole(engines, n: int, chunk: int, oracle_chunk, buffers=BUFFERS, threads: int | None = None):
    """oracle_chunk(lo, length) -> one oracle Worker per engine for elements
    [lo, lo + length).  Compares every element of every buffer of every engine
    bit for bit; returns the number of elements compared."""
    lock = threading.Lock()
    bad = []
    done = [0]

    def task(lo):
        length = min(chunk, n - lo)
        ws = oracle_chunk(lo, length)
        with lock:  # one download at a time (each synchronises the engine stream)
            for wi, e in enumerate(engines):
                for which, attr in buffers:
                    got = e.download_range(which, lo, length)
                    diff = np.flatnonzero(bits(got) != bits(getattr(ws[wi], attr)))
                    if diff.size:
                        bad.append((wi, which, lo + int(diff[0]), int(diff.size)))
            done[0] += length * len(engines) * len(buffers)

    threads = threads or max(1, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(task, range(0, n, chunk)))
    assert not bad, f"{len(bad)} mismatching chunks, first (worker, buffer, element, count): {bad[:8]}"
    return done[0]
