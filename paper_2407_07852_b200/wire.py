"""Device data plane of the reference's cross-box all-reduce.

``Node::Impl::all_reduce`` (collective.cpp:1347-1595) averages pseudo-gradients
between boxes over TCP: encode once at the source, scatter every foreign
partition to its owner as ``reduce_chunk`` frames, owner fold in peer order,
owner encode once, ring all-gather of the owner partitions as
``reduce_result`` frames, then ``DilocoEngine::outer_step``.  ``WireRound``
drives exactly that sequence on one device engine: every frame is produced from
/ consumed into device memory by ``libdiloco_cuda.so`` (include/diloco_cuda.h
section 5), byte-exact with the reference's framing, so a transport only moves
bytes.  The control plane (barrier, commit, membership, retries) stays with the
transport and is out of scope here.
"""
from __future__ import annotations

from . import _capi as A
from .diloco import partition_ranges

DEFAULT_CHUNK_BYTES = 1 << 20  # NodeOptions::chunk_size_bytes, collective.hpp:93


def make_tags(msg_type: int, precision: int, outer_epoch: int, attempt: int, partition: int, peer_id: tuple[int, int],
              chunk_size_bytes: int = DEFAULT_CHUNK_BYTES) -> A.WireTags:
    """Tags of send_chunk_span (collective.cpp:1318-1345); peer_id = PeerId (hi, lo)."""
    return A.WireTags(msg_type, precision, outer_epoch, attempt, partition, peer_id[0], peer_id[1],
                      chunk_size_bytes)


class WireRound:
    """One worker's side of a committed all-reduce round (attempt `attempt`).

    peer_ids: the round's contributors in peer-sorted order (their PeerIds);
    `rank` is this worker's index among them (collective.cpp:1379-1387)."""

    def __init__(self, engine, rank: int, peer_ids, attempt: int = 0, chunk_size_bytes: int = DEFAULT_CHUNK_BYTES):
        self.e = engine
        self.rank = rank
        self.ids = list(peer_ids)
        self.k = len(self.ids)
        self.attempt = attempt
        self.chunk = chunk_size_bytes
        self.prec = engine.config.reduce_precision
        self.ranges = partition_ranges(engine.n, self.k)  # reduce.cpp:20-31
        self.epoch = engine.wire_begin()  # K2, encode once at the source

    def _tags(self, msg_type: int, partition: int, owner: int) -> A.WireTags:
        return make_tags(msg_type, self.prec, self.epoch, self.attempt, partition, self.ids[owner], self.chunk)

    def scatter_frames(self, p: int):
        """reduce_chunk frames of partition p for its owner (collective.cpp:1400-1426)."""
        off, ln = self.ranges[p]
        return self.e.wire_encode(A.WIRE_DELTA, off, ln, self._tags(A.MSG_REDUCE_CHUNK, p, self.rank))

    def accept_contribution(self, j: int, frames):
        """Contributor j's frames for our partition (collective.cpp:1428-1453)."""
        off, ln = self.ranges[self.rank]
        return self.e.wire_decode(A.WIRE_ROW, j, off, ln, frames)

    def fold(self) -> None:
        """Owner fold in peer order + encode once (collective.cpp:1455-1489)."""
        off, ln = self.ranges[self.rank]
        self.e.wire_fold(self.rank, self.k, off, ln)

    def result_frames(self, p: int):
        """reduce_result frames of owner partition p for the ring successor (collective.cpp:1491-1531)."""
        off, ln = self.ranges[p]
        return self.e.wire_encode(A.WIRE_MEAN, off, ln, self._tags(A.MSG_REDUCE_RESULT, p, p))

    def accept_result(self, frames):
        return self.e.wire_decode(A.WIRE_MEAN, 0, 0, self.e.n, frames)

    def finish(self):
        """DilocoEngine::outer_step on the assembled mean (engine.cpp:128-146)."""
        return self.e.wire_finish(self.epoch)


def all_reduce_local(engines, peer_ids, attempt: int = 0, chunk_size_bytes: int = DEFAULT_CHUNK_BYTES,
                     deliver=None):
    """Every worker's round in one process; `deliver(src, dst, frames)` (default:
    identity) is the transport, e.g. a socket pair.  Returns the outer results."""
    k = len(engines)
    deliver = deliver or (lambda src, dst, frames: frames)
    rounds = [WireRound(e, r, peer_ids, attempt, chunk_size_bytes) for r, e in enumerate(engines)]
    for r, rd in enumerate(rounds):  # scatter: every foreign partition to its owner
        for p in range(k):
            if p != r and rd.ranges[p][1]:
                rounds[p].accept_contribution(r, deliver(r, p, rd.scatter_frames(p)))
    for rd in rounds:
        rd.fold()
    for s in range(k - 1):  # ring relay all-gather
        for r, rd in enumerate(rounds):
            send_p = (r + k - s) % k
            if rd.ranges[send_p][1]:
                succ = (r + 1) % k
                rounds[succ].accept_result(deliver(r, succ, rd.result_frames(send_p)))
    return [rd.finish() for rd in rounds]
