"""Message accounting of the reference's virtual topology.

The reference runs its "ranks" as threads and logs every inter-rank
transfer in a ``MessageLog`` (comms.py:112-155): the time->space exchange
(comms.py:516-535), the two block transposes of each plane's distributed
FFT (transform.py:152-172) and the reduce choreography of the chosen
``ReduceStrategy`` (comms.py:338-417). ``run_pipeline`` reports the byte
and message totals of that log in ``ops`` (pipeline.py:178-186) and writes
it to ``messages.csv`` (pipeline.py:166-168).

On the GPU the image is computed once for any topology (the reference's
result does not depend on it, gridder.py:267-268), so the drop-in derives
the log the reference would have written for ``topo`` instead of running
the choreography: message sizes follow from the mesh, the slab rows and the
per-(source, destination) record counts of the exchange (counted on the GPU
with the reference's halo predicate, ``wsb_route_count``). The entries,
their order-independent CSV and every ``ops`` total equal the reference's.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass

PREPARED_RECORD_BYTES = 48      # comms.py:62-64: gu, gv, plane, time, gindex, value
CELL_BYTES = 16                 # complex128
REDUCE_KINDS = ("direct", "hybrid_ring", "ring_rdma_like")


@dataclass(frozen=True)
class Message:
    phase: str
    src_rank: int
    dst_rank: int
    intra_node: bool
    nbytes: int


class MessageLog:
    """Same interface as the reference's MessageLog (comms.py:119-155)."""

    def __init__(self, entries=None):
        self._entries = list(entries or [])

    def append(self, msg: Message) -> None:
        self._entries.append(msg)

    def entries(self, phase=None, intra_node=None):
        return [m for m in self._entries
                if (phase is None or m.phase == phase)
                and (intra_node is None or m.intra_node == intra_node)]

    def count(self, phase=None, intra_node=None) -> int:
        return len(self.entries(phase, intra_node))

    def total_bytes(self, phase=None, intra_node=None) -> int:
        return sum(m.nbytes for m in self.entries(phase, intra_node))

    def to_csv(self, path) -> None:
        """Rows in canonical (sorted) order under the reference's header
        ``phase,src_rank,dst_rank,intra_node,bytes`` (comms.py:145-155)."""
        rows = sorted((m.phase, m.src_rank, m.dst_rank, int(m.intra_node), m.nbytes)
                      for m in self._entries)
        with open(path, "w", newline="") as fh:
            wr = csv.writer(fh)
            wr.writerow(["phase", "src_rank", "dst_rank", "intra_node", "bytes"])
            wr.writerows(rows)


def _split(n: int, parts: int, index: int):
    """partition_1d (mesh.py:34-45): (start, count)."""
    q, r = divmod(n, parts)
    return (index * (q + 1), q + 1) if index < r else (r * (q + 1) + (index - r) * q, q)


class _Topo:
    """The fields of a reference Topology (comms.py:67-97) this module needs."""

    def __init__(self, topo):
        self.n_nodes = int(topo.n_nodes)
        self.per_node = int(topo.ranks_per_node)
        self.n_ranks = self.n_nodes * self.per_node

    def node(self, rank: int) -> int:
        return rank // self.per_node

    def ranks(self, node: int):
        return range(node * self.per_node, (node + 1) * self.per_node)

    def msg(self, phase, src, dst, nbytes):
        return Message(phase, src, dst, self.node(src) == self.node(dst), int(nbytes))


def exchange_messages(topo, counts):
    """One (possibly empty) message from every rank to every other rank,
    ``counts[s][d]`` prepared records each (comms.py:516-524)."""
    t = _Topo(topo)
    R = t.n_ranks
    return [t.msg("exchange", s, d, counts[s][d] * PREPARED_RECORD_BYTES)
            for s in range(R) for d in range(R) if d != s]


def fft_messages(topo, n_u: int, n_v: int, n_w: int):
    """Per plane, the forward block transpose (rank r's rows x d's columns)
    and the transpose back (r's columns x d's rows) of fft2d_slab
    (transform.py:152-172)."""
    t = _Topo(topo)
    R = t.n_ranks
    rows = [_split(n_v, R, r)[1] for r in range(R)]
    cols = [_split(n_u, R, r)[1] for r in range(R)]
    one = [t.msg("fft", r, d, rows[r] * cols[d] * CELL_BYTES) for r in range(R) for d in range(R)
           if d != r]
    one += [t.msg("fft", r, d, cols[r] * rows[d] * CELL_BYTES) for r in range(R) for d in range(R)
            if d != r]
    return one * n_w


def _reduce_target(t: _Topo, kind: str, length: int, target: int):
    """Messages of one reduce onto ``target`` of a flat partial of ``length``
    complex128 values held by every rank (comms.py:338-417)."""
    R = t.n_ranks
    out = []
    if kind == "direct":
        return [t.msg("reduce", r, target, length * CELL_BYTES) for r in range(R) if r != target]
    P = t.per_node
    seg = math.ceil(length / P) if P > 1 else length
    # intra-node ring reduce-scatter: P-1 steps, every member forwards one
    # (padded) segment to its successor (comms.py:310-335)
    if P > 1:
        for node in range(t.n_nodes):
            grp = list(t.ranks(node))
            for _ in range(P - 1):
                for pos, r in enumerate(grp):
                    out.append(t.msg("reduce", r, grp[(pos + 1) % P], seg * CELL_BYTES))
    t_node = t.node(target)
    chain = [n for n in range(t.n_nodes) if n != t_node] + [t_node]
    if kind == "hybrid_ring":
        for node in range(t.n_nodes):       # segments gathered on the node master
            grp = list(t.ranks(node))
            for r in grp[1:]:
                out.append(t.msg("reduce", r, grp[0], seg * CELL_BYTES))
        for k in range(len(chain) - 1):     # node sums chained master to master
            out.append(t.msg("reduce", chain[k] * P, chain[k + 1] * P, length * CELL_BYTES))
        if target != t_node * P:            # the target node's master delivers
            out.append(t.msg("reduce", t_node * P, target, length * CELL_BYTES))
        return out
    # ring_rdma_like: segment owners chain straight to their peers on the
    # next node, then deliver to the target inside the target node
    for k in range(len(chain) - 1):
        for pos in range(P):
            out.append(t.msg("reduce", chain[k] * P + pos, chain[k + 1] * P + pos,
                             seg * CELL_BYTES))
    for r in t.ranks(t_node):
        if r != target:
            out.append(t.msg("reduce", r, target, seg * CELL_BYTES))
    return out


def reduce_messages(topo, kind: str, n_u: int, n_v: int, n_w: int):
    """run_pipeline's reduce phase: one reduce per target slab, every rank
    contributing a partial of that slab's size (pipeline.py:117-122)."""
    if kind not in REDUCE_KINDS:
        raise ValueError(f"reduce kind must be one of {REDUCE_KINDS}, got {kind!r}")
    t = _Topo(topo)
    out = []
    for target in range(t.n_ranks):
        rows = _split(n_v, t.n_ranks, target)[1]
        out += _reduce_target(t, kind, n_w * rows * n_u, target)
    return out


def virtual_log(topo, kind: str, n_u: int, n_v: int, n_w: int, counts) -> MessageLog:
    """The MessageLog of run_pipeline on ``topo`` (exchange, reduce, fft)."""
    log = MessageLog()
    for m in exchange_messages(topo, counts):
        log.append(m)
    for m in reduce_messages(topo, kind, n_u, n_v, n_w):
        log.append(m)
    for m in fft_messages(topo, n_u, n_v, n_w):
        log.append(m)
    return log
