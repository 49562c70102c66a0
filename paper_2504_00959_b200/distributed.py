"""Multi-GPU w-stacking: v-slab decomposition over one process per GPU.

Mirrors the reference's distributed structure:
  1. time->space exchange of the prepared records to the slab owners, with
     the +-S halo duplicates (exchange_to_space_order, comms.py:495-547),
     as one NCCL all-to-all-v;
  2. per-slab gridding (grid_sector, gridder.py:186-259);
  3. distributed inverse FFT: row pass on the slab, one all-to-all block
     transpose per plane (fft2d_slab, transform.py:130-177), column pass on
     full columns; the reference's transpose back is not needed because the
     column pass also applies the w screen and stacks the planes
     (transform.py:192-230);
  4. gather of the image strips and of the per-column residual norms to the
     root (assemble_image, transform.py:233-241).
The reference's reduce phase (comms.py:420-454) is the identity after the
exchange (pipeline.py:117-122) and has no counterpart here.

Every numeric stage runs through a backend; the product backend is
``CudaBackend`` (libwsb.so). The collectives are torch.distributed calls,
NCCL over NVLink on the GPU box. In this v-slab mode (the default,
deterministic=True) the image is bit-identical to the single-GPU image for
any number of ranks whose slab starts lie on the gridder's 128-row item
boundaries (partition_1d of a power-of-two mesh over 2/4/8 ranks; balanced
starts are rounded to them): records reach each slab in gindex order, every
cell is accumulated in (anchor row, record) order inside an item that holds
the same records on any GPU count, and the norms are summed per column in
global column order. The w-plane decomposition (decomposition="planes") is
a faster mode whose image agrees to ~1e-16 relative (the plane sum
associates differently).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .imager import (FinalImage, _ptr, as_grid_spec, as_kernel_spec, context, grid_slab_device,
                     last_timings, partition_1d, prepare_device)

G = L.P_GROUP


class CudaBackend:
    """Stage implementations on the local GPU (libwsb.so)."""

    def __init__(self, device=None):
        self.ctx = context(device)
        self.device = torch.device("cuda", self.ctx.device)

    def prepare(self, u, v, w, vis, weight, spec):
        return prepare_device(u, v, w, vis, weight, spec, device=self.device)

    def row_histogram(self, rec, spec):
        """Records per anchor row floor(gv), int64 [n_v] on the device."""
        g = spec.c_struct()
        h = torch.empty(spec.n_v, dtype=torch.int32, device=self.device)
        L.check(L.lib().wsb_row_histogram(self.ctx.handle, C.byref(g), _ptr(rec), rec.shape[0],
                                          _ptr(h)))
        return h.to(torch.int64)

    def route(self, rec, plane, spec, S, R, starts=None):
        g = spec.c_struct()
        n = rec.shape[0]
        counts = (C.c_int64 * R)()
        st = None if starts is None else (C.c_int32 * (R + 1))(*starts)
        L.check(L.lib().wsb_route_count(self.ctx.handle, C.byref(g), S, R, st, _ptr(rec), n, counts))
        counts = [int(c) for c in counts]
        tot = sum(counts)
        srec = torch.empty((max(tot, 1), 4), dtype=torch.float64, device=self.device)
        spl = torch.empty(max(tot, 1), dtype=torch.int32, device=self.device)
        L.check(L.lib().wsb_route_pack(self.ctx.handle, C.byref(g), S, R, st, _ptr(rec), _ptr(plane),
                                       n, _ptr(srec), _ptr(spl), None))
        return srec[:tot], spl[:tot], counts

    def grid_slab(self, rec, plane, spec, kern, v0, vc):
        return grid_slab_device(rec, plane, spec, kern, v0, vc)

    def fft_rows(self, grid_s, spec, vc, dest_pairs, plane_lo=0, plane_hi=None):
        """Row pass of planes [plane_lo, plane_hi): strip-layout slab in; out:
        float64 buffer laid out [dest][plane - plane_lo][pair][row][G][2] (the
        all-to-all send buffer)."""
        plane_hi = spec.n_w if plane_hi is None else plane_hi
        g = spec.c_struct()
        grid_p = torch.empty((plane_hi - plane_lo) * spec.n_u * vc * 2, dtype=torch.float64,
                             device=self.device)
        pairs = (C.c_int32 * len(dest_pairs))(*dest_pairs)
        L.check(L.lib().wsb_fft_rows(self.ctx.handle, C.byref(g), int(vc), _ptr(grid_s),
                                     _ptr(grid_p), int(plane_lo), int(plane_hi), len(dest_pairs),
                                     pairs))
        return grid_p

    def fft_rows_peer(self, grid_s, spec, vc, dest_cols, dest_ptrs):
        """Row pass of all planes stored into the destinations' column-pass
        inputs through device pointers (peer memory)."""
        g = spec.c_struct()
        R = len(dest_cols)
        cols = (C.c_int32 * R)(*dest_cols)
        ptrs = (C.c_void_p * R)(*dest_ptrs)
        L.check(L.lib().wsb_fft_rows_peer(self.ctx.handle, C.byref(g), int(vc), _ptr(grid_s), 0,
                                          spec.n_w, R, cols, ptrs))

    def push_blocks(self, srcs, dsts, nbytes, stream):
        """One launch copying block d: srcs[d] -> dsts[d] (device addresses,
        dsts may be peer memory), enqueued on ``stream``."""
        R = len(srcs)
        lib, h = L.lib(), self.ctx.handle
        L.check(lib.wsb_ctx_set_stream(h, C.c_void_p(stream.cuda_stream)))
        try:
            L.check(lib.wsb_push_blocks(h, R, (C.c_void_p * R)(*srcs), (C.c_void_p * R)(*dsts),
                                        (C.c_int64 * R)(*nbytes)))
        finally:
            L.check(lib.wsb_ctx_set_stream(h, C.c_void_p(torch.cuda.current_stream(self.device)
                                                         .cuda_stream)))

    def fft_cols_stack(self, tgrid, spec, src_rows, g0, ng, plane_lo=0, plane_hi=None):
        """Column pass + stack of planes [plane_lo, plane_hi) (ranges in
        descending order; the context carries the running stack). Returns
        (strip, partials) after the range starting at plane 0, (None, None)
        before."""
        plane_hi = spec.n_w if plane_hi is None else plane_hi
        g = spec.c_struct()
        final = plane_lo == 0
        strip = torch.empty((spec.n_v, ng * G) if final else (1,), dtype=torch.float64,
                            device=self.device)
        partials = torch.empty((col_split(spec.n_v), ng * G, 2) if final else (1,),
                               dtype=torch.float64, device=self.device)
        rows = (C.c_int32 * len(src_rows))(*src_rows)
        L.check(L.lib().wsb_fft_cols_stack(self.ctx.handle, C.byref(g), len(src_rows), rows, int(g0),
                                           int(ng), int(plane_lo), int(plane_hi), _ptr(tgrid),
                                           _ptr(strip), _ptr(partials)))
        return (strip, partials) if final else (None, None)

    # ---- w-plane decomposition ------------------------------------------------
    def plane_histogram(self, plane, spec):
        """Records per w plane, int64 [n_w] on the device."""
        g = spec.c_struct()
        h = torch.empty(spec.n_w, dtype=torch.int32, device=self.device)
        L.check(L.lib().wsb_plane_histogram(self.ctx.handle, C.byref(g), _ptr(plane),
                                            plane.shape[0], _ptr(h)))
        return h.to(torch.int64)

    def route_planes(self, rec, plane, spec, R, starts):
        """Records to the owners of their planes; planes rebased per owner."""
        g = spec.c_struct()
        n = rec.shape[0]
        counts = (C.c_int64 * R)()
        st = (C.c_int32 * (R + 1))(*starts)
        lib, h = L.lib(), self.ctx.handle
        L.check(lib.wsb_route_planes_count(h, C.byref(g), R, st, _ptr(rec), _ptr(plane), n, counts))
        counts = [int(c) for c in counts]
        tot = sum(counts)
        srec = torch.empty((max(tot, 1), 4), dtype=torch.float64, device=self.device)
        spl = torch.empty(max(tot, 1), dtype=torch.int32, device=self.device)
        L.check(lib.wsb_route_planes_pack(h, C.byref(g), R, st, _ptr(rec), _ptr(plane), n,
                                          _ptr(srec), _ptr(spl), None))
        return srec[:tot], spl[:tot], counts

    def fft_cols_partial(self, tgrid, spec, plane_lo, plane_hi, rank_lo, rank_hi, pimg):
        """Column pass + stack of planes [plane_lo, plane_hi) of this rank's
        [rank_lo, rank_hi); the call starting at rank_lo writes ``pimg``
        (complex128 [n_v][n_u] as float64 [..., 2])."""
        g = spec.c_struct()
        L.check(L.lib().wsb_fft_cols_partial(self.ctx.handle, C.byref(g), int(plane_lo),
                                             int(plane_hi), int(rank_lo), int(rank_hi),
                                             _ptr(tgrid), _ptr(pimg)))

    def image_finish(self, pimg, spec):
        """Summed partial stacks -> (image [n_v, n_u], norm partials [RS, n_u, 2])."""
        g = spec.c_struct()
        img = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, device=self.device)
        parts = torch.empty((finish_split(spec.n_v), spec.n_u, 2), dtype=torch.float64,
                            device=self.device)
        L.check(L.lib().wsb_image_finish(self.ctx.handle, C.byref(g), _ptr(pimg), _ptr(img),
                                         _ptr(parts)))
        return img, parts


def finish_split(n_v: int) -> int:
    """WSB_FINISH_SPLIT: row blocks of wsb_image_finish's norm partials."""
    return 16 if n_v >= 4096 else (n_v // 256 if n_v >= 256 else 1)


def _a2a(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group, async_op=False):
    return dist.all_to_all_single(out, inp, output_split_sizes=list(out_splits),
                                  input_split_sizes=list(in_splits), group=group,
                                  async_op=async_op)


def plane_ranges(n_w: int, n_ranges: int):
    """Contiguous plane ranges of the pipelined transpose (partition_1d)."""
    n_ranges = max(1, min(n_ranges, n_w))
    return [(a, a + c) for a, c in (partition_1d(n_w, n_ranges, i) for i in range(n_ranges))]


class _Stages:
    """CUDA events on the compute stream between pipeline stages (optional)."""

    def __init__(self, on: bool, device):
        self.on, self.device, self.marks = on, device, []

    def mark(self, name):
        if self.on:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(self.device))
            self.marks.append((name, ev))

    def ms(self):
        if not self.on or len(self.marks) < 2:
            return {}
        torch.cuda.current_stream(self.device).synchronize()
        return {b[0]: a[1].elapsed_time(b[1]) for a, b in zip(self.marks, self.marks[1:])}


ITEM_ROWS = 128       # csrc/wsb_internal.cuh kItemRows: the gridder's row blocks


def balanced_slab_starts(row_counts, n_ranks: int, row_weight: float = 10_000.0,
                         max_rows: int | None = None, align: int = ITEM_ROWS):
    """Slab rows with equal estimated work instead of partition_1d's equal
    rows. A slab's cost is modelled as records + row_weight * rows (the
    gridder scales with the records, the row pass and the sweep's row
    emission with the rows; row_weight ~ records-equivalent of one row,
    measured on cfg3). Returns starts[0..R] with starts[R] = n_v and every
    slab at least one row. The image does not depend on the slab rows.
    ``align``: slab starts are rounded to multiples of it when the mesh has
    room (n_v >= align * n_ranks): slabs that start on the gridder's 128-row
    item boundaries grid every cell exactly as one GPU does, so the image is
    bit-identical for any rank count."""
    import numpy as np
    h = np.asarray(row_counts, dtype=np.float64)
    n_v = h.shape[0]
    cost = np.cumsum(h + row_weight)
    total = cost[-1]
    starts = [0]
    for d in range(1, n_ranks):
        # boundary whose prefix cost (rows above it) is closest to d/R of the total
        target = total * d / n_ranks
        i = int(np.searchsorted(cost, target, side="left"))
        r = i if i > 0 and target - cost[i - 1] <= cost[min(i, n_v - 1)] - target else i + 1
        r = max(r, starts[-1] + 1)
        r = min(r, n_v - (n_ranks - d))
        starts.append(r)
    starts.append(n_v)
    if align > 1 and n_v >= align * n_ranks and n_v % align == 0:
        for d in range(1, n_ranks):
            a_ = int(round(starts[d] / align)) * align
            starts[d] = min(max(a_, starts[d - 1] + align), n_v - (n_ranks - d) * align)
    # memory bound: no slab taller than max_rows (default 1.5x the equal share;
    # the slab's grid and transforms scale with its rows)
    if max_rows is None:
        max_rows = -(-3 * n_v // (2 * n_ranks))
    max_rows = max(max_rows, -(-n_v // n_ranks))
    step = align if (align > 1 and n_v >= align * n_ranks and n_v % align == 0) else 1
    max_rows = max(step, max_rows // step * step)
    for d in range(1, n_ranks):
        starts[d] = min(starts[d], starts[d - 1] + max_rows)
    for d in range(n_ranks - 1, 0, -1):
        starts[d] = max(starts[d], starts[d + 1] - max_rows)
    return starts


ONCHIP_FFT_N = 4096   # include/wsb.h WSB_ONCHIP_FFT_N


def col_split(n_v: int) -> int:
    """WSB_COL_SPLIT: residue classes of the column pass (norm partials are
    [residue][column][2])."""
    return n_v // ONCHIP_FFT_N if n_v > ONCHIP_FFT_N else 1


_SYMM: dict = {}
_ROW_CAP: dict = {}


def _symm_available() -> bool:
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
        return True
    except Exception:
        return False


_SIDE: dict = {}


def _side_stream(dev):
    if dev.index not in _SIDE:
        _SIDE[dev.index] = torch.cuda.Stream(dev)
    return _SIDE[dev.index]


def _symm_buffer(elems: int, dev, group, tag: str = "transpose"):
    """Symmetric (peer-mapped) float64 buffer of 2*elems values on every rank,
    cached per tag: the rendezvous is collective and costly. Keeps the
    largest (all ranks must ask for the same size)."""
    import torch.distributed._symmetric_memory as symm
    key = (tag, id(group), dev.index)
    hit = _SYMM.get(key)
    if hit is None or hit[0].numel() < 2 * elems:
        _SYMM.pop(key, None)
        buf = symm.empty(2 * elems, dtype=torch.float64, device=dev)
        hdl = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
        _SYMM[key] = (buf, hdl)
    return _SYMM[key]


def _exchange(be, srec, spl, counts, group, exchange: str = "auto"):
    """Time->space exchange of packed records: block d of (srec, spl) goes to
    rank d, blocks arrive in source-rank (gindex) order. "push": NVLink stores
    into symmetric memory; "nccl": all-to-all-v. Returns (records, planes, m)."""
    R = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = be.device
    if exchange == "auto":
        exchange = ("push" if (hasattr(be, "push_blocks") and dev.type == "cuda"
                               and _symm_available()) else "nccl")
    if exchange == "push":
        # every rank learns the whole count matrix, then pushes its block for
        # slab d straight into d's receive buffer (symmetric memory, NVLink
        # stores) at the offset of its rank in gindex order
        cm = torch.empty((R, R), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(cm, torch.tensor(counts, dtype=torch.int64, device=dev),
                                    group=group)
        cmat = cm.tolist()                                  # cmat[s][d]
        recv_counts = [cmat[s_][r] for s_ in range(R)]
        m = sum(recv_counts)
        need = max(sum(cmat[s_][d] for s_ in range(R)) for d in range(R))
        cap = max(1, -(-need * 5 // 4))                    # 25% headroom against re-rendezvous
        # records: 4 float64 each (2 * 2cap values); planes: int32, viewed in a float64 buffer
        rbuf, rh = _symm_buffer(2 * cap, dev, group, "records")
        pbuf, ph = _symm_buffer(-(-cap // 4) + 1, dev, group, "planes")
        if rbuf.numel() < 4 * need or pbuf.numel() * 2 < need:
            raise RuntimeError("symmetric exchange buffers out of sync")
        rh.barrier(channel=0)                               # the previous slab has been gridded
        srcs_r, dsts_r, b_r, srcs_p, dsts_p, b_p = [], [], [], [], [], []
        sent = 0
        for d in range(R):
            off = sum(cmat[s_][d] for s_ in range(r))       # my place in d's buffer
            srcs_r.append(srec.data_ptr() + 32 * sent)
            dsts_r.append(rh.buffer_ptrs[d] + 32 * off)
            b_r.append(32 * counts[d])
            srcs_p.append(spl.data_ptr() + 4 * sent)
            dsts_p.append(ph.buffer_ptrs[d] + 4 * off)
            b_p.append(4 * counts[d])
            sent += counts[d]
        cur = torch.cuda.current_stream(dev)
        be.push_blocks(srcs_r, dsts_r, b_r, cur)
        be.push_blocks(srcs_p, dsts_p, b_p, cur)
        rh.barrier(channel=0)                               # every block has landed
        rrec = rbuf[: 4 * m].view(m, 4)
        rpl = pbuf.view(torch.int32)[:m]
    else:
        c_send = torch.tensor(counts, dtype=torch.int64, device=dev)
        c_recv = torch.empty(R, dtype=torch.int64, device=dev)
        dist.all_to_all_single(c_recv, c_send, group=group)
        recv_counts = [int(x) for x in c_recv.tolist()]
        m = sum(recv_counts)
        rrec = torch.empty((m, 4), dtype=torch.float64, device=dev)
        rpl = torch.empty(m, dtype=torch.int32, device=dev)
        _a2a(rrec, srec.contiguous(), recv_counts, counts, group)
        _a2a(rpl, spl.contiguous(), recv_counts, counts, group)
    return rrec, rpl, m


def image_distributed(u, v, w, vis, weight, spec, kern, group=None, backend=None, root: int = 0,
                      to_host: bool = True, n_ranges: int = 4, timings: dict | None = None,
                      balance: bool = True, row_weight: float = 10_000.0,
                      transpose: str = "auto", exchange: str = "auto",
                      decomposition: str = "auto", plane_weight: float | None = None,
                      deterministic: bool = True):
    """Dirty image of the union of every rank's records. Each rank passes its
    own time partition (records in gindex order, rank r holding the r-th
    contiguous block, as visdata.partition_time_ordered produces).

    ``transpose``: "push" (default on GPUs) overlaps NVLink pushes of each
    plane range (a copy kernel into the destinations' inputs in symmetric
    memory) with the row pass of the next range; "peer" fuses the slab
    transpose into the row pass -- its
    results are stored straight into the destination ranks' column-pass
    inputs in symmetric memory over NVLink (wsb_fft_rows_peer); "nccl"
    pipelines an NCCL all-to-all over ``n_ranges`` plane ranges (from the top
    plane down, the stacking order of the column pass): the all-to-all of one
    range runs on NCCL's stream while the row pass of the next range and the
    column pass of the previous one run on the compute stream; "auto" picks
    "push" when the backend and torch's symmetric memory support it. The
    result does not depend on the choice.
    ``timings``, if a dict, receives per-stage milliseconds of the compute
    stream (and the bucket / sweep split of the gridder).
    ``balance`` sizes the v-slabs for equal work from a global histogram of
    the anchor rows (one all-reduce of n_v counts) instead of partition_1d's
    equal rows: Earth-rotation tracks put most records in the central rows.
    ``decomposition``: "auto" (v-slabs when ``deterministic``, the
    default -- the reference's ReduceStrategy default -- else w-plane ranges
    when every rank gets a plane), "slabs" (the reference's v-slabs, above;
    the image is bit-identical to the single-GPU one for any R when the slab
    starts lie on the gridder's 128-row item boundaries: partition_1d of a
    power-of-two mesh over 2/4/8 ranks, and the balanced starts, which are
    rounded to them) or "planes" (a performance mode, measured faster on 2
    and 4 GPUs: cfg2 4.30 vs 4.93 ms/step, cfg3 16.9 vs 21.8 ms/step at N=4
    in round 1): rank d owns a contiguous range of w
    planes (balanced on records per plane + ``plane_weight`` records per
    plane's transforms), grids them over the whole mesh, transforms and
    stacks them locally, and the ranks' complex partial stacks are summed by
    one NCCL reduce to the root -- no grid transpose; the image agrees with
    the single-GPU one to rounding (~1e-16 relative; the stack's association
    over planes depends on R).

    Returns (FinalImage on ``root``, None elsewhere; diag dict on every rank)."""
    spec, kern = as_grid_spec(spec), as_kernel_spec(kern)
    be = backend or CudaBackend()
    R = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = be.device
    S = kern.half_support
    n_groups = spec.n_u // G
    if R > spec.n_v or R > n_groups:
        raise ValueError(f"{R} ranks exceed the mesh ({spec.n_v} rows, {n_groups} column groups)")

    st = _Stages(timings is not None and dev.type == "cuda", dev)
    st.mark("start")

    # 1. prepare + time->space exchange ------------------------------------
    rec, plane = be.prepare(u, v, w, vis, weight, spec)
    st.mark("prepare")
    if decomposition == "auto":
        # deterministic (the reference's ReduceStrategy default): v-slabs,
        # bit-identical for any R; else the faster w-plane ranges
        decomposition = ("slabs" if deterministic or R > spec.n_w or not hasattr(be, "route_planes")
                         else "planes")
    if decomposition == "planes":
        return _image_planes(be, rec, plane, spec, kern, group, root, to_host, timings, st,
                             balance, plane_weight, exchange)
    if decomposition != "slabs":
        raise ValueError(f"unknown decomposition {decomposition!r}")
    if balance and R > 1:
        hist = be.row_histogram(rec, spec)
        dist.all_reduce(hist, group=group)
        # memory bound on a slab's rows: its strip grid and row-pass output
        # (2 x n_w x n_u complex128 per row) within ~60% of the free memory
        # of the tightest rank
        max_rows = None
        if dev.type == "cuda":
            key = (id(group), dev.index, spec.n_u, spec.n_v, spec.n_w, R)
            if key not in _ROW_CAP:     # once per mesh: a collective + host sync
                free = torch.tensor([torch.cuda.mem_get_info(dev)[0]], dtype=torch.float64,
                                    device=dev)
                dist.all_reduce(free, op=dist.ReduceOp.MIN, group=group)
                _ROW_CAP[key] = int(0.6 * float(free.item()) / (2 * spec.n_w * spec.n_u * 16))
            max_rows = _ROW_CAP[key]
        starts = balanced_slab_starts(hist.cpu().numpy(), R, row_weight,
                                      max_rows=min(spec.n_v, max_rows) if max_rows else spec.n_v)
    else:
        starts = [partition_1d(spec.n_v, R, d)[0] for d in range(R)] + [spec.n_v]
    slabs = [(starts[d], starts[d + 1] - starts[d]) for d in range(R)]
    srec, spl, counts = be.route(rec, plane, spec, S, R, starts)
    n_local = int(rec.shape[0])
    del rec, plane                  # large meshes: keep the peak footprint down
    st.mark("route")
    rrec, rpl, m = _exchange(be, srec, spl, counts, group, exchange)
    del srec, spl
    st.mark("exchange")

    # 2. grid this rank's slab ----------------------------------------------
    v0, vc = slabs[r]
    grid_s, updates = be.grid_slab(rrec, rpl, spec, kern, v0, vc)
    st.mark("grid")
    split = last_timings(dev)[0][1:3] if st.on else None
    del rrec, rpl

    # 3. row FFT, all-to-all block transpose, column FFT + w stack, pipelined
    #    over plane ranges ----------------------------------------------------
    cols = [partition_1d(n_groups, R, d) for d in range(R)]
    g0, ng = cols[r]
    dest_pairs = [ng_d for _, ng_d in cols]
    src_rows = [vc_s for _, vc_s in slabs]
    # plane ranges of at most ~4 GiB of row-pass output each (cfg4 meshes)
    n_ranges = max(n_ranges, -(-spec.n_w * spec.n_u * vc * 16 // (4 << 30)))
    if transpose == "auto":
        # measured: the NVLink push beats NCCL's all-to-all on 2 GPUs (cfg2
        # 5.98 vs 6.60 ms/step); on 4 the pushes' CTAs slow the concurrent row
        # pass more than NCCL does (cfg3 27.7 vs 23.0 ms/step)
        transpose = "push" if (R == 2 and hasattr(be, "push_blocks") and dev.type == "cuda"
                               and _symm_available()) else "nccl"
    if transpose == "push":
        # row pass into local destination-major plane ranges; each range is
        # pushed by a copy kernel on a side stream straight into the other
        # ranks' column-pass inputs (symmetric memory, NVLink stores) while
        # the next range is transformed; one device-side barrier, then the
        # column pass over all planes. Every rank's input:
        # [s][plane][g][row - r0_s].
        elems = spec.n_w * max(dest_pairs) * G * spec.n_v
        buf, hdl = _symm_buffer(elems, dev, group)
        cur = torch.cuda.current_stream(dev)
        ps = _side_stream(dev)
        hdl.barrier(channel=0)          # every rank has finished reading the previous image
        ps.wait_stream(cur)
        for k0, k1 in reversed(plane_ranges(spec.n_w, n_ranges)):
            nk = k1 - k0
            grid_p = be.fft_rows(grid_s, spec, vc, dest_pairs, k0, k1)  # [dest][plane][g][row][G]
            srcs, dsts, nbytes = [], [], []
            lo = 0
            for d in range(R):
                n_el = nk * dest_pairs[d] * G * vc              # complex128 elements
                srcs.append(grid_p.data_ptr() + 16 * nk * vc * G * lo)
                blk = spec.n_w * dest_pairs[d] * G * slabs[r][0] + k0 * dest_pairs[d] * G * vc
                dsts.append(hdl.buffer_ptrs[d] + 16 * blk)
                nbytes.append(16 * n_el)
                lo += dest_pairs[d]
            ev = torch.cuda.Event()
            ev.record(cur)
            ps.wait_event(ev)
            be.push_blocks(srcs, dsts, nbytes, ps)
            grid_p.record_stream(ps)    # freed for reuse once its push has run
            del grid_p
        st.mark("rows")
        del grid_s
        cur.wait_stream(ps)
        hdl.barrier(channel=0)          # all slabs' columns have landed
        tgrid = buf[: 2 * spec.n_w * ng * G * spec.n_v]
        strip, partials = be.fft_cols_stack(tgrid, spec, src_rows, g0, ng, 0, spec.n_w)
        st.mark("cols")
    elif transpose == "peer":
        # fused transpose: the row pass stores each destination's columns
        # straight into that rank's column-pass input (symmetric memory,
        # NVLink stores); one device-side barrier orders them before the
        # column pass. Layout of every rank's input: [s][plane][g][row - r0_s].
        elems = spec.n_w * max(dest_pairs) * G * spec.n_v            # complex128 per rank
        buf, hdl = _symm_buffer(elems, dev, group)
        ptrs = [hdl.buffer_ptrs[d] + 16 * spec.n_w * dest_pairs[d] * G * slabs[r][0]
                for d in range(R)]
        hdl.barrier(channel=0)          # every rank has finished reading the previous image
        be.fft_rows_peer(grid_s, spec, vc, dest_pairs, ptrs)
        st.mark("rows")
        del grid_s
        hdl.barrier(channel=0)          # all slabs' columns have landed
        tgrid = buf[: 2 * spec.n_w * ng * G * spec.n_v]
        strip, partials = be.fft_cols_stack(tgrid, spec, src_rows, g0, ng, 0, spec.n_w)
        st.mark("cols")
    else:
        inflight = []
        for k0, k1 in reversed(plane_ranges(spec.n_w, n_ranges)):   # top planes first
            nk = k1 - k0
            grid_p = be.fft_rows(grid_s, spec, vc, dest_pairs, k0, k1)  # [dest][plane][g][row][G]
            in_splits = [nk * ng_d * vc * G * 2 for ng_d in dest_pairs]  # float64 elements per rank
            out_splits = [nk * ng * vc_s * G * 2 for vc_s in src_rows]   # from each source slab
            tgrid = torch.empty(sum(out_splits), dtype=torch.float64, device=dev)
            work = _a2a(tgrid, grid_p, out_splits, in_splits, group, async_op=True)
            inflight.append((k0, k1, work, tgrid, grid_p))
        st.mark("rows")
        del grid_s
        for k0, k1, work, tgrid, grid_p in inflight:
            work.wait()
            strip, partials = be.fft_cols_stack(tgrid, spec, src_rows, g0, ng, k0, k1)
        inflight.clear()
        st.mark("cols")

    # 4. gather to the root ----------------------------------------------------
    upd = torch.tensor([updates], dtype=torch.int64, device=dev)
    dist.all_reduce(upd, group=group)
    maxc = max(dest_pairs) * G
    pad = torch.zeros((spec.n_v, maxc), dtype=torch.float64, device=dev)
    pad[:, : ng * G] = strip
    sp = col_split(spec.n_v)
    ppad = torch.zeros((sp, maxc, 2), dtype=torch.float64, device=dev)
    ppad[:, : ng * G] = partials.reshape(sp, ng * G, 2)
    strips = [torch.empty_like(pad) for _ in range(R)]
    parts = [torch.empty_like(ppad) for _ in range(R)]
    dist.all_gather(strips, pad, group=group)
    dist.all_gather(parts, ppad, group=group)
    st.mark("gather")
    diag = {"grid_updates": int(upd.item()), "records_local": n_local,
            "records_slab": m, "exchange_bytes": int(sum(counts) - counts[r]) * 36,
            "slab_starts": starts}
    if timings is not None:
        timings.update(st.ms())
        if split is not None:
            timings["bucket"], timings["sweep"] = split
    if r != root:
        return None, diag
    pix = torch.empty((spec.n_v, spec.n_u), dtype=torch.float64, device=dev)
    col_parts = []
    for d, (g0_d, ng_d) in enumerate(cols):
        pix[:, g0_d * G:(g0_d + ng_d) * G] = strips[d][:, : ng_d * G]
        col_parts.append(parts[d][:, : ng_d * G])
    return _final(spec, pix, torch.cat(col_parts, dim=1), to_host, diag)


NORM_CHUNK = 64   # k_sum_partials' chunk (csrc/api.cu)


def norm_sum(p) -> tuple:
    """(sum of column 0, sum of column 1) of the norm partials p [n][2] in
    k_sum_partials' association: chunks of NORM_CHUNK consecutive rows summed
    left to right, then the chunk sums left to right (cumsum is left to
    right; padding with +0.0 leaves a sum of squares unchanged)."""
    p = np.asarray(p, dtype=np.float64).reshape(-1, 2)
    nc = -(-len(p) // NORM_CHUNK)
    q = np.zeros((nc * NORM_CHUNK, 2))
    q[: len(p)] = p
    chunks = q.reshape(nc, NORM_CHUNK, 2).cumsum(axis=1)[:, -1, :]
    tot = chunks.cumsum(axis=0)[-1]
    return float(tot[0]), float(tot[1])


def _final(spec, pix, partials, to_host, diag):
    """FinalImage on the root from the device image and the norm partials
    [residue][column][2]."""
    p = partials.reshape(-1, 2).cpu().numpy()
    # residue-major, global column order, the single-GPU association (any R)
    im_sq, re_sq = norm_sum(p)
    if to_host and pix.is_cuda:
        # page-locked destination: the image leaves at DMA speed (a pageable
        # destination costs ~10x). The returned pixels are that buffer itself
        # (the array keeps the tensor alive; torch's caching host allocator
        # recycles it once the caller drops the image): no host-side copy
        stage = torch.empty(pix.shape, dtype=pix.dtype, pin_memory=True)
        stage.copy_(pix)
        pixels = stage.numpy()
    else:
        pixels = pix.numpy() if to_host else pix
    img = FinalImage(spec, pixels, im_sq ** 0.5, re_sq ** 0.5)
    diag.update({"imag_residual_norm": img.imag_residual_norm, "real_norm": img.real_norm})
    return img, diag


_PLANE_CAP: dict = {}


def _image_planes(be, rec, plane, spec, kern, group, root, to_host, timings, st, balance,
                  plane_weight, exchange):
    """w-plane decomposition of image_distributed (see its docstring)."""
    import dataclasses
    R = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = be.device
    n_w, n_u, n_v = spec.n_w, spec.n_u, spec.n_v
    if R > n_w:
        raise ValueError(f"{R} ranks exceed the {n_w} w planes")
    if plane_weight is None:
        # a plane's row + column passes and emission cost about as much as
        # bucketing and gridding n_u n_v / 8 records: measured per rank on cfg3
        # (4 GPUs: grid + transforms 10.8 / 9.8 / 9.6 / 9.9 ms with /8 against
        # 8.5 / 9.8 / 10.3 / 12.1 with /12, 12.5 / 9.8 / 9.2 / 8.2 with /5)
        plane_weight = n_u * n_v / 8.0
    if balance and R > 1:
        hist = be.plane_histogram(plane, spec)
        dist.all_reduce(hist, group=group)
        max_planes = None
        if dev.type == "cuda":
            key = (id(group), dev.index, n_u, n_v, n_w, R)
            if key not in _PLANE_CAP:   # once per mesh: a collective + host sync
                free = torch.tensor([torch.cuda.mem_get_info(dev)[0]], dtype=torch.float64,
                                    device=dev)
                dist.all_reduce(free, op=dist.ReduceOp.MIN, group=group)
                # a plane's strip grid and row-pass output, complex128 each
                _PLANE_CAP[key] = max(1, int(0.6 * float(free.item()) / (2 * n_u * n_v * 16)))
            max_planes = _PLANE_CAP[key]
        starts = balanced_slab_starts(hist.cpu().numpy(), R, plane_weight,
                                      max_rows=min(n_w, max_planes) if max_planes else n_w)
    else:
        starts = [partition_1d(n_w, R, d)[0] for d in range(R)] + [n_w]
    srec, spl, counts = be.route_planes(rec, plane, spec, R, starts)
    n_local = int(rec.shape[0])
    del rec, plane
    st.mark("route")
    rrec, rpl, m = _exchange(be, srec, spl, counts, group, exchange)
    del srec, spl
    st.mark("exchange")

    # 2. grid this rank's planes over the whole mesh ---------------------------
    p0, p1 = starts[r], starts[r + 1]
    nloc = p1 - p0
    spec_l = dataclasses.replace(spec, n_w=nloc)
    grid_s, updates = be.grid_slab(rrec, rpl, spec_l, kern, 0, n_v)
    st.mark("grid")
    split = last_timings(dev)[0][1:3] if st.on else None
    del rrec, rpl

    # 3. row + column passes and the stack of the local planes, top range
    #    first (ranges of at most ~4 GiB of row-pass output) ------------------
    pimg = torch.empty((n_v, n_u, 2), dtype=torch.float64, device=dev)
    n_groups = n_u // G
    n_rng = max(1, -(-nloc * n_u * n_v * 16 // (4 << 30)))
    for l0, l1 in reversed(plane_ranges(nloc, n_rng)):
        grid_p = be.fft_rows(grid_s, spec_l, n_v, [n_groups], l0, l1)
        be.fft_cols_partial(grid_p, spec, p0 + l0, p0 + l1, p0, p1, pimg)
        del grid_p
    del grid_s
    st.mark("fft")

    # 4. sum of the partial stacks on the root, finish there ---------------------
    upd = torch.tensor([updates], dtype=torch.int64, device=dev)
    dist.all_reduce(upd, group=group)
    if R > 1:
        dist.reduce(pimg, dst=dist.get_global_rank(group, root) if group is not None else root,
                    op=dist.ReduceOp.SUM, group=group)
    st.mark("reduce")
    diag = {"grid_updates": int(upd.item()), "records_local": n_local, "records_slab": m,
            "exchange_bytes": int(sum(counts) - counts[r]) * 36, "plane_starts": starts,
            "decomposition": "planes"}
    if timings is not None:
        timings.update(st.ms())
        if split is not None:
            timings["bucket"], timings["sweep"] = split
    if r != root:
        return None, diag
    pix, parts = be.image_finish(pimg, spec)
    return _final(spec, pix, parts, to_host, diag)


def image_distributed_stream(batches, spec, kern, group=None, root: int = 0, **kwargs):
    """``image_distributed`` over a stream of this rank's HOST record batches
    (one image per batch, e.g. successive time chunks), double-buffered: the
    host->device copy of batch i+1 runs on a side stream while batch i is
    imaged. Every batch still makes the full round trip (pinned host records
    in, root image to host); only the copies overlap the device work. Each
    batch is (u, v, w, vis, weight) host arrays (page-locked for DMA speed).
    Yields (FinalImage on ``root`` / None elsewhere, diag)."""
    import numpy as np
    be = kwargs.pop("backend", None) or CudaBackend()
    dev = be.device
    compute = torch.cuda.current_stream(dev)
    s_in = torch.cuda.Stream(dev)
    slots, done = [None, None], [None, None]

    def upload(i, b):
        u, v, w, vis, wt = b
        n = len(u)
        vis = np.asarray(vis, np.complex64).reshape(n, -1)
        wt = np.asarray(wt, np.float32).reshape(n, -1)
        host = [torch.from_numpy(np.ascontiguousarray(x)) for x in
                (np.asarray(u, np.float64), np.asarray(v, np.float64), np.asarray(w, np.float64),
                 vis, wt)]
        slot = i % 2
        if slots[slot] is None or any(d.shape != h.shape for d, h in zip(slots[slot], host)):
            slots[slot] = [torch.empty(h.shape, dtype=h.dtype, device=dev) for h in host]
        with torch.cuda.stream(s_in):
            if done[slot] is not None:
                s_in.wait_event(done[slot])
            for d, h in zip(slots[slot], host):
                d.copy_(h, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
        return ev, host

    it = iter(batches)
    nxt = next(it, None)
    staged = upload(0, nxt) if nxt is not None else None
    i = 0
    while staged is not None:
        ev, _host = staged
        slot = i % 2
        nxt = next(it, None)
        compute.wait_event(ev)
        staged = upload(i + 1, nxt) if nxt is not None else None
        img, diag = image_distributed(*slots[slot], spec, kern, group=group, backend=be, root=root,
                                      to_host=True, **kwargs)
        done[slot] = torch.cuda.Event()
        done[slot].record(compute)
        yield img, diag
        i += 1


def _route_counts_local(rec, spec, half_support: int, R: int):
    """Records of this rank's prepared partition that each v-slab of
    partition_1d(n_v, R) receives under the +-half_support halo predicate
    (comms.py:516-523), counted on the GPU (wsb_route_count): [R] ints."""
    ctx = context(rec.device)
    g = spec.c_struct()
    cnt = (C.c_int64 * R)()
    n = rec.shape[0]
    L.check(L.lib().wsb_route_count(ctx.handle, C.byref(g), int(half_support), R, None,
                                    _ptr(rec) if n else None, n, cnt))
    return [int(x) for x in cnt]


def run_pipeline_distributed(dataset_path, n_u: int, n_v: int, n_w: int, cell_size_lm: float,
                             kernel, group=None, root: int = 0, strategy=None, meter=None,
                             freq_level: str = "default", label: str = "run", out_dir=None,
                             pgm: bool = False, seed=None, **image_kwargs):
    """run_pipeline (pipeline.py:61-191) over a process group, one GPU per
    rank (torchrun). Ingest as the reference's read phase: rank r takes the
    r-th time partition of the RVIS dataset (_partition_for_ranks,
    pipeline.py:47-58 -> partition_time_ordered, visdata.py:344-366:
    contiguous groups of time slices; an unsorted time_index raises its
    ValueError on every rank) and reads only those records of the
    memory-mapped file; image_distributed then exchanges them to their
    v-slabs, grids, transforms and stacks (``image_kwargs`` go to it; the
    default deterministic v-slab decomposition gives run_pipeline's image bit
    for bit). The topology is 1 node x R ranks; the MessageLog / ``ops`` are
    the reference's virtual choreography for it (msglog.py), from exchange
    counts each rank measures on its own records. Returns the PipelineResult
    on ``root`` and None on the other ranks."""
    import time as _time

    from . import msglog
    from .imager import (PipelineResult, RunRecord, GridSpec, _partition_bounds, measure,
                         read_dataset, write_image)

    kern = as_kernel_spec(kernel)
    kind = getattr(strategy, "kind", "direct") if strategy is not None else "direct"
    if kind not in msglog.REDUCE_KINDS:
        raise ValueError(f"reduce kind must be one of {msglog.REDUCE_KINDS}, got {kind!r}")
    R, r = dist.get_world_size(group), dist.get_rank(group)
    if meter is not None and hasattr(meter, "start") and r == root:
        meter.start()
    t_begin = _time.perf_counter()
    times = {}
    # 1. read: this rank's contiguous run of observing time
    t0 = _time.perf_counter()
    header, _ = read_dataset(dataset_path, rows=(0, 0))
    from .imager import _HEADER, _record_dtype
    rec_dt = _record_dtype(header["n_freq"] * header["n_corr"])
    t_idx = (np.asarray(np.memmap(dataset_path, dtype=rec_dt, mode="r", offset=_HEADER.size,
                                  shape=(header["n_records"],))["time_index"])
             if header["n_records"] else np.zeros(0, np.uint32))
    bounds, time_ordered = _partition_bounds(t_idx, R)
    if time_ordered and len(t_idx) > 1 and np.any(np.diff(t_idx.astype(np.int64)) < 0):
        raise ValueError("records must be sorted by time_index")
    lo, hi = bounds[r]
    _, cols = read_dataset(dataset_path, rows=(lo, hi))
    spec = GridSpec(n_u=n_u, n_v=n_v, n_w=n_w, cell_size_lm=cell_size_lm,
                    w_min_native=header["w_min_native"], w_max_native=header["w_max_native"])
    times["read"] = _time.perf_counter() - t0
    # 2-5. exchange, gridding, transforms, w correction, stack
    t0 = _time.perf_counter()
    stage_ms = {}
    img, diag = image_distributed(cols["u"], cols["v"], cols["w"], cols["vis"], cols["weight"],
                                  spec, kern, group=group, root=root, to_host=True,
                                  timings=stage_ms, **image_kwargs)
    wall = _time.perf_counter() - t0
    grid_ms = sum(stage_ms.get(k, 0.0) for k in ("prepare", "route", "exchange", "grid"))
    fft_ms = sum(stage_ms.get(k, 0.0) for k in ("rows", "cols", "fft"))
    fin_ms = sum(stage_ms.get(k, 0.0) for k in ("gather", "reduce"))
    dev_total = max(grid_ms + fft_ms + fin_ms, 1e-9)
    scale = wall / (dev_total / 1e3) if dev_total > 0 else 0.0
    times["gridding"] = grid_ms / 1e3 * scale
    times["reduce"] = 0.0          # the identity after the exchange (pipeline.py:117-122)
    times["fft"] = fft_ms / 1e3 * scale
    times["wcorrect"] = fin_ms / 1e3 * scale
    # the reference's message log for 1 x R ranks: exchange counts per source
    dev = torch.device("cuda", torch.cuda.current_device())
    rec, _pl = prepare_device(cols["u"], cols["v"], cols["w"], cols["vis"], cols["weight"], spec,
                              device=dev)
    mine = torch.tensor(_route_counts_local(rec, spec, kern.half_support, R), dtype=torch.int64,
                        device=dev)
    del rec, _pl
    allc = [torch.empty_like(mine) for _ in range(R)]
    dist.all_gather(allc, mine, group=group)
    if r != root:
        return None
    counts = [c.cpu().tolist() for c in allc]

    class _Topo:   # Topology(n_nodes=1, ranks_per_node=R, threads_per_rank=1)
        n_nodes, ranks_per_node, threads_per_rank, n_ranks = 1, R, 1, R

    topo = _Topo()
    log = msglog.virtual_log(topo, kind, n_u, n_v, n_w, counts) if R > 1 else msglog.MessageLog()
    t0 = _time.perf_counter()
    paths = {}
    if out_dir is not None:
        from pathlib import Path as _Path
        out_dir = _Path(out_dir)
        out_dir.mkdir(parents=True, exist_ok=True)
        prov = {"dataset": str(dataset_path),
                "kernel": {"kind": kern.kind, "half_support": kern.half_support,
                           "shape_param": kern.shape_param},
                "topology": {"n_nodes": 1, "ranks_per_node": R, "threads_per_rank": 1},
                "strategy": {"kind": kind,
                             "deterministic": getattr(strategy, "deterministic", True)},
                "engine": "wsb-b200", "gpus": R, "seed": seed}
        paths = write_image(img, out_dir / "image", prov, pgm=pgm)
        log.to_csv(out_dir / "messages.csv")
        paths["messages"] = out_dir / "messages.csv"
    times["write"] = _time.perf_counter() - t0
    times["total"] = _time.perf_counter() - t_begin
    energy = {}
    if meter is not None:
        energy = measure(meter, {k: v for k, v in times.items() if k != "total"}, freq_level)
    ops = {"records": int(header["n_records"]), "grid_updates": int(diag["grid_updates"]),
           "exchange_bytes": log.total_bytes(phase="exchange"),
           "reduce_bytes": log.total_bytes(phase="reduce"),
           "fft_bytes": log.total_bytes(phase="fft"),
           "reduce_messages": log.count(phase="reduce"), "stack_pixels": n_u * n_v}
    run = RunRecord(label=label, topology=topo, freq_level=freq_level, phase_times=times,
                    energy_joules=energy)
    return PipelineResult(run=run, image=img, log=log, ops=ops, paths=paths)
