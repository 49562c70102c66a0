"""NumPy stand-in for distributed.CudaBackend, built on the oracle, so the
multi-rank host logic (exchange splits, transposes, gathers) can be tested
with gloo on CPU. Test infrastructure only: it follows the same stage
contracts as include/wsb.h (P layout, transposed slab layout, per-column
norm partials)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import wstack_oracle as O
from paper_2504_00959_b200 import _lib as L

G = 1


class NumpyBackend:
    device = torch.device("cpu")

    def prepare(self, u, v, w, vis, weight, spec):
        p = O.prepare(np.asarray(u), np.asarray(v), np.asarray(w), np.zeros(len(u), np.uint32),
                      np.asarray(vis), np.asarray(weight), spec.n_u, spec.n_v, spec.n_w)
        rec = np.stack([p["gu"], p["gv"], p["value"].real, p["value"].imag], axis=1)
        return torch.from_numpy(rec), torch.from_numpy(p["plane"].astype(np.int32))

    def row_histogram(self, rec, spec):
        rows = np.clip(np.floor(rec.numpy()[:, 1]).astype(np.int64), 0, spec.n_v - 1)
        return torch.from_numpy(np.bincount(rows, minlength=spec.n_v).astype(np.int64))

    def route(self, rec, plane, spec, S, R, starts=None):
        r, pl = rec.numpy(), plane.numpy()
        outs, outp, counts = [], [], []
        bounds = (O.slabs(spec.n_v, R) if starts is None
                  else [(starts[d], starts[d + 1] - starts[d]) for d in range(R)])
        for v0, vc in bounds:
            m = O.halo_mask(r[:, 1], S, v0, vc)
            outs.append(r[m])
            outp.append(pl[m])
            counts.append(int(m.sum()))
        return (torch.from_numpy(np.concatenate(outs)), torch.from_numpy(np.concatenate(outp)),
                counts)

    def grid_slab(self, rec, plane, spec, kern, v0, vc):
        r = rec.numpy()
        batch = {"gu": r[:, 0], "gv": r[:, 1], "value": r[:, 2] + 1j * r[:, 3],
                 "plane": plane.numpy().astype(np.uint32), "v_start": v0, "v_count": vc}
        kind = O.KIND_GAUSSIAN if kern.kind == "gaussian" else O.KIND_KAISER_BESSEL
        grid, upd = O.grid_slab(batch, spec.n_u, spec.n_w, kind, kern.half_support, kern.shape_param)
        grid = grid * O.checker_sign(spec.n_u, v0, vc)[None]
        # (plane, row, col) -> strip layout (plane, col/SW, row, col%SW)
        sw = L.STRIP
        ns = (spec.n_u + sw - 1) // sw
        pad = np.zeros((spec.n_w, vc, ns * sw), np.complex128)
        pad[:, :, : spec.n_u] = grid
        s = np.ascontiguousarray(pad.reshape(spec.n_w, vc, ns, sw).transpose(0, 2, 1, 3))
        # each strip row: its sw real parts, then its sw imaginary parts
        split = np.stack([s.real, s.imag], axis=3)             # (n_w, ns, vc, 2, sw)
        return torch.from_numpy(np.ascontiguousarray(split)), upd

    def fft_rows(self, grid_s, spec, vc, dest_pairs, plane_lo=0, plane_hi=None):
        plane_hi = spec.n_w if plane_hi is None else plane_hi
        nk = plane_hi - plane_lo
        sw = L.STRIP
        ns = (spec.n_u + sw - 1) // sw
        g = grid_s.numpy().reshape(spec.n_w, ns, vc, 2, sw)
        a = (g[:, :, :, 0, :] + 1j * g[:, :, :, 1, :])[plane_lo:plane_hi]
        nat = a.transpose(0, 2, 1, 3).reshape(nk, vc, ns * sw)[:, :, : spec.n_u]
        f = np.fft.ifft(nat, axis=-1) * spec.n_u               # unnormalised inverse
        # -> P layout (plane, col/G, row, col%G), then destination major
        p = f.reshape(nk, vc, spec.n_u // G, G).transpose(0, 2, 1, 3)
        out, g0 = [], 0
        for ng in dest_pairs:
            out.append(np.ascontiguousarray(p[:, g0:g0 + ng]).ravel())
            g0 += ng
        return torch.from_numpy(np.concatenate(out).view(np.float64))

    def fft_cols_stack(self, tgrid, spec, src_rows, g0, ng, plane_lo=0, plane_hi=None):
        """Plane ranges come in descending order (the CUDA backend's
        contract); their planes are kept until the range starting at 0."""
        plane_hi = spec.n_w if plane_hi is None else plane_hi
        nk = plane_hi - plane_lo
        t = tgrid.numpy().view(np.complex128)
        ncols = ng * G
        full = np.empty((nk, spec.n_v, ncols), np.complex128)
        off, r0 = 0, 0
        for rows in src_rows:                    # [s][plane][pair][row][G]
            n = nk * ng * rows * G
            blk = t[off:off + n].reshape(nk, ng, rows, G)
            full[:, r0:r0 + rows] = blk.transpose(0, 2, 1, 3).reshape(nk, rows, ncols)
            off += n
            r0 += rows
        planes = np.fft.ifft(full, axis=1) * spec.n_v / (spec.n_u * spec.n_v)
        c0 = g0 * G
        cols = np.arange(c0, c0 + ncols, dtype=np.float64) - spec.n_u // 2
        rowsv = np.arange(spec.n_v, dtype=np.float64) - spec.n_v // 2
        l = np.broadcast_to(cols * spec.cell_size_lm, (spec.n_v, ncols))
        m = np.broadcast_to((rowsv * spec.cell_size_lm)[:, None], (spec.n_v, ncols))
        n = np.sqrt(1.0 - l * l - m * m)
        # ranges arrive top-down; the oracle's order (k ascending) at the end
        if plane_hi == spec.n_w:
            self._planes = {}
        for k in range(plane_lo, plane_hi):
            wk = O.plane_w_native(k, spec.n_w, spec.w_min_native, spec.w_max_native)
            pk = planes[k - plane_lo]
            self._planes[k] = pk if wk == 0.0 else pk * np.exp(2j * np.pi * wk * (n - 1.0))
        if plane_lo > 0:
            return None, None
        acc = np.zeros((spec.n_v, ncols), np.complex128)
        for k in range(spec.n_w):
            acc = acc + self._planes[k]
        acc = acc / spec.n_w * n
        strip = np.ascontiguousarray(acc.real)
        sp = spec.n_v // 4096 if spec.n_v > 4096 else 1      # residue classes of the rows
        partials = np.stack([np.stack([(acc.imag[e::sp] ** 2).sum(axis=0),
                                       (acc.real[e::sp] ** 2).sum(axis=0)], axis=1)
                             for e in range(sp)])
        return torch.from_numpy(strip), torch.from_numpy(np.ascontiguousarray(partials))

    # ---- w-plane decomposition (distributed._image_planes) -------------------
    def plane_histogram(self, plane, spec):
        return torch.from_numpy(np.bincount(plane.numpy().astype(np.int64), minlength=spec.n_w))

    def route_planes(self, rec, plane, spec, R, starts):
        r, pl = rec.numpy(), plane.numpy()
        outs, outp, counts = [], [], []
        for d in range(R):
            m = (pl >= starts[d]) & (pl < starts[d + 1])
            outs.append(r[m])
            outp.append((pl[m] - starts[d]).astype(pl.dtype))
            counts.append(int(m.sum()))
        return (torch.from_numpy(np.concatenate(outs)), torch.from_numpy(np.concatenate(outp)),
                counts)

    def fft_cols_partial(self, tgrid, spec, plane_lo, plane_hi, rank_lo, rank_hi, pimg):
        """Unscaled stack sum_k P_k exp(2 pi i w_k (n-1)) of the rank's planes
        (ranges in descending order), written at the range starting at rank_lo."""
        nk = plane_hi - plane_lo
        ng = spec.n_u // G
        t = tgrid.numpy().view(np.complex128)[: nk * ng * spec.n_v * G]
        full = t.reshape(nk, ng, spec.n_v, G).transpose(0, 2, 1, 3).reshape(nk, spec.n_v, spec.n_u)
        planes = np.fft.ifft(full, axis=1) * spec.n_v            # unnormalised inverse
        if plane_hi == rank_hi:
            self._pacc = np.zeros((spec.n_v, spec.n_u), np.complex128)
        n = self._n(spec)
        for k in range(plane_lo, plane_hi):
            wk = O.plane_w_native(k, spec.n_w, spec.w_min_native, spec.w_max_native)
            pk = planes[k - plane_lo]
            self._pacc = self._pacc + (pk if wk == 0.0 else pk * np.exp(2j * np.pi * wk * (n - 1.0)))
        if plane_lo == rank_lo:
            pimg.numpy().view(np.complex128).reshape(spec.n_v, spec.n_u)[:] = self._pacc

    def image_finish(self, pimg, spec):
        from paper_2504_00959_b200.distributed import finish_split
        acc = pimg.numpy().view(np.complex128).reshape(spec.n_v, spec.n_u)
        acc = acc / (spec.n_u * spec.n_v) / spec.n_w * self._n(spec)
        rs = finish_split(spec.n_v)
        blk = spec.n_v // rs
        partials = np.stack([np.stack([(acc.imag[e * blk:(e + 1) * blk] ** 2).sum(axis=0),
                                       (acc.real[e * blk:(e + 1) * blk] ** 2).sum(axis=0)], axis=1)
                             for e in range(rs)])
        return (torch.from_numpy(np.ascontiguousarray(acc.real)),
                torch.from_numpy(np.ascontiguousarray(partials)))

    @staticmethod
    def _n(spec):
        cols = np.arange(spec.n_u, dtype=np.float64) - spec.n_u // 2
        rowsv = np.arange(spec.n_v, dtype=np.float64) - spec.n_v // 2
        l = np.broadcast_to(cols * spec.cell_size_lm, (spec.n_v, spec.n_u))
        m = np.broadcast_to((rowsv * spec.cell_size_lm)[:, None], (spec.n_v, spec.n_u))
        return np.sqrt(1.0 - l * l - m * m)
