"""Host-side mirror of the reference's hot-path interface, over the C-ABI.

The reference (dspar, C++) exposes this path as

  * SparseTensor::from_parts / pack         tensor.hpp:62-72, tensor.cpp:94-197
  * LevelPartitioner universe / nonzero     level_partition.hpp:23-58
  * plan(...) -> Plan                        planner.hpp:42
  * execute(plan, tensors, machine, ...)     sim.hpp:121-122 -> ExecResult{output, Stats}

This module keeps the same names, argument meaning and error classes
(ValidationError -> SpdValidationError, runtime errors -> SpdError) so the
parity tests read like the reference's own tests, while every computation
runs in libspdistal_b200.so on the GPU.  PyTorch is only used for device
memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import SpdError, SpdValidationError, check

DENSE, COMPRESSED = "d", "s"
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


# ---------------------------------------------------------------- formats ---
@dataclass(frozen=True)
class FormatSpec:
    """FormatSpec (tensor.hpp:19-30): level kind per storage position + mode order."""
    kinds: tuple
    mode_order: tuple

    @property
    def order(self):
        return len(self.kinds)


def parse_format(text: str) -> FormatSpec:
    """parse_format (format_lang.cpp:13-53): "ds" = CSR, "ds:1,0" = CSC."""
    body, _, perm = text.strip().partition(":")
    if not body or any(ch not in "ds" for ch in body):
        raise SpdValidationError(f"bad format '{text}'")
    order = tuple(int(x) for x in perm.split(",")) if perm else tuple(range(len(body)))
    if sorted(order) != list(range(len(body))):
        raise SpdValidationError("format: mode order is not a permutation")
    return FormatSpec(tuple(body), order)


def level_grouping(fmt: FormatSpec) -> List[List[int]]:
    """tensor.cpp:30-41: maximal runs of dense modes collapse into one level."""
    groups: List[List[int]] = []
    for k, kind in enumerate(fmt.kinds):
        if kind == DENSE and groups and fmt.kinds[groups[-1][-1]] == DENSE:
            groups[-1].append(k)
        else:
            groups.append([k])
    return groups


# ----------------------------------------------------------- host tensors ---
@dataclass
class Level:
    kind: str                               # "d" or "s"
    dom: tuple = ()                         # dense extents
    pos: Optional[np.ndarray] = None        # compressed: int64 [npos, 2] inclusive (lo, hi)
    crd: Optional[np.ndarray] = None        # compressed: int64 [nnz]

    def rowptr(self) -> np.ndarray:
        """Lossless pairs -> row pointer (tensor.cpp:258-281)."""
        npos = self.pos.shape[0]
        rp = np.empty(npos + 1, dtype=np.int64)
        rp[:npos] = self.pos[:, 0]
        rp[npos] = self.pos[-1, 1] + 1 if npos else 0
        return rp


@dataclass
class SparseTensor:
    """Host copy of the reference's SparseTensor (coordinate-tree encoding)."""
    dims: tuple
    format: FormatSpec
    levels: List[Level]
    vals: np.ndarray

    @staticmethod
    def from_parts(dims, fmt: FormatSpec, levels: List[Level], vals) -> "SparseTensor":
        t = SparseTensor(tuple(int(d) for d in dims), fmt, levels,
                         np.ascontiguousarray(vals, dtype=np.float64))
        return t

    @staticmethod
    def from_rowptrs(dims, fmt: FormatSpec, rowptrs: Sequence, crds: Sequence, vals) -> "SparseTensor":
        """Device-format constructor: one row pointer + crd per compressed level."""
        levels = []
        ci = 0
        for g in level_grouping(fmt):
            if fmt.kinds[g[0]] == DENSE:
                levels.append(Level(DENSE, dom=tuple(dims[fmt.mode_order[k]] for k in g)))
            else:
                rp = np.ascontiguousarray(rowptrs[ci], dtype=np.int64)
                pos = np.stack([rp[:-1], rp[1:] - 1], axis=1)
                levels.append(Level(COMPRESSED, pos=np.ascontiguousarray(pos),
                                    crd=np.ascontiguousarray(crds[ci], dtype=np.int64)))
                ci += 1
        return SparseTensor.from_parts(dims, fmt, levels, vals)

    @staticmethod
    def pack(dims, fmt: FormatSpec, coords, values) -> "SparseTensor":
        """SparseTensor::pack (tensor.cpp:94-182): sort in storage order, sum
        duplicates (in input order), keep explicit zeros.  Host-side test and
        fixture helper (numpy)."""
        dims = tuple(int(d) for d in dims)
        coords = np.asarray(coords, dtype=np.int64).reshape(-1, len(dims))
        values = np.asarray(values, dtype=np.float64).reshape(-1)
        for k in range(len(dims)):
            if coords.size and (coords[:, k].min() < 0 or coords[:, k].max() >= dims[k]):
                raise SpdValidationError("pack: coordinate out of bounds")
        skeys = coords[:, list(fmt.mode_order)] if coords.size else coords
        if skeys.shape[0]:
            order = np.lexsort(skeys.T[::-1])  # stable: duplicates keep input order
            skeys = skeys[order]
            values = values[order]
            diff = np.any(skeys[1:] != skeys[:-1], axis=1)
            starts = np.concatenate([[True], diff])
            uniq = skeys[starts]
            seg = np.cumsum(starts) - 1
            summed = np.zeros(uniq.shape[0])
            np.add.at(summed, seg, values)  # unbuffered, in input order (std::map +=)
        else:
            uniq = skeys.reshape(0, len(dims))
            summed = np.zeros(0)
        levels: List[Level] = []
        entry_pos = np.zeros(uniq.shape[0], dtype=np.int64)
        parent = 1
        base = 0
        for g in level_grouping(fmt):
            if fmt.kinds[g[0]] == DENSE:
                ext = tuple(dims[fmt.mode_order[k]] for k in g)
                local = np.zeros(uniq.shape[0], dtype=np.int64)
                for j, k in enumerate(g):
                    local = local * ext[j] + uniq[:, base + j]
                total = int(np.prod(ext)) if ext else 1
                entry_pos = entry_pos * total + local
                parent *= total
                levels.append(Level(DENSE, dom=ext))
            else:
                col = uniq[:, base]
                key = np.stack([entry_pos, col], axis=1)
                if key.shape[0]:
                    newp = np.concatenate([[True], np.any(key[1:] != key[:-1], axis=1)])
                else:
                    newp = np.zeros(0, dtype=bool)
                crd = col[newp]
                ids = np.cumsum(newp) - 1
                parents = entry_pos[newp]
                counts = np.bincount(parents, minlength=parent) if parents.size else np.zeros(parent, np.int64)
                rp = np.zeros(parent + 1, dtype=np.int64)
                rp[1:] = np.cumsum(counts)
                pos = np.stack([rp[:-1], rp[1:] - 1], axis=1)
                levels.append(Level(COMPRESSED, pos=np.ascontiguousarray(pos), crd=crd.astype(np.int64)))
                entry_pos = ids.astype(np.int64)
                parent = int(crd.shape[0])
            base += len(g)
        vals = np.zeros(parent)
        if uniq.shape[0]:
            vals[entry_pos] = summed
        return SparseTensor.from_parts(dims, fmt, levels, vals)

    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def compressed_rowptrs(self):
        return [lv.rowptr() for lv in self.levels if lv.kind == COMPRESSED]

    def densify(self) -> np.ndarray:
        """densify (oracle.cpp:39-43) for small tensors."""
        out = np.zeros(self.dims)
        for coords, v in self.leaves():
            out[coords] += v
        return out

    def leaves(self):
        """(logical coords, value) per stored path (tensor.cpp:199-206)."""
        fmt = self.format
        paths = [((), 0)]  # (storage coords so far, position)
        for lv in self.levels:
            nxt = []
            if lv.kind == DENSE:
                total = int(np.prod(lv.dom)) if lv.dom else 1
                for sc, p in paths:
                    for s in range(total):
                        pt = np.unravel_index(s, lv.dom) if lv.dom else ()
                        nxt.append((sc + tuple(int(x) for x in pt), p * total + s))
            else:
                for sc, p in paths:
                    lo, hi = lv.pos[p]
                    for q in range(lo, hi + 1):
                        nxt.append((sc + (int(lv.crd[q]),), q))
            paths = nxt
        out = []
        for sc, p in paths:
            logical = [0] * len(self.dims)
            for k, c in enumerate(sc):
                logical[fmt.mode_order[k]] = c
            out.append((tuple(logical), float(self.vals[p])))
        return out


# ---------------------------------------------------------------- device ---
def _i64arr(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Context:
    """One GPU (spd_context).  `stream` defaults to torch's current stream so
    torch-allocated buffers and the backend's kernels are ordered."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, use_torch_stream: bool = True):
        self.device = device
        if stream is None and use_torch_stream:
            import torch
            torch.cuda.set_device(device)
            stream = torch.cuda.current_stream(device).cuda_stream
            if stream == 0:  # torch's default is the legacy NULL stream: order with it
                stream = CUDA_STREAM_LEGACY
        h = C.c_void_p()
        check(N.lib().spd_context_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.rank, self.world = 0, 1

    def synchronize(self):
        check(N.lib().spd_context_synchronize(self.h))

    def init_comm(self, unique_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(unique_id, 128)
        check(N.lib().spd_context_init_comm(self.h, buf, rank, world))
        self.rank, self.world = rank, world

    def capture(self):
        """Context manager: the ops enqueued inside become a Graph
        (spd_capture_begin/end) replayed with Graph.launch()."""
        ctx = self

        class _Capture:
            def __enter__(self_):
                check(N.lib().spd_capture_begin(ctx.h))
                self_.graph = None
                return self_

            def __exit__(self_, exc_type, *rest):
                h = C.c_void_p()
                rc = N.lib().spd_capture_end(ctx.h, C.byref(h))
                if exc_type is None:
                    check(rc)
                    self_.graph = Graph(ctx, h)
                return False

        return _Capture()

    def allgather(self, dev_buf, bytes_per_rank: int):
        """In-place NCCL all-gather of a device buffer (spd_allgather)."""
        check(N.lib().spd_allgather(self.h, _ptr(dev_buf), int(bytes_per_rank)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(N.lib().spd_nccl_unique_id(buf))
        return buf.raw

    def timing(self, enable):
        """spd_context_timing: False/0 off; True/1 CUDA events around every
        leaf kernel; 2 phase markers (read_timing returns the deltas)."""
        check(N.lib().spd_context_timing(self.h, int(enable)))

    def read_timing(self, cap: int = 1 << 16) -> List[float]:
        buf = (C.c_double * cap)()
        n = C.c_int64()
        check(N.lib().spd_context_read_timing(self.h, buf, cap, C.byref(n)))
        return [buf[i] for i in range(min(n.value, cap))]

    def launches(self) -> int:
        n = C.c_int64()
        check(N.lib().spd_context_launches(self.h, C.byref(n)))
        return n.value

    def close(self):
        if self.h:
            check(N.lib().spd_context_destroy(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _format_arrays(dims, fmt: FormatSpec):
    order = len(dims)
    d = (C.c_int64 * order)(*[int(x) for x in dims])
    kinds = (C.c_int * order)(*[N.SPD_DENSE if k == DENSE else N.SPD_COMPRESSED for k in fmt.kinds])
    mo = (C.c_int * order)(*fmt.mode_order)
    return d, kinds, mo


class Graph:
    """A captured op sequence (spd_graph)."""

    def __init__(self, ctx, handle):
        self.ctx, self.h = ctx, handle

    def launch(self):
        check(N.lib().spd_graph_launch(self.h, self.ctx.h))

    def close(self):
        if self.h:
            check(N.lib().spd_graph_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceTensor:
    """A tensor resident in HBM (spd_tensor)."""

    def __init__(self, ctx: Context, handle, dims, fmt: FormatSpec, keep=None):
        self.ctx, self.h, self.dims, self.format = ctx, handle, tuple(dims), fmt
        self._keep = keep

    @staticmethod
    def upload(ctx: Context, t: SparseTensor) -> "DeviceTensor":
        """spd_tensor_upload: the reference's own (lo,hi) pos pairs; validated on the GPU."""
        d, kinds, mo = _format_arrays(t.dims, t.format)
        nl = len(t.levels)
        keep = []
        pos = (N.i64p * nl)()
        crd = (N.i64p * nl)()
        for l, lv in enumerate(t.levels):
            if lv.kind == COMPRESSED:
                p = _i64arr(lv.pos).reshape(-1)
                c = _i64arr(lv.crd)
                keep += [p, c]
                pos[l] = p.ctypes.data_as(N.i64p)
                crd[l] = c.ctypes.data_as(N.i64p)
        vals = np.ascontiguousarray(t.vals, dtype=np.float64)
        h = C.c_void_p()
        check(N.lib().spd_tensor_upload(ctx.h, len(t.dims), d, kinds, mo, pos, crd,
                                        vals.ctypes.data_as(N.dblp), C.byref(h)))
        return DeviceTensor(ctx, h, t.dims, t.format)

    def restage(self, t: SparseTensor, wait: bool = True):
        """spd_tensor_restage: new contents of the same geometry from host
        arrays, into this tensor's device buffers.  The device validates the
        staged pattern and commits it only if it is valid; the verdict is
        reported by the next call on the tensor, or here when `wait` (the
        default) synchronises the context -- a rejected restage leaves the
        tensor's previous contents in place."""
        nl = len(t.levels)
        keep = []
        pos = (N.i64p * nl)()
        crd = (N.i64p * nl)()
        for l, lv in enumerate(t.levels):
            if lv.kind == COMPRESSED:
                p = _i64arr(lv.pos).reshape(-1)
                c = _i64arr(lv.crd)
                keep += [p, c]
                pos[l] = p.ctypes.data_as(N.i64p)
                crd[l] = c.ctypes.data_as(N.i64p)
        vals = np.ascontiguousarray(t.vals, dtype=np.float64)
        check(N.lib().spd_tensor_restage(self.ctx.h, self.h, pos, crd, vals.ctypes.data_as(N.dblp)))
        if wait:
            check(N.lib().spd_context_synchronize(self.ctx.h))
        return self

    @staticmethod
    def pack(ctx: Context, dims, fmt: FormatSpec, coords, values) -> "DeviceTensor":
        """spd_tensor_pack: SparseTensor::pack (tensor.cpp:94-182) on the GPU.
        `coords`: (nentries, order) host array in logical mode order, or a
        sequence of `order` equal-length arrays (numpy, or torch CUDA tensors
        for device-resident input); `values`: nentries."""
        order = len(dims)
        d, kinds, mo = _format_arrays(dims, fmt)
        on_device = False
        if isinstance(coords, (list, tuple)):
            cols = list(coords)
        else:
            arr = np.asarray(coords, dtype=np.int64).reshape(-1, order)
            cols = [np.ascontiguousarray(arr[:, k]) for k in range(order)]
        if cols and hasattr(cols[0], "is_cuda") and cols[0].is_cuda:
            on_device = True
            n = int(cols[0].numel())
            ptrs = (N.i64p * max(order, 1))(*[C.cast(c.data_ptr(), N.i64p) for c in cols])
            vptr = C.cast(values.data_ptr(), N.dblp)
            keep = (cols, values)
        else:
            cols = [np.ascontiguousarray(np.asarray(c, dtype=np.int64)) for c in cols]
            vals = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
            n = int(vals.shape[0])
            ptrs = (N.i64p * max(order, 1))(*[c.ctypes.data_as(N.i64p) for c in cols])
            vptr = vals.ctypes.data_as(N.dblp)
            keep = (cols, vals)
        h = C.c_void_p()
        check(N.lib().spd_tensor_pack(ctx.h, order, d, kinds, mo, n, ptrs, vptr, int(on_device), C.byref(h)))
        del keep
        return DeviceTensor(ctx, h, dims, fmt)

    @staticmethod
    def load(ctx: Context, path, fmt: FormatSpec, dims=None) -> "DeviceTensor":
        """spd_tensor_load: load_tensor (tensor_io.cpp:136-142) -> device pack."""
        order = len(fmt.kinds)
        kinds = (C.c_int * order)(*[N.SPD_DENSE if k == DENSE else N.SPD_COMPRESSED for k in fmt.kinds])
        mo = (C.c_int * order)(*fmt.mode_order)
        d = (C.c_int64 * order)(*[int(x) for x in dims]) if dims is not None else None
        dout = (C.c_int64 * order)()
        h = C.c_void_p()
        check(N.lib().spd_tensor_load(ctx.h, str(path).encode(), order, kinds, mo, d, C.byref(h), dout))
        return DeviceTensor(ctx, h, tuple(dout), fmt)

    @staticmethod
    def place(ctx: Context, whole, dims, fmt: FormatSpec, split: str = "nonzero", root: int = 0):
        """Collective spd_tensor_place: this GPU's piece of a CSR matrix placed
        by its compute partition ("row" or "nonzero"); `whole` on root only.
        Returns (piece, bytes received)."""
        h = C.c_void_p()
        b = C.c_int64()
        check(N.lib().spd_tensor_place(ctx.h, root, whole.h if whole is not None else None,
                                       1 if split == "row" else 2, C.byref(h), C.byref(b)))
        return DeviceTensor(ctx, h, dims, fmt), b.value

    @staticmethod
    def upload_piece(ctx: Context, t: SparseTensor, split: str = "nonzero"):
        """spd_tensor_upload_piece: this GPU's colour of a CSR-like matrix,
        staged from the host arrays of `t` (whole pos, this colour's crd/vals)."""
        d, kinds, mo = _format_arrays(t.dims, t.format)
        nl = len(t.levels)
        keep = []
        pos = (N.i64p * nl)()
        crd = (N.i64p * nl)()
        for l, lv in enumerate(t.levels):
            if lv.kind == COMPRESSED:
                p = _i64arr(lv.pos).reshape(-1)
                c = _i64arr(lv.crd)
                keep += [p, c]
                pos[l] = p.ctypes.data_as(N.i64p)
                crd[l] = c.ctypes.data_as(N.i64p)
        vals = np.ascontiguousarray(t.vals, dtype=np.float64)
        h = C.c_void_p()
        check(N.lib().spd_tensor_upload_piece(ctx.h, len(t.dims), d, kinds, mo, pos, crd,
                                              vals.ctypes.data_as(N.dblp), 1 if split == "row" else 2,
                                              C.byref(h)))
        return DeviceTensor(ctx, h, t.dims, t.format)

    def repartition(self, split: str):
        """Collective spd_tensor_repartition: this piece moved to colour `rank`
        of the compute split ("row" | "nonzero").  Returns (piece, bytes in)."""
        h = C.c_void_p()
        b = C.c_int64()
        check(N.lib().spd_tensor_repartition(self.ctx.h, self.h, 1 if split == "row" else 2, C.byref(h),
                                             C.byref(b)))
        return DeviceTensor(self.ctx, h, self.dims, self.format), b.value

    def piece_span(self):
        lo, hi = C.c_int64(), C.c_int64()
        check(N.lib().spd_tensor_piece_span(self.h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def store(self, path):
        """spd_tensor_store: write_tensor (tensor_io.cpp:145-155)."""
        check(N.lib().spd_tensor_store(self.h, str(path).encode()))

    @staticmethod
    def upload_rowptr(ctx: Context, dims, fmt: FormatSpec, rowptrs, crds, vals,
                      validate=True) -> "DeviceTensor":
        """spd_tensor_upload_rowptr: device-format host arrays (one per compressed level)."""
        d, kinds, mo = _format_arrays(dims, fmt)
        groups = level_grouping(fmt)
        nl = len(groups)
        pos = (N.i64p * nl)()
        crd = (N.i64p * nl)()
        keep = []
        ci = 0
        for l, g in enumerate(groups):
            if fmt.kinds[g[0]] == COMPRESSED:
                rp = _i64arr(rowptrs[ci])
                c = _i64arr(crds[ci])
                keep += [rp, c]
                pos[l] = rp.ctypes.data_as(N.i64p)
                crd[l] = c.ctypes.data_as(N.i64p)
                ci += 1
        v = np.ascontiguousarray(vals, dtype=np.float64)
        h = C.c_void_p()
        check(N.lib().spd_tensor_upload_rowptr(ctx.h, len(dims), d, kinds, mo, pos, crd,
                                               v.ctypes.data_as(N.dblp), int(bool(validate)),
                                               C.byref(h)))
        return DeviceTensor(ctx, h, dims, fmt)

    @staticmethod
    def wrap(ctx: Context, dims, fmt: FormatSpec, rowptr_ptrs, crd_ptrs, vals_ptr, keep=None):
        """spd_tensor_wrap_device: zero-copy over device arrays (e.g. torch tensors)."""
        d, kinds, mo = _format_arrays(dims, fmt)
        groups = level_grouping(fmt)
        nl = len(groups)
        rp = (C.c_void_p * nl)()
        cr = (C.c_void_p * nl)()
        ci = 0
        for l, g in enumerate(groups):
            if fmt.kinds[g[0]] == COMPRESSED:
                rp[l] = rowptr_ptrs[ci]
                cr[l] = crd_ptrs[ci]
                ci += 1
        h = C.c_void_p()
        check(N.lib().spd_tensor_wrap_device(ctx.h, len(dims), d, kinds, mo, rp, cr,
                                             C.c_void_p(vals_ptr), C.byref(h)))
        return DeviceTensor(ctx, h, dims, fmt, keep)

    def num_levels(self) -> int:
        n = C.c_int()
        check(N.lib().spd_tensor_num_levels(self.h, C.byref(n)))
        return n.value

    def level(self, l):
        kind, par, pos = C.c_int(), C.c_int64(), C.c_int64()
        check(N.lib().spd_tensor_level(self.h, l, C.byref(kind), C.byref(par), C.byref(pos)))
        return kind.value, par.value, pos.value

    def nvals(self) -> int:
        n = C.c_int64()
        check(N.lib().spd_tensor_nvals(self.h, C.byref(n)))
        return n.value

    def vals_ptr(self) -> int:
        p = C.c_void_p()
        check(N.lib().spd_tensor_vals_ptr(self.h, C.byref(p)))
        return p.value

    def download(self) -> SparseTensor:
        levels = []
        for l in range(self.num_levels()):
            kind, par, pos = self.level(l)
            if kind == N.SPD_DENSE:
                levels.append(None)
                continue
            pairs = np.empty((par, 2), dtype=np.int64)
            crd = np.empty(pos, dtype=np.int64)
            check(N.lib().spd_tensor_download_level(self.h, l, pairs.ctypes.data_as(N.i64p),
                                                    crd.ctypes.data_as(N.i64p)))
            levels.append(Level(COMPRESSED, pos=pairs, crd=crd))
        groups = level_grouping(self.format)
        for l, g in enumerate(groups):
            if levels[l] is None:
                levels[l] = Level(DENSE, dom=tuple(self.dims[self.format.mode_order[k]] for k in g))
        vals = np.empty(self.nvals(), dtype=np.float64)
        check(N.lib().spd_tensor_download_vals(self.h, vals.ctypes.data_as(N.dblp)))
        return SparseTensor.from_parts(self.dims, self.format, levels, vals)

    def global_span(self):
        """(row_lo, row_hi, pos_base, global_positions) of this piece."""
        v = [C.c_int64() for _ in range(4)]
        check(N.lib().spd_tensor_global_span(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def gather_rows(self, root: int = 0):
        """Collective: the whole tensor on GPU `root` (None elsewhere)."""
        h = C.c_void_p()
        check(N.lib().spd_gather_rows(self.ctx.h, self.h, root, C.byref(h)))
        return DeviceTensor(self.ctx, h, self.dims, self.format) if h.value else None

    def close(self):
        if self.h:
            check(N.lib().spd_tensor_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ partitions ---
@dataclass
class Colour:
    """One colour of a distributed loop (spd_color), inclusive ranges."""
    color: tuple
    q: tuple
    par: tuple
    top: tuple


def _colours(arr) -> List[Colour]:
    return [Colour((c.color.lo, c.color.hi), (c.q.lo, c.q.hi), (c.par.lo, c.par.hi),
                   (c.top.lo, c.top.hi)) for c in arr]


def partition_universe(ctx: Context, t: DeviceTensor, pieces: int, host=True):
    """host=False keeps the colours on the device (no synchronisation)."""
    arr = (N.spd_color * pieces)() if host else None
    check(N.lib().spd_partition_universe(ctx.h, t.h, pieces, arr))
    return _colours(arr) if host else None


def partition_nonzero(ctx: Context, t: DeviceTensor, level: int, pieces: int, host=True):
    arr = (N.spd_color * pieces)() if host else None
    check(N.lib().spd_partition_nonzero(ctx.h, t.h, level, pieces, arr))
    return _colours(arr) if host else None


# ------------------------------------------------- general deppart (8f.4) ---
class DevicePartition:
    """A materialised partition in HBM: (off[P+1], idx) int64 device tensors,
    colour c = idx[off[c]:off[c+1]] sorted and unique (Partition,
    partition.hpp:16-46)."""

    def __init__(self, off, idx, disjoint=None):
        self.off, self.idx, self.disjoint = off, idx, disjoint

    @property
    def num_colors(self):
        return self.off.numel() - 1

    @staticmethod
    def from_subsets(subsets, device="cuda"):
        import torch

        off = np.zeros(len(subsets) + 1, np.int64)
        for c, sub in enumerate(subsets):
            off[c + 1] = off[c] + len(sub)
        idx = (np.concatenate([np.asarray(x, np.int64) for x in subsets]) if len(subsets)
               else np.zeros(0, np.int64))
        return DevicePartition(torch.from_numpy(off).to(device), torch.from_numpy(idx).to(device))

    def subsets(self):
        off = self.off.cpu().numpy()
        idx = self.idx.cpu().numpy()
        return [idx[off[c]:off[c + 1]].copy() for c in range(len(off) - 1)]


def _deppart_call(fn, ctx, pieces, args):
    """Two-phase call: size, then fill."""
    import torch

    dev = torch.device("cuda", ctx.device)
    out_off = torch.empty(pieces + 1, dtype=torch.int64, device=dev)
    total = C.c_int64()
    disj = C.c_int()
    check(fn(ctx.h, *args, C.c_void_p(out_off.data_ptr()), None, 0, C.byref(total), C.byref(disj)))
    out_idx = torch.empty(max(total.value, 1), dtype=torch.int64, device=dev)
    check(fn(ctx.h, *args, C.c_void_p(out_off.data_ptr()), C.c_void_p(out_idx.data_ptr()), total.value,
             C.byref(total), C.byref(disj)))
    return DevicePartition(out_off, out_idx[:total.value], bool(disj.value))


def _ranges_dev(ranges, device):
    import torch

    if isinstance(ranges, torch.Tensor):
        r = ranges.to(device=device, dtype=torch.int64).contiguous().reshape(-1, 2)
    else:
        r = torch.from_numpy(np.ascontiguousarray(np.asarray(ranges, np.int64).reshape(-1, 2))).to(device)
    return r


def image(ctx: Context, ranges, part: DevicePartition, dest_extent: int) -> DevicePartition:
    """spd_deppart_image: image(source, src_part, dest) (deppart.cpp:15-31)."""
    r = _ranges_dev(ranges, part.off.device)
    return _deppart_call(N.lib().spd_deppart_image, ctx, part.num_colors,
                         (C.c_void_p(r.data_ptr()), r.shape[0], dest_extent, part.num_colors,
                          C.c_void_p(part.off.data_ptr()), C.c_void_p(part.idx.data_ptr())))


def preimage(ctx: Context, ranges, part: DevicePartition, dest_extent: int) -> DevicePartition:
    """spd_deppart_preimage: preimage(source, dest_part, dest) (deppart.cpp:33-53)."""
    r = _ranges_dev(ranges, part.off.device)
    return _deppart_call(N.lib().spd_deppart_preimage, ctx, part.num_colors,
                         (C.c_void_p(r.data_ptr()), r.shape[0], dest_extent, part.num_colors,
                          C.c_void_p(part.off.data_ptr()), C.c_void_p(part.idx.data_ptr())))


def partition_by_bounds(ctx: Context, extents, coloring: dict) -> DevicePartition:
    """spd_deppart_by_bounds: partition_by_bounds(space, coloring)
    (deppart.cpp:55-91); coloring = {colour: [(lo, hi) per dimension]};
    colours absent from the map are empty."""
    ext = np.asarray(extents, np.int64)
    R = len(ext)
    P = (max(coloring) + 1) if coloring else 0
    if any(c < 0 for c in coloring):
        raise N.SpdValidationError("partition_by_bounds: negative color")
    b = np.tile(np.array([1, 0], np.int64), P * R).reshape(P, R, 2)  # empty boxes
    for c, box in coloring.items():
        if len(box) != R:
            raise N.SpdValidationError("partition_by_bounds: bounds rank mismatch")
        b[c] = np.asarray(box, np.int64)
    b = np.ascontiguousarray(b.reshape(-1))
    return _deppart_call(N.lib().spd_deppart_by_bounds, ctx, P,
                         (R, ext.ctypes.data_as(N.i64p), P, b.ctypes.data_as(N.i64p)))


REGION = {"dom": 0, "pos": 1, "crd": 2, "vals": 3}


def materialize(ctx: Context, t: DeviceTensor, level: int, region: str, color: int) -> np.ndarray:
    """K2m: one colour's explicit index set of a bundle region."""
    count = C.c_int64()
    check(N.lib().spd_partition_materialize(ctx.h, t.h, level, REGION[region], color, None, 0,
                                            C.byref(count)))
    out = np.empty(count.value, dtype=np.int64)
    check(N.lib().spd_partition_materialize(ctx.h, t.h, level, REGION[region], color,
                                            out.ctypes.data_as(N.i64p), count.value,
                                            C.byref(count)))
    return out


# ------------------------------------------------------------------ stats ---
@dataclass
class Stats:
    """Stats (sim.hpp:25-36)."""
    workers: int
    work: List[int]
    imbalance: float
    combines: int
    kernel_ms: float = 0.0
    launches: int = 0


def _stats(ctx: Context, st: N.spd_stats, pieces: int) -> Stats:
    work = (C.c_int64 * pieces)()
    check(N.lib().spd_last_work(ctx.h, work, pieces))
    return Stats(st.workers, list(work), st.imbalance, st.combines, st.kernel_ms, st.launches)


def _ptr(x) -> C.c_void_p:
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return C.c_void_p(int(x))


# --------------------------------------------------------------- leaf ops ---
def spmv(ctx, B: DeviceTensor, c, a, first=0, count=None, pieces=None, stats=True):
    st = N.spd_stats()
    count = pieces - first if count is None else count
    check(N.lib().spd_spmv(ctx.h, B.h, _ptr(c), _ptr(a), first, count, C.byref(st) if stats else None))
    return _stats(ctx, st, pieces) if stats else None


def last_owned(ctx, first, count):
    """spd_last_owned: (lo, hi) output rows (fibres for SpTTV) the colours
    [first, first + count) stored in the last row-reducing op."""
    lo, hi = C.c_int64(), C.c_int64()
    check(N.lib().spd_last_owned(ctx.h, first, count, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def split_colour_blocks(costs, world):
    """spd_split_colour_blocks (host only): bounds[0..world] of contiguous
    colour blocks of near-equal total cost."""
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    b = np.zeros(world + 1, dtype=np.int64)
    check(N.lib().spd_split_colour_blocks(costs.ctypes.data_as(N.dblp), len(costs), world,
                                          b.ctypes.data_as(N.i64p)))
    return b


def set_colour_blocks(ctx, pieces, bounds):
    """spd_context_set_colour_blocks; bounds None restores the even blocks."""
    if bounds is None:
        check(N.lib().spd_context_set_colour_blocks(ctx.h, pieces, None))
        return
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    check(N.lib().spd_context_set_colour_blocks(ctx.h, pieces, b.ctypes.data_as(N.i64p)))


def colour_blocks(ctx, pieces):
    """spd_context_colour_blocks: the bounds[0..world] a `pieces`-colour
    partition runs with; rank r runs [bounds[r], bounds[r + 1])."""
    b = np.zeros(ctx.world + 1, dtype=np.int64)
    check(N.lib().spd_context_colour_blocks(ctx.h, pieces, b.ctypes.data_as(N.i64p)))
    return b


def colour_costs(ctx, t: DeviceTensor, pieces):
    """spd_colour_costs: per colour of the current partition of the ds matrix
    t, (positions, output rows W_c, non-empty rows of W_c)."""
    out = [np.zeros(pieces, dtype=np.int64) for _ in range(3)]
    check(N.lib().spd_colour_costs(ctx.h, t.h, *(o.ctypes.data_as(N.i64p) for o in out)))
    return tuple(out)


def balance_colour_blocks(ctx, t: DeviceTensor, pieces, row_cost, empty_row_cost):
    """Cost-balanced colour blocks for an over-decomposed plan (pieces >
    world): cost_c = positions + row_cost * non-empty rows + empty_row_cost *
    empty rows of W_c, split into contiguous blocks of near-equal cost and
    installed on the context.  Deterministic, so every rank computes the same
    blocks from the same partition.  Returns the bounds."""
    pos, rows, ne = colour_costs(ctx, t, pieces)
    cost = pos + row_cost * ne + empty_row_cost * (rows - ne)
    b = split_colour_blocks(cost, ctx.world)
    set_colour_blocks(ctx, pieces, b)
    return b


def spmm(ctx, B: DeviceTensor, Cd, n_cols, A, first=0, count=None, pieces=None, stats=True):
    st = N.spd_stats()
    count = pieces - first if count is None else count
    check(N.lib().spd_spmm(ctx.h, B.h, _ptr(Cd), n_cols, _ptr(A), first, count,
                           C.byref(st) if stats else None))
    return _stats(ctx, st, pieces) if stats else None


SPLITS = {"row": 1, "nonzero": 2, "replicated": 3}


def ledger_bytes(ctx, B: DeviceTensor, need: str, held: str, pieces: int):
    """spd_ledger_bytes: per-worker bytes_by_tensor of B (transfer_bytes,
    sim.cpp:134-147) for compute split `need` ("row" | "nonzero") against
    placement `held` ("row" | "nonzero" | "replicated")."""
    out = (C.c_int64 * pieces)()
    check(N.lib().spd_ledger_bytes(ctx.h, B.h, SPLITS[need], SPLITS[held], pieces, out))
    return list(out)


def divide_bounds(n: int, pieces: int):
    """divide_bounds (planner.cpp:10-20): block = n / pieces (truncating);
    colour c < pieces-1 -> [c*block, c*block+block-1], the last -> [.., n-1]."""
    block = n // pieces
    return [(c * block, c * block + block - 1) if c < pieces - 1 else ((pieces - 1) * block, n - 1)
            for c in range(pieces)]


def spmm_batched(ctx, B: DeviceTensor, Cd, n_cols, A, grid, rank=None, stats=True):
    """SpDISTAL-Batched SpMM (2-D machine grid x=Px, y=Py,
    test_planner.cpp:193-225): rows of B/A divided over x (a universe split
    of B, spd_partition_universe with Px pieces), the columns j of C/A
    divided over y (divide_bounds on N).  Worker (x, y) computes the block
    A[rows_x, slab_y] = B[rows_x, :] * C[:, slab_y] from its column slab of C
    only, so C is partitioned instead of replicated; no combine.

    Single GPU (rank None): every tuple, in worker order x*Py + y
    (MachineGrid::worker_id, machine.cpp:88-92).  With a communicator of
    Px*Py GPUs: this rank's tuple; Cd is then this rank's slab (K x w,
    contiguous) and A its n x w block buffer (rows outside rows_x untouched).
    Stats: work[x*Py+y] = nnz(rows_x) * w_y, combines 0."""
    import torch

    Px, Py = grid
    n = B.dims[0]
    slabs = divide_bounds(n_cols, Py)
    cols = partition_universe(ctx, B, Px)
    if rank is not None:
        x, y = divmod(rank, Py)
        lo, hi = slabs[y]
        w = max(hi - lo + 1, 0)
        if w > 0:
            spmm(ctx, B, Cd, w, A, first=x, count=1, pieces=Px, stats=False)
        tuples = [(x, y)]
    else:
        K = Cd.numel() // n_cols if n_cols else 0
        Cv = Cd.view(K, n_cols)
        Av = A.view(n, n_cols)
        for y, (lo, hi) in enumerate(slabs):
            w = hi - lo + 1
            if w <= 0:
                continue
            Cy = Cv[:, lo:hi + 1].contiguous()
            Ay = torch.empty(n * w, dtype=torch.float64, device=A.device)
            spmm(ctx, B, Cy, w, Ay, pieces=Px, stats=False)
            Av[:, lo:hi + 1] = Ay.view(n, w)
        tuples = [(x, y) for x in range(Px) for y in range(Py)]
    if not stats:
        return None
    nnz_x = [c.q[1] - c.q[0] + 1 if c.q[0] <= c.q[1] else 0 for c in cols]  # crd image of rows_x
    work = [0] * (Px * Py)
    for x in range(Px):
        for y, (lo, hi) in enumerate(slabs):
            work[x * Py + y] = nnz_x[x] * max(hi - lo + 1, 0)
    total, mx = sum(work), max(work) if work else 0
    imb = 1.0 if total == 0 else mx * len(work) / total
    return Stats(Px * Py, work, imb, 0)


def spmttkrp_batched(ctx, B: DeviceTensor, Cd, Dd, R, A, grid, rank=None, stats=True):
    """SpMTTKRP A(i,l) = B(i,j,k) * C(j,l) * D(k,l) on a 2-D machine grid, the
    batched form of spmm_batched: rows i of B/A divided over x (a universe
    split of B's top level), the rank columns l of C, D and A divided over y
    (divide_bounds on R).  Worker (x, y) computes A[rows_x, slab_y] from the
    column slabs C[:, slab_y] and D[:, slab_y] only; no combine.  Same
    schedule shape as test_planner.cpp:193-225 (divide both output modes,
    distribute io over x and lo over y); the reference plans and executes it
    through the same code (planner.cpp:142-359, sim.cpp:816-1010).

    rank None: every tuple on this GPU, in worker order x*Py + y.  With a
    communicator of Px*Py GPUs: this rank's tuple; Cd / Dd are then this
    rank's slabs (J x w and K x w, contiguous) and A its I x w block buffer.
    Stats: work[x*Py+y] = nnz(rows_x) * w_y (each leaf entry times the slab
    width, the reference's per-coordinate count), combines 0."""
    import torch

    Px, Py = grid
    n = B.dims[0]
    slabs = divide_bounds(R, Py)
    cols = partition_universe(ctx, B, Px)
    if rank is not None:
        x, y = divmod(rank, Py)
        lo, hi = slabs[y]
        w = max(hi - lo + 1, 0)
        if w > 0:
            spmttkrp(ctx, B, Cd, Dd, w, A, first=x, count=1, pieces=Px, stats=False)
    else:
        J = Cd.numel() // R if R else 0
        Kd = Dd.numel() // R if R else 0
        Cv, Dv, Av = Cd.view(J, R), Dd.view(Kd, R), A.view(n, R)
        for y, (lo, hi) in enumerate(slabs):
            w = hi - lo + 1
            if w <= 0:
                continue
            Ay = torch.empty(n * w, dtype=torch.float64, device=A.device)
            spmttkrp(ctx, B, Cv[:, lo:hi + 1].contiguous(), Dv[:, lo:hi + 1].contiguous(), w, Ay,
                     pieces=Px, stats=False)
            Av[:, lo:hi + 1] = Ay.view(n, w)
    if not stats:
        return None
    nnz_x = [c.q[1] - c.q[0] + 1 if c.q[0] <= c.q[1] else 0 for c in cols]
    work = [0] * (Px * Py)
    for x in range(Px):
        for y, (lo, hi) in enumerate(slabs):
            work[x * Py + y] = nnz_x[x] * max(hi - lo + 1, 0)
    total, mx = sum(work), max(work) if work else 0
    imb = 1.0 if total == 0 else mx * len(work) / total
    return Stats(Px * Py, work, imb, 0)


def sddmm(ctx, B: DeviceTensor, Cd, Dd, K, dk, dj, Avals, first=0, count=None, pieces=None, stats=True):
    st = N.spd_stats()
    count = pieces - first if count is None else count
    check(N.lib().spd_sddmm(ctx.h, B.h, _ptr(Cd), _ptr(Dd), K, dk, dj, _ptr(Avals), first, count,
                            C.byref(st) if stats else None))
    return _stats(ctx, st, pieces) if stats else None


def spttv(ctx, B: DeviceTensor, c, Avals, first=0, count=None, pieces=None, stats=True):
    st = N.spd_stats()
    count = pieces - first if count is None else count
    check(N.lib().spd_spttv(ctx.h, B.h, _ptr(c), _ptr(Avals), first, count,
                            C.byref(st) if stats else None))
    return _stats(ctx, st, pieces) if stats else None


def spmttkrp(ctx, B: DeviceTensor, Cd, Dd, R, A, first=0, count=None, pieces=None, stats=True):
    st = N.spd_stats()
    count = pieces - first if count is None else count
    check(N.lib().spd_spmttkrp(ctx.h, B.h, _ptr(Cd), _ptr(Dd), R, _ptr(A), first, count,
                               C.byref(st) if stats else None))
    return _stats(ctx, st, pieces) if stats else None


def spadd3(ctx, B: DeviceTensor, Cm: DeviceTensor, D: DeviceTensor, first=0, count=None,
           pieces=None, stats=True):
    st = N.spd_stats()
    count = pieces - first if count is None else count
    h = C.c_void_p()
    check(N.lib().spd_spadd3(ctx.h, B.h, Cm.h, D.h, C.byref(h), first, count,
                             C.byref(st) if stats else None))
    A = DeviceTensor(ctx, h, B.dims, B.format)
    return A, (_stats(ctx, st, pieces) if stats else None)
