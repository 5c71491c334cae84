"""TEST INFRASTRUCTURE: ctypes bindings of the checkers under oracle/.

  * liboracle.so       -- the C restatement (oracle/restate.c)
  * _ref/libdspar_ref.so -- the reference itself (patched, oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs import this module.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")
PORT_LIB = os.path.join(ORACLE, "liboracle.so")
REF_LIB = os.path.join(ORACLE, "_ref", "libdspar_ref.so")
REF_TESTS = os.path.join(ORACLE, "_ref", "dspar_ref_tests")
GPU_LIB = os.path.join(ORACLE, "_ref", "libdspar_gpu.so")  # reference + ExecMode::Gpu adapter

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)


class or_color(C.Structure):
    _fields_ = [(n, i64) for n in
                ("color_lo", "color_hi", "q_lo", "q_hi", "par_lo", "par_hi", "top_lo", "top_hi")]


def colours_to_tuples(arr):
    return [dict(color=(c.color_lo, c.color_hi), q=(c.q_lo, c.q_hi), par=(c.par_lo, c.par_hi),
                 top=(c.top_lo, c.top_hi)) for c in arr]


_port = None
_refs = {}


def ensure_built(ref=True):
    need = [PORT_LIB] + ([REF_LIB] if ref else [])
    if all(os.path.exists(p) for p in need):
        return
    if not os.path.exists("/root/reference/proj"):
        if ref and not os.path.exists(REF_LIB):
            raise FileNotFoundError("oracle/_ref not prebuilt and /root/reference absent")
    targets = ["port"] + (["ref", "ref-tests"] if ref and os.path.exists("/root/reference/proj") else [])
    subprocess.run(["make", "-C", ORACLE, "-j8"] + targets, check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


def port():
    global _port
    if _port is None:
        ensure_built(ref=False)
        L = C.CDLL(PORT_LIB)
        L.or_divide_bounds.argtypes = [i64, i64, i64p, i64p]
        L.or_pos_to_rowptr.argtypes = [i64p, i64, i64, i64p]
        L.or_pos_to_rowptr.restype = C.c_int
        L.or_owner.argtypes = [i64p, i64, i64]
        L.or_owner.restype = i64
        L.or_partition_universe.argtypes = [C.POINTER(i64p), i64p, C.c_int, i64, i64, C.POINTER(or_color)]
        L.or_partition_nonzero.argtypes = [C.POINTER(i64p), i64p, C.c_int, i64, i64, C.POINTER(or_color)]
        L.or_preimage_range.argtypes = [i64p, i64, i64, i64, i64p, i64]
        L.or_preimage_range.restype = i64
        L.or_spmv.argtypes = [i64, i64p, i64p, dblp, dblp, i64, C.POINTER(or_color), dblp, i64p, C.c_int]
        L.or_spmv.restype = i64
        L.or_spmm.argtypes = [i64, i64p, i64p, dblp, dblp, i64, i64, C.POINTER(or_color), dblp, i64p, C.c_int]
        L.or_spmm.restype = i64
        L.or_sddmm.argtypes = [i64, i64p, i64p, dblp, dblp, dblp, i64, i64, i64, i64,
                               C.POINTER(or_color), dblp, i64p, C.c_int]
        L.or_sddmm.restype = i64
        L.or_spttv.argtypes = [i64, i64p, i64p, i64p, i64p, dblp, dblp, i64, C.POINTER(or_color),
                               dblp, i64p, C.c_int]
        L.or_spttv.restype = i64
        L.or_spmttkrp.argtypes = [i64, i64p, i64p, i64p, i64p, dblp, dblp, dblp, i64, i64,
                                  C.POINTER(or_color), dblp, i64p, C.c_int]
        L.or_spmttkrp.restype = i64
        L.or_spadd3_count.argtypes = [i64, C.POINTER(i64p), C.POINTER(i64p), i64p, C.c_int]
        L.or_spadd3_count.restype = i64
        L.or_spadd3_fill.argtypes = [i64, C.POINTER(i64p), C.POINTER(i64p), C.POINTER(dblp), i64p,
                                     i64p, dblp, C.c_int]
        L.or_imbalance.argtypes = [i64p, i64]
        L.or_imbalance.restype = C.c_double
        _port = L
    return _port


def _p(a, t=i64p):
    return a.ctypes.data_as(t)


def I64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def F64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- restatement wrappers ---------------------------------------------------
def divide_bounds(n, pieces):
    lo = np.zeros(pieces, np.int64)
    hi = np.zeros(pieces, np.int64)
    port().or_divide_bounds(n, pieces, _p(lo), _p(hi))
    return list(zip(lo.tolist(), hi.tolist()))


def _rp_args(rowptrs):
    rps = [I64(r) for r in rowptrs]
    arr = (i64p * len(rps))(*[_p(r) for r in rps])
    npos = I64([len(r) - 1 for r in rps])
    return rps, arr, npos


def partition_universe(rowptrs, nrows, pieces):
    rps, arr, npos = _rp_args(rowptrs)
    out = (or_color * pieces)()
    port().or_partition_universe(arr, _p(npos), len(rps), nrows, pieces, out)
    return out


def partition_nonzero(rowptrs, nnz, pieces):
    rps, arr, npos = _rp_args(rowptrs)
    out = (or_color * pieces)()
    port().or_partition_nonzero(arr, _p(npos), len(rps), nnz, pieces, out)
    return out


def preimage_range(rowptr, q_lo, q_hi):
    rp = I64(rowptr)
    n = port().or_preimage_range(_p(rp), len(rp) - 1, q_lo, q_hi, None, 0)
    out = np.empty(n, np.int64)
    port().or_preimage_range(_p(rp), len(rp) - 1, q_lo, q_hi, _p(out), n)
    return out


def spmv(rowptr, crd, vals, c, colours, nthreads=0):
    rp, cr, v, cc = I64(rowptr), I64(crd), F64(vals), F64(c)
    n = len(rp) - 1
    a = np.empty(n)
    work = np.zeros(len(colours), np.int64)
    comb = port().or_spmv(n, _p(rp), _p(cr), _p(v, dblp), _p(cc, dblp), len(colours), colours,
                          _p(a, dblp), _p(work), nthreads)
    return a, work, comb


def spmm(rowptr, crd, vals, Cm, N, colours, nthreads=0):
    rp, cr, v, cm = I64(rowptr), I64(crd), F64(vals), F64(Cm)
    n = len(rp) - 1
    A = np.empty(n * N)
    work = np.zeros(len(colours), np.int64)
    comb = port().or_spmm(n, _p(rp), _p(cr), _p(v, dblp), _p(cm, dblp), N, len(colours), colours,
                          _p(A, dblp), _p(work), nthreads)
    return A.reshape(n, N), work, comb


def sddmm(rowptr, crd, vals, Cm, Dm, K, dk, dj, colours, nthreads=0):
    rp, cr, v, cm, dm = I64(rowptr), I64(crd), F64(vals), F64(Cm), F64(Dm)
    n = len(rp) - 1
    A = np.empty(len(cr))
    work = np.zeros(len(colours), np.int64)
    comb = port().or_sddmm(n, _p(rp), _p(cr), _p(v, dblp), _p(cm, dblp), _p(dm, dblp), K, dk, dj,
                           len(colours), colours, _p(A, dblp), _p(work), nthreads)
    return A, work, comb


def spttv(rp1, crd1, rp2, crd2, vals, c, colours, nthreads=0):
    a1, c1, a2, c2, v, cc = I64(rp1), I64(crd1), I64(rp2), I64(crd2), F64(vals), F64(c)
    I = len(a1) - 1
    A = np.empty(len(c1))
    work = np.zeros(len(colours), np.int64)
    comb = port().or_spttv(I, _p(a1), _p(c1), _p(a2), _p(c2), _p(v, dblp), _p(cc, dblp),
                           len(colours), colours, _p(A, dblp), _p(work), nthreads)
    return A, work, comb


def spmttkrp(rp1, crd1, rp2, crd2, vals, Cm, Dm, R, colours, nthreads=0):
    a1, c1, a2, c2, v, cm, dm = I64(rp1), I64(crd1), I64(rp2), I64(crd2), F64(vals), F64(Cm), F64(Dm)
    I = len(a1) - 1
    A = np.empty(I * R)
    work = np.zeros(len(colours), np.int64)
    comb = port().or_spmttkrp(I, _p(a1), _p(c1), _p(a2), _p(c2), _p(v, dblp), _p(cm, dblp),
                              _p(dm, dblp), R, len(colours), colours, _p(A, dblp), _p(work),
                              nthreads)
    return A.reshape(I, R), work, comb


def spadd3(ops, nthreads=0):
    """ops: three (rowptr, crd, vals) CSR triples with equal row counts."""
    rps = [I64(o[0]) for o in ops]
    crds = [I64(o[1]) for o in ops]
    vals = [F64(o[2]) for o in ops]
    n = len(rps[0]) - 1
    rpa = (i64p * 3)(*[_p(r) for r in rps])
    cra = (i64p * 3)(*[_p(c) for c in crds])
    vaa = (dblp * 3)(*[_p(v, dblp) for v in vals])
    A_rp = np.empty(n + 1, np.int64)
    nnz = port().or_spadd3_count(n, rpa, cra, _p(A_rp), nthreads)
    A_crd = np.empty(nnz, np.int64)
    A_vals = np.empty(nnz)
    port().or_spadd3_fill(n, rpa, cra, vaa, _p(A_rp), _p(A_crd), _p(A_vals, dblp), nthreads)
    return A_rp, A_crd, A_vals


# ---- the reference itself ---------------------------------------------------
class ref_tensor_in(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("order", C.c_int),
        ("dims", i64p),
        ("format", C.c_char_p),
        ("pos_pairs", C.POINTER(i64p)),
        ("pos_len", i64p),
        ("crd", C.POINTER(i64p)),
        ("crd_len", i64p),
        ("vals", dblp),
        ("nvals", i64),
        ("tdn", C.c_char_p),
    ]


def ref(path=REF_LIB):
    if path not in _refs:
        if path == REF_LIB:
            ensure_built(ref=True)
        L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_run.restype = vp
        L.ref_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int,
                              C.POINTER(ref_tensor_in), C.c_int, C.c_char_p, C.c_int]
        for name, res, args in [
            ("ref_free", None, [vp]), ("ref_status", C.c_int, [vp]), ("ref_error", C.c_char_p, [vp]),
            ("ref_plan_seconds", C.c_double, [vp]), ("ref_exec_seconds", C.c_double, [vp]),
            ("ref_rendered_plan", C.c_char_p, [vp]), ("ref_stats_json", C.c_char_p, [vp]),
            ("ref_has_combine", C.c_int, [vp]), ("ref_num_loops", C.c_int, [vp]),
            ("ref_loop_info", C.c_int, [vp, C.c_int, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            ("ref_loop_color_bounds", C.c_int, [vp, C.c_int, i64p]),
            ("ref_step_bounds", C.c_int, [vp, C.c_int, C.c_char_p, C.POINTER(C.c_int), i64p]),
            ("ref_bundle_subset", i64, [vp, C.c_int, C.c_char_p, C.c_int, C.c_int, i64, i64p, i64]),
            ("ref_bundle_disjoint", C.c_int, [vp, C.c_int, C.c_char_p]),
            ("ref_out_nlevels", C.c_int, [vp]),
            ("ref_out_level", C.c_int, [vp, C.c_int, C.POINTER(C.c_int), i64p, i64p]),
            ("ref_out_copy_level", C.c_int, [vp, C.c_int, i64p, i64p]),
            ("ref_out_nvals", i64, [vp]), ("ref_out_copy_vals", C.c_int, [vp, dblp]),
            ("ref_stats_workers", i64, [vp]), ("ref_stats_combines", i64, [vp]),
            ("ref_stats_imbalance", C.c_double, [vp]), ("ref_stats_work", i64, [vp, i64]),
            ("ref_dense_eval", C.c_int, [C.c_char_p, C.c_int, C.POINTER(ref_tensor_in), C.c_int,
                                          i64p, dblp, C.c_char_p, C.c_int]),
            ("ref_pack", vp, [C.c_int, i64p, C.c_char_p, i64, i64p, dblp]),
            ("ref_load", vp, [C.c_char_p, C.c_char_p, C.c_int, i64p]),
            ("ref_out_dims", C.c_int, [vp, i64p]),
            ("ref_store", C.c_int, [vp, C.c_char_p]),
            ("ref_image", vp, [i64p, i64, i64, i64, i64p, i64p]),
            ("ref_preimage", vp, [i64p, i64, i64, i64, i64p, i64p]),
            ("ref_partition_by_bounds", vp, [C.c_int, i64p, i64, i64p, i64p]),
            ("ref_part_status", C.c_int, [vp]), ("ref_part_error", C.c_char_p, [vp]),
            ("ref_part_colors", i64, [vp]), ("ref_part_disjoint", C.c_int, [vp]),
            ("ref_part_copy", None, [vp, i64p, i64p]), ("ref_part_free", None, [vp]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _refs[path] = L
    return _refs[path]


def _ref_inputs(tensors):
    """tensors: dict name -> (host.SparseTensor, format string[, tdn])."""
    keep = []
    arr = (ref_tensor_in * len(tensors))()
    for i, (name, spec) in enumerate(tensors.items()):
        t, fmt = spec[0], spec[1]
        tdn = spec[2] if len(spec) > 2 else None
        nl = len(t.levels)
        dims = I64(t.dims)
        pos_pp = (i64p * nl)()
        crd_pp = (i64p * nl)()
        pos_len = np.zeros(nl, np.int64)
        crd_len = np.zeros(nl, np.int64)
        for l, lv in enumerate(t.levels):
            if lv.kind == "s":
                p = I64(lv.pos).reshape(-1)
                c = I64(lv.crd)
                keep += [p, c]
                pos_pp[l] = _p(p)
                crd_pp[l] = _p(c)
                pos_len[l] = lv.pos.shape[0]
                crd_len[l] = c.shape[0]
        vals = F64(t.vals)
        keep += [dims, pos_len, crd_len, vals, pos_pp, crd_pp]
        nm = name.encode()
        fm = fmt.encode()
        td = tdn.encode() if tdn else None
        keep += [nm, fm, td]
        arr[i] = ref_tensor_in(nm, len(t.dims), _p(dims), fm, C.cast(pos_pp, C.POINTER(i64p)),
                               _p(pos_len), C.cast(crd_pp, C.POINTER(i64p)), _p(crd_len),
                               _p(vals, dblp), len(vals), td)
    return arr, keep


class RefRun:
    """One reference pipeline run (cli.cpp:72-195 with in-memory tensors)."""

    def __init__(self, expr, schedule, grid, out_format, tensors, mode="seq", execute=True,
                 use_placements=False, out_tdn=None, lib=REF_LIB):
        L = ref(lib)
        self._arr, self._keep = _ref_inputs(tensors)
        self.h = L.ref_run(expr.encode(), schedule.encode() if schedule else b"", str(grid).encode(),
                           out_format.encode(), out_tdn.encode() if out_tdn else None,
                           len(tensors), self._arr, int(use_placements), mode.encode(),
                           int(execute))
        self.L = L
        self.status = L.ref_status(self.h)
        self.error = L.ref_error(self.h).decode()

    def __del__(self):
        try:
            self.L.ref_free(self.h)
        except Exception:
            pass

    def ok(self):
        if self.status:
            raise RuntimeError(f"reference failed ({self.status}): {self.error}")
        return self

    def loop(self, k=0):
        pieces = C.c_int64()
        pspace = C.c_int()
        lvl = C.c_int()
        self.L.ref_loop_info(self.h, k, C.byref(pieces), C.byref(pspace), C.byref(lvl))
        b = np.zeros(2 * pieces.value, np.int64)
        self.L.ref_loop_color_bounds(self.h, k, _p(b))
        return dict(pieces=pieces.value, position=bool(pspace.value), split_level=lvl.value,
                    bounds=[tuple(x) for x in b.reshape(-1, 2).tolist()])

    def step_bounds(self, tensor, k=0):
        kind = C.c_int()
        b = np.zeros(2 * 4096, np.int64)
        n = self.L.ref_step_bounds(self.h, k, tensor.encode(), C.byref(kind), _p(b))
        if n < 0:
            return None
        return kind.value, [tuple(x) for x in b[: 2 * n].reshape(-1, 2).tolist()]

    def subset(self, tensor, level, region, color, k=0):
        which = {"dom": 0, "pos": 1, "crd": 2, "vals": 3}[region]
        n = self.L.ref_bundle_subset(self.h, k, tensor.encode(), level, which, color, None, 0)
        if n < 0:
            return None
        out = np.empty(n, np.int64)
        self.L.ref_bundle_subset(self.h, k, tensor.encode(), level, which, color, _p(out), n)
        return out

    def combine(self):
        return bool(self.L.ref_has_combine(self.h))

    def output(self):
        """(levels [(kind, pos_pairs, crd)], vals)."""
        L = self.L
        levels = []
        for l in range(L.ref_out_nlevels(self.h)):
            kind = C.c_int()
            pl = C.c_int64()
            cl = C.c_int64()
            L.ref_out_level(self.h, l, C.byref(kind), C.byref(pl), C.byref(cl))
            if kind.value == 0:
                levels.append(("d", None, None))
            else:
                pos = np.empty(2 * pl.value, np.int64)
                crd = np.empty(cl.value, np.int64)
                L.ref_out_copy_level(self.h, l, _p(pos), _p(crd))
                levels.append(("s", pos.reshape(-1, 2), crd))
        vals = np.empty(L.ref_out_nvals(self.h))
        L.ref_out_copy_vals(self.h, _p(vals, dblp))
        return levels, vals

    @classmethod
    def pack(cls, dims, fmt: str, coords, values, lib=REF_LIB):
        """SparseTensor::pack (tensor.cpp:94-182) run by the reference itself;
        read the result with output()."""
        self = cls.__new__(cls)
        L = ref(lib)
        dims = I64(dims)
        coords = I64(np.asarray(coords).reshape(-1, len(dims)))
        values = F64(np.asarray(values, dtype=np.float64).reshape(-1))
        self._keep = (dims, coords, values)
        self.h = L.ref_pack(len(dims), _p(dims), fmt.encode(), values.shape[0], _p(coords), _p(values, dblp))
        self.L = L
        self.status = L.ref_status(self.h)
        self.error = L.ref_error(self.h).decode()
        return self

    @classmethod
    def load(cls, path, fmt: str, order: int, dims=None, lib=REF_LIB):
        """load_tensor (tensor_io.cpp:136-142) run by the reference itself."""
        self = cls.__new__(cls)
        L = ref(lib)
        d = I64(dims) if dims is not None else None
        self._keep = (d,)
        self.h = L.ref_load(str(path).encode(), fmt.encode(), order, _p(d) if d is not None else None)
        self.L = L
        self.status = L.ref_status(self.h)
        self.error = L.ref_error(self.h).decode()
        return self

    def store(self, path):
        return self.L.ref_store(self.h, str(path).encode())

    def out_dims(self, order):
        d = np.zeros(order, np.int64)
        self.L.ref_out_dims(self.h, _p(d))
        return tuple(int(x) for x in d)

    def stats(self):
        L = self.L
        w = L.ref_stats_workers(self.h)
        return dict(workers=w, combines=L.ref_stats_combines(self.h),
                    imbalance=L.ref_stats_imbalance(self.h),
                    work=[L.ref_stats_work(self.h, i) for i in range(w)])

    def plan_seconds(self):
        return self.L.ref_plan_seconds(self.h)

    def exec_seconds(self):
        return self.L.ref_exec_seconds(self.h)

    def rendered(self):
        return self.L.ref_rendered_plan(self.h).decode()


def dense_eval(expr, tensors, out_dims):
    arr, keep = _ref_inputs(tensors)
    out = np.empty(int(np.prod(out_dims)) if out_dims else 1)
    od = I64(out_dims)
    err = C.create_string_buffer(512)
    st = ref().ref_dense_eval(expr.encode(), len(tensors), arr, len(out_dims), _p(od),
                              _p(out, dblp), err, 512)
    if st:
        raise RuntimeError(err.value.decode())
    return out.reshape(out_dims)


# ---- dependent partitioning through the reference (deppart.cpp:15-101) ----
class RefPartitionError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _flat_partition(subsets):
    off = np.zeros(len(subsets) + 1, np.int64)
    for c, s in enumerate(subsets):
        off[c + 1] = off[c] + len(s)
    idx = np.concatenate([np.asarray(s, np.int64) for s in subsets]) if subsets else np.zeros(0, np.int64)
    return off, np.ascontiguousarray(idx, dtype=np.int64)


def _read_part(L, h):
    try:
        if L.ref_part_status(h):
            raise RefPartitionError(L.ref_part_status(h), L.ref_part_error(h).decode())
        P = L.ref_part_colors(h)
        off = np.zeros(P + 1, np.int64)
        L.ref_part_copy(h, _p(off), None)
        idx = np.zeros(max(int(off[-1]), 1), np.int64)
        L.ref_part_copy(h, _p(off), _p(idx))
        return [idx[off[c]:off[c + 1]].copy() for c in range(P)], bool(L.ref_part_disjoint(h))
    finally:
        L.ref_part_free(h)


def ref_image(ranges, subsets, dest_extent, lib=REF_LIB):
    """The reference's image (deppart.cpp:15-31): (subsets, disjoint)."""
    L = ref(lib)
    r = np.ascontiguousarray(np.asarray(ranges, np.int64).reshape(-1, 2))
    off, idx = _flat_partition(subsets)
    return _read_part(L, L.ref_image(_p(r), len(r), dest_extent, len(subsets), _p(off), _p(idx)))


def ref_preimage(ranges, subsets, dest_extent, lib=REF_LIB):
    """The reference's preimage (deppart.cpp:33-53): (subsets, disjoint)."""
    L = ref(lib)
    r = np.ascontiguousarray(np.asarray(ranges, np.int64).reshape(-1, 2))
    off, idx = _flat_partition(subsets)
    return _read_part(L, L.ref_preimage(_p(r), len(r), dest_extent, len(subsets), _p(off), _p(idx)))


def ref_partition_by_bounds(extents, coloring):
    """The reference's partition_by_bounds (deppart.cpp:55-91); coloring:
    {colour: [(lo, hi) per dimension]}."""
    L = ref()
    ext = np.asarray(extents, np.int64)
    cols = np.asarray(sorted(coloring), np.int64)
    b = np.asarray([coloring[c] for c in sorted(coloring)], np.int64).reshape(-1)
    return _read_part(L, L.ref_partition_by_bounds(len(ext), _p(ext), len(cols), _p(cols), _p(b)))
