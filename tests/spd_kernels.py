"""TEST INFRASTRUCTURE: the six hot-path kernels as the reference states them.

Expressions, formats and schedules are the reference's (checked
against the reference in section 9.2); `instance()` builds small random
inputs the way the reference's tests do (test_util.hpp:48-61: integer values,
duplicate coordinates summed by pack).
"""
import numpy as np

from paper_2207_13901_b200.host import SparseTensor, parse_format

ROW = "divide(i, io, ii, M.x); distribute(io, M.x)"

KERNELS = {
    "spmv": dict(
        expr="a(i) = B(i, j) * c(j)",
        formats={"a": "d", "B": "ds", "c": "d"},
        nonzero="fuse(i, j, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)",
    ),
    "spmm": dict(
        expr="A(i, j) = B(i, k) * C(k, j)",
        formats={"A": "dd", "B": "ds", "C": "dd"},
        nonzero="reorder(i, k, j); fuse(i, k, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)",
    ),
    "sddmm": dict(
        expr="A(i, j) = B(i, j) * C(i, k) * D(k, j)",
        formats={"A": "ds", "B": "ds", "C": "dd", "D": "dd:1,0"},
        nonzero="fuse(i, j, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)",
    ),
    "spttv": dict(
        expr="A(i, j) = B(i, j, k) * c(k)",
        formats={"A": "ds", "B": "dss", "c": "d"},
        nonzero="fuse(i, j, f); fuse(f, k, g); divide(g, go, gi, B.pos, M.x); distribute(go, M.x)",
    ),
    "spmttkrp": dict(
        expr="A(i, l) = B(i, j, k) * C(j, l) * D(k, l)",
        formats={"A": "dd", "B": "dss", "C": "dd", "D": "dd"},
        nonzero="reorder(i, j, k, l); fuse(i, j, f); fuse(f, k, g); divide(g, go, gi, B.pos, M.x); "
                "distribute(go, M.x)",
    ),
    "spadd3": dict(
        expr="A(i, j) = B(i, j) + C(i, j) + D(i, j)",
        formats={"A": "ds", "B": "ds", "C": "ds", "D": "ds"},
        nonzero=None,  # rejected by the reference (schedule.cpp:334-336)
    ),
}

OUTPUT = {"spmv": "a", "spmm": "A", "sddmm": "A", "spttv": "A", "spmttkrp": "A", "spadd3": "A"}


def _values(rng, n, integers):
    if integers:
        return rng.integers(-3, 4, size=n).astype(np.float64)
    return rng.uniform(0.5, 1.5, size=n)


def random_sparse(rng, dims, fmt, density, integers=True):
    total = int(np.prod(dims))
    want = max(1, int(total * density))
    coords = np.stack([rng.integers(0, d, size=want) for d in dims], axis=1)
    return SparseTensor.pack(dims, parse_format(fmt), coords, _values(rng, want, integers))


def dense(rng, dims, fmt="d", integers=True):
    f = parse_format(fmt)
    total = int(np.prod(dims))
    coords = np.array(np.unravel_index(np.arange(total), dims)).T if total else np.zeros((0, len(dims)), np.int64)
    return SparseTensor.pack(dims, f, coords, _values(rng, total, integers))


def instance(kernel, rng, integers=True, density=0.15, max_dim=40, rank=None):
    """Random inputs {name: SparseTensor} for one kernel."""
    d = lambda: int(rng.integers(1, max_dim + 1))
    if kernel == "spmv":
        n, m = d(), d()
        return {"B": random_sparse(rng, (n, m), "ds", density, integers),
                "c": dense(rng, (m,), "d", integers)}
    if kernel == "spmm":
        n, k = d(), d()
        N = rank or int(rng.integers(1, 9))
        return {"B": random_sparse(rng, (n, k), "ds", density, integers),
                "C": dense(rng, (k, N), "dd", integers)}
    if kernel == "sddmm":
        n, m = d(), d()
        K = rank or int(rng.integers(1, 9))
        return {"B": random_sparse(rng, (n, m), "ds", density, integers),
                "C": dense(rng, (n, K), "dd", integers),
                "D": dense(rng, (K, m), "dd:1,0", integers)}
    if kernel == "spttv":
        I, J, K = (int(rng.integers(1, 13)) for _ in range(3))
        return {"B": random_sparse(rng, (I, J, K), "dss", density, integers),
                "c": dense(rng, (K,), "d", integers)}
    if kernel == "spmttkrp":
        I, J, K = (int(rng.integers(1, 13)) for _ in range(3))
        R = rank or int(rng.integers(1, 6))
        return {"B": random_sparse(rng, (I, J, K), "dss", density, integers),
                "C": dense(rng, (J, R), "dd", integers),
                "D": dense(rng, (K, R), "dd", integers)}
    if kernel == "spadd3":
        n, m = d(), d()
        return {X: random_sparse(rng, (n, m), "ds", density, integers) for X in "BCD"}
    raise KeyError(kernel)


def ref_inputs(kernel, tensors):
    fm = KERNELS[kernel]["formats"]
    return {name: (t, fm[name]) for name, t in tensors.items()}
