#!/usr/bin/env python3
"""plan() of the reference's own planner with its CPU dependent partitioning
(oracle/_ref/libdspar_ref.so) and with the GPU operators linked in its place
(oracle/_ref/libdspar_gpu.so, integration/deppart_gpu.cpp), on the C2 SpMM
schedule (nonzero split of the R-MAT CSR, P colours) at growing scales, the
two plans' colour bounds and bundle subsets compared (measurement only)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import oracle_bind as ob  # noqa: E402

from paper_2207_13901_b200.host import Level, SparseTensor, parse_format  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scales", default="18,20,22")
ap.add_argument("--pieces", type=int, default=8)
ap.add_argument("--kernel", default="spmv", choices=["spmv", "spmm"])
a = ap.parse_args()
EXPR = {"spmv": "a(i) = B(i, j) * c(j)", "spmm": "A(i, j) = B(i, k) * C(k, j)"}[a.kernel]
SCHED = {"spmv": "fuse(i, j, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)",
         "spmm": "reorder(i, k, j); fuse(i, k, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)"}[a.kernel]
for sc in (int(x) for x in a.scales.split(",")):
    n, rp, crd, vals = bench.rmat_csr(sc, 10, 42)
    B = SparseTensor.from_rowptrs((n, n), parse_format("ds"), [rp], [crd], vals)
    if a.kernel == "spmv":
        other = {"c": (SparseTensor.from_parts((n,), parse_format("d"), [Level("d", dom=(n,))], np.ones(n)), "d")}
        out_fmt = "d"
    else:
        other = {"C": (SparseTensor.from_parts((n, 4), parse_format("dd"), [Level("d", dom=(n, 4))],
                                               np.ones(n * 4)), "dd")}
        out_fmt = "dd"
    tens = {"B": (B, "ds"), **other}
    cpu = ob.RefRun(EXPR, SCHED, a.pieces, out_fmt, tens, execute=False, lib=ob.REF_LIB).ok()
    gpu = ob.RefRun(EXPR, SCHED, a.pieces, out_fmt, tens, execute=False, lib=ob.GPU_LIB).ok()
    same = cpu.loop()["bounds"] == gpu.loop()["bounds"]
    for c in range(a.pieces):
        for lvl, region in ((1, "pos"), (1, "crd")):
            same = same and np.array_equal(cpu.subset("B", lvl, region, c), gpu.subset("B", lvl, region, c))
    print(json.dumps({"kernel": a.kernel, "scale": sc, "rows": n, "nnz": int(len(crd)), "pieces": a.pieces,
                      "plan_cpu_deppart_s": cpu.plan_seconds(), "plan_gpu_deppart_s": gpu.plan_seconds(),
                      "same_bounds_and_B_subsets": bool(same), "cpu": bench.cpu_model()}), flush=True)
