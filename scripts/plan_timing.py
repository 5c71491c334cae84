#!/usr/bin/env python3
"""plan() of the reference's own planner (oracle/_ref/libdspar_ref.so), with
only dspar::Partition replaced (libdspar_fastpart.so,
integration/partition_fast.cpp), and as the drop-in links it -- the GPU
dependent partitioning (integration/deppart_gpu.cpp) plus the fast Partition
(libdspar_gpu.so) -- on the C2 schedule (nonzero split of the R-MAT CSR, P
colours) at growing scales; the plans' colour bounds and bundle subsets are
compared with the reference's (measurement only)."""
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
ap.add_argument("--kernel", default="spmm", choices=["spmv", "spmm"])
ap.add_argument("--cols", type=int, default=32, help="columns of C (spmm)")
ap.add_argument("--no-gpu", action="store_true")
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
        other = {"C": (SparseTensor.from_parts((n, a.cols), parse_format("dd"), [Level("d", dom=(n, a.cols))],
                                               np.ones(n * a.cols)), "dd")}
        out_fmt = "dd"
    tens = {"B": (B, "ds"), **other}
    FAST = os.path.join(os.path.dirname(ob.REF_LIB), "libdspar_fastpart.so")
    libs = [("reference", ob.REF_LIB), ("fast_partition", FAST)] + ([] if a.no_gpu else [("gpu_deppart_fast_partition",
                                                                                         ob.GPU_LIB)])
    out = {"kernel": a.kernel, "scale": sc, "rows": n, "nnz": int(len(crd)), "pieces": a.pieces,
           "cols": a.cols if a.kernel == "spmm" else None, "cpu": bench.cpu_model()}
    ref = None
    for name, lib in libs:
        run = ob.RefRun(EXPR, SCHED, a.pieces, out_fmt, tens, execute=False, lib=lib).ok()
        out[f"plan_s_{name}"] = run.plan_seconds()
        subs = [run.subset("B", 1, region, c) for region in ("pos", "crd") for c in range(a.pieces)]
        if ref is None:
            ref = (run.loop()["bounds"], subs)
        else:
            out[f"same_as_reference_{name}"] = bool(run.loop()["bounds"] == ref[0] and
                                                    all(np.array_equal(x, y) for x, y in zip(subs, ref[1])))
        del run
    print(json.dumps(out), flush=True)
