#!/usr/bin/env python3
"""The whole reference pipeline on the C2 SpMM schedule (measurement only):
dspar's plan() + execute() in par mode on all host threads
(oracle/_ref/libdspar_ref.so) against the drop-in (oracle/_ref/libdspar_gpu.so:
the same plan() with the GPU dependent partitioning and the fast Partition
class, execute() replaced by execute_gpu on every visible GPU), on the R-MAT
CSR at growing scales; outputs compared at 1e-10 relative.  One JSON line
per scale.  Run the host with GLIBC_TUNABLES=glibc.malloc.hugetlb=1 to give
the planner's multi-GB vectors huge pages (both arms).

  python scripts/dropin_timing.py --scales 18,20,21
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import oracle_bind as ob  # noqa: E402

from paper_2207_13901_b200.host import Level, SparseTensor, parse_format  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scales", default="18,20")
ap.add_argument("--pieces", type=int, default=8)
ap.add_argument("--cols", type=int, default=32)
ap.add_argument("--arms", default="reference_par,dropin_gpu")
a = ap.parse_args()
EXPR = "A(i, j) = B(i, k) * C(k, j)"
SCHED = "reorder(i, k, j); fuse(i, k, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)"
for sc in (int(x) for x in a.scales.split(",")):
    n, rp, crd, vals = bench.rmat_csr(sc, 10, 42)
    B = SparseTensor.from_rowptrs((n, n), parse_format("ds"), [rp], [crd], vals)
    Cm = SparseTensor.from_parts((n, a.cols), parse_format("dd"), [Level("d", dom=(n, a.cols))],
                                 bench.dense_vals(n * a.cols, 43))
    tens = {"B": (B, "ds"), "C": (Cm, "dd")}
    out = {"scale": sc, "rows": n, "nnz": int(len(crd)), "pieces": a.pieces, "cols": a.cols,
           "cpu": bench.cpu_model(), "host_threads": bench.host_cores(),
           "hugetlb": os.environ.get("GLIBC_TUNABLES", "")}
    res = {}
    for name, lib, mode in (("reference_par", ob.REF_LIB, "par"), ("dropin_gpu", ob.GPU_LIB, "gpu")):
        if name not in a.arms.split(","):
            continue
        t0 = time.time()
        run = ob.RefRun(EXPR, SCHED, a.pieces, "dd", tens, mode=mode, lib=lib).ok()
        wall = time.time() - t0
        out[f"{name}_plan_s"] = run.plan_seconds()
        out[f"{name}_exec_s"] = run.exec_seconds()
        out[f"{name}_wall_s"] = wall
        res[name] = np.asarray(run.output()[1])
        out[f"{name}_stats"] = run.stats()
        del run
    if len(res) == 2:
        want, got = res["reference_par"], res["dropin_gpu"]
        out["match_1e-10"] = bool(np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300)))
        out["same_stats"] = out["reference_par_stats"] == out["dropin_gpu_stats"]
    for k in ("reference_par_stats", "dropin_gpu_stats"):
        out.pop(k, None)
    print(json.dumps(out), flush=True)
