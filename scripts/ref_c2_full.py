#!/usr/bin/env python3
"""One full-size run of the reference's own CPU path on the C2 headline
workload (measurement only; verdict round 1 item 9): plan() + execute() of
/root/reference/proj/core (built into oracle/_ref, par mode) on the R-MAT
scale-24 CSR with C 16.8M x 32, nonzero split into P colours, output compared
with the GPU's at 1e-10.  Prints one JSON line; the bench's reference arm
uses a bounded scale-17 sample of the same generator, and this run puts that
sample's rate next to the full-size rate.

  python scripts/ref_c2_full.py [--pieces 8]   (~40-80 GB host memory)
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
import oracle_bind as ob  # noqa: E402  (the reference itself)

ap = argparse.ArgumentParser()
ap.add_argument("--pieces", type=int, default=8)
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--sample-scale", type=int, default=17)
a = ap.parse_args()

from paper_2207_13901_b200.host import Level, SparseTensor, parse_format  # noqa: E402

SCHED = "reorder(i, k, j); fuse(i, k, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)"


def ref_run(scale, pieces):
    n, rp, crd, vals = bench.rmat_csr(scale, 10, 42)
    B = SparseTensor.from_rowptrs((n, n), parse_format("ds"), [rp], [crd], vals)
    Cv = bench.dense_vals(n * 32, 43)
    Cm = SparseTensor.from_parts((n, 32), parse_format("dd"), [Level("d", dom=(n, 32))], Cv)
    t0 = time.time()
    run = ob.RefRun("A(i, j) = B(i, k) * C(k, j)", SCHED, pieces, "dd", {"B": (B, "ds"), "C": (Cm, "dd")},
                    mode="par").ok()
    wall = time.time() - t0
    return n, rp, crd, vals, Cv, run, wall


out = {"cpu": bench.cpu_model(), "host_cores": bench.host_cores(), "pieces": a.pieces}
# the bounded sample the bench's reference arm times
n, rp, crd, vals, Cv, run, wall = ref_run(a.sample_scale, a.pieces)
fl = 2.0 * len(crd) * 32
out["sample"] = {"scale": a.sample_scale, "nnz": int(len(crd)), "plan_s": run.plan_seconds(),
                 "exec_s": run.exec_seconds(), "gflops": fl / (run.plan_seconds() + run.exec_seconds()) / 1e9}
del run
# the full-size workload
n, rp, crd, vals, Cv, run, wall = ref_run(a.scale, a.pieces)
fl = 2.0 * len(crd) * 32
ref_out = np.asarray(run.output()[1])
out["full"] = {"scale": a.scale, "rows": n, "nnz": int(len(crd)), "plan_s": run.plan_seconds(),
               "exec_s": run.exec_seconds(), "wall_s": wall,
               "gflops": fl / (run.plan_seconds() + run.exec_seconds()) / 1e9,
               "gflops_execute_only": fl / run.exec_seconds() / 1e9, "stats": json.loads(
                   run.L.ref_stats_json(run.h).decode())["combines"]}
del run
try:
    import torch

    from paper_2207_13901_b200 import host as H
    dev = torch.device("cuda", 0)
    ctx = H.Context(0)
    rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
    B = H.DeviceTensor.wrap(ctx, (n, n), parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()], vals_d.data_ptr())
    C_d = torch.from_numpy(Cv).to(dev)
    A_d = torch.empty(n * 32, dtype=torch.float64, device=dev)
    H.partition_nonzero(ctx, B, 1, a.pieces)
    st = H.spmm(ctx, B, C_d, 32, A_d, pieces=a.pieces)
    got = A_d.cpu().numpy()
    out["matches_gpu"] = bool(np.all(np.abs(got - ref_out) <= 1e-10 * np.maximum(np.abs(ref_out), 1e-300)))
    out["gpu_combines"] = st.combines
    B.close()
    ctx.close()
except Exception as ex:  # no GPU here: the reference numbers alone
    out["matches_gpu"] = f"not checked: {ex}"
print(json.dumps(out), flush=True)
