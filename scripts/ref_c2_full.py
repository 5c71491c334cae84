#!/usr/bin/env python3
"""The reference's own CPU path on the C2 headline workload at growing R-MAT
scales (measurement only; verdict round 1 item 9): plan() + execute() of
/root/reference/proj/core (built into oracle/_ref, par mode, P colours) on
the R-MAT CSR of each scale with C n x 32, output compared with the GPU's at
1e-10.  One JSON line per scale.  The bench's reference arm times the
scale-17 sample; the ladder shows how the reference's rate depends on the
scale, up to the largest scale the host fits (--scales ... 24 is the full
C2 workload: plan() replicates C per colour and execute() allocates a dense
n x 32 accumulator per task, ~40-80 GB; it was killed for memory on the GPU
box at P = 8).

  python scripts/ref_c2_full.py --scales 16,17,18,19,20 [--pieces 16]
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
ap.add_argument("--pieces", type=int, default=16)
ap.add_argument("--scales", default="16,17,18,19,20")
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


for scale in (int(x) for x in a.scales.split(",")):
    out = {"cpu": bench.cpu_model(), "host_cores": bench.host_cores(), "pieces": a.pieces}
    n, rp, crd, vals, Cv, run, wall = ref_run(scale, a.pieces)
    fl = 2.0 * len(crd) * 32
    ref_out = np.asarray(run.output()[1])
    out.update({"scale": scale, "rows": n, "nnz": int(len(crd)), "plan_s": run.plan_seconds(),
                "exec_s": run.exec_seconds(), "wall_s": wall,
                "gflops": fl / (run.plan_seconds() + run.exec_seconds()) / 1e9,
                "gflops_execute_only": fl / run.exec_seconds() / 1e9,
                "combines": json.loads(run.L.ref_stats_json(run.h).decode())["combines"]})
    del run
    try:
        import torch

        from paper_2207_13901_b200 import host as H
        dev = torch.device("cuda", 0)
        ctx = H.Context(0)
        rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
        B = H.DeviceTensor.wrap(ctx, (n, n), parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                                vals_d.data_ptr())
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
