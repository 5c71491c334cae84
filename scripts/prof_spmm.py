#!/usr/bin/env python3
"""Profiling driver: the bench's C2 SpMM step (R-MAT scale 24, N=32), run
`--steps` times on one GPU; for ncu (-k regex:k_spmm_walk)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--cols", type=int, default=32)
ap.add_argument("--kernel", default="spmm", choices=["spmm", "spmv", "sddmm"])
a = ap.parse_args()

import torch  # noqa: E402

from paper_2207_13901_b200 import host as H  # noqa: E402

n, rp, crd, vals = bench.rmat_csr(a.scale, 10, 42)
dev = torch.device("cuda", 0)
rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
N = a.cols if a.kernel == "spmm" else (128 if a.kernel == "sddmm" else 1)
C_d = torch.from_numpy(bench.dense_vals(n * N, 43)).to(dev)
A_d = torch.empty(n * N if a.kernel != "sddmm" else len(crd), dtype=torch.float64, device=dev)
if a.kernel == "sddmm":
    D_d = torch.from_numpy(bench.dense_vals(n * N, 44)).to(dev)
ctx = H.Context(0)
B = H.DeviceTensor.wrap(ctx, (n, n), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                        vals_d.data_ptr())
ctx.timing(True)
for _ in range(a.steps):
    H.partition_nonzero(ctx, B, 1, 1, host=False)
    if a.kernel == "spmm":
        H.spmm(ctx, B, C_d, N, A_d, pieces=1, stats=False)
    elif a.kernel == "sddmm":
        H.sddmm(ctx, B, C_d, D_d, N, 1, N, A_d, pieces=1, stats=False)
    else:
        H.spmv(ctx, B, C_d, A_d, pieces=1, stats=False)
torch.cuda.synchronize()
print("leaf ms:", [round(x, 3) for x in ctx.read_timing()], "nnz", len(crd))
ctx.close()
