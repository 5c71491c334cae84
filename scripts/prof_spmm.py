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
ap.add_argument("--cols", type=int, default=None, help="N (SpMM, default 32) or K (SDDMM, default 128)")
ap.add_argument("--kernel", default="spmm", choices=["spmm", "spmv", "sddmm"])
ap.add_argument("--slice", default=None, help="q/P: only the rows of nonzero colour q of P (whole rows)")
a = ap.parse_args()
if a.cols is None:
    a.cols = 128 if a.kernel == "sddmm" else 32

import torch  # noqa: E402

from paper_2207_13901_b200 import host as H  # noqa: E402

n, rp, crd, vals = bench.rmat_csr(a.scale, 10, 42)
if a.slice:
    import numpy as np
    q, P = (int(x) for x in a.slice.split("/"))
    nnz = len(crd)
    lo, hi = q * nnz // P, (q + 1) * nnz // P - 1
    r0 = int(np.searchsorted(rp, lo, side="right") - 1)
    r1 = int(np.searchsorted(rp, hi, side="right") - 1)
    crd, vals = crd[rp[r0]:rp[r1 + 1]], vals[rp[r0]:rp[r1 + 1]]
    rp = rp[r0:r1 + 2] - rp[r0]
    print("slice rows", r0, r1, "nnz", len(crd), "non-empty rows", int(np.count_nonzero(np.diff(rp))))
m = n
n = len(rp) - 1
dev = torch.device("cuda", 0)
rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
N = a.cols if a.kernel in ("spmm", "sddmm") else 1  # SDDMM: K (C2 configs use 128)
C_d = torch.from_numpy(bench.dense_vals(m * N, 43)).to(dev)
A_d = torch.empty(n * N if a.kernel != "sddmm" else len(crd), dtype=torch.float64, device=dev)
if a.kernel == "sddmm":
    D_d = torch.from_numpy(bench.dense_vals(m * N, 44)).to(dev)
ctx = H.Context(0)
B = H.DeviceTensor.wrap(ctx, (n, m), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
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
if a.kernel != "sddmm":
    print("digest", int(A_d.view(torch.int64).sum().item()), "nan", bool(torch.isnan(A_d).any().item()))
print("leaf ms:", [round(x, 3) for x in ctx.read_timing()], "nnz", len(crd))
ctx.close()
