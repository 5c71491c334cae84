#!/usr/bin/env python3
"""Profiling driver (ncu target): one BASELINE config's op, run --steps times
on one GPU with the bench's inputs and code path.

  python scripts/prof_configs.py --config c1|spmv|c3|ttv|mttkrp|c5 [--steps 3]
  ncu --set full -k regex:<leaf> -s 2 -c 1 python scripts/prof_configs.py --config c1
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", required=True, choices=["c1", "spmv", "c3", "ttv", "mttkrp", "c5", "spmv_long", "spmv_dense"])
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--scale", type=int, default=24)
a = ap.parse_args()

import torch  # noqa: E402

from paper_2207_13901_b200 import _native as N  # noqa: E402
from paper_2207_13901_b200 import host as H  # noqa: E402

dev = torch.device("cuda", 0)
ctx = H.Context(0)
S = N.synth()
fmt = H.parse_format("ds")


def wrap(n, m, rp, crd, vals):
    rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
    return H.DeviceTensor.wrap(ctx, (n, m), fmt, [rp_d.data_ptr()], [crd_d.data_ptr()], vals_d.data_ptr(),
                               keep=(rp_d, crd_d, vals_d))


ops = []
if a.config == "c1":
    n, nz = 1_000_000, 10_000_000
    rp, crd, vals = np.empty(n + 1, np.int64), np.empty(nz, np.int64), np.empty(nz)
    nnz = S.syn_uniform_csr(n, n, nz, 42, 0, rp.ctypes.data_as(N.i64p), crd.ctypes.data_as(N.i64p),
                            vals.ctypes.data_as(N.dblp))
    B = wrap(n, n, rp, crd[:nnz], vals[:nnz])
    x = torch.from_numpy(bench.dense_vals(n, 43)).to(dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    ops.append(lambda: (H.partition_universe(ctx, B, 1, host=False), H.spmv(ctx, B, x, y, pieces=1, stats=False)))
elif a.config in ("spmv_long", "spmv_dense"):
    # long-row SpMV shapes (no BASELINE config): uniform 400K x 400K with 250
    # per row, R-MAT scale 20 with edge factor 100
    if a.config == "spmv_long":
        n, nz = 400_000, 100_000_000
        rp, crd, vals = np.empty(n + 1, np.int64), np.empty(nz, np.int64), np.empty(nz)
        nnz = S.syn_uniform_csr(n, n, nz, 42, 0, rp.ctypes.data_as(N.i64p), crd.ctypes.data_as(N.i64p),
                                vals.ctypes.data_as(N.dblp))
        crd, vals = crd[:nnz], vals[:nnz]
    else:
        n, rp, crd, vals = bench.rmat_csr(20, 100, 42)
    B = wrap(n, n, rp, crd, vals)
    x = torch.from_numpy(bench.dense_vals(n, 44)).to(dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    ops.append(lambda: (H.partition_nonzero(ctx, B, 1, 1, host=False),
                        H.spmv(ctx, B, x, y, pieces=1, stats=False)))
elif a.config in ("spmv", "c3", "c5"):
    n, rp, crd, vals = bench.rmat_csr(a.scale, 10, 42)
    B = wrap(n, n, rp, crd, vals)
    if a.config == "spmv":
        x = torch.from_numpy(bench.dense_vals(n, 44)).to(dev)
        y = torch.empty(n, dtype=torch.float64, device=dev)
        ops.append(lambda: (H.partition_nonzero(ctx, B, 1, 1, host=False),
                            H.spmv(ctx, B, x, y, pieces=1, stats=False)))
    elif a.config == "c3":
        K = 128
        Cd = torch.from_numpy(bench.dense_vals(n * K, 44)).to(dev)
        Dd = torch.from_numpy(bench.dense_vals(n * K, 45)).to(dev)
        Av = torch.empty(len(crd), dtype=torch.float64, device=dev)
        ops.append(lambda: (H.partition_nonzero(ctx, B, 1, 1, host=False),
                            H.sddmm(ctx, B, Cd, Dd, K, 1, K, Av, pieces=1, stats=False)))
    else:
        Bs = [B]
        for shift in (1, 2):
            rps, e = np.empty(n + 1, np.int64), 10 * n
            cs, vs = np.empty(e, np.int64), np.empty(e)
            k = S.syn_rmat_csr(a.scale, e, bench.A_RMAT, bench.B_RMAT, bench.C_RMAT, 42, 0, 0, shift,
                               rps.ctypes.data_as(N.i64p), cs.ctypes.data_as(N.i64p), vs.ctypes.data_as(N.dblp))
            Bs.append(wrap(n, n, rps, cs[:k], vs[:k]))

        def add3():
            H.partition_universe(ctx, Bs[0], 8, host=False)
            A, _ = H.spadd3(ctx, Bs[0], Bs[1], Bs[2], pieces=8, stats=False)
            A.close()
        ops.append(add3)
else:
    I, J, Kd, Sm, R = 12092, 9184, 28818, 10_000_000, 32
    rp1, crd1 = np.empty(I + 1, np.int64), np.empty(Sm, np.int64)
    rp2, crd2 = np.empty(Sm + 1, np.int64), np.empty(Sm, np.int64)
    vals, F = np.empty(Sm), np.zeros(1, np.int64)
    nnz = S.syn_powerlaw_csf(I, J, Kd, Sm, 4, 0, rp1.ctypes.data_as(N.i64p), crd1.ctypes.data_as(N.i64p),
                             rp2.ctypes.data_as(N.i64p), crd2.ctypes.data_as(N.i64p), vals.ctypes.data_as(N.dblp),
                             F.ctypes.data_as(N.i64p))
    F = int(F[0])
    Bt = H.DeviceTensor.upload_rowptr(ctx, (I, J, Kd), H.parse_format("dss"), [rp1, rp2[:F + 1]],
                                      [crd1[:F], crd2[:nnz]], vals[:nnz])
    if a.config == "ttv":
        c = torch.from_numpy(bench.dense_vals(Kd, 46)).to(dev)
        Av = torch.empty(F, dtype=torch.float64, device=dev)
        ops.append(lambda: (H.partition_nonzero(ctx, Bt, 2, 1, host=False),
                            H.spttv(ctx, Bt, c, Av, pieces=1, stats=False)))
    else:
        Cm = torch.from_numpy(bench.dense_vals(J * R, 47)).to(dev)
        Dm = torch.from_numpy(bench.dense_vals(Kd * R, 48)).to(dev)
        A = torch.empty(I * R, dtype=torch.float64, device=dev)
        ops.append(lambda: (H.partition_nonzero(ctx, Bt, 2, 1, host=False),
                            H.spmttkrp(ctx, Bt, Cm, Dm, R, A, pieces=1, stats=False)))

ctx.timing(True)
for _ in range(a.steps):
    for op in ops:
        op()
torch.cuda.synchronize()
print(a.config, "leaf ms:", [round(x, 4) for x in ctx.read_timing()])
ctx.close()
