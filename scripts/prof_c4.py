#!/usr/bin/env python3
"""Profiling driver for config C4 (SpTTV / SpMTTKRP on the power-law dss tensor)."""
import argparse, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa
from paper_2207_13901_b200 import _native as N  # noqa
ap = argparse.ArgumentParser(); ap.add_argument("--steps", type=int, default=3); ap.add_argument("--kernel", default="spmttkrp"); ap.add_argument("--rank", type=int, default=32)
a = ap.parse_args()
import torch  # noqa
from paper_2207_13901_b200 import host as H  # noqa
I, J, Kd, S = 12092, 9184, 28818, 10_000_000
rp1 = np.empty(I + 1, np.int64); crd1 = np.empty(S, np.int64); rp2 = np.empty(S + 1, np.int64)
crd2 = np.empty(S, np.int64); vals = np.empty(S); F = np.zeros(1, np.int64)
nnz = N.synth().syn_powerlaw_csf(I, J, Kd, S, 4, 0, rp1.ctypes.data_as(N.i64p), crd1.ctypes.data_as(N.i64p),
                                 rp2.ctypes.data_as(N.i64p), crd2.ctypes.data_as(N.i64p), vals.ctypes.data_as(N.dblp),
                                 F.ctypes.data_as(N.i64p))
F = int(F[0]); crd1, rp2, crd2, vals = crd1[:F], rp2[:F + 1], crd2[:nnz], vals[:nnz]
ctx = H.Context(0)
Bt = H.DeviceTensor.upload_rowptr(ctx, (I, J, Kd), H.parse_format("dss"), [rp1, rp2], [crd1, crd2], vals)
dev = torch.device("cuda", 0)
R = a.rank
C_d = torch.from_numpy(bench.dense_vals(J * R, 47)).to(dev); D_d = torch.from_numpy(bench.dense_vals(Kd * R, 48)).to(dev)
c_d = torch.from_numpy(bench.dense_vals(Kd, 46)).to(dev)
A_d = torch.empty(I * R, dtype=torch.float64, device=dev); Av = torch.empty(F, dtype=torch.float64, device=dev)
ctx.timing(True)
for _ in range(a.steps):
    H.partition_nonzero(ctx, Bt, 2, 1, host=False)
    if a.kernel == "spmttkrp":
        H.spmttkrp(ctx, Bt, C_d, D_d, R, A_d, pieces=1, stats=False)
    else:
        H.spttv(ctx, Bt, c_d, Av, pieces=1, stats=False)
torch.cuda.synchronize()
print(a.kernel, "leaf ms:", [round(x, 4) for x in ctx.read_timing()], "nnz", nnz, "fibres", F)
ctx.close()
