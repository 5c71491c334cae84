#!/usr/bin/env python3
"""Vendor yardstick (measurement only, never on the product path): cuSPARSE
SpMV and SpMM (through torch.sparse CSR, which calls cusparseSpMV /
cusparseSpMM) on the C2 R-MAT CSR, timed like the bench leaf (CUDA events,
median of --steps after --warmup) next to this backend's leaf on the same
inputs, with the outputs compared (1e-10 relative)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()

import torch  # noqa: E402

from paper_2207_13901_b200 import host as H  # noqa: E402

dev = torch.device("cuda", 0)
n, rp, crd, vals = bench.rmat_csr(a.scale, 10, 42)
nnz = len(crd)
rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
x = torch.from_numpy(bench.dense_vals(n, 44)).to(dev)
N = 32
C = torch.from_numpy(bench.dense_vals(n * N, 43)).to(dev).view(n, N)


def timed(fn):
    for _ in range(a.warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def rel(got, want):
    got, want = got.reshape(-1).double(), want.reshape(-1).double()
    return float(((got - want).abs() / want.abs().clamp_min(1e-300)).max())


out = {"workload": f"R-MAT scale {a.scale}, {n} rows, {nnz} nnz, fp64", "steps": a.steps}
Acsr = torch.sparse_csr_tensor(rp_d, crd_d, vals_d, size=(n, n))
res = {}
keep = {}
res["spmv_cusparse_ms"] = timed(lambda: keep.__setitem__("y", torch.mv(Acsr, x)))
res["spmm_cusparse_ms"] = timed(lambda: keep.__setitem__("Y", torch.sparse.mm(Acsr, C)))
y_cs, Y_cs = keep["y"], keep["Y"]
ctx = H.Context(0)
B = H.DeviceTensor.wrap(ctx, (n, n), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()], vals_d.data_ptr())
y = torch.empty(n, dtype=torch.float64, device=dev)
Y = torch.empty(n * N, dtype=torch.float64, device=dev)


def ours_spmv():
    H.partition_nonzero(ctx, B, 1, 1, host=False)
    H.spmv(ctx, B, x, y, pieces=1, stats=False)


def ours_spmm():
    H.partition_nonzero(ctx, B, 1, 1, host=False)
    H.spmm(ctx, B, C, N, Y, pieces=1, stats=False)


res["spmv_ours_ms"] = timed(ours_spmv)
res["spmm_ours_ms"] = timed(ours_spmm)
res["spmv_max_rel_diff"] = rel(y, y_cs)
res["spmm_max_rel_diff"] = rel(Y, Y_cs)
sb = 8 * (n + 1) + 16 * nnz + 16 * n
mb = bench.spmm_bytes(n, nnz, n, N)
for k in ("spmv", "spmm"):
    by = sb if k == "spmv" else mb
    for who in ("cusparse", "ours"):
        ms = res[f"{k}_{who}_ms"]
        res[f"{k}_{who}_gbs"] = by / (ms * 1e-3) / 1e9
        res[f"{k}_{who}_gflops"] = (2.0 * nnz * (1 if k == "spmv" else N)) / (ms * 1e-3) / 1e9
out.update(res)
out["note"] = ("whole op time per call (ours: partition step + leaf + combine; cuSPARSE: torch.mv / "
               "torch.sparse.mm on a CSR tensor, output allocated by torch's caching allocator); same "
               "inputs, same device")
print(json.dumps(out))
B.close()
ctx.close()
