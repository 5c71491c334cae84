#!/usr/bin/env python3
"""Experiment (measurement only): how fast would a hot/cold two-pass SpMM be?

Splits the C2 R-MAT matrix B into B_hot (entries whose column is among the H
most referenced ones) and B_cold (the rest), two ordinary CSR matrices of the
same shape, and times the production SpMM leaf on B, on B_hot and on B_cold
(each writing its own output).  leaf(B_hot) + leaf(B_cold) bounds a two-pass
design from below (it omits the read-back of rows holding both kinds)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_13901_b200 import host as H  # noqa: E402

dev = torch.device("cuda", 0)
n, rp, crd, vals = bench.rmat_csr(24, 10, 42)
N = 32
rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
C_d = torch.from_numpy(bench.dense_vals(n * N, 43)).to(dev)
A_d = torch.empty(n * N, dtype=torch.float64, device=dev)
A2_d = torch.empty(n * N, dtype=torch.float64, device=dev)
ctx = H.Context(0)
fmt = H.parse_format("ds")
rows = torch.repeat_interleave(torch.arange(n, device=dev), rp_d[1:] - rp_d[:-1])
counts = torch.bincount(crd_d, minlength=n)
sc = torch.sort(counts, descending=True).values


def timed(B, out, reps=6):
    ctx.timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        H.partition_nonzero(ctx, B, 1, 1, host=False)
        H.spmm(ctx, B, C_d, N, out, pieces=1, stats=False)
    torch.cuda.synchronize()
    ctx.read_timing()
    ev0.record()
    for _ in range(reps):
        H.partition_nonzero(ctx, B, 1, 1, host=False)
        H.spmm(ctx, B, C_d, N, out, pieces=1, stats=False)
    ev1.record()
    torch.cuda.synchronize()
    lm = ctx.read_timing()
    ctx.timing(False)
    return ev0.elapsed_time(ev1) / reps, float(np.mean(lm))


def sub(mask):
    r = rows[mask]
    cnt = torch.bincount(r, minlength=n)
    rpx = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rpx[1:] = torch.cumsum(cnt, 0)
    c = crd_d[mask].contiguous()
    v = vals_d[mask].contiguous()
    return H.DeviceTensor.wrap(ctx, (n, n), fmt, [rpx.data_ptr()], [c.data_ptr()], v.data_ptr(),
                               keep=(rpx, c, v)), int(c.numel())


Bf = H.DeviceTensor.wrap(ctx, (n, n), fmt, [rp_d.data_ptr()], [crd_d.data_ptr()], vals_d.data_ptr())
step, leaf = timed(Bf, A_d)
print(f"full B: nnz {len(crd)} step {step:.3f} ms leaf {leaf:.3f} ms", flush=True)
for Hn in (100000, 160000, 200000, 240000, 280000):
    thr = int(sc[Hn - 1])
    hot = counts[crd_d] >= thr
    Bh, nh = sub(hot)
    Bc, nc = sub(~hot)
    sh, lh = timed(Bh, A_d)
    scd, lc = timed(Bc, A2_d)
    both = int(((torch.bincount(rows[hot], minlength=n) > 0) & (torch.bincount(rows[~hot], minlength=n) > 0)).sum())
    print(f"H={Hn} thr={thr} hot nnz {nh} ({nh / len(crd):.3f}) cold nnz {nc}: hot step {sh:.3f} leaf {lh:.3f} | "
          f"cold step {scd:.3f} leaf {lc:.3f} | sum steps {sh + scd:.3f} leaves {lh + lc:.3f} ms; both rows {both}",
          flush=True)
    Bh.close()
    Bc.close()
ctx.close()
