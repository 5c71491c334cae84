#!/usr/bin/env python3
"""The five BASELINE configs on N GPUs of one box, one process per GPU.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/mgpu_configs.py

Rank 0 generates every input on the host (the same generators and seeds as
scripts/bench_configs.py) and broadcasts it over NVLink; each GPU runs the
colour equal to its rank of a P = N partition (C1 row split, C2-C4 nonzero
split, C5 row split -- the schedules of SURVEY 8d), rows cut between GPUs are
combined inside the backend over NCCL.  Time = CUDA events on each rank,
median of --steps, max over ranks.

Check: rank 0 also runs ALL N colours of the same partition on its own GPU
(no communicator involved) and compares them with the distributed result
gathered from the ranks' owned output ranges -- bit-exact, because the
combine order is the colour order in both.  The full-size comparison with
the CPU oracle at P = 1 is scripts/bench_configs.py; small multi-GPU cases
against the oracle are scripts/mgpu_check.py.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2207_13901_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--scale", type=int, default=24)
args = ap.parse_args()

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2207_13901_b200 import host as H  # noqa: E402
from paper_2207_13901_b200.distributed import init_comm, owned_rows  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = H.Context(local)
init_comm(ctx, dist, rank, world, dev)
P = world
PEAK = 6650.0
if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", PEAK)
if rank == 0:
    N.synth().syn_set_threads(bench.host_cores())


def bcast(arr, dtype):
    """numpy array on rank 0 -> identical device tensor on every rank."""
    n = torch.tensor([arr.size if rank == 0 else 0], dtype=torch.int64, device=dev)
    dist.broadcast(n, 0)
    t = torch.from_numpy(arr).to(dev) if rank == 0 else torch.empty(int(n[0]), dtype=dtype, device=dev)
    dist.broadcast(t, 0)
    return t


def timed(fn):
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = torch.tensor([float(np.median(ts))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def gather_ranges(buf, ranges, width):
    """Rank r's rows ranges[r] of `buf` (rows x width) assembled on rank 0."""
    out = torch.zeros_like(buf) if rank == 0 else None
    v = buf.view(-1, width)
    for r, (lo, hi) in enumerate(ranges):
        if lo > hi:
            continue
        if r == 0 and rank == 0:
            out.view(-1, width)[lo:hi + 1] = v[lo:hi + 1]
        elif rank == r:
            dist.send(v[lo:hi + 1].contiguous(), 0)
        elif rank == 0:
            tmp = torch.empty((hi - lo + 1, width), dtype=buf.dtype, device=dev)
            dist.recv(tmp, r)
            out.view(-1, width)[lo:hi + 1] = tmp
    return out


def report(name, workload, flops, bytes_, ms, check):
    if rank == 0:
        print(json.dumps({"config": name, "workload": workload, "n_gpus": world, "gflops": flops / ms / 1e6,
                          "ms": ms, "effective_gbs": bytes_ / ms / 1e6,
                          "roofline_frac_per_gpu": bytes_ / ms / 1e6 / PEAK / world, "peak_gbs": PEAK,
                          "check_vs_single_gpu_all_colours": check}), flush=True)


def wrap(n, m, rp_d, crd_d, vals_d):
    return H.DeviceTensor.wrap(ctx, (n, m), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                               vals_d.data_ptr(), keep=(rp_d, crd_d, vals_d))


def same(a, b):
    return bool(torch.equal(a, b)) if rank == 0 else None


configs = args.configs.split(",")

if "c1" in configs:
    n, S = 1_000_000, 10_000_000
    if rank == 0:
        rp = np.empty(n + 1, np.int64)
        crd = np.empty(S, np.int64)
        vals = np.empty(S)
        nnz = N.synth().syn_uniform_csr(n, n, S, 42, 0, rp.ctypes.data_as(N.i64p), crd.ctypes.data_as(N.i64p),
                                         vals.ctypes.data_as(N.dblp))
        crd, vals, x = crd[:nnz], vals[:nnz], bench.dense_vals(n, 43)
    else:
        rp = crd = vals = x = None
    rp_d, crd_d, vals_d = bcast(rp, torch.int64), bcast(crd, torch.int64), bcast(vals, torch.float64)
    x_d = bcast(x, torch.float64)
    nnz = crd_d.numel()
    B = wrap(n, n, rp_d, crd_d, vals_d)
    y_d = torch.zeros(n, dtype=torch.float64, device=dev)
    cols = H.partition_universe(ctx, B, P)

    def op():
        H.partition_universe(ctx, B, P, host=False)
        H.spmv(ctx, B, x_d, y_d, first=rank, count=1, pieces=P, stats=False)

    ms = timed(op)
    got = gather_ranges(y_d, owned_rows(cols, rp_d.cpu().numpy(), "row", n), 1)
    ok = None
    if rank == 0:
        ref = torch.zeros_like(y_d)
        H.partition_universe(ctx, B, P, host=False)
        H.spmv(ctx, B, x_d, ref, first=0, count=P, pieces=P, stats=False)
        ok = same(got, ref)
    report("C1", "SpMV uniform 1M x 1M (%d nnz), row split P=%d" % (nnz, P), 2.0 * nnz,
           8 * (n + 1) + 16 * nnz + 8 * n + 8 * n, ms, ok)
    B.close()
    del rp_d, crd_d, vals_d, x_d, y_d

if any(c in configs for c in ("c2", "c3", "c5")):
    if rank == 0:
        n, rp, crd, vals = bench.rmat_csr(args.scale, 10, 42)
    else:
        rp = crd = vals = None
    rm = [bcast(rp, torch.int64), bcast(crd, torch.int64), bcast(vals, torch.float64)]
    n = rm[0].numel() - 1
    nnz = rm[1].numel()
    rp_h = rm[0].cpu().numpy()

if "c2" in configs:
    Nc = 32
    B = wrap(n, n, *rm)
    C_d = bcast(bench.dense_vals(n * Nc, 43) if rank == 0 else None, torch.float64)
    A_d = torch.empty(n * Nc, dtype=torch.float64, device=dev)
    cols = H.partition_nonzero(ctx, B, 1, P)

    def op():
        H.partition_nonzero(ctx, B, 1, P, host=False)
        H.spmm(ctx, B, C_d, Nc, A_d, first=rank, count=1, pieces=P, stats=False)

    ms = timed(op)
    got = gather_ranges(A_d, owned_rows(cols, rp_h, "nonzero", n), Nc)
    ok = None
    if rank == 0:
        ref = torch.empty_like(A_d)
        H.partition_nonzero(ctx, B, 1, P, host=False)
        H.spmm(ctx, B, C_d, Nc, ref, first=0, count=P, pieces=P, stats=False)
        ok = same(got, ref)
        del ref
    del got
    report("C2", "SpMM N=32, R-MAT scale %d (%d nnz), nonzero split P=%d" % (args.scale, nnz, P),
           2.0 * nnz * Nc, bench.spmm_bytes(n, nnz, n, Nc), ms, ok)
    B.close()
    del C_d, A_d

if "c3" in configs:
    K = 128
    B = wrap(n, n, *rm)
    C_d = bcast(bench.dense_vals(n * K, 44) if rank == 0 else None, torch.float64)
    D_d = bcast(bench.dense_vals(n * K, 45) if rank == 0 else None, torch.float64)
    A_d = torch.zeros(nnz, dtype=torch.float64, device=dev)
    cols = H.partition_nonzero(ctx, B, 1, P)

    def op():
        H.partition_nonzero(ctx, B, 1, P, host=False)
        H.sddmm(ctx, B, C_d, D_d, K, 1, K, A_d, first=rank, count=1, pieces=P, stats=False)

    ms = timed(op)
    # the output lives on B's pattern: colour c owns its positions q_c
    got = gather_ranges(A_d, [tuple(c.q) for c in cols], 1)
    ok = None
    if rank == 0:
        ref = torch.zeros_like(A_d)
        H.partition_nonzero(ctx, B, 1, P, host=False)
        H.sddmm(ctx, B, C_d, D_d, K, 1, K, ref, first=0, count=P, pieces=P, stats=False)
        ok = same(got, ref)
        del ref
    del got
    report("C3", "SDDMM K=128, R-MAT scale %d (%d nnz), nonzero split P=%d" % (args.scale, nnz, P),
           2.0 * nnz * K, 8 * (n + 1) + 16 * nnz + 8 * nnz + 8 * n * K + 8 * n * K, ms, ok)
    B.close()
    del C_d, D_d, A_d

if "c4" in configs:
    I, J, Kd, S = 12092, 9184, 28818, 10_000_000
    if rank == 0:
        rp1 = np.empty(I + 1, np.int64)
        crd1 = np.empty(S, np.int64)
        rp2 = np.empty(S + 1, np.int64)
        crd2 = np.empty(S, np.int64)
        vals = np.empty(S)
        F = np.zeros(1, np.int64)
        nz = N.synth().syn_powerlaw_csf(I, J, Kd, S, 4, 0, rp1.ctypes.data_as(N.i64p), crd1.ctypes.data_as(N.i64p),
                                        rp2.ctypes.data_as(N.i64p), crd2.ctypes.data_as(N.i64p),
                                        vals.ctypes.data_as(N.dblp), F.ctypes.data_as(N.i64p))
        F = int(F[0])
        crd1, rp2, crd2, vals = crd1[:F], rp2[:F + 1], crd2[:nz], vals[:nz]
        arrs = [rp1, crd1, rp2, crd2, vals]
    else:
        arrs = [None] * 5
    rp1_d, crd1_d, rp2_d, crd2_d = (bcast(a, torch.int64) for a in arrs[:4])
    vals_d = bcast(arrs[4], torch.float64)
    F, nz = crd1_d.numel(), crd2_d.numel()
    Bt = H.DeviceTensor.wrap(ctx, (I, J, Kd), H.parse_format("dss"), [rp1_d.data_ptr(), rp2_d.data_ptr()],
                             [crd1_d.data_ptr(), crd2_d.data_ptr()], vals_d.data_ptr(),
                             keep=(rp1_d, crd1_d, rp2_d, crd2_d, vals_d))
    rp1_h, rp2_h = rp1_d.cpu().numpy(), rp2_d.cpu().numpy()
    cols = H.partition_nonzero(ctx, Bt, 2, P)
    c_d = bcast(bench.dense_vals(Kd, 46) if rank == 0 else None, torch.float64)
    Av = torch.zeros(F, dtype=torch.float64, device=dev)

    def op_ttv():
        H.partition_nonzero(ctx, Bt, 2, P, host=False)
        H.spttv(ctx, Bt, c_d, Av, first=rank, count=1, pieces=P, stats=False)

    ms = timed(op_ttv)
    got = gather_ranges(Av, owned_rows(cols, rp2_h, "nonzero", F), 1)
    ok = None
    if rank == 0:
        ref = torch.zeros_like(Av)
        H.partition_nonzero(ctx, Bt, 2, P, host=False)
        H.spttv(ctx, Bt, c_d, ref, first=0, count=P, pieces=P, stats=False)
        ok = same(got, ref)
    report("C4-SpTTV", "SpTTV %dx%dx%d power-law dss (%d nnz, %d fibres), nonzero split P=%d" % (I, J, Kd, nz, F, P),
           2.0 * nz, 8 * (I + 1) + 8 * F + 8 * (F + 1) + 16 * nz + 8 * Kd + 8 * F, ms, ok)
    R = 32
    C_d = bcast(bench.dense_vals(J * R, 47) if rank == 0 else None, torch.float64)
    D_d = bcast(bench.dense_vals(Kd * R, 48) if rank == 0 else None, torch.float64)
    A_d = torch.zeros(I * R, dtype=torch.float64, device=dev)

    def op_mttkrp():
        H.partition_nonzero(ctx, Bt, 2, P, host=False)
        H.spmttkrp(ctx, Bt, C_d, D_d, R, A_d, first=rank, count=1, pieces=P, stats=False)

    ms = timed(op_mttkrp)
    leaf_rp = rp2_h[rp1_h]  # rows i -> leaf positions
    got = gather_ranges(A_d, owned_rows(cols, leaf_rp, "nonzero", I), R)
    ok = None
    if rank == 0:
        ref = torch.zeros_like(A_d)
        H.partition_nonzero(ctx, Bt, 2, P, host=False)
        H.spmttkrp(ctx, Bt, C_d, D_d, R, ref, first=0, count=P, pieces=P, stats=False)
        ok = same(got, ref)
    report("C4-SpMTTKRP", "SpMTTKRP R=32, same tensor, nonzero split P=%d" % P, 3.0 * nz * R,
           8 * (I + 1) + 8 * F + 8 * (F + 1) + 16 * nz + 8 * (J + Kd + I) * R, ms, ok)
    Bt.close()

if "c5" in configs:
    ops = [wrap(n, n, *rm)]
    sizes = [nnz]
    for shift in (1, 2):
        if rank == 0:
            e = 10 * n
            rps, cs, vs = np.empty(n + 1, np.int64), np.empty(e, np.int64), np.empty(e)
            nzs = N.synth().syn_rmat_csr(args.scale, e, bench.A_RMAT, bench.B_RMAT, bench.C_RMAT, 42, 0, 0, shift,
                                         rps.ctypes.data_as(N.i64p), cs.ctypes.data_as(N.i64p),
                                         vs.ctypes.data_as(N.dblp))
            arrs = [rps, cs[:nzs], vs[:nzs]]
        else:
            arrs = [None] * 3
        crd_s = bcast(arrs[1], torch.int64)
        sizes.append(crd_s.numel())
        ops.append(wrap(n, n, bcast(arrs[0], torch.int64), crd_s, bcast(arrs[2], torch.float64)))
    state = {}

    def op():
        if "A" in state:
            state.pop("A").close()
        H.partition_universe(ctx, ops[0], P, host=False)
        state["A"], _ = H.spadd3(ctx, ops[0], ops[1], ops[2], first=rank, count=1, pieces=P, stats=False)

    ms = timed(op)
    full = state["A"].gather_rows(0)
    ok = None
    if rank == 0:
        H.partition_universe(ctx, ops[0], P, host=False)
        ref, _ = H.spadd3(ctx, ops[0], ops[1], ops[2], first=0, count=P, pieces=P, stats=False)
        g, w = full.download(), ref.download()
        ok = bool(np.array_equal(g.levels[1].rowptr(), w.levels[1].rowptr())
                  and np.array_equal(g.levels[1].crd, w.levels[1].crd) and np.array_equal(g.vals, w.vals))
        nA = len(w.levels[1].crd)
        full.close()
        ref.close()
    else:
        nA = 0
    report("C5", "SpAdd3 R-MAT scale %d + shifted copies (%d input nnz -> %d), row split P=%d"
           % (args.scale, sum(sizes), nA, P), float(sum(sizes)),
           sum(8 * (n + 1) + 16 * z for z in sizes) + 8 * (n + 1) + 16 * nA, ms, ok)

ctx.close()
dist.destroy_process_group()
