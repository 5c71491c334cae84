#!/usr/bin/env python3
"""All five BASELINE configs on one B200, each with a full-size parity check
against the CPU restatement (the oracle) and the restatement's time on the
host cores beside it.

  C1  SpMV, uniform 1M x 1M, 10M samples, row split
  C2  SpMM N=32, R-MAT scale 24, nonzero split       (bench.py's headline)
  C3  SDDMM K=128 on the same R-MAT, D stored j-major (dd:1,0)
  C4  SpTTV / SpMTTKRP R=32, power-law 12092 x 9184 x 28818 dss tensor, 10M samples
  C5  SpAdd3, R-MAT B, C/D = B with columns shifted +1/+2, row split

Prints one JSON line per config; values are device-resident throughput
(CUDA events around the op, median of --steps after --warmup).
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
from paper_2207_13901_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--sddmm-scale", type=int, default=24)
ap.add_argument("--no-check", action="store_true")
ap.add_argument("--no-reference", action="store_true",
                help="skip the reference's own plan() + execute() timings (C1, C4)")
args = ap.parse_args()

import torch  # noqa: E402

import oracle_bind as ob  # noqa: E402  (checker + CPU baseline only)
import spd_kernels as SK  # noqa: E402
from paper_2207_13901_b200 import host as H  # noqa: E402

dev = torch.device("cuda", 0)
ctx = H.Context(0)
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
CORES = bench.host_cores()


def timed(fn):
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


GSTREAM = torch.cuda.Stream()
gctx = H.Context(0, stream=GSTREAM.cuda_stream)  # an explicit stream: capturable


def graph_timed(op_on):
    """The op captured once into a CUDA graph (spd_capture_begin/end) and
    replayed: device time without per-launch host overhead."""
    with torch.cuda.stream(GSTREAM):
        op_on(gctx)  # warm: derived indices, scratch sizes
    GSTREAM.synchronize()
    with gctx.capture() as cap:
        op_on(gctx)
    g = cap.graph
    for _ in range(args.warmup):
        g.launch()
    GSTREAM.synchronize()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(GSTREAM)
        g.launch()
        e1.record(GSTREAM)
        GSTREAM.synchronize()
        ts.append(e0.elapsed_time(e1))
    g.close()
    return float(np.median(ts))


def report(name, workload, flops, bytes_, ms, check, cpu_s, extra=None):
    line = {"config": name, "workload": workload, "gflops": flops / ms / 1e6, "ms": ms,
            "effective_gbs": bytes_ / ms / 1e6, "roofline_frac": bytes_ / ms / 1e6 / PEAK,
            "peak_gbs": PEAK, "check": check,
            "cpu_restatement": {"seconds": cpu_s, "gflops": flops / cpu_s / 1e9 if cpu_s else None,
                                "cores": CORES, "kind": "port"}}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)


def ref_timings(kernel, sched, out_fmt, tensors, flops, pieces_list, gpu_out):
    """The reference's own CPU path (oracle/_ref: plan() + execute() in par
    mode, SURVEY 8d "CPU timing beside the GPU"): one run per colour count P
    (its thread pool is min(cores, P), sim.cpp:960-961), output compared with
    the GPU's at 1e-10."""
    if args.no_reference:
        return None
    spec = SK.KERNELS[kernel]
    rows = []
    for P in pieces_list:
        run = ob.RefRun(spec["expr"], sched, P, out_fmt, tensors, mode="par").ok()
        ex = run.exec_seconds()
        rows.append({"pieces": P, "threads": min(CORES, P), "plan_s": run.plan_seconds(), "exec_s": ex,
                     "gflops": flops / ex / 1e9 if ex else None,
                     "matches_gpu": rel_ok(gpu_out, run.output()[1])})
    return {"kind": "reference", "cpu": bench.cpu_model(), "runs": rows}


def rel_ok(got, want, exact=False):
    got = np.asarray(got).reshape(-1)
    want = np.asarray(want).reshape(-1)
    if exact:
        return bool(np.array_equal(got, want))
    return bool(np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300)))


def wrap_csr(n, m, rp, crd, vals):
    rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
    B = H.DeviceTensor.wrap(ctx, (n, m), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                            vals_d.data_ptr(), keep=(rp_d, crd_d, vals_d))
    return B


configs = args.configs.split(",")

if "c1" in configs:
    n = 1_000_000
    rp = np.empty(n + 1, np.int64)
    crd = np.empty(10_000_000, np.int64)
    vals = np.empty(10_000_000)
    nnz = N.synth().syn_uniform_csr(n, n, 10_000_000, 42, 0, rp.ctypes.data_as(N.i64p),
                                     crd.ctypes.data_as(N.i64p), vals.ctypes.data_as(N.dblp))
    crd, vals = crd[:nnz], vals[:nnz]
    x = bench.dense_vals(n, 43)
    B = wrap_csr(n, n, rp, crd, vals)
    x_d = torch.from_numpy(x).to(dev)
    y_d = torch.empty(n, dtype=torch.float64, device=dev)

    def op():
        H.partition_universe(ctx, B, 1, host=False)
        H.spmv(ctx, B, x_d, y_d, pieces=1, stats=False)

    ms = timed(op)
    Bg = H.DeviceTensor.wrap(gctx, (n, n), H.parse_format("ds"), [B._keep[0].data_ptr()], [B._keep[1].data_ptr()],
                             B._keep[2].data_ptr())
    yg = torch.empty(n, dtype=torch.float64, device=dev)

    def op_g(c):
        H.partition_universe(c, Bg, 1, host=False)
        H.spmv(c, Bg, x_d, yg, pieces=1, stats=False)

    ms_graph = graph_timed(op_g)
    t0 = time.time()
    want, _, _ = ob.spmv(rp, crd, vals, x, ob.partition_universe([rp], n, 1))
    cpu = time.time() - t0
    ok = args.no_check or (rel_ok(y_d.cpu().numpy(), want) and rel_ok(yg.cpu().numpy(), want))
    Bh = H.SparseTensor.from_rowptrs((n, n), H.parse_format("ds"), [rp], [crd], vals)
    xh = H.SparseTensor.from_parts((n,), H.parse_format("d"), [H.Level("d", dom=(n,))], x)
    ref = ref_timings("spmv", SK.ROW, "d", {"B": (Bh, "ds"), "c": (xh, "d")}, 2.0 * nnz,
                      sorted({1, 2, 4, 8, CORES}), y_d.cpu().numpy())
    report("C1", "SpMV uniform 1M x 1M, 10M samples (%d nnz), row split" % nnz, 2.0 * nnz,
           8 * (n + 1) + 16 * nnz + 8 * n + 8 * n, ms, ok, cpu, {"ms_cuda_graph": ms_graph, "cpu_reference": ref})

rm = None
if any(c in configs for c in ("c2", "c3", "c5")):
    rm = bench.rmat_csr(args.scale, 10, 42)

if "c2" in configs:
    n, rp, crd, vals = rm
    Nc = 32
    Cv = bench.dense_vals(n * Nc, 43)
    B = wrap_csr(n, n, rp, crd, vals)
    C_d = torch.from_numpy(Cv).to(dev)
    A_d = torch.empty(n * Nc, dtype=torch.float64, device=dev)

    def op():
        H.partition_nonzero(ctx, B, 1, 1, host=False)
        H.spmm(ctx, B, C_d, Nc, A_d, pieces=1, stats=False)

    ms = timed(op)
    t0 = time.time()
    want, _, _ = ob.spmm(rp, crd, vals, Cv, Nc, ob.partition_nonzero([rp], len(crd), 1))
    cpu = time.time() - t0
    ok = args.no_check or rel_ok(A_d.cpu().numpy(), want)
    report("C2", "SpMM N=32, R-MAT scale %d (%d nnz), nonzero split" % (args.scale, len(crd)),
           2.0 * len(crd) * Nc, bench.spmm_bytes(n, len(crd), n, Nc), ms, ok, cpu)
    del C_d, A_d, B

if "c3" in configs:
    n, rp, crd, vals = rm if args.sddmm_scale == args.scale else bench.rmat_csr(args.sddmm_scale, 10, 42)
    K = 128
    B = wrap_csr(n, n, rp, crd, vals)
    Cv = bench.dense_vals(n * K, 44)
    Dv = bench.dense_vals(n * K, 45)  # D(k, j) stored j-major: D[j*K + k]
    C_d = torch.from_numpy(Cv).to(dev)
    D_d = torch.from_numpy(Dv).to(dev)
    A_d = torch.empty(len(crd), dtype=torch.float64, device=dev)

    def op():
        H.partition_nonzero(ctx, B, 1, 1, host=False)
        H.sddmm(ctx, B, C_d, D_d, K, 1, K, A_d, pieces=1, stats=False)

    ms = timed(op)
    t0 = time.time()
    want, _, _ = ob.sddmm(rp, crd, vals, Cv, Dv, K, 1, K, ob.partition_nonzero([rp], len(crd), 1))
    cpu = time.time() - t0
    ok = args.no_check or rel_ok(A_d.cpu().numpy(), want)
    nnz = len(crd)
    report("C3", "SDDMM K=128, R-MAT scale %d (%d nnz), nonzero split" % (args.sddmm_scale, nnz),
           2.0 * nnz * K, 8 * (n + 1) + 16 * nnz + 8 * nnz + 8 * n * K + 8 * n * K, ms, ok, cpu)
    del C_d, D_d, A_d, B

if "c4" in configs:
    I, J, Kd = 12092, 9184, 28818
    S = 10_000_000
    rp1 = np.empty(I + 1, np.int64)
    crd1 = np.empty(S, np.int64)
    rp2 = np.empty(S + 1, np.int64)
    crd2 = np.empty(S, np.int64)
    vals = np.empty(S)
    F = np.zeros(1, np.int64)
    nnz = N.synth().syn_powerlaw_csf(I, J, Kd, S, 4, 0, rp1.ctypes.data_as(N.i64p), crd1.ctypes.data_as(N.i64p),
                                     rp2.ctypes.data_as(N.i64p), crd2.ctypes.data_as(N.i64p),
                                     vals.ctypes.data_as(N.dblp), F.ctypes.data_as(N.i64p))
    F = int(F[0])
    crd1, rp2, crd2, vals = crd1[:F], rp2[:F + 1], crd2[:nnz], vals[:nnz]
    t = H.SparseTensor.from_rowptrs((I, J, Kd), H.parse_format("dss"), [rp1, rp2], [crd1, crd2], vals)
    Bt = H.DeviceTensor.upload_rowptr(ctx, (I, J, Kd), H.parse_format("dss"), [rp1, rp2], [crd1, crd2], vals)
    c = bench.dense_vals(Kd, 46)
    c_d = torch.from_numpy(c).to(dev)
    Av = torch.empty(F, dtype=torch.float64, device=dev)

    def op_ttv():
        H.partition_nonzero(ctx, Bt, 2, 1, host=False)
        H.spttv(ctx, Bt, c_d, Av, pieces=1, stats=False)

    ms = timed(op_ttv)
    Btg = H.DeviceTensor.upload_rowptr(gctx, (I, J, Kd), H.parse_format("dss"), [rp1, rp2], [crd1, crd2], vals)
    Avg = torch.empty(F, dtype=torch.float64, device=dev)

    def op_ttv_g(c):
        H.partition_nonzero(c, Btg, 2, 1, host=False)
        H.spttv(c, Btg, c_d, Avg, pieces=1, stats=False)

    ms_graph = graph_timed(op_ttv_g)
    t0 = time.time()
    want, _, _ = ob.spttv(rp1, crd1, rp2, crd2, vals, c, ob.partition_nonzero([rp1, rp2], nnz, 1))
    cpu = time.time() - t0
    ok = args.no_check or (rel_ok(Av.cpu().numpy(), want) and rel_ok(Avg.cpu().numpy(), want))
    ch = H.SparseTensor.from_parts((Kd,), H.parse_format("d"), [H.Level("d", dom=(Kd,))], c)
    ref = ref_timings("spttv", SK.KERNELS["spttv"]["nonzero"], "ds", {"B": (t, "dss"), "c": (ch, "d")}, 2.0 * nnz,
                      sorted({8, CORES}), Av.cpu().numpy())
    report("C4-SpTTV", "SpTTV, %dx%dx%d power-law dss, %d nnz, %d fibres, nonzero split" % (I, J, Kd, nnz, F),
           2.0 * nnz, 8 * (I + 1) + 8 * F + 8 * (F + 1) + 16 * nnz + 8 * Kd + 8 * F, ms, ok, cpu,
           {"ms_cuda_graph": ms_graph, "cpu_reference": ref})
    R = 32
    Cm = bench.dense_vals(J * R, 47)
    Dm = bench.dense_vals(Kd * R, 48)
    C_d = torch.from_numpy(Cm).to(dev)
    D_d = torch.from_numpy(Dm).to(dev)
    A_d = torch.empty(I * R, dtype=torch.float64, device=dev)

    def op_mttkrp():
        H.partition_nonzero(ctx, Bt, 2, 1, host=False)
        H.spmttkrp(ctx, Bt, C_d, D_d, R, A_d, pieces=1, stats=False)

    ms = timed(op_mttkrp)
    A_g = torch.empty(I * R, dtype=torch.float64, device=dev)

    def op_mttkrp_g(c):
        H.partition_nonzero(c, Btg, 2, 1, host=False)
        H.spmttkrp(c, Btg, C_d, D_d, R, A_g, pieces=1, stats=False)

    ms_graph = graph_timed(op_mttkrp_g)
    t0 = time.time()
    want, _, _ = ob.spmttkrp(rp1, crd1, rp2, crd2, vals, Cm, Dm, R, ob.partition_nonzero([rp1, rp2], nnz, 1))
    cpu = time.time() - t0
    ok = args.no_check or (rel_ok(A_d.cpu().numpy(), want) and rel_ok(A_g.cpu().numpy(), want))
    Ch = H.SparseTensor.from_parts((J, R), H.parse_format("dd"), [H.Level("d", dom=(J, R))], Cm)
    Dh = H.SparseTensor.from_parts((Kd, R), H.parse_format("dd"), [H.Level("d", dom=(Kd, R))], Dm)
    ref = ref_timings("spmttkrp", SK.KERNELS["spmttkrp"]["nonzero"], "dd",
                      {"B": (t, "dss"), "C": (Ch, "dd"), "D": (Dh, "dd")}, 3.0 * nnz * R, [CORES],
                      A_d.cpu().numpy())
    report("C4-SpMTTKRP", "SpMTTKRP R=32, same tensor, nonzero split", 3.0 * nnz * R,
           8 * (I + 1) + 8 * F + 8 * (F + 1) + 16 * nnz + 8 * (J + Kd + I) * R, ms, ok, cpu,
           {"ms_cuda_graph": ms_graph, "cpu_reference": ref})

if "c5" in configs:
    n, rp, crd, vals = rm
    ops = [(rp, crd, vals)]
    for shift in (1, 2):
        rps = np.empty(n + 1, np.int64)
        # shifted copies: same generator, columns + shift (mod n), re-sorted per row
        e = 10 * n
        cs = np.empty(e, np.int64)
        vs = np.empty(e)
        nz = N.synth().syn_rmat_csr(args.scale, e, bench.A_RMAT, bench.B_RMAT, bench.C_RMAT, 42, 0, 0, shift,
                                    rps.ctypes.data_as(N.i64p), cs.ctypes.data_as(N.i64p), vs.ctypes.data_as(N.dblp))
        ops.append((rps, cs[:nz], vs[:nz]))
    Bs = [wrap_csr(n, n, *o) for o in ops]

    def op():
        H.partition_universe(ctx, Bs[0], 8, host=False)
        A, _ = H.spadd3(ctx, Bs[0], Bs[1], Bs[2], pieces=8, stats=False)
        return A

    for _ in range(args.warmup):
        op().close()
    torch.cuda.synchronize()
    ts = []
    last = None
    for _ in range(args.steps):
        if last is not None:  # the previous output goes back to the pool first
            last.close()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A = op()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        last = A
    ms = float(np.median(ts))
    At = last.download()
    t0 = time.time()
    want = ob.spadd3(ops)
    cpu = time.time() - t0
    ok = args.no_check or (np.array_equal(At.levels[1].rowptr(), want[0]) and np.array_equal(At.levels[1].crd, want[1])
                           and np.array_equal(At.vals, want[2]))
    nin = sum(len(o[1]) for o in ops)
    nA = len(want[1])
    report("C5", "SpAdd3 R-MAT scale %d + shifted copies (%d input nnz -> %d), row split P=8" % (args.scale, nin, nA),
           float(nin), sum(8 * (n + 1) + 16 * len(o[1]) for o in ops) + 8 * (n + 1) + 16 * nA, ms, ok, cpu,
           {"pattern_bit_exact": bool(ok)})

ctx.close()
