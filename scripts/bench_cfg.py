"""The BASELINE configs besides bench.py's C2 headline, measured inside the
same bench run (bench.py imports this; it is not a stand-alone script).

Each leg returns one JSON object with the headline line's keys: `value` /
`unit` / `ms_per_step` (device-resident inputs, one step = the partition step
+ the leaf + the combine), `roofline` of the leaf kernel (algorithmic bytes
per launch, over the leaf's CUDA-event time), `e2e` (the same
metric through the C-ABI with host buffers: the sparse operand re-staged from
pinned host memory as the reference stores it, dense operands copied H2D,
the output copied D2H, every step) and, on rank 0 at N = 1, `cpu_baseline`:
the reference's own plan() + execute() (oracle/_ref, par mode, every host
thread) at full size where it fits (C1, C4), else on a bounded R-MAT sample.

  C1          SpMV, uniform 1M x 1M, 10M samples, row split
  SpMV-RMAT   SpMV on the C2 R-MAT (scale 24), nonzero split
  C3          SDDMM K=128 on the R-MAT, D stored j-major (dd:1,0), nonzero split
  C4-SpTTV    SpTTV on a 12092 x 9184 x 28818 power-law dss tensor, nonzero split
  C4-SpMTTKRP SpMTTKRP R=32 on the same tensor, nonzero split
  C5          SpAdd3 of the R-MAT and two column-shifted copies, row split P=8

At N > 1 every GPU runs the colour equal to its rank of a P = N partition
(C5: P = 8 colours over the N GPUs when N divides 8 is not required -- it is
P = N), time = max over ranks; e2e and the CPU baseline are N = 1 only.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L2_GATHER_PEAK_GBS = 20776.5  # profiles/r02_probe_gather.jsonl, uniform_16MB, best variant


def _ob():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob  # the CPU baseline only (never on the measured path)
    return ob


def _sk():
    """The six kernels' expressions and schedules as the reference states
    them (tests/spd_kernels.py), for the CPU baseline's reference runs."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import spd_kernels
    return spd_kernels


class Env:
    def __init__(self, ctx, torch, dev, rank, world, args, peak, host_cores, cpu_model):
        self.ctx, self.torch, self.dev = ctx, torch, dev
        self.rank, self.world, self.args, self.peak = rank, world, args, peak
        self.host_cores, self.cpu_model = host_cores, cpu_model
        import torch.distributed as dist
        self.dist = dist

    def maxr(self, vals):
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]

    def bcast(self, arr, dtype):
        """numpy array on rank 0 -> device tensor on every rank (NVLink)."""
        torch = self.torch
        if self.world == 1:
            return torch.from_numpy(arr).to(self.dev)
        n = torch.tensor([arr.size if self.rank == 0 else 0], dtype=torch.int64, device=self.dev)
        self.dist.broadcast(n, 0)
        t = torch.from_numpy(arr).to(self.dev) if self.rank == 0 else torch.empty(int(n[0]), dtype=dtype,
                                                                                    device=self.dev)
        self.dist.broadcast(t, 0)
        return t

    def colours(self):
        """(first, count, pieces) of this GPU's share of a P = N partition."""
        return (self.rank, 1, self.world) if self.world > 1 else (0, 1, 1)


def _block_times(env, step):
    """Median leaf time of a few steps on every GPU (all-gathered): the
    measurement the colour-block refinement re-weights by."""
    torch = env.torch
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    env.ctx.timing(True)
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    env.ctx.timing(False)
    t = torch.tensor([float(np.median(env.ctx.read_timing()))], dtype=torch.float64, device=env.dev)
    allt = [torch.zeros_like(t) for _ in range(env.world)]
    env.dist.all_gather(allt, t)
    return [float(x[0]) for x in allt]


def measure(env, step, kernel_share=1.0):
    """W warm-up steps, then K timed steps bracketed by barrier + synchronize,
    CUDA events on the launching stream; the leaf's own CUDA-event pairs
    (spd_context_timing) give the roofline time.  Max over ranks."""
    torch, ctx, args = env.torch, env.ctx, env.args
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ctx.read_timing()
    ctx.timing(True)
    l0 = ctx.launches()
    if env.world > 1:
        env.dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if env.world > 1:
        env.dist.barrier()
    nl = ctx.launches() - l0
    lm = ctx.read_timing()
    ctx.timing(False)
    ms = e0.elapsed_time(e1) / args.steps
    leaf = float(np.mean(lm[-args.steps:])) if lm else 0.0
    ms, leaf = env.maxr([ms, leaf])
    return ms, leaf, nl


def roofline(env, bytes_per_launch, leaf_ms, kernel, traffic=None):
    ach = bytes_per_launch / (leaf_ms * 1e-3) / 1e9 if leaf_ms > 0 else None
    return {"bound": "hbm", "achieved": ach, "peak": env.peak, "unit": "GB/s",
            "frac": ach / env.peak if ach else None, "traffic": traffic, "kernel": kernel,
            "bytes_per_launch": bytes_per_launch, "leaf_ms": leaf_ms, "peak_source": "measured"}


def cpu_reference(env, kernel, schedule, out_fmt, tensors, flops, pieces, what):
    """The reference's plan() + execute() (par mode; its pool is min(cores,
    tasks) threads, sim.cpp:958-961) on host buffers: the CPU baseline."""
    ob = _ob()
    SK = _sk()
    spec = SK.KERNELS[kernel]
    run = ob.RefRun(spec["expr"], schedule, pieces, out_fmt, tensors, mode="par").ok()
    t = run.exec_seconds() + run.plan_seconds()
    return {"value": flops / t / 1e9, "unit": "GFLOP/s", "cores": min(env.host_cores, pieces), "kind": "reference",
            "sample": f"{what}; reference plan() {run.plan_seconds():.2f} s + execute() {run.exec_seconds():.2f} s, "
                      f"{pieces} colours, par mode, {env.cpu_model}"}, run


def e2e_loop(env, one_step, flops, h2d, d2h):
    """The metric end to end: `one_step` does this step's H2D + op + D2H;
    timed over --steps after 2 warm steps, host clock around synchronised
    steps (max over ranks)."""
    torch, args = env.torch, env.args
    one_step()
    one_step()
    torch.cuda.synchronize()
    if env.world > 1:
        env.dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.steps
    dt = env.maxr([dt])[0]
    return {"value": flops / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3}


def mgpu_check(env, H, out_d, width, span, reference):
    """N > 1: this rank's share of the distributed output (`span` = (lo, hi)
    rows / fibres / positions it stores, `width` values each) is sent to rank
    0 and compared bit-exactly with `reference()` -- rank 0 running every
    colour of the same partition on its own GPU without a communicator (same
    combine order, same bits).  Outside the timed region."""
    torch, dist = env.torch, env.dist
    spans = [None] * env.world
    dist.all_gather_object(spans, tuple(int(x) for x in span))
    ref = reference() if env.rank == 0 else None
    ok = True
    for r, (lo, hi) in enumerate(spans):
        if lo > hi:
            continue
        if r == env.rank == 0:
            ok = ok and bool(torch.equal(out_d[lo * width:(hi + 1) * width], ref[lo * width:(hi + 1) * width]))
        elif env.rank == r:
            dist.send(out_d[lo * width:(hi + 1) * width].contiguous(), 0)
        elif env.rank == 0:
            buf = torch.empty((hi - lo + 1) * width, dtype=out_d.dtype, device=env.dev)
            dist.recv(buf, r)
            ok = ok and bool(torch.equal(buf, ref[lo * width:(hi + 1) * width]))
    t = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device=env.dev)
    dist.broadcast(t, 0)
    return {"bit_exact_vs_one_gpu": bool(t[0] > 0.5),
            "what": "this config's distributed output (each rank's owned share) vs all colours of the same "
                    "partition on rank 0's GPU"}


def _ctx1(env, H):
    """A communicator-free context on this GPU (every colour locally)."""
    return H.Context(env.dev.index)


def _pinned(torch, arr):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.pin_memory()


def _csr_host(H, n, m, rp, crd, vals):
    return H.SparseTensor.from_rowptrs((n, m), H.parse_format("ds"), [rp], [crd], vals)


def _restager(env, H, dims, fmt, rowptrs, crds, vals):
    """A device tensor re-staged every step from pinned host arrays in the
    reference's storage (inclusive pos pairs per compressed level, crd, vals)
    through spd_tensor_upload / spd_tensor_restage.  Returns (step_fn, bytes)."""
    from paper_2207_13901_b200 import _native as NN
    torch = env.torch
    nl = len(rowptrs) + 1
    pairs = [None] + [_pinned(torch, np.stack([r[:-1], r[1:] - 1], axis=1).reshape(-1)) for r in rowptrs]
    crd_h = [None] + [_pinned(torch, c) for c in crds]
    vals_h = _pinned(torch, vals)
    # levels: a dense top then compressed levels (ds / dss)
    pos_pp = (NN.i64p * nl)(*([None] + [C.cast(p.data_ptr(), NN.i64p) for p in pairs[1:]]))
    crd_pp = (NN.i64p * nl)(*([None] + [C.cast(c.data_ptr(), NN.i64p) for c in crd_h[1:]]))
    d = (C.c_int64 * len(dims))(*dims)
    kinds = (C.c_int * len(dims))(*([0] + [1] * (len(dims) - 1)))
    mo = (C.c_int * len(dims))(*range(len(dims)))
    state = {"t": None}
    nbytes = sum(p.numel() * 8 for p in pairs[1:]) + sum(c.numel() * 8 for c in crd_h[1:]) + vals_h.numel() * 8

    def step():
        if state["t"] is None:
            h = C.c_void_p()
            NN.check(NN.lib().spd_tensor_upload(env.ctx.h, len(dims), d, kinds, mo, pos_pp, crd_pp,
                                                C.cast(vals_h.data_ptr(), NN.dblp), C.byref(h)))
            state["t"] = H.DeviceTensor(env.ctx, h, tuple(dims), fmt)
        else:
            NN.check(NN.lib().spd_tensor_restage(env.ctx.h, state["t"].h, pos_pp, crd_pp,
                                                 C.cast(vals_h.data_ptr(), NN.dblp)))
        return state["t"]

    step.keep = (pairs, crd_h, vals_h)
    return step, nbytes, state


# ------------------------------------------------------------------ C1 ---
def config_c1(env, H, synth):
    from paper_2207_13901_b200 import _native as NN
    torch = env.torch
    n, S = 1_000_000, 10_000_000
    if env.rank == 0:
        rp = np.empty(n + 1, np.int64)
        crd = np.empty(S, np.int64)
        vals = np.empty(S)
        nnz = synth.syn_uniform_csr(n, n, S, 42, 0, rp.ctypes.data_as(NN.i64p), crd.ctypes.data_as(NN.i64p),
                                    vals.ctypes.data_as(NN.dblp))
        crd, vals = crd[:nnz], vals[:nnz]
        x = np.empty(n)
        synth.syn_dense(n, 43, 0, x.ctypes.data_as(NN.dblp))
    else:
        rp = crd = vals = x = np.empty(0)
    rp_d, crd_d, vals_d = env.bcast(rp, torch.int64), env.bcast(crd, torch.int64), env.bcast(vals, torch.float64)
    x_d = env.bcast(x, torch.float64)
    nnz = crd_d.numel()
    B = H.DeviceTensor.wrap(env.ctx, (n, n), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                            vals_d.data_ptr(), keep=(rp_d, crd_d, vals_d))
    y_d = torch.empty(n, dtype=torch.float64, device=env.dev)
    first, count, P = env.colours()

    def step():
        H.partition_universe(env.ctx, B, P, host=False)
        H.spmv(env.ctx, B, x_d, y_d, first=first, count=count, pieces=P, stats=False)

    ms, leaf, nl = measure(env, step)
    flops = 2.0 * nnz
    by = 8 * (n + 1) + 16 * nnz + 8 * n + 8 * n
    out = {"workload": f"C1: SpMV a(i)=B(i,j)*c(j), uniform 1M x 1M, 10M samples ({nnz} nnz), row split "
                       f"into {P} colour(s), one per GPU",
           "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms, "gpu_launches": nl,
           "roofline": roofline(env, by / env.world, leaf, "k_spmv_win<4>"),
           "effective_gbs": by / (ms * 1e-3) / 1e9}
    if env.world > 1:
        step()

        def ref():
            c1 = _ctx1(env, H)
            B1 = H.DeviceTensor.wrap(c1, (n, n), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                                     vals_d.data_ptr())
            y1 = torch.empty_like(y_d)
            H.partition_universe(c1, B1, P, host=False)
            H.spmv(c1, B1, x_d, y1, pieces=P, stats=False)
            torch.cuda.synchronize()
            B1.close()
            c1.close()
            return y1

        out["multi_gpu_check"] = mgpu_check(env, H, y_d, 1, H.last_owned(env.ctx, first, count), ref)
    B.close()
    if env.world == 1:
        rs, nbytes, st = _restager(env, H, (n, n), H.parse_format("ds"), [rp], [crd], vals)
        x_h = _pinned(torch, x)
        y_h = torch.empty(n, dtype=torch.float64).pin_memory()
        xd2 = torch.empty(n, dtype=torch.float64, device=env.dev)
        yd2 = torch.empty(n, dtype=torch.float64, device=env.dev)

        def one():
            Bs = rs()
            xd2.copy_(x_h, non_blocking=True)
            H.partition_universe(env.ctx, Bs, 1, host=False)
            H.spmv(env.ctx, Bs, xd2, yd2, pieces=1, stats=False)
            y_h.copy_(yd2, non_blocking=True)

        out["e2e"] = e2e_loop(env, one, flops, nbytes + n * 8, n * 8)
        st["t"].close()
        if not env.args.no_cpu_baseline:
            Bh = _csr_host(H, n, n, rp, crd, vals)
            xh = H.SparseTensor.from_parts((n,), H.parse_format("d"), [H.Level("d", dom=(n,))], x)
            SK = _sk()
            cb, run = cpu_reference(env, "spmv", SK.ROW, "d", {"B": (Bh, "ds"), "c": (xh, "d")}, flops,
                                    env.host_cores, "C1 at full size (1M x 1M, 10M samples)")
            cb["matches_gpu"] = bool(np.allclose(run.output()[1], y_h.numpy(), rtol=1e-10, atol=0))
            out["cpu_baseline"] = cb
    return out


# ------------------------------------------------------------ SpMV-RMAT ---
def config_spmv_rmat(env, H, rm, x_seed):
    torch = env.torch
    n, rp_d, crd_d, vals_d, Bstep = rm["n"], rm["rp_d"], rm["crd_d"], rm["vals_d"], rm["Bstep"]
    nnz = crd_d.numel()
    x_d = env.bcast(rm["dense"](n, x_seed) if env.rank == 0 else np.empty(0), torch.float64)
    y_d = torch.empty(n, dtype=torch.float64, device=env.dev)
    first, count, P = env.colours()
    if rm.get("blocks") is not None:
        # the headline's over-decomposed nonzero split and its cost-balanced
        # colour blocks (B placed by them), reused for the SpMV of the same matrix
        Bstep, P, bounds = rm["blocks"]
        H.set_colour_blocks(env.ctx, P, bounds)
        first, count = int(bounds[env.rank]), int(bounds[env.rank + 1] - bounds[env.rank])

    def step():
        H.partition_nonzero(env.ctx, Bstep, 1, P, host=False)
        H.spmv(env.ctx, Bstep, x_d, y_d, first=first, count=count, pieces=P, stats=False)

    ms, leaf, nl = measure(env, step)
    flops = 2.0 * nnz
    by = 8 * (n + 1) + 16 * nnz + 8 * n + 8 * n
    out = {"workload": f"SpMV a(i)=B(i,j)*c(j) on the C2 R-MAT (scale {rm['scale']}, {nnz} nnz), nonzero split "
                       f"into {P} colour(s)" + ("" if rm.get("blocks") is None else
                                                 ", the headline's cost-balanced block of them per GPU"),
           "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms, "gpu_launches": nl,
           "roofline": roofline(env, by / env.world, leaf, "k_spmv_win<6,int> over compacted columns"),
           "effective_gbs": by / (ms * 1e-3) / 1e9}
    if env.world > 1:
        step()

        def ref():
            c1 = _ctx1(env, H)
            B1 = H.DeviceTensor.wrap(c1, (n, n), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                                     vals_d.data_ptr())
            y1 = torch.empty_like(y_d)
            H.partition_nonzero(c1, B1, 1, P, host=False)
            H.spmv(c1, B1, x_d, y1, pieces=P, stats=False)
            torch.cuda.synchronize()
            B1.close()
            c1.close()
            return y1

        out["multi_gpu_check"] = mgpu_check(env, H, y_d, 1, H.last_owned(env.ctx, first, count), ref)
    if rm.get("blocks") is not None:
        H.set_colour_blocks(env.ctx, P, None)
    if env.world == 1:
        rp, crd, vals = rm["host"]
        rs, nbytes, st = _restager(env, H, (n, n), H.parse_format("ds"), [rp], [crd], vals)
        x_h = x_d.cpu().pin_memory()
        y_h = torch.empty(n, dtype=torch.float64).pin_memory()
        xd2 = torch.empty_like(x_d)

        def one():
            Bs = rs()
            xd2.copy_(x_h, non_blocking=True)
            H.partition_nonzero(env.ctx, Bs, 1, 1, host=False)
            H.spmv(env.ctx, Bs, xd2, y_d, pieces=1, stats=False)
            y_h.copy_(y_d, non_blocking=True)

        out["e2e"] = e2e_loop(env, one, flops, nbytes + n * 8, n * 8)
        st["t"].close()
        if not env.args.no_cpu_baseline:
            sc = env.args.ref_scale
            n2, rp2, crd2, vals2 = rm["gen"](sc)
            x2 = rm["dense"](n2, x_seed)
            Bh = _csr_host(H, n2, n2, rp2, crd2, vals2)
            xh = H.SparseTensor.from_parts((n2,), H.parse_format("d"), [H.Level("d", dom=(n2,))], x2)
            SK = _sk()
            out["cpu_baseline"], _ = cpu_reference(
                env, "spmv", SK.KERNELS["spmv"]["nonzero"], "d", {"B": (Bh, "ds"), "c": (xh, "d")},
                2.0 * len(crd2), max(1, min(env.host_cores, 64)),
                f"bounded sample: R-MAT scale {sc} ({n2} rows, {len(crd2)} nnz) of the same generator")
    return out


# ------------------------------------------------------------------ C3 ---
def config_c3(env, H, rm):
    torch = env.torch
    K = 128
    n, Bstep = rm["n"], rm["Bstep"]
    nnz = rm["crd_d"].numel()
    from paper_2207_13901_b200 import _native as NN
    first, count, P = env.colours()
    placement = None
    C_h = D_h = None
    if env.rank == 0:  # host operands, pinned (the e2e leg copies them every step)
        C_h = torch.empty(n * K, dtype=torch.float64).pin_memory()
        NN.synth().syn_dense(n * K, 44, 0, C.cast(C_h.data_ptr(), NN.dblp))
        D_h = torch.empty(n * K, dtype=torch.float64).pin_memory()
        NN.synth().syn_dense(n * K, 45, 0, C.cast(D_h.data_ptr(), NN.dblp))
    if env.world == 1:
        C_d = C_h.to(env.dev)
        D_d = D_h.to(env.dev)
        C_ptr = C_d
    else:
        # D block-distributed over the GPUs, then all-gathered over
        # NVLink (spd_allgather) -- reported as placement, outside the step;
        # C held only as the projected row slab of this GPU's colour
        # (planner.cpp:278-293): the leaf reads rows [top.lo, top.hi] only.
        dist = env.dist
        cols = H.partition_nonzero(env.ctx, Bstep, 1, P)
        per = -(-n // env.world)
        D_d = torch.zeros(env.world * per * K, dtype=torch.float64, device=env.dev)
        t_lo, t_hi = cols[env.rank].top
        rows = max(t_hi - t_lo + 1, 0)
        C_slab = torch.empty(max(rows, 1) * K, dtype=torch.float64, device=env.dev)
        for r in range(env.world):
            d_lo, d_hi = r * per, min(n, (r + 1) * per) - 1
            c_lo, c_hi = cols[r].top
            if env.rank == 0:
                dblk = D_h[d_lo * K:(d_hi + 1) * K].to(env.dev) if d_hi >= d_lo else None
                cblk = C_h[c_lo * K:(c_hi + 1) * K].to(env.dev) if c_hi >= c_lo else None
                if r == 0:
                    if dblk is not None:
                        D_d[d_lo * K:(d_hi + 1) * K].copy_(dblk)
                    if cblk is not None:
                        C_slab[:cblk.numel()].copy_(cblk)
                else:
                    if dblk is not None:
                        dist.send(dblk, r)
                    if cblk is not None:
                        dist.send(cblk, r)
            elif env.rank == r:
                if d_hi >= d_lo:
                    dist.recv(D_d[d_lo * K:(d_hi + 1) * K], 0)
                if c_hi >= c_lo:
                    buf = torch.empty((c_hi - c_lo + 1) * K, dtype=torch.float64, device=env.dev)
                    dist.recv(buf, 0)
                    C_slab[:buf.numel()].copy_(buf)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        env.ctx.allgather(D_d, per * K * 8)
        e1.record()
        torch.cuda.synchronize()
        ag_ms = env.maxr([e0.elapsed_time(e1)])[0]
        placement = {"D_allgather_ms": ag_ms, "D_bytes_received_per_gpu": (env.world - 1) * per * K * 8,
                     "C_slab_rows": rows, "C_slab_bytes": rows * K * 8,
                     "note": "D (n x 128, j-major) block-distributed then all-gathered over NVLink; C held as "
                             "this GPU's projected row slab; outside the timed step"}
        C_ptr = C_slab.data_ptr() - t_lo * K * 8  # global row i at C_ptr + i*K
    A_d = torch.empty(nnz, dtype=torch.float64, device=env.dev)

    def step():
        H.partition_nonzero(env.ctx, Bstep, 1, P, host=False)
        H.sddmm(env.ctx, Bstep, C_ptr, D_d, K, 1, K, A_d, first=first, count=count, pieces=P, stats=False)

    ms, leaf, nl = measure(env, step)
    flops = 2.0 * nnz * K
    by = 8 * (n + 1) + 16 * nnz + 8 * nnz + 8 * n * K + 8 * n * K
    out = {"workload": f"C3: SDDMM A(i,j)=B(i,j)*C(i,k)*D(k,j), K=128, on the C2 R-MAT ({nnz} nnz), D stored "
                       f"j-major (dd:1,0), nonzero split into {P} colour(s)",
           "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms, "gpu_launches": nl,
           "roofline": roofline(env, by / env.world, leaf, "k_sddmm_nz<4,3>"),
           "effective_gbs": by / (ms * 1e-3) / 1e9, "placement": placement}
    if env.world > 1:
        step()

        def ref():
            c1 = _ctx1(env, H)
            B1 = H.DeviceTensor.wrap(c1, (n, n), H.parse_format("ds"), [rm["rp_d"].data_ptr()],
                                     [rm["crd_d"].data_ptr()], rm["vals_d"].data_ptr())
            Cfull = C_h.to(env.dev)
            a1 = torch.empty_like(A_d)
            H.partition_nonzero(c1, B1, 1, P, host=False)
            H.sddmm(c1, B1, Cfull, D_d, K, 1, K, a1, pieces=P, stats=False)
            torch.cuda.synchronize()
            B1.close()
            c1.close()
            del Cfull
            return a1

        out["multi_gpu_check"] = mgpu_check(env, H, A_d, 1, tuple(cols[env.rank].q), ref)
    if env.world == 1:
        rp, crd, vals = rm["host"]
        rs, nbytes, st = _restager(env, H, (n, n), H.parse_format("ds"), [rp], [crd], vals)
        A_h = torch.empty(nnz, dtype=torch.float64).pin_memory()

        def one():
            Bs = rs()
            C_d.copy_(C_h, non_blocking=True)
            D_d.copy_(D_h, non_blocking=True)
            H.partition_nonzero(env.ctx, Bs, 1, 1, host=False)
            H.sddmm(env.ctx, Bs, C_d, D_d, K, 1, K, A_d, pieces=1, stats=False)
            A_h.copy_(A_d, non_blocking=True)

        out["e2e"] = e2e_loop(env, one, flops, nbytes + 2 * n * K * 8, nnz * 8)
        st["t"].close()
        if not env.args.no_cpu_baseline:
            sc = env.args.sddmm_ref_scale
            n2, rp2, crd2, vals2 = rm["gen"](sc)
            Bh = _csr_host(H, n2, n2, rp2, crd2, vals2)
            Ch = H.SparseTensor.from_parts((n2, K), H.parse_format("dd"), [H.Level("d", dom=(n2, K))],
                                           rm["dense"](n2 * K, 44))
            Dh = H.SparseTensor.from_parts((K, n2), H.parse_format("dd:1,0"), [H.Level("d", dom=(n2, K))],
                                           rm["dense"](n2 * K, 45))
            SK = _sk()
            out["cpu_baseline"], _ = cpu_reference(
                env, "sddmm", SK.KERNELS["sddmm"]["nonzero"], "ds",
                {"B": (Bh, "ds"), "C": (Ch, "dd"), "D": (Dh, "dd:1,0")}, 2.0 * len(crd2) * K,
                max(1, min(env.host_cores, 16)),
                f"bounded sample: R-MAT scale {sc} ({n2} rows, {len(crd2)} nnz) -- execute() allocates a dense "
                f"accumulator of the whole output space per task (sim.cpp:949-950), so scale 24 cannot run")
    del D_d, A_d, C_h, D_h
    return out


# ------------------------------------------------------------------ C4 ---
def config_c4(env, H, synth):
    from paper_2207_13901_b200 import _native as NN
    torch = env.torch
    I, J, Kd, S, R = 12092, 9184, 28818, 10_000_000, 32
    if env.rank == 0:
        rp1 = np.empty(I + 1, np.int64)
        crd1 = np.empty(S, np.int64)
        rp2 = np.empty(S + 1, np.int64)
        crd2 = np.empty(S, np.int64)
        vals = np.empty(S)
        F = np.zeros(1, np.int64)
        nnz = synth.syn_powerlaw_csf(I, J, Kd, S, 4, 0, rp1.ctypes.data_as(NN.i64p), crd1.ctypes.data_as(NN.i64p),
                                     rp2.ctypes.data_as(NN.i64p), crd2.ctypes.data_as(NN.i64p),
                                     vals.ctypes.data_as(NN.dblp), F.ctypes.data_as(NN.i64p))
        F = int(F[0])
        crd1, rp2, crd2, vals = crd1[:F], rp2[:F + 1], crd2[:nnz], vals[:nnz]
        c = np.empty(Kd)
        synth.syn_dense(Kd, 46, 0, c.ctypes.data_as(NN.dblp))
        Cm = np.empty(J * R)
        synth.syn_dense(J * R, 47, 0, Cm.ctypes.data_as(NN.dblp))
        Dm = np.empty(Kd * R)
        synth.syn_dense(Kd * R, 48, 0, Dm.ctypes.data_as(NN.dblp))
    else:
        rp1 = crd1 = rp2 = crd2 = vals = c = Cm = Dm = np.empty(0)
    arrs = [env.bcast(a, dt) for a, dt in ((rp1, torch.int64), (crd1, torch.int64), (rp2, torch.int64),
                                            (crd2, torch.int64), (vals, torch.float64))]
    c_d, C_d, D_d = (env.bcast(a, torch.float64) for a in (c, Cm, Dm))
    F, nnz = arrs[1].numel(), arrs[3].numel()
    fmt = H.parse_format("dss")
    Bt = H.DeviceTensor.wrap(env.ctx, (I, J, Kd), fmt, [arrs[0].data_ptr(), arrs[2].data_ptr()],
                             [arrs[1].data_ptr(), arrs[3].data_ptr()], arrs[4].data_ptr(), keep=tuple(arrs))
    Av = torch.empty(F, dtype=torch.float64, device=env.dev)
    A_d = torch.empty(I * R, dtype=torch.float64, device=env.dev)
    first, count, P = env.colours()

    def step_ttv():
        H.partition_nonzero(env.ctx, Bt, 2, P, host=False)
        H.spttv(env.ctx, Bt, c_d, Av, first=first, count=count, pieces=P, stats=False)

    def step_mttkrp():
        H.partition_nonzero(env.ctx, Bt, 2, P, host=False)
        H.spmttkrp(env.ctx, Bt, C_d, D_d, R, A_d, first=first, count=count, pieces=P, stats=False)

    res = {}
    bB = 8 * (I + 1) + 8 * F + 8 * (F + 1) + 16 * nnz

    def ref_of(name):
        def ref():
            c1 = _ctx1(env, H)
            B1 = H.DeviceTensor.wrap(c1, (I, J, Kd), fmt, [arrs[0].data_ptr(), arrs[2].data_ptr()],
                                     [arrs[1].data_ptr(), arrs[3].data_ptr()], arrs[4].data_ptr())
            H.partition_nonzero(c1, B1, 2, P, host=False)
            if name == "C4-SpTTV":
                o = torch.empty_like(Av)
                H.spttv(c1, B1, c_d, o, pieces=P, stats=False)
            else:
                o = torch.empty_like(A_d)
                H.spmttkrp(c1, B1, C_d, D_d, R, o, pieces=P, stats=False)
            torch.cuda.synchronize()
            B1.close()
            c1.close()
            return o
        return ref

    for name, step, flops, by, kern in (
            ("C4-SpTTV", step_ttv, 2.0 * nnz, bB + 8 * Kd + 8 * F, "k_spmv_win<6> over fibres"),
            ("C4-SpMTTKRP", step_mttkrp, 3.0 * nnz * R, bB + 8 * (J + Kd + I) * R, "k_mttkrp32_nz<4,3>")):
        ms, leaf, nl = measure(env, step)
        check = None
        if env.world > 1:
            step()
            out_d, width = (Av, 1) if name == "C4-SpTTV" else (A_d, R)
            check = mgpu_check(env, H, out_d, width, H.last_owned(env.ctx, first, count), ref_of(name))
        res[name] = {"workload": f"{name[3:]} on a {I}x{J}x{Kd} power-law dss tensor ({nnz} nnz, {F} fibres), "
                                 f"nonzero split into {P} colour(s)" + (", R=32" if "MTT" in name else ""),
                     "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms, "gpu_launches": nl,
                     "roofline": roofline(env, by / env.world, leaf, kern),
                     "effective_gbs": by / (ms * 1e-3) / 1e9, "multi_gpu_check": check}
        if "MTT" in name and leaf > 0:
            # both factors (C 2.4 MB, D 7.4 MB) sit in L2: the leaf is bound by
            # L2 -> SM bytes, two 256-byte row reads per position, against the
            # measured L2-resident gather ceiling (profiles/r02_probe_gather.jsonl)
            l2b = 2.0 * 256 * nnz / env.world
            ach = l2b / (leaf * 1e-3) / 1e9
            res[name]["roofline_l2"] = {"bound": "l2", "achieved": ach, "peak": L2_GATHER_PEAK_GBS, "unit": "GB/s",
                                        "frac": ach / L2_GATHER_PEAK_GBS, "bytes_per_launch": l2b,
                                        "peak_source": "measured: 256-byte row gathers from a 16 MB working set, "
                                                       "scripts/probe_gather.py"}
    Bt.close()
    if env.world == 1:
        rs, nbytes, st = _restager(env, H, (I, J, Kd), fmt, [rp1, rp2], [crd1, crd2], vals)
        c_h, C_h, D_h = _pinned(torch, c), _pinned(torch, Cm), _pinned(torch, Dm)
        Av_h = torch.empty(F, dtype=torch.float64).pin_memory()
        A_h = torch.empty(I * R, dtype=torch.float64).pin_memory()

        def one_ttv():
            Bs = rs()
            c_d.copy_(c_h, non_blocking=True)
            H.partition_nonzero(env.ctx, Bs, 2, 1, host=False)
            H.spttv(env.ctx, Bs, c_d, Av, pieces=1, stats=False)
            Av_h.copy_(Av, non_blocking=True)

        def one_mttkrp():
            Bs = rs()
            C_d.copy_(C_h, non_blocking=True)
            D_d.copy_(D_h, non_blocking=True)
            H.partition_nonzero(env.ctx, Bs, 2, 1, host=False)
            H.spmttkrp(env.ctx, Bs, C_d, D_d, R, A_d, pieces=1, stats=False)
            A_h.copy_(A_d, non_blocking=True)

        res["C4-SpTTV"]["e2e"] = e2e_loop(env, one_ttv, 2.0 * nnz, nbytes + Kd * 8, F * 8)
        res["C4-SpMTTKRP"]["e2e"] = e2e_loop(env, one_mttkrp, 3.0 * nnz * R, nbytes + (J + Kd) * R * 8, I * R * 8)
        st["t"].close()
        if not env.args.no_cpu_baseline:
            SK = _sk()
            t = H.SparseTensor.from_rowptrs((I, J, Kd), fmt, [rp1, rp2], [crd1, crd2], vals)
            ch = H.SparseTensor.from_parts((Kd,), H.parse_format("d"), [H.Level("d", dom=(Kd,))], c)
            Ch = H.SparseTensor.from_parts((J, R), H.parse_format("dd"), [H.Level("d", dom=(J, R))], Cm)
            Dh = H.SparseTensor.from_parts((Kd, R), H.parse_format("dd"), [H.Level("d", dom=(Kd, R))], Dm)
            cores = max(1, min(env.host_cores, 64))
            cb, run = cpu_reference(env, "spttv", SK.KERNELS["spttv"]["nonzero"], "ds",
                                    {"B": (t, "dss"), "c": (ch, "d")}, 2.0 * nnz, cores, "C4 SpTTV at full size")
            cb["matches_gpu"] = bool(np.allclose(run.output()[1], Av_h.numpy(), rtol=1e-10, atol=0))
            res["C4-SpTTV"]["cpu_baseline"] = cb
            cb, run = cpu_reference(env, "spmttkrp", SK.KERNELS["spmttkrp"]["nonzero"], "dd",
                                    {"B": (t, "dss"), "C": (Ch, "dd"), "D": (Dh, "dd")}, 3.0 * nnz * R, cores,
                                    "C4 SpMTTKRP R=32 at full size")
            cb["matches_gpu"] = bool(np.allclose(run.output()[1], A_h.numpy(), rtol=1e-10, atol=0))
            res["C4-SpMTTKRP"]["cpu_baseline"] = cb
    return res


# ------------------------------------------------------------------ C5 ---
def config_c5(env, H, rm):
    torch = env.torch
    n = rm["n"]
    ops_host = rm["spadd3_inputs"]()  # rank 0: [(rp, crd, vals)] * 3, others: None
    devs = []
    for i in range(3):
        if env.rank == 0:
            rp, crd, vals = ops_host[i]
        else:
            rp = crd = vals = np.empty(0)
        a = [env.bcast(rp, torch.int64), env.bcast(crd, torch.int64), env.bcast(vals, torch.float64)]
        devs.append(H.DeviceTensor.wrap(env.ctx, (n, n), H.parse_format("ds"), [a[0].data_ptr()], [a[1].data_ptr()],
                                        a[2].data_ptr(), keep=tuple(a)))
    nin = sum(d._keep[1].numel() for d in devs)
    P = 8 if env.world == 1 else env.world
    sel = {"first": 0, "count": P} if env.world == 1 else {"first": env.rank, "count": 1}
    live = {"A": None}

    def step():
        if live["A"] is not None:
            live["A"].close()
        H.partition_universe(env.ctx, devs[0], P, host=False)
        live["A"], _ = H.spadd3(env.ctx, devs[0], devs[1], devs[2], first=sel["first"], count=sel["count"],
                                pieces=P, stats=False)

    balance = None
    if env.world > 1 and env.args.colours_per_gpu > 1:
        # the row split over-decomposed into colours_per_gpu x N row blocks,
        # each GPU running a contiguous block of them balanced by the inputs'
        # stored entries (3 x B's positions: C and D are B shifted) + rows,
        # then refined by measured times (as the C2 headline)
        P = env.args.colours_per_gpu * env.world
        H.partition_universe(env.ctx, devs[0], P)
        pos, nrow, _ = H.colour_costs(env.ctx, devs[0], P)
        cur = (3.0 * pos + nrow).astype(np.float64)
        bounds = H.split_colour_blocks(cur, env.world)
        balance = {"model": "3 x positions + rows", "rounds": []}
        for it in range(env.args.balance_rounds + 1):
            H.set_colour_blocks(env.ctx, P, bounds)
            sel["first"], sel["count"] = int(bounds[env.rank]), int(bounds[env.rank + 1] - bounds[env.rank])
            if it == env.args.balance_rounds:
                break
            lt = _block_times(env, step)
            balance["rounds"].append({"blocks": [int(b) for b in bounds], "leaf_ms": lt})
            for r in range(env.world):
                seg = slice(int(bounds[r]), int(bounds[r + 1]))
                cur[seg] *= lt[r] / max(cur[seg].sum(), 1e-30)
            nb = H.split_colour_blocks(cur, env.world)
            if np.array_equal(nb, bounds):
                break
            bounds = nb
        balance["final_blocks"] = [int(b) for b in bounds]
    first, count = sel["first"], sel["count"]

    ms, leaf, nl = measure(env, step)
    A = live["A"]
    nA = int(np.sum(env.maxr([float(A.global_span()[3] if env.world > 1 else A.nvals())])))
    by = sum(8 * (n + 1) + 16 * d._keep[1].numel() for d in devs) + 8 * (n + 1) + 16 * nA
    out = {"workload": f"C5: SpAdd3 A=B+C+D, the C2 R-MAT and two copies with columns shifted +1/+2 "
                       f"({nin} input nnz -> {nA}), row split into {P} colour(s)" +
                       ("" if balance is None else ", a contiguous cost-balanced block of them per GPU"),
           "block_balance": balance,
           "value": float(nin) / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms, "gpu_launches": nl,
           "roofline": roofline(env, by / env.world, ms,
                                "the SpAdd3 step (count, scan, allocate, fill; leaf = whole step)"),
           "effective_gbs": by / (ms * 1e-3) / 1e9}
    if env.world > 1:
        # the row blocks gathered on rank 0 (spd_gather_rows) vs every colour on rank 0's GPU
        whole = A.gather_rows(0)
        ok = True
        if env.rank == 0:
            got = whole.download()
            whole.close()
            c1 = _ctx1(env, H)
            Bs1 = [H.DeviceTensor.wrap(c1, (n, n), H.parse_format("ds"), [d._keep[0].data_ptr()],
                                       [d._keep[1].data_ptr()], d._keep[2].data_ptr()) for d in devs]
            H.partition_universe(c1, Bs1[0], P, host=False)
            A1, _ = H.spadd3(c1, Bs1[0], Bs1[1], Bs1[2], pieces=P, stats=False)
            want = A1.download()
            A1.close()
            for b in Bs1:
                b.close()
            c1.close()
            ok = (np.array_equal(got.levels[1].rowptr(), want.levels[1].rowptr()) and
                  np.array_equal(got.levels[1].crd, want.levels[1].crd) and np.array_equal(got.vals, want.vals))
        t = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device=env.dev)
        env.dist.broadcast(t, 0)
        out["multi_gpu_check"] = {"bit_exact_vs_one_gpu": bool(t[0] > 0.5),
                                  "what": "the row blocks gathered on rank 0 (spd_gather_rows) vs every colour "
                                          "of the same partition on rank 0's GPU: row pointer, crd, vals"}
    A.close()
    live["A"] = None
    if balance is not None:
        H.set_colour_blocks(env.ctx, P, None)
    if env.world == 1:
        steps = []
        nbytes = 0
        for rp, crd, vals in ops_host:
            rs, nb, st = _restager(env, H, (n, n), H.parse_format("ds"), [rp], [crd], vals)
            steps.append((rs, st))
            nbytes += nb
        bufs = {}

        def one():
            Bs = [rs() for rs, _ in steps]
            H.partition_universe(env.ctx, Bs[0], 8, host=False)
            Ad, _ = H.spadd3(env.ctx, Bs[0], Bs[1], Bs[2], pieces=8, stats=False)
            _, par, pos = Ad.level(1)
            if "crd" not in bufs or bufs["crd"].numel() < pos:
                bufs["pairs"] = np.empty((par, 2), np.int64)
                bufs["crd"] = torch.empty(pos, dtype=torch.int64).pin_memory()
                bufs["vals"] = torch.empty(pos, dtype=torch.float64).pin_memory()
            from paper_2207_13901_b200 import _native as NN
            NN.check(NN.lib().spd_tensor_download_level(Ad.h, 1, bufs["pairs"].ctypes.data_as(NN.i64p),
                                                        C.cast(bufs["crd"].data_ptr(), NN.i64p)))
            NN.check(NN.lib().spd_tensor_download_vals(Ad.h, C.cast(bufs["vals"].data_ptr(), NN.dblp)))
            bufs["nA"] = pos
            Ad.close()

        out["e2e"] = e2e_loop(env, one, float(nin), nbytes, 16 * (n + 0) + 16 * nA)
        for _, st in steps:
            st["t"].close()
        if not env.args.no_cpu_baseline:
            sc = env.args.sddmm_ref_scale
            ins = rm["spadd3_inputs"](sc)
            n2 = len(ins[0][0]) - 1
            SK = _sk()
            tens = {nm: (_csr_host(H, n2, n2, *o), "ds") for nm, o in zip("BCD", ins)}
            out["cpu_baseline"], _ = cpu_reference(
                env, "spadd3", SK.ROW, "ds", tens, float(sum(len(o[1]) for o in ins)), 8,
                f"bounded sample: R-MAT scale {sc} ({n2} rows) + shifted copies -- execute() allocates a dense "
                f"accumulator of the whole output space per task (sim.cpp:949-950)")
    for d in devs:
        d.close()
    return out
