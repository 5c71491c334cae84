#!/usr/bin/env python3
"""Multi-GPU parity check (run under torchrun, one process per GPU).

Each rank runs one colour of a nonzero (or row) split of the same matrix
through the C-ABI with an NCCL communicator; rows cut between GPUs are
combined by the backend over NCCL.  Rank 0 gathers every rank's owned rows
(the write ranges W_c, recomputed here from the colours) and compares the
assembled output with the CPU restatement run with the same number of
colours -- bit-exact for integer values, 1e-10 relative otherwise.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/mgpu_check.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import torch
    import torch.distributed as dist

    import oracle_bind as ob
    import oracle_exec
    import spd_kernels as K
    from paper_2207_13901_b200 import host as H
    from paper_2207_13901_b200.distributed import assemble, init_comm, owned_rows

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctx = H.Context(local)
    init_comm(ctx, dist, rank, world, dev)

    failures = 0
    for kernel, N in (("spmv", 1), ("spmm", 32), ("spmm", 8)):
        for schedule in ("nonzero", "row"):
            for integers in (True, False):
                rng = np.random.default_rng(1234)
                # a matrix with a hub row spanning several colours plus random rows
                n, m = 3000, 2500
                rows = np.concatenate([np.full(40000, 17), rng.integers(0, n, 60000)])
                cols = rng.integers(0, m, rows.shape[0])
                vals = (rng.integers(1, 5, rows.shape[0]).astype(float) if integers
                        else rng.uniform(0.5, 1.5, rows.shape[0]))
                B = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, cols], 1), vals)
                t = {"B": B}
                if kernel == "spmv":
                    t["c"] = K.dense(rng, (m,), "d", integers)
                else:
                    t["C"] = K.dense(rng, (m, N), "dd", integers)
                Bd = H.DeviceTensor.upload(ctx, B)
                if schedule == "row":
                    cols_ = H.partition_universe(ctx, Bd, world)
                else:
                    cols_ = H.partition_nonzero(ctx, Bd, 1, world)
                rp = B.levels[1].rowptr()
                if kernel == "spmv":
                    c = torch.from_numpy(t["c"].vals).to(dev)
                    out = torch.zeros(n, dtype=torch.float64, device=dev)
                    st = H.spmv(ctx, Bd, c, out, first=rank, count=1, pieces=world)
                else:
                    Cd = torch.from_numpy(t["C"].vals).to(dev)
                    out = torch.zeros(n * N, dtype=torch.float64, device=dev)
                    st = H.spmm(ctx, Bd, Cd, N, out, first=rank, count=1, pieces=world)
                W = owned_rows(cols_, rp, schedule, n)
                width = 1 if kernel == "spmv" else N
                full = out.view(n, width)
                gathered = [torch.zeros_like(full) for _ in range(world)]
                dist.all_gather(gathered, full)
                if rank == 0:
                    got = assemble([x.cpu().numpy() for x in gathered], W, width, n)
                    want = np.asarray(oracle_exec.oracle_execute(kernel, t, schedule, world)["out"]).reshape(n, width)
                    if integers:
                        ok = np.array_equal(got, want)
                    else:
                        ok = np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300))
                    print(f"[mgpu world={world}] {kernel} N={N} {schedule} {'int' if integers else 'real'}: "
                          f"{'OK' if ok else 'MISMATCH'} combines={st.combines}", flush=True)
                    failures += 0 if ok else 1
                Bd.close()
    # Placed operands (spd_tensor_place): every GPU holds the row pointer and
    # only its colour's crd/vals; the leaf ops run on the pieces.
    for schedule in ("nonzero", "row"):
        rng = np.random.default_rng(4321)
        n, m = 3000, 2500
        rows = np.concatenate([np.full(30000, 5), rng.integers(0, n, 50000)])
        cols = rng.integers(0, m, rows.shape[0])
        vals = rng.uniform(0.5, 1.5, rows.shape[0])
        B = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, cols], 1), vals)
        whole = H.DeviceTensor.upload(ctx, B) if rank == 0 else None
        piece, nbytes = H.DeviceTensor.place(ctx, whole, (n, m), H.parse_format("ds"), schedule)
        lo, hi = piece.piece_span()
        Cm = K.dense(rng, (m, 32), "dd", False)
        Cd = torch.from_numpy(Cm.vals).to(dev)
        out = torch.zeros(n * 32, dtype=torch.float64, device=dev)
        cols_ = (H.partition_universe(ctx, piece, world) if schedule == "row"
                 else H.partition_nonzero(ctx, piece, 1, world))
        H.spmm(ctx, piece, Cd, 32, out, first=rank, count=1, pieces=world)
        W = owned_rows(cols_, B.levels[1].rowptr(), schedule, n)
        gathered = [torch.zeros_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        # SDDMM on the piece (hot-column index over the piece's positions)
        Kd = 128
        Cs = K.dense(rng, (n, Kd), "dd", False)
        Ds = K.dense(rng, (Kd, m), "dd:1,0", False)
        A = torch.zeros(len(B.vals), dtype=torch.float64, device=dev)
        (H.partition_universe(ctx, piece, world) if schedule == "row" else H.partition_nonzero(ctx, piece, 1, world))
        H.sddmm(ctx, piece, torch.from_numpy(Cs.vals).to(dev), torch.from_numpy(Ds.vals).to(dev), Kd, 1, Kd, A,
                first=rank, count=1, pieces=world)
        ga = [torch.zeros_like(A) for _ in range(world)]
        dist.all_gather(ga, A)
        # SpMV on the piece (compacted-column index over the piece's positions
        # when SPD_XC=2)
        cv = K.dense(rng, (m,), "d", False)
        yv = torch.zeros(n, dtype=torch.float64, device=dev)
        (H.partition_universe(ctx, piece, world) if schedule == "row" else H.partition_nonzero(ctx, piece, 1, world))
        H.spmv(ctx, piece, torch.from_numpy(cv.vals).to(dev), yv, first=rank, count=1, pieces=world)
        gy = [torch.zeros_like(yv) for _ in range(world)]
        dist.all_gather(gy, yv)
        spans = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(spans, torch.tensor([lo, hi], dtype=torch.int64, device=dev))
        if rank == 0:
            got = assemble([x.cpu().numpy() for x in gathered], W, 32, n)
            want = np.asarray(oracle_exec.oracle_execute("spmm", {"B": B, "C": Cm}, schedule, world)["out"]).reshape(n, 32)
            ok = np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300))
            gs = np.zeros(len(B.vals))
            for r in range(world):
                a, b = (int(x) for x in spans[r].cpu())
                gs[a:b + 1] = ga[r].cpu().numpy()[a:b + 1]
            wsd = np.asarray(oracle_exec.oracle_execute("sddmm", {"B": B, "C": Cs, "D": Ds}, schedule, world)["out"])
            ok2 = np.all(np.abs(gs - wsd) <= 1e-10 * np.maximum(np.abs(wsd), 1e-300))
            goty = assemble([x.cpu().numpy().reshape(n, 1) for x in gy], W, 1, n).reshape(-1)
            wy = np.asarray(oracle_exec.oracle_execute("spmv", {"B": B, "c": cv}, schedule, world)["out"]).reshape(-1)
            ok3 = np.all(np.abs(goty - wy) <= 1e-10 * np.maximum(np.abs(wy), 1e-300))
            print(f"[mgpu world={world}] placed {schedule}: spmm {'OK' if ok else 'MISMATCH'} sddmm "
                  f"{'OK' if ok2 else 'MISMATCH'} spmv {'OK' if ok3 else 'MISMATCH'} piece=[{lo},{hi}] "
                  f"bytes_in={nbytes}", flush=True)
            failures += (0 if ok else 1) + (0 if ok2 else 1) + (0 if ok3 else 1)
        piece.close()
        if whole is not None:
            whole.close()

    # Host-staged pieces (spd_tensor_upload_piece): every GPU copies the pos
    # level and only its colour's crd/vals from host memory; then a second
    # matrix with the same nnz is re-staged into the same buffers.
    for schedule in ("nonzero", "row"):
        rng = np.random.default_rng(99)
        n, m = 3000, 2500
        mats = []
        for _ in range(2):  # a full hub row 9 + 57500 distinct random entries elsewhere
            other = rng.choice((n - 1) * m, size=57500, replace=False)
            other = other + np.where(other >= 9 * m, m, 0)
            lin = np.concatenate([9 * m + np.arange(m), other])
            mats.append(H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([lin // m, lin % m], 1),
                                            rng.uniform(0.5, 1.5, len(lin))))
        Cm = K.dense(rng, (m, 32), "dd", False)
        Cd = torch.from_numpy(Cm.vals).to(dev)
        piece = None
        for i, B in enumerate(mats):
            if piece is None:
                piece = H.DeviceTensor.upload_piece(ctx, B, schedule)
            else:
                piece.restage(B)
            lo, hi = piece.piece_span()
            out = torch.zeros(n * 32, dtype=torch.float64, device=dev)
            cols_ = (H.partition_universe(ctx, piece, world) if schedule == "row"
                     else H.partition_nonzero(ctx, piece, 1, world))
            H.spmm(ctx, piece, Cd, 32, out, first=rank, count=1, pieces=world)
            W = owned_rows(cols_, B.levels[1].rowptr(), schedule, n)
            gathered = [torch.zeros_like(out) for _ in range(world)]
            dist.all_gather(gathered, out)
            if rank == 0:
                got = assemble([x.cpu().numpy() for x in gathered], W, 32, n)
                want = np.asarray(oracle_exec.oracle_execute("spmm", {"B": B, "C": Cm}, schedule, world)["out"]).reshape(n, 32)
                ok = np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300))
                print(f"[mgpu world={world}] host piece {schedule} {'upload' if i == 0 else 'restage'}: spmm "
                      f"{'OK' if ok else 'MISMATCH'} piece=[{lo},{hi}]", flush=True)
                failures += 0 if ok else 1
        piece.close()

    # Mismatched placement: a piece placed by one split moved to the other
    # (spd_tensor_repartition); SpMM on the moved piece; bytes received equal
    # the crd + vals part of the reference ledger (16 B per missing position).
    for held, need in (("row", "nonzero"), ("nonzero", "row")):
        rng = np.random.default_rng(808)
        n, m = 3000, 2500
        rows = np.concatenate([np.full(20000, 11), (rng.pareto(1.1, 60000) * 40).astype(np.int64) % n])
        cols = rng.integers(0, m, rows.shape[0])
        B = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, cols], 1),
                                rng.uniform(0.5, 1.5, rows.shape[0]))
        Cm = K.dense(rng, (m, 32), "dd", False)
        Cd = torch.from_numpy(Cm.vals).to(dev)
        piece = H.DeviceTensor.upload_piece(ctx, B, held)
        moved, nbytes = piece.repartition(need)
        lo, hi = moved.piece_span()
        out = torch.zeros(n * 32, dtype=torch.float64, device=dev)
        cols_ = (H.partition_universe(ctx, moved, world) if need == "row"
                 else H.partition_nonzero(ctx, moved, 1, world))
        H.spmm(ctx, moved, Cd, 32, out, first=rank, count=1, pieces=world)
        W = owned_rows(cols_, B.levels[1].rowptr(), need, n)
        gathered = [torch.zeros_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        # expected bytes: positions of my needed span outside my held span
        hl, hh = piece.piece_span()
        exp = 16 * max(hi - lo + 1, 0) - 16 * max(min(hi, hh) - max(lo, hl) + 1, 0)
        okb = torch.tensor([int(nbytes == exp)], device=dev)
        dist.all_reduce(okb, op=dist.ReduceOp.MIN)
        if rank == 0:
            got = assemble([x.cpu().numpy() for x in gathered], W, 32, n)
            want = np.asarray(oracle_exec.oracle_execute("spmm", {"B": B, "C": Cm}, need, world)["out"]).reshape(n, 32)
            ok = np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300)) and bool(okb.item())
            print(f"[mgpu world={world}] repartition {held}->{need}: spmm {'OK' if ok else 'MISMATCH'} "
                  f"bytes_in(rank0)={nbytes}", flush=True)
            failures += 0 if ok else 1
        moved.close()
        piece.close()

    # CSF pieces (dss / sss): upper levels whole, this GPU's colour of the
    # leaf crd / vals from host memory; SpTTV and SpMTTKRP on the pieces.
    for fmt in ("dss", "sss"):
        rng = np.random.default_rng(4242)
        I, J, Kd, R = 60, 50, 70, 32
        B = K.random_sparse(rng, (I, J, Kd), fmt, 0.03, False)
        piece = H.DeviceTensor.upload_piece(ctx, B, "nonzero")
        Cm, Dm, cv = K.dense(rng, (J, R), "dd", False), K.dense(rng, (Kd, R), "dd", False), K.dense(rng, (Kd,), "d", False)
        cols_ = H.partition_nonzero(ctx, piece, 2, world)
        A = torch.zeros(I * R, dtype=torch.float64, device=dev)
        H.spmttkrp(ctx, piece, torch.from_numpy(Cm.vals).to(dev), torch.from_numpy(Dm.vals).to(dev), R, A,
                   first=rank, count=1, pieces=world)
        F = B.levels[1].crd.shape[0]
        Av = torch.zeros(max(F, 1), dtype=torch.float64, device=dev)
        H.partition_nonzero(ctx, piece, 2, world)
        H.spttv(ctx, piece, torch.from_numpy(cv.vals).to(dev), Av, first=rank, count=1, pieces=world)
        # owned output rows: i via the leaf row pointer (rows absent from an sss top are empty), fibres via rp2
        rp2 = B.levels[2].rowptr()
        if fmt == "dss":
            leaf_rp = rp2[B.levels[1].rowptr()]
        else:
            top = B.levels[0].crd
            rp1 = B.levels[1].rowptr()
            leaf_rp = np.array([rp2[rp1[np.searchsorted(top, i)]] for i in range(I + 1)], np.int64)
        Wm = owned_rows(cols_, leaf_rp, "nonzero", I)
        Wt = owned_rows(cols_, rp2, "nonzero", F)
        ga = [torch.zeros_like(A) for _ in range(world)]
        dist.all_gather(ga, A)
        gt = [torch.zeros_like(Av) for _ in range(world)]
        dist.all_gather(gt, Av)
        if rank == 0:
            got = assemble([x.cpu().numpy() for x in ga], Wm, R, I)
            spec = K.KERNELS["spmttkrp"]
            fm = dict(spec["formats"], B=fmt)
            run = ob.RefRun(spec["expr"], spec["nonzero"], world, "dd",
                            {"B": (B, fmt), "C": (Cm, "dd"), "D": (Dm, "dd")}).ok()
            want = run.output()[1].reshape(I, R)
            ok1 = np.all(np.abs(got - want) <= 1e-10 * np.maximum(np.abs(want), 1e-300))
            gotv = assemble([x.cpu().numpy()[:F].reshape(F, 1) for x in gt], Wt, 1, F).reshape(-1)
            spec2 = K.KERNELS["spttv"]
            run2 = ob.RefRun(spec2["expr"], spec2["nonzero"], world, "ss" if fmt == "sss" else "ds",
                             {"B": (B, fmt), "c": (cv, "d")}).ok()
            want2 = run2.output()[1]
            ok2 = np.all(np.abs(gotv - want2) <= 1e-10 * np.maximum(np.abs(want2), 1e-300))
            lo, hi = piece.piece_span()
            print(f"[mgpu world={world}] csf piece {fmt}: spmttkrp {'OK' if ok1 else 'MISMATCH'} spttv "
                  f"{'OK' if ok2 else 'MISMATCH'} piece=[{lo},{hi}] nnz={len(B.vals)}", flush=True)
            failures += (0 if ok1 else 1) + (0 if ok2 else 1)
        piece.close()

    # SpDISTAL-Batched SpMM on a 2-D grid of the GPUs (x = rows, y = column
    # slabs of C / A): every GPU holds only its slab of C, no combine.
    BATCHED = ("divide(i, io, ii, M.x); divide(j, jo, ji, M.y); reorder(io, jo, ii, ji, k); "
               "distribute(io, M.x); distribute(jo, M.y); communicate({B}, io); communicate({A, C}, jo)")
    for Px in [d for d in range(1, world + 1) if world % d == 0]:
        Py = world // Px
        rng = np.random.default_rng(500 + Px)
        n, m, N = 700, 500, 24
        B = K.random_sparse(rng, (n, m), "ds", 0.05, True)
        Cm = K.dense(rng, (m, N), "dd", True)
        Bd = H.DeviceTensor.upload(ctx, B)
        x, y = divmod(rank, Py)
        lo, hi = H.divide_bounds(N, Py)[y]
        w = hi - lo + 1
        Cs = torch.from_numpy(np.ascontiguousarray(Cm.vals.reshape(m, N)[:, lo:hi + 1])).to(dev)
        Ab = torch.full((n * max(w, 1),), float("nan"), dtype=torch.float64, device=dev)
        H.spmm_batched(ctx, Bd, Cs, N, Ab, (Px, Py), rank=rank, stats=False)
        cols_ = H.partition_universe(ctx, Bd, Px)
        r0, r1 = cols_[x].top
        block = Ab.view(n, max(w, 1))[r0:r1 + 1, :w].cpu().numpy() if r0 <= r1 else np.zeros((0, w))
        blocks = [None] * world
        dist.all_gather_object(blocks, (r0, r1, lo, hi, block))
        if rank == 0:
            got = np.full((n, N), np.nan)
            for (a, b, c0, c1, blk) in blocks:
                if a <= b and c0 <= c1:
                    got[a:b + 1, c0:c1 + 1] = blk
            run = ob.RefRun("A(i, j) = B(i, k) * C(k, j)", BATCHED, f"x={Px},y={Py}", "dd",
                            K.ref_inputs("spmm", {"B": B, "C": Cm})).ok()
            want = run.output()[1].reshape(n, N)
            ok = np.array_equal(got, want)
            print(f"[mgpu world={world}] batched spmm grid x={Px},y={Py}: {'OK' if ok else 'MISMATCH'}", flush=True)
            failures += 0 if ok else 1
        Bd.close()

    # Batched SpMTTKRP on the same 2-D grids: rows of B / A over x, rank
    # columns of C, D, A over y; every GPU holds only its slabs of C and D.
    BATCHED_MT = ("divide(i, io, ii, M.x); divide(l, lo, li, M.y); reorder(io, lo, ii, j, k, li); "
                  "distribute(io, M.x); distribute(lo, M.y); communicate({B}, io); communicate({A, C, D}, lo)")
    for Px in [d for d in range(1, world + 1) if world % d == 0]:
        Py = world // Px
        rng = np.random.default_rng(600 + Px)
        I, J, Kd, R = 300, 120, 150, 32
        B = K.random_sparse(rng, (I, J, Kd), "dss", 0.002, True)
        Cm = K.dense(rng, (J, R), "dd", True)
        Dm = K.dense(rng, (Kd, R), "dd", True)
        Bd = H.DeviceTensor.upload(ctx, B)
        x, y = divmod(rank, Py)
        lo, hi = H.divide_bounds(R, Py)[y]
        w = hi - lo + 1
        Cs = torch.from_numpy(np.ascontiguousarray(Cm.vals.reshape(J, R)[:, lo:hi + 1])).to(dev)
        Ds = torch.from_numpy(np.ascontiguousarray(Dm.vals.reshape(Kd, R)[:, lo:hi + 1])).to(dev)
        Ab = torch.full((I * max(w, 1),), float("nan"), dtype=torch.float64, device=dev)
        H.spmttkrp_batched(ctx, Bd, Cs, Ds, R, Ab, (Px, Py), rank=rank, stats=False)
        cols_ = H.partition_universe(ctx, Bd, Px)
        r0, r1 = cols_[x].top
        block = Ab.view(I, max(w, 1))[r0:r1 + 1, :w].cpu().numpy() if r0 <= r1 else np.zeros((0, w))
        blocks = [None] * world
        dist.all_gather_object(blocks, (r0, r1, lo, hi, block))
        if rank == 0:
            got = np.full((I, R), np.nan)
            for (a, b, c0, c1, blk) in blocks:
                if a <= b and c0 <= c1:
                    got[a:b + 1, c0:c1 + 1] = blk
            run = ob.RefRun("A(i, l) = B(i, j, k) * C(j, l) * D(k, l)", BATCHED_MT, f"x={Px},y={Py}", "dd",
                            K.ref_inputs("spmttkrp", {"B": B, "C": Cm, "D": Dm})).ok()
            want = run.output()[1].reshape(I, R)
            ok = np.array_equal(got, want)
            print(f"[mgpu world={world}] batched spmttkrp grid x={Px},y={Py}: {'OK' if ok else 'MISMATCH'}",
                  flush=True)
            failures += 0 if ok else 1
        Bd.close()

    # SpAdd3: every GPU assembles its row block, global pos offsets from the
    # all-gathered per-GPU nnz, pieces gathered on rank 0 with NCCL send/recv.
    for integers in (True, False):
        rng = np.random.default_rng(77)
        n, m = 3000, 4000
        rows = np.concatenate([np.full(5000, 11), rng.integers(0, n, 30000)])
        cols = rng.integers(0, m, rows.shape[0])
        lin = np.unique(rows * m + cols)
        ops, devs = {}, {}
        for k, X in enumerate("BCD"):
            l2 = np.unique((lin // m) * m + (lin % m + k) % m)  # shifted copies, overlapping
            v = (rng.integers(-3, 4, l2.shape[0]).astype(float) if integers
                 else rng.uniform(-1, 1, l2.shape[0]))
            ops[X] = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([l2 // m, l2 % m], 1), v)
            devs[X] = H.DeviceTensor.upload(ctx, ops[X])
        H.partition_universe(ctx, devs["B"], world)
        A, _ = H.spadd3(ctx, devs["B"], devs["C"], devs["D"], first=rank, count=1, pieces=world, stats=False)
        span = A.global_span()
        F = A.gather_rows(0)
        if rank == 0:
            got = F.download()
            want = oracle_exec.oracle_execute("spadd3", ops, "row", world)["out"]
            g = (got.levels[1].rowptr(), got.levels[1].crd, got.vals)
            ok = np.array_equal(g[0], want[0]) and np.array_equal(g[1], want[1])
            if integers:
                ok = ok and np.array_equal(g[2], want[2])
            else:
                ok = ok and np.all(np.abs(g[2] - want[2]) <= 1e-10 * np.maximum(np.abs(want[2]), 1e-300))
            print(f"[mgpu world={world}] spadd3 {'int' if integers else 'real'}: {'OK' if ok else 'MISMATCH'} "
                  f"span={span} nnz={len(want[1])}", flush=True)
            failures += 0 if ok else 1
            F.close()
        A.close()
        for d in devs.values():
            d.close()
    # Uneven colour blocks (spd_context_set_colour_blocks): P = 5 x world
    # colours, each GPU a contiguous block of a different size; the leaf ops on
    # the whole matrix and on a piece placed by the blocks, SpAdd3 by blocks.
    from paper_2207_13901_b200.distributed import block_owned_rows
    P = 5 * world
    rng = np.random.default_rng(2024)
    costs = rng.uniform(0.2, 3.0, P)
    bounds = H.split_colour_blocks(costs, world)
    n, m = 3000, 2500
    rows = np.concatenate([np.full(25000, 13), rng.integers(0, n, 60000)])
    cols = rng.integers(0, m, rows.shape[0])
    B = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, cols], 1),
                            rng.integers(1, 5, rows.shape[0]).astype(float))
    rp = B.levels[1].rowptr()
    Cm = K.dense(rng, (m, 32), "dd", True)
    cv = K.dense(rng, (m,), "d", True)
    Cd, cd = torch.from_numpy(Cm.vals).to(dev), torch.from_numpy(cv.vals).to(dev)
    H.set_colour_blocks(ctx, P, bounds)
    first, count = int(bounds[rank]), int(bounds[rank + 1] - bounds[rank])
    Bd = H.DeviceTensor.upload(ctx, B)
    whole = H.DeviceTensor.upload(ctx, B) if rank == 0 else None
    piece, _ = H.DeviceTensor.place(ctx, whole, (n, m), H.parse_format("ds"), "nonzero")
    for schedule in ("nonzero", "row"):
        for name, T in (("whole", Bd), ("placed", piece)):
            if name == "placed" and schedule == "row":
                continue  # the piece follows the nonzero blocks
            cols_ = H.partition_universe(ctx, T, P) if schedule == "row" else H.partition_nonzero(ctx, T, 1, P)
            own = block_owned_rows(owned_rows(cols_, rp, schedule, n), bounds)
            for kernel, width in (("spmm", 32), ("spmv", 1)):
                out = torch.zeros(n * width, dtype=torch.float64, device=dev)
                if kernel == "spmm":
                    H.spmm(ctx, T, Cd, 32, out, first=first, count=count, pieces=P)
                else:
                    H.spmv(ctx, T, cd, out, first=first, count=count, pieces=P)
                gathered = [torch.zeros_like(out) for _ in range(world)]
                dist.all_gather(gathered, out)
                if rank == 0:
                    got = assemble([x.cpu().numpy() for x in gathered], own, width, n)
                    t = {"B": B, "C": Cm} if kernel == "spmm" else {"B": B, "c": cv}
                    want = np.asarray(oracle_exec.oracle_execute(kernel, t, schedule, P)["out"]).reshape(n, width)
                    ok = np.array_equal(got, want)
                    print(f"[mgpu world={world}] blocks {[int(b) for b in bounds]} {name} {kernel} {schedule}: "
                          f"{'OK' if ok else 'MISMATCH'}", flush=True)
                    failures += 0 if ok else 1
    # SpAdd3 over the blocks of a row split
    D2 = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, (cols + 1) % m], 1),
                             rng.integers(1, 5, rows.shape[0]).astype(float))
    D3 = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, (cols + 2) % m], 1),
                             rng.integers(1, 5, rows.shape[0]).astype(float))
    d2, d3 = H.DeviceTensor.upload(ctx, D2), H.DeviceTensor.upload(ctx, D3)
    H.partition_universe(ctx, Bd, P)
    A, _ = H.spadd3(ctx, Bd, d2, d3, first=first, count=count, pieces=P)
    F = A.gather_rows(0)
    if rank == 0:
        g = F.download()
        want = oracle_exec.oracle_execute("spadd3", {"B": B, "C": D2, "D": D3}, "row", P)["out"]
        ok = (np.array_equal(g.levels[1].rowptr(), want[0]) and np.array_equal(g.levels[1].crd, want[1]) and
              np.array_equal(g.vals, want[2]))
        print(f"[mgpu world={world}] blocks {[int(b) for b in bounds]} spadd3 row: {'OK' if ok else 'MISMATCH'}", flush=True)
        failures += 0 if ok else 1
        F.close()
    A.close()
    for d in (d2, d3, Bd, piece):
        d.close()
    if whole is not None:
        whole.close()
    H.set_colour_blocks(ctx, P, None)

    ctx.close()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_RESULT", "PASS" if failures == 0 else f"FAIL ({failures})", flush=True)
        sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
