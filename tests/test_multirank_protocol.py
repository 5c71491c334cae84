"""N>1 host logic on CPU with world_size-2 gloo (no GPU).

Emulates one process per GPU: every rank computes its colour's partial
output the way the device leaf does (rows it starts store complete sums,
the row it starts but does not finish is a tail partial, the row it
continues is a head partial), the head records are all-gathered (the
backend's NCCL all-gather), each owner adds the later colours' partials in
ascending colour order (the K9 combine), and rank 0 assembles the owned
rows with paper_2207_13901_b200.distributed.  The result must equal the
single-process oracle bit-exactly (integer values) -- for row and nonzero
splits, including a hub row spanning both ranks.
"""
import os
import socket

import numpy as np
import pytest

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(seed=5):
    rng = np.random.default_rng(seed)
    n, m = 200, 150
    rows = np.concatenate([np.full(900, 3), rng.integers(0, n, 1500)])
    cols = rng.integers(0, m, rows.shape[0])
    vals = rng.integers(1, 5, rows.shape[0]).astype(float)
    c = rng.integers(-2, 3, m).astype(float)
    return n, m, rows, cols, vals, c


def _worker(rank, port, schedule, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist

    import oracle_bind as ob
    from paper_2207_13901_b200.distributed import assemble, owned_rows
    from paper_2207_13901_b200.host import Colour, SparseTensor, parse_format

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    n, m, rows, cols, vals, c = _matrix()
    B = SparseTensor.pack((n, m), parse_format("ds"), np.stack([rows, cols], 1), vals)
    rp, crd, v = B.levels[1].rowptr(), B.levels[1].crd, B.vals
    part = ob.partition_universe([rp], n, WORLD) if schedule == "row" else ob.partition_nonzero([rp], len(v), WORLD)
    colours = [Colour(**d) for d in ob.colours_to_tuples(part)]
    W = owned_rows(colours, rp, schedule, n)
    # this rank's leaf (the device computes exactly these partial sums)
    q_lo, q_hi = colours[rank].q
    y = np.zeros(n)
    head = None  # (row, partial, continues past this colour)
    tail = None
    if q_lo <= q_hi:
        r0 = int(np.searchsorted(rp, q_lo, side="right") - 1)
        r1 = int(np.searchsorted(rp, q_hi, side="right") - 1)
        for r in range(r0, r1 + 1):
            s_, e_ = max(rp[r], q_lo), min(rp[r + 1] - 1, q_hi)
            if s_ > e_:
                continue
            part_sum = float(np.sum(v[s_:e_ + 1] * c[crd[s_:e_ + 1]]))
            if rp[r] < q_lo:
                head = (r, part_sum, rp[r + 1] - 1 > q_hi)
            elif rp[r + 1] - 1 > q_hi:
                tail = (r, part_sum)
            else:
                y[r] = part_sum
    heads = [None] * WORLD
    dist.all_gather_object(heads, head)
    if tail is not None:  # K9: owner adds later colours' partials in ascending order
        r, total = tail
        for c2 in range(rank + 1, WORLD):
            h = heads[c2]
            if h is None or h[0] != r:
                break
            total += h[1]
            if not h[2]:
                break
        y[r] = total
    parts = [None] * WORLD
    dist.all_gather_object(parts, y)
    if rank == 0:
        got = assemble(parts, W, 1, n).reshape(-1)
        want, _, _ = ob.spmv(rp, crd, v, c, part)
        q.put((np.array_equal(got, want), W))
    dist.destroy_process_group()


@pytest.mark.parametrize("schedule", ["row", "nonzero"])
def test_two_rank_ownership_and_combine(schedule):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, schedule, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    ok, W = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    # the write ranges tile the rows in order
    assert W[0][0] == 0 and all(W[i][1] + 1 == W[i + 1][0] for i in range(WORLD - 1))


def test_owned_rows_edge_cases():
    from paper_2207_13901_b200.distributed import owned_rows
    from paper_2207_13901_b200.host import Colour

    # P > nnz: leading colours empty, the last owns everything
    rp = np.array([0, 0, 2, 2, 3])  # rows: empty, 2 nnz, empty, 1 nnz
    cols = [Colour((0, -1), (0, -1), (0, -1), (0, -1)), Colour((0, 2), (0, 2), (1, 3), (1, 3))]
    W = owned_rows(cols, rp, "nonzero", 4)
    assert W[0][0] > W[0][1] and W[1] == (0, 3)
    # no positions at all
    cols = [Colour((0, -1), (0, -1), (0, -1), (0, -1))] * 3
    W = owned_rows(cols, np.zeros(5, np.int64), "nonzero", 4)
    assert all(lo > hi for lo, hi in W[:2]) and W[2] == (0, 3)


def test_divide_bounds_host_mirror_matches_oracle():
    """host.divide_bounds (used by the batched grid's column slabs) is the
    reference's divide_bounds (planner.cpp:10-20) as the oracle restates it."""
    import oracle_bind as ob
    from paper_2207_13901_b200.host import divide_bounds

    for n in (0, 1, 5, 7, 32, 100, 16777216):
        for p in (1, 2, 3, 4, 7, 8, 9):
            assert divide_bounds(n, p) == ob.divide_bounds(n, p)


def _batched_worker(rank, port, grid, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist

    import oracle_bind as ob
    import spd_kernels as K
    from paper_2207_13901_b200.host import divide_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    Px, Py = grid
    rng = np.random.default_rng(3)
    n, m, N = 60, 40, 10
    B = K.random_sparse(rng, (n, m), "ds", 0.2, True)
    Cm = K.dense(rng, (m, N), "dd", True)
    rp, crd, v = B.levels[1].rowptr(), B.levels[1].crd, B.vals
    # rank -> worker (x, y) (machine.cpp:88-92); rows of colour x, slab y of C
    x, y = divmod(rank, Py)
    (r0, r1) = divide_bounds(n, Px)[x]
    (c0, c1) = divide_bounds(N, Py)[y]
    C = Cm.vals.reshape(m, N)[:, c0:c1 + 1]  # the only part of C this rank holds
    blk = np.zeros((max(r1 - r0 + 1, 0), c1 - c0 + 1))
    for i in range(r0, r1 + 1):
        for p in range(rp[i], rp[i + 1]):
            blk[i - r0] += v[p] * C[crd[p]]
    work = int(rp[r1 + 1] - rp[r0]) * (c1 - c0 + 1) if r0 <= r1 else 0
    got = [None] * WORLD
    dist.all_gather_object(got, (r0, r1, c0, c1, blk, work))
    if rank == 0:
        A = np.zeros((n, N))
        works = [0] * WORLD
        for w, (a, b, lo, hi, bl, wk) in enumerate(got):
            A[a:b + 1, lo:hi + 1] = bl
            works[w] = wk
        run = ob.RefRun("A(i, j) = B(i, k) * C(k, j)",
                        "divide(i, io, ii, M.x); divide(j, jo, ji, M.y); reorder(io, jo, ii, ji, k); "
                        "distribute(io, M.x); distribute(jo, M.y); communicate({B}, io); communicate({A, C}, jo)",
                        f"x={Px},y={Py}", "dd", K.ref_inputs("spmm", {"B": B, "C": Cm})).ok()
        ok = np.array_equal(A.reshape(-1), run.output()[1]) and works == run.stats()["work"]
        q.put(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(1, 2), (2, 1)])
def test_two_rank_batched_grid(grid):
    """SpDISTAL-Batched on a 2-rank grid: each rank holds only its column
    slab of C; the assembled blocks and per-worker work equal the
    reference's plan + execute with the same grid."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batched_worker, args=(r, port, grid, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok
