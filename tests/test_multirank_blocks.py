"""Uneven colour blocks per GPU (spd_context_set_colour_blocks) on CPU with
world_size-2 gloo (no GPU).

A plan with more colours than GPUs runs each GPU on a contiguous block of
colours; the bench chooses the blocks with a cost model
(spd_split_colour_blocks, host-only, exercised here through the library).
Every rank computes, colour by colour, the partials the device leaf leaves
(complete rows stored, head / tail records of rows cut by a colour
boundary); the head records travel in the device's layout -- cmax = the
largest block slots per rank, all-gathered, then moved to their colours'
slots (host mirror of k_unpack_heads) -- and each owner adds the later
colours' heads to its tails in ascending colour order (the K9 combine).
Rank 0 assembles the rows each GPU owns under its block
(distributed.block_owned_rows); the result must equal the single-process
oracle bit-exactly (integer values)."""
import os
import socket

import numpy as np
import pytest

WORLD = 2
PIECES = 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(seed=11):
    rng = np.random.default_rng(seed)
    n, m = 240, 180
    # a hub row spanning several colours, a dense head and a sparse tail
    rows = np.concatenate([np.full(700, 5), rng.integers(0, 40, 900), rng.integers(0, n, 300)])
    cols = rng.integers(0, m, rows.shape[0])
    vals = rng.integers(1, 5, rows.shape[0]).astype(float)
    c = rng.integers(-2, 3, m).astype(float)
    return n, m, rows, cols, vals, c


def _colour_records(rp, crd, v, c, q_lo, q_hi, y):
    """One colour's leaf: complete rows into y; (head, tail) records."""
    head = tail = None
    if q_lo > q_hi:
        return head, tail
    r0 = int(np.searchsorted(rp, q_lo, side="right") - 1)
    r1 = int(np.searchsorted(rp, q_hi, side="right") - 1)
    for r in range(r0, r1 + 1):
        s_, e_ = max(rp[r], q_lo), min(rp[r + 1] - 1, q_hi)
        if s_ > e_:
            continue
        part = float(np.sum(v[s_:e_ + 1] * c[crd[s_:e_ + 1]]))
        if rp[r] < q_lo:
            head = (r, part, bool(rp[r + 1] - 1 > q_hi))
        elif rp[r + 1] - 1 > q_hi:
            tail = (r, part)
        else:
            y[r] = part
    return head, tail


def _worker(rank, port, bounds, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist

    import oracle_bind as ob
    from paper_2207_13901_b200.distributed import assemble, block_owned_rows, owned_rows, unpack_head_records
    from paper_2207_13901_b200.host import Colour, SparseTensor, parse_format

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    n, m, rows, cols, vals, c = _matrix()
    B = SparseTensor.pack((n, m), parse_format("ds"), np.stack([rows, cols], 1), vals)
    rp, crd, v = B.levels[1].rowptr(), B.levels[1].crd, B.vals
    part = ob.partition_nonzero([rp], len(v), PIECES)
    colours = [Colour(**d) for d in ob.colours_to_tuples(part)]
    W = owned_rows(colours, rp, "nonzero", n)
    first, last = int(bounds[rank]), int(bounds[rank + 1])
    y = np.zeros(n)
    heads, tails = {}, {}
    for k in range(first, last):
        heads[k], tails[k] = _colour_records(rp, crd, v, c, *colours[k].q, y)
    cmax = int(max(bounds[r + 1] - bounds[r] for r in range(WORLD)))
    mine = [heads[k] for k in range(first, last)] + [None] * (cmax - (last - first))
    gathered = [None] * WORLD
    dist.all_gather_object(gathered, mine)
    stage = [rec for blk in gathered for rec in blk]
    all_heads = unpack_head_records(stage, bounds, heads, cmax)
    for k in range(first, last):  # K9: ascending colour order
        if tails[k] is None:
            continue
        r, total = tails[k]
        for c2 in range(k + 1, PIECES):
            h = all_heads[c2]
            if h is None or h[0] != r:
                break
            total += h[1]
            if not h[2]:
                break
        y[r] = total
    parts = [None] * WORLD
    dist.all_gather_object(parts, y)
    if rank == 0:
        own = block_owned_rows(W, bounds)
        got = assemble(parts, own, 1, n).reshape(-1)
        want, _, _ = ob.spmv(rp, crd, v, c, part)
        q.put((np.array_equal(got, want), own))
    dist.destroy_process_group()


def _run(bounds):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, list(bounds), q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    ok, own = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return ok, own


@pytest.mark.parametrize("bounds", [(0, 1, PIECES), (0, 5, PIECES), (0, 3, PIECES)])
def test_two_rank_uneven_blocks(bounds):
    ok, own = _run(bounds)
    assert ok
    # the GPUs' owned rows tile the output rows in order
    assert own[0][0] == 0 and own[0][1] + 1 == own[1][0]


def test_split_colour_blocks_known_answers():
    from paper_2207_13901_b200.host import split_colour_blocks
    from paper_2207_13901_b200._native import SpdValidationError

    assert list(split_colour_blocks([1.0] * 8, 2)) == [0, 4, 8]
    assert list(split_colour_blocks([1.0] * 8, 4)) == [0, 2, 4, 6, 8]
    # a heavy tail colour: the first GPU takes every light colour
    assert list(split_colour_blocks([1, 1, 1, 1, 1, 1, 6], 2)) == [0, 6, 7]
    # a heavy head colour: it stays alone
    assert list(split_colour_blocks([9, 1, 1, 1, 1], 2)) == [0, 1, 5]
    # every block keeps at least one colour, even at zero cost
    b = split_colour_blocks([0, 0, 0, 10], 3)
    assert b[0] == 0 and b[-1] == 4 and all(b[i + 1] > b[i] for i in range(3)) and b[2] == 3
    # nearest prefix to each r / world of the total
    b = split_colour_blocks(np.arange(1, 17, dtype=float), 4)
    pre = np.concatenate([[0], np.cumsum(np.arange(1, 17))])
    for r in range(1, 4):
        t = pre[-1] * r / 4
        assert abs(pre[b[r]] - t) <= min(abs(pre[b[r] - 1] - t), abs(pre[b[r] + 1] - t))
    for bad in ([1.0], [1.0, -1.0]):
        with pytest.raises(SpdValidationError):
            split_colour_blocks(bad, 2)


def test_block_owned_rows_tile():
    from paper_2207_13901_b200.distributed import block_owned_rows

    W = [(0, 9), (10, 9), (10, 30), (31, 31), (32, 99)]  # colour 1 stores no row
    assert block_owned_rows(W, [0, 2, 5]) == [(0, 9), (10, 99)]
    assert block_owned_rows(W, [0, 1, 2, 5]) == [(0, 9), (0, -1), (10, 99)]
