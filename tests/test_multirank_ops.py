"""N>1 host protocols of SDDMM, the CSF kernels and SpAdd3 on CPU with
world_size-2 gloo (no GPU), like test_multirank_protocol.py for SpMV/SpMM.

Every rank computes its colour's share the way the device does:
  * SDDMM: the vals of its own positions (output on B's pattern, disjoint:
    no collective) -- rank 0 keeps each rank's q span;
  * SpTTV / SpMTTKRP (nonzero split of the leaf level): complete fibres / rows
    directly, the boundary fibre / row as head / tail partials that the owner
    combines in ascending colour order after an all-gather of head records;
  * SpAdd3 (row split): the union of its row block as a local CSR piece, the
    piece sizes all-gathered into global pos offsets, rank 0 concatenating.
The assembled result must equal the single-process oracle bit-exactly
(integer values)."""
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


def _run(target, *args):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, port, q) + args) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _init(rank, port):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    return dist


def _segment_partials(rp, q_lo, q_hi, value_of_range):
    """The row walk of one colour over row pointer rp: complete rows, the head
    row (began before the colour: row, partial, continues past it) and the tail
    row (continues past it: row, partial)."""
    full, head, tail = {}, None, None
    if q_lo > q_hi:
        return full, head, tail
    r0 = int(np.searchsorted(rp, q_lo, side="right") - 1)
    r1 = int(np.searchsorted(rp, q_hi, side="right") - 1)
    for r in range(r0, r1 + 1):
        s_, e_ = max(rp[r], q_lo), min(rp[r + 1] - 1, q_hi)
        if s_ > e_:
            continue
        val = value_of_range(s_, e_)
        if rp[r] < q_lo:
            head = (r, val, rp[r + 1] - 1 > q_hi)
        elif rp[r + 1] - 1 > q_hi:
            tail = (r, val)
        else:
            full[r] = val
    return full, head, tail


def _combine(dist, rank, full, head, tail, width, nrows):
    """All-gather of head records, then the owner's ascending-colour sum (K9)."""
    heads = [None] * WORLD
    dist.all_gather_object(heads, head)
    out = np.zeros((nrows, width))
    for r, v in full.items():
        out[r] = v
    if tail is not None:
        r, total = tail
        total = np.array(total, dtype=float)
        for c2 in range(rank + 1, WORLD):
            h = heads[c2]
            if h is None or h[0] != r:
                break
            total = total + h[1]
            if not h[2]:
                break
        out[r] = total
    return out


def _csf(rng):
    import spd_kernels as K

    t = K.instance("spmttkrp", rng, integers=True, rank=6, max_dim=25)
    t["B"] = K.random_sparse(rng, t["B"].dims, "dss", 0.25, True)
    return t


def _sddmm_worker(rank, port, q):
    dist = _init(rank, port)
    import oracle_bind as ob
    import spd_kernels as K
    from paper_2207_13901_b200.distributed import assemble_positions

    rng = np.random.default_rng(8)
    t = K.instance("sddmm", rng, integers=True, max_dim=30)
    B, Cm, Dm = t["B"], t["C"], t["D"]
    rp, crd, v = B.levels[1].rowptr(), B.levels[1].crd, B.vals
    n, m = B.dims
    Kd = Cm.dims[1]
    Cmat = Cm.vals.reshape(n, Kd)
    Dmat = Dm.vals.reshape(m, Kd)  # dd:1,0 -> D[j, k]
    part = ob.partition_nonzero([rp], len(v), WORLD)
    spans = [tuple(x["q"]) for x in ob.colours_to_tuples(part)]
    lo, hi = spans[rank]
    a = np.zeros(len(v))
    for p in range(lo, hi + 1):
        i = int(np.searchsorted(rp, p, side="right") - 1)
        a[p] = v[p] * float(np.dot(Cmat[i], Dmat[crd[p]]))
    parts = [None] * WORLD
    dist.all_gather_object(parts, a)  # test transport only; the device keeps its span
    if rank == 0:
        got = assemble_positions(parts, spans, len(v))
        want, _, _ = ob.sddmm(rp, crd, v, Cm.vals, Dm.vals, Kd, 1, Kd, part)
        q.put(bool(np.array_equal(got, want)))
    dist.destroy_process_group()


def _spttv_worker(rank, port, q):
    dist = _init(rank, port)
    import oracle_bind as ob
    import spd_kernels as K
    from paper_2207_13901_b200.distributed import assemble_positions, owned_rows
    from paper_2207_13901_b200.host import Colour

    rng = np.random.default_rng(12)
    t = K.instance("spttv", rng, integers=True, max_dim=25)
    B, c = t["B"], t["c"]
    rp1, crd1 = B.levels[1].rowptr(), B.levels[1].crd
    rp2, crd2, v = B.levels[2].rowptr(), B.levels[2].crd, B.vals
    F = len(crd1)
    part = ob.partition_nonzero([rp1, rp2], len(v), WORLD)
    cols = [Colour(**d) for d in ob.colours_to_tuples(part)]
    lo, hi = cols[rank].q
    full, head, tail = _segment_partials(rp2, lo, hi, lambda s, e: float(np.sum(v[s:e + 1] * c.vals[crd2[s:e + 1]])))
    out = _combine(dist, rank, full, head, tail, 1, F).reshape(-1)
    W = owned_rows(cols, rp2, "nonzero", F)  # owned fibres of the leaf level
    parts = [None] * WORLD
    dist.all_gather_object(parts, out)
    if rank == 0:
        got = assemble_positions(parts, W, F)
        want, _, _ = ob.spttv(rp1, crd1, rp2, crd2, v, c.vals, part)
        q.put(bool(np.array_equal(got, want)))
    dist.destroy_process_group()


def _spmttkrp_worker(rank, port, q):
    dist = _init(rank, port)
    import oracle_bind as ob
    from paper_2207_13901_b200.distributed import assemble, leaf_rowptr, owned_rows
    from paper_2207_13901_b200.host import Colour

    rng = np.random.default_rng(13)
    t = _csf(rng)
    B, Cm, Dm = t["B"], t["C"], t["D"]
    I, J, Kd = B.dims
    R = Cm.dims[1]
    rp1, crd1 = B.levels[1].rowptr(), B.levels[1].crd
    rp2, crd2, v = B.levels[2].rowptr(), B.levels[2].crd, B.vals
    Cmat, Dmat = Cm.vals.reshape(J, R), Dm.vals.reshape(Kd, R)
    jleaf = np.repeat(crd1, np.diff(rp2))  # middle coordinate of every leaf
    R_i = leaf_rowptr(rp1, rp2)
    part = ob.partition_nonzero([rp1, rp2], len(v), WORLD)
    cols = [Colour(**d) for d in ob.colours_to_tuples(part)]
    lo, hi = cols[rank].q

    def val(s, e):
        acc = np.zeros(R)
        for p in range(s, e + 1):
            acc += (v[p] * Cmat[jleaf[p]]) * Dmat[crd2[p]]
        return acc

    full, head, tail = _segment_partials(R_i, lo, hi, val)
    out = _combine(dist, rank, full, head, tail, R, I)
    W = owned_rows(cols, R_i, "nonzero", I)
    parts = [None] * WORLD
    dist.all_gather_object(parts, out)
    if rank == 0:
        got = assemble(parts, W, R, I)
        want, _, _ = ob.spmttkrp(rp1, crd1, rp2, crd2, v, Cm.vals, Dm.vals, R, part)
        q.put(bool(np.array_equal(got.reshape(-1), np.asarray(want).reshape(-1))))
    dist.destroy_process_group()


def _spadd3_worker(rank, port, q):
    dist = _init(rank, port)
    import oracle_bind as ob
    import spd_kernels as K
    from paper_2207_13901_b200.distributed import assemble_csr, csr_offsets
    from paper_2207_13901_b200.host import divide_bounds

    rng = np.random.default_rng(21)
    t = K.instance("spadd3", rng, integers=True, max_dim=40)
    ops = [(t[x].levels[1].rowptr(), t[x].levels[1].crd, t[x].vals) for x in "BCD"]
    n = len(ops[0][0]) - 1
    r0, r1 = divide_bounds(n, WORLD)[rank]
    # this rank's rows: the union of the three operands, crd sorted, values summed in term order
    lrp, lcrd, lval = [0], [], []
    for i in range(r0, r1 + 1):
        row = {}
        for rp, crd, v in ops:
            for p in range(rp[i], rp[i + 1]):
                row[int(crd[p])] = row.get(int(crd[p]), 0.0) + v[p]
        for j in sorted(row):
            lcrd.append(j)
            lval.append(row[j])
        lrp.append(len(lcrd))
    sizes = [None] * WORLD
    dist.all_gather_object(sizes, len(lcrd))  # the backend's one-int64-per-GPU all-gather
    offs, total = csr_offsets(sizes)
    pieces = [None] * WORLD
    dist.all_gather_object(pieces, (r0, r1, lrp, lcrd, lval))
    if rank == 0:
        rp, crd, vals = assemble_csr(pieces, n)
        w_rp, w_crd, w_vals = ob.spadd3(ops)
        ok = (np.array_equal(rp, w_rp) and np.array_equal(crd, w_crd) and np.array_equal(vals, w_vals)
              and total == len(w_crd) and list(offs) == [int(w_rp[divide_bounds(n, WORLD)[r][0]]) for r in range(WORLD)])
        q.put(bool(ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("worker", ["sddmm", "spttv", "spmttkrp", "spadd3"])
def test_two_rank_protocol(worker):
    target = {"sddmm": _sddmm_worker, "spttv": _spttv_worker, "spmttkrp": _spmttkrp_worker,
              "spadd3": _spadd3_worker}[worker]
    assert _run(target)


def test_colour_blocks_tile_the_partition():
    """Every colour runs on exactly one GPU, in ascending blocks, every used
    GPU gets at least one colour (the execute_gpu / require_partition rule)."""
    from paper_2207_13901_b200.distributed import colour_blocks

    for P in range(1, 40):
        for G in range(1, 10):
            blocks = colour_blocks(P, G)
            assert 1 <= len(blocks) <= min(P, G)
            cmax = blocks[0][1]
            seen = []
            for r, (f, c) in enumerate(blocks):
                assert c >= 1 and f == r * cmax and c <= cmax
                seen += list(range(f, f + c))
            assert seen == list(range(P))
    assert colour_blocks(8, 8) == [(c, 1) for c in range(8)]  # the bench: one colour per GPU
    assert colour_blocks(5, 4) == [(0, 2), (2, 2), (4, 1)]
