"""Host-side plumbing for one process per GPU (torch.distributed bootstrap).

The data path between GPUs is inside libspdistal_b200.so (NCCL all-gather of
boundary records, rowwalk.cuh); this module only
  * bootstraps the backend's NCCL communicator from a torch.distributed group
    (the 128-byte ncclUniqueId travels over whatever backend the group uses);
  * states the output-ownership rule the device code applies (k_setup,
    leaf_rows.cu): colour c stores rows W_c, and the W_c tile [0, rows);
  * assembles a distributed dense output on one rank for checking/download.
"""
from __future__ import annotations

import numpy as np


def init_comm(ctx, dist, rank: int, world: int, device=None):
    """Create the backend communicator of `ctx` for this rank."""
    import torch

    from .host import Context

    dev = device if device is not None else "cpu"
    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(Context.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    ctx.init_comm(bytes(uid.cpu().numpy().tobytes()), rank, world)


def owned_rows(colours, rowptr, schedule: str, nrows: int):
    """W_c for every colour: its row block for a universe ("row") split; for a
    nonzero split, from the first row starting inside the colour up to the row
    before the next colour's first such row (the first non-empty colour starts
    at row 0; with no positions at all the last colour owns every row).
    `colours` are host.Colour-like objects with `.q` and `.top` spans."""
    P = len(colours)
    if schedule == "row":
        return [tuple(c.top) for c in colours]
    rowptr = np.asarray(rowptr)
    starts = []
    for c in colours:
        lo, hi = c.q
        if lo > hi:
            starts.append(None)
            continue
        o = int(np.searchsorted(rowptr, lo, side="right") - 1)
        starts.append(o if rowptr[o] == lo else o + 1)
    W = [None] * P
    nxt, first = nrows, None
    for c in range(P - 1, -1, -1):
        if starts[c] is None:
            W[c] = (nxt, nxt - 1)
        else:
            W[c] = (starts[c], nxt - 1)
            nxt = starts[c]
            first = c
    if first is not None:
        W[first] = (0, W[first][1])
    else:
        W[P - 1] = (0, nrows - 1)
    return W


def assemble(parts, W, width: int, nrows: int):
    """Dense output from every rank's (full-size) buffer, keeping W_c rows of
    rank c."""
    out = np.zeros((nrows, width))
    for r, (lo, hi) in enumerate(W):
        if lo <= hi:
            out[lo:hi + 1] = np.asarray(parts[r]).reshape(nrows, width)[lo:hi + 1]
    return out


def assemble_positions(parts, spans, npos: int):
    """Output vals on an input's pattern (SDDMM, SpTTV's fibre level) from
    every rank's full-size buffer, keeping rank c's position span spans[c]
    (the colour's q range for SDDMM, its owned fibres for SpTTV)."""
    out = np.zeros(npos)
    for r, (lo, hi) in enumerate(spans):
        if lo <= hi:
            out[lo:hi + 1] = np.asarray(parts[r]).reshape(-1)[lo:hi + 1]
    return out


def leaf_rowptr(rp1, rp2):
    """Rows i of a dss CSF -> leaf positions (rp2[rp1[i]]), the derived row
    pointer the SpMTTKRP leaf walks (k_leaf_rowptr, leaf_rows.cu)."""
    return np.asarray(rp2)[np.asarray(rp1)]


def csr_offsets(counts):
    """Global position offset of every rank's row-block piece of an assembled
    CSR output (SpAdd3): the exclusive prefix sum of the all-gathered piece
    sizes (spd_spadd3 with a communicator, spd_tensor_global_span)."""
    c = np.asarray(counts, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(c)[:-1]]), int(c.sum())


def assemble_csr(pieces, nrows: int):
    """One CSR from row-block pieces [(row_lo, row_hi, rowptr_local, crd,
    vals)] in rank order; rowptr_local has row_hi - row_lo + 2 entries from 0."""
    rp = np.zeros(nrows + 1, np.int64)
    crds, vals = [], []
    base = 0
    for lo, hi, lrp, c, v in pieces:
        if lo <= hi:
            rp[lo + 1:hi + 2] = base + np.asarray(lrp)[1:]
        crds.append(np.asarray(c))
        vals.append(np.asarray(v))
        base += len(c)
    # rows outside every piece keep the running offset
    for i in range(1, nrows + 1):
        if rp[i] < rp[i - 1]:
            rp[i] = rp[i - 1]
    return rp, (np.concatenate(crds) if crds else np.zeros(0, np.int64)), \
        (np.concatenate(vals) if vals else np.zeros(0))


def colour_blocks(pieces: int, gpus: int):
    """The colour-to-GPU mapping of a P-colour plan on G GPUs (the
    integration adapter's execute_gpu, the library's require_partition):
    cmax = ceil(P / G) consecutive colours per GPU, rank r running
    [r * cmax, min(P, (r + 1) * cmax)); only as many GPUs as get a colour are
    used.  Returns [(first, count)] per used GPU."""
    g = max(1, min(gpus, max(pieces, 1)))
    cmax = -(-max(pieces, 1) // g)
    used = max(1, -(-max(pieces, 1) // cmax))
    return [(r * cmax, min(cmax, pieces - r * cmax)) for r in range(used)]


def block_owned_rows(W, bounds):
    """Owned output rows per GPU under colour blocks (spd_context_colour_blocks):
    GPU r stores the union of W_c over its block [bounds[r], bounds[r + 1]) --
    contiguous, since the W_c tile the rows in colour order.  Returns
    [(lo, hi)] per GPU, (0, -1) when its block stores no row."""
    out = []
    for r in range(len(bounds) - 1):
        rng = [(lo, hi) for lo, hi in W[bounds[r]:bounds[r + 1]] if lo <= hi]
        out.append((min(lo for lo, _ in rng), max(hi for _, hi in rng)) if rng else (0, -1))
    return out


def unpack_head_records(stage, bounds, own, cmax):
    """Host mirror of k_unpack_heads: the all-gathered head records (cmax
    slots per rank, rank r's block in its first bounds[r+1]-bounds[r] slots)
    to one record per colour; the caller's own block is taken from `own`
    (its records by colour).  Returns the per-colour list."""
    P = int(bounds[-1])
    out = [None] * P
    for r in range(len(bounds) - 1):
        for j in range(int(bounds[r + 1] - bounds[r])):
            c = int(bounds[r]) + j
            out[c] = own[c] if c in own else stage[r * cmax + j]
    return out

