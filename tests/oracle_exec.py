"""TEST INFRASTRUCTURE: run a kernel through the CPU restatement (oracle) or
the reference, returning results in one comparable form:

    {"out": dense ndarray | vals ndarray | (rowptr, crd, vals),
     "work": [per colour], "combines": int, "imbalance": float}
"""
import numpy as np

import oracle_bind as ob
from spd_kernels import KERNELS, OUTPUT, ROW, ref_inputs


def _rp(t, level):
    return t.levels[level].rowptr()


def oracle_colours(kernel, tensors, schedule, pieces):
    B = tensors["B"]
    rps = B.compressed_rowptrs()
    if schedule == "row":
        return ob.partition_universe(rps, B.dims[0], pieces)
    return ob.partition_nonzero(rps, B.nnz(), pieces)


def oracle_execute(kernel, tensors, schedule, pieces, nthreads=0):
    cols = oracle_colours(kernel, tensors, schedule, pieces)
    B = tensors["B"]
    if kernel == "spmv":
        out, work, comb = ob.spmv(_rp(B, 1), B.levels[1].crd, B.vals, tensors["c"].vals, cols, nthreads)
    elif kernel == "spmm":
        Cm = tensors["C"]
        out, work, comb = ob.spmm(_rp(B, 1), B.levels[1].crd, B.vals, Cm.vals, Cm.dims[1], cols, nthreads)
    elif kernel == "sddmm":
        Cm, Dm = tensors["C"], tensors["D"]
        K = Cm.dims[1]
        out, work, comb = ob.sddmm(_rp(B, 1), B.levels[1].crd, B.vals, Cm.vals, Dm.vals, K,
                                   1, K, cols, nthreads)  # D stored j-major (dd:1,0)
    elif kernel == "spttv":
        out, work, comb = ob.spttv(_rp(B, 1), B.levels[1].crd, _rp(B, 2), B.levels[2].crd, B.vals,
                                   tensors["c"].vals, cols, nthreads)
    elif kernel == "spmttkrp":
        Cm, Dm = tensors["C"], tensors["D"]
        out, work, comb = ob.spmttkrp(_rp(B, 1), B.levels[1].crd, _rp(B, 2), B.levels[2].crd,
                                      B.vals, Cm.vals, Dm.vals, Cm.dims[1], cols, nthreads)
    elif kernel == "spadd3":
        ops = [(_rp(tensors[X], 1), tensors[X].levels[1].crd, tensors[X].vals) for X in "BCD"]
        out = ob.spadd3(ops, nthreads)
        rps = [o[0] for o in ops]
        work = np.zeros(pieces, np.int64)
        for c, col in enumerate(cols):
            lo, hi = col.top_lo, col.top_hi
            if lo <= hi:
                work[c] = sum(int(r[hi + 1] - r[lo]) for r in rps)
        comb = 0
    else:
        raise KeyError(kernel)
    work = np.asarray(work, np.int64)
    return dict(out=out, work=work.tolist(), combines=int(comb),
                imbalance=ob.port().or_imbalance(ob._p(work), pieces), colours=ob.colours_to_tuples(cols))


def reference_execute(kernel, tensors, schedule, pieces, mode="seq"):
    spec = KERNELS[kernel]
    sched = ROW if schedule == "row" else spec["nonzero"]
    out_name = OUTPUT[kernel]
    run = ob.RefRun(spec["expr"], sched, pieces, spec["formats"][out_name],
                    ref_inputs(kernel, tensors), mode=mode).ok()
    levels, vals = run.output()
    B = tensors["B"]
    if kernel in ("spmv",):
        out = vals
    elif kernel == "spmm":
        out = vals.reshape(B.dims[0], tensors["C"].dims[1])
    elif kernel == "spmttkrp":
        out = vals.reshape(B.dims[0], tensors["C"].dims[1])
    elif kernel in ("sddmm", "spttv"):
        out = vals
    else:  # spadd3: (rowptr, crd, vals)
        pos, crd = levels[1][1], levels[1][2]
        rp = np.empty(pos.shape[0] + 1, np.int64)
        rp[:-1] = pos[:, 0]
        rp[-1] = pos[-1, 1] + 1 if pos.shape[0] else 0
        out = (rp, crd, vals)
    st = run.stats()
    return dict(out=out, work=st["work"], combines=st["combines"], imbalance=st["imbalance"],
                run=run)
