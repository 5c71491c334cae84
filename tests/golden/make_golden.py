#!/usr/bin/env python3
"""Generates tests/golden/cases.npz + index.json from the REFERENCE itself.

Runs the (patched, see oracle/patch_ref.py) reference pipeline -- plan() and
execute() of /root/reference/proj/core, built into oracle/_ref -- on seeded
small instances of the six kernels under row and nonzero schedules and
several piece counts, plus the reference tests' known-answer tensors
(test_util.hpp:16-27) and the SURVEY 9.6 hub-row example, and stores inputs,
partition bounds, bundle subsets, outputs and Stats.  The committed fixtures
pin the oracle and the GPU path on machines where /root/reference is absent.

    python tests/golden/make_golden.py      (needs /root/reference)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]

import oracle_bind as ob  # noqa: E402
import spd_kernels as K  # noqa: E402
from oracle_exec import reference_execute  # noqa: E402
from paper_2207_13901_b200.host import SparseTensor, parse_format  # noqa: E402


def kat_tensors():
    """Known-answer inputs of the reference's own tests + SURVEY 9.6."""
    csr = SparseTensor.pack((3, 3), parse_format("ds"), [[0, 0], [0, 1], [1, 1], [2, 2]], [2, 3, 4, 5])
    straddle = SparseTensor.pack((2, 4), parse_format("ds"), [[0, 0], [0, 1], [0, 2], [1, 3]], [1, 2, 3, 4])
    # 6x8, hub row 0 with 7 nnz, empty rows 1 and 3: 12 nnz
    hub_coords = [[0, j] for j in range(7)] + [[2, 5], [4, 1], [4, 6], [5, 2], [5, 7]]
    hub = SparseTensor.pack((6, 8), parse_format("ds"), hub_coords, np.arange(1, 13, dtype=float))
    return {"csr_example": csr, "straddle_example": straddle, "hub_6x8": hub}


def ones_vec(m):
    return SparseTensor.pack((m,), parse_format("d"), [[j] for j in range(m)], np.ones(m))


def add_tensor(store, key, t):
    store[key + "/vals"] = t.vals
    for l, lv in enumerate(t.levels):
        if lv.kind == "s":
            store[f"{key}/pos{l}"] = lv.pos
            store[f"{key}/crd{l}"] = lv.crd
    return dict(dims=list(t.dims), format="".join(t.format.kinds) +
                (":" + ",".join(map(str, t.format.mode_order)) if list(t.format.mode_order) != sorted(t.format.mode_order) else ""))


def main():
    store = {}
    index = []
    rng = np.random.default_rng(20261018)
    cases = []
    for name, B in kat_tensors().items():
        for P in (1, 2, 3, 4, 5):
            for sched in ("row", "nonzero"):
                cases.append(("spmv", {"B": B, "c": ones_vec(B.dims[1])}, sched, P, "kat:" + name))
    for kernel in K.KERNELS:
        for sched in ("row", "nonzero"):
            if sched == "nonzero" and K.KERNELS[kernel]["nonzero"] is None:
                continue
            for P in (1, 2, 3, 4, 7):
                for rep in range(2):
                    integers = rep == 0
                    cases.append((kernel, K.instance(kernel, rng, integers=integers), sched, P,
                                  f"random:{'int' if integers else 'real'}"))
    for ci, (kernel, tensors, sched, P, origin) in enumerate(cases):
        res = reference_execute(kernel, tensors, sched, P)
        run = res["run"]
        key = f"c{ci}"
        entry = dict(kernel=kernel, schedule=sched, pieces=P, origin=origin, key=key, tensors={})
        for tname, t in tensors.items():
            entry["tensors"][tname] = add_tensor(store, f"{key}/{tname}", t)
        out = res["out"]
        if kernel == "spadd3":
            store[f"{key}/out_rowptr"], store[f"{key}/out_crd"], store[f"{key}/out_vals"] = out
        else:
            store[f"{key}/out_vals"] = np.asarray(out).reshape(-1)
        loop = run.loop(0)
        entry["color_bounds"] = loop["bounds"]
        entry["combine"] = run.combine()
        entry["work"] = [int(w) for w in res["work"]]
        entry["combines"] = int(res["combines"])
        entry["imbalance"] = float(res["imbalance"])
        out_name = K.OUTPUT[kernel]
        sb = run.step_bounds(out_name)
        entry["out_bounds"] = sb[1] if sb else None
        # B's bundle subsets per colour (pos/crd of the split-relevant levels, dom, vals)
        Bt = tensors["B"]
        subsets = {}
        for c in range(P):
            for l, lv in enumerate(Bt.levels):
                regions = ["dom"] if lv.kind == "d" else ["pos", "crd"]
                for r in regions:
                    s = run.subset("B", l, r, c)
                    if s is not None:
                        store[f"{key}/B_{r}{l}_c{c}"] = s
                        subsets.setdefault(f"{r}{l}", []).append(c)
            s = run.subset("B", 0, "vals", c)
            store[f"{key}/B_vals_c{c}"] = s
        entry["subsets"] = sorted(subsets)
        index.append(entry)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **store)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=0)
    print(f"{len(index)} cases written")


if __name__ == "__main__":
    main()
