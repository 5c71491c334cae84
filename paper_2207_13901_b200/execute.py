"""execute() for the six hot-path statements on the GPU.

Mirrors the reference's `execute(plan, tensors, machine, residency, mode)`
(sim.hpp:121-122, sim.cpp:816-1010) for the statements of SURVEY.md 8d: the
plan's partition step (universe "row" or nonzero split) runs as GPU kernels,
the leaf runs on sm_100a, colour partials are combined deterministically,
and the output is assembled like assemble_output (sim.cpp:647-789):
dense outputs for SpMV / SpMM / SpMTTKRP, pattern reuse for SDDMM / SpTTV,
two-phase union assembly for SpAdd3.  Statements outside the six raise
SpdValidationError("unsupported on gpu") -- there is no CPU fallback.
"""
from __future__ import annotations

import numpy as np

from . import host as H
from ._native import SpdValidationError

STATEMENTS = {
    "a(i) = B(i, j) * c(j)": "spmv",
    "A(i, j) = B(i, k) * C(k, j)": "spmm",
    "A(i, j) = B(i, j) * C(i, k) * D(k, j)": "sddmm",
    "A(i, j) = B(i, j, k) * c(k)": "spttv",
    "A(i, l) = B(i, j, k) * C(j, l) * D(k, l)": "spmttkrp",
    "A(i, j) = B(i, j) + C(i, j) + D(i, j)": "spadd3",
}


def _dense_dev(t: H.SparseTensor, torch):
    return torch.from_numpy(np.ascontiguousarray(t.vals)).cuda()


def partition(ctx, B: H.DeviceTensor, schedule: str, pieces: int):
    """The plan's partition step for B (PlanLoop colours)."""
    if schedule == "row":
        return H.partition_universe(ctx, B, pieces)
    if schedule == "nonzero":
        return H.partition_nonzero(ctx, B, B.num_levels() - 1, pieces)
    raise SpdValidationError(f"unknown schedule '{schedule}'")


def execute(kernel: str, tensors: dict, schedule: str, pieces: int, ctx: H.Context | None = None):
    """Runs one statement over host tensors; returns (out, Stats, colours) with
    `out` in the layout of oracle_execute: dense ndarray / vals / (rowptr, crd, vals)."""
    import torch

    kernel = STATEMENTS.get(kernel, kernel)
    own = ctx is None
    if own:
        ctx = H.Context(0)
    try:
        B = H.DeviceTensor.upload(ctx, tensors["B"])
        cols = partition(ctx, B, schedule, pieces)
        Bt = tensors["B"]
        if kernel == "spmv":
            c = _dense_dev(tensors["c"], torch)
            a = torch.empty(Bt.dims[0], dtype=torch.float64, device="cuda")
            st = H.spmv(ctx, B, c, a, pieces=pieces)
            out = a.cpu().numpy()
        elif kernel == "spmm":
            Cm = tensors["C"]
            N = Cm.dims[1]
            Cd = _dense_dev(Cm, torch)
            A = torch.empty(Bt.dims[0] * N, dtype=torch.float64, device="cuda")
            st = H.spmm(ctx, B, Cd, N, A, pieces=pieces)
            out = A.cpu().numpy().reshape(Bt.dims[0], N)
        elif kernel == "sddmm":
            Cm, Dm = tensors["C"], tensors["D"]
            K = Cm.dims[1]
            if Dm.format.mode_order == (1, 0):
                dk, dj = 1, K           # D stored j-major ("dd:1,0")
            else:
                dk, dj = Dm.dims[1], 1  # D stored k-major ("dd")
            A = torch.empty(max(Bt.nnz(), 1), dtype=torch.float64, device="cuda")
            st = H.sddmm(ctx, B, _dense_dev(Cm, torch), _dense_dev(Dm, torch), K, dk, dj, A,
                         pieces=pieces)
            out = A.cpu().numpy()[: Bt.nnz()]
        elif kernel == "spttv":
            F = Bt.levels[1].crd.shape[0]
            A = torch.empty(max(F, 1), dtype=torch.float64, device="cuda")
            st = H.spttv(ctx, B, _dense_dev(tensors["c"], torch), A, pieces=pieces)
            out = A.cpu().numpy()[:F]
        elif kernel == "spmttkrp":
            Cm, Dm = tensors["C"], tensors["D"]
            R = Cm.dims[1]
            A = torch.empty(Bt.dims[0] * R, dtype=torch.float64, device="cuda")
            st = H.spmttkrp(ctx, B, _dense_dev(Cm, torch), _dense_dev(Dm, torch), R, A,
                            pieces=pieces)
            out = A.cpu().numpy().reshape(Bt.dims[0], R)
        elif kernel == "spadd3":
            Cd = H.DeviceTensor.upload(ctx, tensors["C"])
            Dd = H.DeviceTensor.upload(ctx, tensors["D"])
            Ad, st = H.spadd3(ctx, B, Cd, Dd, pieces=pieces)
            At = Ad.download()
            out = (At.levels[1].rowptr(), At.levels[1].crd, At.vals)
            for t in (Cd, Dd, Ad):
                t.close()
        else:
            raise SpdValidationError(f"unsupported on gpu: {kernel}")
        B.close()
        return out, st, cols
    finally:
        if own:
            ctx.close()
