"""The drop-in: the reference's own pipeline (parse -> validate_schedule ->
plan) with execute() replaced by the ExecMode::Gpu adapter
(integration/gpu_execute.cpp, built into oracle/_ref/libdspar_gpu.so against
the reference headers), compared with the reference's execute()."""
import os

import numpy as np
import pytest

import oracle_bind as ob
import spd_kernels as K
from spd_kernels import KERNELS, OUTPUT, ROW, ref_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu_lib():
    if not os.path.exists(ob.GPU_LIB):
        pytest.skip("integration library not built (make -C oracle integration)")
    return ob.GPU_LIB


@pytest.mark.parametrize("kernel", list(KERNELS))
@pytest.mark.parametrize("schedule", ["row", "nonzero"])
def test_reference_pipeline_with_gpu_execute(gpu_lib, kernel, schedule):
    if schedule == "nonzero" and KERNELS[kernel]["nonzero"] is None:
        pytest.skip("position split rejected for union statements")
    spec = KERNELS[kernel]
    sched = ROW if schedule == "row" else spec["nonzero"]
    rng = np.random.default_rng(99)
    for pieces in (1, 3, 4):
        t = K.instance(kernel, rng, integers=True)
        args = (spec["expr"], sched, pieces, spec["formats"][OUTPUT[kernel]], ref_inputs(kernel, t))
        want = ob.RefRun(*args, mode="seq").ok()
        got = ob.RefRun(*args, mode="gpu", lib=gpu_lib).ok()
        wl, wv = want.output()
        gl, gv = got.output()
        assert np.array_equal(wv, gv)
        for (wk, wp, wc), (gk, gp, gc) in zip(wl, gl):
            assert wk == gk
            if wk == "s":
                assert np.array_equal(wp, gp) and np.array_equal(wc, gc)
        ws, gs = want.stats(), got.stats()
        assert ws["work"] == gs["work"] and ws["combines"] == gs["combines"]
        assert ws["imbalance"] == gs["imbalance"]


def test_unsupported_statement_is_a_validation_error(gpu_lib):
    from paper_2207_13901_b200.host import SparseTensor, parse_format

    B = SparseTensor.pack((4, 4), parse_format("ds"), [[0, 1], [2, 3]], [1.0, 2.0])
    run = ob.RefRun("A(i, j) = B(i, j)", ROW, 2, "ds", {"B": (B, "ds")}, mode="gpu", lib=gpu_lib)
    assert run.status == 2 and "unsupported on gpu" in run.error


BATCHED = ("divide(i, io, ii, M.x); divide(j, jo, ji, M.y); reorder(io, jo, ii, ji, k); "
           "distribute(io, M.x); distribute(jo, M.y); communicate({B}, io); communicate({A, C}, jo)")


@pytest.mark.parametrize("grid", ["x=2,y=2", "x=3,y=2", "x=1,y=3"])
def test_batched_spmm_plan_with_gpu_execute(gpu_lib, grid):
    """The reference's two-loop SpDISTAL-Batched plan (test_planner.cpp:193-225)
    through the adapter: output, per-worker work, imbalance."""
    spec = KERNELS["spmm"]
    rng = np.random.default_rng(7)
    t = K.instance("spmm", rng, integers=True, max_dim=30, rank=10)
    args = (spec["expr"], BATCHED, grid, "dd", ref_inputs("spmm", t))
    want = ob.RefRun(*args, mode="seq").ok()
    got = ob.RefRun(*args, mode="gpu", lib=gpu_lib).ok()
    assert np.array_equal(want.output()[1], got.output()[1])
    ws, gs = want.stats(), got.stats()
    assert ws["work"] == gs["work"] and ws["combines"] == gs["combines"] and ws["imbalance"] == gs["imbalance"]


BATCHED_MTTKRP = ("divide(i, io, ii, M.x); divide(l, lo, li, M.y); reorder(io, lo, ii, j, k, li); "
                  "distribute(io, M.x); distribute(lo, M.y); communicate({B}, io); communicate({A, C, D}, lo)")


@pytest.mark.parametrize("grid", ["x=2,y=2", "x=3,y=2", "x=1,y=4"])
def test_batched_spmttkrp_plan_with_gpu_execute(gpu_lib, grid):
    """The two-loop batched SpMTTKRP plan (rows over x, rank columns over y)
    through the adapter: output, per-worker work, imbalance."""
    spec = KERNELS["spmttkrp"]
    rng = np.random.default_rng(9)
    t = K.instance("spmttkrp", rng, integers=True, rank=12)
    args = (spec["expr"], BATCHED_MTTKRP, grid, "dd", ref_inputs("spmttkrp", t))
    want = ob.RefRun(*args, mode="seq").ok()
    got = ob.RefRun(*args, mode="gpu", lib=gpu_lib).ok()
    assert np.array_equal(want.output()[1], got.output()[1])
    ws, gs = want.stats(), got.stats()
    assert ws["work"] == gs["work"] and ws["combines"] == gs["combines"] and ws["imbalance"] == gs["imbalance"]


@pytest.mark.parametrize("kernel", ["spttv", "spmttkrp"])
def test_sss_plan_with_gpu_execute(gpu_lib, kernel):
    spec = KERNELS[kernel]
    rng = np.random.default_rng(5)
    out_fmt = "ss" if kernel == "spttv" else "dd"
    for pieces in (1, 3):
        t = K.instance(kernel, rng, integers=True, rank=32 if kernel == "spmttkrp" else None)
        t["B"] = K.random_sparse(rng, t["B"].dims, "sss", 0.2, True)
        fm = dict(spec["formats"], B="sss", A=out_fmt)
        inputs = {nm: (x, fm[nm]) for nm, x in t.items()}
        want = ob.RefRun(spec["expr"], spec["nonzero"], pieces, out_fmt, inputs, mode="seq").ok()
        got = ob.RefRun(spec["expr"], spec["nonzero"], pieces, out_fmt, inputs, mode="gpu", lib=gpu_lib).ok()
        assert np.array_equal(want.output()[1], got.output()[1])
        assert want.stats()["work"] == got.stats()["work"]
