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


def _stats_json(run):
    import json

    return json.loads(run.L.ref_stats_json(run.h).decode())


# Explicit placements (tensor distribution notation): row blocks,
# nonzero blocks and replication, so the ledger charges real bytes.
EXPLICIT_TDN = {
    "spmv": {"B": "B(x, y) onto M(x)", "c": "c(x) onto M(x)", "a": "a(x) onto M(x)"},
    "spmm": {"B": "B(x, y) fuse(x, y -> f) onto M(~f)", "C": "C(x, y) onto M(x)", "A": "A(x, y) onto M(x)"},
    "sddmm": {"B": "B(x, y) onto M(x)", "C": "C(x, y) onto M(z)", "D": "D(x, y) onto M(x)", "A": "A(x, y) onto M(x)"},
    "spttv": {"B": "B(x, y, z) onto M(x)", "c": "c(x) onto M(x)", "A": "A(x, y) onto M(x)"},
    "spmttkrp": {"B": "B(x, y, z) onto M(x)", "C": "C(x, y) onto M(x)", "D": "D(x, y) onto M(z)",
                 "A": "A(x, y) onto M(x)"},
    "spadd3": {"B": "B(x, y) onto M(x)", "C": "C(x, y) fuse(x, y -> f) onto M(~f)", "D": "D(x, y) onto M(z)",
               "A": "A(x, y) onto M(x)"},
}


@pytest.mark.parametrize("kernel", list(KERNELS))
@pytest.mark.parametrize("schedule", ["row", "nonzero"])
@pytest.mark.parametrize("tdns", ["default", "explicit"])
def test_residency_ledger_matches_reference(gpu_lib, kernel, schedule, tdns):
    """execute_gpu(plan, tensors, machine, residency): with the TDN placements
    lowered into a Residency (cli.cpp:152-160), the whole Stats JSON --
    per-worker bytes_by_tensor (the ledger, sim.cpp:868-887), work, imbalance,
    combines -- equals the reference's execute in par mode."""
    if schedule == "nonzero" and KERNELS[kernel]["nonzero"] is None:
        pytest.skip("position split rejected for union statements")
    spec = KERNELS[kernel]
    sched = ROW if schedule == "row" else spec["nonzero"]
    rng = np.random.default_rng(1234)
    out = OUTPUT[kernel]
    for pieces in (1, 3, 4):
        t = K.instance(kernel, rng, integers=True)
        inputs = ref_inputs(kernel, t)
        out_tdn = None
        if tdns == "explicit":
            inputs = {nm: (x[0], x[1], EXPLICIT_TDN[kernel][nm]) for nm, x in inputs.items()}
            out_tdn = EXPLICIT_TDN[kernel][out]
        args = (spec["expr"], sched, pieces, spec["formats"][out], inputs)
        want = ob.RefRun(*args, mode="par", use_placements=True, out_tdn=out_tdn).ok()
        got = ob.RefRun(*args, mode="gpu", use_placements=True, out_tdn=out_tdn, lib=gpu_lib).ok()
        ws, gs = _stats_json(want), _stats_json(got)
        assert gs == ws, (kernel, schedule, tdns, pieces)
        if pieces > 1 and tdns == "explicit":
            assert any(b for w in ws["per_worker"] for b in w["bytes_by_tensor"].values())


@pytest.mark.parametrize("kernel", ["spmv", "spmm", "spttv"])
def test_worker_mapping_on_a_2d_machine(gpu_lib, kernel):
    """A one-loop schedule on a 2-D grid (x=2,y=2, distribute over M.x): the
    colours map to workers through tuple_worker (sim.cpp:535-544) and the
    imbalance is over all four workers (sim.cpp:1000-1005)."""
    spec = KERNELS[kernel]
    rng = np.random.default_rng(3)
    t = K.instance(kernel, rng, integers=True)
    args = (spec["expr"], ROW, "x=2,y=2", spec["formats"][OUTPUT[kernel]], ref_inputs(kernel, t))
    want = ob.RefRun(*args, mode="par", use_placements=True).ok()
    got = ob.RefRun(*args, mode="gpu", use_placements=True, lib=gpu_lib).ok()
    assert _stats_json(got) == _stats_json(want)
    assert np.array_equal(want.output()[1], got.output()[1])


@pytest.mark.parametrize("case", ["csc_B", "colmajor_C", "colmajor_out"])
def test_transposed_storage_is_rejected(gpu_lib, case):
    """A CSC B ('ds:1,0') or a column-major dense operand / output is valid
    for the reference but would be read in the wrong order by the leaf
    kernels: the adapter rejects it as unsupported (no wrong results)."""
    from paper_2207_13901_b200.host import SparseTensor, parse_format

    rng = np.random.default_rng(11)
    n, k, N = 6, 5, 3
    fmtB = "ds:1,0" if case == "csc_B" else "ds"
    fmtC = "dd:1,0" if case == "colmajor_C" else "dd"
    fmtA = "dd:1,0" if case == "colmajor_out" else "dd"
    B = K.random_sparse(rng, (n, k), fmtB, 0.4)
    C = K.dense(rng, (k, N), fmtC)
    sched = "divide(i, io, ii, M.x); distribute(io, M.x)"
    if case == "csc_B":
        sched = "reorder(k, i, j); fuse(k, i, f); divide(f, fo, fi, B.pos, M.x); distribute(fo, M.x)"
    run = ob.RefRun("A(i, j) = B(i, k) * C(k, j)", sched, 2, fmtA, {"B": (B, fmtB), "C": (C, fmtC)},
                    mode="gpu", lib=gpu_lib)
    if run.status == 2 and "unsupported on gpu" not in run.error:
        pytest.skip(f"the reference itself rejects this schedule: {run.error}")
    assert run.status == 2 and "unsupported on gpu" in run.error, run.error


@pytest.mark.parametrize("kernel", list(KERNELS))
def test_every_visible_gpu_gives_the_one_gpu_result(gpu_lib, kernel):
    """execute_gpu spreads the colours over every visible GPU (one host thread
    per GPU, NCCL boundary combine, SpAdd3 row blocks gathered); capped to one
    GPU with DSPAR_GPUS=1 it runs them all on device 0.  Both give the same
    output and Stats as the reference (on a one-GPU box both runs take the
    one-GPU path)."""
    import torch

    spec = KERNELS[kernel]
    sched = spec["nonzero"] or ROW
    rng = np.random.default_rng(31)
    for pieces in (3, 5):
        # SpMM and SpMTTKRP at width / rank 32 too: their leaves opt in to
        # dynamic shared memory, a per-device attribute every GPU must get
        rank = 32 if pieces == 5 and kernel in ("spmm", "spmttkrp") else None
        t = K.instance(kernel, rng, integers=True, rank=rank)
        args = (spec["expr"], sched, pieces, spec["formats"][OUTPUT[kernel]], ref_inputs(kernel, t))
        want = ob.RefRun(*args, mode="par", use_placements=True).ok()
        outs = []
        for cap in (None, "1"):
            if cap:
                os.environ["DSPAR_GPUS"] = cap
            try:
                got = ob.RefRun(*args, mode="gpu", use_placements=True, lib=gpu_lib).ok()
            finally:
                os.environ.pop("DSPAR_GPUS", None)
            outs.append(got.output())
            assert _stats_json(got) == _stats_json(want), (kernel, pieces, cap, torch.cuda.device_count())
        (l0, v0), (l1, v1) = outs
        assert np.array_equal(v0, v1) and np.array_equal(v0, want.output()[1])


GRID = ("divide(i, io, ii, M.x); divide(j, jo, ji, M.y); reorder(io, jo, ii, ji, k); "
        "distribute(io, M.x); distribute(jo, M.y)")


@pytest.mark.parametrize("kernel", ["sddmm", "spttv"])
@pytest.mark.parametrize("grid", ["x=2,y=2", "x=3,y=2", "x=1,y=4", "x=4,y=3"])
def test_two_dimensional_grid_with_bucketed_columns(gpu_lib, kernel, grid):
    """Rows over M.x, the compressed level's coordinate j over M.y (the inner
    universe split, level_partition.cpp:193-205): output, per-worker work,
    imbalance and the ledger equal the reference's execute."""
    spec = KERNELS[kernel]
    rng = np.random.default_rng(17)
    for _ in range(2):
        t = K.instance(kernel, rng, integers=True, max_dim=30)
        args = (spec["expr"], GRID, grid, spec["formats"]["A"], ref_inputs(kernel, t))
        want = ob.RefRun(*args, mode="par", use_placements=True).ok()
        got = ob.RefRun(*args, mode="gpu", use_placements=True, lib=gpu_lib).ok()
        assert np.array_equal(want.output()[1], got.output()[1])
        assert _stats_json(got) == _stats_json(want)


@pytest.mark.parametrize("kernel", ["sddmm", "spttv"])
@pytest.mark.parametrize("pieces", [1, 2, 3, 5, 40])
def test_bucket_split_equals_the_reference_bundle(gpu_lib, kernel, pieces):
    """spd_partition_bucket's colour sets are the reference's crd partition of
    B's level 1 for the bucketed loop (bucketCoords), empty colours included."""
    import ctypes as C

    import torch

    from paper_2207_13901_b200 import _native as N
    from paper_2207_13901_b200 import host as H

    spec = KERNELS[kernel]
    rng = np.random.default_rng(pieces)
    t = K.instance(kernel, rng, integers=True, max_dim=30)
    run = ob.RefRun(spec["expr"], GRID, f"x=1,y={pieces}", spec["formats"]["A"], ref_inputs(kernel, t),
                    execute=False).ok()
    ctx = H.Context(0)
    try:
        dev = H.DeviceTensor.upload(ctx, t["B"])
        counts = np.zeros(pieces, np.int64)
        N.check(N.lib().spd_partition_bucket(ctx.h, dev.h, 1, pieces, counts.ctypes.data_as(N.i64p)))
        for c in range(pieces):
            want = run.subset("B", 1, "crd", c, k=1)
            buf = np.zeros(max(int(counts[c]), 1), np.int64)
            n = C.c_int64()
            N.check(N.lib().spd_bucket_positions(ctx.h, c, buf.ctypes.data_as(N.i64p), len(buf), C.byref(n)))
            assert n.value == counts[c] == len(want)
            assert np.array_equal(buf[:n.value], want)
        dev.close()
    finally:
        ctx.close()


def test_reference_suite_with_gpu_dependent_partitioning(gpu_lib):
    """The reference's own doctest suite (64 cases, 1886 checks) linked with
    integration/deppart_gpu.cpp in place of deppart.cpp: image, preimage,
    partition_by_bounds and copy_partition on the GPU under the reference's
    planner, LevelPartitioner and tests -- the same single known failure as
    the CPU build (test_planner.cpp:233, a validation gap of planner.cpp:84)."""
    import subprocess

    exe = os.path.join(os.path.dirname(ob.REF_TESTS), "dspar_ref_tests_gpudeppart")
    if not os.path.exists(exe):
        pytest.skip("GPU-deppart reference suite not built (make -C oracle integration)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    # the three render-golden cases read /root/reference/proj/tests/golden,
    # which only exists where the reference is mounted (not on a GPU box):
    # there they report "golden file created"; the rendered plans are
    # compared library against library in test_rendered_plans_equal_with_gpu_deppart
    missing = out.count("golden file created")
    assert f"test cases: 64 | failed: {1 + missing}" in out, out[-3000:]
    assert "test_planner.cpp:233" in r.stderr and r.stderr.count("CHECK FAILED") == 1 + missing


@pytest.mark.parametrize("schedule,pieces", [("row", 2), ("row", 1), ("nonzero", 2), ("nonzero", 4)])
def test_rendered_plans_equal_with_gpu_deppart(gpu_lib, schedule, pieces):
    """render_plan of the reference's planner with the GPU dependent
    partitioning equals the CPU build's, colour bounds and every bundle subset
    included (the golden-file cases of test_planner.cpp:302-315, library
    against library)."""
    spec = KERNELS["spmv"]
    sched = ROW if schedule == "row" else spec["nonzero"]
    rng = np.random.default_rng(pieces)
    t = K.instance("spmv", rng, integers=True, max_dim=30)
    args = (spec["expr"], sched, pieces, "d", ref_inputs("spmv", t))
    cpu = ob.RefRun(*args, execute=False).ok()
    gpu = ob.RefRun(*args, execute=False, lib=gpu_lib).ok()
    assert cpu.L.ref_rendered_plan(cpu.h) == gpu.L.ref_rendered_plan(gpu.h)
    for c in range(pieces):
        for lvl, region in ((0, "dom"), (1, "pos"), (1, "crd")):
            a, b = cpu.subset("B", lvl, region, c), gpu.subset("B", lvl, region, c)
            assert (a is None and b is None) or np.array_equal(a, b)
