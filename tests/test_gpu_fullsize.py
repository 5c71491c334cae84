"""Parity at the production sizes, through the exact code paths bench.py
times (verdict round 1: full-size parity was builder-run only).

  C1         SpMV, uniform 1M x 1M, 10M samples, row split -- against the
             reference's own plan() + execute() (oracle/_ref, par mode)
  C2         SpMM N=32 on the R-MAT scale-24 CSR (16.8M rows, 165.6M nnz):
             the cp.async-ring leaf, 1 colour and 4 colours on one GPU
  SpMV-RMAT  the same matrix, nonzero split: the lane-per-row leaf over
             compacted columns with 2048-position chunks (>= 2^26 positions)
  C3         SDDMM K=128 on the same matrix, D stored j-major
  C4         SpTTV and SpMTTKRP R=32 on the 10M-nnz power-law dss tensor
  C5         SpAdd3 of the R-MAT and two column-shifted copies, row split P=8

C2-C5 are checked against the C restatement (oracle/restate.c, the
reference's summation semantics, OpenMP), the reference being infeasible at
these sizes.  Values within 1e-10 relative per entry (north
star), partition statistics and the SpAdd3 pattern bit-exact.
"""
import os
import sys

import numpy as np
import pytest

import oracle_bind as ob

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel_close(got, want):
    got = np.asarray(got).reshape(-1)
    want = np.asarray(want).reshape(-1)
    assert got.shape == want.shape
    bad = np.abs(got - want) > 1e-10 * np.maximum(np.abs(want), 1e-300)
    assert not bad.any(), f"{int(bad.sum())} entries differ, first at {int(np.argmax(bad))}"


@pytest.fixture(scope="module")
def ctx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2207_13901_b200 import host as H

    c = H.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch, torch.device("cuda", 0)


@pytest.fixture(scope="module")
def rmat():
    import bench

    n, rp, crd, vals = bench.rmat_csr(24, 10, 42)
    return n, rp, crd, vals


@pytest.fixture(scope="module")
def rmat_dev(ctx, torch_dev, rmat):
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    n, rp, crd, vals = rmat
    rp_d, crd_d, vals_d = (torch.from_numpy(x).to(dev) for x in (rp, crd, vals))
    B = H.DeviceTensor.wrap(ctx, (n, n), H.parse_format("ds"), [rp_d.data_ptr()], [crd_d.data_ptr()],
                            vals_d.data_ptr(), keep=(rp_d, crd_d, vals_d))
    yield B
    B.close()


def test_c1_spmv_full_size_against_the_reference(ctx, torch_dev):
    """C1 at full size through the reference's own pipeline: the GPU output
    equals plan() + execute() at 1e-10 and the Stats agree (P = 1 and 4)."""
    import bench
    import spd_kernels as SK
    from paper_2207_13901_b200 import _native as N
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    n, S = 1_000_000, 10_000_000
    rp, crd, vals = np.empty(n + 1, np.int64), np.empty(S, np.int64), np.empty(S)
    nnz = N.synth().syn_uniform_csr(n, n, S, 42, 0, rp.ctypes.data_as(N.i64p), crd.ctypes.data_as(N.i64p),
                                    vals.ctypes.data_as(N.dblp))
    crd, vals = crd[:nnz], vals[:nnz]
    x = bench.dense_vals(n, 43)
    Bh = H.SparseTensor.from_rowptrs((n, n), H.parse_format("ds"), [rp], [crd], vals)
    xh = H.SparseTensor.from_parts((n,), H.parse_format("d"), [H.Level("d", dom=(n,))], x)
    B = H.DeviceTensor.upload(ctx, Bh)
    x_d = torch.from_numpy(x).to(dev)
    y_d = torch.empty(n, dtype=torch.float64, device=dev)
    try:
        for P in (1, 4):
            H.partition_universe(ctx, B, P)
            st = H.spmv(ctx, B, x_d, y_d, pieces=P)
            run = ob.RefRun(SK.KERNELS["spmv"]["expr"], SK.ROW, P, "d", {"B": (Bh, "ds"), "c": (xh, "d")},
                            mode="par").ok()
            rel_close(y_d.cpu().numpy(), run.output()[1])
            ws = run.stats()
            assert st.work == ws["work"] and st.combines == ws["combines"] and st.imbalance == ws["imbalance"]
    finally:
        B.close()


@pytest.mark.parametrize("pieces", [1, 4])
def test_c2_spmm_full_size(ctx, torch_dev, rmat, rmat_dev, pieces):
    import bench
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    n, rp, crd, vals = rmat
    N = 32
    Cv = bench.dense_vals(n * N, 43)
    C_d = torch.from_numpy(Cv).to(dev)
    A_d = torch.empty(n * N, dtype=torch.float64, device=dev)
    H.partition_nonzero(ctx, rmat_dev, 1, pieces)
    st = H.spmm(ctx, rmat_dev, C_d, N, A_d, pieces=pieces)
    want, work, comb = ob.spmm(rp, crd, vals, Cv, N, ob.partition_nonzero([rp], len(crd), pieces))
    rel_close(A_d.cpu().numpy(), want)
    assert st.work == list(work) and st.combines == comb


def test_spmv_rmat_full_size(ctx, torch_dev, rmat, rmat_dev):
    """>= 2^26 positions: the production instantiation (6 CTAs/SM, compacted
    columns, 2048-position chunks)."""
    import bench
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    n, rp, crd, vals = rmat
    x = bench.dense_vals(n, 44)
    x_d = torch.from_numpy(x).to(dev)
    y_d = torch.empty(n, dtype=torch.float64, device=dev)
    for P in (1, 3):
        H.partition_nonzero(ctx, rmat_dev, 1, P)
        st = H.spmv(ctx, rmat_dev, x_d, y_d, pieces=P)
        want, work, comb = ob.spmv(rp, crd, vals, x, ob.partition_nonzero([rp], len(crd), P))
        rel_close(y_d.cpu().numpy(), want)
        assert st.work == list(work) and st.combines == comb


def test_c3_sddmm_full_size(ctx, torch_dev, rmat, rmat_dev):
    import bench
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    n, rp, crd, vals = rmat
    K = 128
    Cv = bench.dense_vals(n * K, 44)
    Dv = bench.dense_vals(n * K, 45)  # D(k, j) stored j-major
    C_d = torch.from_numpy(Cv).to(dev)
    D_d = torch.from_numpy(Dv).to(dev)
    A_d = torch.empty(len(crd), dtype=torch.float64, device=dev)
    H.partition_nonzero(ctx, rmat_dev, 1, 1)
    st = H.sddmm(ctx, rmat_dev, C_d, D_d, K, 1, K, A_d, pieces=1)
    del C_d, D_d
    want, work, comb = ob.sddmm(rp, crd, vals, Cv, Dv, K, 1, K, ob.partition_nonzero([rp], len(crd), 1))
    rel_close(A_d.cpu().numpy(), want)
    assert st.work == list(work) and st.combines == comb


def test_c4_spttv_spmttkrp_full_size(ctx, torch_dev):
    import bench
    from paper_2207_13901_b200 import _native as N
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    I, J, Kd, S, R = 12092, 9184, 28818, 10_000_000, 32
    rp1, crd1 = np.empty(I + 1, np.int64), np.empty(S, np.int64)
    rp2, crd2 = np.empty(S + 1, np.int64), np.empty(S, np.int64)
    vals, F = np.empty(S), np.zeros(1, np.int64)
    nnz = N.synth().syn_powerlaw_csf(I, J, Kd, S, 4, 0, rp1.ctypes.data_as(N.i64p), crd1.ctypes.data_as(N.i64p),
                                     rp2.ctypes.data_as(N.i64p), crd2.ctypes.data_as(N.i64p),
                                     vals.ctypes.data_as(N.dblp), F.ctypes.data_as(N.i64p))
    F = int(F[0])
    crd1, rp2, crd2, vals = crd1[:F], rp2[:F + 1], crd2[:nnz], vals[:nnz]
    Bt = H.DeviceTensor.upload_rowptr(ctx, (I, J, Kd), H.parse_format("dss"), [rp1, rp2], [crd1, crd2], vals)
    try:
        c = bench.dense_vals(Kd, 46)
        Cm, Dm = bench.dense_vals(J * R, 47), bench.dense_vals(Kd * R, 48)
        c_d, C_d, D_d = (torch.from_numpy(a).to(dev) for a in (c, Cm, Dm))
        Av = torch.empty(F, dtype=torch.float64, device=dev)
        A_d = torch.empty(I * R, dtype=torch.float64, device=dev)
        for P in (1, 4):
            cols = ob.partition_nonzero([rp1, rp2], nnz, P)
            H.partition_nonzero(ctx, Bt, 2, P)
            st = H.spttv(ctx, Bt, c_d, Av, pieces=P)
            want, work, comb = ob.spttv(rp1, crd1, rp2, crd2, vals, c, cols)
            rel_close(Av.cpu().numpy(), want)
            assert st.work == list(work) and st.combines == comb
            H.partition_nonzero(ctx, Bt, 2, P)
            st = H.spmttkrp(ctx, Bt, C_d, D_d, R, A_d, pieces=P)
            want, work, comb = ob.spmttkrp(rp1, crd1, rp2, crd2, vals, Cm, Dm, R, cols)
            rel_close(A_d.cpu().numpy(), want)
            assert st.work == list(work) and st.combines == comb
    finally:
        Bt.close()


def test_c5_spadd3_full_size(ctx, torch_dev, rmat, rmat_dev):
    """The structural union of 3 x 165M entries: pattern bit-exact."""
    import bench
    from paper_2207_13901_b200 import _native as N
    from paper_2207_13901_b200 import host as H

    torch, dev = torch_dev
    n, rp, crd, vals = rmat
    ops = [(rp, crd, vals)]
    for shift in (1, 2):
        rps, e = np.empty(n + 1, np.int64), 10 * n
        cs, vs = np.empty(e, np.int64), np.empty(e)
        nz = N.synth().syn_rmat_csr(24, e, bench.A_RMAT, bench.B_RMAT, bench.C_RMAT, 42, 0, 0, shift,
                                    rps.ctypes.data_as(N.i64p), cs.ctypes.data_as(N.i64p), vs.ctypes.data_as(N.dblp))
        ops.append((rps, cs[:nz], vs[:nz]))
    devs = [rmat_dev] + [H.DeviceTensor.upload_rowptr(ctx, (n, n), H.parse_format("ds"), [o[0]], [o[1]], o[2])
                         for o in ops[1:]]
    try:
        H.partition_universe(ctx, devs[0], 8)
        A, st = H.spadd3(ctx, devs[0], devs[1], devs[2], pieces=8)
        At = A.download()
        A.close()
        w_rp, w_crd, w_vals = ob.spadd3(ops)
        assert np.array_equal(At.levels[1].rowptr(), w_rp)
        assert np.array_equal(At.levels[1].crd, w_crd)
        rel_close(At.vals, w_vals)
    finally:
        for d in devs[1:]:
            d.close()
