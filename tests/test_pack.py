"""Tensor construction: SparseTensor::pack (tensor.cpp:94-182).

* CPU: the reference's own pack (oracle/_ref, `RefRun.pack`) reproduces the
  known answers of test_tensor_core.cpp:211-244, and the host restatement
  (host.SparseTensor.pack, used to build every test input) matches the
  reference bit-for-bit on random COO with duplicates, explicit zeros and
  -0.0 over many formats.
* GPU: the device-side pack (spd_tensor_pack) matches the
  reference bit-for-bit: pos pairs, crd, vals (including the sign of zero),
  host- and device-resident inputs, the LSD multi-pass path (storage key
  wider than 64 bits), empty input and the out-of-bounds error.
"""
import numpy as np
import pytest

import oracle_bind as ob
from paper_2207_13901_b200.host import SparseTensor, parse_format

FORMATS = {
    1: ["s", "d"],
    2: ["ds", "ds:1,0", "ss", "sd", "dd", "ss:1,0"],
    3: ["dss", "sss", "dds", "sds", "ssd", "dss:2,0,1", "sss:1,2,0", "dsd"],
}


def _entries(rng, dims, n, dup_frac=0.3):
    base = np.stack([rng.integers(0, d, n) for d in dims], axis=1)
    ndup = int(n * dup_frac)
    if n and ndup:
        base = np.concatenate([base, base[rng.integers(0, n, ndup)]])
        rng.shuffle(base)
    vals = rng.integers(-3, 4, base.shape[0]).astype(float)
    vals[rng.random(vals.shape[0]) < 0.1] = -0.0
    return base, vals


def _ref_levels(r):
    levels, vals = r.output()
    return [(k, None if p is None else p.reshape(-1, 2), c) for k, p, c in levels], vals


def _same(levels_a, vals_a, levels_b, vals_b):
    assert len(levels_a) == len(levels_b)
    for (ka, pa, ca), (kb, pb, cb) in zip(levels_a, levels_b):
        assert ka == kb
        if ka == "s":
            assert np.array_equal(np.asarray(pa).reshape(-1, 2), np.asarray(pb).reshape(-1, 2))
            assert np.array_equal(ca, cb)
    va, vb = np.asarray(vals_a), np.asarray(vals_b)
    assert np.array_equal(va, vb)
    assert np.array_equal(np.signbit(va), np.signbit(vb))


def _host_levels(t):
    return [(lv.kind, lv.pos, lv.crd) for lv in t.levels], t.vals


def test_reference_pack_known_answers():
    r = ob.RefRun.pack((3, 3), "ds", [[0, 0], [0, 1], [1, 1], [2, 2]], [2.0, 3.0, 4.0, 5.0]).ok()
    levels, vals = _ref_levels(r)
    assert levels[1][1].tolist() == [[0, 1], [2, 2], [3, 3]] and levels[1][2].tolist() == [0, 1, 1, 2]
    assert vals.tolist() == [2, 3, 4, 5]
    r = ob.RefRun.pack((3, 3), "ds:1,0", [[0, 0], [0, 1], [1, 1], [2, 2]], [2.0, 3.0, 4.0, 5.0]).ok()
    levels, vals = _ref_levels(r)
    assert levels[1][1].tolist() == [[0, 0], [1, 2], [3, 3]] and levels[1][2].tolist() == [0, 0, 1, 2]
    r = ob.RefRun.pack((2,), "s", [[1], [1], [0]], [1.5, 2.5, 1.0]).ok()
    assert _ref_levels(r)[1].tolist() == [1.0, 4.0]
    r = ob.RefRun.pack((3, 3), "ds", np.zeros((0, 2)), []).ok()
    levels, vals = _ref_levels(r)
    assert len(vals) == 0 and all(p[1] < p[0] for p in levels[1][1])
    r = ob.RefRun.pack((3, 3), "ds", [[0, 3]], [1.0])
    assert r.status == 2 and "out of bounds" in r.error


@pytest.mark.parametrize("order", [1, 2, 3])
def test_host_pack_matches_reference(order):
    rng = np.random.default_rng(order)
    for fmt in FORMATS[order]:
        for trial in range(3):
            dims = tuple(int(x) for x in rng.integers(1, 9, order))
            coords, vals = _entries(rng, dims, int(rng.integers(0, 40)))
            want = _ref_levels(ob.RefRun.pack(dims, fmt, coords, vals).ok())
            got = _host_levels(SparseTensor.pack(dims, parse_format(fmt), coords, vals))
            _same(*got, *want)


def _device_case(ctx, dims, fmt, coords, vals, on_device=False):
    from paper_2207_13901_b200.host import DeviceTensor

    if on_device:
        import torch

        cols = [torch.from_numpy(np.ascontiguousarray(coords[:, k])).cuda() for k in range(len(dims))]
        t = DeviceTensor.pack(ctx, dims, parse_format(fmt), cols, torch.from_numpy(vals).cuda())
    else:
        t = DeviceTensor.pack(ctx, dims, parse_format(fmt), coords, vals)
    host = t.download()
    t.close()
    return _host_levels(host)


@pytest.fixture(scope="module")
def ctx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2207_13901_b200.host import Context

    c = Context(0)
    yield c
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 2, 3])
def test_device_pack_matches_reference(ctx, order):
    rng = np.random.default_rng(100 + order)
    for fmt in FORMATS[order]:
        for trial in range(4):
            dims = tuple(int(x) for x in rng.integers(1, 40, order))
            coords, vals = _entries(rng, dims, int(rng.integers(0, 3000)))
            want = _ref_levels(ob.RefRun.pack(dims, fmt, coords, vals).ok())
            got = _device_case(ctx, dims, fmt, coords, vals, on_device=bool(trial % 2))
            _same(*got, *want)


@pytest.mark.gpu
def test_device_pack_wide_keys_and_errors(ctx):
    from paper_2207_13901_b200._native import SpdValidationError
    from paper_2207_13901_b200.host import DeviceTensor

    rng = np.random.default_rng(7)
    # storage key of 3 x 31 bits: the multi-pass (LSD) sort
    dims = (2**31 - 1, 2**31 - 5, 2**30 + 3)
    coords, vals = _entries(rng, dims, 5000)
    coords[:50] = coords[0]  # a heavy duplicate
    want = _ref_levels(ob.RefRun.pack(dims, "sss", coords, vals).ok())
    _same(*_device_case(ctx, dims, "sss", coords, vals), *want)
    # empty input
    want = _ref_levels(ob.RefRun.pack((5, 4), "ds", np.zeros((0, 2), np.int64), []).ok())
    _same(*_device_case(ctx, (5, 4), "ds", np.zeros((0, 2), np.int64), np.zeros(0)), *want)
    # out of bounds
    with pytest.raises(SpdValidationError):
        DeviceTensor.pack(ctx, (3, 3), parse_format("ds"), np.array([[0, 3]]), np.array([1.0]))
    with pytest.raises(SpdValidationError):
        DeviceTensor.pack(ctx, (3, 3), parse_format("ds"), np.array([[-1, 0]]), np.array([1.0]))


@pytest.mark.gpu
def test_device_pack_rmat_matches_generator(ctx):
    """A scale-16 R-MAT edge list with its duplicates: the packed CSR equals
    the host restatement (the generator's own CSR build sums duplicates the
    same way)."""
    import bench
    from paper_2207_13901_b200 import _native as N
    from paper_2207_13901_b200.host import DeviceTensor

    n, rp, crd, vals = bench.rmat_csr(16, 10, 5)
    rows = np.repeat(np.arange(n), np.diff(rp))
    coords = np.stack([rows, crd], axis=1)
    perm = np.random.default_rng(3).permutation(coords.shape[0])
    t = DeviceTensor.pack(ctx, (n, n), parse_format("ds"), coords[perm], vals[perm])
    h = t.download()
    t.close()
    assert np.array_equal(h.levels[1].rowptr(), rp)
    assert np.array_equal(h.levels[1].crd, crd)
    assert np.array_equal(h.vals, vals)
    del N


# ------------------------------------------------------------------ loaders ---
def _write_tns(path, coords, vals, comments=True):
    with open(path, "w") as f:
        if comments:
            f.write("# a comment\n\n% another\n")
        for c, v in zip(coords, vals):
            f.write(" ".join(str(int(x) + 1) for x in c) + " %r\n" % float(v))
            if comments and np.random.random() < 0.01:
                f.write("   \n")


def _write_mtx(path, dims, coords, vals):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n% comment\n\n")
        f.write(f"{dims[0]} {dims[1]} {len(vals)}\n")
        for c, v in zip(coords, vals):
            f.write(f"{c[0] + 1} {c[1] + 1} {float(v)!r}\n")


def test_reference_load_known_answer(tmp_path):
    p = tmp_path / "csr.tns"
    p.write_text("1 1 2\n1 2 3\n2 2 4\n3 3 5\n")
    r = ob.RefRun.load(p, "ds", 2, (3, 3)).ok()
    levels, vals = _ref_levels(r)
    assert levels[1][1].tolist() == [[0, 1], [2, 2], [3, 3]] and vals.tolist() == [2, 3, 4, 5]


@pytest.mark.gpu
def test_device_load_matches_reference(ctx, tmp_path):
    from paper_2207_13901_b200.host import DeviceTensor

    rng = np.random.default_rng(9)
    cases = []
    for order, fmt in ((2, "ds"), (2, "ds:1,0"), (3, "dss"), (3, "sss")):
        dims = tuple(int(x) for x in rng.integers(5, 300, order))
        coords, vals = _entries(rng, dims, 20000)
        p = tmp_path / f"t{order}{fmt.replace(':', '_').replace(',', '')}.tns"
        _write_tns(p, coords, vals)
        cases += [(p, fmt, order, None), (p, fmt, order, tuple(d + 3 for d in dims))]
    dims = (400, 300)
    coords, vals = _entries(rng, dims, 30000, dup_frac=0.0)
    mp = tmp_path / "m.mtx"
    _write_mtx(mp, dims, coords, vals)
    cases += [(mp, "ds", 2, None), (mp, "ds", 2, dims)]
    for path, fmt, order, d in cases:
        r = ob.RefRun.load(path, fmt, order, d).ok()
        want = _ref_levels(r)
        t = DeviceTensor.load(ctx, path, parse_format(fmt), d)
        assert t.dims == r.out_dims(order)
        _same(*_host_levels(t.download()), *want)
        # write_tensor: byte-identical files
        a, b = tmp_path / "ours.tns", tmp_path / "ref.tns"
        t.store(a)
        assert r.store(b) == 0
        assert a.read_bytes() == b.read_bytes()
        t.close()


@pytest.mark.gpu
def test_device_load_errors_match_reference(ctx, tmp_path):
    from paper_2207_13901_b200._native import SpdValidationError
    from paper_2207_13901_b200.host import DeviceTensor

    bad = {
        "malformed.tns": ("1 1 2\n1 x 3\n", "ds", (3, 3)),
        "short.tns": ("1 1 2\n\n2 2\n", "ds", (3, 3)),
        "trailing.tns": ("1 1 2\n2 2 4 9\n", "ds", (3, 3)),
        "bounds.tns": ("1 1 2\n4 1 1\n", "ds", (3, 3)),
        "zero.tns": ("0 1 2\n", "ds", None),
        "count.mtx": ("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n", "ds", None),
        "header.mtx": ("%%MatrixMarket matrix coordinate integer general\n3 3 1\n1 1 1\n", "ds", None),
        "dims.mtx": ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 1\n", "ds", (4, 3)),
    }
    for name, (text, fmt, d) in bad.items():
        p = tmp_path / name
        p.write_text(text)
        r = ob.RefRun.load(p, fmt, 2, d)
        assert r.status == 2, name
        with pytest.raises(SpdValidationError) as ei:
            DeviceTensor.load(ctx, p, parse_format(fmt), d)
        assert str(ei.value) == r.error, (name, str(ei.value), r.error)
    with pytest.raises(SpdValidationError, match="cannot open tensor file"):
        DeviceTensor.load(ctx, tmp_path / "missing.tns", parse_format("ds"))
