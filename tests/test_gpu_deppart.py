"""GPU dependent partitioning (spd_deppart_*, csrc/deppart.cu) against the
reference's own image / preimage / partition_by_bounds (oracle/_ref):
known answers, 200 seeded random trials (overlapping and empty ranges,
uncoloured indices), large pos-level cases, and the validation errors."""
import numpy as np
import pytest

import deppart_cases as D
import oracle_bind as ob

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2207_13901_b200 import host as H

    c = H.Context(0)
    yield c
    c.close()


def _gpu(ctx, op, ranges, subsets, dest):
    from paper_2207_13901_b200 import host as H

    part = H.DevicePartition.from_subsets(subsets)
    out = (H.image if op == "image" else H.preimage)(ctx, ranges, part, dest)
    return D.as_lists(out.subsets()), out.disjoint


@pytest.mark.parametrize("case", D.IMAGE_KATS)
def test_gpu_image_known_answers(ctx, case):
    ranges, dest, subsets, want, disj = case
    assert _gpu(ctx, "image", ranges, subsets, dest) == (want, disj)


@pytest.mark.parametrize("case", D.PREIMAGE_KATS)
def test_gpu_preimage_known_answers(ctx, case):
    ranges, dest, subsets, want, disj = case
    assert _gpu(ctx, "preimage", ranges, subsets, dest) == (want, disj)


@pytest.mark.parametrize("case", D.BOUNDS_KATS)
def test_gpu_by_bounds_known_answers(ctx, case):
    from paper_2207_13901_b200 import host as H

    ext, coloring, want = case
    out = H.partition_by_bounds(ctx, ext, coloring)
    assert D.as_lists(out.subsets()) == want
    ref, disj = ob.ref_partition_by_bounds(ext, coloring)
    assert out.disjoint == disj


def test_gpu_deppart_matches_reference_random(ctx):
    rng = np.random.default_rng(20260810)
    for _ in range(200):
        ranges, dest, src, dst = D.random_trial(rng)
        want, disj = ob.ref_image(ranges, src, dest)
        assert _gpu(ctx, "image", ranges, src, dest) == (D.as_lists(want), disj)
        want, disj = ob.ref_preimage(ranges, dst, dest)
        assert _gpu(ctx, "preimage", ranges, dst, dest) == (D.as_lists(want), disj)


def test_gpu_by_bounds_random_boxes(ctx):
    from paper_2207_13901_b200 import host as H

    rng = np.random.default_rng(3)
    for _ in range(40):
        R = int(rng.integers(1, 4))
        ext = [int(x) for x in rng.integers(1, 7, R)]
        coloring = {}
        for c in range(int(rng.integers(0, 5))):
            if rng.integers(0, 4) == 0:
                continue
            box = []
            for d in range(R):
                lo = int(rng.integers(0, ext[d]))
                hi = int(rng.integers(lo - 1, ext[d]))
                box.append((lo, hi))
            coloring[c] = box
        want, disj = ob.ref_partition_by_bounds(ext, coloring)
        out = H.partition_by_bounds(ctx, ext, coloring)
        assert D.as_lists(out.subsets()) == D.as_lists(want)
        assert out.disjoint == disj


def test_gpu_deppart_pos_level_at_scale(ctx):
    """A CSR pos level (1M rows, power-law lengths): image of a strided
    (non-contiguous) row colouring and preimage of a random position
    colouring, against the reference."""
    rng = np.random.default_rng(9)
    n = 1 << 20
    lens = np.minimum(rng.zipf(1.6, n) - 1, 400)
    lo = np.concatenate([[0], np.cumsum(lens)[:-1]])
    ranges = np.stack([lo, lo + lens - 1], 1)
    nnz = int(lens.sum())
    P = 5
    rows = [np.arange(c, n, P * 3) for c in range(P)]  # strided, some rows uncoloured
    want, disj = ob.ref_image(ranges, rows, nnz)
    got, gd = _gpu(ctx, "image", ranges, rows, nnz)
    assert gd == disj and all(np.array_equal(a, b) for a, b in zip(got, D.as_lists(want)))
    colour = rng.integers(0, P, nnz)
    pos = [np.nonzero(colour == c)[0][::7] for c in range(P)]
    want, disj = ob.ref_preimage(ranges, pos, nnz)
    got, gd = _gpu(ctx, "preimage", ranges, pos, nnz)
    assert gd == disj and all(np.array_equal(a, b) for a, b in zip(got, D.as_lists(want)))


def test_gpu_deppart_validation(ctx):
    from paper_2207_13901_b200 import host as H
    from paper_2207_13901_b200._native import SpdValidationError

    with pytest.raises(SpdValidationError):  # range outside the destination (region.cpp:38-40)
        H.image(ctx, [(0, 7)], H.DevicePartition.from_subsets([[0]]), 5)
    with pytest.raises(SpdValidationError):  # subset index outside the parent space
        H.image(ctx, [(0, 1)], H.DevicePartition.from_subsets([[3]]), 5)
    with pytest.raises(SpdValidationError):  # unsorted subset
        H.preimage(ctx, [(0, 1), (2, 3)], H.DevicePartition.from_subsets([[3, 1]]), 5)
    with pytest.raises(SpdValidationError):  # bound outside the space (deppart.cpp:72-73)
        H.partition_by_bounds(ctx, (4,), {0: [(0, 9)]})
