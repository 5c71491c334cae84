"""The deppart oracle -- the reference's own image / preimage /
partition_by_bounds (deppart.cpp:15-101, built into oracle/_ref) -- pinned
against the reference's known answers (test_tensor_core.cpp:83-199) and the
formal definitions folded directly, before it judges the GPU path
(tests/test_gpu_deppart.py).  CPU only."""
import numpy as np
import pytest

import deppart_cases as D
import oracle_bind as ob


@pytest.mark.parametrize("case", D.IMAGE_KATS)
def test_reference_image_known_answers(case):
    ranges, dest, subsets, want, disj = case
    got, d = ob.ref_image(ranges, subsets, dest)
    assert D.as_lists(got) == want and d == disj


@pytest.mark.parametrize("case", D.PREIMAGE_KATS)
def test_reference_preimage_known_answers(case):
    ranges, dest, subsets, want, disj = case
    got, d = ob.ref_preimage(ranges, subsets, dest)
    assert D.as_lists(got) == want and d == disj


@pytest.mark.parametrize("case", D.BOUNDS_KATS)
def test_reference_by_bounds_known_answers(case):
    ext, coloring, want = case
    got, _ = ob.ref_partition_by_bounds(ext, coloring)
    assert D.as_lists(got) == want


def test_reference_deppart_matches_folds():
    rng = np.random.default_rng(20260810)
    for _ in range(200):
        ranges, dest, src, dst = D.random_trial(rng)
        got, d = ob.ref_image(ranges, src, dest)
        want = D.image_fold(ranges, src)
        assert D.as_lists(got) == want and d == D.disjoint(want)
        got, d = ob.ref_preimage(ranges, dst, dest)
        want = D.preimage_fold(ranges, dst)
        assert D.as_lists(got) == want and d == D.disjoint(want)


def test_reference_deppart_errors():
    with pytest.raises(ob.RefPartitionError) as e:
        ob.ref_image([(0, 7)], [[0]], 5)  # range outside the destination
    assert e.value.status == 2
    with pytest.raises(ob.RefPartitionError):
        ob.ref_partition_by_bounds((4,), {0: [(0, 9)]})
