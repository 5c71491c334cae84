"""Shared cases for the dependent-partitioning tests (deppart.cpp:15-101):
the reference's own known answers (test_tensor_core.cpp:83-199) and seeded
random trials in the style of its brute-force test (:118-149)."""
import numpy as np

# (ranges, dest_extent, subsets, expected image, expected disjoint)
IMAGE_KATS = [
    ([(0, 1), (2, 2), (3, 4)], 5, [[0], [1, 2]], [[0, 1], [2, 3, 4]], True),   # :83-90
    ([(0, 1), (2, 2), (3, 4)], 5, [[0, 1, 2]], [[0, 1, 2, 3, 4]], True),       # :92-95
]
# (ranges, dest_extent, dest subsets, expected preimage, expected disjoint)
PREIMAGE_KATS = [
    ([(0, 2), (3, 3)], 4, [[0, 1], [2, 3]], [[0], [0, 1]], False),             # :98-104
    ([(0, 1), (2, 1), (2, 3)], 4, [[0, 1, 2, 3]], [[0, 2]], True),             # :106-110
]
# (extents, coloring, expected subsets)
BOUNDS_KATS = [
    ((6,), {0: [(0, 2)], 1: [(3, 5)]}, [[0, 1, 2], [3, 4, 5]]),               # :179-183
    ((5,), {0: [(0, 2)], 1: [(3, 4)]}, [[0, 1, 2], [3, 4]]),                  # :185-188
    ((4,), {}, []),                                                          # :190-191
    ((2, 3), {0: [(0, 1), (1, 2)]}, [[1, 2, 4, 5]]),                          # :196-198
]


def random_trial(rng):
    """One trial of test_tensor_core.cpp:118-149's generator shape: ranges
    with hi in [lo-1, dest-1] (so some are empty), some indices uncoloured."""
    src_n = int(rng.integers(1, 33))
    dest_n = int(rng.integers(1, 41))
    ranges = []
    for _ in range(src_n):
        lo = int(rng.integers(0, dest_n))
        hi = int(rng.integers(lo - 1, dest_n))
        ranges.append((lo, hi))
    colors = int(rng.integers(1, 7))
    src = [[] for _ in range(colors)]
    dst = [[] for _ in range(colors)]
    for i in range(src_n):
        if rng.integers(0, 4) == 0:
            continue
        src[int(rng.integers(0, colors))].append(i)
    for i in range(dest_n):
        if rng.integers(0, 4) == 0:
            continue
        dst[int(rng.integers(0, colors))].append(i)
    return ranges, dest_n, src, dst


def image_fold(ranges, subsets):
    """The formal definition, folded directly (test_tensor_core.cpp:26-35)."""
    out = []
    for sub in subsets:
        s = set()
        for i in sub:
            lo, hi = ranges[i]
            s.update(range(lo, hi + 1))
        out.append(sorted(s))
    return out


def preimage_fold(ranges, subsets):
    out = []
    for sub in subsets:
        ss = set(sub)
        out.append([i for i, (lo, hi) in enumerate(ranges) if lo <= hi and any(d in ss for d in range(lo, hi + 1))])
    return out


def disjoint(subsets):
    seen = set()
    for sub in subsets:
        for v in sub:
            if v in seen:
                return False
            seen.add(v)
    return True


def as_lists(parts):
    return [list(map(int, p)) for p in parts]
