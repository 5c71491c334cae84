#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY -- builds the checker, never the product.

Writes a patched copy of the reference's leaf executor into oracle/_ref/patched/sim.cpp.

The reference's `execute()` (/root/reference/proj/core/src/sim.cpp:816) has two
documented defects that make it unusable as an oracle:

  1. use-after-move at sim.cpp:451 -- `lists.push_back(std::move(*c))` empties
     the candidate lists that `visit()` then binary-searches (sim.cpp:437-439),
     so every coordinate-value (row) leaf does zero work;
  2. `locate_coord` (sim.cpp:307-320) binary-searches the whole pos range of a
     row through a WorkerView that only holds the colour's crd positions, so a
     nonzero split that straddles a row throws ClosureViolation.

This script applies the minimal fix of SURVEY.md section 9.3 (one line + an
owned-span search) to a copy under oracle/_ref/ (git-ignored).  Nothing is ever
written to /root/reference and no reference source is committed: only the
few-line edit below lives in the repository.
"""
import os
import sys

REF = os.environ.get("DSPAR_REF", "/root/reference/proj")
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "patched")

EDITS = [
    # (1) WorkerView gains an owned-span search over its snapshot (fix for sim.cpp:307-320).
    (
        "  void set_color(int64_t c) { color_ = c; }\n",
        "  void set_color(int64_t c) { color_ = c; }\n"
        "\n"
        "  // [graft oracle patch] owned crd positions of `level` inside [lo, hi]\n"
        "  std::pair<int64_t, int64_t> owned_span(int level, int64_t lo, int64_t hi) const {\n"
        "    const auto& idx = levels_[level].crd_idx;\n"
        "    auto b = std::lower_bound(idx.begin(), idx.end(), lo);\n"
        "    auto e = std::upper_bound(idx.begin(), idx.end(), hi);\n"
        "    return {b - idx.begin(), e - idx.begin()};\n"
        "  }\n"
        "  int64_t owned_crd_index(int level, int64_t k) const { return levels_[level].crd_idx[k]; }\n",
    ),
    # (2) locate_coord searches only the owned part of the row.
    (
        "    int64_t lo = r.lo, hi = r.hi;\n"
        "    while (lo <= hi) {\n"
        "      int64_t mid = (lo + hi) / 2;\n"
        "      int64_t c = a.view->crd_at(level, mid);\n"
        "      if (c == coord) return mid;\n",
        "    auto [ob, oe] = a.view->owned_span(level, r.lo, r.hi);  // [graft oracle patch]\n"
        "    int64_t lo = ob, hi = oe - 1;\n"
        "    while (lo <= hi) {\n"
        "      int64_t mid = (lo + hi) / 2;\n"
        "      int64_t c = a.view->crd_at(level, a.view->owned_crd_index(level, mid));\n"
        "      if (c == coord) return a.view->owned_crd_index(level, mid);\n",
    ),
    # (3) copy, do not move, the candidate lists (fix for sim.cpp:451).
    (
        "      for (auto& c : candidates) lists.push_back(std::move(*c));\n",
        "      for (auto& c : candidates) lists.push_back(*c);  // [graft oracle patch]\n",
    ),
]


def main() -> int:
    src = os.path.join(REF, "core", "src", "sim.cpp")
    with open(src) as f:
        text = f.read()
    for old, new in EDITS:
        if text.count(old) != 1:
            print(f"patch_ref: anchor not found exactly once in {src}:\n{old}", file=sys.stderr)
            return 1
        text = text.replace(old, new)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "sim.cpp"), "w") as f:
        f.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
