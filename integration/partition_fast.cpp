// dspar::Partition (/root/reference/proj/core/include/dspar/partition.hpp)
// for the drop-in library, linked in place of partition.cpp.
//
// Same contract as the reference's class (partition.cpp:10-60): subsets are
// stored sorted and deduplicated, an index outside the parent space throws
// std::invalid_argument("Partition: subset index outside parent space"),
// disjointness is computed from the subsets, never assumed.  The difference
// is cost: every subset the GPU dependent partitioning hands to plan()
// (integration/deppart_gpu.cpp) and every contiguous block the planner builds
// is already strictly increasing, so the constructor checks that in one pass
// and sorts only a subset that is not (over the colours on all host
// threads); disjointness is decided from the subsets' spans where they settle
// it, with the reference's full bitmap scan only as the fallback.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <thread>
#include <vector>

#include "dspar/partition.hpp"

namespace dspar {

namespace {

bool strictly_increasing(const std::vector<int64_t>& s) {
  for (size_t k = 1; k < s.size(); k++)
    if (s[k - 1] >= s[k]) return false;
  return true;
}

// Runs f(c) for c in [0, n) on up to hardware_concurrency threads (a plain
// loop below ~1 M indices, where threads cost more than they save).
template <class F>
void for_colours(size_t n, size_t work, F f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  if (n < 2 || work < (size_t(1) << 20) || hw == 1) {
    for (size_t c = 0; c < n; c++) f(c);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::atomic<bool> failed{false};
  for (unsigned t = 0; t < std::min<size_t>(hw, n); t++)
    pool.emplace_back([&] {
      for (size_t c = next++; c < n && !failed; c = next++) {
        try {
          f(c);
        } catch (...) {
          if (!failed.exchange(true)) err = std::current_exception();
        }
      }
    });
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

Partition::Partition(IndexSpace parent, std::vector<std::vector<int64_t>> subsets)
    : parent_(std::move(parent)), subsets_(std::move(subsets)) {
  const int64_t total = parent_.total();
  size_t work = 0;
  for (const auto& s : subsets_) work += s.size();
  // canonical subsets (sorted, unique) and the range check
  for_colours(subsets_.size(), work, [&](size_t c) {
    auto& s = subsets_[c];
    if (!strictly_increasing(s)) {
      std::sort(s.begin(), s.end());
      s.erase(std::unique(s.begin(), s.end()), s.end());
    }
    if (!s.empty() && (s.front() < 0 || s.back() >= total))
      throw std::invalid_argument("Partition: subset index outside parent space");
  });
  // disjointness: an index owned by two colours.  Colours whose [min, max]
  // spans do not overlap cannot share an index (contiguous blocks: no scan);
  // two overlapping spans are intersected by a merge with early exit (the
  // replicated partitions stop at their first element); only when spans
  // overlap without a common element does the exact bitmap scan run.
  std::vector<std::pair<int64_t, size_t>> spans;  // (min, colour) of the non-empty subsets
  for (size_t c = 0; c < subsets_.size(); c++)
    if (!subsets_[c].empty()) spans.emplace_back(subsets_[c].front(), c);
  std::sort(spans.begin(), spans.end());
  disjoint_ = true;
  bool exact_scan = false;
  int64_t reach = -1;  // largest max so far, and its colour
  size_t reach_c = 0;
  for (const auto& [lo, c] : spans) {
    const auto& s = subsets_[c];
    if (lo <= reach) {
      const auto& t = subsets_[reach_c];
      auto a = s.begin(), b = t.begin();
      while (a != s.end() && b != t.end()) {
        if (*a < *b) ++a;
        else if (*b < *a) ++b;
        else { disjoint_ = false; return; }
      }
      exact_scan = true;  // overlapping spans, no common index with that colour
    }
    if (s.back() > reach) reach = s.back(), reach_c = c;
  }
  if (!exact_scan) return;
  std::vector<uint64_t> seen(static_cast<size_t>((total + 63) / 64), 0);
  for (const auto& s : subsets_)
    for (int64_t i : s) {
      uint64_t& w = seen[static_cast<size_t>(i >> 6)];
      const uint64_t bit = uint64_t(1) << (i & 63);
      if (w & bit) {
        disjoint_ = false;
        return;
      }
      w |= bit;
    }
}

bool Partition::contains(int64_t color, int64_t index) const {
  const auto& s = subsets_[color];
  return std::binary_search(s.begin(), s.end(), index);
}

std::vector<int64_t> Partition::colors_of(int64_t index) const {
  std::vector<int64_t> out;
  for (int64_t c = 0; c < num_colors(); c++)
    if (contains(c, index)) out.push_back(c);
  return out;
}

Partition Partition::replicated(IndexSpace parent, int64_t colors) {
  std::vector<int64_t> every(static_cast<size_t>(parent.total()));
  std::iota(every.begin(), every.end(), int64_t(0));
  return Partition(std::move(parent), std::vector<std::vector<int64_t>>(static_cast<size_t>(colors), every));
}

std::string Partition::to_string() const {
  std::ostringstream s;
  for (int64_t c = 0; c < num_colors(); c++) {
    if (c) s << " ";
    s << c << ": {";
    const auto& sub = subsets_[c];
    for (size_t k = 0; k < sub.size(); k++) s << (k ? ", " : "") << sub[k];
    s << "}";
  }
  return s.str();
}

}  // namespace dspar
