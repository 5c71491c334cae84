// GPU dependent partitioning for the reference's own planner: the operators
// of /root/reference/proj/core/include/dspar/deppart.hpp (image, preimage,
// partition_by_bounds, copy_partition) implemented over the C-ABI, so that
// plan() (planner.cpp:142-359), LevelPartitioner::finalize
// (level_partition.cpp:134-212), partition_from_parent / partition_from_child
// (:214-251) -- the paper's format-abstraction layer -- run their set
// algebra on the GPU.  A dspar build links this translation unit in place of
// deppart.cpp; oracle/Makefile builds the reference's own
// doctest suite both ways (oracle/_ref/dspar_ref_tests_gpudeppart is the GPU
// one) and the integration library with it.
//
// Semantics are the reference's: the same preconditions (std::invalid_argument
// on a non-range source, a partition over the wrong space, negative colours,
// out-of-space bounds, a mismatched copy), the result a Partition built from
// sorted unique subsets (its constructor recomputes disjointness).
#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dspar/deppart.hpp"
#include "spdistal_b200.h"

namespace dspar {

namespace {

spd_context* gpu() {
  static spd_context* ctx = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (spd_context_create(0, nullptr, &ctx) != SPD_OK)
      throw std::runtime_error(std::string("deppart on gpu: ") + spd_last_error());
  });
  return ctx;
}

void check(int st) {
  if (st == SPD_OK) return;
  if (st == SPD_ERR_VALIDATION) throw std::invalid_argument(spd_last_error());
  throw std::runtime_error(spd_last_error());
}

// A Partition as the ABI's (off[P+1], idx) arrays.
void flatten(const Partition& p, std::vector<int64_t>& off, std::vector<int64_t>& idx) {
  off.assign(static_cast<size_t>(p.num_colors()) + 1, 0);
  size_t total = 0;
  for (int64_t c = 0; c < p.num_colors(); c++) total += p.subset(c).size();
  idx.clear();
  idx.reserve(total);
  for (int64_t c = 0; c < p.num_colors(); c++) {
    const auto& s = p.subset(c);
    idx.insert(idx.end(), s.begin(), s.end());
    off[static_cast<size_t>(c) + 1] = static_cast<int64_t>(idx.size());
  }
}

Partition unflatten(const IndexSpace& space, int64_t P, const std::vector<int64_t>& off,
                    const std::vector<int64_t>& idx) {
  std::vector<std::vector<int64_t>> subsets(static_cast<size_t>(P));
  for (int64_t c = 0; c < P; c++)
    subsets[static_cast<size_t>(c)].assign(idx.begin() + off[static_cast<size_t>(c)],
                                           idx.begin() + off[static_cast<size_t>(c) + 1]);
  return Partition(space, std::move(subsets));
}

const int64_t* range_pairs(const Region& r) {
  static_assert(sizeof(CoordRange) == 2 * sizeof(int64_t), "CoordRange is two int64");
  return reinterpret_cast<const int64_t*>(r.range_values().data());
}

using HostOp = int (*)(spd_context*, const int64_t*, int64_t, int64_t, int64_t, const int64_t*, const int64_t*,
                       int64_t*, int64_t*, int64_t, int64_t*, int*);

// `bound`: an upper bound of the result's size when it is cheap to state, so
// one call both sizes and fills; else -1 and the result is sized first.
Partition run_op(HostOp op, const Region& source, const Partition& part, const IndexSpace& out_space,
                 int64_t dest_extent, int64_t bound) {
  std::vector<int64_t> off, idx;
  flatten(part, off, idx);
  const int64_t P = part.num_colors();
  std::vector<int64_t> out_off(static_cast<size_t>(P) + 1, 0);
  int64_t total = 0;
  int disjoint = -1;
  std::vector<int64_t> out_idx(static_cast<size_t>(std::max<int64_t>(bound, 0)));
  check(op(gpu(), range_pairs(source), source.size(), dest_extent, P, off.data(), idx.data(), out_off.data(),
           bound >= 0 ? out_idx.data() : nullptr, std::max<int64_t>(bound, 0), &total, &disjoint));
  if (total > bound) {
    out_idx.assign(static_cast<size_t>(total), 0);
    check(op(gpu(), range_pairs(source), source.size(), dest_extent, P, off.data(), idx.data(), out_off.data(),
             out_idx.data(), total, &total, &disjoint));
  }
  out_idx.resize(static_cast<size_t>(total));
  return unflatten(out_space, P, out_off, out_idx);
}

}  // namespace

Partition image(const Region& source, const Partition& src_part, const IndexSpace& dest) {
  if (source.kind() != ValueKind::Range)
    throw std::invalid_argument("image: source region must hold coordinate ranges");
  if (source.range_dest_extent() != dest.total())
    throw std::invalid_argument("image: source ranges do not reference dest");
  if (!(src_part.parent() == source.space()))
    throw std::invalid_argument("image: partition is not over the source's space");
  int64_t bound = 0;  // the expansion's length: every range of every coloured source entry
  const auto& ranges = source.range_values();
  for (int64_t c = 0; c < src_part.num_colors(); c++)
    for (int64_t i : src_part.subset(c)) bound += std::max<int64_t>(ranges[static_cast<size_t>(i)].hi -
                                                                    ranges[static_cast<size_t>(i)].lo + 1, 0);
  return run_op(spd_deppart_image_host, source, src_part, dest, dest.total(), bound);
}

Partition preimage(const Region& source, const Partition& dest_part, const IndexSpace& dest) {
  if (source.kind() != ValueKind::Range)
    throw std::invalid_argument("preimage: source region must hold coordinate ranges");
  if (source.range_dest_extent() != dest.total())
    throw std::invalid_argument("preimage: source ranges do not reference dest");
  if (!(dest_part.parent() == dest)) throw std::invalid_argument("preimage: partition is not over dest");
  const int64_t all = dest_part.num_colors() * source.size();  // every colour holding every source entry
  return run_op(spd_deppart_preimage_host, source, dest_part, source.space(), dest.total(),
                all <= (int64_t(1) << 27) ? all : -1);
}

Partition partition_by_bounds(const IndexSpace& space, const std::map<int64_t, std::vector<CoordRange>>& coloring) {
  int64_t P = 0;
  for (const auto& entry : coloring) {
    if (entry.first < 0) throw std::invalid_argument("partition_by_bounds: negative color");
    P = std::max(P, entry.first + 1);
  }
  const int R = space.rank();
  // colours absent from the map colour nothing: an empty box
  std::vector<int64_t> bounds(static_cast<size_t>(P) * R * 2, 0);
  for (int64_t c = 0; c < P; c++) bounds[static_cast<size_t>(c) * R * 2 + 1] = -1;
  for (const auto& [color, box] : coloring) {
    if (static_cast<int>(box.size()) != R) throw std::invalid_argument("partition_by_bounds: bounds rank mismatch");
    for (int d = 0; d < R; d++) {
      bounds[(static_cast<size_t>(color) * R + d) * 2] = box[d].lo;
      bounds[(static_cast<size_t>(color) * R + d) * 2 + 1] = box[d].hi;
    }
  }
  if (R == 0) {  // a rank-0 space has one point; every listed colour holds it
    std::vector<std::vector<int64_t>> subsets(static_cast<size_t>(P));
    for (const auto& entry : coloring) subsets[static_cast<size_t>(entry.first)] = {0};
    return Partition(space, std::move(subsets));
  }
  std::vector<int64_t> extents(space.extents().begin(), space.extents().end());
  std::vector<int64_t> out_off(static_cast<size_t>(P) + 1, 0);
  int64_t total = 0;
  int disjoint = -1;
  check(spd_deppart_by_bounds_host(gpu(), R, extents.data(), P, bounds.data(), out_off.data(), nullptr, 0, &total,
                                   &disjoint));
  std::vector<int64_t> out_idx(static_cast<size_t>(total));
  check(spd_deppart_by_bounds_host(gpu(), R, extents.data(), P, bounds.data(), out_off.data(), out_idx.data(), total,
                                   &total, &disjoint));
  return unflatten(space, P, out_off, out_idx);
}

Partition copy_partition(const Partition& part, const IndexSpace& target) {
  if (part.parent().total() != target.total()) throw std::invalid_argument("copy_partition: extent mismatch");
  return Partition(target, part.subsets());  // a reinterpretation: the same linear indices
}

Partition copy_partition(const Partition& part, const Region& target) { return copy_partition(part, target.space()); }

}  // namespace dspar
