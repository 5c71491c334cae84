// Dependent partitioning on the GPU (K1 universe / K2 nonzero / K2m materialise).
//
// The reference materialises every partition as sorted index sets
// (Partition, partition.cpp:10-24) and derives them with image / preimage
// (deppart.cpp:15-53) level by level (level_partition.cpp:134-276).  For the
// schedules on the hot path every colour's sub-region is a contiguous span
// per level (filtered to non-empty entries by preimage), so the GPU computes
// the spans directly:
//   * universe split of the top level: divide_bounds (planner.cpp:10-20) on
//     the coordinate extent, then each compressed level maps a span [a,b] to
//     [rowptr[a], rowptr[b+1]-1] -- the image of contiguous pos entries;
//   * nonzero split of level L: divide_bounds on the level's positions, then
//     each level up maps a position to its owner entry (the preimage of a
//     contiguous crd range is the non-empty entries between the owners of its
//     ends) with a warp-parallel 32-ary search, and the top-level coordinates
//     of the ends are project_to_universe's [min, max] (planner.cpp:50-69).
// One warp per colour; O(P) probes, so this is a latency kernel.
#include <algorithm>
#include <cub/cub.cuh>

#include "common.cuh"

namespace spd {

struct TreeView {
  int nlevels = 0;
  int kind[8];
  int64_t parent[8], positions[8], fanout[8], dom0[8];
  const int64_t* rowptr[8];
  const int64_t* crd[8];
  int64_t top_extent = 0;  // extent of the top level's first mode
};

static TreeView make_view(const spd_tensor* t) {
  if (t->levels.size() > 8) throw ValidationError("at most 8 stored levels are supported");
  TreeView v;
  v.nlevels = (int)t->levels.size();
  for (int l = 0; l < v.nlevels; l++) {
    const auto& L = t->levels[l];
    v.kind[l] = L.kind;
    v.parent[l] = L.parent_positions;
    v.positions[l] = L.positions;
    int64_t f = 1;
    for (int64_t e : L.dom) f *= e;
    v.fanout[l] = f;
    v.dom0[l] = L.dom.empty() ? 0 : L.dom[0];
    v.rowptr[l] = L.rowptr;
    v.crd[l] = L.crd;
  }
  if (v.nlevels > 0) v.top_extent = t->dims[t->mode_order[t->groups[0][0]]];
  return v;
}

__device__ __forceinline__ void divide_bounds_dev(int64_t n, int64_t pieces, int64_t c,
                                                  int64_t& lo, int64_t& hi) {
  int64_t block = pieces > 0 ? n / pieces : 0;
  lo = c * block;
  hi = c + 1 == pieces ? n - 1 : lo + block - 1;
}

// Top-level coordinate of a top position (planner.cpp:40-46).
__device__ __forceinline__ int64_t top_coordinate(const TreeView& v, int64_t p) {
  if (v.kind[0] == SPD_DENSE) return p / (v.fanout[0] / (v.dom0[0] > 0 ? v.dom0[0] : 1));
  return __ldg(v.crd[0] + p);
}

__global__ void k_partition_universe(TreeView v, int64_t pieces, DevColor* __restrict__ out) {
  const int64_t c = blockIdx.x;
  const int lane = lane_id();
  int64_t lo, hi;
  divide_bounds_dev(v.top_extent, pieces, c, lo, hi);
  int64_t a, b;  // positions of level 0
  if (v.kind[0] == SPD_DENSE) {
    int64_t rest = v.fanout[0] / (v.dom0[0] > 0 ? v.dom0[0] : 1);
    a = lo * rest;
    b = lo <= hi ? (hi + 1) * rest - 1 : a - 1;
  } else {  // bucket sorted top crd by coordinate range (level_partition.cpp:193-205)
    int64_t n0 = v.positions[0];
    a = warp_upper_bound(v.crd[0], n0, lo - 1);
    b = lo <= hi ? warp_upper_bound(v.crd[0], n0, hi) - 1 : a - 1;
  }
  int64_t pa = 0, pb = lo <= hi ? 0 : -1;
  for (int l = 1; l < v.nlevels; l++) {
    pa = a, pb = b;
    if (v.kind[l] == SPD_COMPRESSED) {
      if (a <= b) {
        int64_t na = __ldg(v.rowptr[l] + a), nb = __ldg(v.rowptr[l] + b + 1) - 1;
        a = na, b = nb;
      } else {
        int64_t at = __ldg(v.rowptr[l] + (a < v.parent[l] ? a : v.parent[l]));
        a = at, b = at - 1;
      }
    } else {
      int64_t f = v.fanout[l];
      int64_t na = a * f;
      b = a <= b ? b * f + f - 1 : na - 1;
      a = na;
    }
  }
  if (v.nlevels == 1) pa = 0, pb = a <= b ? 0 : -1;
  if (lane == 0) {
    DevColor d;
    d.pub.color = {lo, hi};
    d.pub.top = {lo, hi};
    d.pub.par = {pa, pb};
    d.pub.q = {a, b};
    d.w_lo = 1, d.w_hi = 0, d.chunk_begin = 0, d.pad = 0;
    out[c] = d;
  }
}

__global__ void k_partition_nonzero(TreeView v, int level, int64_t pieces,
                                    DevColor* __restrict__ out) {
  const int64_t c = blockIdx.x;
  const int lane = lane_id();
  int64_t lo, hi;
  divide_bounds_dev(v.positions[level], pieces, c, lo, hi);
  DevColor d;
  d.pub.color = {lo, hi};
  d.pub.q = {lo, hi};
  d.w_lo = 1, d.w_hi = 0, d.chunk_begin = 0, d.pad = 0;
  if (lo > hi) {
    d.pub.par = {0, -1};
    d.pub.top = {0, -1};
  } else {
    int64_t a = lo, b = hi;
    d.pub.par = {0, 0};
    for (int l = level; l >= 1; l--) {
      if (v.kind[l] == SPD_COMPRESSED) {
        a = warp_owner(v.rowptr[l], v.parent[l], a);
        b = warp_owner(v.rowptr[l], v.parent[l], b);
      } else {
        a /= v.fanout[l];
        b /= v.fanout[l];
      }
      if (l == level) d.pub.par = {a, b};
    }
    d.pub.top = {top_coordinate(v, a), top_coordinate(v, b)};
  }
  if (lane == 0) out[c] = d;
}

// ---- K2m: materialisation for bit-exact comparison with the reference ----
// Flags over a candidate span of one level's entries.
__global__ void k_flag_nonempty(const int64_t* __restrict__ rowptr, int64_t lo, int64_t hi,
                                unsigned char* __restrict__ flags) {
  for (int64_t p = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= hi;
       p += (int64_t)gridDim.x * blockDim.x)
    flags[p - lo] = __ldg(rowptr + p + 1) > __ldg(rowptr + p);
}
// Parent entry r is coloured iff its (non-empty) range meets the coloured
// child set (preimage, deppart.cpp:33-53): child flags over [clo, chi].
__global__ void k_flag_preimage(const int64_t* __restrict__ rowptr, int64_t lo, int64_t hi,
                                const unsigned char* __restrict__ child, int64_t clo, int64_t chi,
                                unsigned char* __restrict__ flags) {
  for (int64_t r = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= hi;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = max(__ldg(rowptr + r), clo), e = min(__ldg(rowptr + r + 1) - 1, chi);
    unsigned char f = 0;
    for (int64_t q = s; q <= e && !f; q++) f = child[q - clo];
    flags[r - lo] = f;
  }
}


// ---- universe split of a compressed level (bucketCoords) ------------------
// LevelPartitioner::finalize, compressed universe entry
// (level_partition.cpp:193-205): colour c holds the positions of the level
// whose coordinate lies in divide_bounds(extent, P)[c] -- bucketed by
// coordinate, not contiguous in position space.
__device__ __forceinline__ int64_t bucket_of(int64_t j, int64_t extent, int64_t pieces) {
  const int64_t block = extent / pieces;  // divide_bounds: the last colour takes the rest
  if (block == 0) return pieces - 1;
  const int64_t c = j / block;
  return c < pieces - 1 ? c : pieces - 1;
}

__global__ void k_bucket_keys(const int64_t* __restrict__ crd, int64_t n, int64_t extent, int64_t pieces,
                              int32_t* __restrict__ keys, int64_t* __restrict__ pos) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    keys[q] = (int32_t)bucket_of(__ldg(crd + q), extent, pieces);
    pos[q] = q;
  }
}

// weight of a bucketed position: its leaf count (the rows of the next level
// it spans, product of dense extents below) -- 1 on the leaf level
__global__ void k_bucket_weights(const int64_t* __restrict__ sorted_pos, int64_t n,
                                 const int64_t* __restrict__ next_rowptr, int64_t* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = sorted_pos[i];
    w[i] = next_rowptr ? __ldg(next_rowptr + q + 1) - __ldg(next_rowptr + q) : 1;
  }
}

// colour boundaries in the sorted keys
__global__ void k_bucket_bounds(const int32_t* __restrict__ keys, int64_t n, int64_t pieces,
                                int64_t* __restrict__ off) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= pieces; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;  // first index with key >= c
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < c) lo = mid + 1; else hi = mid;
    }
    off[c] = lo;
  }
}

// leaf positions of bucket y inside level-position span x: two searches in
// the bucket's ascending positions, a difference of the weight prefix sums
__global__ void k_bucket_grid(const int64_t* __restrict__ pos, const int64_t* __restrict__ pref,
                              const int64_t* __restrict__ off, int64_t Y, const int64_t* __restrict__ spans,
                              int64_t X, int64_t* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= X * Y) return;
  const int64_t x = t / Y, y = t % Y;
  const int64_t lo = spans[2 * x], hi = spans[2 * x + 1];
  if (lo > hi) {
    out[t] = 0;
    return;
  }
  int64_t a = off[y], b = off[y + 1];
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (pos[mid] < lo) a = mid + 1; else b = mid;
  }
  int64_t c = a, d = off[y + 1];
  while (c < d) {
    const int64_t mid = (c + d) >> 1;
    if (pos[mid] <= hi) c = mid + 1; else d = mid;
  }
  out[t] = pref[c] - pref[a];
}

}  // namespace spd

using namespace spd;

static void run_bucket(spd_context* ctx, const spd_tensor* t, int level, int64_t pieces, int64_t* counts_out) {
  checked(ctx);
  if (!t) throw ValidationError("null tensor");
  if (pieces < 1) throw ValidationError("pieces must be positive");
  if (level < 1 || level >= (int)t->levels.size() || t->levels[level].kind != SPD_COMPRESSED)
    throw ValidationError("unsupported on gpu: the bucket split needs an inner compressed level");
  if (t->piece) throw ValidationError("unsupported on gpu: bucket split of a placed piece");
  activate(ctx);
  settle_restage(t);
  const spd_level_store& L = t->levels[level];
  const int64_t n = L.positions;
  const int64_t extent = t->dims[t->mode_order[t->groups[level][0]]];
  cudaStream_t s = ctx->stream;
  auto& B = ctx->bucket;
  B.n = n;
  B.pieces = pieces;
  int32_t* keys = (int32_t*)B.keys.reserve(sizeof(int32_t) * 2 * (n > 0 ? n : 1));
  int32_t* keys_out = keys + (n > 0 ? n : 1);
  int64_t* pos_in = (int64_t*)B.tmp.reserve(sizeof(int64_t) * 2 * (n + 1));
  int64_t* w = pos_in + (n + 1);
  B.pos = (int64_t*)B.pos_buf.reserve(sizeof(int64_t) * (n > 0 ? n : 1));
  B.pref = (int64_t*)B.pref_buf.reserve(sizeof(int64_t) * (n + 1));
  B.off = (int64_t*)B.off_buf.reserve(sizeof(int64_t) * (pieces + 1));
  const unsigned grid = (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), ctx->num_sms * 16);
  SPD_CUDA(cudaMemsetAsync(B.pref, 0, sizeof(int64_t), s));
  if (n > 0) {
    k_bucket_keys<<<grid, 256, 0, s>>>(L.crd, n, extent, pieces, keys, pos_in);
    SPD_CHECK_LAUNCH();
    int bits = 1;
    while ((int64_t(1) << bits) < pieces) bits++;
    size_t bytes = 0;  // stable: positions stay ascending within a colour
    SPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, pos_in, B.pos, n, 0, bits, s));
    void* tmp = ctx->scratch[5].reserve(bytes);
    SPD_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, keys_out, pos_in, B.pos, n, 0, bits, s));
    const bool leaf = level + 1 == (int)t->levels.size();
    k_bucket_weights<<<grid, 256, 0, s>>>(B.pos, n, leaf ? nullptr : t->levels[level + 1].rowptr, w);
    SPD_CHECK_LAUNCH();
    bytes = 0;
    SPD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, w, B.pref + 1, n, s));
    tmp = ctx->scratch[5].reserve(bytes);
    SPD_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, w, B.pref + 1, n, s));
    ctx->launches += 4;
  }
  k_bucket_bounds<<<(unsigned)ceil_div(pieces + 1, 256), 256, 0, s>>>(keys_out, n, pieces, B.off);
  SPD_CHECK_LAUNCH();
  ctx->launches++;
  B.tensor = t;
  B.level = level;
  std::vector<int64_t> off(pieces + 1);
  SPD_CUDA(cudaMemcpyAsync(off.data(), B.off, sizeof(int64_t) * (pieces + 1), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  if (counts_out)
    for (int64_t c = 0; c < pieces; c++) counts_out[c] = off[c + 1] - off[c];
}

extern "C" {

int spd_partition_bucket(spd_context* ctx, const spd_tensor* t, int level, int64_t pieces, int64_t* counts_out) {
  return guarded([&] { run_bucket(ctx, t, level, pieces, counts_out); });
}

int spd_bucket_positions(spd_context* ctx, int64_t color, int64_t* out, int64_t cap, int64_t* count) {
  return guarded([&] {
    checked(ctx);
    auto& B = ctx->bucket;
    if (!B.tensor) throw ValidationError("no bucket split on the context: call spd_partition_bucket first");
    if (color < 0 || color >= B.pieces) throw ValidationError("no such colour");
    if (!count) throw ValidationError("null argument");
    activate(ctx);
    int64_t o[2];
    SPD_CUDA(cudaMemcpy(o, B.off + color, sizeof(o), cudaMemcpyDeviceToHost));
    *count = o[1] - o[0];
    const int64_t k = std::min<int64_t>(*count, cap);
    if (k > 0 && out) SPD_CUDA(cudaMemcpy(out, B.pos + o[0], sizeof(int64_t) * k, cudaMemcpyDeviceToHost));
  });
}

int spd_bucket_grid_work(spd_context* ctx, const int64_t* spans, int64_t nspans, int64_t* out) {
  return guarded([&] {
    checked(ctx);
    auto& B = ctx->bucket;
    if (!B.tensor) throw ValidationError("no bucket split on the context: call spd_partition_bucket first");
    if (nspans < 0 || (nspans > 0 && (!spans || !out))) throw ValidationError("null argument");
    if (nspans == 0) return;
    activate(ctx);
    cudaStream_t s = ctx->stream;
    const int64_t cells = nspans * B.pieces;
    int64_t* d = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (2 * nspans + cells));
    SPD_CUDA(cudaMemcpyAsync(d, spans, sizeof(int64_t) * 2 * nspans, cudaMemcpyHostToDevice, s));
    k_bucket_grid<<<(unsigned)ceil_div(cells, 256), 256, 0, s>>>(B.pos, B.pref, B.off, B.pieces, d, nspans,
                                                                  d + 2 * nspans);
    SPD_CHECK_LAUNCH();
    ctx->launches++;
    SPD_CUDA(cudaMemcpyAsync(out, d + 2 * nspans, sizeof(int64_t) * cells, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    dev_free(ctx, d);
  });
}

}  // extern "C"

static void run_partition(spd_context* ctx, const spd_tensor* t, int level, int64_t pieces,
                          bool nonzero, spd_color* colors_out) {
  checked(ctx);
  if (!t) throw ValidationError("null tensor");
  if (pieces < 1) throw ValidationError("pieces must be positive");
  if (t->levels.empty()) throw ValidationError("cannot partition a rank-0 tensor");
  activate(ctx);
  settle_restage(t);
  TreeView v = make_view(t);
  ctx->colors_dev.reserve(sizeof(DevColor) * pieces);
  DevColor* cols = (DevColor*)ctx->colors_dev.ptr;
  if (nonzero) {
    if (level < 0 || level >= v.nlevels) throw ValidationError("no such level");
    k_partition_nonzero<<<(unsigned)pieces, 32, 0, ctx->stream>>>(v, level, pieces, cols);
  } else {
    k_partition_universe<<<(unsigned)pieces, 32, 0, ctx->stream>>>(v, pieces, cols);
  }
  SPD_CHECK_LAUNCH();
  ctx->launches++;
  ctx->split = nonzero ? SplitKind::NonZero : SplitKind::Universe;
  ctx->split_tensor = t;
  ctx->split_level = nonzero ? level : 0;
  ctx->pieces = pieces;
  ctx->colors_host_valid = false;
  if (colors_out) {
    const auto& h = host_colors(ctx);
    std::copy(h.begin(), h.end(), colors_out);
  }
}

extern "C" {

int spd_partition_universe(spd_context* ctx, const spd_tensor* t, int64_t pieces,
                           spd_color* colors_out) {
  return guarded([&] { run_partition(ctx, t, 0, pieces, false, colors_out); });
}

int spd_partition_nonzero(spd_context* ctx, const spd_tensor* t, int level, int64_t pieces,
                          spd_color* colors_out) {
  return guarded([&] { run_partition(ctx, t, level, pieces, true, colors_out); });
}

int spd_partition_materialize(spd_context* ctx, const spd_tensor* t, int level, int which,
                              int64_t color, int64_t* out, int64_t cap, int64_t* count) {
  return guarded([&] {
    checked(ctx);
    if (ctx->split == SplitKind::None || ctx->split_tensor != t)
      throw ValidationError("no partition of this tensor on the context");
    if (color < 0 || color >= ctx->pieces) throw ValidationError("no such colour");
    activate(ctx);
    const spd_color col = host_colors(ctx)[color];
    const int nl = (int)t->levels.size();
    std::vector<int64_t> result;
    auto push_span = [&](int64_t a, int64_t b) {
      for (int64_t i = a; i <= b; i++) result.push_back(i);
    };
    if (which == 3) {
      push_span(col.q.lo, col.q.hi);  // vals = copy of the leaf partition
    } else {
      if (level < 0 || level >= nl) throw ValidationError("no such level");
      const auto& L = t->levels[level];
      if ((which == 0) != (L.kind == SPD_DENSE))
        throw ValidationError("region does not exist on this level");
      if (ctx->split == SplitKind::Universe) {
        // Spans per level walking down from the top (copy + image); a dense
        // level's dom partition is the projection of its positions.
        int64_t a = col.top.lo, b = col.top.hi;
        const auto& L0 = t->levels[0];
        if (L0.kind == SPD_DENSE) {
          int64_t rest = 1;
          for (size_t k = 1; k < L0.dom.size(); k++) rest *= L0.dom[k];
          int64_t na = a * rest;
          b = a <= b ? (b + 1) * rest - 1 : na - 1;
          a = na;
        } else {
          std::vector<int64_t> crd0(L0.positions);
          if (L0.positions)
            SPD_CUDA(cudaMemcpy(crd0.data(), L0.crd, 8 * L0.positions, cudaMemcpyDeviceToHost));
          int64_t lo = a, hi = b;
          a = std::lower_bound(crd0.begin(), crd0.end(), lo) - crd0.begin();
          b = lo <= hi ? (std::upper_bound(crd0.begin(), crd0.end(), hi) - crd0.begin()) - 1 : a - 1;
        }
        int64_t pa = 0, pb = a <= b ? 0 : -1;  // parent span of level 0 = the root
        for (int l = 1; l <= level; l++) {
          pa = a, pb = b;
          const auto& Ll = t->levels[l];
          if (Ll.kind == SPD_COMPRESSED) {
            int64_t ra = 0, rb = 0;
            if (a <= b) {
              SPD_CUDA(cudaMemcpy(&ra, Ll.rowptr + a, 8, cudaMemcpyDeviceToHost));
              SPD_CUDA(cudaMemcpy(&rb, Ll.rowptr + b + 1, 8, cudaMemcpyDeviceToHost));
              a = ra, b = rb - 1;
            } else {
              b = a - 1;
            }
          } else {
            int64_t f = 1;
            for (int64_t e : Ll.dom) f *= e;
            int64_t na = a * f;
            b = a <= b ? b * f + f - 1 : na - 1;
            a = na;
          }
        }
        if (which == 2) push_span(a, b);                 // crd = image
        else if (which == 1) push_span(pa, pb);          // pos = copy of the parent colouring
        else {                                           // dom: projected positions
          int64_t f = 1;
          for (int64_t e : L.dom) f *= e;
          std::vector<char> seen(f, 0);
          for (int64_t p = a; p <= b; p++) seen[p % f] = 1;
          for (int64_t s = 0; s < f; s++)
            if (seen[s]) result.push_back(s);
        }
      } else {
        // Nonzero: walk up from the split level with exact flags.
        int split = ctx->split_level;
        if (level > split) throw ValidationError("levels below the split level are not derived here");
        // coloured span + flags at the current level's positions
        int64_t lo = col.q.lo, hi = col.q.hi;
        std::vector<unsigned char> flags(hi >= lo ? hi - lo + 1 : 0, 1);
        unsigned char* dflags = nullptr;
        for (int l = split; l >= level; l--) {
          const auto& Ll = t->levels[l];
          if (l == level && which == 2) {  // crd of this level = coloured positions
            for (int64_t i = lo; i <= hi; i++)
              if (flags[i - lo]) result.push_back(i);
            break;
          }
          if (l == level && which == 0) {  // dense dom: projected positions
            int64_t f = 1;
            for (int64_t e : Ll.dom) f *= e;
            std::vector<char> seen(f, 0);
            for (int64_t i = lo; i <= hi; i++)
              if (flags[i - lo]) seen[i % f] = 1;
            for (int64_t s = 0; s < f; s++)
              if (seen[s]) result.push_back(s);
            break;
          }
          // go up one level: parent positions coloured
          int64_t nlo, nhi;
          std::vector<unsigned char> nflags;
          if (lo > hi) {
            nlo = 0, nhi = -1;
          } else if (Ll.kind == SPD_COMPRESSED) {
            std::vector<int64_t> rp(Ll.parent_positions + 1);
            SPD_CUDA(cudaMemcpy(rp.data(), Ll.rowptr, 8 * rp.size(), cudaMemcpyDeviceToHost));
            nlo = (std::upper_bound(rp.begin(), rp.end(), lo) - rp.begin()) - 1;
            nhi = (std::upper_bound(rp.begin(), rp.end(), hi) - rp.begin()) - 1;
            int64_t n = nhi - nlo + 1;
            unsigned char *dchild = nullptr, *dout = nullptr;
            SPD_CUDA(cudaMalloc(&dchild, flags.size()));
            SPD_CUDA(cudaMalloc(&dout, n));
            SPD_CUDA(cudaMemcpy(dchild, flags.data(), flags.size(), cudaMemcpyHostToDevice));
            k_flag_preimage<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0,
                              ctx->stream>>>(Ll.rowptr, nlo, nhi, dchild, lo, hi, dout);
            SPD_CHECK_LAUNCH();
            nflags.resize(n);
            SPD_CUDA(cudaMemcpyAsync(nflags.data(), dout, n, cudaMemcpyDeviceToHost, ctx->stream));
            SPD_CUDA(cudaStreamSynchronize(ctx->stream));
            cudaFree(dchild);
            cudaFree(dout);
          } else {
            int64_t f = 1;
            for (int64_t e : Ll.dom) f *= e;
            nlo = lo / f, nhi = hi / f;
            nflags.assign(nhi - nlo + 1, 0);
            for (int64_t i = lo; i <= hi; i++)
              if (flags[i - lo]) nflags[i / f - nlo] = 1;
          }
          if (l == level && which == 1) {  // pos of this level = coloured parent entries
            for (int64_t i = nlo; i <= nhi; i++)
              if (nflags[i - nlo]) result.push_back(i);
            break;
          }
          lo = nlo, hi = nhi;
          flags.swap(nflags);
        }
        (void)dflags;
      }
    }
    *count = (int64_t)result.size();
    for (int64_t k = 0; k < *count && k < cap; k++) out[k] = result[k];
  });
}

}  // extern "C"
