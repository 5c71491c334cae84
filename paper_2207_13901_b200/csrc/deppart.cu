// General dependent partitioning on the GPU: image,
// preimage and partition_by_bounds over MATERIALISED partitions -- arbitrary,
// possibly non-contiguous and overlapping colour subsets -- as the reference
// computes them on the host (deppart.cpp:15-101, Partition ctor
// partition.cpp:10-24).  The row / nonzero splits of partition.cu never
// materialise sets (their subsets are contiguous ranges); these entry points
// cover every other partition a plan or a user can build.
//
// A partition is (P, off[P+1], idx[off[P]]) in device memory: colour c's
// subset is idx[off[c] .. off[c+1]), sorted and unique, as Partition holds it.
// Outputs use the same layout; *total receives the output size and the index
// array is written only when it fits `cap` (call once with cap 0 to size it).
// *disjoint is Partition::disjoint(): no index in two colours.
//
//   image     P'[c] = U_{i in P[c]} [lo_i, hi_i]            deppart.cpp:15-31
//             item lengths -> exclusive scan -> expansion by a per-output
//             binary search over the item starts; colours whose expansion is
//             not already increasing (overlapping / unordered ranges) get a
//             segmented sort, then per-colour unique.
//   preimage  i in P'[c] iff [lo_i, hi_i] non-empty and meets P[c]
//             (lower_bound in the sorted subset, deppart.cpp:42-48): one
//             thread per (colour, i), flags, one ordered select.
//   by_bounds one box per colour enumerated row-major (deppart.cpp:55-91):
//             one thread per output index, unravel + linearise.
#include <cub/cub.cuh>

#include "common.cuh"

namespace spd {

namespace {

constexpr int kT = 256;

unsigned grid_of(spd_context* ctx, int64_t n) {
  int64_t g = ceil_div(n > 0 ? n : 1, kT);
  return (unsigned)std::min<int64_t>(g, (int64_t)ctx->num_sms * 16);
}

// First k in [0, n) with a[k] > v (n if none).
__device__ __forceinline__ int64_t upper_bound_dev(const int64_t* __restrict__ a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Partition input checks: every index in [0, extent), strictly increasing
// inside its colour.  err bit 1: outside, bit 2: not sorted/unique.
__global__ void k_check_partition(const int64_t* __restrict__ off, int64_t P, const int64_t* __restrict__ idx,
                                  int64_t extent, int* __restrict__ err) {
  const int64_t m = off[P];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = idx[k];
    if (v < 0 || v >= extent) atomicOr(err, 1);
    if (k > 0) {
      const int64_t c = upper_bound_dev(off, P + 1, k) - 1;  // colour of item k
      if (k > off[c] && v <= idx[k - 1]) atomicOr(err, 2);
    }
  }
}

// Range checks (Region::ranges, region.cpp:33-46): non-empty ranges inside
// [0, dest).  err bit 4.
__global__ void k_check_ranges(const int64_t* __restrict__ ranges, int64_t n, int64_t dest, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = ranges[2 * i], hi = ranges[2 * i + 1];
    if (lo <= hi && (lo < 0 || hi >= dest)) atomicOr(err, 4);
  }
}

__global__ void k_image_len(const int64_t* __restrict__ ranges, const int64_t* __restrict__ idx, int64_t m,
                            int64_t* __restrict__ len) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[k];
    const int64_t lo = ranges[2 * i], hi = ranges[2 * i + 1];
    len[k] = hi >= lo ? hi - lo + 1 : 0;
  }
}

// Expansion: output slot e belongs to item k = (last start <= e); its value
// is lo_k + (e - start_k).  Flags slots that break the increasing order
// inside their colour (seg = colour start slots).
__global__ void k_image_expand(const int64_t* __restrict__ ranges, const int64_t* __restrict__ idx, int64_t m,
                               const int64_t* __restrict__ start, int64_t L, const int64_t* __restrict__ seg,
                               int64_t P, int64_t* __restrict__ E, int* __restrict__ unsorted) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = upper_bound_dev(start, m, e) - 1;
    const int64_t i = idx[k];
    const int64_t v = ranges[2 * i] + (e - start[k]);
    E[e] = v;
    if (e > 0 && e != start[k]) continue;  // inside one range: increasing by construction
    if (e == 0) continue;
    // first slot of item k: compare with the last slot of the previous item
    // unless e starts a colour
    const int64_t c = upper_bound_dev(seg, P + 1, e) - 1;
    if (seg[c] == e) continue;
    const int64_t kp = upper_bound_dev(start, m, e - 1) - 1;
    const int64_t ip = idx[kp];
    const int64_t prev = ranges[2 * ip] + (e - 1 - start[kp]);
    if (v <= prev) atomicOr(unsorted, 1);
  }
}

// counts[c] += hit, aggregated over the lanes of a warp with the same colour.
__device__ __forceinline__ void count_hit(int64_t* counts, int64_t c, bool hit) {
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, (unsigned long long)c);
  const unsigned hits = __ballot_sync(act, hit) & peers;
  if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1) && hits)
    atomicAdd((unsigned long long*)(counts + c), (unsigned long long)__popc(hits));
}

// keep[e] = e starts its colour or E[e] != E[e-1]; per-colour kept counts.
__global__ void k_unique_flags(const int64_t* __restrict__ E, int64_t L, const int64_t* __restrict__ seg, int64_t P,
                               unsigned char* __restrict__ keep, int64_t* __restrict__ counts) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = upper_bound_dev(seg, P + 1, e) - 1;
    const bool k = seg[c] == e || E[e] != E[e - 1];
    keep[e] = k;
    count_hit(counts, c, k);
  }
}

// flags[c*n + i] for the preimage; per-colour counts.
__global__ void k_preimage_flags(const int64_t* __restrict__ ranges, int64_t n, const int64_t* __restrict__ off,
                                 const int64_t* __restrict__ idx, int64_t P, unsigned char* __restrict__ flags,
                                 int64_t* __restrict__ counts) {
  const int64_t total = n * P;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / n, i = t - c * n;
    const int64_t lo = ranges[2 * i], hi = ranges[2 * i + 1];
    bool hit = false;
    if (lo <= hi) {  // empty ranges are never coloured (deppart.cpp:46)
      const int64_t a = off[c], len = off[c + 1] - a;
      // lower_bound(lo) in the sorted subset, then test <= hi (deppart.cpp:47-48)
      int64_t l = 0, h = len;
      while (l < h) {
        const int64_t mid = (l + h) >> 1;
        if (idx[a + mid] < lo) l = mid + 1; else h = mid;
      }
      hit = l < len && idx[a + l] <= hi;
    }
    flags[t] = hit;
    count_hit(counts, c, hit);
  }
}

__global__ void k_gather_starts(const int64_t* __restrict__ start, const int64_t* __restrict__ off, int64_t P,
                                int64_t* __restrict__ seg) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= P; c += (int64_t)gridDim.x * blockDim.x)
    seg[c] = start[off[c]];
}

struct ModN {
  int64_t n;
  __host__ __device__ int64_t operator()(int64_t t) const { return t % n; }
};

// counts -> off (exclusive), off[P] = total.  P is small: one thread.
__global__ void k_counts_to_off(const int64_t* __restrict__ counts, int64_t P, int64_t* __restrict__ off) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t o = 0;
    for (int64_t c = 0; c < P; c++) off[c] = o, o += counts[c];
    off[P] = o;
  }
}

// Partition::disjoint: some index present in two colours.
__global__ void k_multiplicity(const int64_t* __restrict__ idx, int64_t m, int32_t* __restrict__ seen,
                               int* __restrict__ overlap) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    if (atomicAdd(seen + idx[k], 1) > 0) *overlap = 1;
}

// Row-major enumeration of colour boxes: box c covers lo[c*R + d] .. hi,
// its volume vol[c], output offset off[c].
__global__ void k_boxes(int R, const int64_t* __restrict__ ext, const int64_t* __restrict__ lo,
                        const int64_t* __restrict__ hi, const int64_t* __restrict__ off, int64_t P,
                        int64_t* __restrict__ out) {
  const int64_t total = off[P];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = upper_bound_dev(off, P + 1, e) - 1;
    int64_t r = e - off[c], lin = 0, stride = 1;
    for (int d = R - 1; d >= 0; d--) {
      const int64_t w = hi[c * R + d] - lo[c * R + d] + 1;
      const int64_t q = r % w;
      r /= w;
      lin += (lo[c * R + d] + q) * stride;
      stride *= ext[d];
    }
    out[e] = lin;
  }
}

struct Scratch {
  spd_context* ctx;
  std::vector<void*> ptrs;
  explicit Scratch(spd_context* c) : ctx(c) {}
  template <class T>
  T* get(int64_t n) {
    void* p = dev_alloc(ctx, sizeof(T) * (size_t)std::max<int64_t>(n, 1));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~Scratch() {
    for (void* p : ptrs) dev_free(ctx, p);
  }
};

int read_err(spd_context* ctx, int* err_d) {
  int e = 0;
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 13, err_d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(&e, ctx->pinned_counters + 13, sizeof(int));
  return e;
}

std::vector<int64_t> host_off(spd_context* ctx, const int64_t* off, int64_t P) {
  std::vector<int64_t> h(P + 1);
  SPD_CUDA(cudaMemcpyAsync(h.data(), off, sizeof(int64_t) * (P + 1), cudaMemcpyDeviceToHost, ctx->stream));
  SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h[0] != 0) throw ValidationError("partition: off[0] must be 0");
  for (int64_t c = 0; c < P; c++)
    if (h[c + 1] < h[c]) throw ValidationError("partition: off must be non-decreasing");
  return h;
}

void check_partition(spd_context* ctx, const int64_t* off, int64_t P, const int64_t* idx, int64_t extent,
                     int* err_d, const char* what) {
  SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), ctx->stream));
  k_check_partition<<<grid_of(ctx, 1 << 20), kT, 0, ctx->stream>>>(off, P, idx, extent, err_d);
  SPD_CHECK_LAUNCH();
  const int e = read_err(ctx, err_d);
  if (e & 1) throw ValidationError(std::string(what) + ": Partition: subset index outside parent space");
  if (e & 2) throw ValidationError(std::string(what) + ": partition subsets must be sorted and unique");
}

void check_ranges(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest, int* err_d) {
  SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), ctx->stream));
  k_check_ranges<<<grid_of(ctx, n), kT, 0, ctx->stream>>>(ranges, n, dest, err_d);
  SPD_CHECK_LAUNCH();
  if (read_err(ctx, err_d) & 4) throw ValidationError("Region: range outside destination region");
}

// Writes off (device, P+1) from counts, the total, and disjointness.
int64_t finish(spd_context* ctx, Scratch& S, const int64_t* counts, int64_t P, int64_t* out_off,
               const int64_t* idx_for_disjoint, int64_t extent, int* disjoint, bool have_idx, int* err_d) {
  cudaStream_t s = ctx->stream;
  k_counts_to_off<<<1, 32, 0, s>>>(counts, P, out_off);
  SPD_CHECK_LAUNCH();
  int64_t total = 0;
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 14, out_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  total = ctx->pinned_counters[14];
  if (disjoint && have_idx) {
    int32_t* seen = S.get<int32_t>(extent);
    SPD_CUDA(cudaMemsetAsync(seen, 0, sizeof(int32_t) * std::max<int64_t>(extent, 1), s));
    SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), s));
    k_multiplicity<<<grid_of(ctx, total), kT, 0, s>>>(idx_for_disjoint, total, seen, err_d);
    SPD_CHECK_LAUNCH();
    *disjoint = read_err(ctx, err_d) ? 0 : 1;
  } else if (disjoint) {
    *disjoint = -1;  // not computed: no index array written
  }
  return total;
}

void run_image(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest, int64_t P, const int64_t* off,
               const int64_t* idx, int64_t* out_off, int64_t* out_idx, int64_t cap, int64_t* total_out,
               int* disjoint) {
  checked(ctx);
  if (n < 0 || dest < 0 || P < 0) throw ValidationError("image: negative size");
  if (!out_off || !total_out) throw ValidationError("image: null output");
  if ((n > 0 && !ranges) || !off) throw ValidationError("image: null input");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  Scratch S(ctx);
  int* err_d = S.get<int>(1);
  check_ranges(ctx, ranges, n, dest, err_d);
  const std::vector<int64_t> hoff = host_off(ctx, off, P);
  const int64_t m = hoff[P];
  if (m > 0 && !idx) throw ValidationError("image: null input");
  if (m > 0) check_partition(ctx, off, P, idx, n, err_d, "image");
  // item lengths -> starts
  int64_t* len = S.get<int64_t>(m + 1);
  int64_t* start = S.get<int64_t>(m + 1);
  SPD_CUDA(cudaMemsetAsync(len + m, 0, sizeof(int64_t), s));
  if (m > 0) {
    k_image_len<<<grid_of(ctx, m), kT, 0, s>>>(ranges, idx, m, len);
    SPD_CHECK_LAUNCH();
  }
  size_t tb = 0;
  SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len, start, m + 1, s));
  void* tmp = S.get<char>((int64_t)tb);
  SPD_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, len, start, m + 1, s));
  // colour segment starts in the expansion: seg[c] = start[off[c]]
  int64_t* seg = S.get<int64_t>(P + 1);
  k_gather_starts<<<grid_of(ctx, P + 1), kT, 0, s>>>(start, off, P, seg);
  SPD_CHECK_LAUNCH();
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 15, seg + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  const int64_t L = ctx->pinned_counters[15];
  if (L >= (int64_t(1) << 31)) throw ValidationError("image: more than 2^31 expanded indices");
  int64_t* E = S.get<int64_t>(L);
  SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), s));
  if (L > 0) {
    k_image_expand<<<grid_of(ctx, L), kT, 0, s>>>(ranges, idx, m, start, L, seg, P, E, err_d);
    SPD_CHECK_LAUNCH();
  }
  if (read_err(ctx, err_d)) {  // overlapping / unordered ranges: sort each colour
    int64_t* E2 = S.get<int64_t>(L);
    size_t sb = 0;
    SPD_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, sb, E, E2, (int)L, (int)P, seg, seg + 1, s));
    void* st = S.get<char>((int64_t)sb);
    SPD_CUDA(cub::DeviceSegmentedSort::SortKeys(st, sb, E, E2, (int)L, (int)P, seg, seg + 1, s));
    E = E2;
  }
  unsigned char* keep = S.get<unsigned char>(L);
  int64_t* counts = S.get<int64_t>(P);
  SPD_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * std::max<int64_t>(P, 1), s));
  if (L > 0) {
    k_unique_flags<<<grid_of(ctx, L), kT, 0, s>>>(E, L, seg, P, keep, counts);
    SPD_CHECK_LAUNCH();
  }
  k_counts_to_off<<<1, 32, 0, s>>>(counts, P, out_off);
  SPD_CHECK_LAUNCH();
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 14, out_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  const int64_t total = ctx->pinned_counters[14];
  *total_out = total;
  const bool write = out_idx && cap >= total;
  if (write && L > 0) {
    int64_t* nsel = S.get<int64_t>(1);
    size_t fb = 0;
    SPD_CUDA(cub::DeviceSelect::Flagged(nullptr, fb, E, keep, out_idx, nsel, L, s));
    void* ft = S.get<char>((int64_t)fb);
    SPD_CUDA(cub::DeviceSelect::Flagged(ft, fb, E, keep, out_idx, nsel, L, s));
  }
  finish(ctx, S, counts, P, out_off, out_idx, dest, disjoint, write, err_d);
  ctx->launches += 6;
}

void run_preimage(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest, int64_t P, const int64_t* off,
                  const int64_t* idx, int64_t* out_off, int64_t* out_idx, int64_t cap, int64_t* total_out,
                  int* disjoint) {
  checked(ctx);
  if (n < 0 || dest < 0 || P < 0) throw ValidationError("preimage: negative size");
  if (!out_off || !total_out) throw ValidationError("preimage: null output");
  if ((n > 0 && !ranges) || !off) throw ValidationError("preimage: null input");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  Scratch S(ctx);
  int* err_d = S.get<int>(1);
  check_ranges(ctx, ranges, n, dest, err_d);
  const std::vector<int64_t> hoff = host_off(ctx, off, P);
  if (hoff[P] > 0 && !idx) throw ValidationError("preimage: null input");
  if (hoff[P] > 0) check_partition(ctx, off, P, idx, dest, err_d, "preimage");
  const int64_t tot = n * P;
  unsigned char* flags = S.get<unsigned char>(tot);
  int64_t* counts = S.get<int64_t>(P);
  SPD_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * std::max<int64_t>(P, 1), s));
  if (tot > 0) {
    k_preimage_flags<<<grid_of(ctx, tot), kT, 0, s>>>(ranges, n, off, idx, P, flags, counts);
    SPD_CHECK_LAUNCH();
  }
  k_counts_to_off<<<1, 32, 0, s>>>(counts, P, out_off);
  SPD_CHECK_LAUNCH();
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 14, out_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  const int64_t total = ctx->pinned_counters[14];
  *total_out = total;
  const bool write = out_idx && cap >= total;
  if (write && tot > 0) {
    cub::CountingInputIterator<int64_t> cnt(0);
    cub::TransformInputIterator<int64_t, ModN, cub::CountingInputIterator<int64_t>> it(cnt, ModN{n});
    int64_t* nsel = S.get<int64_t>(1);
    size_t fb = 0;
    SPD_CUDA(cub::DeviceSelect::Flagged(nullptr, fb, it, flags, out_idx, nsel, tot, s));
    void* ft = S.get<char>((int64_t)fb);
    SPD_CUDA(cub::DeviceSelect::Flagged(ft, fb, it, flags, out_idx, nsel, tot, s));
  }
  finish(ctx, S, counts, P, out_off, out_idx, n, disjoint, write, err_d);
  ctx->launches += 4;
}

void run_by_bounds(spd_context* ctx, int R, const int64_t* extents, int64_t P, const int64_t* bounds,
                   int64_t* out_off, int64_t* out_idx, int64_t cap, int64_t* total_out, int* disjoint) {
  checked(ctx);
  if (R < 1 || P < 0 || !extents || (P > 0 && !bounds) || !out_off || !total_out)
    throw ValidationError("partition_by_bounds: bad arguments");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  Scratch S(ctx);
  int64_t space = 1;
  for (int d = 0; d < R; d++) {
    if (extents[d] < 0) throw ValidationError("partition_by_bounds: negative extent");
    space *= extents[d];
  }
  // host: validate boxes (deppart.cpp:64-75), volumes, offsets
  std::vector<int64_t> lo(std::max<int64_t>(P * R, 1)), hi(std::max<int64_t>(P * R, 1)), hoff(P + 1, 0);
  for (int64_t c = 0; c < P; c++) {
    bool empty = false;
    int64_t vol = 1;
    for (int d = 0; d < R; d++) {
      const int64_t a = bounds[(c * R + d) * 2], b = bounds[(c * R + d) * 2 + 1];
      lo[c * R + d] = a;
      hi[c * R + d] = b;
      if (a > b) {
        empty = true;
        continue;
      }
      if (a < 0 || b >= extents[d]) throw ValidationError("partition_by_bounds: bound outside space");
      vol *= b - a + 1;
    }
    hoff[c + 1] = hoff[c] + (empty ? 0 : vol);
  }
  const int64_t total = hoff[P];
  *total_out = total;
  SPD_CUDA(cudaMemcpyAsync(out_off, hoff.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, s));
  const bool write = out_idx && cap >= total;
  if (write && total > 0) {
    int64_t* dext = S.get<int64_t>(R);
    int64_t* dlo = S.get<int64_t>(P * R);
    int64_t* dhi = S.get<int64_t>(P * R);
    SPD_CUDA(cudaMemcpyAsync(dext, extents, sizeof(int64_t) * R, cudaMemcpyHostToDevice, s));
    SPD_CUDA(cudaMemcpyAsync(dlo, lo.data(), sizeof(int64_t) * P * R, cudaMemcpyHostToDevice, s));
    SPD_CUDA(cudaMemcpyAsync(dhi, hi.data(), sizeof(int64_t) * P * R, cudaMemcpyHostToDevice, s));
    k_boxes<<<grid_of(ctx, total), kT, 0, s>>>(R, dext, dlo, dhi, out_off, P, out_idx);
    SPD_CHECK_LAUNCH();
  }
  if (disjoint) {
    if (write) {
      int* err_d = S.get<int>(1);
      int32_t* seen = S.get<int32_t>(space);
      SPD_CUDA(cudaMemsetAsync(seen, 0, sizeof(int32_t) * std::max<int64_t>(space, 1), s));
      SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), s));
      k_multiplicity<<<grid_of(ctx, total), kT, 0, s>>>(out_idx, total, seen, err_d);
      SPD_CHECK_LAUNCH();
      *disjoint = read_err(ctx, err_d) ? 0 : 1;
    } else {
      *disjoint = -1;
    }
  }
  SPD_CUDA(cudaStreamSynchronize(s));
  ctx->launches += 2;
}

}  // namespace

}  // namespace spd

using namespace spd;

extern "C" int spd_deppart_image(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                                 int64_t pieces, const int64_t* off, const int64_t* idx, int64_t* out_off,
                                 int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint) {
  return guarded([&] {
    run_image(ctx, ranges, n, dest_extent, pieces, off, idx, out_off, out_idx, cap, total, disjoint);
  });
}

extern "C" int spd_deppart_preimage(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                                    int64_t pieces, const int64_t* off, const int64_t* idx, int64_t* out_off,
                                    int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint) {
  return guarded([&] {
    run_preimage(ctx, ranges, n, dest_extent, pieces, off, idx, out_off, out_idx, cap, total, disjoint);
  });
}

extern "C" int spd_deppart_by_bounds(spd_context* ctx, int rank, const int64_t* extents, int64_t pieces,
                                     const int64_t* bounds, int64_t* out_off, int64_t* out_idx, int64_t cap,
                                     int64_t* total, int* disjoint) {
  return guarded([&] { run_by_bounds(ctx, rank, extents, pieces, bounds, out_off, out_idx, cap, total, disjoint); });
}

// Host-memory variants for host callers (the reference's own planner through
// integration/deppart_gpu.cpp): inputs are staged to the device once, the
// operator runs twice (size, then fill) on the device, the result comes
// back into the caller's arrays.  cap < total: only out_off and *total.
namespace {
template <class Run>
void host_call(spd_context* ctx, int64_t n_ranges, const int64_t* ranges, int64_t P, const int64_t* off,
               const int64_t* idx, int64_t* out_off, int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint,
               Run run) {
  checked(ctx);
  if (P < 0 || n_ranges < 0) throw ValidationError("deppart: negative size");
  if (!out_off || !total || (P > 0 && !off) || (n_ranges > 0 && !ranges)) throw ValidationError("deppart: null argument");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  const int64_t m = P > 0 ? off[P] : 0;
  if (m > 0 && !idx) throw ValidationError("deppart: null argument");
  int64_t* d_r = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * std::max<int64_t>(2 * n_ranges, 1));
  int64_t* d_off = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (P + 1));
  int64_t* d_idx = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * std::max<int64_t>(m, 1));
  int64_t* d_out_off = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (P + 1));
  int64_t* d_out_idx = nullptr;
  auto release = [&] {
    for (void* q : {(void*)d_r, (void*)d_off, (void*)d_idx, (void*)d_out_off, (void*)d_out_idx}) dev_free(ctx, q);
  };
  try {
    if (n_ranges > 0) SPD_CUDA(cudaMemcpyAsync(d_r, ranges, sizeof(int64_t) * 2 * n_ranges, cudaMemcpyHostToDevice, s));
    if (P >= 0) SPD_CUDA(cudaMemcpyAsync(d_off, off, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, s));
    if (m > 0) SPD_CUDA(cudaMemcpyAsync(d_idx, idx, sizeof(int64_t) * m, cudaMemcpyHostToDevice, s));
    int64_t t = 0;
    run(d_r, d_off, d_idx, d_out_off, (int64_t*)nullptr, (int64_t)0, &t, (int*)nullptr);
    *total = t;
    if (out_idx && cap >= t) {
      d_out_idx = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * std::max<int64_t>(t, 1));
      run(d_r, d_off, d_idx, d_out_off, d_out_idx, t, &t, disjoint);
      if (t > 0) SPD_CUDA(cudaMemcpyAsync(out_idx, d_out_idx, sizeof(int64_t) * t, cudaMemcpyDeviceToHost, s));
    } else if (disjoint) {
      *disjoint = -1;
    }
    SPD_CUDA(cudaMemcpyAsync(out_off, d_out_off, sizeof(int64_t) * (P + 1), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    release();
    throw;
  }
  release();
}
}  // namespace

extern "C" int spd_deppart_image_host(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                                      int64_t pieces, const int64_t* off, const int64_t* idx, int64_t* out_off,
                                      int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint) {
  return guarded([&] {
    host_call(ctx, n, ranges, pieces, off, idx, out_off, out_idx, cap, total, disjoint,
              [&](const int64_t* r, const int64_t* o, const int64_t* x, int64_t* oo, int64_t* oi, int64_t c,
                  int64_t* t, int* d) { run_image(ctx, r, n, dest_extent, pieces, o, x, oo, oi, c, t, d); });
  });
}

extern "C" int spd_deppart_preimage_host(spd_context* ctx, const int64_t* ranges, int64_t n, int64_t dest_extent,
                                         int64_t pieces, const int64_t* off, const int64_t* idx, int64_t* out_off,
                                         int64_t* out_idx, int64_t cap, int64_t* total, int* disjoint) {
  return guarded([&] {
    host_call(ctx, n, ranges, pieces, off, idx, out_off, out_idx, cap, total, disjoint,
              [&](const int64_t* r, const int64_t* o, const int64_t* x, int64_t* oo, int64_t* oi, int64_t c,
                  int64_t* t, int* d) { run_preimage(ctx, r, n, dest_extent, pieces, o, x, oo, oi, c, t, d); });
  });
}

extern "C" int spd_deppart_by_bounds_host(spd_context* ctx, int rank, const int64_t* extents, int64_t pieces,
                                          const int64_t* bounds, int64_t* out_off, int64_t* out_idx, int64_t cap,
                                          int64_t* total, int* disjoint) {
  return guarded([&] {
    checked(ctx);
    if (pieces < 0 || !out_off || !total) throw ValidationError("partition_by_bounds: bad arguments");
    activate(ctx);
    cudaStream_t s = ctx->stream;
    int64_t* d_off = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (pieces + 1));
    int64_t* d_idx = nullptr;
    try {
      int64_t t = 0;
      run_by_bounds(ctx, rank, extents, pieces, bounds, d_off, nullptr, 0, &t, nullptr);
      *total = t;
      if (out_idx && cap >= t) {
        d_idx = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * std::max<int64_t>(t, 1));
        run_by_bounds(ctx, rank, extents, pieces, bounds, d_off, d_idx, t, &t, disjoint);
        if (t > 0) SPD_CUDA(cudaMemcpyAsync(out_idx, d_idx, sizeof(int64_t) * t, cudaMemcpyDeviceToHost, s));
      } else if (disjoint) {
        *disjoint = -1;
      }
      SPD_CUDA(cudaMemcpyAsync(out_off, d_off, sizeof(int64_t) * (pieces + 1), cudaMemcpyDeviceToHost, s));
      SPD_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      dev_free(ctx, d_off);
      dev_free(ctx, d_idx);
      throw;
    }
    dev_free(ctx, d_off);
    dev_free(ctx, d_idx);
  });
}
