// SpAdd3 leaf + two-phase assembly (K8): A = B + C + D over CSR operands.
//
// Reference: a coordinate-value loop over rows, the union of the three
// sorted crd lists per row (iterate_coords + union_merge, sim.cpp:46-66,
// 389-454), value ((0.0 + B) + C) + D over the present terms in term order
// (accumulate, sim.cpp:326-354), then two-phase assembly: a symbolic count
// sizes pos/crd exactly and a fill pass writes them (sim.cpp:676-788).
//
// B200 design -- rows binned by their total input length L = |B_i|+|C_i|+|D_i|:
//   short rows (L <= T, almost every row of a power-law matrix): one thread
//           per row runs the sequential three-way merge, once to count and
//           once to fill; consecutive threads own consecutive rows so the
//           warp's loads stay within a few sectors;
//   long rows (the hubs): one CTA per row, element-parallel rank-based union:
//           C's elements absent from B's row and D's absent from B's and C's
//           rows are flagged by binary search, block-scanned into row-local
//           prefixes, and every element first in term order computes its rank
//           in the union from searches + prefix lookups (no serial merge).
//   count -> exclusive scan (cub) -> exact allocation -> fill is the
//   reference's two-phase assembly.  With a communicator each GPU builds its
//   row block; the per-GPU nnz are all-gathered over NCCL to give global pos
//   offsets (spd_tensor_global_span) and spd_gather_rows collects the pieces
//   on one GPU with grouped NCCL send/recv.
// The pattern is the structural union (explicit zeros kept, P6), crd sorted,
// empties canonical -- bit-exact with the reference; values are exact because
// each output sums the same terms in the same order.
#include <cub/cub.cuh>
#include <cuda/std/limits>

#include "common.cuh"

namespace spd {

constexpr int kSaBlock = 256;
constexpr int64_t kTile = 1024;  // merge tile: positions of a row's longest operand
constexpr int64_t kNone = INT64_MAX;

// lower_bound of x in a[lo, hi): first index with a[idx] >= x.
__device__ __forceinline__ int64_t lb(const int64_t* __restrict__ a, int64_t lo, int64_t hi,
                                      int64_t x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct Csr {
  const int64_t* rp;
  const int64_t* crd;
  const double* vals;
};

struct Row3 {
  int64_t b0, b1, c0, c1, d0, d1;
};

__device__ __forceinline__ Row3 row3(const Csr& B, const Csr& C, const Csr& D, int64_t i) {
  return {__ldg(B.rp + i), __ldg(B.rp + i + 1), __ldg(C.rp + i), __ldg(C.rp + i + 1),
          __ldg(D.rp + i), __ldg(D.rp + i + 1)};
}

__device__ __forceinline__ int64_t head(const int64_t* __restrict__ crd, int64_t p, int64_t e) {
  return p < e ? __ldg(crd + p) : kNone;
}

// Short rows: sequential three-way merge (the union_merge of sim.cpp:46-66
// over three sorted lists).  Long rows are appended to `longrows`.
// Appends `row` to list[*n] for the lanes with `take`, one atomic per warp.
__device__ __forceinline__ void warp_append(bool take, int64_t row, int32_t* __restrict__ list,
                                            int32_t* __restrict__ n) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, take);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane_id() == leader) base = atomicAdd(n, __popc(m));
  base = __shfl_sync(act, base, leader);
  if (take) list[base + __popc(m & ((1u << lane_id()) - 1u))] = (int32_t)row;
}

__global__ void __launch_bounds__(kSaBlock) k_sa_count(Csr B, Csr C, Csr D, int64_t lo, int64_t hi,
                                                       int64_t T, int64_t* __restrict__ cnt,
                                                       int32_t* __restrict__ midrows,
                                                       int32_t* __restrict__ hubrows,
                                                       int32_t* __restrict__ nlists) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Row3 r = row3(B, C, D, i);
    const int64_t L = (r.b1 - r.b0) + (r.c1 - r.c0) + (r.d1 - r.d0);
    const int64_t mx = max(r.b1 - r.b0, max(r.c1 - r.c0, r.d1 - r.d0));
    warp_append(L > T && mx <= kTile, i, midrows, nlists);
    warp_append(L > T && mx > kTile, i, hubrows, nlists + 1);
    if (L > T) continue;
    int64_t pb = r.b0, pc = r.c0, pd = r.d0;
    int64_t xb = head(B.crd, pb, r.b1), xc = head(C.crd, pc, r.c1), xd = head(D.crd, pd, r.d1);
    int64_t n = 0;
    while (true) {
      const int64_t x = min(xb, min(xc, xd));
      if (x == kNone) break;
      n++;
      if (xb == x) xb = head(B.crd, ++pb, r.b1);
      if (xc == x) xc = head(C.crd, ++pc, r.c1);
      if (xd == x) xd = head(D.crd, ++pd, r.d1);
    }
    cnt[i] = n;
  }
}

__global__ void __launch_bounds__(kSaBlock) k_sa_fill(Csr B, Csr C, Csr D, int64_t lo, int64_t hi,
                                                      int64_t T, const int64_t* __restrict__ rpA,
                                                      int64_t* __restrict__ Acrd,
                                                      double* __restrict__ Avals) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Row3 r = row3(B, C, D, i);
    const int64_t L = (r.b1 - r.b0) + (r.c1 - r.c0) + (r.d1 - r.d0);
    if (L > T || L == 0) continue;
    int64_t o = __ldg(rpA + i);
    int64_t pb = r.b0, pc = r.c0, pd = r.d0;
    int64_t xb = head(B.crd, pb, r.b1), xc = head(C.crd, pc, r.c1), xd = head(D.crd, pd, r.d1);
    while (true) {
      const int64_t x = min(xb, min(xc, xd));
      if (x == kNone) break;
      // accumulate (sim.cpp:326-354): 0.0, then the present terms in order
      double v = 0.0;
      if (xb == x) { v += __ldg(B.vals + pb); xb = head(B.crd, ++pb, r.b1); }
      if (xc == x) { v += __ldg(C.vals + pc); xc = head(C.crd, ++pc, r.c1); }
      if (xd == x) { v += __ldg(D.vals + pd); xd = head(D.crd, ++pd, r.d1); }
      Acrd[o] = x;
      Avals[o] = 0.0 + v;
      o++;
    }
  }
}

// ---------------------------------------------------------------------------
// Rows above the thread-merge threshold: warp-cooperative three-way merge.
// A row is cut into tiles of about kTile positions of its longest operand
// (value splitters taken from that operand, the other operands' tile starts
// found by warp binary search).  A warp merges a tile in steps: it holds a
// 32-entry window of each operand in registers, takes xmax = the smallest of
// the three windows' last entries -- every entry <= xmax of every operand is
// then inside its window -- and resolves all of them at once: membership
// flags and ranks come from 5-step shuffle searches between the windows and
// popcounts of the "first in term order" ballots, so each step emits up to
// 96 union entries with coalesced loads and no global searches.  Pass 0
// counts (and records the tile starts), pass 1 writes crd and values.

// First index in a[lo, hi) with a[idx] >= x (warp-cooperative 32-ary search;
// full converged warp, same x on every lane).
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t* __restrict__ a, int64_t lo,
                                                    int64_t hi, int64_t x) {
  const int lane = lane_id();
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + lane * step;
    const bool below = idx < hi && __ldg(a + idx) < x;
    const int cnt = __popc(__ballot_sync(0xffffffffu, below));
    if (cnt == 0) return lo;
    const int64_t nlo = lo + (int64_t)(cnt - 1) * step + 1;
    const int64_t nhi = lo + (int64_t)cnt * step;
    hi = nhi < hi ? nhi : hi;
    lo = nlo;
  }
  const int64_t idx = lo + lane;
  const bool below = idx < hi && __ldg(a + idx) < x;
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// Number of window entries (sorted across lanes, invalid = max) below x, and
// whether x itself is present.  Every lane calls it (shuffles are warp-wide).
template <typename KEY>
__device__ __forceinline__ int win_below(KEY w, KEY x, bool& eq) {
  int c = 0;
#pragma unroll
  for (int st = 16; st >= 1; st >>= 1)
    if (__shfl_sync(0xffffffffu, w, c + st - 1) < x) c += st;
  const KEY w31 = __shfl_sync(0xffffffffu, w, 31);
  if (c == 31 && w31 < x) c = 32;
  const KEY wc = __shfl_sync(0xffffffffu, w, c & 31);
  eq = c < 32 && wc == x;
  return c;
}

__device__ __forceinline__ unsigned below_mask(int k) { return k >= 32 ? 0xffffffffu : (1u << k) - 1u; }

template <typename KEY>
__device__ __forceinline__ KEY win_load(const int64_t* __restrict__ crd, int64_t p, int64_t e) {
  return p < e ? (KEY)__ldg(crd + p) : cuda::std::numeric_limits<KEY>::max();
}

__global__ void k_sa_tiles(Csr B, Csr C, Csr D, const int32_t* __restrict__ longrows, int64_t nl,
                           int64_t* __restrict__ tilecnt) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nl;
       li += (int64_t)gridDim.x * blockDim.x) {
    const Row3 r = row3(B, C, D, longrows[li]);
    const int64_t mx = max(r.b1 - r.b0, max(r.c1 - r.c0, r.d1 - r.d0));
    tilecnt[li] = max((int64_t)1, ceil_div(mx, kTile));
  }
}

template <typename KEY, int MODE>
__device__ __forceinline__ int64_t merge_steps(const Csr& B, const Csr& C, const Csr& D, int64_t pb,
                                               int64_t eb, int64_t pc, int64_t ec, int64_t pd,
                                               int64_t ed, int64_t out, int64_t* __restrict__ Acrd,
                                               double* __restrict__ Avals) {
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  while (pb < eb || pc < ec || pd < ed) {
    const KEY wb = win_load<KEY>(B.crd, pb + lane, eb);
    const KEY wc = win_load<KEY>(C.crd, pc + lane, ec);
    const KEY wd = win_load<KEY>(D.crd, pd + lane, ed);
    double vb = 0.0, vc = 0.0, vd = 0.0;
    if (MODE == 1) {
      if (pb + lane < eb) vb = __ldg(B.vals + pb + lane);
      if (pc + lane < ec) vc = __ldg(C.vals + pc + lane);
      if (pd + lane < ed) vd = __ldg(D.vals + pd + lane);
    }
    const KEY xmax = min(__shfl_sync(0xffffffffu, wb, 31),
                         min(__shfl_sync(0xffffffffu, wc, 31), __shfl_sync(0xffffffffu, wd, 31)));
    const int nB = __popc(__ballot_sync(0xffffffffu, pb + lane < eb && wb <= xmax));
    const int nC = __popc(__ballot_sync(0xffffffffu, pc + lane < ec && wc <= xmax));
    const int nD = __popc(__ballot_sync(0xffffffffu, pd + lane < ed && wd <= xmax));
    // C entries present in B; D entries present in B or C
    bool cInB, dInB, dInC;
    const int kBc = win_below(wb, wc, cInB);
    const int kBd = win_below(wb, wd, dInB);
    const int kCd = win_below(wc, wd, dInC);
    const bool fc = lane < nC && !cInB;
    const bool fd = lane < nD && !dInB && !dInC;
    const unsigned mC = __ballot_sync(0xffffffffu, fc);
    const unsigned mD = __ballot_sync(0xffffffffu, fd);
    if (MODE == 1) {
      bool bInC, bInD, cInD;
      const int kCb = win_below(wc, wb, bInC);
      const int kDb = win_below(wd, wb, bInD);
      const int kDc = win_below(wd, wc, cInD);
      const double vcb = __shfl_sync(0xffffffffu, vc, kCb & 31);
      const double vdb = __shfl_sync(0xffffffffu, vd, kDb & 31);
      const double vdc = __shfl_sync(0xffffffffu, vd, kDc & 31);
      if (lane < nB) {  // accumulate (sim.cpp:326-354): 0.0, then terms in order
        const int64_t o = out + lane + __popc(mC & below_mask(kCb)) + __popc(mD & below_mask(kDb));
        double v = 0.0;
        v += vb;
        if (bInC) v += vcb;
        if (bInD) v += vdb;
        Acrd[o] = (int64_t)wb;
        Avals[o] = 0.0 + v;
      }
      if (fc) {
        const int64_t o = out + kBc + __popc(mC & lt) + __popc(mD & below_mask(kDc));
        double v = 0.0;
        v += vc;
        if (cInD) v += vdc;
        Acrd[o] = (int64_t)wc;
        Avals[o] = 0.0 + v;
      }
      if (fd) {
        const int64_t o = out + kBd + __popc(mC & below_mask(kCd)) + __popc(mD & lt);
        double v = 0.0;
        v += vd;
        Acrd[o] = (int64_t)wd;
        Avals[o] = 0.0 + v;
      }
    }
    out += nB + __popc(mC) + __popc(mD);
    pb += nB, pc += nC, pd += nD;
  }
  return out;
}

template <typename KEY, int MODE>
__global__ void __launch_bounds__(kSaBlock) k_sa_merge(Csr B, Csr C, Csr D,
                                                       const int32_t* __restrict__ longrows, int64_t nl,
                                                       const int64_t* __restrict__ tileof,
                                                       int64_t* __restrict__ tstart,
                                                       int64_t* __restrict__ tcount,
                                                       const int64_t* __restrict__ toff,
                                                       const int64_t* __restrict__ rpA,
                                                       int64_t* __restrict__ Acrd,
                                                       double* __restrict__ Avals) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = tileof[nl];
  for (int64_t t = gw; t < total; t += nw) {
    const int64_t li = warp_lower_bound(tileof, 0, nl + 1, t + 1) - 1;
    const int64_t i = longrows[li];
    const Row3 r = row3(B, C, D, i);
    const int64_t j = t - tileof[li], nt = tileof[li + 1] - tileof[li];
    int64_t pb, pc, pd, eb = r.b1, ec = r.c1, ed = r.d1;
    if (MODE == 0) {
      pb = r.b0, pc = r.c0, pd = r.d0;
      if (nt > 1) {  // value splitters from the longest operand
        const int64_t lb_ = r.b1 - r.b0, lc = r.c1 - r.c0, ld = r.d1 - r.d0;
        const int64_t* X = lb_ >= lc && lb_ >= ld ? B.crd : (lc >= ld ? C.crd : D.crd);
        const int64_t x0 = lb_ >= lc && lb_ >= ld ? r.b0 : (lc >= ld ? r.c0 : r.d0);
        if (j > 0) {
          const int64_t v = __ldg(X + x0 + j * kTile);
          pb = warp_lower_bound(B.crd, r.b0, r.b1, v);
          pc = warp_lower_bound(C.crd, r.c0, r.c1, v);
          pd = warp_lower_bound(D.crd, r.d0, r.d1, v);
        }
        if (j + 1 < nt) {
          const int64_t v = __ldg(X + x0 + (j + 1) * kTile);
          eb = warp_lower_bound(B.crd, pb, r.b1, v);
          ec = warp_lower_bound(C.crd, pc, r.c1, v);
          ed = warp_lower_bound(D.crd, pd, r.d1, v);
        }
      }
      if (lane == 0) tstart[3 * t] = pb, tstart[3 * t + 1] = pc, tstart[3 * t + 2] = pd;
    } else {
      pb = tstart[3 * t], pc = tstart[3 * t + 1], pd = tstart[3 * t + 2];
      if (j + 1 < nt) eb = tstart[3 * t + 3], ec = tstart[3 * t + 4], ed = tstart[3 * t + 5];
    }
    int64_t out = MODE == 1 ? __ldg(rpA + i) + (toff[t] - toff[tileof[li]]) : 0;
    out = merge_steps<KEY, MODE>(B, C, D, pb, eb, pc, ec, pd, ed, out, Acrd, Avals);
    if (MODE == 0 && lane == 0) tcount[t] = out;
  }
}

// Rows whose operands all fit one tile: one warp per row, no tile search.
template <typename KEY, int MODE>
__global__ void __launch_bounds__(kSaBlock) k_sa_mid(Csr B, Csr C, Csr D,
                                                     const int32_t* __restrict__ rows, int64_t nr,
                                                     int64_t* __restrict__ cnt,
                                                     const int64_t* __restrict__ rpA,
                                                     int64_t* __restrict__ Acrd,
                                                     double* __restrict__ Avals,
                                                     unsigned long long* __restrict__ ticket) {
  // batches of kMidBatch rows handed out by an atomic ticket: row lengths
  // vary by two orders of magnitude, a static stride leaves a long tail
  constexpr int64_t kMidBatch = 8;
  const int lane = lane_id();
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    const int64_t w0 = (int64_t)__shfl_sync(0xffffffffu, t, 0) * kMidBatch;
    if (w0 >= nr) break;
    // the batch's row extents (and output offsets) loaded together, lane b
    // holding row w0 + b's: one dependent round trip per batch, not per row
    // (C5 fill window 4.87 -> 4.74 ms; also prefetching the next batch's
    // extents measured no better)
    const int64_t nb = min(nr - w0, kMidBatch);
    int64_t i_l = 0, o_l = 0;
    Row3 r_l{0, 0, 0, 0, 0, 0};
    if (lane < nb) {
      i_l = rows[w0 + lane];
      r_l = row3(B, C, D, i_l);
      if (MODE == 1) o_l = __ldg(rpA + i_l);
    }
    for (int b = 0; b < nb; b++) {
      const int64_t i = __shfl_sync(0xffffffffu, i_l, b);
      const int64_t b0 = __shfl_sync(0xffffffffu, r_l.b0, b), b1 = __shfl_sync(0xffffffffu, r_l.b1, b);
      const int64_t c0 = __shfl_sync(0xffffffffu, r_l.c0, b), c1 = __shfl_sync(0xffffffffu, r_l.c1, b);
      const int64_t d0 = __shfl_sync(0xffffffffu, r_l.d0, b), d1 = __shfl_sync(0xffffffffu, r_l.d1, b);
      const int64_t out0 = MODE == 1 ? __shfl_sync(0xffffffffu, o_l, b) : 0;
      const int64_t out = merge_steps<KEY, MODE>(B, C, D, b0, b1, c0, c1, d0, d1, out0, Acrd, Avals);
      if (MODE == 0 && lane == 0) cnt[i] = out;
    }
  }
}

// Union size of every merged row: the sum of its tiles' counts.
__global__ void k_sa_cnt_long(const int32_t* __restrict__ longrows, int64_t nl,
                              const int64_t* __restrict__ tileof, const int64_t* __restrict__ toff,
                              int64_t* __restrict__ cnt) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nl;
       li += (int64_t)gridDim.x * blockDim.x)
    cnt[longrows[li]] = toff[tileof[li + 1]] - toff[tileof[li]];
}

// Stats::work per colour: the inputs' stored entries in the colour's rows.
__global__ void k_sa_work(const DevColor* __restrict__ cols, int64_t P, Csr B, Csr C, Csr D,
                          int64_t* __restrict__ work) {
  for (int64_t k = threadIdx.x; k < P; k += blockDim.x) {
    const int64_t lo = cols[k].pub.top.lo, hi = cols[k].pub.top.hi;
    work[k] = lo > hi ? 0
                      : (B.rp[hi + 1] - B.rp[lo]) + (C.rp[hi + 1] - C.rp[lo]) +
                            (D.rp[hi + 1] - D.rp[lo]);
  }
}

__global__ void k_add_offset(int64_t* __restrict__ a, int64_t n, int64_t off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] += off;
}

static int grid_n(spd_context* ctx, int64_t n) {
  int64_t g = ceil_div(n, kSaBlock);
  int64_t cap = (int64_t)ctx->num_sms * 8;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

static int64_t long_threshold() {
  static int64_t t = [] {
    const char* e = getenv("SPD_SA_T");
    return e ? atoll(e) : (int64_t)16;
  }();
  return t;
}

static void run_spadd3(spd_context* ctx, const spd_tensor* B, const spd_tensor* C,
                       const spd_tensor* D, spd_tensor** A_out, int64_t first, int64_t count,
                       spd_stats* stats) {
  checked(ctx);
  if (!B || !C || !D || !A_out) throw ValidationError("null argument");
  for (const spd_tensor* X : {B, C, D}) settle_restage(X);
  require_partition(ctx, B, first, count);
  activate(ctx);
  if (ctx->split != SplitKind::Universe)
    throw ValidationError(
        "SpAdd3 is a union (multi-term) statement: position-space split is rejected "
        "(schedule.cpp:334-336)");
  const spd_tensor* T[3] = {B, C, D};
  for (const spd_tensor* X : T) {
    if (X->levels.size() != 2 || X->levels[0].kind != SPD_DENSE ||
        X->levels[1].kind != SPD_COMPRESSED)
      throw ValidationError("unsupported on gpu: SpAdd3 operands must be ds (CSR-like)");
    if (X->dims != B->dims || X->mode_order != B->mode_order)
      throw ValidationError("SpAdd3 operands must share dimensions and storage order");
  }
  const int64_t n = B->levels[1].parent_positions;
  Csr b{B->levels[1].rowptr, B->levels[1].crd, B->vals};
  Csr c{C->levels[1].rowptr, C->levels[1].crd, C->vals};
  Csr d{D->levels[1].rowptr, D->levels[1].crd, D->vals};
  const int64_t nc = C->levels[1].positions, nd = D->levels[1].positions;
  const bool distributed = ctx->comm && ctx->world > 1 && ctx->pieces > 1 && !(first == 0 && count == ctx->pieces);
  // rows of this call: the colours' row blocks (a universe split is contiguous)
  const auto& hc = host_colors(ctx);
  int64_t lo = n, hi = -1;
  for (int64_t k = first; k < first + count; k++)
    if (hc[k].top.lo <= hc[k].top.hi) lo = std::min(lo, hc[k].top.lo), hi = std::max(hi, hc[k].top.hi);
  cudaStream_t s = ctx->stream;
  int64_t launches = 0;
  if (stats) SPD_CUDA(cudaEventRecord(ctx->ev0, s));
  const int64_t Tl = long_threshold();
  int64_t* cnt = (int64_t*)ctx->scratch[0].reserve(sizeof(int64_t) * (n + 1));
  // rows above the thread-merge threshold: one-tile rows (midrows) and hub
  // rows (longest operand > kTile, tiled)
  int32_t* midrows = (int32_t*)ctx->scratch[1].reserve(sizeof(int32_t) * 2 * (n + 1));
  int32_t* longrows = midrows + (n + 1);
  int32_t* nlists = (int32_t*)ctx->counters.reserve(64);
  unsigned long long* tickets = reinterpret_cast<unsigned long long*>(nlists) + 2;  // one per merge pass
  SPD_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n + 1), s));
  SPD_CUDA(cudaMemsetAsync(nlists, 0, 32, s));
  if (lo <= hi) {
    k_sa_count<<<grid_n(ctx, hi - lo + 1), kSaBlock, 0, s>>>(b, c, d, lo, hi, Tl, cnt, midrows, longrows,
                                                             nlists);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters, nlists, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  const int64_t nmid = reinterpret_cast<int32_t*>(ctx->pinned_counters)[0];
  const int64_t nl = reinterpret_cast<int32_t*>(ctx->pinned_counters)[1];
  const bool key32 = B->dims[B->mode_order[1]] < INT32_MAX;
  const int lgrid = ctx->num_sms * 8;
  if (nmid > 0) {
    if (key32)
      k_sa_mid<int, 0><<<lgrid, kSaBlock, 0, s>>>(b, c, d, midrows, nmid, cnt, nullptr, nullptr, nullptr, tickets);
    else
      k_sa_mid<long long, 0><<<lgrid, kSaBlock, 0, s>>>(b, c, d, midrows, nmid, cnt, nullptr, nullptr,
                                                        nullptr, tickets);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  // Merged rows: tiles per row -> tile offsets; pass 0 counts every tile.
  int64_t* tileof = (int64_t*)ctx->scratch[4].reserve(sizeof(int64_t) * (nl + 1) * 2);
  int64_t* tilecnt = tileof + (nl + 1);
  int64_t ntiles = 0;
  int64_t *tstart = nullptr, *tcount = nullptr, *toff = nullptr;
  if (nl > 0) {
    SPD_CUDA(cudaMemsetAsync(tilecnt + nl, 0, sizeof(int64_t), s));
    k_sa_tiles<<<grid_n(ctx, nl), kSaBlock, 0, s>>>(b, c, d, longrows, nl, tilecnt);
    SPD_CHECK_LAUNCH();
    size_t bytes = 0;
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, tilecnt, tileof, nl + 1, s));
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(ctx->scratch[5].reserve(bytes), bytes, tilecnt, tileof, nl + 1, s));
    SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters, tileof + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    ntiles = ctx->pinned_counters[0];
    tstart = (int64_t*)ctx->scratch[2].reserve(sizeof(int64_t) * 5 * (ntiles + 1));
    tcount = tstart + 3 * (ntiles + 1);
    toff = tcount + (ntiles + 1);
    SPD_CUDA(cudaMemsetAsync(tcount + ntiles, 0, sizeof(int64_t), s));
    if (key32)
      k_sa_merge<int, 0><<<lgrid, kSaBlock, 0, s>>>(b, c, d, longrows, nl, tileof, tstart, tcount,
                                                    nullptr, nullptr, nullptr, nullptr);
    else
      k_sa_merge<long long, 0><<<lgrid, kSaBlock, 0, s>>>(b, c, d, longrows, nl, tileof, tstart,
                                                          tcount, nullptr, nullptr, nullptr, nullptr);
    SPD_CHECK_LAUNCH();
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, tcount, toff, ntiles + 1, s));
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(ctx->scratch[5].reserve(bytes), bytes, tcount, toff, ntiles + 1, s));
    k_sa_cnt_long<<<grid_n(ctx, nl), kSaBlock, 0, s>>>(longrows, nl, tileof, toff, cnt);
    SPD_CHECK_LAUNCH();
    launches += 6;
  }
  // Phase 1 (symbolic): A's row pointer = exclusive scan of the row counts.
  int64_t* rpA = nullptr;
  SPD_CUDA(cudaMallocAsync((void**)&rpA, sizeof(int64_t) * (n + 1), s));
  {
    size_t bytes = 0;
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, rpA, n + 1, s));
    void* t = ctx->scratch[5].reserve(bytes);
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, cnt, rpA, n + 1, s));
    launches++;
  }
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters, rpA + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  const int64_t nnzA = ctx->pinned_counters[0];
  // Phase 2 (fill): exactly-sized buffers.
  int64_t* Acrd = nullptr;
  double* Avals = nullptr;
  SPD_CUDA(cudaMallocAsync((void**)&Acrd, sizeof(int64_t) * (nnzA > 0 ? nnzA : 1), s));
  SPD_CUDA(cudaMallocAsync((void**)&Avals, sizeof(double) * (nnzA > 0 ? nnzA : 1), s));
  leaf_timing_begin(ctx);
  if (lo <= hi && nnzA > 0) {
    k_sa_fill<<<grid_n(ctx, hi - lo + 1), kSaBlock, 0, s>>>(b, c, d, lo, hi, Tl, rpA, Acrd, Avals);
    SPD_CHECK_LAUNCH();
    launches++;
    if (nmid > 0) {
      if (key32)
        k_sa_mid<int, 1><<<lgrid, kSaBlock, 0, s>>>(b, c, d, midrows, nmid, nullptr, rpA, Acrd, Avals,
                                                    tickets + 1);
      else
        k_sa_mid<long long, 1><<<lgrid, kSaBlock, 0, s>>>(b, c, d, midrows, nmid, nullptr, rpA, Acrd,
                                                          Avals, tickets + 1);
      SPD_CHECK_LAUNCH();
      launches++;
    }
    if (nl > 0) {
      if (key32)
        k_sa_merge<int, 1><<<lgrid, kSaBlock, 0, s>>>(b, c, d, longrows, nl, tileof, tstart, tcount,
                                                      toff, rpA, Acrd, Avals);
      else
        k_sa_merge<long long, 1><<<lgrid, kSaBlock, 0, s>>>(b, c, d, longrows, nl, tileof, tstart,
                                                            tcount, toff, rpA, Acrd, Avals);
      SPD_CHECK_LAUNCH();
      launches++;
    }
  }
  leaf_timing_end(ctx);
  // Global pos offsets of the distributed pieces (all-gather of per-GPU nnz).
  int64_t base = 0, total = nnzA;
  if (distributed) {
    int64_t* g = (int64_t*)ctx->counters.reserve(sizeof(int64_t) * (ctx->world + 8));
    SPD_CUDA(cudaMemcpyAsync(g + ctx->rank, rpA + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    SPD_NCCL(ncclAllGather(g + ctx->rank, g, 1, ncclInt64, ctx->comm, s));
    std::vector<int64_t> all(ctx->world);
    SPD_CUDA(cudaMemcpyAsync(all.data(), g, sizeof(int64_t) * ctx->world, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    total = 0;
    for (int r = 0; r < ctx->world; r++) {
      if (r == ctx->rank) base = total;
      total += all[r];
    }
  }
  ctx->launches += launches;
  auto* A = new spd_tensor();
  A->ctx = ctx;
  A->order = B->order;
  A->dims = B->dims;
  A->kinds = B->kinds;
  A->mode_order = B->mode_order;
  A->groups = B->groups;
  A->levels.resize(2);
  A->levels[0] = B->levels[0];
  A->levels[0].rowptr = nullptr;
  A->levels[0].crd = nullptr;
  A->levels[1].kind = SPD_COMPRESSED;
  A->levels[1].parent_positions = n;
  A->levels[1].positions = nnzA;
  A->levels[1].rowptr = rpA;
  A->levels[1].crd = Acrd;
  A->nvals = nnzA;
  A->vals = Avals;
  A->owns = true;
  A->row_lo = lo;
  A->row_hi = hi;
  A->pos_base = base;
  A->global_positions = total;
  *A_out = A;
  std::vector<int64_t> work(ctx->pieces, 0);
  if (ctx->pieces > 0) {
    int64_t* w = (int64_t*)ctx->scratch[4].reserve(sizeof(int64_t) * ctx->pieces);
    k_sa_work<<<1, 256, 0, s>>>((const DevColor*)ctx->colors_dev.ptr, ctx->pieces, b, c, d, w);
    SPD_CHECK_LAUNCH();
    SPD_CUDA(cudaMemcpyAsync(work.data(), w, sizeof(int64_t) * ctx->pieces, cudaMemcpyDeviceToHost, s));
  }
  if (stats) SPD_CUDA(cudaEventRecord(ctx->ev1, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  fill_stats(ctx, stats, 0, work, launches, stats != nullptr);
}

// Collects the row blocks of a distributed SpAdd3 output on `root`: every
// rank sends its rows' pointers and its positions' crd/vals (grouped NCCL
// send/recv); the root rebases each block's pointers by the block's global
// pos offset.
static void run_gather_rows(spd_context* ctx, const spd_tensor* A, int root, spd_tensor** out) {
  checked(ctx);
  if (!A || !out) throw ValidationError("null argument");
  if (!ctx->comm) throw ValidationError("spd_gather_rows needs a communicator");
  if (root < 0 || root >= ctx->world) throw ValidationError("root outside the communicator");
  if (A->levels.size() != 2 || A->levels[1].kind != SPD_COMPRESSED)
    throw ValidationError("spd_gather_rows gathers ds (CSR-like) tensors");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  const int64_t n = A->levels[1].parent_positions;
  // every rank's (row_lo, row_hi, pos_base, positions)
  int64_t* g = (int64_t*)ctx->counters.reserve(sizeof(int64_t) * 4 * (ctx->world + 1));
  const int64_t mine[4] = {A->row_lo, A->row_hi, A->pos_base, A->levels[1].positions};
  SPD_CUDA(cudaMemcpyAsync(g + 4 * ctx->rank, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
  SPD_NCCL(ncclAllGather(g + 4 * ctx->rank, g, 4, ncclInt64, ctx->comm, s));
  std::vector<int64_t> all(4 * ctx->world);
  SPD_CUDA(cudaMemcpyAsync(all.data(), g, sizeof(int64_t) * all.size(), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  int64_t total = 0;
  for (int r = 0; r < ctx->world; r++) total += all[4 * r + 3];
  spd_tensor* F = nullptr;
  if (ctx->rank == root) {
    F = new spd_tensor();
    F->ctx = ctx;
    F->order = A->order;
    F->dims = A->dims;
    F->kinds = A->kinds;
    F->mode_order = A->mode_order;
    F->groups = A->groups;
    F->levels = A->levels;
    F->levels[1].positions = total;
    F->nvals = total;
    F->owns = true;
    F->row_lo = 0;
    F->row_hi = n - 1;
    F->global_positions = total;
    SPD_CUDA(cudaMallocAsync((void**)&F->levels[1].rowptr, sizeof(int64_t) * (n + 1), s));
    SPD_CUDA(cudaMallocAsync((void**)&F->levels[1].crd, sizeof(int64_t) * std::max<int64_t>(total, 1), s));
    SPD_CUDA(cudaMallocAsync((void**)&F->vals, sizeof(double) * std::max<int64_t>(total, 1), s));
    // rows before the first block start at 0; the final pointer is the total
    SPD_CUDA(cudaMemsetAsync(F->levels[1].rowptr, 0, sizeof(int64_t) * (n + 1), s));
    SPD_CUDA(cudaMemcpyAsync(F->levels[1].rowptr + n, &total, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  }
  SPD_NCCL(ncclGroupStart());
  if (A->row_lo <= A->row_hi) {
    const int64_t rows = A->row_hi - A->row_lo + 1;
    SPD_NCCL(ncclSend(A->levels[1].rowptr + A->row_lo, rows, ncclInt64, root, ctx->comm, s));
    if (A->levels[1].positions > 0) {
      SPD_NCCL(ncclSend(A->levels[1].crd, A->levels[1].positions, ncclInt64, root, ctx->comm, s));
      SPD_NCCL(ncclSend(A->vals, A->levels[1].positions, ncclFloat64, root, ctx->comm, s));
    }
  }
  if (ctx->rank == root) {
    for (int r = 0; r < ctx->world; r++) {
      const int64_t rl = all[4 * r], rh = all[4 * r + 1], pb = all[4 * r + 2], np = all[4 * r + 3];
      if (rl > rh) continue;
      SPD_NCCL(ncclRecv(F->levels[1].rowptr + rl, rh - rl + 1, ncclInt64, r, ctx->comm, s));
      if (np > 0) {
        SPD_NCCL(ncclRecv(F->levels[1].crd + pb, np, ncclInt64, r, ctx->comm, s));
        SPD_NCCL(ncclRecv(F->vals + pb, np, ncclFloat64, r, ctx->comm, s));
      }
    }
  }
  SPD_NCCL(ncclGroupEnd());
  if (ctx->rank == root) {
    for (int r = 0; r < ctx->world; r++) {
      const int64_t rl = all[4 * r], rh = all[4 * r + 1], pb = all[4 * r + 2];
      if (rl > rh || pb == 0) continue;
      k_add_offset<<<grid_n(ctx, rh - rl + 1), kSaBlock, 0, s>>>(F->levels[1].rowptr + rl,
                                                                  rh - rl + 1, pb);
      SPD_CHECK_LAUNCH();
    }
    // rows after the last non-empty block keep the total
    int64_t last = -1;
    for (int r = 0; r < ctx->world; r++)
      if (all[4 * r] <= all[4 * r + 1]) last = std::max(last, all[4 * r + 1]);
    if (last + 1 < n) {
      k_add_offset<<<grid_n(ctx, n - last - 1), kSaBlock, 0, s>>>(F->levels[1].rowptr + last + 1,
                                                                  n - last - 1, total);
      SPD_CHECK_LAUNCH();
    }
  }
  SPD_CUDA(cudaStreamSynchronize(s));
  *out = F;
}

}  // namespace spd

using namespace spd;

extern "C" int spd_spadd3(spd_context* ctx, const spd_tensor* B, const spd_tensor* C,
                          const spd_tensor* D, spd_tensor** A_out, int64_t first_color,
                          int64_t ncolors, spd_stats* stats) {
  return guarded([&] { run_spadd3(ctx, B, C, D, A_out, first_color, ncolors, stats); });
}

extern "C" int spd_gather_rows(spd_context* ctx, const spd_tensor* A, int root, spd_tensor** out) {
  return guarded([&] { run_gather_rows(ctx, A, root, out); });
}

extern "C" int spd_tensor_global_span(const spd_tensor* t, int64_t* row_lo, int64_t* row_hi,
                                      int64_t* pos_base, int64_t* global_positions) {
  return guarded([&] {
    if (!t) throw ValidationError("null spd_tensor");
    *row_lo = t->row_lo;
    *row_hi = t->row_hi;
    *pos_base = t->pos_base;
    *global_positions = t->global_positions;
  });
}
