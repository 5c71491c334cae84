// Row-reducing leaf kernels on sm_100a: SpMV (K3), SpMM (K4), SpTTV (K6),
// SpMTTKRP (K7), plus the chunk fixup and the deterministic colour combine
// (K9, reduce_combine sim.cpp:791-811).  See rowwalk.cuh for the execution
// scheme and DESIGN.md for the rooflines.
//
// Leaf semantics follow the reference's LeafRun (sim.cpp:258-494) as rendered
// by plan.cpp:158-365 (tests/golden/plan_spmv_row.txt:28-33,
// plan_spmv_nonzero.txt:23-28): for every stored position of the colour the
// product of the accessed values is added to the output entry, in position
// order within a row; this backend reassociates that sum (FMA, chunk and
// colour partials), which north_star allows within 1e-10 relative.
#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <cub/cub.cuh>

#include "rowwalk.cuh"

namespace spd {

#define FULL 0xffffffffu

// ---------------------------------------------------------------------------
// Setup: output write ranges W_c and chunk starts for every colour, and the
// chunk range of the colours this GPU runs.  k_setup_rows: one warp per
// colour finds the first row starting inside it (a 32-ary search);
// k_setup: one CTA links the colours -- W_c of a nonzero split ends before
// the next non-empty colour's first row -- and numbers the chunks (prefix
// sum); O(log P) block steps up to 1024 colours, a serial pass above.
__global__ void k_setup_rows(DevColor* __restrict__ cols, int64_t P, int split, int out_level,
                             const int64_t* __restrict__ R, int64_t nrows, int64_t* __restrict__ counters,
                             int64_t* __restrict__ ff0, int64_t n0, int64_t* __restrict__ ff1, int64_t n1) {
  // the call's scratch: combines / ticket counters zeroed, record slots -1
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) counters[0] = 0, counters[3] = 0;
  for (int64_t i = tid; i < n0; i += nt) ff0[i] = -1;
  for (int64_t i = tid; i < n1; i += nt) ff1[i] = -1;
  const int64_t c = tid >> 5;
  if (c >= P) return;
  const spd_color pc = cols[c].pub;
  int64_t wl = 1, wh = 0;
  if (split == (int)SplitKind::Universe) {
    spd_range w = out_level == 0 ? pc.top : pc.par;
    wl = w.lo, wh = w.hi;
  } else if (pc.q.lo <= pc.q.hi) {
    int64_t o = warp_owner(R, nrows, pc.q.lo);
    wl = ld64(R + o) == pc.q.lo ? o : o + 1;  // first row starting inside the colour
  }
  if (lane_id() == 0) cols[c].w_lo = wl, cols[c].w_hi = wh;
}

constexpr int kSetupMax = 1024;

__global__ void __launch_bounds__(kSetupMax) k_setup(DevColor* __restrict__ cols, int64_t P, int split,
                                                     int64_t nrows, int64_t CH, int64_t c_first, int64_t c_count,
                                                     int64_t* __restrict__ counters) {
  __shared__ int64_t a[kSetupMax], b[kSetupMax];
  const int t = threadIdx.x;
  if (P <= kSetupMax) {
    const bool live = t < P;
    const bool ne = live && cols[t].pub.q.lo <= cols[t].pub.q.hi;
    int64_t wl = live ? cols[t].w_lo : 0;
    if (split == (int)SplitKind::NonZero) {
      // nxt(t) = w_lo of the first non-empty colour after t (nrows if none):
      // a suffix minimum (non-empty colours' w_lo ascend); first = the
      // smallest non-empty colour
      a[t] = ne ? wl : INT64_MAX;
      b[t] = ne ? t : INT64_MAX;
      __syncthreads();
      for (int off = 1; off < kSetupMax; off <<= 1) {
        const int64_t va = t + off < kSetupMax ? a[t + off] : INT64_MAX;
        const int64_t vb = t >= off ? b[t - off] : INT64_MAX;
        __syncthreads();
        a[t] = min(a[t], va);
        b[t] = min(b[t], vb);
        __syncthreads();
      }
      const int64_t nxt_incl_next = t + 1 < kSetupMax ? a[t + 1] : INT64_MAX;
      const int64_t nxt = nxt_incl_next == INT64_MAX ? nrows : nxt_incl_next;
      const int64_t first_ne = b[kSetupMax - 1];
      __syncthreads();
      if (live) {
        int64_t lo = ne ? wl : nxt, hi = nxt - 1;
        if (first_ne == INT64_MAX) {  // no positions at all: the last colour stores the zero rows
          if (t == P - 1) lo = 0, hi = nrows - 1;
        } else if (t == first_ne) {
          lo = 0;
        }
        cols[t].w_lo = lo, cols[t].w_hi = hi;
        wl = lo;
      }
    }
    // chunks per colour, exclusive prefix sum
    int64_t n = 0;
    if (live) {
      const DevColor& d = cols[t];
      n = ne ? (d.pub.q.hi - d.pub.q.lo + CH) / CH : (d.w_lo <= d.w_hi ? 1 : 0);
    }
    a[t] = n;
    __syncthreads();
    for (int off = 1; off < kSetupMax; off <<= 1) {
      const int64_t v = t >= off ? a[t - off] : 0;
      __syncthreads();
      a[t] += v;
      __syncthreads();
    }
    const int64_t run = a[t] - n;  // exclusive
    if (live) {
      cols[t].chunk_begin = run;
      if (t == c_first) counters[1] = run;
      if (t == c_first + c_count - 1) counters[2] = a[t];
    }
    return;
  }
  if (t != 0) return;
  if (split == (int)SplitKind::NonZero) {
    int64_t next = nrows, first_ne = -1;
    for (int64_t c = P - 1; c >= 0; c--) {
      if (cols[c].pub.q.lo <= cols[c].pub.q.hi) {
        cols[c].w_hi = next - 1;
        next = cols[c].w_lo;
        first_ne = c;
      } else {
        cols[c].w_lo = next;
        cols[c].w_hi = next - 1;
      }
    }
    if (first_ne >= 0) {
      cols[first_ne].w_lo = 0;
    } else {  // no positions at all: the last colour stores the zero rows
      cols[P - 1].w_lo = 0;
      cols[P - 1].w_hi = nrows - 1;
    }
  }
  int64_t run = 0;
  for (int64_t c = 0; c < P; c++) {
    const DevColor& d = cols[c];
    int64_t n = d.pub.q.lo <= d.pub.q.hi ? (d.pub.q.hi - d.pub.q.lo + CH) / CH
                                           : (d.w_lo <= d.w_hi ? 1 : 0);
    if (c == c_first) counters[1] = run;
    cols[c].chunk_begin = run;
    run += n;
    if (c == c_first + c_count - 1) counters[2] = run;
  }
}

void launch_setup(cudaStream_t s, DevColor* cols, int64_t P, int split, int out_level, const int64_t* R,
                  int64_t nrows, int64_t CH, int64_t c_first, int64_t c_count, int64_t* counters, int64_t* ff0,
                  int64_t n0, int64_t* ff1, int64_t n1) {
  const int64_t blocks = std::max<int64_t>(ceil_div(P * 32, 256), std::min<int64_t>(ceil_div(n0 + n1, 256), 148));
  k_setup_rows<<<(unsigned)blocks, 256, 0, s>>>(cols, P, split, out_level, R, nrows, counters, ff0, n0, ff1, n1);
  SPD_CHECK_LAUNCH();
  k_setup<<<1, kSetupMax, 0, s>>>(cols, P, split, nrows, CH, c_first, c_count, counters);
  SPD_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// SpMM / SpMTTKRP family: lane = output column, positions streamed serially
// per warp with UNR independent 256-byte row gathers in flight.
constexpr int kUnr = 8;

template <int CPL>
struct ColAcc {
  double v[CPL];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int t = 0; t < CPL; t++) v[t] = 0.0;
  }
};

template <int CPL>
__device__ __forceinline__ void store_row(double* __restrict__ out, int64_t W, int64_t r,
                                          const ColAcc<CPL>& a) {
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < CPL; t++) {
    int64_t col = lane + 32 * t;
    if (col < W) out[r * W + col] = a.v[t];
  }
}

template <int CPL>
__device__ __forceinline__ void store_rec(double* __restrict__ val, int64_t slot, int64_t W,
                                          const ColAcc<CPL>& a) {
  store_row<CPL>(val, W, slot, a);
}

// Row-transition bookkeeping shared by the column kernels.
struct ColState {
  int64_t r, nb;       // current output row and its end (exclusive)
  bool head;           // current row started before the chunk
  int64_t head_row;    // head record row (-1 none)
  int head_cont;
};

template <int CPL>
__device__ __forceinline__ void col_row_end(const WalkGeom& g, ColState& st, ColAcc<CPL>& acc,
                                            int64_t q, double* __restrict__ out,
                                            const ChunkRecs& rec, int64_t k,
                                            const ChunkInfo& ci) {
  if (st.head) {
    store_rec<CPL>(rec.val, 2 * k, g.W, acc);
    st.head_row = st.r;
    st.head_cont = 0;
    st.head = false;
  } else {
    store_row<CPL>(out, g.W, st.r, acc);
  }
  acc.zero();
  st.r = skip_empty_rows(g, st.r + 1, q, st.nb, out, ci.w_lo, ci.w_hi);
}

template <int CPL>
__device__ __forceinline__ void col_chunk_end(const WalkGeom& g, ColState& st, ColAcc<CPL>& acc,
                                              double* __restrict__ out, const ChunkRecs& rec,
                                              int64_t k, const ChunkInfo& ci) {
  int64_t tail_row = -1;
  if (st.nb == ci.e + 1) {
    if (st.head) {
      store_rec<CPL>(rec.val, 2 * k, g.W, acc);
      st.head_row = st.r;
      st.head_cont = 0;
    } else {
      store_row<CPL>(out, g.W, st.r, acc);
    }
    int64_t nb;
    if (st.r + 1 < g.nrows) skip_empty_rows(g, st.r + 1, ci.e + 1, nb, out, ci.w_lo, ci.w_hi);
  } else if (st.head) {
    store_rec<CPL>(rec.val, 2 * k, g.W, acc);
    st.head_row = st.r;
    st.head_cont = 1;
  } else {
    store_rec<CPL>(rec.val, 2 * k + 1, g.W, acc);
    tail_row = st.r;
  }
  if (lane_id() == 0) {
    rec.row[2 * k] = st.head_row;
    rec.row[2 * k + 1] = tail_row;
    rec.cont[k] = st.head_cont;
  }
}

__device__ __forceinline__ void empty_chunk(const WalkGeom& g, const ChunkInfo& ci,
                                            double* __restrict__ out, const ChunkRecs& rec) {
  zero_rows(out, g.W, ci.w_lo, ci.w_hi);
  if (lane_id() == 0) {
    rec.row[2 * ci.local] = -1;
    rec.row[2 * ci.local + 1] = -1;
    rec.cont[ci.local] = 0;
  }
}

// SpMM: A(i,j) = sum_k B(i,k) * C(k,j).  Row stride of C and A is W = N.
template <int CPL>
__global__ void __launch_bounds__(kBlock) k_spmm_walk(WalkGeom g, const int64_t* __restrict__ crd,
                                                      const double* __restrict__ vals,
                                                      const double* __restrict__ C,
                                                      double* __restrict__ A, ChunkRecs rec,
                                                      const int64_t* __restrict__ counters) {
  const int lane = lane_id();
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t N = g.W;
  for (int64_t v = begin + chunk_ticket(counters); v < end; v = begin + chunk_ticket(counters)) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) {
      empty_chunk(g, ci, A, rec);
      continue;
    }
    const int64_t k = ci.local, s = ci.s, e = ci.e;
    ColState st;
    st.r = warp_owner(g.R, g.nrows, s);
    st.nb = ld64(g.R + st.r + 1);
    st.head = ld64(g.R + st.r) < s;
    st.head_row = -1;
    st.head_cont = 0;
    if (s == ci.q_lo) zero_rows(A, N, ci.w_lo, st.r - 1);
    ColAcc<CPL> acc;
    acc.zero();
    for (int64_t base = s; base <= e; base += 32) {
      const int cnt = (int)min((int64_t)32, e - base + 1);
      int64_t my_k = 0;
      double my_v = 0.0;
      if (lane < cnt) {
        my_k = ld64(crd + base + lane);
        my_v = __ldg(vals + base + lane);
      }
      for (int u0 = 0; u0 < cnt; u0 += kUnr) {
        double cv[kUnr][CPL];
#pragma unroll
        for (int i = 0; i < kUnr; i++) {
          const int64_t kk = __shfl_sync(FULL, my_k, (u0 + i) & 31);
#pragma unroll
          for (int t = 0; t < CPL; t++) {
            const int64_t col = lane + 32 * t;
            cv[i][t] = (u0 + i < cnt && col < N) ? __ldg(C + kk * N + col) : 0.0;
          }
        }
#pragma unroll
        for (int i = 0; i < kUnr; i++) {
          if (u0 + i < cnt) {
            const int64_t q = base + u0 + i;
            if (q == st.nb) col_row_end<CPL>(g, st, acc, q, A, rec, k, ci);
            const double bv = __shfl_sync(FULL, my_v, u0 + i);
#pragma unroll
            for (int t = 0; t < CPL; t++) acc.v[t] = fma(bv, cv[i][t], acc.v[t]);
          }
        }
      }
    }
    col_chunk_end<CPL>(g, st, acc, A, rec, k, ci);
  }
}

// ---------------------------------------------------------------------------
// SpMM, N == 32 specialisation (the C2 configuration).  Half a warp per
// stored position: lane l covers columns 2(l%16), 2(l%16)+1 with one 128-bit
// load, so a warp instruction gathers the 256-byte C rows of two positions.
// Row starts inside each 32-position window come from one coalesced load of
// the row pointer (a 32-bit mask), so the per-position work is a shuffle, a
// 128-bit gather, two FMAs and a bit test.  C rows are gathered with L2
// evict_last priority; crd / vals / A stream with evict_first so the 7 GB of
// streamed data does not push the reused C rows out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_f64x2_hint(const double* ptr, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_i32_hint(const int32_t* ptr, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_i64_hint(const int64_t* ptr, uint64_t pol) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_f64_hint(const double* ptr, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_f64x2_hint(double* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

// SpMTTKRP over a dss CSF: A(i,l) = sum_{j,k} B(i,j,k) * C(j,l) * D(k,l).
// Output rows are i; g.R is the derived leaf row pointer rp2[rp1[i]].  The
// fibre (j) of each position is tracked alongside; W = R (rank).
template <int CPL>
__global__ void __launch_bounds__(kBlock) k_mttkrp_walk(
    WalkGeom g, const int64_t* __restrict__ rp2, int64_t F, const int64_t* __restrict__ crd1,
    const int64_t* __restrict__ crd2, const double* __restrict__ vals,
    const double* __restrict__ C, const double* __restrict__ D, double* __restrict__ A,
    ChunkRecs rec, const int64_t* __restrict__ counters) {
  const int lane = lane_id();
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t Rk = g.W;
  for (int64_t v = begin + chunk_ticket(counters); v < end; v = begin + chunk_ticket(counters)) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) {
      empty_chunk(g, ci, A, rec);
      continue;
    }
    const int64_t k = ci.local, s = ci.s, e = ci.e;
    ColState st;
    st.r = warp_owner(g.R, g.nrows, s);
    st.nb = ld64(g.R + st.r + 1);
    st.head = ld64(g.R + st.r) < s;
    st.head_row = -1;
    st.head_cont = 0;
    if (s == ci.q_lo) zero_rows(A, Rk, ci.w_lo, st.r - 1);
    int64_t f = warp_owner(rp2, F, s);
    int64_t fe = ld64(rp2 + f + 1);
    double cj[CPL];
    {
      const int64_t j = ld64(crd1 + f);
#pragma unroll
      for (int t = 0; t < CPL; t++) {
        const int64_t col = lane + 32 * t;
        cj[t] = col < Rk ? __ldg(C + j * Rk + col) : 0.0;
      }
    }
    ColAcc<CPL> acc;
    acc.zero();
    for (int64_t base = s; base <= e; base += 32) {
      const int cnt = (int)min((int64_t)32, e - base + 1);
      int64_t my_k = 0;
      double my_v = 0.0;
      if (lane < cnt) {
        my_k = ld64(crd2 + base + lane);
        my_v = __ldg(vals + base + lane);
      }
      for (int u0 = 0; u0 < cnt; u0 += kUnr) {
        double dv[kUnr][CPL];
#pragma unroll
        for (int i = 0; i < kUnr; i++) {
          const int64_t kk = __shfl_sync(FULL, my_k, (u0 + i) & 31);
#pragma unroll
          for (int t = 0; t < CPL; t++) {
            const int64_t col = lane + 32 * t;
            dv[i][t] = (u0 + i < cnt && col < Rk) ? __ldg(D + kk * Rk + col) : 0.0;
          }
        }
#pragma unroll
        for (int i = 0; i < kUnr; i++) {
          if (u0 + i < cnt) {
            const int64_t q = base + u0 + i;
            if (q == st.nb) col_row_end<CPL>(g, st, acc, q, A, rec, k, ci);
            if (q == fe) {
              do {
                f++;
                fe = ld64(rp2 + f + 1);
              } while (fe == q);
              const int64_t j = ld64(crd1 + f);
#pragma unroll
              for (int t = 0; t < CPL; t++) {
                const int64_t col = lane + 32 * t;
                cj[t] = col < Rk ? __ldg(C + j * Rk + col) : 0.0;
              }
            }
            const double bv = __shfl_sync(FULL, my_v, u0 + i);
#pragma unroll
            for (int t = 0; t < CPL; t++) acc.v[t] = fma(bv * cj[t], dv[i][t], acc.v[t]);
          }
        }
      }
    }
    col_chunk_end<CPL>(g, st, acc, A, rec, k, ci);
  }
}

// ---------------------------------------------------------------------------
// SpMV / SpTTV family: lane = position.  Each warp streams its chunk in
// windows of 32 positions with coalesced crd/vals loads; products are
// reduced per row with a warp segmented scan (heads from the row pointer
// window held one row per lane), so a window costs the same whether it holds
// one row or 32.
__device__ __forceinline__ void load_rows(const WalkGeom& g, int64_t rb, int64_t& S, int64_t& E) {
  const int64_t rr = rb + lane_id();
  if (rr < g.nrows) {
    S = ld64(g.R + rr);
    E = ld64(g.R + rr + 1);
  } else {
    S = INT64_MAX;
    E = INT64_MAX;
  }
}


}  // namespace spd
#include "leaf_nz.cuh"
namespace spd {

// ---------------------------------------------------------------------------
// Non-empty rows in each colour's write range W_c (spd_colour_costs): the
// compacted row ids inside [w_lo, w_hi], one warp per colour.
__global__ void k_colour_nonempty(const DevColor* __restrict__ cols, int64_t P, NzView z, int64_t* __restrict__ out) {
  z.m = nz_count(z);
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= P) return;
  const int64_t lo = cols[c].w_lo, hi = cols[c].w_hi;
  // rows < lo and rows <= hi among the m sorted ids
  const int64_t a = warp_upper_bound(z.id, z.m, lo - 1), b = warp_upper_bound(z.id, z.m, hi);
  if (lane_id() == 0) out[c] = lo <= hi ? b - a : 0;
}

// ---------------------------------------------------------------------------
// Uneven colour blocks: the all-gathered head records, cmax slots per rank,
// to their colours' slots (the calling rank's own block is already there).
__global__ void k_unpack_heads(const int64_t* __restrict__ stage, const int64_t* __restrict__ bounds, int world,
                               int own, int64_t cmax, int64_t rec_words, int64_t* __restrict__ head_pack) {
  const int64_t total = (int64_t)world * cmax * rec_words;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = i / rec_words, w = i - slot * rec_words;
    const int r = (int)(slot / cmax);
    const int64_t j = slot - (int64_t)r * cmax;
    if (r == own || j >= bounds[r + 1] - bounds[r]) continue;
    head_pack[(bounds[r] + j) * rec_words + w] = stage[i];
  }
}

// ---------------------------------------------------------------------------
// Chunk fixup: sums each cut row's records in chunk order.  Rows cut by the
// end of a colour become colour tail records; the head chain at the start of
// a colour becomes its packed head record.
// sum + vals[k0*stride], ..., vals[k1*stride] added in that order, 16 loads
// in flight (a hub row's chain spans hundreds of chunk records)
__device__ __forceinline__ double chain_sum(double sum, const double* __restrict__ vals, int64_t stride,
                                            int64_t k0, int64_t k1) {
  int64_t k2 = k0;
  for (; k2 + 15 <= k1; k2 += 16) {
    double t[16];
#pragma unroll
    for (int i = 0; i < 16; i++) t[i] = vals[(k2 + i) * stride];
#pragma unroll
    for (int i = 0; i < 16; i++) sum += t[i];
  }
  for (; k2 <= k1; k2++) sum += vals[k2 * stride];
  return sum;
}

__device__ __forceinline__ int64_t chain_stop(const int* __restrict__ cont, int64_t from,
                                              int64_t to) {
  const int lane = lane_id();
  for (int64_t b = from; b < to; b += 128) {  // 128 flags per round, loads issued together
    int f[4];
#pragma unroll
    for (int i = 0; i < 4; i++) f[i] = b + 32 * i + lane < to ? cont[b + 32 * i + lane] : 1;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const unsigned m = __ballot_sync(FULL, b + 32 * i + lane < to && f[i] == 0);
      if (m) return b + 32 * i + __ffs(m) - 1;
    }
  }
  return to;
}

constexpr int kFixupColours = 1024;  // colours whose chunk starts the fixup keeps in shared memory

// One warp per 8 consecutive chunks, 4 lanes per chunk: the common case -- a
// tail record whose row ends in the next chunk (or at the colour's end) --
// is summed by its own 4 lanes (tail + the next chunk's head, 16-byte pairs
// interleaved over the row's W values), so the records of 8 chunks are in
// flight together; rows spanning several chunks and colour-start head
// records go through the warp-cooperative chain sums, one chunk at a time
// (few per warp: hub-dense stretches of the matrix put several in a group).
// `vec2`: W even and the output 16-byte aligned.
__global__ void __launch_bounds__(kBlock) k_chunk_fixup(WalkGeom g, ChunkRecs rec, ColorRecs col,
                                                        double* __restrict__ out, int vec2) {
  // the chunk starts of this GPU's colours, so a chunk's colour is a search
  // in shared memory instead of log2(P) dependent global loads
  __shared__ int64_t cb_s[kFixupColours];
  const bool in_smem = g.c_count <= kFixupColours;
  if (in_smem)
    for (int64_t i = threadIdx.x; i < g.c_count; i += blockDim.x) cb_s[i] = g.cols[g.c_first + i].chunk_begin;
  __syncthreads();
  const int lane = lane_id();
  const int64_t begin = col.counters[1], end = col.counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t W = g.W;
  const int sub = lane & 3;  // 4 lanes per chunk, 8 chunks per warp
  for (int64_t v0 = begin + gw * 8; v0 < end; v0 += nw * 8) {
    const int64_t v = v0 + (lane >> 2);
    const bool live = v < end;
    int64_t c = g.c_first;
    if (live) {
      if (in_smem) {
        int64_t lo = 0, hi = g.c_count - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi + 1) >> 1;
          if (cb_s[mid] <= v) lo = mid; else hi = mid - 1;
        }
        c = g.c_first + lo;
      } else {
        c = colour_of_chunk(g, v);
      }
    }
    const int64_t k = v - begin;
    const int64_t cstart = live ? (in_smem ? cb_s[c - g.c_first] : g.cols[c].chunk_begin) : -1;
    const int64_t cend =
        (c + 1 < g.c_first + g.c_count ? (in_smem ? cb_s[c + 1 - g.c_first] : g.cols[c + 1].chunk_begin) : end) -
        begin;
    const int64_t trow = live ? rec.row[2 * k + 1] : -1;
    const int64_t hrow = live ? rec.row[2 * k] : -1;
    const bool has_next = k + 1 < cend;
    const int next_cont = trow >= 0 && has_next ? rec.cont[k + 1] : 0;
    const bool fast = trow >= 0 && next_cont == 0;
    if (fast) {  // tail + next head (or the colour's tail record): 4 lanes, interleaved 16-byte pairs
      const double* t = rec.val + (2 * k + 1) * W;
      const double* h = rec.val + (2 * k + 2) * W;
      double* o = has_next ? out + trow * W : col.tail_val + c * W;
      if (vec2 && has_next) {  // (the colour tail records are 8-byte aligned only)
        for (int64_t j0 = 2 * sub; j0 < W; j0 += 32) {
          double2 a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; i++)
            if (j0 + 8 * i < W) {
              a[i] = __ldg(reinterpret_cast<const double2*>(t + j0 + 8 * i));
              b[i] = __ldg(reinterpret_cast<const double2*>(h + j0 + 8 * i));
            }
#pragma unroll
          for (int i = 0; i < 4; i++)
            if (j0 + 8 * i < W)
              *reinterpret_cast<double2*>(o + j0 + 8 * i) = make_double2(a[i].x + b[i].x, a[i].y + b[i].y);
        }
      } else {
        for (int64_t j = sub; j < W; j += 4) o[j] = has_next ? __ldg(t + j) + __ldg(h + j) : __ldg(t + j);
      }
      if (!has_next && sub == 0) col.tail_row[c] = trow;
    }
    unsigned slow = __ballot_sync(FULL, sub == 0 && ((trow >= 0 && !fast) || (v == cstart && hrow >= 0)));
    while (slow) {
      const int src = __ffs(slow) - 1;
      slow &= slow - 1;
      const int64_t kk = __shfl_sync(FULL, k, src), cc = __shfl_sync(FULL, c, src);
      const int64_t ce = __shfl_sync(FULL, cend, src);
      const int64_t tr = __shfl_sync(FULL, trow, src), hr = __shfl_sync(FULL, hrow, src);
      const bool tslow = __shfl_sync(FULL, (int)(trow >= 0 && !fast), src) != 0;
      const bool cs = __shfl_sync(FULL, (int)(v == cstart), src) != 0;
      if (tslow) {
        const int64_t stop = chain_stop(rec.cont, kk + 1, ce);
        const int64_t last = stop < ce ? stop : ce - 1;
        for (int64_t j = lane; j < W; j += 32) {
          const double sum = chain_sum(rec.val[(2 * kk + 1) * W + j], rec.val + j, 2 * W, kk + 1, last);
          if (stop < ce) out[tr * W + j] = sum;
          else col.tail_val[cc * W + j] = sum;
        }
        if (stop >= ce && lane == 0) col.tail_row[cc] = tr;
      }
      if (cs && hr >= 0) {
        const int64_t stop = rec.cont[kk] == 0 ? kk : chain_stop(rec.cont, kk + 1, ce);
        const int64_t last = stop < ce ? stop : ce - 1;
        int64_t* pack = col.head_pack + cc * (W + 2);
        for (int64_t j = lane; j < W; j += 32)
          reinterpret_cast<double*>(pack)[2 + j] = chain_sum(0.0, rec.val + j, 2 * W, kk, last);
        if (lane == 0) {
          pack[0] = hr;
          pack[1] = stop < ce ? 0 : 1;
        }
      }
    }
  }
}

// K9: colour combine.  A row cut between colours is owned by the colour
// where it starts (its tail record); the partials of the following colours
// that continue it (their head records) are added in ascending colour order,
// exactly the order of reduce_combine (sim.cpp:797-808).  Also counts
// Stats::combines = W per extra contributing colour.
__global__ void k_colour_combine(ColorRecs col, const DevColor* __restrict__ cols, int64_t P,
                                 int64_t W, int64_t c_first, int64_t c_count,
                                 double* __restrict__ out) {
  const int lane = lane_id();
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= P) return;
  const int64_t* hp = col.head_pack + c * (W + 2);
  if (hp[0] >= 0 && lane == 0) atomicAdd((unsigned long long*)&col.counters[0], (unsigned long long)W);
  if (c < c_first || c >= c_first + c_count) return;
  const int64_t r = col.tail_row[c];
  if (r < 0) return;
  for (int64_t j = lane; j < W; j += 32) {
    double sum = col.tail_val[c * W + j];
    for (int64_t c2 = c + 1; c2 < P; c2++) {
      if (cols[c2].pub.q.lo > cols[c2].pub.q.hi) continue;  // colours without positions
      const int64_t* h2 = col.head_pack + c2 * (W + 2);
      if (h2[0] != r) break;
      sum += reinterpret_cast<const double*>(h2)[2 + j];
      if (!h2[1]) break;
    }
    out[r * W + j] = sum;
  }
}

__global__ void k_leaf_rowptr(const int64_t* __restrict__ rp1, const int64_t* __restrict__ rp2,
                              int64_t I, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= I;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rp2[rp1[i]];
}

// Compressed top level (an sss CSF): output row i's leaves start at the
// first top position whose coordinate is >= i (rows absent from crd0 are
// empty), so out is a dense row pointer over [0, I] like the dss one.
__global__ void k_leaf_rowptr_sparse_top(const int64_t* __restrict__ crd0, int64_t n0,
                                         const int64_t* __restrict__ rp1, const int64_t* __restrict__ rp2,
                                         int64_t I, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= I;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n0;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (crd0[mid] < i) lo = mid + 1; else hi = mid;
    }
    out[i] = rp2[rp1[lo]];
  }
}

// ---------------------------------------------------------------------------
enum class Op { SpMV, SpMM, SpTTV, SpMTTKRP };

struct OpArgs {
  Op op;
  const spd_tensor* B;
  const double* x;  // c (SpMV, SpTTV) / C (SpMM, SpMTTKRP)
  const double* D;  // SpMTTKRP
  int64_t W;        // values per output row (1, N, R)
  double* out;
};

template <class K>
static int occupancy_grid(spd_context* ctx, K kernel) {
  int per_sm = 0;
  SPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, 0));
  if (per_sm < 1) per_sm = 1;
  return ctx->num_sms * per_sm;
}

// Compacted non-empty-row view of row pointer R of tensor t (cached on t).
// Built without a host synchronisation: the row-id and start arrays are sized
// by the row count (an upper bound of the non-empty rows) and the count stays
// on the device (NzView::m_dev, read by the kernels); `need_host_m` also
// copies it to the host (the SpMV leaf choice depends on it).
static NzView nz_view(spd_context* ctx, spd_tensor* t, const int64_t* R, int64_t nrows, bool need_host_m = false) {
  cudaStream_t s = ctx->stream;
  auto host_m = [&](spd_tensor::NzCache& e) {
    if (need_host_m && e.m < 0) {
      SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 8, e.m_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      SPD_CUDA(cudaStreamSynchronize(s));
      e.m = ctx->pinned_counters[8];
    }
  };
  for (auto& e : t->nz)
    if (e.R == R) {
      host_m(e);
      return NzView{e.ptr, e.id, e.m, e.m_dev};
    }
  spd_tensor::NzCache* slot = nullptr;
  for (auto& e : t->nz)
    if (!e.R && (!slot || e.cap_id > slot->cap_id)) slot = &e;  // prefer reusable buffers
  if (!slot) {
    slot = &t->nz[0];
    slot->R = nullptr;
  }
  unsigned char* flags = nullptr;
  const int64_t nid = nrows > 0 ? nrows : 1;
  if (t->stage_flags_cap >= nid) {
    flags = t->stage_flags;  // a restaged tensor's staging buffer, idle here
  } else {
    SPD_CUDA(cudaMallocAsync((void**)&flags, nid, s));
  }
  if (!slot->m_dev) SPD_CUDA(cudaMallocAsync((void**)&slot->m_dev, sizeof(int64_t), s));
  if (slot->cap_id < nid) {
    if (slot->id) cudaFreeAsync(slot->id, s);
    if (slot->ptr) cudaFreeAsync(slot->ptr, s);
    SPD_CUDA(cudaMallocAsync((void**)&slot->id, sizeof(int64_t) * nid, s));
    SPD_CUDA(cudaMallocAsync((void**)&slot->ptr, sizeof(int64_t) * (nid + 1), s));
    slot->cap_id = nid;
  }
  SPD_CUDA(cudaMemsetAsync(slot->m_dev, 0, sizeof(int64_t), s));
  if (nrows > 0) {
    k_nz_flags<<<(unsigned)std::min<int64_t>(ceil_div(nrows, 256), ctx->num_sms * 16), 256, 0, s>>>(R, nrows, flags);
    SPD_CHECK_LAUNCH();
    cub::CountingInputIterator<int64_t> it(0);
    size_t bytes = 0;
    SPD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, slot->id, slot->m_dev, nrows, s));
    void* tmp = ctx->scratch[5].reserve(bytes);
    SPD_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, it, flags, slot->id, slot->m_dev, nrows, s));
  }
  k_nz_ptr<<<(unsigned)std::min<int64_t>(ceil_div(nid + 1, 256), ctx->num_sms * 16), 256, 0, s>>>(
      R, nrows, slot->id, slot->m_dev, slot->ptr);
  SPD_CHECK_LAUNCH();
  if (flags != t->stage_flags) cudaFreeAsync(flags, s);
  slot->R = R;
  slot->m = -1;
  ctx->launches += 3;
  host_m(*slot);
  return NzView{slot->ptr, slot->id, slot->m, slot->m_dev};
}

// Non-empty rows of row pointer R (of t) inside each span [lo, hi]: two
// binary searches over the compacted view's sorted row ids.
__global__ void k_nonempty_in_spans(const int64_t* __restrict__ ids, const int64_t* __restrict__ m_dev,
                                    const int64_t* __restrict__ spans, int64_t nspans, int64_t* __restrict__ out) {
  const int64_t m = *m_dev;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nspans; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = spans[2 * j], hi = spans[2 * j + 1];
    if (lo > hi) {
      out[j] = 0;
      continue;
    }
    int64_t a = 0, b = m;  // first id >= lo
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (ids[mid] < lo) a = mid + 1; else b = mid;
    }
    int64_t c = a, d = m;  // first id > hi
    while (c < d) {
      const int64_t mid = (c + d) >> 1;
      if (ids[mid] <= hi) c = mid + 1; else d = mid;
    }
    out[j] = c - a;
  }
}

std::vector<int64_t> nonempty_in_spans(spd_context* ctx, spd_tensor* t, const int64_t* R, int64_t nrows,
                                       const std::vector<int64_t>& spans) {
  const NzView z = nz_view(ctx, t, R, nrows);
  const int64_t ns = (int64_t)spans.size() / 2;
  std::vector<int64_t> out(ns, 0);
  if (ns == 0) return out;
  cudaStream_t s = ctx->stream;
  int64_t* d = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * 3 * ns);
  SPD_CUDA(cudaMemcpyAsync(d, spans.data(), sizeof(int64_t) * 2 * ns, cudaMemcpyHostToDevice, s));
  k_nonempty_in_spans<<<(unsigned)std::min<int64_t>(ceil_div(ns, 256), 1024), 256, 0, s>>>(z.id, z.m_dev, d, ns,
                                                                                             d + 2 * ns);
  SPD_CHECK_LAUNCH();
  SPD_CUDA(cudaMemcpyAsync(out.data(), d + 2 * ns, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  dev_free(ctx, d);
  return out;
}

// int32 leaf crd with hot-column bit for dense rows of `rowbytes` (cached on
// t): the most referenced columns whose rows fit in ~70% of L2 are hot and
// gathered with L2 evict_last, the rest with evict_first -- an LFU-like L2
// policy for the power-law column distribution.
static const int32_t* hot_crd(spd_context* ctx, spd_tensor* t, int64_t rowbytes) {
  if (t->crd32h && t->crd32h_rowbytes == rowbytes) return t->crd32h;
  const spd_level_store& L = t->levels.back();
  // positions held: all of them, or a placed piece's range
  const int64_t lo = t->piece ? t->piece_lo : 0;
  const int64_t nnz = t->piece ? t->piece_hi - t->piece_lo + 1 : L.positions;
  const int64_t ncols = t->dims[t->mode_order[t->groups.back()[0]]];
  cudaStream_t s = ctx->stream;
  int l2 = 0;
  SPD_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
  static double frac = [] {
    const char* e = getenv("SPD_HOT_FRAC");
    return e ? atof(e) : 0.7;
  }();
  const int64_t k = std::max<int64_t>(1, (int64_t)(frac * l2) / rowbytes);
  int32_t *counts = nullptr, *sorted = nullptr;
  SPD_CUDA(cudaMallocAsync((void**)&counts, sizeof(int32_t) * (ncols > 0 ? ncols : 1), s));
  SPD_CUDA(cudaMallocAsync((void**)&sorted, sizeof(int32_t) * (ncols > 0 ? ncols : 1), s));
  SPD_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (ncols > 0 ? ncols : 1), s));
  if (!t->crd32h_alloc)
    SPD_CUDA(cudaMallocAsync((void**)&t->crd32h_alloc, sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
  t->crd32h = t->crd32h_alloc - lo;  // indexed by global position
  const unsigned grid = (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(nnz, 256), 1), ctx->num_sms * 16);
  if (nnz > 0) {
    k_col_count<<<grid, 256, 0, s>>>(L.crd + lo, nnz, counts);
    SPD_CHECK_LAUNCH();
    size_t bytes = 0;
    SPD_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, bytes, counts, sorted, ncols, 0, 32, s));
    void* tmp = ctx->scratch[5].reserve(bytes);
    SPD_CUDA(cub::DeviceRadixSort::SortKeysDescending(tmp, bytes, counts, sorted, ncols, 0, 32, s));
    k_crd32h<<<grid, 256, 0, s>>>(L.crd + lo, nnz, counts, sorted, k, ncols, t->crd32h_alloc);
    SPD_CHECK_LAUNCH();
    ctx->launches += 3;
  }
  cudaFreeAsync(counts, s);
  cudaFreeAsync(sorted, s);
  t->crd32h_rowbytes = rowbytes;
  return t->crd32h;
}

// Compacted-column SpMV (SPD_XC: 1 auto, 0 off, 2 always): when x is wider
// than a quarter of L2, the leaf reads x through a dense renumbering of the
// referenced columns (crdc / cref, built once per pattern, cached on the
// tensor) and a per-call packed copy xc, so the x gathers hit an L2-resident
// array and the crd stream is int32.  Same positions, same order, same x
// values: the sums are unchanged.  < 2^31 columns; for a piece the index
// covers the piece's positions (its referenced columns only).
static int xc_mode() {
  static int v = [] {
    const char* e = getenv("SPD_XC");
    return e ? atoi(e) : 1;
  }();
  return v;
}

static bool xc_wanted(spd_context* ctx, const spd_tensor* B, int64_t ncols) {
  const int m = xc_mode();
  if (m == 0 || ncols >= (int64_t(1) << 31)) return false;
  if (m == 2) return true;
  int l2 = 0;
  SPD_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
  return ncols * 8 > l2 / 4;
}

static void xc_index(spd_context* ctx, spd_tensor* t, int64_t ncols) {
  if (t->nref >= 0) return;
  const spd_level_store& L = t->levels.back();
  const int64_t lo = t->piece ? t->piece_lo : 0;
  const int64_t nnz = t->piece ? t->piece_hi - t->piece_lo + 1 : L.positions;
  cudaStream_t s = ctx->stream;
  const unsigned gc = (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(ncols, 256), 1), ctx->num_sms * 16);
  const unsigned gq = (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(nnz, 256), 1), ctx->num_sms * 16);
  int32_t *counts = nullptr, *flags = nullptr, *rank = nullptr;
  const size_t cb = sizeof(int32_t) * (ncols > 0 ? ncols : 1);
  SPD_CUDA(cudaMallocAsync((void**)&counts, cb, s));
  SPD_CUDA(cudaMallocAsync((void**)&flags, cb, s));
  SPD_CUDA(cudaMallocAsync((void**)&rank, cb, s));
  SPD_CUDA(cudaMemsetAsync(counts, 0, cb, s));
  SPD_CUDA(cudaMallocAsync((void**)&t->crdc_alloc, sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
  t->crdc = t->crdc_alloc - lo;  // indexed by global position
  int64_t nref = 0;
  if (nnz > 0 && ncols > 0) {
    k_col_count<<<gq, 256, 0, s>>>(L.crd + lo, nnz, counts);
    SPD_CHECK_LAUNCH();
    k_ref_flags<<<gc, 256, 0, s>>>(counts, ncols, flags);
    SPD_CHECK_LAUNCH();
    size_t bytes = 0;
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags, rank, ncols, s));
    void* tmp = ctx->scratch[5].reserve(bytes);
    SPD_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, flags, rank, ncols, s));
    int32_t last[2] = {0, 0};
    SPD_CUDA(cudaMemcpyAsync(&last[0], rank + ncols - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaMemcpyAsync(&last[1], flags + ncols - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    nref = (int64_t)last[0] + last[1];
    SPD_CUDA(cudaMallocAsync((void**)&t->cref, sizeof(int32_t) * (nref > 0 ? nref : 1), s));
    k_ref_list<<<gc, 256, 0, s>>>(flags, rank, ncols, t->cref);
    SPD_CHECK_LAUNCH();
    k_crd_rank<<<gq, 256, 0, s>>>(L.crd + lo, nnz, rank, t->crdc_alloc);
    SPD_CHECK_LAUNCH();
    ctx->launches += 4;
  } else {
    SPD_CUDA(cudaMallocAsync((void**)&t->cref, sizeof(int32_t), s));
  }
  cudaFreeAsync(counts, s);
  cudaFreeAsync(flags, s);
  cudaFreeAsync(rank, s);
  t->nref = nref;
}

// SDDMM over the compacted view (called by sddmm.cu): K = 128, D j-major.
bool sddmm_nz_launch(spd_context* ctx, const spd_tensor* B, const WalkGeom& g, const double* C,
                     const double* D, int64_t K, int64_t dk, int64_t dj, double* Avals,
                     const int64_t* counters) {
  if ((K != 32 && K != 64 && K != 128 && K != 256) || dk != 1 || dj != K ||
      B->dims[1] >= (int64_t(1) << 31))
    return false;
  NzView z = nz_view(ctx, const_cast<spd_tensor*>(B), g.R, g.nrows);
  const int32_t* h = hot_crd(ctx, const_cast<spd_tensor*>(B), K * 8);
  static int minb = [] {
    const char* e = getenv("SPD_SDDMM_MINB");
    return e ? atoi(e) : 3;
  }();
  if (K == 32) {
    static int grid = 0;
    if (!grid) grid = occupancy_grid(ctx, k_sddmm_nz<1, 4>);
    k_sddmm_nz<1, 4><<<grid, kBlock, 0, ctx->stream>>>(g, z, h, B->vals, C, D, K, Avals, counters);
  } else if (K == 64) {
    static int grid = 0;
    if (!grid) grid = occupancy_grid(ctx, k_sddmm_nz<2, 4>);
    k_sddmm_nz<2, 4><<<grid, kBlock, 0, ctx->stream>>>(g, z, h, B->vals, C, D, K, Avals, counters);
  } else if (K == 256) {
    static int grid = 0;
    if (!grid) grid = occupancy_grid(ctx, k_sddmm_nz<8, 2>);
    k_sddmm_nz<8, 2><<<grid, kBlock, 0, ctx->stream>>>(g, z, h, B->vals, C, D, K, Avals, counters);
  } else if (minb == 4) {
    static int grid = 0;
    if (!grid) grid = occupancy_grid(ctx, k_sddmm_nz<4, 4>);
    k_sddmm_nz<4, 4><<<grid, kBlock, 0, ctx->stream>>>(g, z, h, B->vals, C, D, K, Avals, counters);
  } else {
    static int grid = 0;
    if (!grid) grid = occupancy_grid(ctx, k_sddmm_nz<4, 3>);
    k_sddmm_nz<4, 3><<<grid, kBlock, 0, ctx->stream>>>(g, z, h, B->vals, C, D, K, Avals, counters);
  }
  SPD_CHECK_LAUNCH();
  return true;
}

// int32 copy of the leaf crd (cached on t, rebuilt after a restage): the
// N = 32 SpMM leaf streams 4-byte columns and forms addresses with one
// 32x32->64-bit multiply-add.  Indexed by global position (offset for a piece).
static const int32_t* crd32_index(spd_context* ctx, spd_tensor* t) {
  if (t->crd32) return t->crd32;
  const spd_level_store& L = t->levels.back();
  const int64_t lo = t->piece ? t->piece_lo : 0;
  const int64_t nnz = t->piece ? t->piece_hi - t->piece_lo + 1 : L.positions;
  cudaStream_t s = ctx->stream;
  if (!t->crd32_alloc || t->crd32_cap < nnz) {
    if (t->crd32_alloc) cudaFreeAsync(t->crd32_alloc, s);
    SPD_CUDA(cudaMallocAsync((void**)&t->crd32_alloc, sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
    t->crd32_cap = nnz;
  }
  if (nnz > 0) {
    k_crd_to_i32<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), ctx->num_sms * 16), 256, 0, s>>>(L.crd + lo, nnz,
                                                                                                   t->crd32_alloc);
    SPD_CHECK_LAUNCH();
    ctx->launches++;
  }
  t->crd32 = t->crd32_alloc - lo;
  return t->crd32;
}

static void run_rowwalk(spd_context* ctx, const OpArgs& a, int64_t first, int64_t count,
                        spd_stats* stats) {
  HostTrace ht("rowwalk");
  checked(ctx);
  const spd_tensor* B = a.B;
  if (!B) throw ValidationError("null tensor");
  settle_restage(B);
  require_partition(ctx, B, first, count, true);
  activate(ctx);
  const int nl = (int)B->levels.size();
  const bool csf = a.op == Op::SpTTV || a.op == Op::SpMTTKRP;
  if (csf) {
    // dss (the paper's Dense-outer CSF) or sss (every level compressed)
    const bool top_ok = (B->levels[0].kind == SPD_DENSE && B->levels[0].dom.size() == 1) ||
                        (B->levels[0].kind == SPD_COMPRESSED && B->levels[0].parent_positions == 1);
    if (nl != 3 || !top_ok || B->levels[1].kind != SPD_COMPRESSED || B->levels[2].kind != SPD_COMPRESSED ||
        B->groups[0].size() != 1 || B->groups[1].size() != 1 || B->groups[2].size() != 1)
      throw ValidationError("unsupported on gpu: this kernel needs a dss or sss 3-tensor (CSF)");
  } else if (nl != 2 || B->levels[0].kind != SPD_DENSE || B->levels[1].kind != SPD_COMPRESSED ||
             B->levels[0].dom.size() != 1) {
    throw ValidationError("unsupported on gpu: this kernel needs a ds (CSR-like) matrix");
  }
  require_identity_order(B, csf ? "the CSF operand" : "the sparse operand");
  if (ctx->split == SplitKind::NonZero && ctx->split_level != nl - 1)
    throw ValidationError("unsupported on gpu: nonzero split must be on the leaf level");
  if (a.W < 0 || a.W > 128) throw ValidationError("unsupported on gpu: inner extent must be in [0, 128]");
  const int64_t P = ctx->pieces;
  const int64_t nnz = B->levels[nl - 1].positions;

  WalkGeom g;
  int out_level = 0;
  switch (a.op) {
    case Op::SpMV:
    case Op::SpMM:
      g.R = B->levels[1].rowptr;
      g.nrows = B->levels[1].parent_positions;
      break;
    case Op::SpTTV:
      g.R = B->levels[2].rowptr;
      g.nrows = B->levels[2].parent_positions;
      out_level = 1;
      break;
    case Op::SpMTTKRP: {
      const bool sparse_top = B->levels[0].kind == SPD_COMPRESSED;
      const int64_t I = sparse_top ? B->dims[B->mode_order[0]] : B->levels[1].parent_positions;
      spd_tensor* Bm = const_cast<spd_tensor*>(B);
      if (!Bm->leaf_rowptr) {
        SPD_CUDA(cudaMallocAsync((void**)&Bm->leaf_rowptr, sizeof(int64_t) * (I + 1), ctx->stream));
        const unsigned gr = (unsigned)std::min<int64_t>(ceil_div(I + 1, 256), 4096);
        if (sparse_top)
          k_leaf_rowptr_sparse_top<<<gr, 256, 0, ctx->stream>>>(B->levels[0].crd, B->levels[0].positions,
                                                                B->levels[1].rowptr, B->levels[2].rowptr, I,
                                                                Bm->leaf_rowptr);
        else
          k_leaf_rowptr<<<gr, 256, 0, ctx->stream>>>(B->levels[1].rowptr, B->levels[2].rowptr, I,
                                                     Bm->leaf_rowptr);
        SPD_CHECK_LAUNCH();
      }
      g.R = B->leaf_rowptr;
      g.nrows = I;
      break;
    }
  }
  g.cols = (const DevColor*)ctx->colors_dev.ptr;
  g.c_first = first;
  g.c_count = count;
  g.W = a.W;
  // Positions per chunk: ~256 KB of operand traffic per warp-chunk for the
  // column kernels, 2048 positions for the scalar ones.
  // (the lane-per-row SpMV kernel balances small problems better with 1024)
  // SpTTV over CSF fibres (~1.5 positions per fibre on C4): 512-position
  // chunks and 6 CTAs/SM (0.190 -> 0.160 ms, profiles/README.md)
  g.CH = (a.op == Op::SpMV || a.op == Op::SpTTV) ? (nnz < (int64_t(1) << 26) ? 1024 : 2048) : 1024;
  if (a.op == Op::SpTTV && nnz < (int64_t(1) << 26)) g.CH = 512;
  {
    static int64_t ch_override = [] {
      const char* e = getenv("SPD_CH");
      return e ? atoll(e) : 0;
    }();
    if (ch_override >= 32 && (a.op == Op::SpMM || a.op == Op::SpMTTKRP)) g.CH = ch_override;
    static int64_t ch_spmv = [] {
      const char* e = getenv("SPD_CH_SPMV");
      return e ? atoll(e) : 0;
    }();
    if (ch_spmv >= 32 && (a.op == Op::SpMV || a.op == Op::SpTTV)) g.CH = ch_spmv;
  }
  const bool spmm32 = a.op == Op::SpMM && a.W == 32 && B->dims[1] < (int64_t(1) << 31) && g.nrows < (int64_t(1) << 31);
  const bool spmmv = a.op == Op::SpMM && (a.W == 8 || a.W == 16 || a.W == 64 || a.W == 128) &&
                     B->dims[1] < (int64_t(1) << 31);
  const int64_t W = a.W > 0 ? a.W : 1;
  const int64_t max_chunks = nnz / g.CH + 2 * P + 2;

  ChunkRecs rec;
  rec.row = (int64_t*)ctx->scratch[0].reserve(sizeof(int64_t) * 2 * max_chunks);
  rec.cont = (int*)ctx->scratch[1].reserve(sizeof(int) * max_chunks);
  rec.val = (double*)ctx->scratch[2].reserve(sizeof(double) * 2 * max_chunks * W);
  ColorRecs col;
  // colour blocks per GPU (require_partition): with the even blocks rank r's
  // head records sit at slots [r * cmax, r * cmax + cmax), so one all-gather
  // of cmax slots per rank lays every colour's record at its own slot; with
  // uneven blocks (spd_context_set_colour_blocks) the all-gather goes to a
  // staging area of cmax = the largest block per rank and k_unpack_heads
  // moves each record to its colour's slot
  const bool cross_gpu = ctx->comm && ctx->world > 1 && P > 1 && ctx->split != SplitKind::Universe &&
                         !(first == 0 && count == P);
  const bool even = !cross_gpu || even_blocks(ctx);
  int64_t cmax = 1;
  if (cross_gpu)
    for (int r = 0; r < ctx->world; r++) {
      int64_t f, c;
      colour_block(ctx, r, f, c);
      cmax = std::max(cmax, c);
    }
  // even: every rank's window inside P rounded up; uneven: a short block's
  // window may run past its colours (the extra slots are ignored)
  const int64_t pack_slots = cross_gpu ? (even ? cmax * ctx->world : P + cmax) : P;
  col.head_pack = (int64_t*)ctx->scratch[3].reserve(sizeof(int64_t) * pack_slots * (W + 2));
  char* cr = (char*)ctx->scratch[4].reserve(sizeof(int64_t) * (P + 4) + sizeof(double) * P * W);
  col.counters = (int64_t*)cr;
  col.tail_row = col.counters + 4;
  col.tail_val = (double*)(col.tail_row + P);

  cudaStream_t s = ctx->stream;
  int64_t launches = 0;
  if (stats) SPD_CUDA(cudaEventRecord(ctx->ev0, s));
  trace_mark(ctx);
  ht.mark("scratch");
  launch_setup(s, (DevColor*)ctx->colors_dev.ptr, P, (int)ctx->split, out_level, g.R, g.nrows, g.CH, first, count,
               col.counters, col.head_pack, pack_slots * (W + 2), col.tail_row, P);
  launches += 2;

  const spd_level_store& leaf = B->levels[nl - 1];
  const bool mttkrp32 = a.op == Op::SpMTTKRP && a.W == 32 && B->dims[1] < (int64_t(1) << 31) &&
                        B->dims[2] < (int64_t(1) << 31);
  const bool mttkrpv = a.op == Op::SpMTTKRP && (a.W == 8 || a.W == 16 || a.W == 64 || a.W == 128) &&
                       B->dims[1] < (int64_t(1) << 31) && B->dims[2] < (int64_t(1) << 31);
  // the compacted-row walks cover SpMV / SpTTV and the widths with a
  // specialised leaf; other widths use the lane-per-column walks
  const bool use_nz = a.op == Op::SpMV || a.op == Op::SpTTV || mttkrp32 || mttkrpv || spmm32 || spmmv;
  NzView z{nullptr, nullptr, 0, nullptr};
  bool zero_joined = false;
  if (use_nz) {
    z = nz_view(ctx, const_cast<spd_tensor*>(B), g.R, g.nrows, a.op == Op::SpMV || a.op == Op::SpTTV);
    ht.mark("nz_view");
    // SpMV/SpTTV walks zero the empty rows between consecutive non-empty
    // rows themselves (8 bytes each); the W-wide outputs use this pass.
    if (a.op == Op::SpMM || a.op == Op::SpMTTKRP) {
      static int zgrid = 0;
      if (!zgrid) zgrid = occupancy_grid(ctx, k_zero_empty);
      // zero-fill CTAs on the aux stream, concurrent with the leaf (its
      // late-starting CTAs just draw the remaining chunk tickets): 4 per SM
      // measured best (step 6.05 -> 5.95 ms, profiles/README.md);
      // SPD_ZCONC=0 runs the pass before the leaf instead.
      static int zconc = [ctx] {
        const char* e = getenv("SPD_ZCONC");
        return e ? atoi(e) : 4 * ctx->num_sms;
      }();
      trace_mark(ctx);
      if (zconc > 0 && ctx->aux) {
        SPD_CUDA(cudaEventRecord(ctx->fork, s));
        SPD_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->fork, 0));
        k_zero_empty<<<zconc, kBlock, 0, ctx->aux>>>(g.R, g.nrows, (const DevColor*)ctx->colors_dev.ptr, first,
                                                    count, a.W, a.out);
        SPD_CUDA(cudaEventRecord(ctx->join, ctx->aux));
        zero_joined = true;
      } else {
        k_zero_empty<<<zgrid, kBlock, 0, s>>>(g.R, g.nrows, (const DevColor*)ctx->colors_dev.ptr, first, count,
                                             a.W, a.out);
      }
      SPD_CHECK_LAUNCH();
      launches++;
    }
  }
  trace_mark(ctx);
  leaf_timing_begin(ctx);
  if (use_nz) {
    if (a.op == Op::SpMTTKRP) {
      spd_tensor* Bm = const_cast<spd_tensor*>(B);
      const spd_level_store& L1 = B->levels[1];
      const spd_level_store& L2 = B->levels[2];
      if (!Bm->jleaf) {
        SPD_CUDA(cudaMallocAsync((void**)&Bm->jleaf, sizeof(int32_t) * (L2.positions > 0 ? L2.positions : 1), s));
        k_jleaf<<<(unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(L2.parent_positions, 256), 1),
                                               ctx->num_sms * 16), 256, 0, s>>>(L2.rowptr, L1.crd, L2.parent_positions,
                                                                               Bm->jleaf);
        SPD_CHECK_LAUNCH();
        ctx->launches++;
      }
      if (mttkrpv) {  // R in {8, 16, 64, 128}
        switch (a.W) {
#define SPD_MTV(NN, UU, MB)                                                                              \
  case NN: {                                                                                             \
    static int grid = 0;                                                                                 \
    if (!grid) grid = occupancy_grid(ctx, k_spmm_nzv<NN, UU, MB, true>);                                \
    k_spmm_nzv<NN, UU, MB, true><<<grid, kBlock, 0, s>>>(g, z, leaf.crd, B->vals, a.D, a.out, rec,     \
                                                          col.counters, B->jleaf, a.x);                  \
    break;                                                                                               \
  }
          SPD_MTV(8, 4, 3)
          SPD_MTV(16, 4, 3)
          SPD_MTV(64, 4, 3)
          SPD_MTV(128, 2, 3)
#undef SPD_MTV
        }
      } else {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_mttkrp32_nz<4, 3, false>);
        k_mttkrp32_nz<4, 3, false><<<grid, kBlock, 0, s>>>(g, z, leaf.crd, B->jleaf, a.x, B->vals, a.D, a.out,
                                                           rec, col.counters);
      }
    } else if (spmmv) {  // N in {8, 16, 64, 128}
      switch (a.W) {
#define SPD_SPMMV(NN, UU, MB)                                                                        \
  case NN: {                                                                                         \
    static int grid = 0;                                                                             \
    if (!grid) grid = occupancy_grid(ctx, k_spmm_nzv<NN, UU, MB>);                                  \
    k_spmm_nzv<NN, UU, MB><<<grid, kBlock, 0, s>>>(g, z, leaf.crd, B->vals, a.x, a.out, rec, col.counters); \
    break;                                                                                           \
  }
        SPD_SPMMV(8, 4, 4)
        SPD_SPMMV(16, 4, 4)
        SPD_SPMMV(64, 4, 4)
        SPD_SPMMV(128, 2, 4)
#undef SPD_SPMMV
      }
    } else if (a.op == Op::SpMM) {  // N == 32 (C2): cp.async ring of 4 slots, 3 CTAs / SM
      const int32_t* c32 = crd32_index(ctx, const_cast<spd_tensor*>(B));
      constexpr int kS = 4, kMinB = 3;
      const int smem = (kBlock / 32) * kS * 8 * 16 * (int)sizeof(double2);
      // the dynamic shared-memory opt-in is a per-device function attribute:
      // set once on every device a context of this process uses (the
      // drop-in runs one host thread per GPU)
      static std::mutex attr_mu;
      static uint64_t attr_done = 0;
      static int grid = 0;
      {
        std::lock_guard<std::mutex> lk(attr_mu);
        const uint64_t bit = uint64_t(1) << (ctx->device & 63);
        if (!(attr_done & bit)) {
          SPD_CUDA(cudaFuncSetAttribute(k_spmm32_nz<kS, kMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          int per_sm = 0;
          SPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmm32_nz<kS, kMinB>, kBlock, smem));
          grid = ctx->num_sms * (per_sm > 0 ? per_sm : 1);
          attr_done |= bit;
        }
      }
      k_spmm32_nz<kS, kMinB><<<grid, kBlock, smem, s>>>(g, z, c32, B->vals, a.x, a.out, rec, col.counters);
    } else {  // SpMV / SpTTV: the windowed row reduction
      // 6 CTAs/SM win on large matrices and CSF fibres, 4 on small ones (C1)
      static int minb_env = [] {
        const char* e = getenv("SPD_SPMV_MINB");
        return e ? atoi(e) : 0;
      }();
      const int minb = minb_env ? minb_env : (nnz >= (int64_t(1) << 26) || a.op == Op::SpTTV ? 6 : 4);
      const int64_t ncols = B->dims[B->mode_order[B->groups.back()[0]]];
      const int32_t* c32 = nullptr;  // compacted columns (SpMV over a wide x)
      const double* xv = a.x;
      if (a.op == Op::SpMV && xc_wanted(ctx, B, ncols)) {  // compacted x, int32 crd
        spd_tensor* Bm = const_cast<spd_tensor*>(B);
        xc_index(ctx, Bm, ncols);
        double* xc = (double*)ctx->scratch[7].reserve(sizeof(double) * (Bm->nref > 0 ? Bm->nref : 1));
        if (Bm->nref > 0) {
          k_gather_ref<<<(unsigned)std::min<int64_t>(ceil_div(Bm->nref, 256), ctx->num_sms * 16), 256, 0, s>>>(
              a.x, Bm->cref, Bm->nref, xc);
          SPD_CHECK_LAUNCH();
          launches++;
        }
        c32 = Bm->crdc;
        xv = xc;
      } else if (ncols < (int64_t(1) << 31)) {
        // int32 columns (built once per pattern, like the SpMM leaf's): 4 of
        // the 16 bytes a position streams (SpTTV 0.120 -> 0.117 ms)
        c32 = crd32_index(ctx, const_cast<spd_tensor*>(B));
      }
#define SPD_LEAF(KERN, CI, CRD)                                                                         \
  do {                                                                                                  \
    static int gr = 0;                                                                                  \
    if (!gr) gr = occupancy_grid(ctx, KERN);                                                            \
    KERN<<<gr, kBlock, 0, s>>>(g, z, (const CI*)(CRD), B->vals, xv, a.out, rec, col.counters);          \
  } while (0)
      if (c32) {
        if (minb == 6) SPD_LEAF((k_spmv_win<6, int32_t>), int32_t, c32);
        else SPD_LEAF((k_spmv_win<4, int32_t>), int32_t, c32);
      } else {
        if (minb == 6) SPD_LEAF((k_spmv_win<6, int64_t>), int64_t, leaf.crd);
        else SPD_LEAF((k_spmv_win<4, int64_t>), int64_t, leaf.crd);
      }
#undef SPD_LEAF
    }
  } else
  switch (a.op) {  // SpMM at other widths, SpMTTKRP at other ranks
    case Op::SpMM: {
      if (a.W <= 32) {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_spmm_walk<1>);
        k_spmm_walk<1><<<grid, kBlock, 0, s>>>(g, leaf.crd, B->vals, a.x, a.out, rec, col.counters);
      } else if (a.W <= 64) {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_spmm_walk<2>);
        k_spmm_walk<2><<<grid, kBlock, 0, s>>>(g, leaf.crd, B->vals, a.x, a.out, rec, col.counters);
      } else {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_spmm_walk<4>);
        k_spmm_walk<4><<<grid, kBlock, 0, s>>>(g, leaf.crd, B->vals, a.x, a.out, rec, col.counters);
      }
      break;
    }
    case Op::SpMTTKRP: {
      const spd_level_store& L1 = B->levels[1];
      const spd_level_store& L2 = B->levels[2];
      if (a.W <= 32) {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_mttkrp_walk<1>);
        k_mttkrp_walk<1><<<grid, kBlock, 0, s>>>(g, L2.rowptr, L2.parent_positions, L1.crd,
                                                 L2.crd, B->vals, a.x, a.D, a.out, rec,
                                                 col.counters);
      } else if (a.W <= 64) {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_mttkrp_walk<2>);
        k_mttkrp_walk<2><<<grid, kBlock, 0, s>>>(g, L2.rowptr, L2.parent_positions, L1.crd,
                                                 L2.crd, B->vals, a.x, a.D, a.out, rec,
                                                 col.counters);
      } else {
        static int grid = 0;
        if (!grid) grid = occupancy_grid(ctx, k_mttkrp_walk<4>);
        k_mttkrp_walk<4><<<grid, kBlock, 0, s>>>(g, L2.rowptr, L2.parent_positions, L1.crd,
                                                 L2.crd, B->vals, a.x, a.D, a.out, rec,
                                                 col.counters);
      }
      break;
    }
  }
  SPD_CHECK_LAUNCH();
  ht.mark("leaf launch");
  leaf_timing_end(ctx);
  if (zero_joined) SPD_CUDA(cudaStreamWaitEvent(s, ctx->join, 0));
  trace_mark(ctx);
  launches++;
  {
    static int grid = 0;
    if (!grid) grid = occupancy_grid(ctx, k_chunk_fixup);
    const int vec2 = W % 2 == 0 && reinterpret_cast<uintptr_t>(a.out) % 16 == 0;
    k_chunk_fixup<<<grid, kBlock, 0, s>>>(g, rec, col, a.out, vec2);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  trace_mark(ctx);
  if (cross_gpu && even) {  // rows cut between GPUs: every colour's head record to every GPU
    const size_t bytes = sizeof(int64_t) * cmax * (W + 2);
    SPD_NCCL(ncclAllGather(col.head_pack + first * (W + 2), col.head_pack, bytes, ncclUint8, ctx->comm, s));
  } else if (cross_gpu) {
    const size_t bytes = sizeof(int64_t) * cmax * (W + 2);
    int64_t* stage = (int64_t*)ctx->scratch[6].reserve(bytes * ctx->world);
    SPD_NCCL(ncclAllGather(col.head_pack + first * (W + 2), stage, bytes, ncclUint8, ctx->comm, s));
    const int64_t words = cmax * ctx->world * (W + 2);
    k_unpack_heads<<<(unsigned)std::min<int64_t>(ceil_div(words, 256), 1024), 256, 0, s>>>(
        stage, (const int64_t*)ctx->blocks_dev.ptr, ctx->world, ctx->rank, cmax, W + 2, col.head_pack);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  trace_mark(ctx);
  k_colour_combine<<<(unsigned)ceil_div(P * 32, 256), 256, 0, s>>>(
      col, (const DevColor*)ctx->colors_dev.ptr, P, W, first, count, a.out);
  SPD_CHECK_LAUNCH();
  trace_mark(ctx);
  launches++;
  ctx->launches += launches;
  ht.mark("tail launches");
  if (stats) {
    SPD_CUDA(cudaEventRecord(ctx->ev1, s));
    SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters, col.counters, sizeof(int64_t) * 4,
                             cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    const auto& hc = host_colors(ctx);
    std::vector<int64_t> work(P);
    const int64_t inner = a.op == Op::SpMV || a.op == Op::SpTTV ? 1 : a.W;
    for (int64_t c = 0; c < P; c++)
      work[c] = hc[c].q.lo <= hc[c].q.hi ? (hc[c].q.hi - hc[c].q.lo + 1) * inner : 0;
    fill_stats(ctx, stats, ctx->pinned_counters[0], work, launches, true);
  }
}

}  // namespace spd

using namespace spd;

extern "C" {

int spd_spmv(spd_context* ctx, const spd_tensor* B, const double* c_dev, double* a_dev,
             int64_t first_color, int64_t ncolors, spd_stats* stats) {
  return guarded([&] {
    run_rowwalk(ctx, OpArgs{Op::SpMV, B, c_dev, nullptr, 1, a_dev}, first_color, ncolors, stats);
  });
}

int spd_spmm(spd_context* ctx, const spd_tensor* B, const double* C_dev, int64_t N,
             double* A_dev, int64_t first_color, int64_t ncolors, spd_stats* stats) {
  return guarded([&] {
    run_rowwalk(ctx, OpArgs{Op::SpMM, B, C_dev, nullptr, N, A_dev}, first_color, ncolors, stats);
  });
}

int spd_spttv(spd_context* ctx, const spd_tensor* B, const double* c_dev, double* Avals_dev,
              int64_t first_color, int64_t ncolors, spd_stats* stats) {
  return guarded([&] {
    run_rowwalk(ctx, OpArgs{Op::SpTTV, B, c_dev, nullptr, 1, Avals_dev}, first_color, ncolors,
                stats);
  });
}

int spd_spmttkrp(spd_context* ctx, const spd_tensor* B, const double* C_dev,
                 const double* D_dev, int64_t R, double* A_dev, int64_t first_color,
                 int64_t ncolors, spd_stats* stats) {
  return guarded([&] {
    run_rowwalk(ctx, OpArgs{Op::SpMTTKRP, B, C_dev, D_dev, R, A_dev}, first_color, ncolors,
                stats);
  });
}


int spd_colour_costs(spd_context* ctx, const spd_tensor* t, int64_t* positions, int64_t* rows,
                     int64_t* nonempty) {
  return guarded([&] {
    checked(ctx);
    if (!t || !positions || !rows || !nonempty) throw ValidationError("null argument");
    settle_restage(t);
    if (ctx->split == SplitKind::None || ctx->split_tensor != t)
      throw ValidationError("no partition of this tensor on the context: call spd_partition_* first");
    if (t->levels.size() != 2 || t->levels[0].kind != SPD_DENSE || t->levels[1].kind != SPD_COMPRESSED)
      throw ValidationError("colour costs: a ds (CSR-like) matrix");
    activate(ctx);
    cudaStream_t s = ctx->stream;
    const int64_t P = ctx->pieces;
    const spd_level_store& L = t->levels[1];
    int64_t* cnt = (int64_t*)ctx->scratch[6].reserve(sizeof(int64_t) * (P + 4));
    // W_c as the row-reducing ops store them, then the non-empty rows in W_c
    launch_setup(s, (DevColor*)ctx->colors_dev.ptr, P, (int)ctx->split, 0, L.rowptr, L.parent_positions, 1024, 0,
                 P, cnt + P, nullptr, 0, nullptr, 0);
    NzView z = nz_view(ctx, const_cast<spd_tensor*>(t), L.rowptr, L.parent_positions);
    k_colour_nonempty<<<(unsigned)ceil_div(P * 32, 256), 256, 0, s>>>((const DevColor*)ctx->colors_dev.ptr, P, z,
                                                                     cnt);
    SPD_CHECK_LAUNCH();
    std::vector<DevColor> d(P);
    SPD_CUDA(cudaMemcpyAsync(d.data(), ctx->colors_dev.ptr, sizeof(DevColor) * P, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaMemcpyAsync(nonempty, cnt, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    for (int64_t c = 0; c < P; c++) {
      positions[c] = d[c].pub.q.lo <= d[c].pub.q.hi ? d[c].pub.q.hi - d[c].pub.q.lo + 1 : 0;
      rows[c] = d[c].w_lo <= d[c].w_hi ? d[c].w_hi - d[c].w_lo + 1 : 0;
    }
  });
}

}  // extern "C"
