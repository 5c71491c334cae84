// Leaf kernels over the compacted non-empty-row view (included by leaf_rows.cu).
//
// A compressed level of a power-law matrix is mostly empty rows (58% of the
// R-MAT scale-24 rows).  Walking `rowptr` directly puts a dependent row-pointer
// load on every warp's critical path at every row end.  Instead each tensor
// lazily builds, once, the compacted view of its non-empty rows -- `nzp`
// (their start positions, strictly increasing, m+1 entries) and `nzid` (their
// row ids) -- a DCSR-style auxiliary index.  A warp walking a chunk keeps 64
// consecutive entries of both in registers (two 32-lane blocks), so the row
// starts inside a 32-position window are one ballot-like OR away, and the next
// block is loaded ~20 windows before it is needed.  Empty rows of the dense
// output are zeroed by a separate coalesced pass (k_zero_empty) over the
// colours' write ranges, so the walks never touch them.
#pragma once

#include "rowwalk.cuh"

namespace spd {

#ifndef FULL
#define FULL 0xffffffffu
#endif

struct NzView {
  const int64_t* __restrict__ ptr;  // m + 1 starts
  const int64_t* __restrict__ id;   // m row ids
  int64_t m;
};

// Register-resident window of 64 compacted rows [cb, cb + 64).
struct NzCursor {
  int64_t cb, ic;  // block base, current compacted row
  int64_t P0, P1;  // starts of rows cb + lane, cb + 32 + lane
  int64_t I0, I1;  // ids of the same rows
};

__device__ __forceinline__ void nz_load(const NzView& z, int64_t j0, int64_t& P, int64_t& I) {
  const int64_t j = j0 + lane_id();
  P = j <= z.m ? ld64(z.ptr + j) : INT64_MAX;
  I = j < z.m ? ld64(z.id + j) : -1;
}

__device__ __forceinline__ void nz_start(const NzView& z, NzCursor& c, int64_t s) {
  c.ic = warp_owner(z.ptr, z.m, s);  // compacted row containing position s
  c.cb = c.ic;
  nz_load(z, c.cb, c.P0, c.I0);
  nz_load(z, c.cb + 32, c.P1, c.I1);
}

// Value of row (cb + idx) from a (v0, v1) block pair, idx in [0, 64); may
// differ per lane.
__device__ __forceinline__ int64_t nz_get(int64_t v0, int64_t v1, int idx) {
  const int64_t a = __shfl_sync(FULL, v0, idx & 31);
  const int64_t b = __shfl_sync(FULL, v1, idx & 31);
  return idx < 32 ? a : b;
}

__device__ __noinline__ void nz_slide(const NzView& z, NzCursor& c) {
  while (c.ic - c.cb >= 32) {  // slide the register window; the new block is far ahead
    c.cb += 32;
    c.P0 = c.P1;
    c.I0 = c.I1;
    nz_load(z, c.cb + 32, c.P1, c.I1);
  }
}

__device__ __forceinline__ void nz_advance(const NzView& z, NzCursor& c, int64_t by) {
  c.ic += by;
  if (c.ic - c.cb >= 32) nz_slide(z, c);
}

// Offsets in [base, last] where a row after the current one starts.
__device__ __forceinline__ unsigned nz_window_mask(const NzCursor& c, int64_t base, int64_t last) {
  const int lane = lane_id();
  const int64_t j0 = c.cb + lane;
  unsigned b0 = (j0 > c.ic && c.P0 >= base && c.P0 <= last) ? 1u << (int)(c.P0 - base) : 0u;
  unsigned bm = __reduce_or_sync(FULL, b0);
  if (__shfl_sync(FULL, c.P0, 31) <= last) {
    const int64_t j1 = j0 + 32;
    unsigned b1 = (j1 > c.ic && c.P1 >= base && c.P1 <= last) ? 1u << (int)(c.P1 - base) : 0u;
    bm |= __reduce_or_sync(FULL, b1);
  }
  return bm;
}

// Zeroes the empty rows of the union of the write ranges of colours
// [c_first, c_first + c_count): one warp per 32 rows, one coalesced W-wide
// store per empty row.
__global__ void __launch_bounds__(kBlock) k_zero_empty(const int64_t* __restrict__ R, int64_t nrows,
                                                       const DevColor* __restrict__ cols, int64_t c_first,
                                                       int64_t c_count, int64_t W, double* __restrict__ out) {
  const int lane = lane_id();
  int64_t lo = INT64_MAX, hi = -1;
  for (int64_t c = c_first; c < c_first + c_count; c++) {
    if (cols[c].w_lo <= cols[c].w_hi) {
      lo = min(lo, cols[c].w_lo);
      hi = max(hi, cols[c].w_hi);
    }
  }
  if (lo > hi) return;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g0 = lo + gw * 32; g0 <= hi; g0 += nw * 32) {
    const int64_t r = g0 + lane;
    const bool empty = r <= hi && ld64(R + r + 1) == ld64(R + r);
    if (W == 1) {
      if (empty) out[r] = 0.0;
      continue;
    }
    unsigned m = __ballot_sync(FULL, empty);
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      double* row = out + (g0 + b) * W;
      for (int64_t j = lane; j < W; j += 32) row[j] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// SpMV / SpTTV over the compacted view: lane = position, 32-position windows
// (kSpmvBatch of them loaded together), per window one segmented scan; the
// rows completing in a window are handled one per lane: lane t finds the end
// of row ic+t with __fns on the head mask.
__global__ void __launch_bounds__(kBlock) k_spmv_nz(WalkGeom g, NzView z, const int64_t* __restrict__ crd,
                                                    const double* __restrict__ vals,
                                                    const double* __restrict__ x, double* __restrict__ y,
                                                    ChunkRecs rec, const int64_t* __restrict__ counters) {
  const int lane = lane_id();
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_stream = l2_policy_evict_first();
  for (int64_t v = begin + gw; v < end; v += nw) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) {
      if (lane == 0) rec.row[2 * ci.local] = -1, rec.row[2 * ci.local + 1] = -1, rec.cont[ci.local] = 0;
      continue;
    }
    const int64_t k = ci.local, s = ci.s, e = ci.e;
    NzCursor c;
    nz_start(z, c, s);
    bool head = __shfl_sync(FULL, c.P0, 0) < s;
    int64_t head_row = -1;
    int head_cont = 0;
    double head_val = 0.0, acc = 0.0;
    for (int64_t bbase = s; bbase <= e; bbase += 32 * kSpmvBatch) {
      int64_t kk[kSpmvBatch];
      double vv[kSpmvBatch], prods[kSpmvBatch];
#pragma unroll
      for (int bi = 0; bi < kSpmvBatch; bi++) {
        const int64_t q = bbase + 32 * bi + lane;
        kk[bi] = 0;
        vv[bi] = 0.0;
        if (q <= e) {
          kk[bi] = ld_i64_hint(crd + q, pol_stream);
          vv[bi] = ld_f64_hint(vals + q, pol_stream);
        }
      }
#pragma unroll
      for (int bi = 0; bi < kSpmvBatch; bi++) {
        const int64_t q = bbase + 32 * bi + lane;
        prods[bi] = q <= e ? vv[bi] * __ldg(x + kk[bi]) : 0.0;
      }
#pragma unroll
      for (int bi = 0; bi < kSpmvBatch; bi++) {
        const int64_t base = bbase + 32 * bi;
        if (base > e) break;
        const int64_t last = min(base + 31, e);
        const int cnt = (int)(last - base + 1);
        const unsigned heads = nz_window_mask(c, base, last);
        if (heads == 0u) {
          acc += warp_sum(prods[bi]);
          continue;
        }
        double sv = prods[bi];
        unsigned f = (heads >> lane) & 1u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double tv = __shfl_up_sync(FULL, sv, off);
          const unsigned tf = __shfl_up_sync(FULL, f, off);
          if (lane >= off) {
            if (!f) sv += tv;
            f |= tf;
          }
        }
        const int nh = __popc(heads);
        // lane t < nh: row ic + t ends just before the t-th head
        const int endl = lane < nh ? (int)__fns(heads, 0, lane + 1) - 1 : -1;
        double sum = __shfl_sync(FULL, sv, endl < 0 ? 0 : endl);
        if (endl < 0) sum = 0.0;
        if (lane == 0) sum += acc;
        const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb) + lane);
        if (lane < nh) {
          if (lane == 0 && head) {
            head_row = id;
            head_val = sum;
            head_cont = 0;
          } else {
            y[id] = sum;
          }
        }
        head_row = __shfl_sync(FULL, head_row, 0);
        head_val = __shfl_sync(FULL, head_val, 0);
        head = false;
        acc = __shfl_sync(FULL, sv, cnt - 1);
        nz_advance(z, c, nh);
      }
    }
    // chunk end: the current row ends exactly at e, or continues past it
    const int64_t next = nz_get(c.P0, c.P1, (int)(c.ic - c.cb) + 1);
    const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
    int64_t tail_row = -1;
    double tail_val = 0.0;
    if (next == e + 1) {
      if (head) head_row = id, head_val = acc, head_cont = 0;
      else if (lane == 0) y[id] = acc;
    } else if (head) {
      head_row = id, head_val = acc, head_cont = 1;
    } else {
      tail_row = id, tail_val = acc;
    }
    if (lane == 0) {
      rec.row[2 * k] = head_row;
      rec.row[2 * k + 1] = tail_row;
      rec.cont[k] = head_cont;
      rec.val[2 * k] = head_val;
      rec.val[2 * k + 1] = tail_val;
    }
  }
}

// ---------------------------------------------------------------------------
// SpMM N == 32 over the compacted view: half a warp per position, 128-bit
// register gathers UNR pairs deep, crd/vals of the next window prefetched,
// row switches from the window mask (no dependent loads on the critical path).
template <int UNR, int MINB, bool HOT>
__global__ void __launch_bounds__(kBlock, MINB) k_spmm32_nz(WalkGeom g, NzView z, const int64_t* __restrict__ crd,
                                                      const int32_t* __restrict__ crd32h,
                                                      const double* __restrict__ vals,
                                                      const double* __restrict__ C,
                                                      double* __restrict__ A, ChunkRecs rec,
                                                      const int64_t* __restrict__ counters) {
  const int lane = lane_id();
  const int half = lane >> 4, hl = lane & 15;
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_keep = l2_policy_evict_last();
  const uint64_t pol_stream = l2_policy_evict_first();
  const double* Cl = C + 2 * hl;
  for (int64_t v = begin + gw; v < end; v += nw) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) {
      if (lane == 0) rec.row[2 * ci.local] = -1, rec.row[2 * ci.local + 1] = -1, rec.cont[ci.local] = 0;
      continue;
    }
    const int64_t k = ci.local, s = ci.s, e = ci.e;
    NzCursor c;
    nz_start(z, c, s);
    bool head = __shfl_sync(FULL, c.P0, 0) < s;
    int64_t head_row = -1;
    int head_cont = 0;
    double2 acc = make_double2(0.0, 0.0);
    // prefetched crd/vals of the next window
    int kn = 0;
    double vn = 0.0;
    if (lane <= e - s) {
      kn = HOT ? ld_i32_hint(crd32h + s + lane, pol_stream) : (int)ld_i64_hint(crd + s + lane, pol_stream);
      vn = ld_f64_hint(vals + s + lane, pol_stream);
    }
    for (int64_t base = s; base <= e; base += 32) {
      const int last_off = (int)min((int64_t)31, e - base);
      const int cnt = last_off + 1;
      const int my_k = kn;
      const double my_v = vn;
      if (base + 32 + lane <= e) {
        kn = HOT ? ld_i32_hint(crd32h + base + 32 + lane, pol_stream)
                 : (int)ld_i64_hint(crd + base + 32 + lane, pol_stream);
        vn = ld_f64_hint(vals + base + 32 + lane, pol_stream);
      }
      const unsigned bm = nz_window_mask(c, base, base + last_off);
      // Fixed-trip groups of 2*UNR positions: positions past `cnt` carry
      // crd 0 / val 0 (their loads are predicated off), so the fast path is
      // branch-free; one mask test per group selects the row-switch path.
#pragma unroll 1
      for (int u = 0; u < 32; u += 2 * UNR) {
        if (u >= cnt) break;
        double2 cv[UNR];
        double bv[UNR];
#pragma unroll
        for (int i = 0; i < UNR; i++) {
          const int p = u + 2 * i + half;
          const int kk = __shfl_sync(FULL, my_k, p);
          bv[i] = __shfl_sync(FULL, my_v, p);
          const double* src = Cl + (int64_t)(kk & 0x7fffffff) * 32;
          if (HOT) {  // two uniform-policy loads instead of a per-lane policy
            cv[i] = make_double2(0.0, 0.0);
            if (p < cnt && kk < 0) cv[i] = ld_f64x2_hint(src, pol_keep);
            if (p < cnt && kk >= 0) cv[i] = ld_f64x2_hint(src, pol_stream);
          } else {
            cv[i] = p < cnt ? ld_f64x2_hint(src, pol_keep) : make_double2(0.0, 0.0);
          }
        }
        const unsigned gm = (bm >> u) & ((1u << (2 * UNR)) - 1u);
        if (gm == 0u) {
#pragma unroll
          for (int i = 0; i < UNR; i++) {
            acc.x = fma(bv[i], cv[i].x, acc.x);
            acc.y = fma(bv[i], cv[i].y, acc.y);
          }
        } else {
#pragma unroll
          for (int i = 0; i < UNR; i++) {
            const unsigned two = (gm >> (2 * i)) & 3u;
#pragma unroll
            for (int h = 0; h < 2; h++) {
              if ((two >> h) & 1u) {  // a new row starts at position u + 2i + h
                double2 o;
                o.x = acc.x + __shfl_xor_sync(FULL, acc.x, 16);
                o.y = acc.y + __shfl_xor_sync(FULL, acc.y, 16);
                const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
                if (head) {
                  if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
                  head_row = id;
                  head_cont = 0;
                  head = false;
                } else if (lane < 16) {
                  st_f64x2_hint(A + id * 32 + 2 * lane, o, pol_stream);
                }
                acc = make_double2(0.0, 0.0);
                nz_advance(z, c, 1);
              }
              if (half == h) {
                acc.x = fma(bv[i], cv[i].x, acc.x);
                acc.y = fma(bv[i], cv[i].y, acc.y);
              }
            }
          }
        }
      }
    }
    double2 o;
    o.x = acc.x + __shfl_xor_sync(FULL, acc.x, 16);
    o.y = acc.y + __shfl_xor_sync(FULL, acc.y, 16);
    const int64_t next = nz_get(c.P0, c.P1, (int)(c.ic - c.cb) + 1);
    const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
    int64_t tail_row = -1;
    if (next == e + 1) {
      if (head) {
        if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
        head_row = id, head_cont = 0;
      } else if (lane < 16) {
        st_f64x2_hint(A + id * 32 + 2 * lane, o, pol_stream);
      }
    } else if (head) {
      if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
      head_row = id, head_cont = 1;
    } else {
      if (lane < 16) reinterpret_cast<double2*>(rec.val + (2 * k + 1) * 32)[lane] = o;
      tail_row = id;
    }
    if (lane == 0) {
      rec.row[2 * k] = head_row;
      rec.row[2 * k + 1] = tail_row;
      rec.cont[k] = head_cont;
    }
  }
}

__global__ void k_nz_flags(const int64_t* __restrict__ R, int64_t nrows, unsigned char* __restrict__ f) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x)
    f[r] = ld64(R + r + 1) > ld64(R + r);
}

__global__ void k_nz_ptr(const int64_t* __restrict__ R, int64_t nrows, const int64_t* __restrict__ id,
                         const int64_t* __restrict__ m_dev, int64_t* __restrict__ ptr) {
  const int64_t m = *m_dev;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= m;
       j += (int64_t)gridDim.x * blockDim.x)
    ptr[j] = j < m ? ld64(R + id[j]) : ld64(R + nrows);
}

}  // namespace spd

namespace spd {

// ---------------------------------------------------------------------------
// SpMM N == 32 over the compacted view with cp.async gathers: per warp an
// S-stage ring of 32-position windows in shared memory (8 KB of C rows + the
// window's vals per stage).  Lane (h, hl) copies 16 B of the C row of
// position 2i+h and later reads back exactly that slot, so completion is a
// per-thread cp.async.wait_group.  (S-1) windows = (S-1) x 8 KB of gathers
// stay in flight per warp without registers.
constexpr int kAsyncWarps = 4;

template <int S>
__global__ void __launch_bounds__(kAsyncWarps * 32) k_spmm32_nz_async(
    WalkGeom g, NzView z, const int64_t* __restrict__ crd, const double* __restrict__ vals,
    const double* __restrict__ C, double* __restrict__ A, ChunkRecs rec, const int64_t* __restrict__ counters) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = lane_id();
  const int half = lane >> 4, hl = lane & 15;
  const int wc = threadIdx.x >> 5;
  double2* ring = reinterpret_cast<double2*>(smem + (size_t)wc * S * (kBulkStageBytes + 256));
  double* vslot = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ring) + (size_t)S * kBulkStageBytes);
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_keep = l2_policy_evict_last();
  const uint64_t pol_stream = l2_policy_evict_first();
  const double* Cl = C + 2 * hl;
  for (int64_t v = begin + gw; v < end; v += nw) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) {
      if (lane == 0) rec.row[2 * ci.local] = -1, rec.row[2 * ci.local + 1] = -1, rec.cont[ci.local] = 0;
      continue;
    }
    const int64_t k = ci.local, s = ci.s, e = ci.e;
    const int nwin = (int)((e - s + 32) >> 5);
    NzCursor c;
    nz_start(z, c, s);
    bool head = __shfl_sync(FULL, c.P0, 0) < s;
    int64_t head_row = -1;
    int head_cont = 0;
    double2 acc = make_double2(0.0, 0.0);

    // kpre/vpre: crd/vals of the next window to issue (loaded one window ahead)
    int kpre = 0;
    double vpre = 0.0;
    auto load_pre = [&](int w) {
      const int64_t q = s + 32 * (int64_t)w + lane;
      kpre = 0;
      vpre = 0.0;
      if (w < nwin && q <= e) {
        kpre = (int)ld_i64_hint(crd + q, pol_stream);
        vpre = ld_f64_hint(vals + q, pol_stream);
      }
    };
    auto issue = [&](int w) {  // copies + vals of window w (kpre/vpre hold it)
      if (w < nwin) {
        const int stage = w % S;
        const int cnt = (int)min((int64_t)32, e - (s + 32 * (int64_t)w) + 1);
        vslot[stage * 32 + lane] = vpre;
        double2* dst = ring + (size_t)stage * 512 + hl;
#pragma unroll 4
        for (int i = 0; i < 16; i++) {
          const int p = 2 * i + half;
          const int kk = __shfl_sync(FULL, kpre, p);
          if (p < cnt) cp_async16(dst + p * 16, Cl + (int64_t)kk * 32, pol_keep);
        }
      }
      cp_async_commit();
    };
    load_pre(0);
    for (int w = 0; w < S - 1; w++) {
      issue(w);
      load_pre(w + 1);
    }
    for (int w = 0; w < nwin; w++) {
      const int stage = w % S;
      const int64_t base = s + 32 * (int64_t)w;
      const int cnt = (int)min((int64_t)32, e - base + 1);
      const unsigned bm = nz_window_mask(c, base, base + cnt - 1);
      cp_async_wait<S - 2>();
      __syncwarp();
      const double2* buf = ring + (size_t)stage * 512 + hl;
      const double* vb = vslot + stage * 32;
#pragma unroll 2
      for (int p0 = 0; p0 < cnt; p0 += 2) {
        const int p = p0 + half;
        const double2 cv = p < cnt ? buf[p * 16] : make_double2(0.0, 0.0);
        const double b = p < cnt ? vb[p] : 0.0;
        const unsigned two = (bm >> p0) & 3u;
        if (two == 0u) {
          acc.x = fma(b, cv.x, acc.x);
          acc.y = fma(b, cv.y, acc.y);
        } else {
#pragma unroll
          for (int h = 0; h < 2; h++) {
            if ((two >> h) & 1u) {
              double2 o;
              o.x = acc.x + __shfl_xor_sync(FULL, acc.x, 16);
              o.y = acc.y + __shfl_xor_sync(FULL, acc.y, 16);
              const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
              if (head) {
                if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
                head_row = id;
                head_cont = 0;
                head = false;
              } else if (lane < 16) {
                st_f64x2_hint(A + id * 32 + 2 * lane, o, pol_stream);
              }
              acc = make_double2(0.0, 0.0);
              nz_advance(z, c, 1);
            }
            if (half == h) {
              acc.x = fma(b, cv.x, acc.x);
              acc.y = fma(b, cv.y, acc.y);
            }
          }
        }
      }
      __syncwarp();
      issue(w + S - 1);
      load_pre(w + S);
    }
    cp_async_wait<0>();
    double2 o;
    o.x = acc.x + __shfl_xor_sync(FULL, acc.x, 16);
    o.y = acc.y + __shfl_xor_sync(FULL, acc.y, 16);
    const int64_t next = nz_get(c.P0, c.P1, (int)(c.ic - c.cb) + 1);
    const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
    int64_t tail_row = -1;
    if (next == e + 1) {
      if (head) {
        if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
        head_row = id, head_cont = 0;
      } else if (lane < 16) {
        st_f64x2_hint(A + id * 32 + 2 * lane, o, pol_stream);
      }
    } else if (head) {
      if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
      head_row = id, head_cont = 1;
    } else {
      if (lane < 16) reinterpret_cast<double2*>(rec.val + (2 * k + 1) * 32)[lane] = o;
      tail_row = id;
    }
    if (lane == 0) {
      rec.row[2 * k] = head_row;
      rec.row[2 * k + 1] = tail_row;
      rec.cont[k] = head_cont;
    }
  }
}

}  // namespace spd

namespace spd {

// Column reference counts of a crd array (warp-aggregated atomics).
__global__ void k_col_count(const int64_t* __restrict__ crd, int64_t nnz, int32_t* __restrict__ counts) {
  const int lane = lane_id();
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; b < nnz;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = b + lane;
    const bool ok = q < nnz;
    const unsigned long long col = ok ? (unsigned long long)ld64(crd + q) : ~0ull;
    const unsigned active = __ballot_sync(FULL, ok);
    if (!ok) continue;
    const unsigned peers = __match_any_sync(active, col);
    if (lane == __ffs(peers) - 1) atomicAdd(counts + col, __popc(peers));
  }
}

__global__ void k_crd32h(const int64_t* __restrict__ crd, int64_t nnz, const int32_t* __restrict__ counts,
                         const int32_t* __restrict__ sorted_desc, int64_t k, int64_t ncols,
                         int32_t* __restrict__ out) {
  // threshold: the k-th largest count (every column with a count >= it is hot)
  const int32_t t = k >= ncols ? 1 : max(sorted_desc[k - 1], 1);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = ld64(crd + q);
    out[q] = (int32_t)col | (counts[col] >= t ? (int32_t)0x80000000 : 0);
  }
}

}  // namespace spd
