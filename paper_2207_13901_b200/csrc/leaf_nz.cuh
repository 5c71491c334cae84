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
  int64_t m;                        // count, or -1: read it from *m_dev
  const int64_t* __restrict__ m_dev;  // device-side count (built without a host sync)
};

// The compacted-row count as the kernel sees it (kernels start with
// `z.m = nz_count(z)`): the build leaves it on the device, so no host
// synchronisation sits between building the view and using it.
__device__ __forceinline__ int64_t nz_count(const NzView& z) { return z.m >= 0 ? z.m : __ldg(z.m_dev); }

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

__device__ __forceinline__ void nz_slide(const NzView& z, NzCursor& c) {
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

// Zeroes rows [lo, hi] of a W-wide dense output (contiguous), warp-cooperative.
__device__ __forceinline__ void zero_gap(double* __restrict__ out, int64_t W, int64_t lo, int64_t hi) {
  if (lo > hi) return;
  const int lane = lane_id();
  if (W % 2 == 0) {
    double2* p = reinterpret_cast<double2*>(out + lo * W);
    const int64_t cnt = (hi - lo + 1) * (W / 2);
    for (int64_t i = lane; i < cnt; i += 32) p[i] = make_double2(0.0, 0.0);
  } else {
    double* p = out + lo * W;
    const int64_t cnt = (hi - lo + 1) * W;
    for (int64_t i = lane; i < cnt; i += 32) p[i] = 0.0;
  }
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
  const uint64_t pol = l2_policy_evict_first();
  // the next group's row pointers are loaded before the current group's
  // stores, so the dependent row-pointer latency overlaps them
  int64_t g0 = lo + gw * 32;
  int64_t ra = 0, rb = 0;
  if (g0 + lane <= hi) ra = ld64(R + g0 + lane), rb = ld64(R + g0 + lane + 1);
  for (; g0 <= hi; g0 += nw * 32) {
    const int64_t r = g0 + lane;
    const bool empty = r <= hi && rb == ra;
    const int64_t gn = g0 + nw * 32;
    if (gn + lane <= hi) ra = ld64(R + gn + lane), rb = ld64(R + gn + lane + 1);
    if (W == 1) {
      if (empty) out[r] = 0.0;
      continue;
    }
    const unsigned m = __ballot_sync(FULL, empty);
    const int ne = __popc(m);
    if (W == 32) {  // a half-warp per row: one 128-bit store per lane writes two 256-byte rows
      const int half = lane >> 4, hl = lane & 15;
      double* base = out + g0 * 32 + 2 * hl;
      if (m == FULL) {  // a fully empty group (the sparse tail): 8 KB of contiguous zeros
#pragma unroll
        for (int t = 0; t < 32; t += 2) st_f64x2_hint(base + (t + half) * 32, make_double2(0.0, 0.0), pol);
        continue;
      }
      // otherwise the empty rows two at a time, lowest first (warp-uniform;
      // the k-th-set-bit search it replaces dominated the kernel's issue)
      unsigned left = m;
      while (left) {
        const int b0 = __ffs(left) - 1;
        left &= left - 1u;
        const int b1 = left ? __ffs(left) - 1 : -1;
        if (left) left &= left - 1u;
        const int b = half ? b1 : b0;
        if (b >= 0) st_f64x2_hint(base + b * 32, make_double2(0.0, 0.0), pol);
      }
      continue;
    }
    for (int t = 0; t < ne; t++) {
      const int b = (int)__fns(m, 0, t + 1);
      double* row = out + (g0 + b) * W;
      for (int64_t j = lane; j < W; j += 32) row[j] = 0.0;
    }
  }
}

__device__ __forceinline__ int64_t ld_crd_hint(const int64_t* p, uint64_t pol) { return ld_i64_hint(p, pol); }
__device__ __forceinline__ int64_t ld_crd_hint(const int32_t* p, uint64_t pol) { return ld_i32_hint(p, pol); }

// Compacted-column index build (once per pattern) and the per-call gather.
__global__ void k_ref_flags(const int32_t* __restrict__ counts, int64_t ncols, int32_t* __restrict__ flags) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x)
    flags[c] = counts[c] > 0 ? 1 : 0;
}
__global__ void k_ref_list(const int32_t* __restrict__ flags, const int32_t* __restrict__ rank, int64_t ncols,
                           int32_t* __restrict__ cref) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x)
    if (flags[c]) cref[rank[c]] = (int32_t)c;
}
__global__ void k_crd_rank(const int64_t* __restrict__ crd, int64_t n, const int32_t* __restrict__ rank,
                           int32_t* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = rank[crd[q]];
}
__global__ void k_gather_ref(const double* __restrict__ x, const int32_t* __restrict__ cref, int64_t nref,
                             double* __restrict__ xc) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nref; r += (int64_t)gridDim.x * blockDim.x)
    xc[r] = __ldg(x + cref[r]);
}

// ---------------------------------------------------------------------------
// SpMV / SpTTV, windowed: a warp streams its chunk in windows of kWin
// positions.  Per window every lane loads kWin/32 positions lane-consecutive
// (coalesced crd and vals, kWin/32 independent x gathers in flight per lane),
// and the products go to the warp's shared-memory window.  The rows touching
// the window are then reduced one per lane, serially in stored-position order
// (sim.cpp:326-354) from shared memory; a row segment of kSegLong or more
// positions is summed by the whole warp instead (lane-strided partials and a
// butterfly).  A row continuing past the window carries its partial into the
// next one, and a window lying inside one row that continues past it is summed
// in registers (hub rows).  Versus a lane walking its own row in global memory
// (the round-1 k_spmv_rows: 92 B of spills at 6 CTAs/SM), the stream loads
// touch one or two lines per instruction instead of up to 32; measured
// (profiles/README.md) C1 0.085 -> 0.073 ms, SpTTV 0.125 -> 0.121 ms, R-MAT
// SpMV 0.960 -> 0.940 ms, and faster than the round-1 window scan (k_spmv_nz)
// on long rows too, so it is the one SpMV / SpTTV leaf.
constexpr int kWin = 256;
constexpr int kSegLong = 64;

template <int MINB, typename CI>
__global__ void __launch_bounds__(kBlock, MINB) k_spmv_win(WalkGeom g, NzView z, const CI* __restrict__ crd,
                                                     const double* __restrict__ vals,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     ChunkRecs rec, const int64_t* __restrict__ counters) {
  __shared__ double win_s[kBlock / 32][kWin];
  const int lane = lane_id();
  double* buf = win_s[threadIdx.x >> 5];
  z.m = nz_count(z);
  const int64_t begin = counters[1], end = counters[2];
  const uint64_t pol = l2_policy_evict_first();
  for (int64_t v = begin + chunk_ticket(counters); v < end; v = begin + chunk_ticket(counters)) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) {
      zero_gap(y, 1, ci.w_lo, ci.w_hi);
      if (lane == 0) rec.row[2 * ci.local] = -1, rec.row[2 * ci.local + 1] = -1, rec.cont[ci.local] = 0;
      continue;
    }
    const int64_t k = ci.local, s = ci.s, e = ci.e;
    int64_t r = warp_owner(z.ptr, z.m, s);  // compacted row holding the window's first position
    bool at_head = ld64(z.ptr + r) < s;     // r began before the chunk: its partial is the head record
    if (s == ci.q_lo && !at_head) zero_gap(y, 1, ci.w_lo, ld64(z.id + r) - 1);
    int64_t head_row = -1;
    int head_cont = 0;
    double head_val = 0.0, carry = 0.0;
    int64_t rend = ld64(z.ptr + r + 1) - 1;  // last position of row r
    for (int64_t wb = s; wb <= e; wb += kWin) {
      const int64_t we = min(wb + kWin - 1, e);
      if (rend > we) {  // the window lies inside row r, which continues: no row ends here
        double part = 0.0;
#pragma unroll
        for (int h = 0; h < kWin / 32; h += 4) {
          CI kk[4];
          double vv[4];
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int64_t q = wb + 32 * (h + i) + lane;
            kk[i] = 0;
            vv[i] = 0.0;
            if (q <= we) kk[i] = ld_crd_hint(crd + q, pol), vv[i] = ld_f64_hint(vals + q, pol);
          }
#pragma unroll
          for (int i = 0; i < 4; i++)
            if (wb + 32 * (h + i) + lane <= we) part += vv[i] * __ldg(x + kk[i]);
        }
        carry += warp_sum(part);
        continue;
      }
#pragma unroll
      for (int h = 0; h < kWin / 32; h += 4) {
        CI kk[4];
        double vv[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int64_t q = wb + 32 * (h + i) + lane;
          kk[i] = 0;
          vv[i] = 0.0;
          if (q <= we) kk[i] = ld_crd_hint(crd + q, pol), vv[i] = ld_f64_hint(vals + q, pol);
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int64_t q = wb + 32 * (h + i) + lane;
          buf[32 * (h + i) + lane] = q <= we ? vv[i] * __ldg(x + kk[i]) : 0.0;
        }
      }
      __syncwarp();
      for (;;) {  // the rows touching [wb, we], 32 at a time
        const int64_t rr = r + lane;
        const int64_t pa = rr < z.m ? ld64(z.ptr + rr) : INT64_MAX;
        const bool act = pa <= we;  // lane 0's row holds wb
        const int64_t pe = act ? ld64(z.ptr + rr + 1) - 1 : -1;
        const int a = act ? (int)(max(pa, wb) - wb) : 0;
        const int b = act ? (int)(min(pe, we) - wb) : -1;
        double sum = lane == 0 ? carry : 0.0;
        const bool lng = b - a + 1 >= kSegLong;
        if (!lng)
          for (int q = a; q <= b; q++) sum += buf[q];
        unsigned long_mask = __ballot_sync(FULL, lng);
        while (long_mask) {
          const int t = __ffs(long_mask) - 1;
          long_mask &= long_mask - 1;
          const int aa = __shfl_sync(FULL, a, t), bb = __shfl_sync(FULL, b, t);
          double part = 0.0;
          for (int q = aa + lane; q <= bb; q += 32) part += buf[q];
          part = warp_sum(part);
          if (lane == t) sum += part;
        }
        // a row ending here is stored (or is the head record); the empty rows
        // up to the next non-empty one are zeroed, bounded by W_c at the chunk end
        int64_t glo = 1, ghi = 0;
        if (act && pe <= we) {
          const int64_t id = ld64(z.id + rr);
          const int64_t nid = rr + 1 < z.m ? ld64(z.id + rr + 1) : -1;
          if (lane == 0 && at_head) {
            head_row = id;
            head_val = sum;
            head_cont = 0;
          } else {
            y[id] = sum;
          }
          glo = id + 1;
          ghi = pe == e ? (nid < 0 ? ci.w_hi : min(nid - 1, ci.w_hi)) : nid - 1;
        }
        const bool long_gap = ghi - glo + 1 > 64;
        if (!long_gap)
          for (int64_t q = glo; q <= ghi; q++) y[q] = 0.0;
        unsigned gaps = __ballot_sync(FULL, long_gap);
        while (gaps) {
          const int t = __ffs(gaps) - 1;
          gaps &= gaps - 1;
          zero_gap(y, 1, __shfl_sync(FULL, glo, t), __shfl_sync(FULL, ghi, t));
        }
        const unsigned am = __ballot_sync(FULL, act);
        const int nact = __popc(am);
        const int64_t pe_last = __shfl_sync(FULL, pe, nact - 1);
        if (nact == 32 && pe_last < we) {  // more rows start in this window
          r += 32;
          carry = 0.0;
          at_head = false;
          continue;
        }
        if (pe_last <= we) {  // the window ends exactly at a row end
          r += nact;
          carry = 0.0;
          at_head = false;
          rend = r < z.m ? ld64(z.ptr + r + 1) - 1 : INT64_MAX;
        } else {  // the last row continues: carry its partial
          r += nact - 1;
          carry = __shfl_sync(FULL, sum, nact - 1);
          at_head = at_head && nact == 1;
          rend = pe_last;
        }
        break;
      }
      __syncwarp();
    }
    // chunk end: a row still open continues past e
    int64_t tail_row = -1;
    double tail_val = 0.0;
    if (r < z.m && ld64(z.ptr + r) <= e) {
      const int64_t id = ld64(z.id + r);
      if (at_head) head_row = id, head_val = carry, head_cont = 1;
      else tail_row = id, tail_val = carry;
    }
    head_row = __shfl_sync(FULL, head_row, 0);
    head_val = __shfl_sync(FULL, head_val, 0);
    head_cont = __shfl_sync(FULL, head_cont, 0);
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
// Register cursor of the N == 32 SpMM leaf: 64 consecutive compacted rows
// (two 32-lane blocks) with their starts relative to the chunk start and
// their ids as 32-bit values (rows < 2^31), so the walk fits the register
// budget that leaves room for 24 warps per SM.
struct NzCur32 {
  int64_t cb;  // block base (compacted row index)
  int off;     // current compacted row - cb, in [0, 32) between windows
  int P0, P1;  // starts of rows cb + lane, cb + 32 + lane, relative to the chunk start (clamped)
  int I0, I1;  // ids of the same rows
};

__device__ __forceinline__ void nz32_load(const NzView& z, int64_t j0, int64_t s, int& P, int& I) {
  const int64_t j = j0 + lane_id();
  const int64_t p = j <= z.m ? ld64(z.ptr + j) - s : (int64_t)INT32_MAX;
  P = (int)max(min(p, (int64_t)INT32_MAX), (int64_t)-1);
  I = j < z.m ? (int)ld64(z.id + j) : -1;
}

__device__ __forceinline__ int shfl_pair(int v0, int v1, int idx) {
  const int a = __shfl_sync(FULL, v0, idx & 31), b = __shfl_sync(FULL, v1, idx & 31);
  return idx < 32 ? a : b;
}

// ---------------------------------------------------------------------------
// SpMM N == 32 over the compacted view (the C2 leaf).  Half a warp per stored
// position: lane l copies columns 2(l%16), 2(l%16)+1 of C(k,:), so a warp
// instruction covers two positions.  Per 32-position window the warp holds
// the window's int32 columns and values (one per lane; columns two windows
// ahead, values one) and the row-start mask.  The 256-byte C rows land in a
// per-warp shared-memory ring through cp.async (16 B per lane, L2 evict_last):
// the warp keeps S-1 groups of 8 positions in flight while it consumes the
// oldest, so the bytes in flight per SM do not cost registers.  Each lane
// reads back exactly the 16 bytes it copied: no warp barrier.  A full group
// without a row start is 8 FMAs per lane; a group holding row starts walks
// only its starts (products before each start added under a predicate, the
// finished row flushed with one xor-shuffle, the next row's id read from the
// register cursor).  Positions past the chunk end copy row 0 and are never
// added.  Measured history (profiles/r02_*): the round-1 leaf issued ~16
// instructions per position (64-bit address arithmetic, per-position row
// tests) and stalled on register-held gathers; the register-lean rewrite cut
// that to ~11 but stayed gather-latency bound (16 warps stalled per issue);
// the ring holds 3 groups ahead per warp and moves DRAM to ~65% of its peak.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint64_t pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int S, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) k_spmm32_nz(WalkGeom g, NzView z, const int32_t* __restrict__ crd32,
                                                        const double* __restrict__ vals,
                                                        const double* __restrict__ C, double* __restrict__ A,
                                                        ChunkRecs rec, const int64_t* __restrict__ counters) {
  static_assert(S >= 2 && S <= 5, "lookahead stays within the next window");
  constexpr int UNR = 4;  // gathers per lane per group of 8 positions
  extern __shared__ double2 smem_ring[];
  const int lane = lane_id();
  const int half = lane >> 4, hl = lane & 15;
  // this warp's ring: S slots x 8 positions x 16 lanes of 16 bytes; lane
  // (half, hl) owns element [slot][2i + half][hl]
  double2* ring = smem_ring + (threadIdx.x >> 5) * (S * 8 * 16) + half * 16 + hl;
  z.m = nz_count(z);
  const int64_t begin = counters[1], end = counters[2];
  const double* Cl = C + 2 * hl;
  const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
  const int nchunks = (int)(end - begin);  // < 2^31 (positions < 2^31 here), one register
  for (int t = (int)chunk_ticket(counters); t < nchunks; t = (int)chunk_ticket(counters)) {
    const ChunkInfo ci = chunk_info(g, begin + t, begin);
    if (ci.q_lo > ci.q_hi) {
      if (lane == 0) rec.row[2 * ci.local] = -1, rec.row[2 * ci.local + 1] = -1, rec.cont[ci.local] = 0;
      continue;
    }
    const int64_t s = ci.s;
    const int ne = (int)(ci.e - s);  // last offset of the chunk
    const int ngroups = (ne + 8) / 8;
    const int32_t* cp = crd32 + s;
    const double* vp = vals + s;
    NzCur32 c;
    c.cb = warp_owner32(z.ptr, (int)z.m, s);
    c.off = 0;
    nz32_load(z, c.cb, s, c.P0, c.I0);
    nz32_load(z, c.cb + 32, s, c.P1, c.I1);
    bool head = __shfl_sync(FULL, c.P0, 0) < 0;
    int cur = __shfl_sync(FULL, c.I0, 0);
    int head_row = -1;
    double2 acc = make_double2(0.0, 0.0);
    // column indices of windows w, w+1, w+2 and values of windows w, w+1
    int k0 = lane <= ne ? ld_i32_hint(cp + lane, pol_stream) : 0;
    int k1 = 32 + lane <= ne ? ld_i32_hint(cp + 32 + lane, pol_stream) : 0;
    int k2 = 64 + lane <= ne ? ld_i32_hint(cp + 64 + lane, pol_stream) : 0;
    double v0 = lane <= ne ? ld_f64_hint(vp + lane, pol_stream) : 0.0;
    double v1 = 32 + lane <= ne ? ld_f64_hint(vp + 32 + lane, pol_stream) : 0.0;
    // issue group gi (positions 8 gi .. 8 gi + 7) from the window registers
    // (kw: the column indices of gi's window)
    auto issue = [&](int gi, int kw) {
      if (gi < ngroups) {
        double2* slot = ring + (gi % S) * (8 * 16);
#pragma unroll
        for (int i = 0; i < UNR; i++) {
          const int kk = __shfl_sync(FULL, kw, ((gi & 3) << 3) + 2 * i + half);
          cp_async16(slot + i * 32, Cl + (int64_t)kk * 32, pol_keep);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int gi = 0; gi < S - 1; gi++) issue(gi, k0);
    for (int b0 = 0; b0 <= ne; b0 += 32) {
      const int cnt = min(32, ne - b0 + 1);
      const int last = b0 + cnt - 1;
      unsigned bm = __reduce_or_sync(
          FULL, (lane > c.off && c.P0 >= b0 && c.P0 <= last) ? 1u << (c.P0 - b0) : 0u);
      if (__shfl_sync(FULL, c.P0, 31) <= last)
        bm |= __reduce_or_sync(FULL, (c.P1 >= b0 && c.P1 <= last) ? 1u << (c.P1 - b0) : 0u);
      int j = c.off + 1;
      const int gw = b0 >> 3;  // first group of this window
#pragma unroll 1
      for (int u = 0; u < cnt; u += 8) {
        const int gi = gw + (u >> 3);
        // keep S-1 groups in flight: issue gi + S - 1 (its window is this one or the next)
        {
          const int ga = gi + S - 1;
          issue(ga, (ga >> 2) == (gi >> 2) ? k0 : k1);
        }
        cp_async_wait<S - 1>();
        const double2* slot = ring + (gi % S) * (8 * 16);
        double2 cv[UNR];
        double bv[UNR];
#pragma unroll
        for (int i = 0; i < UNR; i++) {
          cv[i] = slot[i * 32];
          bv[i] = __shfl_sync(FULL, v0, u + 2 * i + half);
        }
        unsigned gm = (bm >> u) & 0xffu;
        if (gm == 0u && u + 8 <= cnt) {
#pragma unroll
          for (int i = 0; i < UNR; i++) {
            acc.x = fma(bv[i], cv[i].x, acc.x);
            acc.y = fma(bv[i], cv[i].y, acc.y);
          }
          continue;
        }
        const int lim = min(8, cnt - u);
        int lo = 0;
        for (;;) {
          const int hi = gm ? __ffs(gm) - 1 : lim;
#pragma unroll
          for (int i = 0; i < UNR; i++) {
            const int o = 2 * i + half;
            if (o >= lo && o < hi) {
              acc.x = fma(bv[i], cv[i].x, acc.x);
              acc.y = fma(bv[i], cv[i].y, acc.y);
            }
          }
          if (!gm) break;
          double2 o;
          o.x = acc.x + __shfl_xor_sync(FULL, acc.x, 16);
          o.y = acc.y + __shfl_xor_sync(FULL, acc.y, 16);
          if (head) {
            if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * ci.local * 32)[lane] = o;
            head_row = cur;
            head = false;
          } else if (lane < 16) {
            st_f64x2_hint(A + (int64_t)cur * 32 + 2 * lane, o, pol_stream);
          }
          acc = make_double2(0.0, 0.0);
          cur = shfl_pair(c.I0, c.I1, j);
          j++;
          lo = hi;
          gm &= gm - 1u;
        }
      }
      c.off = j - 1;
      if (c.off >= 32) {
        c.cb += 32;
        c.off -= 32;
        c.P0 = c.P1;
        c.I0 = c.I1;
        nz32_load(z, c.cb + 32, s, c.P1, c.I1);
      }
      // advance the window registers: w+1 becomes current, w+3 is prefetched
      k0 = k1;
      k1 = k2;
      k2 = b0 + 96 + lane <= ne ? ld_i32_hint(cp + b0 + 96 + lane, pol_stream) : 0;
      v0 = v1;
      v1 = b0 + 64 + lane <= ne ? ld_f64_hint(vp + b0 + 64 + lane, pol_stream) : 0.0;
    }
    cp_async_wait<0>();  // drain the look-ahead past the chunk (empty groups)
    double2 o;
    o.x = acc.x + __shfl_xor_sync(FULL, acc.x, 16);
    o.y = acc.y + __shfl_xor_sync(FULL, acc.y, 16);
    const int next = shfl_pair(c.P0, c.P1, c.off + 1);
    const int64_t k = ci.local;
    int tail_row = -1, head_cont = 0;
    if (next == ne + 1) {
      if (head) {
        if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
        head_row = cur;
      } else if (lane < 16) {
        st_f64x2_hint(A + (int64_t)cur * 32 + 2 * lane, o, pol_stream);
      }
    } else if (head) {
      if (lane < 16) reinterpret_cast<double2*>(rec.val + 2 * k * 32)[lane] = o;
      head_row = cur, head_cont = 1;
    } else {
      if (lane < 16) reinterpret_cast<double2*>(rec.val + (2 * k + 1) * 32)[lane] = o;
      tail_row = cur;
    }
    if (lane == 0) {
      rec.row[2 * k] = head_row;
      rec.row[2 * k + 1] = tail_row;
      rec.cont[k] = head_cont;
    }
  }
}

// ---------------------------------------------------------------------------
// SpMM for N in {8, 16, 64, 128}: k_spmm32_nz generalised.  LP = min(N/2, 32)
// lanes gather one position's C row with 128-bit loads (VPL = N/64 of them
// per lane when N = 128), so a warp instruction covers PPI = 32/LP positions
// (8 at N = 8, 4 at N = 16, 1 at N >= 64).  Positions go in fixed-trip
// groups of PPI*UNR; a group without a row start adds every product; a group
// with one walks its PPI sub-positions in order (runtime loop, to keep the
// code small), flushing the finished row -- the sub-lane partials summed by
// an xor butterfly over the sub index -- at each start.  Chunk tickets,
// records and ownership as k_spmm32_nz.
//
// MT: SpMTTKRP instead (R = N): C is D(k,:) gathered by the leaf crd, and a
// second gather Cj(j,:) by jleaf; the value is (B * C(j,l)) * D(k,l) as the
// reference multiplies (sim.cpp:328-337), added with a unit FMA.
template <int N, int UNR, int MINB, bool MT = false>
__global__ void __launch_bounds__(kBlock, MINB) k_spmm_nzv(WalkGeom g, NzView z, const int64_t* __restrict__ crd,
                                                     const double* __restrict__ vals,
                                                     const double* __restrict__ C, double* __restrict__ A,
                                                     ChunkRecs rec, const int64_t* __restrict__ counters,
                                                     const int32_t* __restrict__ jleaf = nullptr,
                                                     const double* __restrict__ Cj = nullptr) {
  constexpr int LP = N / 2 < 32 ? N / 2 : 32;  // lanes per position
  constexpr int VPL = N / 64 > 1 ? N / 64 : 1;  // double2 per lane
  constexpr int PPI = 32 / LP;                 // positions per warp instruction
  constexpr int GP = PPI * UNR;                // positions per group
  static_assert(GP <= 32, "a group must fit one 32-position window");
  const int lane = lane_id();
  z.m = nz_count(z);
  const int sub = lane / LP, sl = lane % LP;
  const int64_t begin = counters[1], end = counters[2];
  const uint64_t pol_keep = l2_policy_evict_last();
  const uint64_t pol_stream = l2_policy_evict_first();
  const double* Cl = C + 2 * sl;
  const double* Cjl = MT ? Cj + 2 * sl : nullptr;
  const int64_t tmax = end - begin;
  for (int64_t t = chunk_ticket(counters); t < tmax; t = chunk_ticket(counters)) {
    const int64_t v = begin + t;
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
    double2 acc[VPL];
#pragma unroll
    for (int w = 0; w < VPL; w++) acc[w] = make_double2(0.0, 0.0);
    // finished row: sum the sub-lane partials, store (or record) it, reset
    auto flush = [&](double* dst_row_base, bool to_record, double* rec_base) {
      double2 o[VPL];
#pragma unroll
      for (int w = 0; w < VPL; w++) {
        o[w] = acc[w];
#pragma unroll
        for (int m = LP; m < 32; m <<= 1) {
          o[w].x += __shfl_xor_sync(FULL, o[w].x, m);
          o[w].y += __shfl_xor_sync(FULL, o[w].y, m);
        }
      }
      if (sub == 0) {
#pragma unroll
        for (int w = 0; w < VPL; w++) {
          if (to_record)
            reinterpret_cast<double2*>(rec_base)[sl + w * 32] = o[w];
          else
            st_f64x2_hint(dst_row_base + 2 * sl + w * 64, o[w], pol_stream);
        }
      }
#pragma unroll
      for (int w = 0; w < VPL; w++) acc[w] = make_double2(0.0, 0.0);
    };
    int kn = 0, jn = 0;
    double vn = 0.0;
    if (lane <= e - s) {
      kn = (int)ld_i64_hint(crd + s + lane, pol_stream);
      if (MT) jn = ld_i32_hint(jleaf + s + lane, pol_stream);
      vn = ld_f64_hint(vals + s + lane, pol_stream);
    }
    for (int64_t base = s; base <= e; base += 32) {
      const int last_off = (int)min((int64_t)31, e - base);
      const int cnt = last_off + 1;
      const int my_k = kn, my_j = jn;
      const double my_v = vn;
      if (base + 32 + lane <= e) {
        kn = (int)ld_i64_hint(crd + base + 32 + lane, pol_stream);
        if (MT) jn = ld_i32_hint(jleaf + base + 32 + lane, pol_stream);
        vn = ld_f64_hint(vals + base + 32 + lane, pol_stream);
      }
      const unsigned bm = nz_window_mask(c, base, base + last_off);
#pragma unroll 1
      for (int u = 0; u < 32; u += GP) {
        if (u >= cnt) break;
        double2 cv[UNR][VPL];
        double bv[UNR];
#pragma unroll
        for (int i = 0; i < UNR; i++) {
          const int p = u + PPI * i + sub;
          const int kk = __shfl_sync(FULL, my_k, p & 31);
          bv[i] = __shfl_sync(FULL, my_v, p & 31);
          const double* src = Cl + (int64_t)kk * N;
#pragma unroll
          for (int w = 0; w < VPL; w++)
            cv[i][w] = p < cnt ? ld_f64x2_hint(src + w * 64, pol_keep) : make_double2(0.0, 0.0);
          if (MT) {
            const int jj = __shfl_sync(FULL, my_j, p & 31);
            const double* srcj = Cjl + (int64_t)jj * N;
#pragma unroll
            for (int w = 0; w < VPL; w++) {
              const double2 cj = p < cnt ? ld_f64x2_hint(srcj + w * 64, pol_keep) : make_double2(0.0, 0.0);
              cv[i][w] = make_double2((bv[i] * cj.x) * cv[i][w].x, (bv[i] * cj.y) * cv[i][w].y);
            }
            bv[i] = 1.0;
          }
        }
        const unsigned gm = GP == 32 ? (bm >> u) : ((bm >> u) & ((1u << GP) - 1u));
        if (gm == 0u) {
#pragma unroll
          for (int i = 0; i < UNR; i++)
#pragma unroll
            for (int w = 0; w < VPL; w++) {
              acc[w].x = fma(bv[i], cv[i][w].x, acc[w].x);
              acc[w].y = fma(bv[i], cv[i][w].y, acc[w].y);
            }
        } else {
#pragma unroll
          for (int i = 0; i < UNR; i++) {
            const unsigned bits = (gm >> (PPI * i)) & ((1u << PPI) - 1u);
            if (bits == 0u) {
#pragma unroll
              for (int w = 0; w < VPL; w++) {
                acc[w].x = fma(bv[i], cv[i][w].x, acc[w].x);
                acc[w].y = fma(bv[i], cv[i][w].y, acc[w].y);
              }
              continue;
            }
#pragma unroll 1
            for (int h = 0; h < PPI; h++) {
              if ((bits >> h) & 1u) {  // a new row starts at position u + PPI*i + h
                const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
                if (head) {
                  flush(nullptr, true, rec.val + 2 * k * N);
                  head_row = id;
                  head_cont = 0;
                  head = false;
                } else {
                  flush(A + id * N, false, nullptr);
                }
                nz_advance(z, c, 1);
              }
              if (sub == h) {
#pragma unroll
                for (int w = 0; w < VPL; w++) {
                  acc[w].x = fma(bv[i], cv[i][w].x, acc[w].x);
                  acc[w].y = fma(bv[i], cv[i][w].y, acc[w].y);
                }
              }
            }
          }
        }
      }
    }
    const int64_t next = nz_get(c.P0, c.P1, (int)(c.ic - c.cb) + 1);
    const int64_t id = nz_get(c.I0, c.I1, (int)(c.ic - c.cb));
    int64_t tail_row = -1;
    if (next == e + 1) {
      if (head) {
        flush(nullptr, true, rec.val + 2 * k * N);
        head_row = id, head_cont = 0;
      } else {
        flush(A + id * N, false, nullptr);
      }
    } else if (head) {
      flush(nullptr, true, rec.val + 2 * k * N);
      head_row = id, head_cont = 1;
    } else {
      flush(nullptr, true, rec.val + (2 * k + 1) * N);
      tail_row = id;
    }
    if (lane == 0) {
      rec.row[2 * k] = head_row;
      rec.row[2 * k + 1] = tail_row;
      rec.cont[k] = head_cont;
    }
  }
}

// ---------------------------------------------------------------------------
// SpMTTKRP, R == 32, over the compacted rows i (leaf row pointer): the
// k_spmm32_nz walk with two gathers per position -- D(k,:) by the leaf crd and
// C(j,:) by the position's fibre coordinate (jleaf, a per-leaf copy of crd1
// built once per tensor) -- and value ((B*C)*D) as the reference multiplies.
template <int UNR, int MINB, bool HOT>
__global__ void __launch_bounds__(kBlock, MINB) k_mttkrp32_nz(WalkGeom g, NzView z, const int64_t* __restrict__ crd,
                                                      const int32_t* __restrict__ jleaf, const double* __restrict__ Cj,
                                                      const double* __restrict__ vals,
                                                      const double* __restrict__ C,
                                                      double* __restrict__ A, ChunkRecs rec,
                                                      const int64_t* __restrict__ counters) {
  const int lane = lane_id();
  z.m = nz_count(z);
  const int half = lane >> 4, hl = lane & 15;
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_keep = l2_policy_evict_last();
  const uint64_t pol_stream = l2_policy_evict_first();
  const double* Cl = C + 2 * hl;
  const double* Cjl = Cj + 2 * hl;
  for (int64_t v = begin + chunk_ticket(counters); v < end; v = begin + chunk_ticket(counters)) {
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
    int kn = 0, jn = 0;
    double vn = 0.0;
    if (lane <= e - s) {
      kn = (int)ld_i64_hint(crd + s + lane, pol_stream);
      jn = ld_i32_hint(jleaf + s + lane, pol_stream);
      vn = ld_f64_hint(vals + s + lane, pol_stream);
    }
    for (int64_t base = s; base <= e; base += 32) {
      const int last_off = (int)min((int64_t)31, e - base);
      const int cnt = last_off + 1;
      const int my_k = kn, my_j = jn;
      const double my_v = vn;
      if (base + 32 + lane <= e) {
        kn = (int)ld_i64_hint(crd + base + 32 + lane, pol_stream);
        jn = ld_i32_hint(jleaf + base + 32 + lane, pol_stream);
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
          const int jj = __shfl_sync(FULL, my_j, p);
          bv[i] = __shfl_sync(FULL, my_v, p);
          double2 dv = make_double2(0.0, 0.0), cj = make_double2(0.0, 0.0);
          if (p < cnt) {
            dv = ld_f64x2_hint(Cl + (int64_t)kk * 32, pol_keep);
            cj = ld_f64x2_hint(Cjl + (int64_t)jj * 32, pol_keep);
          }
          // ((b * C(j,l)) * D(k,l)) as the reference multiplies (sim.cpp:328-337),
          // then added with a unit FMA
          cv[i] = make_double2((bv[i] * cj.x) * dv.x, (bv[i] * cj.y) * dv.y);
          bv[i] = 1.0;
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

__global__ void k_crd_to_i32(const int64_t* __restrict__ crd, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)crd[i];
}

}  // namespace spd

namespace spd {

// ---------------------------------------------------------------------------
// SDDMM over the compacted view, K = 32 * KT.  Lane l owns k in
// [KT*l, KT*l + KT): one group of 4 positions loads 4 D columns (KT doubles
// per lane each, contiguous -> coalesced K*8-byte rows when D is j-major) and
// the C row of each position's row (kept in registers while the row lasts),
// forms 4 per-lane partial dot products and reduces all four across the warp
// with one butterfly (2+1+3 shuffles instead of 4 x 5).  Row ids of the
// positions come from the window's row-start mask, so no row-pointer loads
// sit on the critical path.
__device__ __forceinline__ double ld_f64_keep(const double* ptr, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}

template <int KT, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) k_sddmm_nz(WalkGeom g, NzView z, const int32_t* __restrict__ crd32h,
                                                      const double* __restrict__ vals,
                                                      const double* __restrict__ C,
                                                      const double* __restrict__ D, int64_t K,
                                                      double* __restrict__ Avals,
                                                      const int64_t* __restrict__ counters) {
  // lane l owns k in [KT*l, KT*l + KT): NV 128-bit loads of D (and C) per
  // position (a single 64-bit load when KT == 1)
  static_assert(KT == 1 || KT == 2 || KT == 4 || KT == 8, "K must be 32, 64, 128 or 256");
  constexpr int NV = KT >= 2 ? KT / 2 : 1;
  const int lane = lane_id();
  z.m = nz_count(z);
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_stream = l2_policy_evict_first();
  const uint64_t pol_keep = l2_policy_evict_last();
  const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1;
  const int nchunks = (int)(end - begin);
  for (int t = (int)chunk_ticket(counters); t < nchunks; t = (int)chunk_ticket(counters)) {
    const ChunkInfo ci = chunk_info(g, begin + t, begin);
    if (ci.q_lo > ci.q_hi) continue;
    const int64_t s = ci.s, e = ci.e;
    NzCursor c;
    nz_start(z, c, s);
    int64_t cur_i = -1;
    double2 cr[NV];
#pragma unroll
    for (int w = 0; w < NV; w++) cr[w] = make_double2(0.0, 0.0);
    for (int64_t base = s; base <= e; base += 32) {
      const int cnt = (int)min((int64_t)32, e - base + 1);
      // crd with the hot-column bit (hot_crd): D columns referenced often
      // enough to stay in L2 are read with evict_last, the rest evict_first;
      // the whole warp reads one column at a time, so the policy is uniform.
      int my_j = 0;
      double my_b = 0.0;
      if (lane < cnt) {
        my_j = ld_i32_hint(crd32h + base + lane, pol_stream);
        my_b = ld_f64_hint(vals + base + lane, pol_stream);
      }
      const unsigned heads = nz_window_mask(c, base, base + cnt - 1);
      // row of this lane's position: rows starting at or before it
      const int kth = __popc(heads & (0xffffffffu >> (31 - lane)));
      const int64_t my_i = nz_get(c.I0, c.I1, (int)(c.ic - c.cb) + kth);
      double res = 0.0;
#pragma unroll 1
      for (int g4 = 0; g4 < cnt; g4 += 4) {
        double2 dd[4][NV];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int p = g4 + u;
          const int jh = __shfl_sync(FULL, my_j, p & 31);
          const int64_t j = jh & 0x7fffffff;
          const double* dp = D + j * K + KT * lane;
          // one column per load instruction: the policy is uniform per branch
#pragma unroll
          for (int w = 0; w < NV; w++) {
            if (p < cnt && jh < 0)
              dd[u][w] = KT == 1 ? make_double2(ld_f64_keep(dp, pol_keep), 0.0) : ld_f64x2_hint(dp + 2 * w, pol_keep);
            else if (p < cnt)
              dd[u][w] = KT == 1 ? make_double2(ld_f64_keep(dp, pol_stream), 0.0)
                                 : ld_f64x2_hint(dp + 2 * w, pol_stream);
            else
              dd[u][w] = make_double2(0.0, 0.0);
          }
        }
        double part[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int p = g4 + u;
          const int64_t i = __shfl_sync(FULL, my_i, p & 31);
          if (i != cur_i && p < cnt) {  // uniform: a new row's C slice
            const double* cp = C + i * K + KT * lane;
#pragma unroll
            for (int w = 0; w < NV; w++)
              cr[w] = KT == 1 ? make_double2(ld_f64_hint(cp, pol_stream), 0.0) : ld_f64x2_hint(cp + 2 * w, pol_stream);
            cur_i = i;
          }
          // the k's of this lane in ascending order, accumulated from the last
          double acc = cr[NV - 1].y * dd[u][NV - 1].y;
          acc = fma(cr[NV - 1].x, dd[u][NV - 1].x, acc);
#pragma unroll
          for (int w = NV - 2; w >= 0; w--) {
            acc = fma(cr[w].y, dd[u][w].y, acc);
            acc = fma(cr[w].x, dd[u][w].x, acc);
          }
          part[u] = acc;
        }
        // butterfly: four warp sums at once
        double a0 = b4 ? part[2] : part[0], a1 = b4 ? part[3] : part[1];
        const double s0 = b4 ? part[0] : part[2], s1 = b4 ? part[1] : part[3];
        a0 += __shfl_xor_sync(FULL, s0, 16);
        a1 += __shfl_xor_sync(FULL, s1, 16);
        double bsum = b3 ? a1 : a0;
        const double sb = b3 ? a0 : a1;
        bsum += __shfl_xor_sync(FULL, sb, 8);
        bsum += __shfl_xor_sync(FULL, bsum, 4);
        bsum += __shfl_xor_sync(FULL, bsum, 2);
        bsum += __shfl_xor_sync(FULL, bsum, 1);
        // lanes 8*v .. 8*v+7 hold the dot product of position g4 + v
        // (v = 2*b4 + b3); lane g4 + v collects it for the final store
        const double dot = __shfl_sync(FULL, bsum, ((lane - g4) & 3) * 8);
        if (lane >= g4 && lane < g4 + 4) res = dot;
      }
      if (lane < cnt) Avals[base + lane] = my_b * res;
      nz_advance(z, c, __popc(heads));
    }
  }
}

}  // namespace spd

namespace spd {
// jleaf[q] = crd1[fibre of q]: the middle-mode coordinate of every leaf.
__global__ void k_jleaf(const int64_t* __restrict__ rp2, const int64_t* __restrict__ crd1, int64_t F,
                        int32_t* __restrict__ jleaf) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = (int32_t)crd1[f];
    for (int64_t q = rp2[f]; q < rp2[f + 1]; q++) jleaf[q] = j;
  }
}
}  // namespace spd
