// Chunked row walks: the execution skeleton shared by the row-reducing leaf
// kernels (SpMV, SpMM, SpTTV, SpMTTKRP).
//
// The reference runs one task per colour (sim.cpp:864-956): each accumulates
// its contributions in stored-position order into a private dense
// accumulator (sim.cpp:326-354, 949-950) and reduce_combine sums the
// partials in ascending colour order (sim.cpp:791-811).  Here a colour's
// leaf positions [q.lo, q.hi] are cut into fixed-size chunks of CH positions,
// one warp per chunk (persistent grid-stride), so hub rows of power-law
// matrices are split across warps and every warp streams the same number of
// positions.  Rows that a chunk holds entirely are stored directly; a row cut
// by a chunk boundary leaves a "head" record (row began before the chunk) and
// / or a "tail" record (row continues after it).  A fixup pass sums each
// row's records in chunk order, and rows cut by a colour boundary become
// colour records that the colour combine (K9) sums in ascending colour order
// -- over NCCL when the colours live on different GPUs.  Every step has a
// fixed order, so results are bit-reproducible run to run.
//
// Output ownership: colour c stores exactly the output rows
// W_c = [w_lo, w_hi]; the W_c tile [0, rows) in order.  For a universe split
// W_c is the colour's own row block; for a nonzero split W_c runs from the
// first row starting inside the colour to the row before the next colour's
// first such row, so a row cut between colours belongs to the colour where it
// starts and empty rows belong to the colour holding the position just before
// them.  Untouched (empty) rows are stored as 0.0, like assemble_output's
// all-dense path (sim.cpp:665-674).
#pragma once

#include "common.cuh"

namespace spd {

constexpr int kBlock = 256;

struct ChunkRecs {
  int64_t* row;  // [2*nchunks]: head row, tail row (-1: none)
  int* cont;     // [nchunks]: head record continues past the chunk end
  double* val;   // [2*nchunks*W]
};

struct ColorRecs {
  // Packed head records, one per colour: [row, cont, val[0..W)] as 8-byte
  // slots -- the unit the multi-GPU combine all-gathers.
  int64_t* head_pack;  // [P*(W+2)]
  int64_t* tail_row;   // [P]
  double* tail_val;    // [P*W]
  int64_t* counters;   // [0]: combines, [1]: chunk range begin, [2]: chunk range end
};

struct WalkGeom {
  const int64_t* __restrict__ R;  // output rows -> leaf positions (nrows + 1)
  int64_t nrows;
  const DevColor* __restrict__ cols;
  int64_t c_first, c_count;
  int64_t CH;
  int64_t W;  // values per output row
};

__device__ __forceinline__ int64_t ld64(const int64_t* p) { return __ldg(p); }

// Colour of virtual chunk v among [c_first, c_first + c_count).
__device__ __forceinline__ int64_t colour_of_chunk(const WalkGeom& g, int64_t v) {
  int64_t lo = g.c_first, hi = g.c_first + g.c_count - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (g.cols[mid].chunk_begin <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Stores zeros into rows [a, b] (contiguous W-wide rows), warp-cooperative.
__device__ __forceinline__ void zero_rows(double* __restrict__ out, int64_t W, int64_t a,
                                         int64_t b) {
  if (a > b) return;
  const int lane = lane_id();
  for (int64_t i = a * W + lane; i < (b + 1) * W; i += 32) out[i] = 0.0;
}

// Rows r, r+1, ... all start at position q.  Zeroes the empty ones inside
// [w_lo, w_hi] and returns the first non-empty row; *nb receives its end
// (exclusive).  Returns nrows (nb = INT64_MAX) when no row follows.
__device__ __forceinline__ int64_t skip_empty_rows(const WalkGeom& g, int64_t r, int64_t q,
                                                   int64_t& nb, double* __restrict__ out,
                                                   int64_t w_lo, int64_t w_hi) {
  const int lane = lane_id();
  for (;;) {
    int64_t idx = r + 1 + lane;
    int64_t x = idx <= g.nrows ? ld64(g.R + idx) : INT64_MAX;
    unsigned m = __ballot_sync(0xffffffffu, x == q);
    int run = m == 0xffffffffu ? 32 : __ffs(~m) - 1;
    int64_t za = max(r, w_lo), zb = min(r + run - 1, w_hi);
    zero_rows(out, g.W, za, zb);
    if (run < 32) {
      nb = __shfl_sync(0xffffffffu, x, run);
      return r + run < g.nrows ? r + run : g.nrows;
    }
    r += 32;
  }
}

// Resolves the chunk handled by virtual chunk index v.
struct ChunkInfo {
  int64_t colour, s, e, q_lo, q_hi, w_lo, w_hi, local;
};
__device__ __forceinline__ ChunkInfo chunk_info(const WalkGeom& g, int64_t v, int64_t begin) {
  ChunkInfo ci;
  ci.colour = colour_of_chunk(g, v);
  const DevColor& d = g.cols[ci.colour];
  ci.q_lo = d.pub.q.lo;
  ci.q_hi = d.pub.q.hi;
  ci.w_lo = d.w_lo;
  ci.w_hi = d.w_hi;
  ci.s = ci.q_lo + (v - d.chunk_begin) * g.CH;
  ci.e = min(ci.s + g.CH - 1, ci.q_hi);
  ci.local = v - begin;
  return ci;
}

// Next chunk ticket of a warp (lane 0 draws, the warp shares it).
__device__ __forceinline__ int64_t chunk_ticket(const int64_t* counters) {
  unsigned long long t = 0;
  if ((threadIdx.x & 31) == 0)
    t = atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<int64_t*>(counters) + 3), 1ull);
  return (int64_t)__shfl_sync(0xffffffffu, t, 0);
}

}  // namespace spd
