// SDDMM leaf (K5): A(i,j) = B(i,j) * C(i,k) * D(k,j) on B's pattern.
//
// The output shares B's pos/crd (pattern reuse, pattern_reuse_source
// sim.cpp:571-606) so only vals are written, one per stored position, and no
// position is owned by two colours (the reference reports combines == 0).
// Reference leaf: for every position of the colour, sum over k of
// ((1.0*B)*C(i,k))*D(k,j) (sim.cpp:328-337); here B * sum_k C(i,k)*D(k,j),
// a reassociation within north_star's 1e-10 relative.
//
// One warp per chunk of positions; lane l owns k = l, l+32, ...: the C row of
// the current i stays in registers while the row lasts, each position gathers
// the K-long D column j (contiguous when D is stored j-major, "dd:1,0") with
// coalesced 256-byte loads, KT-deep in flight, and a warp sum finishes the
// dot product.  Results of 32 positions are written with one coalesced store.
#include "rowwalk.cuh"

namespace spd {

#define FULL 0xffffffffu

void launch_setup(cudaStream_t s, DevColor* cols, int64_t P, int split, int out_level, const int64_t* R,
                  int64_t nrows, int64_t CH, int64_t c_first, int64_t c_count, int64_t* counters, int64_t* ff0,
                  int64_t n0, int64_t* ff1, int64_t n1);

bool sddmm_nz_launch(spd_context* ctx, const spd_tensor* B, const WalkGeom& g, const double* C,
                     const double* D, int64_t K, int64_t dk, int64_t dj, double* Avals,
                     const int64_t* counters);

template <int KT>
__global__ void __launch_bounds__(kBlock) k_sddmm_walk(WalkGeom g, const int64_t* __restrict__ crd,
                                                       const double* __restrict__ vals,
                                                       const double* __restrict__ C,
                                                       const double* __restrict__ D, int64_t K,
                                                       int64_t dk, int64_t dj,
                                                       double* __restrict__ Avals,
                                                       const int64_t* __restrict__ counters) {
  const int lane = lane_id();
  const int64_t begin = counters[1], end = counters[2];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int U = 4;
  for (int64_t v = begin + chunk_ticket(counters); v < end; v = begin + chunk_ticket(counters)) {
    const ChunkInfo ci = chunk_info(g, v, begin);
    if (ci.q_lo > ci.q_hi) continue;
    const int64_t s = ci.s, e = ci.e;
    int64_t r = warp_owner(g.R, g.nrows, s);
    int64_t nb = ld64(g.R + r + 1);
    double cr[KT];
#pragma unroll
    for (int t = 0; t < KT; t++) {
      const int64_t kk = lane + 32 * t;
      cr[t] = kk < K ? __ldg(C + r * K + kk) : 0.0;
    }
    for (int64_t base = s; base <= e; base += 32) {
      const int cnt = (int)min((int64_t)32, e - base + 1);
      int64_t my_j = 0;
      double my_b = 0.0, res = 0.0;
      if (lane < cnt) {
        my_j = ld64(crd + base + lane);
        my_b = __ldg(vals + base + lane);
      }
      for (int u0 = 0; u0 < cnt; u0 += U) {
        double dv[U][KT];
#pragma unroll
        for (int i = 0; i < U; i++) {
          const int64_t jj = __shfl_sync(FULL, my_j, (u0 + i) & 31);
#pragma unroll
          for (int t = 0; t < KT; t++) {
            const int64_t kk = lane + 32 * t;
            dv[i][t] = (u0 + i < cnt && kk < K) ? __ldg(D + jj * dj + kk * dk) : 0.0;
          }
        }
#pragma unroll
        for (int i = 0; i < U; i++) {
          if (u0 + i < cnt) {
            const int64_t q = base + u0 + i;
            if (q == nb) {  // next non-empty row starting at q
              int64_t nbn;
              r = skip_empty_rows(g, r + 1, q, nbn, Avals, 1, 0);
              nb = nbn;
#pragma unroll
              for (int t = 0; t < KT; t++) {
                const int64_t kk = lane + 32 * t;
                cr[t] = kk < K ? __ldg(C + r * K + kk) : 0.0;
              }
            }
            double dot = 0.0;
#pragma unroll
            for (int t = 0; t < KT; t++) dot = fma(cr[t], dv[i][t], dot);
            dot = warp_sum(dot);
            const double b = __shfl_sync(FULL, my_b, u0 + i);
            if (lane == u0 + i) res = b * dot;
          }
        }
      }
      if (lane < cnt) Avals[base + lane] = res;
    }
  }
}

template <class Kern>
static int grid_of(spd_context* ctx, Kern k) {
  int per_sm = 0;
  SPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBlock, 0));
  return ctx->num_sms * (per_sm > 0 ? per_sm : 1);
}

static void run_sddmm(spd_context* ctx, const spd_tensor* B, const double* C, const double* D,
                      int64_t K, int64_t dk, int64_t dj, double* Avals, int64_t first,
                      int64_t count, spd_stats* stats) {
  checked(ctx);
  if (!B) throw ValidationError("null tensor");
  settle_restage(B);
  require_partition(ctx, B, first, count);
  activate(ctx);
  if (B->levels.size() != 2 || B->levels[0].kind != SPD_DENSE ||
      B->levels[1].kind != SPD_COMPRESSED)
    throw ValidationError("unsupported on gpu: SDDMM needs a ds (CSR-like) matrix");
  require_identity_order(B, "the sparse operand");
  if (ctx->split == SplitKind::NonZero && ctx->split_level != 1)
    throw ValidationError("unsupported on gpu: nonzero split must be on the leaf level");
  if (K < 0 || K > 256) throw ValidationError("unsupported on gpu: K must be in [0, 256]");
  const int64_t P = ctx->pieces;
  const spd_level_store& L = B->levels[1];
  WalkGeom g;
  g.R = L.rowptr;
  g.nrows = L.parent_positions;
  g.cols = (const DevColor*)ctx->colors_dev.ptr;
  g.c_first = first;
  g.c_count = count;
  g.CH = 512;
  g.W = 1;
  int64_t* counters = (int64_t*)ctx->scratch[4].reserve(sizeof(int64_t) * 4);
  cudaStream_t s = ctx->stream;
  int64_t launches = 0;
  if (stats) SPD_CUDA(cudaEventRecord(ctx->ev0, s));
  launch_setup(s, (DevColor*)ctx->colors_dev.ptr, P, (int)ctx->split, 0, g.R, g.nrows, g.CH, first, count, counters,
               nullptr, 0, nullptr, 0);
  launches += 2;
  const int64_t kt = ceil_div(K > 0 ? K : 1, 32);
  leaf_timing_begin(ctx);
  if (sddmm_nz_launch(ctx, B, g, C, D, K, dk, dj, Avals, counters)) {
  } else
#define SDDMM_CASE(KT_)                                                                    \
  {                                                                                        \
    static int grid = 0;                                                                   \
    if (!grid) grid = grid_of(ctx, k_sddmm_walk<KT_>);                                     \
    k_sddmm_walk<KT_><<<grid, kBlock, 0, s>>>(g, L.crd, B->vals, C, D, K, dk, dj, Avals,   \
                                              counters);                                   \
  }
  if (kt <= 1) SDDMM_CASE(1)
  else if (kt <= 2) SDDMM_CASE(2)
  else if (kt <= 4) SDDMM_CASE(4)
  else SDDMM_CASE(8)
#undef SDDMM_CASE
  SPD_CHECK_LAUNCH();
  leaf_timing_end(ctx);
  launches++;
  ctx->launches += launches;
  if (stats) {
    SPD_CUDA(cudaEventRecord(ctx->ev1, s));
    const auto& hc = host_colors(ctx);
    std::vector<int64_t> work(P);
    for (int64_t c = 0; c < P; c++)
      work[c] = hc[c].q.lo <= hc[c].q.hi ? (hc[c].q.hi - hc[c].q.lo + 1) * K : 0;
    fill_stats(ctx, stats, 0, work, launches, true);
  }
}

}  // namespace spd

using namespace spd;

extern "C" int spd_sddmm(spd_context* ctx, const spd_tensor* B, const double* C_dev,
                         const double* D_dev, int64_t K, int64_t dk, int64_t dj,
                         double* Avals_dev, int64_t first_color, int64_t ncolors,
                         spd_stats* stats) {
  return guarded([&] {
    run_sddmm(ctx, B, C_dev, D_dev, K, dk, dj, Avals_dev, first_color, ncolors, stats);
  });
}
