// SpAdd3 leaf + two-phase assembly (K8): A = B + C + D over CSR operands.
//
// Reference: a coordinate-value loop over rows, the union of the three
// sorted crd lists per row (iterate_coords + union_merge, sim.cpp:46-66,
// 389-454), value ((0.0 + B) + C) + D over the present terms in term order
// (accumulate, sim.cpp:326-354), then two-phase assembly: a symbolic count
// sizes pos/crd exactly and a fill pass writes them (sim.cpp:676-788).
//
// B200 design -- rank-based union, element-parallel so hub rows of power-law
// matrices split evenly over threads instead of serialising a merge:
//   flags   fC[p] = C's element p is absent from B's row; fD[p] = D's element
//           is absent from B's and C's rows (binary searches inside the row);
//   count   exclusive scans PC, PD of the flags; then with no further pass
//           A.rowptr[i] = rpB[i] + PC[rpC[i]] + PD[rpD[i]] -- the symbolic
//           phase of the two-phase assembly, exact by construction;
//   fill    every element that is first in term order (all of B, flagged C
//           and D) computes its rank in the row union from its index and two
//           searches + prefix lookups, and writes crd and the summed value.
// The pattern is the structural union (explicit zeros kept, P6), crd sorted,
// empties canonical -- bit-exact with the reference; values are exact because
// each output sums the same terms in the same order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace spd {

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

// Row of position p (owner search; p < nnz).
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ rp, int64_t n, int64_t p) {
  int64_t lo = 0, hi = n;  // last i with rp[i] <= p
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(rp + mid) <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Flags for the positions of X in rows [r_lo, r_hi]; `against` 1 or 2 tensors.
__global__ void k_flags(Csr X, int64_t n, int64_t p_lo, int64_t p_hi, Csr A1, Csr A2, int use2,
                        int32_t* __restrict__ flags) {
  for (int64_t p = p_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= p_hi;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row_of(X.rp, n, p);
    const int64_t x = __ldg(X.crd + p);
    int64_t a0 = __ldg(A1.rp + i), a1 = __ldg(A1.rp + i + 1);
    int64_t k = lb(A1.crd, a0, a1, x);
    bool present = k < a1 && __ldg(A1.crd + k) == x;
    if (use2 && !present) {
      int64_t b0 = __ldg(A2.rp + i), b1 = __ldg(A2.rp + i + 1);
      int64_t k2 = lb(A2.crd, b0, b1, x);
      present = k2 < b1 && __ldg(A2.crd + k2) == x;
    }
    flags[p] = present ? 0 : 1;
  }
}

__global__ void k_rowptr_union(const int64_t* __restrict__ rpB, const int64_t* __restrict__ rpC,
                               const int64_t* __restrict__ rpD, const int64_t* __restrict__ PC,
                               const int64_t* __restrict__ PD, int64_t n,
                               int64_t* __restrict__ rpA) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    rpA[i] = rpB[i] + PC[rpC[i]] + PD[rpD[i]];
}

// Fill for the elements of term t (0 B, 1 C, 2 D) in positions [p_lo, p_hi].
__global__ void k_fill(int t, Csr B, Csr C, Csr D, int64_t n, int64_t p_lo, int64_t p_hi,
                       const int32_t* __restrict__ fC, const int32_t* __restrict__ fD,
                       const int64_t* __restrict__ PC, const int64_t* __restrict__ PD,
                       const int64_t* __restrict__ rpA, int64_t* __restrict__ Acrd,
                       double* __restrict__ Avals) {
  const Csr& X = t == 0 ? B : (t == 1 ? C : D);
  for (int64_t p = p_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= p_hi;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (t == 1 && !fC[p]) continue;
    if (t == 2 && !fD[p]) continue;
    const int64_t i = row_of(X.rp, n, p);
    const int64_t x = __ldg(X.crd + p);
    const int64_t b0 = __ldg(B.rp + i), b1 = __ldg(B.rp + i + 1);
    const int64_t c0 = __ldg(C.rp + i), c1 = __ldg(C.rp + i + 1);
    const int64_t d0 = __ldg(D.rp + i), d1 = __ldg(D.rp + i + 1);
    int64_t rank = 0;
    double v = 0.0;
    // B part: elements of B below x, and B's value at x
    int64_t kb = t == 0 ? p : lb(B.crd, b0, b1, x);
    rank += kb - b0;
    if (t == 0) v += 1.0 * __ldg(B.vals + p);
    // C part: C elements below x that are not in B, and C's value at x
    int64_t kc = t == 1 ? p : lb(C.crd, c0, c1, x);
    rank += PC[kc] - PC[c0];
    if (t == 1) v += 1.0 * __ldg(C.vals + p);
    else if (t == 0 && kc < c1 && __ldg(C.crd + kc) == x) v += 1.0 * __ldg(C.vals + kc);
    // D part
    int64_t kd = t == 2 ? p : lb(D.crd, d0, d1, x);
    rank += PD[kd] - PD[d0];
    if (t == 2) v += 1.0 * __ldg(D.vals + p);
    else if (kd < d1 && __ldg(D.crd + kd) == x) v += 1.0 * __ldg(D.vals + kd);
    const int64_t o = __ldg(rpA + i) + rank;
    Acrd[o] = x;
    Avals[o] = 0.0 + v;
  }
}

static int grid_n(spd_context* ctx, int64_t n) {
  int64_t g = ceil_div(n, 256);
  int64_t cap = (int64_t)ctx->num_sms * 16;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

static void exclusive_scan(spd_context* ctx, const int32_t* flags, int64_t n, int64_t* out,
                           DeviceBuffer& tmp) {
  // out has n + 1 entries: out[0] = 0, out[p+1] = sum flags[0..p]
  SPD_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), ctx->stream));
  if (n == 0) return;
  size_t bytes = 0;
  SPD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, flags, out + 1, n, ctx->stream));
  void* t = tmp.reserve(bytes);
  SPD_CUDA(cub::DeviceScan::InclusiveSum(t, bytes, flags, out + 1, n, ctx->stream));
}

static void run_spadd3(spd_context* ctx, const spd_tensor* B, const spd_tensor* C,
                       const spd_tensor* D, spd_tensor** A_out, int64_t first, int64_t count,
                       spd_stats* stats) {
  checked(ctx);
  if (!B || !C || !D || !A_out) throw ValidationError("null argument");
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
  if (ctx->comm && count == 1 && ctx->pieces > 1)
    throw ValidationError("unsupported on gpu: multi-GPU SpAdd3 assembly is not implemented yet");
  const int64_t n = B->levels[1].parent_positions;
  Csr b{B->levels[1].rowptr, B->levels[1].crd, B->vals};
  Csr c{C->levels[1].rowptr, C->levels[1].crd, C->vals};
  Csr d{D->levels[1].rowptr, D->levels[1].crd, D->vals};
  const int64_t nb = B->levels[1].positions, nc = C->levels[1].positions,
                nd = D->levels[1].positions;
  cudaStream_t s = ctx->stream;
  int64_t launches = 0;
  if (stats) SPD_CUDA(cudaEventRecord(ctx->ev0, s));
  int32_t* fC = (int32_t*)ctx->scratch[0].reserve(sizeof(int32_t) * (nc + 1));
  int32_t* fD = (int32_t*)ctx->scratch[1].reserve(sizeof(int32_t) * (nd + 1));
  int64_t* PC = (int64_t*)ctx->scratch[2].reserve(sizeof(int64_t) * (nc + 1));
  int64_t* PD = (int64_t*)ctx->scratch[3].reserve(sizeof(int64_t) * (nd + 1));
  if (nc > 0) {
    k_flags<<<grid_n(ctx, nc), 256, 0, s>>>(c, n, 0, nc - 1, b, b, 0, fC);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  if (nd > 0) {
    k_flags<<<grid_n(ctx, nd), 256, 0, s>>>(d, n, 0, nd - 1, b, c, 1, fD);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  exclusive_scan(ctx, fC, nc, PC, ctx->scratch[5]);
  exclusive_scan(ctx, fD, nd, PD, ctx->scratch[5]);
  launches += 2;
  // Phase 1 (symbolic): A's row pointer.
  int64_t* rpA = nullptr;
  SPD_CUDA(cudaMallocAsync((void**)&rpA, sizeof(int64_t) * (n + 1), s));
  k_rowptr_union<<<grid_n(ctx, n + 1), 256, 0, s>>>(b.rp, c.rp, d.rp, PC, PD, n, rpA);
  SPD_CHECK_LAUNCH();
  launches++;
  int64_t nnzA = 0;
  SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters, rpA + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  nnzA = ctx->pinned_counters[0];
  // Phase 2 (fill): exactly-sized buffers.
  int64_t* Acrd = nullptr;
  double* Avals = nullptr;
  SPD_CUDA(cudaMallocAsync((void**)&Acrd, sizeof(int64_t) * (nnzA > 0 ? nnzA : 1), s));
  SPD_CUDA(cudaMallocAsync((void**)&Avals, sizeof(double) * (nnzA > 0 ? nnzA : 1), s));
  const int64_t np[3] = {nb, nc, nd};
  leaf_timing_begin(ctx);
  for (int t = 0; t < 3; t++) {
    if (np[t] == 0) continue;
    k_fill<<<grid_n(ctx, np[t]), 256, 0, s>>>(t, b, c, d, n, 0, np[t] - 1, fC, fD, PC, PD, rpA,
                                               Acrd, Avals);
    SPD_CHECK_LAUNCH();
    launches++;
  }
  leaf_timing_end(ctx);
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
  *A_out = A;
  if (stats) {
    SPD_CUDA(cudaEventRecord(ctx->ev1, s));
    const auto& hc = host_colors(ctx);
    // work = contributions summed per colour: sum of the three inputs' stored
    // entries in the colour's rows (sim.cpp:352).
    std::vector<int64_t> work(ctx->pieces, 0);
    std::vector<int64_t> rb(n + 1), rc(n + 1), rd(n + 1);
    SPD_CUDA(cudaMemcpy(rb.data(), b.rp, 8 * (n + 1), cudaMemcpyDeviceToHost));
    SPD_CUDA(cudaMemcpy(rc.data(), c.rp, 8 * (n + 1), cudaMemcpyDeviceToHost));
    SPD_CUDA(cudaMemcpy(rd.data(), d.rp, 8 * (n + 1), cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < ctx->pieces; k++) {
      int64_t lo = hc[k].top.lo, hi = hc[k].top.hi;
      if (lo > hi) continue;
      work[k] = (rb[hi + 1] - rb[lo]) + (rc[hi + 1] - rc[lo]) + (rd[hi + 1] - rd[lo]);
    }
    fill_stats(ctx, stats, 0, work, launches, true);
  }
}

}  // namespace spd

using namespace spd;

extern "C" int spd_spadd3(spd_context* ctx, const spd_tensor* B, const spd_tensor* C,
                          const spd_tensor* D, spd_tensor** A_out, int64_t first_color,
                          int64_t ncolors, spd_stats* stats) {
  return guarded([&] { run_spadd3(ctx, B, C, D, A_out, first_color, ncolors, stats); });
}
