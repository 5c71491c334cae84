/* TEST INFRASTRUCTURE ONLY -- the CPU restatement ("port") of the reference's
 * hot path, used as the full-scale parity checker and as bench.py's
 * cpu_baseline "port" leg.  Never linked into or called by the product.
 *
 * Parity of this restatement is PINNED against the patched reference
 * (oracle/_ref, built from /root/reference by oracle/Makefile) and against the
 * reference's own known-answer tests -- see tests/test_oracle_pins.py and
 * tests/golden/.
 *
 * Device-format conventions: a compressed level is an
 * int64 row pointer of (parent positions + 1) entries, lossless versus the
 * reference's inclusive (lo, hi) pos pairs (tensor.cpp:258-281); crd int64,
 * vals fp64.  Summation follows the reference exactly: every colour
 * accumulates its contributions in stored-position order from 0.0
 * (sim.cpp:326-354, 949-950) and colour partials are summed in ascending colour
 * order from 0.0 (reduce_combine, sim.cpp:791-811), so results are
 * bit-identical to the reference's execute().
 */
#ifndef SPD_ORACLE_RESTATE_H
#define SPD_ORACLE_RESTATE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One colour of one distributed loop, in compact (range) form.
 *   color_lo/hi: PlanLoop::color_bounds[c] (rows for universe, positions for nonzero)
 *   q_lo/hi:     leaf-level crd/vals positions owned (image / nonzero entry)
 *   par_lo/hi:   span of the split level's pos partition (the parent positions
 *                whose range meets [q_lo,q_hi]; preimage colours only the
 *                non-empty ones)
 *   top_lo/hi:   top-level coordinate bounds: the universe entry (row split) or
 *                project_to_universe's [min,max] (nonzero split) */
typedef struct {
  int64_t color_lo, color_hi;
  int64_t q_lo, q_hi;
  int64_t par_lo, par_hi;
  int64_t top_lo, top_hi;
} or_color;

/* planner.cpp:10-20 */
void or_divide_bounds(int64_t n, int64_t pieces, int64_t* lo, int64_t* hi);

/* tensor.cpp:241-286 (compressed-level invariants) then lossless pairs -> rowptr.
 * Returns 0 ok, 2 on a violated invariant. */
int or_pos_to_rowptr(const int64_t* pos_pairs, int64_t npos, int64_t nnz, int64_t* rowptr);
void or_rowptr_to_pos(const int64_t* rowptr, int64_t npos, int64_t* pos_pairs);

/* Parent entry whose range contains position q (tensor.cpp:221-235). */
int64_t or_owner(const int64_t* rowptr, int64_t npos, int64_t q);

/* Universe (row) split of a tree Dense(n) -> Compressed... with `ncomp`
 * compressed levels below: level_partition.cpp:142-181, partition_from_parent
 * :214-232 (copy + image, deppart.cpp:15-31). rowptrs[k] is compressed level k+1. */
void or_partition_universe(const int64_t* const* rowptrs, const int64_t* npos, int ncomp,
                           int64_t nrows, int64_t pieces, or_color* out);

/* Nonzero split of the leaf level: level_partition.cpp:186-211 (nonzero entry),
 * preimage deppart.cpp:33-53 / partition_from_child :234-251 up the tree,
 * project_to_universe planner.cpp:50-69. */
void or_partition_nonzero(const int64_t* const* rowptrs, const int64_t* npos, int ncomp,
                          int64_t nnz, int64_t pieces, or_color* out);

/* Exact preimage of a position range at one compressed level (deppart.cpp:33-53
 * with a contiguous destination subset): non-empty entries meeting [q_lo,q_hi].
 * Writes up to `cap` entries into out (may be NULL); returns the count. */
int64_t or_preimage_range(const int64_t* rowptr, int64_t npos, int64_t q_lo, int64_t q_hi,
                          int64_t* out, int64_t cap);

/* Leaf kernels over `pieces` colours + reduce_combine.  `work` (per colour,
 * may be NULL) is Stats::PerWorker::work (sim.cpp:352); the return value is
 * Stats::combines (sim.cpp:804). nthreads <= 0: all OpenMP threads. */

/* a(i) = B(i,j) * c(j); B CSR, a dense (n). */
int64_t or_spmv(int64_t n, const int64_t* rowptr, const int64_t* crd, const double* vals,
                const double* c, int64_t pieces, const or_color* colors, double* a,
                int64_t* work, int nthreads);

/* A(i,j) = B(i,k) * C(k,j); C dense K x N row-major, A dense n x N. */
int64_t or_spmm(int64_t n, const int64_t* rowptr, const int64_t* crd, const double* vals,
                const double* C, int64_t N, int64_t pieces, const or_color* colors, double* A,
                int64_t* work, int nthreads);

/* A(i,j) = B(i,j) * C(i,k) * D(k,j); A shares B's pattern (pattern reuse,
 * sim.cpp:571-606): A_vals has nnz entries.  C dense I x K row-major; D(k,j)
 * is read at D[k*dk + j*dj] (dd: dk=J,dj=1; dd:1,0: dk=1,dj=K). */
int64_t or_sddmm(int64_t n, const int64_t* rowptr, const int64_t* crd, const double* vals,
                 const double* C, const double* D, int64_t K, int64_t dk, int64_t dj,
                 int64_t pieces, const or_color* colors, double* A_vals, int64_t* work,
                 int nthreads);

/* A(i,j) = B(i,j,k) * c(k); B `dss` CSF (rp1: I+1 over fibers, crd1: F,
 * rp2: F+1 over leaves, crd2: nnz); A shares B's first two levels: F vals. */
int64_t or_spttv(int64_t I, const int64_t* rp1, const int64_t* crd1, const int64_t* rp2,
                 const int64_t* crd2, const double* vals, const double* c, int64_t pieces,
                 const or_color* colors, double* A_vals, int64_t* work, int nthreads);

/* A(i,l) = B(i,j,k) * C(j,l) * D(k,l); C: J x R, D: K x R, A: I x R dense. */
int64_t or_spmttkrp(int64_t I, const int64_t* rp1, const int64_t* crd1, const int64_t* rp2,
                    const int64_t* crd2, const double* vals, const double* C, const double* D,
                    int64_t R, int64_t pieces, const or_color* colors, double* A, int64_t* work,
                    int nthreads);

/* A = B + C + D, all CSR, row split (two-phase assembly, sim.cpp:676-788).
 * Phase 1 (count): returns nnz(A) and fills A_rowptr (n+1).  Phase 2 (fill):
 * A_crd / A_vals sized nnz(A).  Colours only decide `work` (rows are disjoint). */
int64_t or_spadd3_count(int64_t n, const int64_t* const rp[3], const int64_t* const crd[3],
                        int64_t* A_rowptr, int nthreads);
void or_spadd3_fill(int64_t n, const int64_t* const rp[3], const int64_t* const crd[3],
                    const double* const vals[3], const int64_t* A_rowptr, int64_t* A_crd,
                    double* A_vals, int nthreads);

/* Stats::imbalance (sim.cpp:997-1005). */
double or_imbalance(const int64_t* work, int64_t workers);

#ifdef __cplusplus
}
#endif
#endif
