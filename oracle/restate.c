/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's hot path.
 * See restate.h for the contract.  Each function cites the reference code it
 * restates (paths relative to /root/reference/proj/core/src/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * load this library; the product never does. */
#include "restate.h"

#include <omp.h>
#include <stdlib.h>
#include <string.h>

static int threads_or_all(int nthreads) { return nthreads > 0 ? nthreads : omp_get_max_threads(); }

/* planner.cpp:10-20: truncating block, the last piece absorbs the remainder. */
void or_divide_bounds(int64_t n, int64_t pieces, int64_t* lo, int64_t* hi) {
  int64_t block = pieces > 0 ? n / pieces : 0;
  for (int64_t c = 0; c < pieces; c++) {
    lo[c] = c * block;
    hi[c] = c + 1 == pieces ? n - 1 : lo[c] + block - 1;
  }
}

/* tensor.cpp:258-281: non-empty ranges tile [0,nnz) in order, empties are the
 * canonical (k, k-1); then rowptr[p] = lo(p), rowptr[npos] = nnz. */
int or_pos_to_rowptr(const int64_t* pos_pairs, int64_t npos, int64_t nnz, int64_t* rowptr) {
  int64_t cursor = 0;
  for (int64_t p = 0; p < npos; p++) {
    int64_t lo = pos_pairs[2 * p], hi = pos_pairs[2 * p + 1];
    if (lo > hi) {
      if (lo != cursor || hi != cursor - 1) return 2;
    } else if (lo != cursor) {
      return 2;
    }
    rowptr[p] = cursor;
    if (lo <= hi) cursor = hi + 1;
  }
  rowptr[npos] = cursor;
  return cursor == nnz ? 0 : 2;
}

void or_rowptr_to_pos(const int64_t* rowptr, int64_t npos, int64_t* pos_pairs) {
  for (int64_t p = 0; p < npos; p++) {
    pos_pairs[2 * p] = rowptr[p];
    pos_pairs[2 * p + 1] = rowptr[p + 1] - 1;
  }
}

/* tensor.cpp:221-235: the entry whose (non-empty) range contains q, i.e. the
 * last p with rowptr[p] <= q (upper_bound - 1 skips the empty entries). */
int64_t or_owner(const int64_t* rowptr, int64_t npos, int64_t q) {
  int64_t lo = 0, hi = npos; /* search rowptr[0..npos] */
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (rowptr[mid] <= q) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

/* Universe split on the top dense level (level_partition.cpp:142-181), derived
 * down the tree by partition_from_parent (:214-232): pos = copy of the parent
 * colouring, crd = image (deppart.cpp:15-31), which on contiguous parents is
 * the contiguous range [rowptr[lo], rowptr[hi+1]-1]. */
void or_partition_universe(const int64_t* const* rowptrs, const int64_t* npos, int ncomp,
                           int64_t nrows, int64_t pieces, or_color* out) {
  int64_t* lo = malloc(sizeof(int64_t) * (pieces > 0 ? pieces : 1));
  int64_t* hi = malloc(sizeof(int64_t) * (pieces > 0 ? pieces : 1));
  or_divide_bounds(nrows, pieces, lo, hi);
  for (int64_t c = 0; c < pieces; c++) {
    or_color* o = &out[c];
    o->color_lo = o->top_lo = lo[c];
    o->color_hi = o->top_hi = hi[c];
    int64_t a = lo[c], b = hi[c]; /* positions of the current level, inclusive */
    int64_t pa = a, pb = b;
    for (int k = 0; k < ncomp; k++) {
      pa = a, pb = b; /* parent span of level k+1 */
      if (a > b) { /* empty stays empty, canonical at the image start */
        int64_t at = a <= npos[k] - 1 ? rowptrs[k][a] : rowptrs[k][npos[k]];
        a = at, b = at - 1;
      } else {
        int64_t na = rowptrs[k][a], nb = rowptrs[k][b + 1] - 1;
        a = na, b = nb;
      }
    }
    o->par_lo = pa, o->par_hi = pb;
    o->q_lo = a, o->q_hi = b;
  }
  free(lo);
  free(hi);
}

/* Nonzero split of the leaf level (level_partition.cpp:186-211): colour c owns
 * positions divide_bounds(nnz)[c]; pos partitions up the tree are preimages
 * (deppart.cpp:33-53 via partition_from_child :234-251), colouring exactly the
 * non-empty entries whose range meets the colour; project_to_universe
 * (planner.cpp:50-69) takes [min,max] of the coloured top positions, which on
 * a contiguous position range is the owner chain of q_lo and of q_hi. */
void or_partition_nonzero(const int64_t* const* rowptrs, const int64_t* npos, int ncomp,
                          int64_t nnz, int64_t pieces, or_color* out) {
  int64_t* lo = malloc(sizeof(int64_t) * (pieces > 0 ? pieces : 1));
  int64_t* hi = malloc(sizeof(int64_t) * (pieces > 0 ? pieces : 1));
  or_divide_bounds(nnz, pieces, lo, hi);
  for (int64_t c = 0; c < pieces; c++) {
    or_color* o = &out[c];
    o->color_lo = o->q_lo = lo[c];
    o->color_hi = o->q_hi = hi[c];
    if (lo[c] > hi[c]) {
      o->par_lo = o->top_lo = 0;
      o->par_hi = o->top_hi = -1;
      continue;
    }
    int64_t a = lo[c], b = hi[c];
    for (int k = ncomp - 1; k >= 0; k--) {
      a = or_owner(rowptrs[k], npos[k], a);
      b = or_owner(rowptrs[k], npos[k], b);
      if (k == ncomp - 1) o->par_lo = a, o->par_hi = b;
    }
    o->top_lo = a, o->top_hi = b;
  }
  free(lo);
  free(hi);
}

int64_t or_preimage_range(const int64_t* rowptr, int64_t npos, int64_t q_lo, int64_t q_hi,
                          int64_t* out, int64_t cap) {
  int64_t n = 0;
  if (q_lo > q_hi) return 0;
  for (int64_t p = 0; p < npos; p++) {
    int64_t s = rowptr[p], e = rowptr[p + 1] - 1;
    if (s > e) continue; /* deppart.cpp:46: empty ranges are never coloured */
    if (s <= q_hi && q_lo <= e) {
      if (out && n < cap) out[n] = p;
      n++;
    }
  }
  return n;
}

/* Stats::combines for colour partials over contiguous position ranges: a row
 * touched by k colours contributes (k-1) * entries (reduce_combine,
 * sim.cpp:797-808).  `owner_of(q)` maps a leaf position to its output row. */
typedef int64_t (*owner_fn)(const void* ctx, int64_t q);

static int64_t count_combines(const or_color* colors, int64_t pieces, owner_fn owner,
                              const void* ctx, int64_t entries_per_row) {
  int64_t combines = 0, prev_last = -1;
  int have_prev = 0;
  for (int64_t c = 0; c < pieces; c++) {
    if (colors[c].q_lo > colors[c].q_hi) continue;
    int64_t first = owner(ctx, colors[c].q_lo);
    if (have_prev && first == prev_last) combines += entries_per_row;
    prev_last = owner(ctx, colors[c].q_hi);
    have_prev = 1;
  }
  return combines;
}

typedef struct {
  const int64_t* rp;
  int64_t n;
  const int64_t* rp1;
  int64_t n1;
} owner_ctx;

static int64_t owner1(const void* v, int64_t q) {
  const owner_ctx* o = v;
  return or_owner(o->rp, o->n, q);
}
static int64_t owner2(const void* v, int64_t q) {
  const owner_ctx* o = v;
  return or_owner(o->rp1, o->n1, or_owner(o->rp, o->n, q));
}

static inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* SpMV leaf (plan_spmv_row.txt:28-33, plan_spmv_nonzero.txt:23-28): per colour,
 * each row's contributions in position order, value (1.0*B)*c (sim.cpp:328-337),
 * accumulated from 0.0 (:350); colours combined in ascending order (:797-808). */
int64_t or_spmv(int64_t n, const int64_t* rowptr, const int64_t* crd, const double* vals,
                const double* c, int64_t pieces, const or_color* colors, double* a,
                int64_t* work, int nthreads) {
  int nt = threads_or_all(nthreads);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = 0; i < n; i++) a[i] = 0.0;
  for (int64_t col = 0; col < pieces; col++) {
    int64_t q_lo = colors[col].q_lo, q_hi = colors[col].q_hi;
    if (work) work[col] = q_hi >= q_lo ? q_hi - q_lo + 1 : 0;
    if (q_lo > q_hi) continue;
    int64_t r0 = or_owner(rowptr, n, q_lo), r1 = or_owner(rowptr, n, q_hi);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
    for (int64_t r = r0; r <= r1; r++) {
      int64_t s = max64(rowptr[r], q_lo), e = min64(rowptr[r + 1] - 1, q_hi);
      if (s > e) continue;
      double partial = 0.0;
      for (int64_t q = s; q <= e; q++) partial += (1.0 * vals[q]) * c[crd[q]];
      a[r] += partial;
    }
  }
  owner_ctx oc = {rowptr, n, 0, 0};
  return count_combines(colors, pieces, owner1, &oc, 1);
}

/* SpMM: as SpMV with a dense inner loop over j in 0..N-1 (LeafVar Full). */
int64_t or_spmm(int64_t n, const int64_t* rowptr, const int64_t* crd, const double* vals,
                const double* C, int64_t N, int64_t pieces, const or_color* colors, double* A,
                int64_t* work, int nthreads) {
  int nt = threads_or_all(nthreads);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = 0; i < n * N; i++) A[i] = 0.0;
  for (int64_t col = 0; col < pieces; col++) {
    int64_t q_lo = colors[col].q_lo, q_hi = colors[col].q_hi;
    if (work) work[col] = q_hi >= q_lo ? (q_hi - q_lo + 1) * N : 0;
    if (q_lo > q_hi) continue;
    int64_t r0 = or_owner(rowptr, n, q_lo), r1 = or_owner(rowptr, n, q_hi);
#pragma omp parallel num_threads(nt)
    {
      double* partial = malloc(sizeof(double) * (N > 0 ? N : 1));
#pragma omp for schedule(dynamic, 1024)
      for (int64_t r = r0; r <= r1; r++) {
        int64_t s = max64(rowptr[r], q_lo), e = min64(rowptr[r + 1] - 1, q_hi);
        if (s > e) continue;
        for (int64_t j = 0; j < N; j++) partial[j] = 0.0;
        for (int64_t q = s; q <= e; q++) {
          double b = 1.0 * vals[q];
          const double* crow = C + crd[q] * N;
          for (int64_t j = 0; j < N; j++) partial[j] += b * crow[j];
        }
        double* arow = A + r * N;
        for (int64_t j = 0; j < N; j++) arow[j] += partial[j];
      }
      free(partial);
    }
  }
  owner_ctx oc = {rowptr, n, 0, 0};
  return count_combines(colors, pieces, owner1, &oc, N);
}

/* SDDMM: output positions are B's (pattern reuse, sim.cpp:656-663); each
 * position is owned by exactly one colour, so no combines. value
 * ((1.0*B)*C(i,k))*D(k,j) summed over k ascending. */
int64_t or_sddmm(int64_t n, const int64_t* rowptr, const int64_t* crd, const double* vals,
                 const double* C, const double* D, int64_t K, int64_t dk, int64_t dj,
                 int64_t pieces, const or_color* colors, double* A_vals, int64_t* work,
                 int nthreads) {
  int nt = threads_or_all(nthreads);
  int64_t nnz = rowptr[n];
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t q = 0; q < nnz; q++) A_vals[q] = 0.0;
  for (int64_t col = 0; col < pieces; col++) {
    int64_t q_lo = colors[col].q_lo, q_hi = colors[col].q_hi;
    if (work) work[col] = q_hi >= q_lo ? (q_hi - q_lo + 1) * K : 0;
    if (q_lo > q_hi) continue;
    int64_t r0 = or_owner(rowptr, n, q_lo), r1 = or_owner(rowptr, n, q_hi);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 256)
    for (int64_t r = r0; r <= r1; r++) {
      int64_t s = max64(rowptr[r], q_lo), e = min64(rowptr[r + 1] - 1, q_hi);
      const double* crow = C + r * K;
      for (int64_t q = s; q <= e; q++) {
        double b = 1.0 * vals[q];
        const double* dcol = D + crd[q] * dj;
        double partial = 0.0;
        for (int64_t k = 0; k < K; k++) partial += (b * crow[k]) * dcol[k * dk];
        A_vals[q] += partial;
      }
    }
  }
  return 0;
}

/* SpTTV over a dss CSF: output vals per (i,j) fiber (pattern reuse of B's
 * first two levels); boundary fibers combine across colours. */
int64_t or_spttv(int64_t I, const int64_t* rp1, const int64_t* crd1, const int64_t* rp2,
                 const int64_t* crd2, const double* vals, const double* c, int64_t pieces,
                 const or_color* colors, double* A_vals, int64_t* work, int nthreads) {
  (void)crd1;
  int nt = threads_or_all(nthreads);
  int64_t F = rp1[I];
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t f = 0; f < F; f++) A_vals[f] = 0.0;
  for (int64_t col = 0; col < pieces; col++) {
    int64_t q_lo = colors[col].q_lo, q_hi = colors[col].q_hi;
    if (work) work[col] = q_hi >= q_lo ? q_hi - q_lo + 1 : 0;
    if (q_lo > q_hi) continue;
    int64_t f0 = or_owner(rp2, F, q_lo), f1 = or_owner(rp2, F, q_hi);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
    for (int64_t f = f0; f <= f1; f++) {
      int64_t s = max64(rp2[f], q_lo), e = min64(rp2[f + 1] - 1, q_hi);
      if (s > e) continue;
      double partial = 0.0;
      for (int64_t q = s; q <= e; q++) partial += (1.0 * vals[q]) * c[crd2[q]];
      A_vals[f] += partial;
    }
  }
  owner_ctx oc = {rp2, F, 0, 0};
  return count_combines(colors, pieces, owner1, &oc, 1);
}

/* SpMTTKRP over a dss CSF: A(i,l) += ((1.0*B)*C(j,l))*D(k,l) in position order. */
int64_t or_spmttkrp(int64_t I, const int64_t* rp1, const int64_t* crd1, const int64_t* rp2,
                    const int64_t* crd2, const double* vals, const double* C, const double* D,
                    int64_t R, int64_t pieces, const or_color* colors, double* A, int64_t* work,
                    int nthreads) {
  int nt = threads_or_all(nthreads);
  int64_t F = rp1[I];
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = 0; i < I * R; i++) A[i] = 0.0;
  for (int64_t col = 0; col < pieces; col++) {
    int64_t q_lo = colors[col].q_lo, q_hi = colors[col].q_hi;
    if (work) work[col] = q_hi >= q_lo ? (q_hi - q_lo + 1) * R : 0;
    if (q_lo > q_hi) continue;
    int64_t f0 = or_owner(rp2, F, q_lo), f1 = or_owner(rp2, F, q_hi);
    int64_t i0 = or_owner(rp1, I, f0), i1 = or_owner(rp1, I, f1);
#pragma omp parallel num_threads(nt)
    {
      double* partial = malloc(sizeof(double) * (R > 0 ? R : 1));
#pragma omp for schedule(dynamic, 64)
      for (int64_t i = i0; i <= i1; i++) {
        int64_t fs = max64(rp1[i], f0), fe = min64(rp1[i + 1] - 1, f1);
        int touched = 0;
        for (int64_t l = 0; l < R; l++) partial[l] = 0.0;
        for (int64_t f = fs; f <= fe; f++) {
          int64_t s = max64(rp2[f], q_lo), e = min64(rp2[f + 1] - 1, q_hi);
          const double* crow = C + crd1[f] * R;
          for (int64_t q = s; q <= e; q++) {
            double b = 1.0 * vals[q];
            const double* drow = D + crd2[q] * R;
            for (int64_t l = 0; l < R; l++) partial[l] += (b * crow[l]) * drow[l];
            touched = 1;
          }
        }
        if (!touched) continue;
        double* arow = A + i * R;
        for (int64_t l = 0; l < R; l++) arow[l] += partial[l];
      }
      free(partial);
    }
  }
  owner_ctx oc = {rp2, F, rp1, I};
  return count_combines(colors, pieces, owner2, &oc, R);
}

/* SpAdd3 phase 1: per row, |union| of the three sorted crd lists
 * (iterate_coords + union_merge, sim.cpp:46-66, 389-454; two-phase count
 * sim.cpp:696-732). */
int64_t or_spadd3_count(int64_t n, const int64_t* const rp[3], const int64_t* const crd[3],
                        int64_t* A_rowptr, int nthreads) {
  int nt = threads_or_all(nthreads);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; r++) {
    int64_t at[3], end[3], cnt = 0;
    for (int t = 0; t < 3; t++) at[t] = rp[t][r], end[t] = rp[t][r + 1];
    for (;;) {
      int64_t next = INT64_MAX;
      for (int t = 0; t < 3; t++)
        if (at[t] < end[t] && crd[t][at[t]] < next) next = crd[t][at[t]];
      if (next == INT64_MAX) break;
      for (int t = 0; t < 3; t++)
        if (at[t] < end[t] && crd[t][at[t]] == next) at[t]++;
      cnt++;
    }
    A_rowptr[r + 1] = cnt;
  }
  A_rowptr[0] = 0;
  for (int64_t r = 0; r < n; r++) A_rowptr[r + 1] += A_rowptr[r];
  return A_rowptr[n];
}

/* SpAdd3 phase 2: fill; value = 0.0 + (((0.0 + B) + C) + D) over the present
 * terms in term order (accumulate sim.cpp:326-354, combine :806). */
void or_spadd3_fill(int64_t n, const int64_t* const rp[3], const int64_t* const crd[3],
                    const double* const vals[3], const int64_t* A_rowptr, int64_t* A_crd,
                    double* A_vals, int nthreads) {
  int nt = threads_or_all(nthreads);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; r++) {
    int64_t at[3], end[3], w = A_rowptr[r];
    for (int t = 0; t < 3; t++) at[t] = rp[t][r], end[t] = rp[t][r + 1];
    for (;;) {
      int64_t next = INT64_MAX;
      for (int t = 0; t < 3; t++)
        if (at[t] < end[t] && crd[t][at[t]] < next) next = crd[t][at[t]];
      if (next == INT64_MAX) break;
      double v = 0.0;
      for (int t = 0; t < 3; t++)
        if (at[t] < end[t] && crd[t][at[t]] == next) v += 1.0 * vals[t][at[t]++];
      A_crd[w] = next;
      A_vals[w] = 0.0 + v;
      w++;
    }
  }
}

double or_imbalance(const int64_t* work, int64_t workers) {
  int64_t total = 0, mx = 0;
  for (int64_t w = 0; w < workers; w++) {
    total += work[w];
    if (work[w] > mx) mx = work[w];
  }
  return total == 0 ? 1.0 : (double)mx * (double)workers / (double)total;
}
