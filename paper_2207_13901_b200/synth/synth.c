/* Deterministic synthetic inputs for the BASELINE configs.
 *
 * Counter-based hashing (splitmix64 of seed, stream, index) makes every
 * generator order-independent and thread-count-independent, so the GPU
 * bench, the CPU oracle and the tests all see identical arrays.  Duplicate
 * coordinates are summed in generation order, the semantics of
 * SparseTensor::pack (tensor.cpp:100-113); coordinates are sorted in storage
 * order and packed into device format (int64 row pointers, crd, fp64 vals).
 *
 *   uniform CSR      n x m, `samples` (row, col) draws         (config 1)
 *   R-MAT CSR        Graph500 recursive matrix, scale s, edges   (configs 2/3/5)
 *   power-law CSF    I x J x K `dss`, coordinates floor(N*u^3)   (config 4)
 *   dense operands   fp64 U[0.5, 1.5) or small integers {1..8}
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t i) {
  return splitmix64(splitmix64(seed * 0x100000001B3ull ^ stream) ^ (i * 0xD6E8FEB86659FD93ull));
}
static inline double unit53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

/* value kinds: 0 -> U[0.5,1.5), 1 -> integers {1..8} */
static inline double value_of(uint64_t seed, uint64_t stream, uint64_t i, int kind) {
  uint64_t h = hash3(seed, stream, i);
  return kind ? (double)(1 + (h >> 61)) : 0.5 + unit53(h);
}

void syn_dense(int64_t n, uint64_t seed, int kind, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) out[i] = value_of(seed, 7, (uint64_t)i, kind);
}

/* ---- COO -> CSR with pack semantics -------------------------------------- */
typedef struct {
  int64_t col;
  double val;
  int64_t order; /* generation index: duplicates sum in this order */
} ent;

static int ent_cmp(const void* a, const void* b) {
  const ent* x = a;
  const ent* y = b;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return x->order < y->order ? -1 : (x->order > y->order);
}

/* Sorts each row by column (stable in generation order), sums duplicates.
 * rows/cols/vals: `cnt` entries.  Outputs rowptr (n+1); returns nnz and
 * writes crd/vals into caller buffers sized >= cnt. */
static int64_t coo_to_csr(int64_t n, int64_t cnt, const int64_t* rows, const int64_t* cols,
                          const double* vals, int64_t* rowptr, int64_t* crd, double* out_vals) {
  int64_t* start = calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < cnt; e++) start[rows[e] + 1]++;
  for (int64_t i = 0; i < n; i++) start[i + 1] += start[i];
  ent* buf = malloc(sizeof(ent) * (size_t)(cnt > 0 ? cnt : 1));
  int64_t* fill = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(fill, start, sizeof(int64_t) * (size_t)n);
  for (int64_t e = 0; e < cnt; e++) {
    int64_t at = fill[rows[e]]++;
    buf[at].col = cols[e];
    buf[at].val = vals[e];
    buf[at].order = e;
  }
  free(fill);
  int64_t* uniq = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; i++) {
    ent* r = buf + start[i];
    int64_t len = start[i + 1] - start[i];
    if (len > 1) qsort(r, (size_t)len, sizeof(ent), ent_cmp);
    int64_t u = 0;
    for (int64_t k = 0; k < len; k++) {
      if (u > 0 && r[u - 1].col == r[k].col) {
        r[u - 1].val += r[k].val;
      } else {
        r[u++] = r[k];
      }
    }
    uniq[i] = u;
  }
  rowptr[0] = 0;
  for (int64_t i = 0; i < n; i++) rowptr[i + 1] = rowptr[i] + uniq[i];
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; i++) {
    const ent* r = buf + start[i];
    for (int64_t k = 0; k < uniq[i]; k++) {
      crd[rowptr[i] + k] = r[k].col;
      out_vals[rowptr[i] + k] = r[k].val;
    }
  }
  int64_t nnz = rowptr[n];
  free(uniq);
  free(buf);
  free(start);
  return nnz;
}

/* Uniform CSR: `samples` draws of (row, col); returns nnz. crd/vals must hold
 * `samples` entries. */
int64_t syn_uniform_csr(int64_t n, int64_t m, int64_t samples, uint64_t seed, int kind,
                        int64_t* rowptr, int64_t* crd, double* vals) {
  int64_t* rows = malloc(sizeof(int64_t) * (size_t)(samples > 0 ? samples : 1));
  int64_t* cols = malloc(sizeof(int64_t) * (size_t)(samples > 0 ? samples : 1));
  double* v = malloc(sizeof(double) * (size_t)(samples > 0 ? samples : 1));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < samples; e++) {
    rows[e] = (int64_t)(hash3(seed, 1, (uint64_t)e) % (uint64_t)n);
    cols[e] = (int64_t)(hash3(seed, 2, (uint64_t)e) % (uint64_t)m);
    v[e] = value_of(seed, 3, (uint64_t)e, kind);
  }
  int64_t nnz = coo_to_csr(n, samples, rows, cols, v, rowptr, crd, vals);
  free(rows);
  free(cols);
  free(v);
  return nnz;
}

/* Graph500-style R-MAT (no noise, no label scrambling unless `scramble`):
 * each of `edges` edges descends `scale` levels, choosing quadrant
 * (0,0)/(0,1)/(1,0)/(1,1) with probabilities a/b/c/1-a-b-c; 21 bits of a
 * 64-bit hash per level.  Optional column shift (mod n) builds the SpAdd3
 * operands C, D = B shifted by +1, +2.  crd/vals must
 * hold `edges` entries. */
int64_t syn_rmat_csr(int scale, int64_t edges, double a, double b, double c, uint64_t seed,
                     int kind, int scramble, int64_t col_shift, int64_t* rowptr, int64_t* crd,
                     double* vals) {
  const int64_t n = (int64_t)1 << scale;
  int64_t* rows = malloc(sizeof(int64_t) * (size_t)(edges > 0 ? edges : 1));
  int64_t* cols = malloc(sizeof(int64_t) * (size_t)(edges > 0 ? edges : 1));
  double* v = malloc(sizeof(double) * (size_t)(edges > 0 ? edges : 1));
  const double ab = a + b, abc = a + b + c;
  const uint64_t mul = 0x9E3779B97F4A7C15ull; /* odd: a bijection of [0, 2^scale) */
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < edges; e++) {
    int64_t r = 0, cc = 0;
    uint64_t h = 0;
    for (int l = 0; l < scale; l++) {
      int slot = l % 3;
      if (slot == 0) h = hash3(seed, 11, (uint64_t)e * 16 + (uint64_t)(l / 3));
      double u = (double)((h >> (slot * 21)) & 0x1FFFFF) * (1.0 / 2097152.0);
      int rb = 0, cb = 0;
      if (u < a) {
      } else if (u < ab) {
        cb = 1;
      } else if (u < abc) {
        rb = 1;
      } else {
        rb = 1, cb = 1;
      }
      r = (r << 1) | rb;
      cc = (cc << 1) | cb;
    }
    if (scramble) {
      r = (int64_t)(((uint64_t)r * mul) & (uint64_t)(n - 1));
      cc = (int64_t)(((uint64_t)cc * mul) & (uint64_t)(n - 1));
    }
    rows[e] = r;
    cols[e] = (cc + col_shift) % n;
    v[e] = value_of(seed, 12 + (uint64_t)col_shift, (uint64_t)e, kind);
  }
  int64_t nnz = coo_to_csr(n, edges, rows, cols, v, rowptr, crd, vals);
  free(rows);
  free(cols);
  free(v);
  return nnz;
}

/* Power-law 3-tensor in `dss` (CSF) form: `samples` draws with per-mode
 * coordinate floor(N * u^3).  Outputs rp1 (I+1), crd1 (F <= samples),
 * rp2 (F+1), crd2 / vals (nnz <= samples); returns nnz, *F_out = fibres. */
int64_t syn_powerlaw_csf(int64_t I, int64_t J, int64_t K, int64_t samples, uint64_t seed,
                         int kind, int64_t* rp1, int64_t* crd1, int64_t* rp2, int64_t* crd2,
                         double* vals, int64_t* F_out) {
  int64_t* rows = malloc(sizeof(int64_t) * (size_t)(samples > 0 ? samples : 1));
  int64_t* keys = malloc(sizeof(int64_t) * (size_t)(samples > 0 ? samples : 1));
  double* v = malloc(sizeof(double) * (size_t)(samples > 0 ? samples : 1));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < samples; e++) {
    double u0 = unit53(hash3(seed, 21, (uint64_t)e));
    double u1 = unit53(hash3(seed, 22, (uint64_t)e));
    double u2 = unit53(hash3(seed, 23, (uint64_t)e));
    int64_t i = (int64_t)((double)I * u0 * u0 * u0);
    int64_t j = (int64_t)((double)J * u1 * u1 * u1);
    int64_t k = (int64_t)((double)K * u2 * u2 * u2);
    if (i >= I) i = I - 1;
    if (j >= J) j = J - 1;
    if (k >= K) k = K - 1;
    rows[e] = i;
    keys[e] = j * K + k;
    v[e] = value_of(seed, 24, (uint64_t)e, kind);
  }
  /* rows x (j,k) keys: a CSR over i whose "columns" are the fused (j,k) */
  int64_t* rp = malloc(sizeof(int64_t) * (size_t)(I + 1));
  int64_t* jk = malloc(sizeof(int64_t) * (size_t)(samples > 0 ? samples : 1));
  int64_t nnz = coo_to_csr(I, samples, rows, keys, v, rp, jk, vals);
  /* split fused keys into fibres */
  int64_t F = 0;
  rp1[0] = 0;
  for (int64_t i = 0; i < I; i++) {
    int64_t prev_j = -1;
    for (int64_t p = rp[i]; p < rp[i + 1]; p++) {
      int64_t j = jk[p] / K, k = jk[p] % K;
      if (j != prev_j) {
        crd1[F] = j;
        rp2[F] = p;
        F++;
        prev_j = j;
      }
      crd2[p] = k;
    }
    rp1[i + 1] = F;
  }
  rp2[F] = nnz;
  *F_out = F;
  free(rp);
  free(jk);
  free(rows);
  free(keys);
  free(v);
  return nnz;
}

/* Thread count of the generators (launchers such as torchrun export
 * OMP_NUM_THREADS=1 to every rank; the rank that generates inputs raises it). */
void syn_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}

int syn_max_threads(void) { return omp_get_max_threads(); }
