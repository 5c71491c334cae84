// Context, NCCL communicator, and device-resident tensor storage (K0).
//
// Storage follows the reference's coordinate-tree encoding
// (SparseTensor, /root/reference/proj/core/include/dspar/tensor.hpp:54-114):
// levels grouped like level_grouping (tensor.cpp:30-41), a compressed level
// kept as an int64 row pointer (lossless versus the reference's inclusive
// (lo,hi) pos pairs, tensor.cpp:258-281), crd int64 and vals fp64, all in HBM.
#include <algorithm>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace spd {

// A whole (non-distributed) tensor: every top-level row, pos base 0.
void set_whole_span(spd_tensor* t) {
  t->row_lo = 0;
  t->row_hi = (t->levels.size() >= 2 ? t->levels[1].parent_positions : 1) - 1;
  t->pos_base = 0;
  t->global_positions = t->nvals;
}

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

spd_context* checked(spd_context* ctx) {
  if (!ctx) throw ValidationError("null spd_context");
  return ctx;
}

void activate(spd_context* ctx) { SPD_CUDA(cudaSetDevice(ctx->device)); }

// ---------------------------------------------------------------------------
// K0: pos pairs -> row pointer, with SparseTensor::validate's compressed-level
// checks (tensor.cpp:258-281) evaluated element-parallel:
//   every range is canonical-empty or non-empty, and starts where the previous
//   one ended: lo_p == hi_{p-1} + 1 (lo_0 == 0); the last ends at nnz - 1.
// Error bits: 1 tiling / canonical form, 2 crd order, 4 crd bounds.
__global__ void k_pairs_to_rowptr(const int64_t* __restrict__ pairs, int64_t npos, int64_t nnz,
                                  int64_t* __restrict__ rowptr, int* __restrict__ err) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; p < npos; p += stride) {
    int64_t lo = pairs[2 * p], hi = pairs[2 * p + 1];
    int64_t prev_end = p == 0 ? -1 : pairs[2 * p - 1];
    bool ok = hi >= lo - 1 && lo == prev_end + 1;
    if (p == npos - 1) ok = ok && hi + 1 == nnz;
    if (!ok) atomicOr(err, 1);
    rowptr[p] = lo;
    if (p == npos - 1) rowptr[npos] = nnz;
  }
}

__global__ void k_check_rowptr(const int64_t* __restrict__ rowptr, int64_t npos, int64_t nnz,
                               int* __restrict__ err) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; p < npos; p += stride) {
    bool ok = rowptr[p + 1] >= rowptr[p];
    if (p == 0) ok = ok && rowptr[0] == 0;
    if (p == npos - 1) ok = ok && rowptr[npos] == nnz;
    if (!ok) atomicOr(err, 1);
  }
}

// crd strictly increasing inside every range and within [0, dim): a position
// q > 0 is compared with q-1 unless q starts a range.  Range starts are found
// with a per-position owner test that needs no extra buffer: q starts a range
// iff rowptr[owner(q)] == q, evaluated here by marking starts first.
__global__ void k_mark_starts(const int64_t* __restrict__ rowptr, int64_t npos,
                              unsigned char* __restrict__ start, int64_t lo, int64_t hi) {
  // start is indexed by global position; only [lo, hi] is held
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; p < npos; p += stride) {
    const int64_t a = rowptr[p];
    if (rowptr[p + 1] > a && a >= lo && a <= hi) start[a] = 1;
  }
}

// Positions [lo, hi] of crd (indexed by global position); the position
// before lo, when it exists and is held elsewhere, is passed as prev.
__global__ void k_check_crd(const int64_t* __restrict__ crd, int64_t lo, int64_t hi, int64_t dim,
                            const unsigned char* __restrict__ start, int has_prev, int64_t prev,
                            int* __restrict__ err) {
  int64_t q = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; q <= hi; q += stride) {
    int64_t c = crd[q];
    if (c < 0 || c >= dim) atomicOr(err, 4);
    if (!start[q]) {
      if (q > lo && c <= crd[q - 1]) atomicOr(err, 2);
      if (q == lo && has_prev && c <= prev) atomicOr(err, 2);
    }
  }
}

__global__ void k_rowptr_to_pairs(const int64_t* __restrict__ rowptr, int64_t npos,
                                  int64_t* __restrict__ pairs) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; p < npos; p += stride) {
    pairs[2 * p] = rowptr[p];
    pairs[2 * p + 1] = rowptr[p + 1] - 1;
  }
}

// Commit of a restage: copies the staged array over the live one only when
// no validation flag was raised.
__global__ void k_commit(const int* __restrict__ err, const int64_t* __restrict__ src, int64_t* __restrict__ dst,
                         int64_t n) {
  if (*err) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

static const char* restage_message(int err) {
  if (err & 1) return "tensor: pos ranges must tile [0, nnz) with canonical empties";
  if (err & 2) return "tensor: crd must be strictly increasing per range";
  return "tensor: crd value out of dimension bounds";
}

void settle_restage(const spd_tensor* tc, bool block) {
  spd_tensor* t = const_cast<spd_tensor*>(tc);
  if (!t) return;
  if (t->restage_pending) {
    if (block) {
      SPD_CUDA(cudaEventSynchronize(t->restage_done));
    } else {
      const cudaError_t q = cudaEventQuery(t->restage_done);
      if (q == cudaErrorNotReady) return;
      SPD_CUDA(q);
    }
    t->restage_pending = false;
    auto& pend = t->ctx->pending_restage;
    pend.erase(std::remove(pend.begin(), pend.end(), t), pend.end());
    const int err = *t->restage_err_host;
    if (err) {
      if (t->restage_moved) t->poisoned = true;  // its range moved with the rejected pattern
      throw ValidationError(std::string(restage_message(err)) +
                            (t->poisoned ? " (spd_tensor_restage rejected it; the row-split piece is unusable, "
                                           "destroy it)"
                                         : " (spd_tensor_restage rejected it; the tensor keeps its previous "
                                           "contents)"));
    }
  }
  if (t->poisoned) throw ValidationError("tensor: a rejected restage left this piece unusable");
}

static int grid_for(spd_context* ctx, int64_t n, int block = 256) {
  int64_t g = ceil_div(n, block);
  int64_t cap = (int64_t)ctx->num_sms * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

void* dev_alloc(spd_context* ctx, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 8;
  SPD_CUDA(cudaMallocAsync(&p, bytes, ctx->stream));
  return p;
}

void dev_free(spd_context* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

// Builds the level skeleton from the FormatSpec (tensor.cpp:30-41, 81-92).
spd_tensor* make_skeleton(spd_context* ctx, int order, const int64_t* dims,
                                 const int* kinds, const int* mode_order) {
  if (order < 0) throw ValidationError("tensor order must be non-negative");
  std::vector<bool> seen(order, false);
  for (int k = 0; k < order; k++) {
    int m = mode_order[k];
    if (m < 0 || m >= order || seen[m]) throw ValidationError("format: mode order is not a permutation");
    seen[m] = true;
    if (kinds[k] != SPD_DENSE && kinds[k] != SPD_COMPRESSED)
      throw ValidationError("format: unknown level kind");
    if (dims[k] < 0) throw ValidationError("tensor: negative dimension");
  }
  auto* t = new spd_tensor();
  t->ctx = ctx;
  t->order = order;
  t->dims.assign(dims, dims + order);
  t->kinds.assign(kinds, kinds + order);
  t->mode_order.assign(mode_order, mode_order + order);
  for (int k = 0; k < order; k++) {
    if (kinds[k] == SPD_DENSE && !t->groups.empty() && kinds[t->groups.back().back()] == SPD_DENSE)
      t->groups.back().push_back(k);
    else
      t->groups.push_back({k});
  }
  t->levels.resize(t->groups.size());
  return t;
}

struct LevelInput {
  const int64_t* pos_pairs;  // or rowptr
  const int64_t* crd;
};

// Uploads/validates all levels. `pairs`: pos given as (lo,hi) pairs.
static spd_tensor* upload_impl(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                               const int* mode_order, const int64_t* const* pos,
                               const int64_t* const* crd, const double* vals, bool pairs,
                               bool validate, bool skip_leaf = false) {
  HostTrace ht("upload");
  activate(ctx);
  spd_tensor* t = make_skeleton(ctx, order, dims, kinds, mode_order);
  int* err_d = nullptr;
  int err_h = 0;
  try {
    SPD_CUDA(cudaMallocAsync((void**)&err_d, sizeof(int), ctx->stream));
    SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), ctx->stream));
    int64_t parent = 1;
    for (size_t l = 0; l < t->groups.size(); l++) {
      spd_level_store& L = t->levels[l];
      L.parent_positions = parent;
      int k0 = t->groups[l][0];
      if (kinds[k0] == SPD_DENSE) {
        L.kind = SPD_DENSE;
        int64_t total = 1;
        for (int k : t->groups[l]) {
          L.dom.push_back(dims[mode_order[k]]);
          total *= dims[mode_order[k]];
        }
        parent *= total;
        L.positions = parent;
        continue;
      }
      L.kind = SPD_COMPRESSED;
      if (!pos || (!pos[l] && parent > 0))
        throw ValidationError("compressed level " + std::to_string(l) + " needs pos");
      int64_t nnz;
      if (parent == 0)
        nnz = 0;
      else if (pairs)
        nnz = pos[l][2 * (parent - 1) + 1] + 1;
      else
        nnz = pos[l][parent];
      if (nnz < 0) throw ValidationError("tensor: pos ranges must cover exactly [0, nnz)");
      if (nnz > 0 && (!crd || !crd[l]))
        throw ValidationError("compressed level " + std::to_string(l) + " needs crd");
      L.positions = nnz;
      // skip_leaf: the leaf's crd / vals are staged later as a piece
      const bool leaf_piece = skip_leaf && l + 1 == t->groups.size();
      L.rowptr = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (parent + 1));
      L.crd = leaf_piece ? nullptr : (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (nnz > 0 ? nnz : 1));
      if (pairs) {
        int64_t* tmp = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * 2 * (parent > 0 ? parent : 1));
        if (parent > 0) {
          SPD_CUDA(cudaMemcpyAsync(tmp, pos[l], sizeof(int64_t) * 2 * parent,
                                   cudaMemcpyHostToDevice, ctx->stream));
          k_pairs_to_rowptr<<<grid_for(ctx, parent), 256, 0, ctx->stream>>>(tmp, parent, nnz,
                                                                            L.rowptr, err_d);
          SPD_CHECK_LAUNCH();
        } else {
          SPD_CUDA(cudaMemsetAsync(L.rowptr, 0, sizeof(int64_t), ctx->stream));
        }
        dev_free(ctx, tmp);
      } else if (parent == 0) {
        SPD_CUDA(cudaMemsetAsync(L.rowptr, 0, sizeof(int64_t), ctx->stream));
      } else {
        SPD_CUDA(cudaMemcpyAsync(L.rowptr, pos[l], sizeof(int64_t) * (parent + 1),
                                 cudaMemcpyHostToDevice, ctx->stream));
        if (validate && parent > 0) {
          k_check_rowptr<<<grid_for(ctx, parent), 256, 0, ctx->stream>>>(L.rowptr, parent, nnz,
                                                                         err_d);
          SPD_CHECK_LAUNCH();
        }
      }
      if (nnz > 0 && !leaf_piece)
        SPD_CUDA(cudaMemcpyAsync(L.crd, crd[l], sizeof(int64_t) * nnz, cudaMemcpyHostToDevice,
                                 ctx->stream));
      if ((validate || pairs) && nnz > 0 && !leaf_piece) {
        unsigned char* start = (unsigned char*)dev_alloc(ctx, nnz);
        SPD_CUDA(cudaMemsetAsync(start, 0, nnz, ctx->stream));
        k_mark_starts<<<grid_for(ctx, parent), 256, 0, ctx->stream>>>(L.rowptr, parent, start, 0, nnz - 1);
        SPD_CHECK_LAUNCH();
        int64_t dim = dims[mode_order[k0]];
        k_check_crd<<<grid_for(ctx, nnz), 256, 0, ctx->stream>>>(L.crd, 0, nnz - 1, dim, start, 0, 0, err_d);
        SPD_CHECK_LAUNCH();
        dev_free(ctx, start);
      }
      parent = nnz;
    }
    t->nvals = parent;
    set_whole_span(t);
    t->vals = skip_leaf ? nullptr : (double*)dev_alloc(ctx, sizeof(double) * (parent > 0 ? parent : 1));
    if (parent > 0 && !skip_leaf) {
      if (!vals) throw ValidationError("tensor: vals length does not match leaf count");
      SPD_CUDA(cudaMemcpyAsync(t->vals, vals, sizeof(double) * parent, cudaMemcpyHostToDevice,
                               ctx->stream));
    }
    ht.mark("queued");
    SPD_CUDA(cudaMemcpyAsync(&err_h, err_d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
    ht.mark("synced");
    dev_free(ctx, err_d);
    err_d = nullptr;
    if (err_h & 1) throw ValidationError("tensor: pos ranges must tile [0, nnz) with canonical empties");
    if (err_h & 2) throw ValidationError("tensor: crd must be strictly increasing per range");
    if (err_h & 4) throw ValidationError("tensor: crd value out of dimension bounds");
  } catch (...) {
    if (err_d) dev_free(ctx, err_d);
    for (auto& L : t->levels) {
      dev_free(ctx, L.rowptr);
      dev_free(ctx, L.crd);
    }
    dev_free(ctx, t->vals);
    delete t;
    throw;
  }
  return t;
}

const std::vector<spd_color>& host_colors(spd_context* ctx) {
  if (!ctx->colors_host_valid) {
    ctx->colors_host.resize(ctx->pieces);
    std::vector<DevColor> tmp(ctx->pieces);
    if (ctx->pieces > 0) {
      SPD_CUDA(cudaMemcpyAsync(tmp.data(), ctx->colors_dev.ptr, sizeof(DevColor) * ctx->pieces,
                               cudaMemcpyDeviceToHost, ctx->stream));
      SPD_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    for (int64_t c = 0; c < ctx->pieces; c++) ctx->colors_host[c] = tmp[c].pub;
    ctx->colors_host_valid = true;
  }
  return ctx->colors_host;
}

void colour_block(const spd_context* ctx, int64_t P, int r, int64_t& first, int64_t& count) {
  if (ctx->blocks_pieces == P && (int)ctx->blocks.size() == ctx->world + 1) {
    first = ctx->blocks[r];
    count = ctx->blocks[r + 1] - first;
    return;
  }
  const int64_t cmax = ceil_div(std::max<int64_t>(P, 1), ctx->world);
  first = std::min<int64_t>(P, r * cmax);
  count = std::max<int64_t>(0, std::min<int64_t>(cmax, P - first));
}

void colour_block(const spd_context* ctx, int r, int64_t& first, int64_t& count) {
  colour_block(ctx, ctx->pieces, r, first, count);
}

int64_t placement_pieces(const spd_context* ctx) {
  return (int)ctx->blocks.size() == ctx->world + 1 && ctx->blocks_pieces > 0 ? ctx->blocks_pieces : ctx->world;
}

std::vector<spd_range> rank_spans(spd_context* ctx, spd_tensor* t, int split, int64_t P) {
  const int rc = split == 1 ? spd_partition_universe(ctx, t, P, nullptr) : spd_partition_nonzero(ctx, t, 1, P, nullptr);
  if (rc != SPD_OK) throw ValidationError(spd_last_error());
  const auto& hc = host_colors(ctx);
  std::vector<spd_range> out(ctx->world, spd_range{0, -1});
  for (int r = 0; r < ctx->world; r++) {
    int64_t f, c;
    colour_block(ctx, P, r, f, c);
    int64_t lo = INT64_MAX, hi = -1;
    for (int64_t k = f; k < f + c; k++)
      if (hc[k].q.lo <= hc[k].q.hi) lo = std::min(lo, hc[k].q.lo), hi = std::max(hi, hc[k].q.hi);
    if (lo <= hi) out[r] = spd_range{lo, hi};
  }
  return out;
}

bool even_blocks(const spd_context* ctx) {
  const int64_t cmax = ceil_div(std::max<int64_t>(ctx->pieces, 1), ctx->world);
  for (int r = 0; r < ctx->world; r++) {
    int64_t f, c;
    colour_block(ctx, r, f, c);
    if (f != std::min<int64_t>(ctx->pieces, r * cmax)) return false;
  }
  return true;
}

void require_partition(spd_context* ctx, const spd_tensor* t, int64_t first, int64_t count, bool allow_grid) {
  if (ctx->split == SplitKind::None || ctx->split_tensor != t)
    throw ValidationError("no partition of this tensor on the context: call spd_partition_* first");
  if (first < 0 || count < 1 || first + count > ctx->pieces)
    throw ValidationError("colour range outside the partition");
  bool all = first == 0 && count == ctx->pieces;
  // With a communicator a GPU runs one contiguous block of colours: rank r
  // runs [r * cmax, min(P, (r + 1) * cmax)), cmax = ceil(P / world) -- one
  // colour per GPU when P == world, several when the plan has more colours
  // than GPUs (the integration adapter on a smaller box) -- or the blocks set
  // by spd_context_set_colour_blocks (cost-balanced over-decomposition).
  bool one_per_rank = false;
  if (ctx->comm && ctx->pieces >= ctx->world) {
    int64_t f, c;
    colour_block(ctx, ctx->rank, f, c);
    one_per_rank = first == f && count >= 1 && count == c;
  }
  // 2-D machine grid (x major, y minor; MachineGrid::worker_id, machine.cpp:88-92)
  // with the row loop on x: rank r runs row colour r / (world / pieces) of a
  // universe split -- rows never straddle colours, so no cross-GPU combine.
  bool grid_row = allow_grid && ctx->comm && count == 1 && ctx->split == SplitKind::Universe &&
                  ctx->pieces > 0 && ctx->world % ctx->pieces == 0 &&
                  first == ctx->rank / (ctx->world / ctx->pieces);
  if (!all && !one_per_rank && !grid_row)
    throw ValidationError(
        "a GPU runs either every colour of the partition, or (with a communicator) its block of colours "
        "(spd_context_colour_blocks: [rank * ceil(pieces / world), ...) unless set) (row loops of a 2-D grid: "
        "colour rank / (world / pieces))");
}

void fill_stats(spd_context* ctx, spd_stats* st, int64_t combines, const std::vector<int64_t>& work,
                int64_t launches, bool timed) {
  ctx->last_work = work;
  if (!st) return;
  st->workers = (int64_t)work.size();
  st->combines = combines;
  int64_t total = 0, mx = 0;
  for (int64_t w : work) total += w, mx = w > mx ? w : mx;
  st->imbalance = total == 0 ? 1.0 : (double)mx * (double)work.size() / (double)total;
  st->launches = launches;
  st->kernel_ms = 0;
  if (timed) {
    float ms = 0;
    SPD_CUDA(cudaEventSynchronize(ctx->ev1));
    SPD_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    st->kernel_ms = ms;
  }
}

static cudaEvent_t timing_event(spd_context* ctx) {
  if (ctx->timing_used == ctx->timing_events.size()) {
    cudaEvent_t e;
    SPD_CUDA(cudaEventCreate(&e));
    ctx->timing_events.push_back(e);
  }
  return ctx->timing_events[ctx->timing_used++];
}

void leaf_timing_begin(spd_context* ctx) {
  if (ctx->timing == 1) SPD_CUDA(cudaEventRecord(timing_event(ctx), ctx->stream));
}

void leaf_timing_end(spd_context* ctx) {
  if (ctx->timing == 1) SPD_CUDA(cudaEventRecord(timing_event(ctx), ctx->stream));
}

void trace_mark(spd_context* ctx) {
  if (ctx->timing == 2) SPD_CUDA(cudaEventRecord(timing_event(ctx), ctx->stream));
}

}  // namespace spd

using namespace spd;

extern "C" {

int spd_context_timing(spd_context* ctx, int enable) {
  return guarded([&] {
    checked(ctx);
    if (enable < 0 || enable > 2) throw ValidationError("timing mode must be 0, 1 or 2");
    ctx->timing = enable;
  });
}

int spd_context_read_timing(spd_context* ctx, double* leaf_ms, int64_t cap, int64_t* n) {
  return guarded([&] {
    checked(ctx);
    activate(ctx);
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
    // mode 1: (begin, end) pairs around leaf kernels; mode 2: consecutive
    // phase markers, returned as the deltas between them.
    const bool pairs_mode = ctx->timing != 2;
    const int64_t used = (int64_t)ctx->timing_used;
    const int64_t cnt = pairs_mode ? used / 2 : std::max<int64_t>(used - 1, 0);
    for (int64_t i = 0; i < cnt && i < cap; i++) {
      float ms = 0;
      const int64_t a = pairs_mode ? 2 * i : i;
      SPD_CUDA(cudaEventElapsedTime(&ms, ctx->timing_events[a], ctx->timing_events[a + 1]));
      leaf_ms[i] = ms;
    }
    *n = cnt;
    ctx->timing_used = 0;
  });
}

int spd_context_launches(const spd_context* ctx, int64_t* count) {
  return guarded([&] {
    if (!ctx) throw ValidationError("null spd_context");
    *count = ctx->launches;
  });
}

const char* spd_last_error(void) { return g_last_error.c_str(); }
int spd_abi_version(void) { return 100; }

int spd_device_count(int* count) {
  return guarded([&] {
    if (!count) throw ValidationError("null out pointer");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

int spd_context_create(int device, void* stream, spd_context** out) {
  return guarded([&] {
    if (!out) throw ValidationError("null out pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      throw RuntimeError("no CUDA device available: the B200 backend has no CPU fallback");
    if (device < 0 || device >= n) throw ValidationError("device ordinal out of range");
    auto* ctx = new spd_context();
    ctx->device = device;
    SPD_CUDA(cudaSetDevice(device));
    SPD_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (stream) {
      ctx->stream = (cudaStream_t)stream;
    } else {
      SPD_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    // Keep freed blocks in the stream-ordered pool: per-step uploads reuse them.
    cudaMemPool_t pool;
    SPD_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    SPD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    SPD_CUDA(cudaEventCreate(&ctx->ev0));
    SPD_CUDA(cudaEventCreate(&ctx->ev1));
    SPD_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    SPD_CUDA(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming));
    SPD_CUDA(cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming));
    SPD_CUDA(cudaMallocHost((void**)&ctx->pinned_counters, sizeof(int64_t) * 64));
    *out = ctx;
  });
}

int spd_context_destroy(spd_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    ctx->colors_dev.release();
    ctx->blocks_dev.release();
    for (auto& b : ctx->scratch) b.release();
    ctx->counters.release();
    for (auto* b : {&ctx->bucket.keys, &ctx->bucket.tmp, &ctx->bucket.pos_buf, &ctx->bucket.pref_buf,
                    &ctx->bucket.off_buf})
      b->release();
    if (ctx->pinned_counters) cudaFreeHost(ctx->pinned_counters);
    for (cudaEvent_t e : ctx->timing_events) cudaEventDestroy(e);
    if (ctx->aux) cudaStreamSynchronize(ctx->aux), cudaStreamDestroy(ctx->aux);
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    if (ctx->join) cudaEventDestroy(ctx->join);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int spd_context_synchronize(spd_context* ctx) {
  return guarded([&] {
    checked(ctx);
    activate(ctx);
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
    // report the verdicts of restages issued on this context (the first
    // rejection raises; every pending verdict is consumed)
    std::string first;
    while (!ctx->pending_restage.empty()) {
      try {
        settle_restage(ctx->pending_restage.front(), true);
      } catch (const ValidationError& e) {
        if (first.empty()) first = e.what();
      }
    }
    if (!first.empty()) throw ValidationError(first);
  });
}

int spd_nccl_unique_id(void* out128) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    SPD_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
  });
}

int spd_context_init_comm(spd_context* ctx, const void* unique_id128, int rank, int world) {
  return guarded([&] {
    checked(ctx);
    if (world < 1 || rank < 0 || rank >= world) throw ValidationError("bad rank/world");
    activate(ctx);
    ncclUniqueId id;
    std::memcpy(&id, unique_id128, sizeof(id));
    if (ctx->comm) SPD_NCCL(ncclCommDestroy(ctx->comm));
    SPD_NCCL(ncclCommInitRank(&ctx->comm, world, id, rank));
    ctx->rank = rank;
    ctx->world = world;
  });
}

int spd_allgather(spd_context* ctx, void* dev_buf, int64_t bytes_per_rank) {
  return guarded([&] {
    checked(ctx);
    if (!ctx->comm) throw ValidationError("spd_allgather needs a communicator (spd_context_init_comm)");
    if (bytes_per_rank < 0) throw ValidationError("negative size");
    activate(ctx);
    char* b = static_cast<char*>(dev_buf);
    SPD_NCCL(ncclAllGather(b + (size_t)ctx->rank * bytes_per_rank, b, (size_t)bytes_per_rank, ncclUint8,
                           ctx->comm, ctx->stream));
  });
}

int spd_context_abort(spd_context* ctx) {
  return guarded([&] {
    checked(ctx);
    // ncclCommAbort ends this rank's pending collectives (their kernels stop
    // waiting for peers), so a thread blocked on them returns with an error
    if (ctx->comm) {
      ncclComm_t c = ctx->comm;
      ctx->comm = nullptr;
      ncclCommAbort(c);
    }
  });
}

int spd_context_rank(const spd_context* ctx, int* rank, int* world) {
  return guarded([&] {
    if (!ctx) throw ValidationError("null spd_context");
    *rank = ctx->rank;
    *world = ctx->world;
  });
}

int spd_tensor_upload(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                      const int* mode_order, const int64_t* const* pos_pairs,
                      const int64_t* const* crd, const double* vals, spd_tensor** out) {
  return guarded([&] {
    checked(ctx);
    *out = upload_impl(ctx, order, dims, kinds, mode_order, pos_pairs, crd, vals, true, true);
  });
}

namespace spd {

// This GPU's colour of a piece, read off the host pos pairs (no device
// round trip): divide_bounds (planner.cpp:10-20) over the positions for a
// nonzero split, or over the rows for a row split -- then the positions of
// that row block.  The pairs are not validated yet; only the two entries read
// here are range-checked (the device checks the rest).
static spd_range host_piece_range(const int64_t* pairs, int64_t nrows, int64_t nnz, int split,
                                  const spd_context* ctx) {
  // this GPU's block [f, f + c) of the placement's P-colour split
  // (partition_nonzero / partition_universe: colour k of P covers
  // [k * (n / P), ...), the last colour the remainder)
  const int64_t P = placement_pieces(ctx);
  int64_t f, c;
  colour_block(ctx, P, ctx->rank, f, c);
  auto divide = [&](int64_t n) {
    const int64_t block = n / P;
    spd_range r{f * block, f + c < P ? (f + c) * block - 1 : n - 1};
    if (c < 1 || r.lo > r.hi) r = spd_range{0, -1};
    return r;
  };
  if (split == 2) return divide(nnz);
  const spd_range rows = divide(nrows);
  if (rows.lo > rows.hi) return spd_range{0, -1};
  spd_range q{pairs[2 * rows.lo], pairs[2 * rows.hi + 1]};
  if (q.lo < 0 || q.hi >= nnz || q.lo > q.hi + 1)
    throw ValidationError("tensor: pos ranges must tile [0, nnz) with canonical empties");
  if (q.lo > q.hi) q = spd_range{0, -1};
  return q;
}

// Per-GPU piece of a CSR matrix staged from host arrays (spd_tensor_upload_
// piece / spd_tensor_restage of a piece): the whole pos level (O(rows), the
// partition step needs it) converted and checked on the GPU, and only this
// GPU's colour of crd / vals (split 1 = rows, 2 = nonzeros over the
// communicator's GPUs) copied from the host arrays (indexed by global
// position) and checked.  `fresh`: an upload -- allocate, write in place and
// synchronise (the handle is returned validated).  Else a restage: stage,
// validate and commit on the device like spd_tensor_restage, no host
// synchronisation.
static void stage_piece(spd_context* ctx, spd_tensor* t, const int64_t* pairs, const int64_t* crd,
                        const double* vals, int split, bool fresh) {
  cudaStream_t s = ctx->stream;
  spd_level_store& L = t->levels[1];
  const int64_t nrows = L.parent_positions, nnz = L.positions;
  if (nrows > 0 && !pairs) throw ValidationError("compressed level 1 needs pos");
  const spd_range mine = host_piece_range(pairs, nrows, nnz, split, ctx);
  const int64_t cnt = std::max<int64_t>(mine.hi - mine.lo + 1, 0);
  if (cnt > 0 && !crd) throw ValidationError("compressed level 1 needs crd");
  if (cnt > 0 && !vals) throw ValidationError("tensor: vals length does not match leaf count");
  int* err_d = nullptr;
  int64_t *rp = L.rowptr, *cd = nullptr;
  double* vd = nullptr;
  if (fresh) {
    err_d = (int*)ctx->counters.reserve(sizeof(int64_t) * 16) + 2;
    t->piece_cap = std::max<int64_t>(cnt, 1);
    t->piece_crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * t->piece_cap);
    t->piece_vals = (double*)dev_alloc(ctx, sizeof(double) * t->piece_cap);
    cd = t->piece_crd;
    vd = t->piece_vals;
  } else {
    if (!t->restage_err) {
      t->restage_err = (int*)dev_alloc(ctx, sizeof(int));
      SPD_CUDA(cudaMallocHost((void**)&t->restage_err_host, sizeof(int)));
      SPD_CUDA(cudaEventCreateWithFlags(&t->restage_done, cudaEventDisableTiming));
    }
    err_d = t->restage_err;
    if (t->stage_rowptr.size() != 2) {
      t->stage_rowptr.assign(2, nullptr);
      t->stage_crd.assign(2, nullptr);
      t->stage_rowptr[1] = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (nrows + 1));
    }
    if (t->stage_leaf_cap < cnt) {
      dev_free(ctx, t->stage_crd[1]);
      dev_free(ctx, t->stage_vals);
      t->stage_leaf_cap = std::max<int64_t>(cnt, 1);
      t->stage_crd[1] = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * t->stage_leaf_cap);
      t->stage_vals = (double*)dev_alloc(ctx, sizeof(double) * t->stage_leaf_cap);
    }
    rp = t->stage_rowptr[1];
    cd = t->stage_crd[1];
    vd = t->stage_vals;
  }
  SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), s));
  if (nrows > 0) {
    if (t->stage_pairs_cap < 2 * nrows) {
      dev_free(ctx, t->stage_pairs);
      t->stage_pairs = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * 2 * nrows);
      t->stage_pairs_cap = 2 * nrows;
    }
    SPD_CUDA(cudaMemcpyAsync(t->stage_pairs, pairs, sizeof(int64_t) * 2 * nrows, cudaMemcpyHostToDevice, s));
    k_pairs_to_rowptr<<<grid_for(ctx, nrows), 256, 0, s>>>(t->stage_pairs, nrows, nnz, rp, err_d);
    SPD_CHECK_LAUNCH();
  } else {
    SPD_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), s));
  }
  if (cnt > 0) {
    SPD_CUDA(cudaMemcpyAsync(cd, crd + mine.lo, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, s));
    SPD_CUDA(cudaMemcpyAsync(vd, vals + mine.lo, sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
    const int64_t need = std::max<int64_t>(cnt, nrows);  // also the nz_view flags buffer
    if (t->stage_flags_cap < need) {
      dev_free(ctx, t->stage_flags);
      t->stage_flags = (unsigned char*)dev_alloc(ctx, need);
      t->stage_flags_cap = need;
    }
    unsigned char* start = t->stage_flags - mine.lo;  // indexed by global position
    SPD_CUDA(cudaMemsetAsync(t->stage_flags, 0, cnt, s));
    k_mark_starts<<<grid_for(ctx, nrows), 256, 0, s>>>(rp, nrows, start, mine.lo, mine.hi);
    SPD_CHECK_LAUNCH();
    const int64_t dim = t->dims[t->mode_order[1]];
    k_check_crd<<<grid_for(ctx, cnt), 256, 0, s>>>(cd - mine.lo, mine.lo, mine.hi, dim, start, mine.lo > 0 ? 1 : 0,
                                                   mine.lo > 0 ? crd[mine.lo - 1] : 0, err_d);
    SPD_CHECK_LAUNCH();
  }
  const bool moved = !fresh && (mine.lo != t->piece_lo || mine.hi != t->piece_hi);
  t->piece_split = split;
  if (fresh) {
    t->piece_lo = mine.lo;
    t->piece_hi = mine.hi;
    L.crd = t->piece_crd - mine.lo;  // indexed by global position
    t->vals = t->piece_vals - mine.lo;
    int err_h = 0;
    SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 12, err_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&err_h, ctx->pinned_counters + 12, sizeof(int));
    if (err_h) throw ValidationError(restage_message(err_h));
    return;
  }
  // restage: a row split's range follows the new pattern; grow the live piece
  // arrays when it does not fit (a rejection then poisons the piece)
  if (cnt > t->piece_cap) {
    dev_free(ctx, t->piece_crd);
    dev_free(ctx, t->piece_vals);
    t->piece_cap = cnt;
    t->piece_crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * t->piece_cap);
    t->piece_vals = (double*)dev_alloc(ctx, sizeof(double) * t->piece_cap);
    if (t->crd32_alloc) dev_free(ctx, t->crd32_alloc), t->crd32_alloc = nullptr, t->crd32_cap = 0;
  }
  t->piece_lo = mine.lo;
  t->piece_hi = mine.hi;
  L.crd = t->piece_crd - mine.lo;
  t->vals = t->piece_vals - mine.lo;
  t->restage_moved = moved;
  k_commit<<<grid_for(ctx, nrows + 1), 256, 0, s>>>(err_d, rp, L.rowptr, nrows + 1);
  SPD_CHECK_LAUNCH();
  if (cnt > 0) {
    k_commit<<<grid_for(ctx, cnt), 256, 0, s>>>(err_d, cd, t->piece_crd, cnt);
    SPD_CHECK_LAUNCH();
    k_commit<<<grid_for(ctx, cnt), 256, 0, s>>>(err_d, reinterpret_cast<const int64_t*>(vd),
                                                reinterpret_cast<int64_t*>(t->piece_vals), cnt);
    SPD_CHECK_LAUNCH();
  }
  SPD_CUDA(cudaMemcpyAsync(t->restage_err_host, err_d, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaEventRecord(t->restage_done, s));
  t->restage_pending = true;
  ctx->pending_restage.push_back(t);
}

static void restage_piece(spd_context* ctx, spd_tensor* t, const int64_t* const* pos_pairs,
                          const int64_t* const* crd, const double* vals) {
  if (t->piece_split != 1 && t->piece_split != 2)
    throw ValidationError("restage: a placed piece (spd_tensor_place) or a 3-level piece cannot be re-staged "
                          "from the host");
  const int64_t nrows = t->levels[1].parent_positions, nnz = t->levels[1].positions;
  const int64_t got = nrows == 0 ? 0 : (pos_pairs && pos_pairs[1] ? pos_pairs[1][2 * (nrows - 1) + 1] + 1 : -1);
  if (got != nnz)
    throw ValidationError("restage: level 1 holds " + std::to_string(nnz) + " positions, the new pos " +
                          std::to_string(got));
  stage_piece(ctx, t, pos_pairs[1], crd ? crd[1] : nullptr, vals, t->piece_split, false);
  for (auto& z : t->nz) z.R = nullptr;
  t->crd32h = nullptr;
  t->crd32h_rowbytes = 0;
  t->crd32 = nullptr;
  dev_free(ctx, t->crdc_alloc);
  t->crdc_alloc = t->crdc = nullptr;
  dev_free(ctx, t->cref);
  t->cref = nullptr;
  t->nref = -1;
  if (ctx->split_tensor == t) ctx->split = SplitKind::None, ctx->split_tensor = nullptr;
  if (ctx->bucket.tensor == t) ctx->bucket.tensor = nullptr;
}

// 3-level trees (dss / sss, the CSF of SpTTV / SpMTTKRP): the upper levels
// and the leaf row pointer are staged whole (O(fibres), the partition and
// the fibre walk need them); only this GPU's colour of the leaf crd / vals
// (split 2: nonzero split of the leaf level; 1: rows of the top level) is
// copied from the host arrays.  Restaging a 3-level piece is not supported.
static spd_tensor* upload_csf_piece(spd_context* ctx, const int64_t* dims, const int* kinds, const int* mode_order,
                                    const int64_t* const* pos_pairs, const int64_t* const* crd, const double* vals,
                                    int split) {
  spd_tensor* t = upload_impl(ctx, 3, dims, kinds, mode_order, pos_pairs, crd, vals, true, true, true);
  try {
    if (t->levels.size() != 3) throw ValidationError("unsupported on gpu: 3-tensor pieces need dss or sss");
    cudaStream_t s = ctx->stream;
    spd_level_store& L = t->levels[2];
    const int rc = split == 1 ? spd_partition_universe(ctx, t, ctx->world, nullptr)
                              : spd_partition_nonzero(ctx, t, 2, ctx->world, nullptr);
    if (rc != SPD_OK) throw ValidationError(spd_last_error());
    const spd_range mine = host_colors(ctx)[ctx->rank].q;
    const int64_t cnt = std::max<int64_t>(mine.hi - mine.lo + 1, 0);
    t->piece = true;
    t->piece_split = 0;  // not re-stageable
    t->piece_lo = mine.lo;
    t->piece_hi = mine.hi;
    t->piece_cap = std::max<int64_t>(cnt, 1);
    t->piece_crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * t->piece_cap);
    t->piece_vals = (double*)dev_alloc(ctx, sizeof(double) * t->piece_cap);
    L.crd = t->piece_crd - mine.lo;
    t->vals = t->piece_vals - mine.lo;
    int* err_d = (int*)ctx->counters.reserve(sizeof(int64_t) * 16) + 2;
    SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), s));
    if (cnt > 0) {
      if (!crd || !crd[2]) throw ValidationError("compressed level 2 needs crd");
      if (!vals) throw ValidationError("tensor: vals length does not match leaf count");
      SPD_CUDA(cudaMemcpyAsync(t->piece_crd, crd[2] + mine.lo, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, s));
      SPD_CUDA(cudaMemcpyAsync(t->piece_vals, vals + mine.lo, sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
      const int64_t nf = L.parent_positions;
      unsigned char* flags = (unsigned char*)dev_alloc(ctx, cnt);
      unsigned char* start = flags - mine.lo;
      SPD_CUDA(cudaMemsetAsync(flags, 0, cnt, s));
      k_mark_starts<<<grid_for(ctx, nf), 256, 0, s>>>(L.rowptr, nf, start, mine.lo, mine.hi);
      SPD_CHECK_LAUNCH();
      const int64_t dim = dims[mode_order[2]];
      k_check_crd<<<grid_for(ctx, cnt), 256, 0, s>>>(L.crd, mine.lo, mine.hi, dim, start, mine.lo > 0 ? 1 : 0,
                                                     mine.lo > 0 ? crd[2][mine.lo - 1] : 0, err_d);
      SPD_CHECK_LAUNCH();
      dev_free(ctx, flags);
    }
    int err_h = 0;
    SPD_CUDA(cudaMemcpyAsync(ctx->pinned_counters + 12, err_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&err_h, ctx->pinned_counters + 12, sizeof(int));
    if (err_h & 2) throw ValidationError("tensor: crd must be strictly increasing per range");
    if (err_h & 4) throw ValidationError("tensor: crd value out of dimension bounds");
  } catch (...) {
    spd_tensor_destroy(t);
    throw;
  }
  return t;
}

}  // namespace spd

int spd_tensor_upload_piece(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                            const int* mode_order, const int64_t* const* pos_pairs, const int64_t* const* crd,
                            const double* vals, int split, spd_tensor** out) {
  return guarded([&] {
    checked(ctx);
    if (!out) throw ValidationError("null output handle");
    if (split != 1 && split != 2) throw ValidationError("split must be 1 (rows) or 2 (nonzeros)");
    HostTrace ht("upload_piece");
    activate(ctx);
    if (order == 3) {
      *out = upload_csf_piece(ctx, dims, kinds, mode_order, pos_pairs, crd, vals, split);
      ht.mark("staged");
      return;
    }
    if (order != 2 || kinds[0] != SPD_DENSE || kinds[1] != SPD_COMPRESSED)
      throw ValidationError("unsupported on gpu: pieces of ds matrices and dss / sss 3-tensors");
    spd_tensor* t = make_skeleton(ctx, 2, dims, kinds, mode_order);
    try {
      const int64_t nrows = dims[mode_order[0]];
      if (nrows > 0 && (!pos_pairs || !pos_pairs[1])) throw ValidationError("compressed level 1 needs pos");
      const int64_t nnz = nrows == 0 ? 0 : pos_pairs[1][2 * (nrows - 1) + 1] + 1;
      if (nnz < 0) throw ValidationError("tensor: pos ranges must cover exactly [0, nnz)");
      t->levels[0].kind = SPD_DENSE;
      t->levels[0].dom = {nrows};
      t->levels[0].positions = nrows;
      spd_level_store& L = t->levels[1];
      L.kind = SPD_COMPRESSED;
      L.parent_positions = nrows;
      L.positions = nnz;
      L.rowptr = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (nrows + 1));
      t->nvals = nnz;
      t->piece = true;
      set_whole_span(t);
      stage_piece(ctx, t, nrows > 0 ? pos_pairs[1] : nullptr, crd ? crd[1] : nullptr, vals, split, true);
    } catch (...) {
      spd_tensor_destroy(t);
      throw;
    }
    ht.mark("staged");
    *out = t;
  });
}

int spd_tensor_restage(spd_context* ctx, spd_tensor* t, const int64_t* const* pos_pairs,
                       const int64_t* const* crd, const double* vals) {
  return guarded([&] {
    checked(ctx);
    if (!t) throw ValidationError("null tensor");
    if (t->ctx != ctx) throw ValidationError("restage: tensor belongs to another context");
    activate(ctx);
    settle_restage(t, true);  // the previous restage's verdict (its staging buffers are reused)
    if (t->piece) {
      restage_piece(ctx, t, pos_pairs, crd, vals);
      return;
    }
    if (!t->owns) throw ValidationError("restage: needs a tensor uploaded by spd_tensor_upload*");
    HostTrace ht("restage");
    cudaStream_t s = ctx->stream;
    // geometry checks on the host (nothing is queued before they pass)
    for (size_t l = 0; l < t->levels.size(); l++) {
      const spd_level_store& L = t->levels[l];
      if (L.kind != SPD_COMPRESSED) continue;
      const int64_t parent = L.parent_positions, nnz = L.positions;
      if (parent > 0 && (!pos_pairs || !pos_pairs[l]))
        throw ValidationError("compressed level " + std::to_string(l) + " needs pos");
      const int64_t got = parent == 0 ? 0 : pos_pairs[l][2 * (parent - 1) + 1] + 1;
      if (got != nnz) throw ValidationError("restage: level " + std::to_string(l) + " holds " +
                                            std::to_string(nnz) + " positions, the new pos " +
                                            std::to_string(got));
      if (nnz > 0 && (!crd || !crd[l]))
        throw ValidationError("compressed level " + std::to_string(l) + " needs crd");
    }
    if (t->nvals > 0 && !vals) throw ValidationError("tensor: vals length does not match leaf count");
    // staging arrays (allocated on the first restage, reused after)
    const size_t nl = t->levels.size();
    if (t->stage_rowptr.size() != nl) {
      t->stage_rowptr.assign(nl, nullptr);
      t->stage_crd.assign(nl, nullptr);
      for (size_t l = 0; l < nl; l++) {
        const spd_level_store& L = t->levels[l];
        if (L.kind != SPD_COMPRESSED) continue;
        t->stage_rowptr[l] = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (L.parent_positions + 1));
        t->stage_crd[l] = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * std::max<int64_t>(L.positions, 1));
      }
      t->stage_vals = (double*)dev_alloc(ctx, sizeof(double) * std::max<int64_t>(t->nvals, 1));
    }
    if (!t->restage_err) {
      t->restage_err = (int*)dev_alloc(ctx, sizeof(int));
      SPD_CUDA(cudaMallocHost((void**)&t->restage_err_host, sizeof(int)));
      SPD_CUDA(cudaEventCreateWithFlags(&t->restage_done, cudaEventDisableTiming));
    }
    int* err_d = t->restage_err;
    SPD_CUDA(cudaMemsetAsync(err_d, 0, sizeof(int), s));
    for (size_t l = 0; l < nl; l++) {
      spd_level_store& L = t->levels[l];
      if (L.kind != SPD_COMPRESSED) continue;
      const int64_t parent = L.parent_positions, nnz = L.positions;
      int64_t* rp = t->stage_rowptr[l];
      if (parent > 0) {
        if (t->stage_pairs_cap < 2 * parent) {
          dev_free(ctx, t->stage_pairs);
          t->stage_pairs = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * 2 * parent);
          t->stage_pairs_cap = 2 * parent;
        }
        SPD_CUDA(cudaMemcpyAsync(t->stage_pairs, pos_pairs[l], sizeof(int64_t) * 2 * parent,
                                 cudaMemcpyHostToDevice, s));
        k_pairs_to_rowptr<<<grid_for(ctx, parent), 256, 0, s>>>(t->stage_pairs, parent, nnz, rp, err_d);
        SPD_CHECK_LAUNCH();
      } else {
        SPD_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), s));
      }
      if (nnz > 0) {
        SPD_CUDA(cudaMemcpyAsync(t->stage_crd[l], crd[l], sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
        const int64_t need = std::max<int64_t>(nnz, parent);  // also the nz_view flags buffer
        if (t->stage_flags_cap < need) {
          dev_free(ctx, t->stage_flags);
          t->stage_flags = (unsigned char*)dev_alloc(ctx, need);
          t->stage_flags_cap = need;
        }
        SPD_CUDA(cudaMemsetAsync(t->stage_flags, 0, nnz, s));
        k_mark_starts<<<grid_for(ctx, parent), 256, 0, s>>>(rp, parent, t->stage_flags, 0, nnz - 1);
        SPD_CHECK_LAUNCH();
        const int64_t dim = t->dims[t->mode_order[t->groups[l][0]]];
        k_check_crd<<<grid_for(ctx, nnz), 256, 0, s>>>(t->stage_crd[l], 0, nnz - 1, dim, t->stage_flags, 0, 0,
                                                       err_d);
        SPD_CHECK_LAUNCH();
      }
    }
    if (t->nvals > 0)
      SPD_CUDA(cudaMemcpyAsync(t->stage_vals, vals, sizeof(double) * t->nvals, cudaMemcpyHostToDevice, s));
    // commit (skipped on the device when a check failed)
    for (size_t l = 0; l < nl; l++) {
      spd_level_store& L = t->levels[l];
      if (L.kind != SPD_COMPRESSED) continue;
      k_commit<<<grid_for(ctx, L.parent_positions + 1), 256, 0, s>>>(err_d, t->stage_rowptr[l], L.rowptr,
                                                                     L.parent_positions + 1);
      SPD_CHECK_LAUNCH();
      if (L.positions > 0) {
        k_commit<<<grid_for(ctx, L.positions), 256, 0, s>>>(err_d, t->stage_crd[l], L.crd, L.positions);
        SPD_CHECK_LAUNCH();
      }
    }
    if (t->nvals > 0) {
      k_commit<<<grid_for(ctx, t->nvals), 256, 0, s>>>(err_d, reinterpret_cast<const int64_t*>(t->stage_vals),
                                                       reinterpret_cast<int64_t*>(t->vals), t->nvals);
      SPD_CHECK_LAUNCH();
    }
    SPD_CUDA(cudaMemcpyAsync(t->restage_err_host, err_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaEventRecord(t->restage_done, s));
    t->restage_pending = true;
    ctx->pending_restage.push_back(t);
    // derived indices are functions of the old pattern: invalidate, keep buffers
    // (rebuilding them over an unchanged pattern after a rejection is harmless)
    for (auto& z : t->nz) z.R = nullptr;
    t->crd32h = nullptr;
    t->crd32h_rowbytes = 0;
    t->crd32 = nullptr;
    dev_free(ctx, t->crdc_alloc);
    t->crdc_alloc = t->crdc = nullptr;
    dev_free(ctx, t->cref);
    t->cref = nullptr;
    t->nref = -1;
    dev_free(ctx, t->jleaf);
    t->jleaf = nullptr;
    dev_free(ctx, t->leaf_rowptr);
    t->leaf_rowptr = nullptr;
    if (ctx->split_tensor == t) ctx->split = SplitKind::None, ctx->split_tensor = nullptr;
    if (ctx->bucket.tensor == t) ctx->bucket.tensor = nullptr;  // a function of the old pattern
    ht.mark("queued");
  });
}

int spd_tensor_upload_rowptr(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                             const int* mode_order, const int64_t* const* rowptr,
                             const int64_t* const* crd, const double* vals, int validate,
                             spd_tensor** out) {
  return guarded([&] {
    checked(ctx);
    *out = upload_impl(ctx, order, dims, kinds, mode_order, rowptr, crd, vals, false,
                       validate != 0);
  });
}

int spd_tensor_wrap_device(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                           const int* mode_order, int64_t* const* rowptr_dev,
                           int64_t* const* crd_dev, double* vals_dev, spd_tensor** out) {
  return guarded([&] {
    checked(ctx);
    activate(ctx);
    spd_tensor* t = make_skeleton(ctx, order, dims, kinds, mode_order);
    t->owns = false;
    int64_t parent = 1;
    for (size_t l = 0; l < t->groups.size(); l++) {
      spd_level_store& L = t->levels[l];
      L.parent_positions = parent;
      int k0 = t->groups[l][0];
      if (kinds[k0] == SPD_DENSE) {
        int64_t total = 1;
        for (int k : t->groups[l]) L.dom.push_back(dims[mode_order[k]]), total *= dims[mode_order[k]];
        parent *= total;
        L.positions = parent;
        continue;
      }
      L.kind = SPD_COMPRESSED;
      L.rowptr = rowptr_dev[l];
      L.crd = crd_dev[l];
      int64_t nnz = 0;
      SPD_CUDA(cudaMemcpyAsync(&nnz, L.rowptr + parent, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
      SPD_CUDA(cudaStreamSynchronize(ctx->stream));
      L.positions = nnz;
      parent = nnz;
    }
    t->nvals = parent;
    set_whole_span(t);
    t->vals = vals_dev;
    *out = t;
  });
}

int spd_tensor_destroy(spd_tensor* t) {
  return guarded([&] {
    if (!t) return;
    HostTrace ht("destroy");
    spd_context* ctx = t->ctx;
    activate(ctx);
    if (ctx->split_tensor == t) {
      ctx->split = SplitKind::None;
      ctx->split_tensor = nullptr;
    }
    if (ctx->bucket.tensor == t) ctx->bucket.tensor = nullptr;
    if (t->restage_pending) {  // the verdict is dropped with the tensor
      cudaEventSynchronize(t->restage_done);
      auto& pend = ctx->pending_restage;
      pend.erase(std::remove(pend.begin(), pend.end(), t), pend.end());
    }
    for (int64_t* p : t->stage_rowptr) dev_free(ctx, p);
    for (int64_t* p : t->stage_crd) dev_free(ctx, p);
    dev_free(ctx, t->stage_vals);
    dev_free(ctx, t->restage_err);
    if (t->restage_err_host) cudaFreeHost(t->restage_err_host);
    if (t->restage_done) cudaEventDestroy(t->restage_done);
    if (t->piece) {
      for (size_t l = 0; l + 1 < t->levels.size(); l++) {
        dev_free(ctx, t->levels[l].rowptr);
        dev_free(ctx, t->levels[l].crd);
      }
      dev_free(ctx, t->levels.back().rowptr);
      dev_free(ctx, t->piece_crd);
      dev_free(ctx, t->piece_vals);
    } else if (t->owns) {
      for (auto& L : t->levels) {
        dev_free(ctx, L.rowptr);
        dev_free(ctx, L.crd);
      }
      dev_free(ctx, t->vals);
    }
    dev_free(ctx, t->leaf_rowptr);
    dev_free(ctx, t->crd32h_alloc);
    dev_free(ctx, t->crd32_alloc);
    dev_free(ctx, t->crdc_alloc);
    dev_free(ctx, t->cref);
    dev_free(ctx, t->stage_pairs);
    dev_free(ctx, t->stage_flags);
    dev_free(ctx, t->jleaf);
    for (auto& z : t->nz) {
      dev_free(ctx, z.ptr);
      dev_free(ctx, z.id);
      dev_free(ctx, z.m_dev);
    }
    delete t;
    ht.mark("freed");
  });
}

int spd_tensor_num_levels(const spd_tensor* t, int* nlevels) {
  return guarded([&] {
    if (!t) throw ValidationError("null tensor");
    *nlevels = (int)t->levels.size();
  });
}

int spd_tensor_level(const spd_tensor* t, int level, int* kind, int64_t* parent_positions,
                     int64_t* positions) {
  return guarded([&] {
    if (!t || level < 0 || level >= (int)t->levels.size()) throw ValidationError("no such level");
    const auto& L = t->levels[level];
    *kind = L.kind;
    *parent_positions = L.parent_positions;
    *positions = L.positions;
  });
}

int spd_tensor_nvals(const spd_tensor* t, int64_t* nvals) {
  return guarded([&] {
    if (!t) throw ValidationError("null tensor");
    *nvals = t->nvals;
  });
}

int spd_tensor_device_ptrs(const spd_tensor* t, int level, int64_t** rowptr, int64_t** crd) {
  return guarded([&] {
    if (!t || level < 0 || level >= (int)t->levels.size()) throw ValidationError("no such level");
    *rowptr = t->levels[level].rowptr;
    *crd = t->levels[level].crd;
  });
}

int spd_tensor_vals_ptr(const spd_tensor* t, double** vals) {
  return guarded([&] {
    if (!t) throw ValidationError("null tensor");
    *vals = t->vals;
  });
}

int spd_tensor_download_level(const spd_tensor* t, int level, int64_t* pos_pairs, int64_t* crd) {
  return guarded([&] {
    if (!t || level < 0 || level >= (int)t->levels.size()) throw ValidationError("no such level");
    const auto& L = t->levels[level];
    if (L.kind != SPD_COMPRESSED) throw ValidationError("level is dense: nothing stored");
    if (t->piece && crd && level + 1 == (int)t->levels.size())
      throw ValidationError("a placed piece holds only its colour's positions: download the whole tensor");
    spd_context* ctx = t->ctx;
    activate(ctx);
    settle_restage(t, true);
    activate(ctx);
    if (pos_pairs && L.parent_positions > 0) {
      int64_t* tmp = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * 2 * L.parent_positions);
      k_rowptr_to_pairs<<<grid_for(ctx, L.parent_positions), 256, 0, ctx->stream>>>(
          L.rowptr, L.parent_positions, tmp);
      SPD_CHECK_LAUNCH();
      SPD_CUDA(cudaMemcpyAsync(pos_pairs, tmp, sizeof(int64_t) * 2 * L.parent_positions,
                               cudaMemcpyDeviceToHost, ctx->stream));
      dev_free(ctx, tmp);
    }
    if (crd && L.positions > 0)
      SPD_CUDA(cudaMemcpyAsync(crd, L.crd, sizeof(int64_t) * L.positions, cudaMemcpyDeviceToHost,
                               ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int spd_tensor_download_rowptr(const spd_tensor* t, int level, int64_t* rowptr) {
  return guarded([&] {
    if (!t || level < 0 || level >= (int)t->levels.size()) throw ValidationError("no such level");
    const auto& L = t->levels[level];
    if (L.kind != SPD_COMPRESSED) throw ValidationError("level is dense: nothing stored");
    spd_context* ctx = t->ctx;
    activate(ctx);
    settle_restage(t, true);
    activate(ctx);
    SPD_CUDA(cudaMemcpyAsync(rowptr, L.rowptr, sizeof(int64_t) * (L.parent_positions + 1),
                             cudaMemcpyDeviceToHost, ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int spd_tensor_download_vals(const spd_tensor* t, double* vals) {
  return guarded([&] {
    if (!t) throw ValidationError("null tensor");
    if (t->piece) throw ValidationError("a placed piece holds only its colour's positions");
    spd_context* ctx = t->ctx;
    activate(ctx);
    settle_restage(t, true);
    activate(ctx);
    if (t->nvals > 0)
      SPD_CUDA(cudaMemcpyAsync(vals, t->vals, sizeof(double) * t->nvals, cudaMemcpyDeviceToHost,
                               ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int spd_tensor_download_vals_range(const spd_tensor* t, int64_t first, int64_t count,
                                   double* vals) {
  return guarded([&] {
    if (!t) throw ValidationError("null tensor");
    if (first < 0 || count < 0 || first + count > t->nvals) throw ValidationError("range outside vals");
    if (t->piece && count > 0 && (first < t->piece_lo || first + count - 1 > t->piece_hi))
      throw ValidationError("range outside the placed piece");
    spd_context* ctx = t->ctx;
    activate(ctx);
    settle_restage(t, true);
    activate(ctx);
    if (count > 0)
      SPD_CUDA(cudaMemcpyAsync(vals, t->vals + first, sizeof(double) * count,
                               cudaMemcpyDeviceToHost, ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int spd_last_owned(spd_context* ctx, int64_t first, int64_t count, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    checked(ctx);
    if (!lo || !hi) throw ValidationError("null argument");
    if (first < 0 || count < 1 || first + count > ctx->pieces) throw ValidationError("colour range outside the partition");
    activate(ctx);
    std::vector<DevColor> d(count);
    SPD_CUDA(cudaMemcpyAsync(d.data(), (const DevColor*)ctx->colors_dev.ptr + first, sizeof(DevColor) * count,
                             cudaMemcpyDeviceToHost, ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
    *lo = INT64_MAX;
    *hi = -1;
    for (const DevColor& c : d)
      if (c.w_lo <= c.w_hi) *lo = std::min(*lo, c.w_lo), *hi = std::max(*hi, c.w_hi);
    if (*hi < 0) *lo = 0;
  });
}

int spd_split_colour_blocks(const double* cost, int64_t pieces, int world, int64_t* bounds) {
  return guarded([&] {
    if (!cost || !bounds) throw ValidationError("null argument");
    if (world < 1 || pieces < world) throw ValidationError("need at least one colour per GPU");
    std::vector<double> pre(pieces + 1, 0.0);
    for (int64_t c = 0; c < pieces; c++) {
      if (!(cost[c] >= 0.0)) throw ValidationError("colour costs must be non-negative");
      pre[c + 1] = pre[c] + cost[c];
    }
    // boundary r at the prefix nearest r / world of the total, every block non-empty
    bounds[0] = 0;
    for (int r = 1; r < world; r++) {
      const double target = pre[pieces] * r / world;
      const int64_t lo = bounds[r - 1] + 1, hi = pieces - (world - r);
      int64_t b = std::lower_bound(pre.begin() + lo, pre.begin() + hi + 1, target) - pre.begin();
      if (b > hi) b = hi;
      if (b > lo && target - pre[b - 1] <= pre[b] - target) b--;
      bounds[r] = b;
    }
    bounds[world] = pieces;
  });
}

int spd_context_set_colour_blocks(spd_context* ctx, int64_t pieces, const int64_t* bounds) {
  return guarded([&] {
    checked(ctx);
    if (bounds == nullptr) {  // back to even blocks
      ctx->blocks.clear();
      ctx->blocks_pieces = -1;
      return;
    }
    if (pieces < ctx->world) throw ValidationError("need at least one colour per GPU");
    if (bounds[0] != 0 || bounds[ctx->world] != pieces) throw ValidationError("colour blocks must tile [0, pieces)");
    for (int r = 0; r < ctx->world; r++)
      if (bounds[r + 1] <= bounds[r]) throw ValidationError("every GPU needs a non-empty colour block");
    activate(ctx);
    ctx->blocks.assign(bounds, bounds + ctx->world + 1);
    ctx->blocks_pieces = pieces;
    SPD_CUDA(cudaMemcpyAsync(ctx->blocks_dev.reserve(sizeof(int64_t) * (ctx->world + 1)), bounds,
                             sizeof(int64_t) * (ctx->world + 1), cudaMemcpyHostToDevice, ctx->stream));
    SPD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int spd_context_colour_blocks(spd_context* ctx, int64_t pieces, int64_t* bounds) {
  return guarded([&] {
    checked(ctx);
    if (!bounds) throw ValidationError("null argument");
    if (pieces < 1) throw ValidationError("pieces must be positive");
    for (int r = 0; r < ctx->world; r++) {  // the blocks a partition of `pieces` colours gets
      int64_t f, c;
      colour_block(ctx, pieces, r, f, c);
      bounds[r] = f;
    }
    bounds[ctx->world] = pieces;
  });
}

int spd_last_work(spd_context* ctx, int64_t* work, int64_t pieces) {
  return guarded([&] {
    checked(ctx);
    if (pieces != (int64_t)ctx->last_work.size()) throw ValidationError("pieces mismatch");
    for (int64_t c = 0; c < pieces; c++) work[c] = ctx->last_work[c];
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// CUDA graphs: a sequence of ops on a context (partition + leaf + combine of
// a step) captured once and replayed, so launch-bound small problems pay one
// graph launch instead of a dozen host API calls per step.  Ops stay
// capturable as long as they need no host read-back: colours kept on the
// device (colors_out NULL), stats NULL, derived indices already built.
struct spd_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" {

int spd_capture_begin(spd_context* ctx) {
  return guarded([&] {
    checked(ctx);
    if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy || ctx->stream == cudaStreamPerThread)
      throw ValidationError("capture needs a context on an explicit stream (not the legacy default stream)");
    activate(ctx);
    SPD_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  });
}

int spd_capture_end(spd_context* ctx, spd_graph** out) {
  return guarded([&] {
    checked(ctx);
    if (!out) throw ValidationError("null output handle");
    activate(ctx);
    auto* g = new spd_graph();
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g->graph);
    if (e != cudaSuccess) {
      if (g->graph) cudaGraphDestroy(g->graph);
      delete g;
      (void)cudaGetLastError();  // an invalidated capture is not a sticky error: clear it
      throw RuntimeError(std::string("stream capture failed (an op needed a host read-back?): ") +
                         cudaGetErrorString(e));
    }
    e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g->graph);
      delete g;
      SPD_CUDA(e);
    }
    *out = g;
  });
}

int spd_graph_launch(spd_graph* g, spd_context* ctx) {
  return guarded([&] {
    checked(ctx);
    if (!g) throw ValidationError("null spd_graph");
    activate(ctx);
    SPD_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
    ctx->launches += 1;
  });
}

int spd_graph_destroy(spd_graph* g) {
  return guarded([&] {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
  });
}

}  // extern "C"
