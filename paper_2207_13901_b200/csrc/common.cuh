// Internal definitions shared by the sm_100a translation units of
// libspdistal_b200.so.  Nothing here is part of the C-ABI (include/spdistal_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>

#include <chrono>
#include <cstdlib>

#include <stdexcept>
#include <string>
#include <vector>

#include "spdistal_b200.h"

namespace spd {

// Error classes of the reference (errors.hpp:11-40) mapped onto ABI codes.
struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct RuntimeError : std::runtime_error {
  explicit RuntimeError(const std::string& m) : std::runtime_error(m) {}
};

void set_last_error(const std::string& msg);

#define SPD_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t spd_e_ = (call);                                                         \
    if (spd_e_ != cudaSuccess)                                                           \
      throw ::spd::RuntimeError(std::string("CUDA error ") + cudaGetErrorString(spd_e_) + \
                                " at " __FILE__ ":" + std::to_string(__LINE__));         \
  } while (0)
#define SPD_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t spd_r_ = (call);                                                        \
    if (spd_r_ != ncclSuccess)                                                           \
      throw ::spd::RuntimeError(std::string("NCCL error ") + ncclGetErrorString(spd_r_) + \
                                " at " __FILE__ ":" + std::to_string(__LINE__));         \
  } while (0)
#define SPD_CHECK_LAUNCH() SPD_CUDA(cudaGetLastError())

// Runs `f` and maps exceptions onto the ABI status codes.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return SPD_OK;
  } catch (const ValidationError& e) {
    set_last_error(e.what());
    return SPD_ERR_VALIDATION;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return SPD_ERR_VALIDATION;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SPD_ERR_RUNTIME;
  }
}

// Host-side wall-clock trace of an API call's stages (SPD_HOST_TRACE=1,
// stderr): where a caller's thread blocks (syncs, allocations).
struct HostTrace {
  const char* name;
  std::chrono::steady_clock::time_point t0, t;
  bool on;
  explicit HostTrace(const char* n) : name(n) {
    static const bool enabled = [] {
      const char* e = getenv("SPD_HOST_TRACE");
      return e && atoi(e) != 0;
    }();
    on = enabled;
    if (on) t0 = t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[spd %s] %s %.2f ms\n", name, what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Grow-only device scratch buffer.
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* reserve(size_t n) {
    if (n > bytes) {
      if (ptr) SPD_CUDA(cudaFree(ptr));
      ptr = nullptr;
      size_t want = n + n / 4;
      SPD_CUDA(cudaMalloc(&ptr, want));
      bytes = want;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

// One colour as the kernels see it: the public spd_color plus the output
// write range (the rows this colour must store, tiling [0, rows) across
// colours in order).
struct DevColor {
  spd_color pub;
  int64_t w_lo, w_hi;       // output rows written by this colour (op-specific)
  int64_t chunk_begin;      // first virtual chunk of this colour (op-specific)
  int64_t pad;
};
static_assert(sizeof(spd_color) == 64, "spd_color layout");

enum class SplitKind { None = 0, Universe = 1, NonZero = 2 };

}  // namespace spd

struct spd_level_store {
  int kind = SPD_DENSE;
  std::vector<int64_t> dom;   // dense: extents of the collapsed modes
  int64_t parent_positions = 1;
  int64_t positions = 0;      // level_positions
  int64_t* rowptr = nullptr;  // compressed: parent_positions + 1
  int64_t* crd = nullptr;     // compressed: positions
};

struct spd_tensor {
  spd_context* ctx = nullptr;
  int order = 0;
  std::vector<int64_t> dims;
  std::vector<int> kinds, mode_order;
  std::vector<std::vector<int>> groups;  // level grouping (tensor.cpp:30-41)
  std::vector<spd_level_store> levels;
  int64_t nvals = 0;
  double* vals = nullptr;
  bool owns = true;
  // Derived device index for 3-level trees: rows -> leaf positions
  // (rp2[rp1[i]]), built on first use by SpMTTKRP.
  int64_t* leaf_rowptr = nullptr;
  // Compacted non-empty-row views (DCSR-style) of row pointers of this
  // tensor, built on first use by the leaf kernels (leaf_nz.cuh).
  struct NzCache {
    const int64_t* R = nullptr;
    int64_t* ptr = nullptr;
    int64_t* id = nullptr;
    int64_t* m_dev = nullptr;  // count of non-empty rows, on the device
    int64_t m = -1;            // host copy, -1 until read
    int64_t cap_id = 0;        // allocated rows of id (ptr: cap_id + 1), reused after a restage
  } nz[3];
  // Staging buffers of spd_tensor_restage (pos pairs, row-start flags), kept
  // so a per-step re-upload allocates nothing.
  int64_t* stage_pairs = nullptr;
  int64_t stage_pairs_cap = 0;
  unsigned char* stage_flags = nullptr;
  int64_t stage_flags_cap = 0;
  // spd_tensor_restage validates before it swaps: the new row pointers, crd
  // and vals land in these staging arrays, are checked on the device, and a
  // commit kernel copies them over the live arrays only if every check
  // passed -- a rejected restage leaves the tensor exactly as it was.  The
  // verdict travels to the host without a synchronisation (pinned copy +
  // event) and is reported by the next call on the tensor once the event has
  // completed, or by spd_context_synchronize.
  std::vector<int64_t*> stage_rowptr, stage_crd;  // per level
  int64_t stage_leaf_cap = 0;                     // leaf crd / vals entries allocated
  double* stage_vals = nullptr;
  int* restage_err = nullptr;       // device flags of the last restage
  int* restage_err_host = nullptr;  // pinned copy
  cudaEvent_t restage_done = nullptr;
  bool restage_pending = false;
  bool restage_moved = false;  // the last restage moved a row-split piece's range
  // A piece whose row-split range moved in a restage that was then rejected:
  // its arrays no longer match its range, every later call refuses it.
  bool poisoned = false;
  // Leaf crd as int32 with bit 31 = "hot column" (its dense row is among the
  // most referenced ones that fit in L2), for row-gathering kernels; built on
  // first use for a given dense-row size (crd32h_rowbytes).
  int32_t* crd32h = nullptr;
  int64_t crd32h_rowbytes = 0;
  // 3-level trees: middle-mode coordinate of every leaf (crd1 of its fibre).
  int32_t* jleaf = nullptr;
  // Row block and global pos offset of a distributed (per-GPU) piece of an
  // assembled output (spd_spadd3 with a communicator); a whole tensor has
  // rows [0, n) and pos_base 0.  global_positions < 0: not an assembled output.
  int64_t row_lo = 0, row_hi = -1, pos_base = 0, global_positions = -1;
  // A placed piece (spd_tensor_place): the leaf level's crd/vals hold only
  // positions [piece_lo, piece_hi]; the level pointers are offset so global
  // positions index them, the allocations are piece_crd / piece_vals.  The
  // row pointer is whole (O(rows), for the partition step).
  bool piece = false;
  int64_t piece_lo = 0, piece_hi = -1;
  int64_t piece_cap = 0;  // allocated positions of piece_crd / piece_vals
  int piece_split = 0;  // 1 rows / 2 nonzeros: re-stageable from the host (upload_piece, place); 0 not (3-level pieces)
  int64_t* piece_crd = nullptr;
  double* piece_vals = nullptr;
  int32_t* crd32h_alloc = nullptr;  // allocation behind crd32h (offset for pieces)
  // int32 copy of the leaf crd (the N = 32 SpMM leaf), indexed by global
  // position; crd32_alloc / crd32_cap the allocation behind it.
  int32_t* crd32 = nullptr;
  int32_t* crd32_alloc = nullptr;
  int64_t crd32_cap = 0;
  // Compacted-column index (SpMV over a wide x): the referenced columns of
  // the leaf level renumbered densely in ascending order -- crdc[q] = rank of
  // crd[q] among them, cref[r] = the column of rank r, nref of them -- so a
  // per-call gather xc[r] = x[cref[r]] packs every x entry the leaf reads
  // into nref * 8 bytes that stay L2-resident.
  int32_t* crdc = nullptr;        // indexed by global position (offset for pieces)
  int32_t* crdc_alloc = nullptr;  // allocation behind crdc
  int32_t* cref = nullptr;
  int64_t nref = -1;
};

struct spd_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // Auxiliary stream for work that overlaps the leaf (the zero-fill of empty
  // output rows), forked from / joined into `stream` with events.
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;

  // Last partition (spd_partition_*): device + host copies of the colours.
  spd::SplitKind split = spd::SplitKind::None;
  const spd_tensor* split_tensor = nullptr;
  int split_level = 0;
  int64_t pieces = 0;
  spd::DeviceBuffer colors_dev;      // spd::DevColor[pieces]
  std::vector<spd_color> colors_host;
  bool colors_host_valid = false;

  // Colour blocks per GPU: rank r runs colours [blocks[r], blocks[r + 1]) of a
  // `blocks_pieces`-colour partition (spd_context_set_colour_blocks); unset or
  // set for another colour count: even blocks of ceil(P / world) colours.
  std::vector<int64_t> blocks;
  int64_t blocks_pieces = -1;
  spd::DeviceBuffer blocks_dev;      // the same bounds on the device (head-record unpack)

  std::vector<int64_t> last_work;    // per colour
  std::vector<spd_tensor*> pending_restage;  // tensors whose last restage verdict is still on its way
  // Last bucket split (spd_partition_bucket): positions of the level sorted by
  // colour (ascending within a colour), colour offsets, prefix sums of the
  // leaf counts under the sorted positions.
  struct Bucket {
    const spd_tensor* tensor = nullptr;
    int level = 0;
    int64_t n = 0, pieces = 0;
    int64_t *pos = nullptr, *pref = nullptr, *off = nullptr;
    spd::DeviceBuffer keys, tmp, pos_buf, pref_buf, off_buf;
  } bucket;
  spd::DeviceBuffer scratch[8];  // [7]: compacted x (SpMV)
  spd::DeviceBuffer counters;        // small int64 device counters
  int64_t* pinned_counters = nullptr;

  // Instrumentation (spd_context_timing / spd_context_launches).
  int64_t launches = 0;
  int timing = 0;  // 0 off, 1 leaf pairs, 2 phase markers
  std::vector<cudaEvent_t> timing_events;  // pairs, grow-only pool
  size_t timing_used = 0;                  // events in use (2 per leaf launch)
};

namespace spd {

constexpr int kWarp = 32;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// First index i in [0, n) with a[i] > key (n if none): a 32-ary search in
// which every round issues one coalescable load per lane -- 5 dependent
// rounds for 16.7M rows instead of 24 for a scalar binary search.  Must be
// called by a full, converged warp; returns the same value on every lane.
__device__ __forceinline__ int64_t warp_upper_bound(const int64_t* __restrict__ a, int64_t n,
                                                    int64_t key) {
  const int lane = lane_id();
  int64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    int64_t step = (hi - lo + 31) / 32;
    int64_t idx = lo + lane * step;
    bool pred = idx < hi && __ldg(a + idx) <= key;
    unsigned m = __ballot_sync(0xffffffffu, pred);
    int cnt = __popc(m);
    if (cnt == 0) return lo;
    int64_t nlo = lo + (int64_t)(cnt - 1) * step + 1;
    int64_t nhi = lo + (int64_t)cnt * step;
    hi = nhi < hi ? nhi : hi;
    lo = nlo;
  }
  int64_t idx = lo + lane;
  bool pred = idx < hi && __ldg(a + idx) <= key;
  unsigned m = __ballot_sync(0xffffffffu, pred);
  return lo + __popc(m);
}

// Parent entry whose range contains position q (tensor.cpp:221-235):
// the last p with rowptr[p] <= q, over rowptr[0..npos].
__device__ __forceinline__ int64_t warp_owner(const int64_t* __restrict__ rowptr, int64_t npos,
                                              int64_t q) {
  return warp_upper_bound(rowptr, npos + 1, q) - 1;
}

// warp_owner over fewer than 2^31 rows, in 32-bit index arithmetic (keeps the
// register-tight leaves free of spills).
__device__ __forceinline__ int warp_owner32(const int64_t* __restrict__ rowptr, int npos, int64_t q) {
  const int lane = lane_id();
  int lo = 0, hi = npos + 1;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int idx = lo + lane * step;
    const unsigned m = __ballot_sync(0xffffffffu, idx < hi && __ldg(rowptr + idx) <= q);
    const int cnt = __popc(m);
    if (cnt == 0) return lo - 1;
    const int nhi = lo + cnt * step;
    lo = lo + (cnt - 1) * step + 1;
    hi = nhi < hi ? nhi : hi;
  }
  const int idx = lo + lane;
  return lo + __popc(__ballot_sync(0xffffffffu, idx < hi && __ldg(rowptr + idx) <= q)) - 1;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// The leaf kernels read a tensor's levels in mode order (level 0 = output
// row i, ...).  A transposed storage order (a CSC 'ds:1,0', a column-major
// dense 'dd:1,0') is accepted by the reference (format_lang.hpp) but would be
// read as the identity order here, so it is rejected like any other
// unsupported format (advisor finding, round 1).
inline void require_identity_order(const spd_tensor* t, const char* what) {
  for (size_t k = 0; k < t->mode_order.size(); k++)
    if (t->mode_order[k] != (int)k)
      throw ValidationError(std::string("unsupported on gpu: ") + what +
                            " must be stored in mode order (no transposed storage)");
}

// Host-side helpers implemented in context.cu.
spd_context* checked(spd_context* ctx);
// Reports the verdict of t's last spd_tensor_restage (ValidationError when it
// was rejected) once it is known; `block` waits for it.  Also refuses a
// poisoned piece.  Every call that uses a tensor starts with it.
void settle_restage(const spd_tensor* t, bool block = false);
void activate(spd_context* ctx);
const std::vector<spd_color>& host_colors(spd_context* ctx);  // syncs if needed
void require_partition(spd_context* ctx, const spd_tensor* t, int64_t first, int64_t count,
                       bool allow_grid = false);
// Colour block of rank r in a P-colour partition (see spd_context::blocks);
// count 0 when r runs none.  The first form uses the current partition's P.
void colour_block(const spd_context* ctx, int64_t P, int r, int64_t& first, int64_t& count);
void colour_block(const spd_context* ctx, int r, int64_t& first, int64_t& count);
// Colours of the compute partition a piece placement follows: the installed
// blocks' colour count, else one colour per GPU.
int64_t placement_pieces(const spd_context* ctx);
// Leaf position span of every rank's block of a P-colour nonzero (split 2) or
// row (split 1) partition of the CSR t (partitions t on ctx).
std::vector<spd_range> rank_spans(spd_context* ctx, spd_tensor* t, int split, int64_t P);
// Whether the blocks in force are the even ceil(P / world) ones.
bool even_blocks(const spd_context* ctx);
void fill_stats(spd_context* ctx, spd_stats* st, int64_t combines, const std::vector<int64_t>& work,
                int64_t launches, bool timed);
// Brackets the leaf kernel of an op with a timing event pair when enabled.
void leaf_timing_begin(spd_context* ctx);
void leaf_timing_end(spd_context* ctx);
// Tensor construction helpers (context.cu): level skeleton from a FormatSpec
// (tensor.cpp:30-92), whole-tensor span, stream-ordered allocation.
spd_tensor* make_skeleton(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                          const int* mode_order);
void set_whole_span(spd_tensor* t);
void* dev_alloc(spd_context* ctx, size_t bytes);
void dev_free(spd_context* ctx, void* p);
// Phase marker (timing mode 2): per-phase device time of an op.
void trace_mark(spd_context* ctx);

}  // namespace spd
