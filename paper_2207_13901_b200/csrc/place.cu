// Data placement on GPUs: a CSR matrix distributed over
// the communicator's GPUs by the row or nonzero partition of its compute
// schedule -- the matched distribution of lower_tdn + residency_from_
// placements (/root/reference/proj/core/src/planner.cpp:361-439,
// sim.cpp:547-566) for which the compute-time ledger charges 0 bytes
// (SPEC.md:426).
//
// Every GPU receives the row pointer (O(rows): the partition step needs it,
// and it is what the reference's preimage walks) and only its colour's
// crd/vals positions (O(nnz / GPUs)): one NCCL broadcast and grouped
// send/recv from the root, no host staging.  The result is a "piece"
// tensor whose leaf arrays are indexed by global position, so the leaf ops
// run on it unchanged for that colour.  The bytes each GPU received are
// returned (the placement's cost, reported apart from compute).
#include <algorithm>
#include <string>

#include "common.cuh"

namespace spd {
std::vector<int64_t> nonempty_in_spans(spd_context* ctx, spd_tensor* t, const int64_t* R, int64_t nrows,
                                       const std::vector<int64_t>& spans);
}

namespace spd {

namespace {

void run_place(spd_context* ctx, int root, const spd_tensor* whole, int split, spd_tensor** out,
               int64_t* bytes_in) {
  checked(ctx);
  if (!out) throw ValidationError("null output handle");
  if (!ctx->comm) throw ValidationError("spd_tensor_place needs a communicator");
  if (root < 0 || root >= ctx->world) throw ValidationError("root outside the communicator");
  if (split != 1 && split != 2) throw ValidationError("split must be 1 (rows) or 2 (nonzeros)");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  const bool is_root = ctx->rank == root;
  // header: order, dims (2), mode order, nnz, rows, root status.  The root's
  // input checks travel in the header, so every rank fails together instead
  // of the others waiting in a collective the root never joins.
  int64_t hdr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::string root_error;
  if (is_root) {
    if (!whole) root_error = "the root must pass the whole tensor";
    else if (whole->piece) root_error = "cannot place a piece";
    else if (whole->levels.size() != 2 || whole->levels[0].kind != SPD_DENSE ||
             whole->levels[1].kind != SPD_COMPRESSED)
      root_error = "unsupported on gpu: placement of ds (CSR-like) matrices";
    if (root_error.empty()) {
      hdr[0] = whole->order;
      hdr[1] = whole->dims[0];
      hdr[2] = whole->dims[1];
      hdr[3] = whole->mode_order[0];
      hdr[4] = whole->mode_order[1];
      hdr[5] = whole->levels[1].positions;
      hdr[6] = whole->levels[1].parent_positions;
    } else {
      hdr[7] = 1;
    }
  }
  int64_t* dh = (int64_t*)ctx->counters.reserve(sizeof(hdr));
  SPD_CUDA(cudaMemcpyAsync(dh, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
  SPD_NCCL(ncclBroadcast(dh, dh, 8, ncclInt64, root, ctx->comm, s));
  SPD_CUDA(cudaMemcpyAsync(hdr, dh, sizeof(hdr), cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  if (hdr[7]) throw ValidationError(is_root ? root_error : "spd_tensor_place: the root rejected its input");
  const int64_t dims[2] = {hdr[1], hdr[2]};
  const int kinds[2] = {SPD_DENSE, SPD_COMPRESSED};
  const int mo[2] = {(int)hdr[3], (int)hdr[4]};
  const int64_t nnz = hdr[5], nrows = hdr[6];
  spd_tensor* t = make_skeleton(ctx, 2, dims, kinds, mo);
  try {
    t->levels[0].kind = SPD_DENSE;
    t->levels[0].dom = {nrows};
    t->levels[0].positions = nrows;
    spd_level_store& L = t->levels[1];
    L.kind = SPD_COMPRESSED;
    L.parent_positions = nrows;
    L.positions = nnz;
    L.rowptr = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (nrows + 1));
    if (is_root)
      SPD_CUDA(cudaMemcpyAsync(L.rowptr, whole->levels[1].rowptr, sizeof(int64_t) * (nrows + 1),
                               cudaMemcpyDeviceToDevice, s));
    SPD_NCCL(ncclBroadcast(L.rowptr, L.rowptr, nrows + 1, ncclInt64, root, ctx->comm, s));
    t->nvals = nnz;
    t->piece = true;
    t->piece_split = split;
    set_whole_span(t);
    // the compute partition, the same on every GPU: one colour per GPU, or
    // each GPU's block of the installed colour blocks (over-decomposition)
    const std::vector<spd_range> span = rank_spans(ctx, t, split, placement_pieces(ctx));
    const spd_range mine = span[ctx->rank];
    t->piece_lo = mine.lo;
    t->piece_hi = mine.hi;
    const int64_t cnt = std::max<int64_t>(mine.hi - mine.lo + 1, 0);
    t->piece_cap = std::max<int64_t>(cnt, 1);  // a placed piece can be re-staged from the host later
    t->piece_crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * t->piece_cap);
    t->piece_vals = (double*)dev_alloc(ctx, sizeof(double) * t->piece_cap);
    L.crd = t->piece_crd - mine.lo;  // indexed by global position
    t->vals = t->piece_vals - mine.lo;
    SPD_NCCL(ncclGroupStart());
    if (is_root) {
      for (int r = 0; r < ctx->world; r++) {
        const spd_range q = span[r];
        const int64_t c = q.hi - q.lo + 1;
        if (c <= 0) continue;
        if (r == root) {
          SPD_CUDA(cudaMemcpyAsync(t->piece_crd, whole->levels[1].crd + q.lo, sizeof(int64_t) * c,
                                   cudaMemcpyDeviceToDevice, s));
          SPD_CUDA(cudaMemcpyAsync(t->piece_vals, whole->vals + q.lo, sizeof(double) * c,
                                   cudaMemcpyDeviceToDevice, s));
        } else {
          SPD_NCCL(ncclSend(whole->levels[1].crd + q.lo, c, ncclInt64, r, ctx->comm, s));
          SPD_NCCL(ncclSend(whole->vals + q.lo, c, ncclFloat64, r, ctx->comm, s));
        }
      }
    } else if (cnt > 0) {
      SPD_NCCL(ncclRecv(t->piece_crd, cnt, ncclInt64, root, ctx->comm, s));
      SPD_NCCL(ncclRecv(t->piece_vals, cnt, ncclFloat64, root, ctx->comm, s));
    }
    SPD_NCCL(ncclGroupEnd());
    SPD_CUDA(cudaStreamSynchronize(s));
    if (bytes_in) *bytes_in = is_root ? 0 : (int64_t)sizeof(int64_t) * (nrows + 1) + 16 * cnt;
  } catch (...) {
    spd_tensor_destroy(t);
    throw;
  }
  *out = t;
}

// Moves a piece to another compute partition: every GPU computes, from the
// whole row pointer it holds, every GPU's held range (the piece's own split)
// and needed range (need_split) -- contiguous leaf position spans -- and the
// overlaps travel as grouped NCCL send/recv of crd and vals; the local
// overlap is a device copy.  The result is a new piece for colour `rank` of
// need_split; *bytes_in = crd + vals bytes received over NCCL.
void run_repartition(spd_context* ctx, const spd_tensor* t, int need_split, spd_tensor** out, int64_t* bytes_in) {
  checked(ctx);
  if (!t || !out) throw ValidationError("null argument");
  if (!ctx->comm) throw ValidationError("spd_tensor_repartition needs a communicator");
  if (!t->piece || (t->piece_split != 1 && t->piece_split != 2))
    throw ValidationError("spd_tensor_repartition moves a piece (spd_tensor_place / spd_tensor_upload_piece)");
  if (need_split != 1 && need_split != 2) throw ValidationError("need_split must be 1 (rows) or 2 (nonzeros)");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  spd_tensor* tm = const_cast<spd_tensor*>(t);
  const int W = ctx->world;
  auto colours = [&](int split) { return rank_spans(ctx, tm, split, placement_pieces(ctx)); };
  const std::vector<spd_range> held = colours(t->piece_split);
  const std::vector<spd_range> need = colours(need_split);
  const int me = ctx->rank;
  if (held[me].lo != t->piece_lo || (held[me].lo <= held[me].hi && held[me].hi != t->piece_hi))
    throw ValidationError("spd_tensor_repartition: the piece does not hold its split's colour");
  const spd_level_store& L = t->levels[1];
  const int64_t nrows = L.parent_positions, nnz = L.positions;
  const int64_t dims[2] = {t->dims[0], t->dims[1]};
  const int kinds[2] = {SPD_DENSE, SPD_COMPRESSED};
  const int mo[2] = {t->mode_order[0], t->mode_order[1]};
  spd_tensor* r = make_skeleton(ctx, 2, dims, kinds, mo);
  try {
    r->levels[0].kind = SPD_DENSE;
    r->levels[0].dom = {nrows};
    r->levels[0].positions = nrows;
    spd_level_store& R = r->levels[1];
    R.kind = SPD_COMPRESSED;
    R.parent_positions = nrows;
    R.positions = nnz;
    R.rowptr = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (nrows + 1));
    SPD_CUDA(cudaMemcpyAsync(R.rowptr, L.rowptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyDeviceToDevice, s));
    r->nvals = nnz;
    r->piece = true;
    r->piece_split = need_split;
    set_whole_span(r);
    const spd_range mine = need[me];
    const int64_t cnt = std::max<int64_t>(mine.hi - mine.lo + 1, 0);
    r->piece_lo = mine.lo;
    r->piece_hi = mine.hi;
    r->piece_cap = std::max<int64_t>(cnt, 1);
    r->piece_crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * r->piece_cap);
    r->piece_vals = (double*)dev_alloc(ctx, sizeof(double) * r->piece_cap);
    R.crd = r->piece_crd - mine.lo;
    r->vals = r->piece_vals - mine.lo;
    auto overlap = [](spd_range a, spd_range b) {
      return spd_range{std::max(a.lo, b.lo), std::min(a.hi, b.hi)};
    };
    int64_t received = 0;
    const spd_range local = overlap(held[me], mine);
    if (local.lo <= local.hi) {
      const int64_t c = local.hi - local.lo + 1;
      SPD_CUDA(cudaMemcpyAsync(R.crd + local.lo, L.crd + local.lo, sizeof(int64_t) * c, cudaMemcpyDeviceToDevice, s));
      SPD_CUDA(cudaMemcpyAsync(r->vals + local.lo, t->vals + local.lo, sizeof(double) * c, cudaMemcpyDeviceToDevice,
                               s));
    }
    SPD_NCCL(ncclGroupStart());
    for (int p = 0; p < W; p++) {
      if (p == me) continue;
      const spd_range snd = overlap(held[me], need[p]);  // what p needs from my piece
      if (snd.lo <= snd.hi) {
        const int64_t c = snd.hi - snd.lo + 1;
        SPD_NCCL(ncclSend(L.crd + snd.lo, c, ncclInt64, p, ctx->comm, s));
        SPD_NCCL(ncclSend(t->vals + snd.lo, c, ncclFloat64, p, ctx->comm, s));
      }
      const spd_range rcv = overlap(held[p], mine);  // what I need from p's piece
      if (rcv.lo <= rcv.hi) {
        const int64_t c = rcv.hi - rcv.lo + 1;
        SPD_NCCL(ncclRecv(R.crd + rcv.lo, c, ncclInt64, p, ctx->comm, s));
        SPD_NCCL(ncclRecv(r->vals + rcv.lo, c, ncclFloat64, p, ctx->comm, s));
        received += 16 * c;
      }
    }
    SPD_NCCL(ncclGroupEnd());
    SPD_CUDA(cudaStreamSynchronize(s));
    if (bytes_in) *bytes_in = received;
  } catch (...) {
    spd_tensor_destroy(r);
    throw;
  }
  *out = r;
}

// The reference's communication ledger for one CSR-like tensor
// (transfer_bytes sim.cpp:134-147 over worker_needed_sets :505-516 and
// residency_from_placements :547-566; units sim.hpp:21-23): worker w needs
// colour w of the compute partition (need_split 1 rows / 2 nonzeros -- the
// communicate site of a distributed loop, which the planner places there by
// default) and holds colour w of its placement
// (held_split 1 rows / 2 nonzeros; 3 = replicated).  Per level-1 region the
// sets are contiguous spans: crd / vals = q; pos = every row of `par` for a
// row split (partition_from_parent copies the row block) or only its
// non-empty rows for a nonzero split (preimage, deppart.cpp:46).
struct PosSet {
  int64_t lo = 0, hi = -1;
  bool nonempty_only = false;
};

void run_ledger(spd_context* ctx, const spd_tensor* t, int need_split, int held_split, int64_t pieces,
                int64_t* bytes_out) {
  checked(ctx);
  if (!t || !bytes_out) throw ValidationError("null argument");
  if (t->levels.size() != 2 || t->levels[0].kind != SPD_DENSE || t->levels[1].kind != SPD_COMPRESSED)
    throw ValidationError("unsupported on gpu: the ledger covers ds (CSR-like) tensors");
  if (need_split < 1 || need_split > 2) throw ValidationError("need_split must be 1 or 2");
  if (held_split < 1 || held_split > 3) throw ValidationError("held_split must be 1, 2 or 3");
  if (pieces < 1) throw ValidationError("pieces must be positive");
  activate(ctx);
  spd_tensor* tm = const_cast<spd_tensor*>(t);
  const int64_t n = t->levels[1].parent_positions, nnz = t->levels[1].positions;
  auto colours = [&](int split) {
    const int rc = split == 1 ? spd_partition_universe(ctx, tm, pieces, nullptr)
                              : spd_partition_nonzero(ctx, tm, 1, pieces, nullptr);
    if (rc != SPD_OK) throw ValidationError(spd_last_error());
    return host_colors(ctx);
  };
  std::vector<spd_color> held, need;
  if (held_split != 3) held = colours(held_split);
  need = colours(need_split);  // leaves the compute partition on ctx
  auto pos_of = [&](const std::vector<spd_color>& cs, int split, int64_t w) {
    PosSet p;
    if (cs.empty()) {  // full / replicated: every pos entry
      p.lo = 0, p.hi = n - 1;
      return p;
    }
    const spd_color& c = cs[w];
    if (split == 1) {
      p.lo = c.par.lo, p.hi = c.par.hi;
    } else if (c.q.lo <= c.q.hi) {
      p.lo = c.par.lo, p.hi = c.par.hi, p.nonempty_only = true;
    }
    return p;
  };
  auto crd_of = [&](const std::vector<spd_color>& cs, int64_t w) {
    return cs.empty() ? spd_range{0, nnz - 1} : cs[w].q;
  };
  // spans whose non-empty rows are counted on the device: per worker
  // |needed pos| and |needed pos & held pos|
  std::vector<int64_t> spans;
  std::vector<int64_t> need_all(pieces), both_all(pieces);
  for (int64_t w = 0; w < pieces; w++) {
    const PosSet N = pos_of(need, need_split, w), H = pos_of(held, held_split, w);
    const int64_t lo = std::max(N.lo, H.lo), hi = std::min(N.hi, H.hi);
    need_all[w] = N.nonempty_only ? -1 : std::max<int64_t>(N.hi - N.lo + 1, 0);
    both_all[w] = (N.nonempty_only || H.nonempty_only) ? -1 : std::max<int64_t>(hi - lo + 1, 0);
    spans.insert(spans.end(), {N.lo, N.hi, lo, hi});
  }
  const std::vector<int64_t> ne = nonempty_in_spans(ctx, tm, t->levels[1].rowptr, n, spans);
  for (int64_t w = 0; w < pieces; w++) {
    const int64_t npos = need_all[w] >= 0 ? need_all[w] : ne[2 * w];
    const int64_t both = both_all[w] >= 0 ? both_all[w] : ne[2 * w + 1];
    const spd_range nc = crd_of(need, w), hc = crd_of(held, w);
    const int64_t ncount = std::max<int64_t>(nc.hi - nc.lo + 1, 0);
    const int64_t ov = std::max<int64_t>(std::min(nc.hi, hc.hi) - std::max(nc.lo, hc.lo) + 1, 0);
    const int64_t missing_pos = npos - both, missing_crd = ncount - ov;
    bytes_out[w] = 16 * missing_pos + 8 * missing_crd + 8 * missing_crd;  // pos ranges, crd, vals
  }
}

// missing_count (sim.cpp:76-84) for many (needed, held) pairs of sorted,
// duplicate-free index sets at once: one thread per needed entry, a binary
// search in its pair's held set, warp-aggregated counts per pair.
__global__ void k_missing(const int64_t* __restrict__ need, const int64_t* __restrict__ need_off,
                          const int64_t* __restrict__ held, const int64_t* __restrict__ held_off,
                          const int32_t* __restrict__ pair_of, int64_t total,
                          unsigned long long* __restrict__ missing) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = pair_of[i];
    const int64_t v = need[i];
    int64_t lo = held_off[p], hi = held_off[p + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (held[mid] < v) lo = mid + 1; else hi = mid;
    }
    const bool miss = lo == held_off[p + 1] || held[lo] != v;
    if (miss) atomicAdd(missing + p, 1ull);
  }
}

__global__ void k_pair_of(const int64_t* __restrict__ need_off, int64_t npairs, int32_t* __restrict__ pair_of) {
  for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x)
    for (int64_t i = need_off[p] + threadIdx.x; i < need_off[p + 1]; i += blockDim.x) pair_of[i] = (int32_t)p;
}

void run_ledger_missing(spd_context* ctx, int64_t npairs, const int64_t* const* needed, const int64_t* n_needed,
                        const int64_t* const* held, const int64_t* n_held, int64_t* missing) {
  checked(ctx);
  if (npairs < 0) throw ValidationError("npairs must be non-negative");
  if (npairs == 0) return;
  if (!needed || !n_needed || !held || !n_held || !missing) throw ValidationError("null argument");
  if (npairs >= (int64_t(1) << 31)) throw ValidationError("too many set pairs");
  activate(ctx);
  cudaStream_t s = ctx->stream;
  std::vector<int64_t> noff(npairs + 1, 0), hoff(npairs + 1, 0);
  for (int64_t p = 0; p < npairs; p++) {
    if (n_needed[p] < 0 || n_held[p] < 0) throw ValidationError("negative set size");
    if ((n_needed[p] > 0 && !needed[p]) || (n_held[p] > 0 && !held[p])) throw ValidationError("null set");
    noff[p + 1] = noff[p] + n_needed[p];
    hoff[p + 1] = hoff[p] + n_held[p];
  }
  const int64_t tn = noff[npairs], th = hoff[npairs];
  const size_t bytes = sizeof(int64_t) * (tn + th + 2 * (npairs + 1)) + sizeof(int32_t) * (tn + 1) +
                       sizeof(unsigned long long) * npairs + 64;
  char* buf = (char*)dev_alloc(ctx, bytes);
  int64_t* d_need = (int64_t*)buf;
  int64_t* d_held = d_need + tn;
  int64_t* d_noff = d_held + th;
  int64_t* d_hoff = d_noff + npairs + 1;
  unsigned long long* d_miss = (unsigned long long*)(d_hoff + npairs + 1);
  int32_t* d_pair = (int32_t*)(d_miss + npairs);
  for (int64_t p = 0; p < npairs; p++) {
    if (n_needed[p] > 0)
      SPD_CUDA(cudaMemcpyAsync(d_need + noff[p], needed[p], sizeof(int64_t) * n_needed[p], cudaMemcpyHostToDevice, s));
    if (n_held[p] > 0)
      SPD_CUDA(cudaMemcpyAsync(d_held + hoff[p], held[p], sizeof(int64_t) * n_held[p], cudaMemcpyHostToDevice, s));
  }
  SPD_CUDA(cudaMemcpyAsync(d_noff, noff.data(), sizeof(int64_t) * (npairs + 1), cudaMemcpyHostToDevice, s));
  SPD_CUDA(cudaMemcpyAsync(d_hoff, hoff.data(), sizeof(int64_t) * (npairs + 1), cudaMemcpyHostToDevice, s));
  SPD_CUDA(cudaMemsetAsync(d_miss, 0, sizeof(unsigned long long) * npairs, s));
  if (tn > 0) {
    k_pair_of<<<(unsigned)std::min<int64_t>(npairs, 65535), 256, 0, s>>>(d_noff, npairs, d_pair);
    SPD_CHECK_LAUNCH();
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(tn, 256), (int64_t)ctx->num_sms * 16);
    k_missing<<<grid, 256, 0, s>>>(d_need, d_noff, d_held, d_hoff, d_pair, tn, d_miss);
    SPD_CHECK_LAUNCH();
    ctx->launches += 2;
  }
  std::vector<unsigned long long> out(npairs);
  SPD_CUDA(cudaMemcpyAsync(out.data(), d_miss, sizeof(unsigned long long) * npairs, cudaMemcpyDeviceToHost, s));
  SPD_CUDA(cudaStreamSynchronize(s));
  dev_free(ctx, buf);
  for (int64_t p = 0; p < npairs; p++) missing[p] = (int64_t)out[p];
}

}  // namespace

}  // namespace spd

using namespace spd;

extern "C" int spd_tensor_repartition(spd_context* ctx, const spd_tensor* piece, int need_split,
                                      spd_tensor** out, int64_t* bytes_in) {
  return guarded([&] { run_repartition(ctx, piece, need_split, out, bytes_in); });
}

extern "C" int spd_ledger_bytes(spd_context* ctx, const spd_tensor* t, int need_split, int held_split,
                                int64_t pieces, int64_t* bytes_out) {
  return guarded([&] { run_ledger(ctx, t, need_split, held_split, pieces, bytes_out); });
}

extern "C" int spd_ledger_missing(spd_context* ctx, int64_t npairs, const int64_t* const* needed,
                                  const int64_t* n_needed, const int64_t* const* held, const int64_t* n_held,
                                  int64_t* missing) {
  return guarded([&] { run_ledger_missing(ctx, npairs, needed, n_needed, held, n_held, missing); });
}

extern "C" int spd_tensor_place(spd_context* ctx, int root, const spd_tensor* whole, int split,
                                spd_tensor** piece, int64_t* bytes_in) {
  return guarded([&] { run_place(ctx, root, whole, split, piece, bytes_in); });
}

extern "C" int spd_tensor_piece_span(const spd_tensor* t, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    if (!t) throw ValidationError("null spd_tensor");
    *lo = t->piece ? t->piece_lo : 0;
    *hi = t->piece ? t->piece_hi : t->nvals - 1;
  });
}
