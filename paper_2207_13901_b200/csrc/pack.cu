// Device-side tensor construction: SparseTensor::pack
// (/root/reference/proj/core/src/tensor.cpp:94-182) from COO entries.
//
// Reference semantics reproduced exactly:
//   * coordinates are checked against the dimensions (ValidationError
//     "pack: coordinate out of bounds");
//   * entries are keyed in storage order (coords[mode_order[k]]), duplicates
//     summed as std::map's `dedup[key] += value` does -- from 0.0, in input
//     order -- and kept even when the sum is zero (explicit zeros);
//   * levels are built top-down: a dense group linearises its coordinates
//     into the running position, a compressed level gives every distinct
//     (parent position, coordinate) pair a new position in sorted order;
//   * vals has one slot per leaf position, 0.0 where no entry lands (dense
//     trailing levels).
//
// B200 design: one stable LSD radix sort of (bit-packed storage key, input
// index) pairs with cub -- one pass over the packed key when the level
// coordinates fit 64 bits together, else one stable pass per coordinate from
// the last storage level to the first -- then segment heads, an ordered
// per-segment sum (one thread per distinct key: the reference's summation
// order, not a tree), and per level an element-parallel flag / scan / count.
// Everything stays in HBM; the host only reads back three scalars.
#include <cub/cub.cuh>

#include "common.cuh"

namespace spd {

namespace {

int bits_for(int64_t extent) {
  int b = 0;
  while (b < 63 && (int64_t(1) << b) < extent) b++;
  return b;
}

__global__ void k_pack_check(const int64_t* __restrict__ c, int64_t n, int64_t dim, int* __restrict__ err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    if (c[e] < 0 || c[e] >= dim) atomicOr(err, 1);
}

// key |= c << shift (bit-packed storage key), idx = e.
__global__ void k_pack_key(const int64_t* __restrict__ c, int64_t n, int shift, int first,
                           uint64_t* __restrict__ key, int64_t* __restrict__ idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = (uint64_t)c[e] << shift;
    key[e] = first ? v : (key[e] | v);
    if (first) idx[e] = e;
  }
}

// LSD fallback: key = coordinate of the permuted entries.
__global__ void k_pack_gather_key(const int64_t* __restrict__ c, const int64_t* __restrict__ idx, int64_t n,
                                  uint64_t* __restrict__ key) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    key[e] = (uint64_t)c[idx[e]];
}

__global__ void k_iota(int64_t* __restrict__ a, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    a[e] = e;
}

struct Coords {
  const int64_t* c[8];  // storage-order coordinate arrays (input order)
  int order;
};

// Head of a run of equal storage keys (sorted entries e-1, e).
__global__ void k_pack_heads(Coords cs, const int64_t* __restrict__ idx, int64_t n,
                             unsigned char* __restrict__ head) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    bool h = e == 0;
    if (!h) {
      const int64_t a = idx[e - 1], b = idx[e];
      for (int k = 0; k < cs.order && !h; k++) h = cs.c[k][a] != cs.c[k][b];
    }
    head[e] = h;
  }
}

// One distinct key per thread: its value summed in input order from 0.0
// (the stable sort kept duplicates in input order), and its storage
// coordinates.
__global__ void k_pack_reduce(Coords cs, const double* __restrict__ vals, const int64_t* __restrict__ idx,
                              const int64_t* __restrict__ seg, int64_t u_count, int64_t n,
                              double* __restrict__ uval, int64_t* __restrict__ ucoord) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u_count;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = seg[u], e = u + 1 < u_count ? seg[u + 1] : n;
    double v = 0.0;
    for (int64_t q = s; q < e; q++) v += vals[idx[q]];
    uval[u] = v;
    const int64_t first = idx[s];
    for (int k = 0; k < cs.order; k++) ucoord[k * u_count + u] = cs.c[k][first];
  }
}

// Dense level group: pos = pos * total + linearize(coords of the group).
__global__ void k_pack_dense(int64_t* __restrict__ pos, const int64_t* __restrict__ ucoord, int64_t u_count,
                             int base, int ng, int64_t e0, int64_t e1, int64_t e2, int64_t total) {
  const int64_t ext[3] = {e0, e1, e2};
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u_count;
       u += (int64_t)gridDim.x * blockDim.x) {
    int64_t local = 0;
    for (int j = 0; j < ng; j++) local = local * ext[j] + ucoord[(base + j) * u_count + u];
    pos[u] = pos[u] * total + local;
  }
}

// Compressed level: a new position per distinct (parent, coordinate).
__global__ void k_pack_cflags(const int64_t* __restrict__ pos, const int64_t* __restrict__ coord,
                              int64_t u_count, int64_t* __restrict__ flag) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u_count;
       u += (int64_t)gridDim.x * blockDim.x)
    flag[u] = (u == 0 || pos[u] != pos[u - 1] || coord[u] != coord[u - 1]) ? 1 : 0;
}

// incl = inclusive scan of the flags: new position = incl - 1; the first
// entry of every new position writes its crd and counts it for its parent.
__global__ void k_pack_cfill(int64_t* __restrict__ pos, const int64_t* __restrict__ coord,
                             const int64_t* __restrict__ flag, const int64_t* __restrict__ incl,
                             int64_t u_count, int64_t* __restrict__ crd, unsigned long long* __restrict__ cnt) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u_count;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = incl[u] - 1;
    if (flag[u]) {
      crd[q] = coord[u];
      atomicAdd(cnt + pos[u], 1ull);
    }
    pos[u] = q;
  }
}

__global__ void k_pack_vals(const int64_t* __restrict__ pos, const double* __restrict__ uval, int64_t u_count,
                            double* __restrict__ vals) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u_count;
       u += (int64_t)gridDim.x * blockDim.x)
    vals[pos[u]] = uval[u];
}

int grid_of(spd_context* ctx, int64_t n) {
  int64_t g = ceil_div(std::max<int64_t>(n, 1), 256);
  return (int)std::min<int64_t>(g, (int64_t)ctx->num_sms * 16);
}

// RAII over stream-ordered temporaries.
struct Temps {
  spd_context* ctx;
  std::vector<void*> ptrs;
  explicit Temps(spd_context* c) : ctx(c) {}
  template <class T>
  T* get(int64_t count) {
    T* p = (T*)dev_alloc(ctx, sizeof(T) * (size_t)std::max<int64_t>(count, 1));
    ptrs.push_back(p);
    return p;
  }
  ~Temps() {
    for (void* p : ptrs) dev_free(ctx, p);
  }
};

void run_pack(spd_context* ctx, int order, const int64_t* dims, const int* kinds, const int* mode_order,
              int64_t n, const int64_t* const* coords, const double* values, int on_device,
              spd_tensor** out) {
  checked(ctx);
  if (!out) throw ValidationError("null output handle");
  if (n < 0) throw ValidationError("pack: negative entry count");
  if (order > 8) throw ValidationError("unsupported on gpu: pack supports tensors of order <= 8");
  activate(ctx);
  spd_tensor* t = make_skeleton(ctx, order, dims, kinds, mode_order);
  cudaStream_t s = ctx->stream;
  try {
    Temps tmp(ctx);
    // storage-order coordinates (and values) on the device
    Coords cs{};
    cs.order = order;
    for (int k = 0; k < order; k++) {
      const int64_t* src = coords ? coords[mode_order[k]] : nullptr;
      if (n > 0 && !src) throw ValidationError("pack: missing coordinate array");
      if (on_device) {
        cs.c[k] = src;
      } else {
        int64_t* d = tmp.get<int64_t>(n);
        if (n > 0) SPD_CUDA(cudaMemcpyAsync(d, src, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
        cs.c[k] = d;
      }
    }
    if (n > 0 && !values) throw ValidationError("pack: missing values");
    const double* vals = values;
    if (!on_device) {
      double* d = tmp.get<double>(n);
      if (n > 0) SPD_CUDA(cudaMemcpyAsync(d, values, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      vals = d;
    }
    int* err = tmp.get<int>(1);
    SPD_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
    const int g = grid_of(ctx, n);
    for (int k = 0; k < order && n > 0; k++) {
      k_pack_check<<<g, 256, 0, s>>>(cs.c[k], n, dims[mode_order[k]], err);
      SPD_CHECK_LAUNCH();
    }
    // stable sort of the entries by storage key
    int64_t* idx = tmp.get<int64_t>(n);
    int total_bits = 0;
    for (int k = 0; k < order; k++) total_bits += bits_for(dims[mode_order[k]]);
    if (n > 0) {
      uint64_t* key = tmp.get<uint64_t>(n);
      uint64_t* key2 = tmp.get<uint64_t>(n);
      int64_t* idx2 = tmp.get<int64_t>(n);
      size_t bytes = 0;
      if (total_bits <= 64) {
        int shift = total_bits;
        for (int k = 0; k < order; k++) {
          shift -= bits_for(dims[mode_order[k]]);
          k_pack_key<<<g, 256, 0, s>>>(cs.c[k], n, shift, k == 0, key, idx);
          SPD_CHECK_LAUNCH();
        }
        if (order == 0) k_iota<<<g, 256, 0, s>>>(idx, n);
        if (total_bits > 0) {
          SPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key2, idx, idx2, n, 0, total_bits, s));
          void* w = tmp.get<char>((int64_t)bytes);
          SPD_CUDA(cub::DeviceRadixSort::SortPairs(w, bytes, key, key2, idx, idx2, n, 0, total_bits, s));
          SPD_CUDA(cudaMemcpyAsync(idx, idx2, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, s));
        }
      } else {  // one stable pass per storage coordinate, least significant first
        k_iota<<<g, 256, 0, s>>>(idx, n);
        SPD_CHECK_LAUNCH();
        for (int k = order - 1; k >= 0; k--) {
          const int b = bits_for(dims[mode_order[k]]);
          if (b == 0) continue;
          k_pack_gather_key<<<g, 256, 0, s>>>(cs.c[k], idx, n, key);
          SPD_CHECK_LAUNCH();
          SPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key2, idx, idx2, n, 0, b, s));
          void* w = tmp.get<char>((int64_t)bytes);
          SPD_CUDA(cub::DeviceRadixSort::SortPairs(w, bytes, key, key2, idx, idx2, n, 0, b, s));
          SPD_CUDA(cudaMemcpyAsync(idx, idx2, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, s));
        }
      }
    }
    // distinct keys
    unsigned char* head = tmp.get<unsigned char>(n);
    int64_t* seg = tmp.get<int64_t>(n);
    int64_t* nsel = tmp.get<int64_t>(1);
    SPD_CUDA(cudaMemsetAsync(nsel, 0, sizeof(int64_t), s));
    if (n > 0) {
      k_pack_heads<<<g, 256, 0, s>>>(cs, idx, n, head);
      SPD_CHECK_LAUNCH();
      int64_t* iota = tmp.get<int64_t>(n);
      k_iota<<<g, 256, 0, s>>>(iota, n);
      SPD_CHECK_LAUNCH();
      size_t bytes = 0;
      SPD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, iota, head, seg, nsel, n, s));
      void* w = tmp.get<char>((int64_t)bytes);
      SPD_CUDA(cub::DeviceSelect::Flagged(w, bytes, iota, head, seg, nsel, n, s));
    }
    int64_t host2[2] = {0, 0};
    SPD_CUDA(cudaMemcpyAsync(&host2[0], nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaMemcpyAsync(&host2[1], err, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    if ((int)host2[1]) throw ValidationError("pack: coordinate out of bounds");
    const int64_t U = host2[0];
    const int gu = grid_of(ctx, U);
    double* uval = tmp.get<double>(U);
    int64_t* ucoord = tmp.get<int64_t>(U * std::max(order, 1));
    if (U > 0) {
      k_pack_reduce<<<gu, 256, 0, s>>>(cs, vals, idx, seg, U, n, uval, ucoord);
      SPD_CHECK_LAUNCH();
    }
    // levels, top-down (tensor.cpp:129-174)
    int64_t* pos = tmp.get<int64_t>(U);
    SPD_CUDA(cudaMemsetAsync(pos, 0, sizeof(int64_t) * std::max<int64_t>(U, 1), s));
    int64_t* flag = tmp.get<int64_t>(U);
    int64_t* incl = tmp.get<int64_t>(U);
    int64_t parent = 1;
    int base = 0;
    for (size_t l = 0; l < t->groups.size(); l++) {
      spd_level_store& L = t->levels[l];
      const auto& grp = t->groups[l];
      L.parent_positions = parent;
      if (kinds[grp[0]] == SPD_DENSE) {
        L.kind = SPD_DENSE;
        int64_t ext[3] = {1, 1, 1}, total = 1;
        if (grp.size() > 3) throw ValidationError("unsupported on gpu: more than 3 collapsed dense modes");
        for (size_t j = 0; j < grp.size(); j++) {
          ext[j] = dims[mode_order[grp[j]]];
          L.dom.push_back(ext[j]);
          total *= ext[j];
        }
        if (U > 0) {
          k_pack_dense<<<gu, 256, 0, s>>>(pos, ucoord, U, base, (int)grp.size(), ext[0], ext[1], ext[2], total);
          SPD_CHECK_LAUNCH();
        }
        parent *= total;
        L.positions = parent;
      } else {
        L.kind = SPD_COMPRESSED;
        int64_t nl = 0;
        unsigned long long* cnt = (unsigned long long*)tmp.get<int64_t>(parent + 1);
        SPD_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (parent + 1), s));
        if (U > 0) {
          const int64_t* coord = ucoord + (int64_t)base * U;
          k_pack_cflags<<<gu, 256, 0, s>>>(pos, coord, U, flag);
          SPD_CHECK_LAUNCH();
          size_t bytes = 0;
          SPD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, flag, incl, U, s));
          void* w = tmp.get<char>((int64_t)bytes);
          SPD_CUDA(cub::DeviceScan::InclusiveSum(w, bytes, flag, incl, U, s));
          SPD_CUDA(cudaMemcpyAsync(&nl, incl + U - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
          SPD_CUDA(cudaStreamSynchronize(s));
          L.crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * std::max<int64_t>(nl, 1));
          k_pack_cfill<<<gu, 256, 0, s>>>(pos, coord, flag, incl, U, L.crd, cnt);
          SPD_CHECK_LAUNCH();
        } else {
          L.crd = (int64_t*)dev_alloc(ctx, sizeof(int64_t));
        }
        // counts per parent -> row pointer (exclusive scan over parent + 1)
        size_t bytes = 0;
        int64_t* rp = (int64_t*)dev_alloc(ctx, sizeof(int64_t) * (parent + 1));
        L.rowptr = rp;
        SPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t*)cnt, rp, parent + 1, s));
        void* w = tmp.get<char>((int64_t)bytes);
        SPD_CUDA(cub::DeviceScan::ExclusiveSum(w, bytes, (int64_t*)cnt, rp, parent + 1, s));
        L.rowptr = rp;
        L.positions = nl;
        parent = nl;
      }
      base += (int)grp.size();
    }
    t->nvals = parent;
    t->vals = (double*)dev_alloc(ctx, sizeof(double) * std::max<int64_t>(parent, 1));
    SPD_CUDA(cudaMemsetAsync(t->vals, 0, sizeof(double) * std::max<int64_t>(parent, 1), s));
    if (U > 0) {
      k_pack_vals<<<gu, 256, 0, s>>>(pos, uval, U, t->vals);
      SPD_CHECK_LAUNCH();
    }
    t->owns = true;
    set_whole_span(t);
    ctx->launches += 8;
    SPD_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    spd_tensor_destroy(t);
    throw;
  }
  *out = t;
}

}  // namespace

}  // namespace spd

using namespace spd;

extern "C" int spd_tensor_pack(spd_context* ctx, int order, const int64_t* dims, const int* kinds,
                               const int* mode_order, int64_t nentries, const int64_t* const* coords,
                               const double* values, int on_device, spd_tensor** out) {
  return guarded([&] { run_pack(ctx, order, dims, kinds, mode_order, nentries, coords, values, on_device, out); });
}
