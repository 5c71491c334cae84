// Tensor loaders feeding the device: load_tensor /
// read_tensor (/root/reference/proj/core/src/tensor_io.cpp:51-142) for
// .tns and MatrixMarket files, and write_tensor (:145-155).
//
// Reference behaviour kept: MatrixMarket when the first line starts with
// "%%MatrixMarket" (only "matrix coordinate real general"), else .tns;
// coordinates are 1-indexed on disk; blank lines and comment lines ('%', and
// '#' in .tns) are skipped; a line needs exactly `order` integers and one
// value ("malformed line N" / "trailing fields on line N"); .tns dimensions
// are the declared ones or the per-mode maximum; coordinates outside them,
// a MatrixMarket entry count or size line that disagrees, or an unreadable
// file are ParseErrors (SPD_ERR_VALIDATION, the CLI's exit 2).
//
// B200 design: the file is read once, split at line boundaries into one
// chunk per host thread, parsed in parallel straight into pinned staging
// buffers (offsets from a per-chunk entry count), then handed to the
// device-side pack (pack.cu) -- the H2D copy runs from pinned memory and
// sorting / deduplication / level construction happen on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace spd {

namespace {

struct ParseError : ValidationError {
  explicit ParseError(const std::string& m) : ValidationError(m) {}
};

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

bool blank(const char* b, const char* e) {
  for (; b < e; b++)
    if (!is_space(*b)) return false;
  return true;
}

// One token [b, e) of a line; returns false at end of line.
bool token(const char*& p, const char* e, const char*& tb, const char*& te) {
  while (p < e && is_space(*p)) p++;
  if (p >= e) return false;
  tb = p;
  while (p < e && !is_space(*p)) p++;
  te = p;
  return true;
}

bool parse_i64(const char* b, const char* e, int64_t* out) {
  char buf[32];
  const size_t n = (size_t)(e - b);
  if (n == 0 || n >= sizeof buf) return false;
  std::memcpy(buf, b, n);
  buf[n] = 0;
  char* end = nullptr;
  errno = 0;
  long long v = std::strtoll(buf, &end, 10);
  if (errno || *end) return false;
  *out = v;
  return true;
}

bool parse_f64(const char* b, const char* e, double* out) {
  char buf[64];
  const size_t n = (size_t)(e - b);
  if (n == 0 || n >= sizeof buf) return false;
  std::memcpy(buf, b, n);
  buf[n] = 0;
  char* end = nullptr;
  double v = std::strtod(buf, &end);
  if (*end) return false;
  *out = v;
  return true;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t first_line;  // 1-based number of the chunk's first line
  std::vector<int64_t> coords;  // entries x order
  std::vector<double> vals;
  std::string error;
  int64_t error_line = -1;
};

// Parses the entry lines of one chunk (tensor_io.cpp:21-38, 88-91, 100-105).
void parse_chunk(Chunk& c, int order, bool tns, const std::string& name) {
  int64_t line_no = c.first_line;
  const char* p = c.b;
  while (p < c.e) {
    const char* le = (const char*)std::memchr(p, '\n', (size_t)(c.e - p));
    if (!le) le = c.e;
    if (!blank(p, le) && !(*p == '%') && !(tns && *p == '#')) {
      const char* q = p;
      const char *tb, *te;
      for (int k = 0; k < order; k++) {
        int64_t v;
        if (!token(q, le, tb, te) || !parse_i64(tb, te, &v)) {
          c.error = name + ": malformed line " + std::to_string(line_no);
          c.error_line = line_no;
          return;
        }
        c.coords.push_back(v - 1);  // 1-indexed on disk
      }
      double v;
      if (!token(q, le, tb, te) || !parse_f64(tb, te, &v)) {
        c.error = name + ": malformed line " + std::to_string(line_no);
        c.error_line = line_no;
        return;
      }
      if (token(q, le, tb, te)) {
        c.error = name + ": trailing fields on line " + std::to_string(line_no);
        c.error_line = line_no;
        return;
      }
      c.vals.push_back(v);
    }
    p = le + 1;
    line_no++;
  }
}

struct Pinned {
  void* p = nullptr;
  explicit Pinned(size_t bytes) { SPD_CUDA(cudaMallocHost(&p, std::max<size_t>(bytes, 8))); }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

void run_load(spd_context* ctx, const char* path, int order, const int* kinds, const int* mode_order,
              const int64_t* dims, spd_tensor** out, int64_t* dims_out) {
  checked(ctx);
  if (!path || !out) throw ValidationError("null argument");
  if (order < 1 || order > 8) throw ValidationError("load: tensor order must be in [1, 8]");
  const std::string name(path);
  FILE* f = std::fopen(path, "rb");
  if (!f) throw ParseError("cannot open tensor file '" + name + "'");
  std::vector<char> buf;
  {
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize((size_t)std::max(sz, 0L));
    const size_t got = sz > 0 ? std::fread(buf.data(), 1, (size_t)sz, f) : 0;
    std::fclose(f);
    if ((long)got != sz) throw ParseError("cannot open tensor file '" + name + "'");
  }
  const char* b = buf.data();
  const char* e = b + buf.size();
  bool tns = true;
  int64_t line0 = 1;
  std::vector<int64_t> sizes;
  int64_t mm_nnz = -1;
  if (e - b >= 14 && std::memcmp(b, "%%MatrixMarket", 14) == 0) {  // tensor_io.cpp:125-133
    tns = false;
    const char* le = (const char*)std::memchr(b, '\n', (size_t)(e - b));
    if (!le) le = e;
    const std::string banner(b, le);
    char t1[64] = {0}, t2[64] = {0}, t3[64] = {0}, t4[64] = {0}, t5[64] = {0};
    std::sscanf(banner.c_str(), "%63s %63s %63s %63s %63s", t1, t2, t3, t4, t5);
    if (std::strcmp(t2, "matrix") || std::strcmp(t3, "coordinate") || std::strcmp(t4, "real") ||
        std::strcmp(t5, "general"))
      throw ParseError(name + ": unsupported MatrixMarket header '" + banner + "'");
    if (order != 2) throw ValidationError("load: a MatrixMarket file holds a matrix (order 2)");
    b = le < e ? le + 1 : e;
    line0 = 2;
    // comments / blank lines up to the size line (tensor_io.cpp:65-72)
    int64_t rows = 0, cols = 0;
    bool have = false;
    while (b < e) {
      le = (const char*)std::memchr(b, '\n', (size_t)(e - b));
      if (!le) le = e;
      const bool skip = (b < le && *b == '%') || blank(b, le);
      const char* line_b = b;
      b = le < e ? le + 1 : e;
      line0++;
      if (skip) continue;
      const std::string line(line_b, le);
      long long r = 0, c = 0, z = 0;
      if (std::sscanf(line.c_str(), "%lld %lld %lld", &r, &c, &z) != 3)
        throw ParseError(name + ": malformed MatrixMarket size line");
      rows = r, cols = c, mm_nnz = z;
      have = true;
      break;
    }
    if (!have) throw ParseError(name + ": malformed MatrixMarket size line");
    if (dims && (dims[0] != rows || dims[1] != cols))
      throw ParseError(name + ": declared dims disagree with MatrixMarket header");
    sizes = {rows, cols};
  } else if (dims) {
    sizes.assign(dims, dims + order);
  }
  // split at line boundaries, one chunk per host thread
  const int T = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 64));
  std::vector<Chunk> chunks;
  const size_t len = (size_t)(e - b);
  const char* cur = b;
  for (int t = 0; t < T && cur < e; t++) {
    const char* stop = t == T - 1 ? e : b + len * (t + 1) / T;
    if (stop < cur) stop = cur;
    if (stop < e) {
      const char* nl = (const char*)std::memchr(stop, '\n', (size_t)(e - stop));
      stop = nl ? nl + 1 : e;
    }
    chunks.push_back(Chunk{cur, stop, 0, {}, {}, {}, -1});
    cur = stop;
  }
  // line numbers of the chunk starts
  {
    std::vector<int64_t> nls(chunks.size(), 0);
    std::vector<std::thread> th;
    for (size_t i = 0; i < chunks.size(); i++)
      th.emplace_back([&, i] { nls[i] = std::count(chunks[i].b, chunks[i].e, '\n'); });
    for (auto& x : th) x.join();
    int64_t ln = line0;
    for (size_t i = 0; i < chunks.size(); i++) chunks[i].first_line = ln, ln += nls[i];
  }
  {
    std::vector<std::thread> th;
    for (auto& c : chunks) th.emplace_back([&] { parse_chunk(c, order, tns, name); });
    for (auto& x : th) x.join();
  }
  int64_t n = 0;
  for (auto& c : chunks) {
    if (!c.error.empty()) throw ParseError(c.error);  // the first bad line in file order
    n += (int64_t)c.vals.size();
  }
  if (!tns && n != mm_nnz) throw ParseError(name + ": entry count does not match header");
  // pinned staging, one array per mode (SoA), then the device-side pack
  Pinned pc(sizeof(int64_t) * (size_t)n * order), pv(sizeof(double) * (size_t)n);
  int64_t* coords = (int64_t*)pc.p;
  double* vals = (double*)pv.p;
  {
    std::vector<int64_t> off(chunks.size() + 1, 0);
    for (size_t i = 0; i < chunks.size(); i++) off[i + 1] = off[i] + (int64_t)chunks[i].vals.size();
    std::vector<int64_t> maxc((size_t)order * chunks.size(), 0);
    std::vector<std::thread> th;
    for (size_t i = 0; i < chunks.size(); i++)
      th.emplace_back([&, i] {
        const Chunk& c = chunks[i];
        const int64_t m = (int64_t)c.vals.size();
        for (int64_t q = 0; q < m; q++) {
          for (int k = 0; k < order; k++) {
            const int64_t v = c.coords[q * order + k];
            coords[(int64_t)k * n + off[i] + q] = v;
            maxc[i * order + k] = std::max(maxc[i * order + k], v + 1);
          }
          vals[off[i] + q] = c.vals[q];
        }
      });
    for (auto& x : th) x.join();
    if (sizes.empty()) {  // tns without declared dims: per-mode maximum (tensor_io.cpp:108-111)
      sizes.assign(order, 0);
      for (size_t i = 0; i < chunks.size(); i++)
        for (int k = 0; k < order; k++) sizes[k] = std::max(sizes[k], maxc[i * order + k]);
    }
  }
  if ((int)sizes.size() != order) throw ParseError(name + ": declared dims do not match format order");
  // pack_checked (tensor_io.cpp:40-49): bounds are a ParseError here
  for (int k = 0; k < order; k++) {
    const int64_t* c = coords + (int64_t)k * n;
    for (int64_t q = 0; q < n; q++)
      if (c[q] < 0 || c[q] >= sizes[k]) throw ParseError(name + ": coordinate out of declared bounds");
  }
  std::vector<const int64_t*> cp(order);
  for (int k = 0; k < order; k++) cp[k] = coords + (int64_t)k * n;
  const int rc = spd_tensor_pack(ctx, order, sizes.data(), kinds, mode_order, n, cp.data(), vals, 0, out);
  if (rc != SPD_OK) throw ValidationError(spd_last_error());
  if (dims_out)
    for (int k = 0; k < order; k++) dims_out[k] = sizes[k];
}

// write_tensor (tensor_io.cpp:145-155): the stored entries sorted by logical
// coordinates, 1-indexed, value printed with %.17g.
void run_store(const spd_tensor* t, const char* path) {
  if (!t || !path) throw ValidationError("null argument");
  spd_context* ctx = t->ctx;
  activate(ctx);
  const int order = t->order;
  const int nl = (int)t->levels.size();
  // every leaf position's storage coordinates, walking the levels down
  std::vector<std::vector<int64_t>> coord(order);
  std::vector<int64_t> parent(1, 0);  // level positions of the current level
  int base = 0;
  for (int l = 0; l < nl; l++) {
    const spd_level_store& L = t->levels[l];
    const auto& grp = t->groups[l];
    std::vector<int64_t> next;
    std::vector<std::vector<int64_t>> ncoord(order);
    if (L.kind == SPD_DENSE) {
      int64_t total = 1;
      for (int64_t x : L.dom) total *= x;
      const int ng = (int)grp.size();
      std::vector<int64_t> local(ng);
      for (size_t q = 0; q < parent.size(); q++)
        for (int64_t j = 0; j < total; j++) {
          next.push_back(parent[q] * total + j);
          for (int k = 0; k < base; k++) ncoord[k].push_back(coord[k][q]);
          int64_t rem = j;  // delinearize, last mode fastest (IndexSpace)
          for (int g = ng - 1; g >= 0; g--) local[g] = rem % L.dom[g], rem /= L.dom[g];
          for (int g = 0; g < ng; g++) ncoord[base + g].push_back(local[g]);
        }
    } else {
      std::vector<int64_t> rp(L.parent_positions + 1), crd(L.positions);
      SPD_CUDA(cudaMemcpy(rp.data(), L.rowptr, sizeof(int64_t) * rp.size(), cudaMemcpyDeviceToHost));
      if (L.positions)
        SPD_CUDA(cudaMemcpy(crd.data(), L.crd, sizeof(int64_t) * crd.size(), cudaMemcpyDeviceToHost));
      for (size_t q = 0; q < parent.size(); q++)
        for (int64_t p = rp[parent[q]]; p < rp[parent[q] + 1]; p++) {
          next.push_back(p);
          for (int k = 0; k < base; k++) ncoord[k].push_back(coord[k][q]);
          ncoord[base].push_back(crd[p]);
        }
    }
    parent.swap(next);
    for (int k = 0; k <= base + (int)grp.size() - 1 && k < order; k++) coord[k].swap(ncoord[k]);
    base += (int)grp.size();
  }
  std::vector<double> vals(t->nvals);
  if (t->nvals) SPD_CUDA(cudaMemcpy(vals.data(), t->vals, sizeof(double) * vals.size(), cudaMemcpyDeviceToHost));
  // logical coordinates of each leaf, sorted (tensor.cpp leaves() + sort)
  const int64_t m = (int64_t)parent.size();
  std::vector<int64_t> logical((size_t)m * order);
  for (int64_t q = 0; q < m; q++)
    for (int k = 0; k < order; k++) logical[q * order + t->mode_order[k]] = coord[k][q];
  std::vector<int64_t> perm(m);
  for (int64_t q = 0; q < m; q++) perm[q] = q;
  std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
    return std::lexicographical_compare(&logical[a * order], &logical[a * order] + order, &logical[b * order],
                                        &logical[b * order] + order);
  });
  FILE* f = std::fopen(path, "wb");
  if (!f) throw ParseError("cannot open output file '" + std::string(path) + "'");
  char num[64];
  for (int64_t q : perm) {
    for (int k = 0; k < order; k++) std::fprintf(f, "%lld ", (long long)(logical[q * order + k] + 1));
    std::snprintf(num, sizeof num, "%.17g", vals[parent[q]]);
    std::fprintf(f, "%s\n", num);
  }
  if (std::fclose(f) != 0) throw ParseError("failed writing '" + std::string(path) + "'");
}

}  // namespace

}  // namespace spd

using namespace spd;

extern "C" int spd_tensor_load(spd_context* ctx, const char* path, int order, const int* kinds,
                               const int* mode_order, const int64_t* dims, spd_tensor** out,
                               int64_t* dims_out) {
  return guarded([&] { run_load(ctx, path, order, kinds, mode_order, dims, out, dims_out); });
}

extern "C" int spd_tensor_store(const spd_tensor* t, const char* path) {
  return guarded([&] { run_store(t, path); });
}
