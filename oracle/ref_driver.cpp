// TEST INFRASTRUCTURE ONLY -- the checker, never the product.
//
// C-ABI driver over the (patched, see patch_ref.py) reference library built
// into oracle/_ref/.  It mirrors the reference's own pipeline,
// `build_pipeline` + `cmd_run` (/root/reference/proj/core/src/cli.cpp:72-195),
// except that tensors arrive in memory and are built with
// `SparseTensor::from_parts` (tensor.cpp:184-197) instead of `pack`/file I/O,
// exactly as SURVEY.md section 7 step 0 prescribes.  Only tests/, smoke() and
// bench.py's reference / cpu_baseline legs load this library (through ctypes).
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "dspar/deppart.hpp"
#include "dspar/errors.hpp"
#include "dspar/format_lang.hpp"
#include "dspar/machine.hpp"
#include "dspar/oracle.hpp"
#include "dspar/plan.hpp"
#include "dspar/planner.hpp"
#include "dspar/schedule.hpp"
#include "dspar/sim.hpp"
#include "dspar/tensor.hpp"
#include "dspar/tensor_io.hpp"
#include "dspar/tin.hpp"

using namespace dspar;

#ifdef WITH_GPU_EXEC
// integration/gpu_execute.cpp: the ExecMode::Gpu adapter under test.
namespace dspar_gpu {
ExecResult execute_gpu(const Plan& plan, const TensorSet& tensors, const MachineGrid& machine,
                       const Residency& residency);
}
#endif

extern "C" {

// One tensor as the reference stores it: per-level pos as inclusive (lo,hi)
// pairs (index_space.hpp:12-23), crd as int64, vals as fp64.
typedef struct ref_tensor_in {
  const char* name;
  int order;
  const int64_t* dims;
  const char* format;                // format language, format_lang.hpp:15
  const int64_t* const* pos_pairs;   // per level: 2*pos_len int64 (NULL for dense levels)
  const int64_t* pos_len;            // per level
  const int64_t* const* crd;         // per level (NULL for dense levels)
  const int64_t* crd_len;            // per level
  const double* vals;
  int64_t nvals;
  const char* tdn;                   // optional distribution statement (NULL: default_tdn)
} ref_tensor_in;
}

namespace {

struct RefRun {
  int status = 0;  // 0 ok, 1 runtime / closure, 2 validation (cli.cpp:297-319)
  std::string error;
  TinStatement stmt;
  MachineGrid machine;
  std::map<std::string, FormatSpec> formats;
  std::map<std::string, std::vector<int64_t>> dims;
  TensorSet tensors;
  Plan compute;
  bool has_result = false;
  ExecResult result;
  std::string stats_json;
  std::string rendered;
  double plan_seconds = 0, exec_seconds = 0, place_seconds = 0;
};

SparseTensor build_tensor(const ref_tensor_in& in) {
  std::vector<int64_t> dims(in.dims, in.dims + in.order);
  FormatSpec fmt = parse_format(in.format);
  auto groups = level_grouping(fmt);
  std::vector<LevelStorage> levels;
  int64_t parent = 1;
  for (size_t l = 0; l < groups.size(); l++) {
    if (fmt.kinds[groups[l][0]] == LevelKind::Dense) {
      std::vector<int64_t> ext;
      for (int k : groups[l]) ext.push_back(dims[fmt.mode_order[k]]);
      IndexSpace dom(ext);
      parent *= dom.total();
      levels.push_back(DenseLevel{dom});
    } else {
      int64_t np = in.pos_len[l], nc = in.crd_len[l];
      std::vector<CoordRange> pos(static_cast<size_t>(np));
      for (int64_t p = 0; p < np; p++) pos[p] = {in.pos_pairs[l][2 * p], in.pos_pairs[l][2 * p + 1]};
      std::vector<int64_t> crd(in.crd[l], in.crd[l] + nc);
      levels.push_back(CompressedLevel{Region::ranges(IndexSpace({np}), std::move(pos), nc),
                                       Region::coordinates(IndexSpace({nc}), std::move(crd))});
      parent = nc;
    }
  }
  std::vector<double> vals(in.vals, in.vals + in.nvals);
  return SparseTensor::from_parts(dims, fmt, std::move(levels), std::move(vals));
}

template <class F>
void guarded(RefRun* r, F&& f) {
  try {
    f();
  } catch (const ParseError& e) {
    r->status = 2, r->error = e.what();
  } catch (const ValidationError& e) {
    r->status = 2, r->error = e.what();
  } catch (const ClosureViolation& e) {
    r->status = 1, r->error = e.what();
  } catch (const std::invalid_argument& e) {
    r->status = 2, r->error = e.what();
  } catch (const std::exception& e) {
    r->status = 1, r->error = e.what();
  }
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

const TensorPartitionBundle* find_bundle(const RefRun* r, int loop, const char* tensor) {
  if (loop < 0 || loop >= static_cast<int>(r->compute.loops.size())) return nullptr;
  const auto& bo = r->compute.loops[loop].bundle_of;
  auto it = bo.find(tensor);
  if (it == bo.end()) return nullptr;
  return &r->compute.bundles[it->second];
}

}  // namespace

namespace {
struct RefPart {
  int status = 0;
  std::string error;
  Partition part;
};

static std::vector<std::vector<int64_t>> subsets_of(int64_t P, const int64_t* off, const int64_t* idx) {
  std::vector<std::vector<int64_t>> s(static_cast<size_t>(P));
  for (int64_t c = 0; c < P; c++) s[c].assign(idx + off[c], idx + off[c + 1]);
  return s;
}

template <class F>
static void* part_guarded(F&& f) {
  auto* r = new RefPart();
  try {
    r->part = f();
  } catch (const std::invalid_argument& e) {
    r->status = 2;
    r->error = e.what();
  } catch (const std::exception& e) {
    r->status = 1;
    r->error = e.what();
  }
  return r;
}

}  // namespace

extern "C" {

// Runs the reference pipeline (cli.cpp:72-195 with in-memory tensors).
//   out_name/out_format/out_order/out_dims: the output tensor's declaration
//   (out_dims may be NULL: inferred like cli.cpp:107-120)
//   use_placements: 1 lowers TDN placements into a Residency (cli.cpp:152-159),
//                   0 passes an empty Residency (every tensor already resident)
//   mode: "seq" | "par" | "instrumented" (sim.cpp:14-19); do_execute 0 = plan only
void* ref_run(const char* expr, const char* schedule, const char* grid, const char* out_format,
              const char* out_tdn, int ntensors, const ref_tensor_in* inputs,
              int use_placements, const char* mode, int do_execute) {
  auto* r = new RefRun();
  guarded(r, [&] {
    r->stmt = parse_tin(expr);
    r->machine = MachineGrid::parse(grid);
    std::map<std::string, TdnStatement> tdns;
    for (int t = 0; t < ntensors; t++) {
      const ref_tensor_in& in = inputs[t];
      r->formats[in.name] = parse_format(in.format);
      SparseTensor st = build_tensor(in);
      r->dims[in.name] = st.dims();
      r->tensors.emplace(in.name, std::move(st));
      if (in.tdn && *in.tdn) tdns[in.name] = parse_tdn(in.tdn);
    }
    const std::string& out = r->stmt.lhs.tensor;
    r->formats[out] = parse_format(out_format);
    if (out_tdn && *out_tdn) tdns[out] = parse_tdn(out_tdn);
    for (const auto& name : r->stmt.tensor_names())
      if (!r->formats.count(name)) throw ValidationError("no format for tensor '" + name + "'");
    std::vector<int64_t> out_dims;
    for (const auto& v : r->stmt.lhs.vars) {
      int64_t extent = -1;
      for (const auto& a : r->stmt.rhs_accesses())
        for (size_t m = 0; m < a.vars.size(); m++)
          if (a.vars[m] == v) extent = r->dims.at(a.tensor)[m];
      out_dims.push_back(extent);
    }
    r->dims[out] = out_dims;
    r->tensors.emplace(out, make_output_stub(r->stmt, r->formats, r->dims, r->tensors));

    Schedule sched;
    if (schedule && *schedule) {
      sched = Schedule::parse(schedule);
    } else if (!r->stmt.lhs.vars.empty()) {
      const std::string& v = r->stmt.lhs.vars[0];
      const std::string& d = r->machine.names()[0];
      sched = Schedule::parse("divide(" + v + ", " + v + "_o, " + v + "_i, M." + d +
                              "); distribute(" + v + "_o, M." + d + ")");
    }
    double t0 = now();
    ScheduledStatement ss = validate_schedule(r->stmt, sched, r->formats, r->dims, r->machine);
    r->compute = plan(ss, r->tensors);
    r->plan_seconds = now() - t0;
    r->rendered = render_plan(r->compute);

    Residency residency;
    if (use_placements) {
      double tp = now();
      std::map<std::string, Plan> placements;
      for (const auto& name : r->stmt.tensor_names()) {
        TdnStatement tdn = tdns.count(name) ? tdns[name]
                                            : default_tdn(name, r->formats.at(name).order());
        placements.emplace(name, lower_tdn(tdn, r->formats.at(name), r->dims.at(name),
                                           r->machine, r->tensors.at(name)));
      }
      residency = residency_from_placements(placements, r->machine, r->tensors);
      r->place_seconds = now() - tp;
    }
    if (do_execute) {
      double t1 = now();
#ifdef WITH_GPU_EXEC
      if (std::string(mode) == "gpu")
        r->result = dspar_gpu::execute_gpu(r->compute, r->tensors, r->machine, residency);
      else
#endif
        r->result = execute(r->compute, r->tensors, r->machine, residency, parse_exec_mode(mode));
      r->exec_seconds = now() - t1;
      r->has_result = true;
      r->stats_json = r->result.stats.to_json();
    }
  });
  return r;
}

void ref_free(void* h) { delete static_cast<RefRun*>(h); }
int ref_status(void* h) { return static_cast<RefRun*>(h)->status; }
const char* ref_error(void* h) { return static_cast<RefRun*>(h)->error.c_str(); }
double ref_plan_seconds(void* h) { return static_cast<RefRun*>(h)->plan_seconds; }
double ref_exec_seconds(void* h) { return static_cast<RefRun*>(h)->exec_seconds; }
double ref_place_seconds(void* h) { return static_cast<RefRun*>(h)->place_seconds; }
const char* ref_rendered_plan(void* h) { return static_cast<RefRun*>(h)->rendered.c_str(); }
const char* ref_stats_json(void* h) { return static_cast<RefRun*>(h)->stats_json.c_str(); }
int ref_has_combine(void* h) { return static_cast<RefRun*>(h)->compute.combine.has_value(); }
int ref_num_loops(void* h) { return static_cast<int>(static_cast<RefRun*>(h)->compute.loops.size()); }

// PlanLoop summary (plan.hpp:49-62).
int ref_loop_info(void* h, int loop, int64_t* pieces, int* position_space, int* split_level) {
  auto* r = static_cast<RefRun*>(h);
  if (loop < 0 || loop >= static_cast<int>(r->compute.loops.size())) return -1;
  const PlanLoop& pl = r->compute.loops[loop];
  *pieces = pl.pieces;
  *position_space = pl.position_space;
  *split_level = pl.split_level;
  return 0;
}

// PlanLoop::color_bounds as 2*pieces int64 (lo, hi).
int ref_loop_color_bounds(void* h, int loop, int64_t* out) {
  auto* r = static_cast<RefRun*>(h);
  if (loop < 0 || loop >= static_cast<int>(r->compute.loops.size())) return -1;
  const auto& cb = r->compute.loops[loop].color_bounds;
  for (size_t c = 0; c < cb.size(); c++) out[2 * c] = cb[c].lo, out[2 * c + 1] = cb[c].hi;
  return static_cast<int>(cb.size());
}

// PartitionStep::bounds of `tensor` at `loop` (plan.hpp:18-27): kind, then bounds.
int ref_step_bounds(void* h, int loop, const char* tensor, int* kind, int64_t* out) {
  auto* r = static_cast<RefRun*>(h);
  if (loop < 0 || loop >= static_cast<int>(r->compute.loops.size())) return -1;
  for (const auto& st : r->compute.loops[loop].partitions) {
    if (st.tensor != tensor) continue;
    *kind = static_cast<int>(st.bounds.kind);
    for (size_t c = 0; c < st.bounds.bounds.size(); c++)
      out[2 * c] = st.bounds.bounds[c].lo, out[2 * c + 1] = st.bounds.bounds[c].hi;
    return static_cast<int>(st.bounds.bounds.size());
  }
  return -1;
}

// One colour's subset of a bundle region (bundle.hpp:15-33).
//   which: 0 dom, 1 pos, 2 crd (level-indexed); 3 vals (level ignored)
// Returns the subset size (copies up to cap entries), -1 when absent.
int64_t ref_bundle_subset(void* h, int loop, const char* tensor, int level, int which,
                          int64_t color, int64_t* out, int64_t cap) {
  auto* r = static_cast<RefRun*>(h);
  const TensorPartitionBundle* b = find_bundle(r, loop, tensor);
  if (!b) return -1;
  const Partition* p = nullptr;
  if (which == 3) {
    p = &b->vals;
  } else {
    if (level < 0 || level >= static_cast<int>(b->levels.size())) return -1;
    const LevelPartition& lp = b->levels[level];
    const std::optional<Partition>& o = which == 0 ? lp.dom : which == 1 ? lp.pos : lp.crd;
    if (!o) return -1;
    p = &*o;
  }
  if (color < 0 || color >= p->num_colors()) return -1;
  const auto& s = p->subset(color);
  int64_t n = static_cast<int64_t>(s.size());
  for (int64_t k = 0; k < n && k < cap; k++) out[k] = s[k];
  return n;
}

int ref_bundle_disjoint(void* h, int loop, const char* tensor) {
  const TensorPartitionBundle* b = find_bundle(static_cast<RefRun*>(h), loop, tensor);
  return b ? b->vals.disjoint() : -1;
}

// SparseTensor::pack (tensor.cpp:94-182) of n COO entries (coords row-major,
// n x order, logical mode order); the packed tensor is read back with the
// ref_out_* getters.  Pins the device-side pack (spd_tensor_pack).
void* ref_pack(int order, const int64_t* dims, const char* format, int64_t n, const int64_t* coords,
               const double* values) {
  auto* r = new RefRun();
  guarded(r, [&] {
    std::vector<int64_t> d(dims, dims + order);
    std::vector<TensorEntry> entries(static_cast<size_t>(n));
    for (int64_t e = 0; e < n; e++) {
      entries[e].coords.assign(coords + e * order, coords + (e + 1) * order);
      entries[e].value = values[e];
    }
    double t0 = now();
    r->result.output = SparseTensor::pack(d, parse_format(format), std::move(entries));
    r->exec_seconds = now() - t0;
    r->has_result = true;
  });
  return r;
}

// load_tensor (tensor_io.cpp:136-142): .tns or MatrixMarket file -> pack.
// dims may be NULL (inferred / taken from the MatrixMarket header).  Pins the
// device-side loader (spd_tensor_load).
void* ref_load(const char* path, const char* format, int order, const int64_t* dims) {
  auto* r = new RefRun();
  guarded(r, [&] {
    std::optional<std::vector<int64_t>> d;
    if (dims) d = std::vector<int64_t>(dims, dims + order);
    double t0 = now();
    r->result.output = load_tensor(path, parse_format(format), d);
    r->exec_seconds = now() - t0;
    r->has_result = true;
  });
  return r;
}

// store_tensor (tensor_io.cpp:158-163) of the run's output tensor.
int ref_store(void* h, const char* path) {
  auto* r = static_cast<RefRun*>(h);
  if (!r->has_result) return -1;
  guarded(r, [&] { store_tensor(r->result.output, path); });
  return r->status;
}

// Output tensor access.
int ref_out_nlevels(void* h) {
  auto* r = static_cast<RefRun*>(h);
  return r->has_result ? r->result.output.num_levels() : -1;
}
int ref_out_level(void* h, int l, int* kind, int64_t* pos_len, int64_t* crd_len) {
  auto* r = static_cast<RefRun*>(h);
  const SparseTensor& t = r->result.output;
  if (!r->has_result || l < 0 || l >= t.num_levels()) return -1;
  if (t.level_kind(l) == LevelKind::Dense) {
    *kind = 0;
    *pos_len = 0;
    *crd_len = std::get<DenseLevel>(t.level(l)).dom.total();
  } else {
    const auto& c = std::get<CompressedLevel>(t.level(l));
    *kind = 1;
    *pos_len = c.pos.size();
    *crd_len = c.crd.size();
  }
  return 0;
}
int ref_out_copy_level(void* h, int l, int64_t* pos_pairs, int64_t* crd) {
  auto* r = static_cast<RefRun*>(h);
  const SparseTensor& t = r->result.output;
  if (!r->has_result || l < 0 || l >= t.num_levels() || t.level_kind(l) != LevelKind::Compressed)
    return -1;
  const auto& c = std::get<CompressedLevel>(t.level(l));
  for (int64_t p = 0; p < c.pos.size(); p++)
    pos_pairs[2 * p] = c.pos.range_at(p).lo, pos_pairs[2 * p + 1] = c.pos.range_at(p).hi;
  for (int64_t q = 0; q < c.crd.size(); q++) crd[q] = c.crd.coord_at(q);
  return 0;
}
int ref_out_dims(void* h, int64_t* dims) {
  auto* r = static_cast<RefRun*>(h);
  if (!r->has_result) return -1;
  const auto& d = r->result.output.dims();
  for (size_t k = 0; k < d.size(); k++) dims[k] = d[k];
  return 0;
}
int64_t ref_out_nvals(void* h) {
  auto* r = static_cast<RefRun*>(h);
  return r->has_result ? r->result.output.leaf_count() : -1;
}
int ref_out_copy_vals(void* h, double* out) {
  auto* r = static_cast<RefRun*>(h);
  if (!r->has_result) return -1;
  const auto& v = r->result.output.vals().scalar_values();
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return 0;
}

// Stats (sim.hpp:25-36) without JSON parsing.
// ---- dependent partitioning (deppart.cpp:15-101) over flat arrays; pins the
// device deppart (spd_deppart_*).  Partitions are (P, off[P+1], idx); range
// regions are n (lo,hi) pairs pointing into dest_extent.  The result is read
// back with ref_part_*.
void* ref_image(const int64_t* ranges, int64_t n, int64_t dest_extent, int64_t P, const int64_t* off,
                const int64_t* idx) {
  return part_guarded([&] {
    std::vector<CoordRange> rs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; i++) rs[i] = CoordRange{ranges[2 * i], ranges[2 * i + 1]};
    Region src = Region::ranges(IndexSpace({n}), std::move(rs), dest_extent);
    Partition p(IndexSpace({n}), subsets_of(P, off, idx));
    return image(src, p, IndexSpace({dest_extent}));
  });
}

void* ref_preimage(const int64_t* ranges, int64_t n, int64_t dest_extent, int64_t P, const int64_t* off,
                   const int64_t* idx) {
  return part_guarded([&] {
    std::vector<CoordRange> rs(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; i++) rs[i] = CoordRange{ranges[2 * i], ranges[2 * i + 1]};
    Region src = Region::ranges(IndexSpace({n}), std::move(rs), dest_extent);
    Partition p(IndexSpace({dest_extent}), subsets_of(P, off, idx));
    return preimage(src, p, IndexSpace({dest_extent}));
  });
}

// colors[k] with box bounds[k*rank*2 ...] (lo,hi per dimension).
void* ref_partition_by_bounds(int rank, const int64_t* extents, int64_t nentries, const int64_t* colors,
                              const int64_t* bounds) {
  return part_guarded([&] {
    std::map<int64_t, std::vector<CoordRange>> coloring;
    for (int64_t k = 0; k < nentries; k++) {
      std::vector<CoordRange> b(static_cast<size_t>(rank));
      for (int d = 0; d < rank; d++) b[d] = CoordRange{bounds[(k * rank + d) * 2], bounds[(k * rank + d) * 2 + 1]};
      coloring[colors[k]] = b;
    }
    return partition_by_bounds(IndexSpace(std::vector<int64_t>(extents, extents + rank)), coloring);
  });
}

int ref_part_status(void* h) { return static_cast<RefPart*>(h)->status; }
const char* ref_part_error(void* h) { return static_cast<RefPart*>(h)->error.c_str(); }
int64_t ref_part_colors(void* h) { return static_cast<RefPart*>(h)->part.num_colors(); }
int ref_part_disjoint(void* h) { return static_cast<RefPart*>(h)->part.disjoint() ? 1 : 0; }
// off: P+1 entries; idx: off[P] entries (either may be NULL)
void ref_part_copy(void* h, int64_t* off, int64_t* idx) {
  const Partition& p = static_cast<RefPart*>(h)->part;
  int64_t o = 0;
  for (int64_t c = 0; c < p.num_colors(); c++) {
    if (off) off[c] = o;
    for (int64_t v : p.subset(c)) {
      if (idx) idx[o] = v;
      o++;
    }
  }
  if (off) off[p.num_colors()] = o;
}
void ref_part_free(void* h) { delete static_cast<RefPart*>(h); }

int64_t ref_stats_workers(void* h) { return static_cast<RefRun*>(h)->result.stats.workers; }
int64_t ref_stats_combines(void* h) { return static_cast<RefRun*>(h)->result.stats.combines; }
double ref_stats_imbalance(void* h) { return static_cast<RefRun*>(h)->result.stats.imbalance; }
int64_t ref_stats_work(void* h, int64_t w) {
  return static_cast<RefRun*>(h)->result.stats.per_worker.at(w).work;
}

// Independent dense oracle: densify + dense_eval (oracle.cpp:39-43, 111-131).
// Writes the row-major dense result (product of out_dims entries) into `out`.
int ref_dense_eval(const char* expr, int ntensors, const ref_tensor_in* inputs, int out_order,
                   const int64_t* out_dims, double* out, char* err, int errlen) {
  try {
    TinStatement stmt = parse_tin(expr);
    std::map<std::string, DenseTensor> dense;
    std::map<std::string, std::vector<int64_t>> dims;
    for (int t = 0; t < ntensors; t++) {
      SparseTensor st = build_tensor(inputs[t]);
      dims[inputs[t].name] = st.dims();
      dense[inputs[t].name] = densify(st);
    }
    dims[stmt.lhs.tensor] = std::vector<int64_t>(out_dims, out_dims + out_order);
    DenseTensor res = dense_eval(stmt, dense, dims);
    std::memcpy(out, res.values.data(), res.values.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen > 0) {
      std::strncpy(err, e.what(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return 1;
  }
}

}  // extern "C"
