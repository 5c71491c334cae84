// ExecMode::Gpu adapter for the reference runtime (dspar), over the C-ABI of
// include/spdistal_b200.h.  This is the code a dspar maintainer adds next to
// execute() (/root/reference/proj/core/src/sim.cpp:816) to run a Plan on the
// GPU; it compiles against the reference's own headers and the unmodified
// reference library.  See INTEGRATION.md.
//
//   dspar::ExecResult dspar_gpu::execute_gpu(const Plan&, const TensorSet&,
//                                            const MachineGrid&, const Residency&)
//
// (execute()'s signature, sim.hpp:121-122, minus the ExecMode it replaces)
//
// * pattern-matches plan.stmt/formats against the six statements the backend
//   implements and raises ValidationError("unsupported on gpu: ...") for
//   anything else -- no CPU fallback;
// * uploads every tensor straight from the reference's storage: CoordRange is
//   {int64 lo, hi} (index_space.hpp:12-23), so a pos Region's range_values()
//   is passed to spd_tensor_upload as the (lo,hi) pair array, zero-copy;
// * runs the plan's partition step on the GPU (universe or nonzero by
//   plan.loops[0].position_space) and cross-checks the GPU colour bounds
//   against plan.loops[0].color_bounds (a mismatch is a logic_error);
// * runs the leaf + deterministic combine and rebuilds the output with
//   SparseTensor::from_parts, so ExecResult / Stats are drop-in: per-worker
//   work through tuple_worker, imbalance over every worker of the machine,
//   and bytes_by_tensor from the Residency (the reference's ledger).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dspar/errors.hpp"
#include "dspar/plan.hpp"
#include "dspar/planner.hpp"
#include "dspar/sim.hpp"
#include "dspar/tensor.hpp"
#include "spdistal_b200.h"

namespace dspar_gpu {

using namespace dspar;

namespace {

void check(int st) {
  if (st == SPD_OK) return;
  std::string msg = spd_last_error();
  if (st == SPD_ERR_VALIDATION) throw ValidationError(msg);
  throw std::runtime_error(msg);
}

// Contexts (stream, events, scratch, NCCL communicator) live for the process:
// one per device for the single-GPU paths, one group per GPU count for the
// multi-GPU path, so repeated execute() calls do not re-create streams or
// re-initialise NCCL.  Ctx is a non-owning handle on a cached context.
std::mutex g_ctx_mu;
std::map<int, spd_context*> g_single;                    // device -> context
std::map<int, std::vector<spd_context*>> g_groups;       // GPU count -> contexts with a communicator

spd_context* single_context(int device) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto it = g_single.find(device);
  if (it != g_single.end()) return it->second;
  spd_context* h = nullptr;
  check(spd_context_create(device, nullptr, &h));
  g_single[device] = h;
  return h;
}

// The G contexts of a multi-GPU execute (device r = rank r), created once:
// the ranks initialise the communicator together, one host thread each.
std::vector<spd_context*> group_contexts(int G) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto it = g_groups.find(G);
  if (it != g_groups.end()) return it->second;
  std::vector<unsigned char> uid(128, 0);
  check(spd_nccl_unique_id(uid.data()));
  std::vector<spd_context*> cs(G, nullptr);
  std::vector<std::exception_ptr> errors(G);
  std::vector<std::thread> pool;
  for (int r = 0; r < G; r++)
    pool.emplace_back([&, r] {
      try {
        check(spd_context_create(r, nullptr, &cs[r]));
        check(spd_context_init_comm(cs[r], uid.data(), r, G));
      } catch (...) {
        errors[r] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
  g_groups[G] = cs;
  return cs;
}

// A failed multi-GPU call may leave a communicator mid-collective: its group
// is not reused (the next call builds a fresh one).
void drop_group(int G) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  g_groups.erase(G);
}

struct Ctx {
  spd_context* h = nullptr;
  explicit Ctx(int device = 0) : h(single_context(device)) {}
  explicit Ctx(spd_context* c) : h(c) {}
};

struct DevTensor {
  spd_tensor* h = nullptr;
  ~DevTensor() { spd_tensor_destroy(h); }
};

void upload(Ctx& ctx, const SparseTensor& t, DevTensor& out) {
  const FormatSpec& f = t.format();
  std::vector<int> kinds, order(f.mode_order.begin(), f.mode_order.end());
  for (LevelKind k : f.kinds) kinds.push_back(k == LevelKind::Dense ? SPD_DENSE : SPD_COMPRESSED);
  std::vector<const int64_t*> pos(t.num_levels(), nullptr), crd(t.num_levels(), nullptr);
  for (int l = 0; l < t.num_levels(); l++) {
    if (const auto* c = std::get_if<CompressedLevel>(&t.level(l))) {
      static_assert(sizeof(CoordRange) == 2 * sizeof(int64_t), "CoordRange is two int64");
      pos[l] = reinterpret_cast<const int64_t*>(c->pos.range_values().data());
      crd[l] = c->crd.coord_values().data();
    }
  }
  check(spd_tensor_upload(ctx.h, t.order(), t.dims().data(), kinds.data(), order.data(),
                          pos.data(), crd.data(), t.vals().scalar_values().data(), &out.h));
}

// Dense operands live in HBM as their vals (row-major over the format's
// storage order, exactly the reference's vals layout).
const double* dense_vals_dev(const spd_tensor* t) {
  double* p = nullptr;
  check(spd_tensor_vals_ptr(t, &p));
  return p;
}

std::string kernel_of(const Plan& plan) {
  const std::string s = plan.stmt.to_string();
  auto fmt = [&](const std::string& n) {
    const FormatSpec& f = plan.formats.at(n);
    std::string k;
    for (LevelKind x : f.kinds) k += x == LevelKind::Dense ? 'd' : 's';
    return k;
  };
  // The kernels read every operand in mode order: a transposed storage order
  // (CSC 'ds:1,0', column-major 'dd:1,0') is unsupported, except SDDMM's D,
  // whose strides are passed explicitly, and SpAdd3, whose three operands and
  // output only need to share one storage order (the union is per level).
  auto ident = [&](const std::string& n) {
    const auto& mo = plan.formats.at(n).mode_order;
    for (size_t k = 0; k < mo.size(); k++)
      if (mo[k] != static_cast<int>(k)) return false;
    return true;
  };
  auto unsupported = [&](const std::string& why) { return ValidationError("unsupported on gpu: " + why + ": " + s); };
  const auto& terms = plan.stmt.terms;
  const auto& lhs = plan.stmt.lhs;
  if (terms.size() == 3 && lhs.vars.size() == 2) {
    for (const auto& t : terms)
      if (t.size() != 1 || fmt(t[0].tensor) != "ds") throw unsupported("SpAdd3 needs three ds operands");
    for (const auto& t : terms)
      if (plan.formats.at(t[0].tensor).mode_order != plan.formats.at(lhs.tensor).mode_order)
        throw unsupported("SpAdd3 operands and output must share one storage order");
    return "spadd3";
  }
  if (terms.size() != 1) throw unsupported("statement");
  const auto& t = terms[0];
  std::string k;
  if (t.size() == 2 && lhs.vars.size() == 1 && fmt(t[0].tensor) == "ds" && fmt(t[1].tensor) == "d")
    k = "spmv";
  else if (t.size() == 2 && lhs.vars.size() == 2 && fmt(t[0].tensor) == "ds" && fmt(t[1].tensor) == "dd" &&
           fmt(lhs.tensor) == "dd")
    k = "spmm";
  else if (t.size() == 3 && fmt(t[0].tensor) == "ds" && fmt(lhs.tensor) == "ds")
    k = "sddmm";
  else {
    const bool csf = fmt(t[0].tensor) == "dss" || fmt(t[0].tensor) == "sss";
    if (t.size() == 2 && csf && fmt(t[1].tensor) == "d") k = "spttv";
    else if (t.size() == 3 && csf && fmt(lhs.tensor) == "dd") k = "spmttkrp";
    else throw unsupported("statement");
  }
  for (size_t a = 0; a < t.size(); a++)
    if (!(k == "sddmm" && a == 2) && !ident(t[a].tensor)) throw unsupported("transposed storage of " + t[a].tensor);
  if (!ident(lhs.tensor)) throw unsupported("transposed storage of " + lhs.tensor);
  return k;
}


// One task per colour tuple (loop_tuples, sim.cpp:519-533), mapped to its
// worker like tuple_worker (sim.cpp:535-544) and ordered by worker id as
// execute() orders them (sim.cpp:843-847).
struct Task {
  std::vector<int64_t> colors;
  int64_t wid = 0;
};

std::vector<Task> tasks_of(const Plan& plan, const MachineGrid& machine) {
  std::vector<std::vector<int64_t>> tuples{{}};
  for (const auto& loop : plan.loops) {
    std::vector<std::vector<int64_t>> next;
    for (const auto& t : tuples)
      for (int64_t c = 0; c < loop.pieces; c++) {
        auto e = t;
        e.push_back(c);
        next.push_back(std::move(e));
      }
    tuples = std::move(next);
  }
  std::vector<Task> tasks;
  for (auto& colors : tuples) {
    std::vector<int64_t> coords(machine.rank(), 0);
    for (size_t k = 0; k < plan.loops.size(); k++) coords[machine.dim_index(plan.loops[k].machine_dim)] = colors[k];
    tasks.push_back(Task{std::move(colors), machine.worker_id(coords)});
  }
  std::stable_sort(tasks.begin(), tasks.end(), [](const Task& a, const Task& b) { return a.wid < b.wid; });
  return tasks;
}

// Stats of one execute (sim.cpp:824-829, 1000-1005): per-worker work written
// task by task in worker order (a later task of the same worker overwrites,
// as execute does), the communication ledger (bytes_by_tensor), imbalance over
// every worker of the machine.  `task_work[k]` is the work of tasks[k].
//
// Ledger (sim.cpp:851-887): a tensor's needed sets at a task are the full
// sets, or the intersection of its bundle colour sets over the loops up to
// its communicate site (worker_needed_sets, sim.cpp:505-516); bytes are the
// needed entries missing from the worker's Residency sets -- 16 B per pos
// range, 8 B per crd, 8 B per val (sim.hpp:21-23, transfer_bytes :134-147).
// The set construction is the reference's own bookkeeping (full_sets,
// bundle_color_sets, intersect_sets from sim.hpp); the per-entry membership
// counting runs on the GPU (spd_ledger_missing).
Stats make_stats(spd_context* ctx, const Plan& plan, const TensorSet& tensors, const MachineGrid& machine,
                 const Residency& residency, const std::vector<Task>& tasks, const std::vector<int64_t>& task_work) {
  Stats st;
  st.workers = machine.total_workers();
  st.per_worker.resize(static_cast<size_t>(st.workers));
  const auto names = plan.stmt.tensor_names();
  for (auto& w : st.per_worker)
    for (const auto& n : names) w.bytes_by_tensor[n] = 0;
  std::map<std::string, int> site;
  for (const auto& c : plan.root_communicates) site[c.tensor] = -1;
  for (size_t k = 0; k < plan.loops.size(); k++)
    for (const auto& c : plan.loops[k].communicates) site[c.tensor] = static_cast<int>(k);

  // every (needed, held) set pair of every (task, tensor), weighted
  std::vector<RegionIndexSets> keep_needed;
  keep_needed.reserve(tasks.size() * names.size());
  struct Pair {
    const std::vector<int64_t>* need;
    const std::vector<int64_t>* held;
    int64_t weight;
    size_t task;
    std::string name;
  };
  std::vector<Pair> pairs;
  for (size_t k = 0; k < tasks.size(); k++) {
    for (const auto& name : names) {
      auto rit = residency.tensors.find(name);
      if (rit == residency.tensors.end()) continue;  // no declared placement: resident, 0 bytes
      const SparseTensor& t = tensors.at(name);
      RegionIndexSets needed = full_sets(t);
      auto sit = site.find(name);
      if (sit != site.end() && sit->second >= 0)
        for (int l = 0; l <= sit->second; l++) {
          auto b = plan.loops[l].bundle_of.find(name);
          if (b == plan.loops[l].bundle_of.end()) continue;
          needed = intersect_sets(needed, bundle_color_sets(plan.bundles[b->second], tasks[k].colors[l]));
        }
      keep_needed.push_back(std::move(needed));
      const RegionIndexSets& nd = keep_needed.back();
      const RegionIndexSets& held = rit->second.at(static_cast<size_t>(tasks[k].wid));
      for (size_t l = 0; l < nd.levels.size(); l++) {
        pairs.push_back({&nd.levels[l].pos, &held.levels[l].pos, kRangeBytes, k, name});
        pairs.push_back({&nd.levels[l].crd, &held.levels[l].crd, kCoordBytes, k, name});
      }
      pairs.push_back({&nd.vals, &held.vals, kScalarBytes, k, name});
    }
  }
  std::vector<int64_t> missing(pairs.size(), 0);
  if (!pairs.empty()) {
    std::vector<const int64_t*> np, hp;
    std::vector<int64_t> nn, hn;
    for (const auto& p : pairs) {
      np.push_back(p.need->data());
      nn.push_back(static_cast<int64_t>(p.need->size()));
      hp.push_back(p.held->data());
      hn.push_back(static_cast<int64_t>(p.held->size()));
    }
    check(spd_ledger_missing(ctx, static_cast<int64_t>(pairs.size()), np.data(), nn.data(), hp.data(), hn.data(),
                             missing.data()));
  }
  std::vector<std::map<std::string, int64_t>> task_bytes(tasks.size());
  for (size_t i = 0; i < pairs.size(); i++) task_bytes[pairs[i].task][pairs[i].name] += missing[i] * pairs[i].weight;
  for (size_t k = 0; k < tasks.size(); k++) {
    auto& w = st.per_worker[static_cast<size_t>(tasks[k].wid)];
    w.work = task_work[k];
    for (const auto& n : names) w.bytes_by_tensor[n] = task_bytes[k].count(n) ? task_bytes[k][n] : 0;
  }
  int64_t total = 0, mx = 0;
  for (const auto& w : st.per_worker) total += w.work, mx = std::max(mx, w.work);
  st.imbalance = total == 0 ? 1.0 : static_cast<double>(mx) * static_cast<double>(st.workers) / static_cast<double>(total);
  return st;
}
}  // namespace

// SpDISTAL-Batched SpMM: loop 0 divides the rows of B
// / A (a universe split), loop 1 the columns j of C / A (dense).  Every
// (x, y) tuple runs spd_spmm on B's row colour x with the column slab y of C
// (staged contiguous), its block scattered into A; worker ids follow
// tuple_worker (sim.cpp:535-544, machine.cpp:88-92).  Batched SpMTTKRP is the
// same shape: rows i over loop 0, the rank columns l of C, D and A over loop
// 1, spd_spmttkrp on the slabs of both factors.
ExecResult execute_batched(const Plan& plan, const TensorSet& tensors, const MachineGrid& machine,
                           const Residency& residency, const std::string& kernel) {
  const PlanLoop& lx = plan.loops[0];
  const PlanLoop& ly = plan.loops[1];
  const auto& t = plan.stmt.terms[0];
  const std::string out_name = plan.stmt.lhs.tensor;
  const SparseTensor& Bt = tensors.at(t[0].tensor);
  if (lx.position_space || ly.position_space || plan.combine)
    throw ValidationError("unsupported on gpu: batched " + kernel + " needs two universe loops and no combine");
  const std::vector<int64_t>& od = plan.dims.at(out_name);
  const int64_t n = od[0], N = od[1];
  Ctx ctx;
  DevTensor B;
  upload(ctx, Bt, B);
  std::vector<spd_color> cols(lx.pieces);
  check(spd_partition_universe(ctx.h, B.h, lx.pieces, cols.data()));
  for (int64_t c = 0; c < lx.pieces; c++) {
    const CoordRange& want = lx.color_bounds[c];
    const bool same = cols[c].color.lo == want.lo && cols[c].color.hi == want.hi;
    if (!same && !(cols[c].color.lo > cols[c].color.hi && want.empty()))
      throw std::logic_error("gpu partition differs from plan() colour bounds");
  }
  std::vector<double> out(static_cast<size_t>(n * N), 0.0);
  ExecResult r;
  std::vector<std::vector<int64_t>> work_xy(static_cast<size_t>(ly.pieces),
                                            std::vector<int64_t>(static_cast<size_t>(lx.pieces), 0));
  const int kinds[2] = {SPD_DENSE, SPD_DENSE}, order[2] = {0, 1};
  // column slab [lo, lo + w) of a dense rows x N factor, uploaded contiguous
  // (one row copy per factor row)
  auto slab_of = [&](const SparseTensor& F, int64_t lo, int64_t w, DevTensor& dst) {
    const int64_t rows = F.dims()[0];
    const std::vector<double>& fv = F.vals().scalar_values();
    std::vector<double> fy(static_cast<size_t>(rows * w));
    for (int64_t k = 0; k < rows; k++) std::memcpy(fy.data() + k * w, fv.data() + k * N + lo, sizeof(double) * w);
    const int64_t dims[2] = {rows, w};
    check(spd_tensor_upload(ctx.h, 2, dims, kinds, order, nullptr, nullptr, fy.data(), &dst.h));
  };
  for (int64_t y = 0; y < ly.pieces; y++) {
    const CoordRange& slab = ly.color_bounds[y];
    const int64_t w = slab.empty() ? 0 : slab.hi - slab.lo + 1;
    std::vector<int64_t>& work = work_xy[static_cast<size_t>(y)];
    if (w > 0) {
      DevTensor Cy, Dy, Ay;
      const int64_t adims[2] = {n, w};
      std::vector<double> ay(static_cast<size_t>(n * w), 0.0);
      check(spd_tensor_upload(ctx.h, 2, adims, kinds, order, nullptr, nullptr, ay.data(), &Ay.h));
      double* a_dev = const_cast<double*>(dense_vals_dev(Ay.h));
      spd_stats st{};
      slab_of(tensors.at(t[1].tensor), slab.lo, w, Cy);
      if (kernel == "spmm") {
        check(spd_spmm(ctx.h, B.h, dense_vals_dev(Cy.h), w, a_dev, 0, lx.pieces, &st));
      } else {
        slab_of(tensors.at(t[2].tensor), slab.lo, w, Dy);
        check(spd_spmttkrp(ctx.h, B.h, dense_vals_dev(Cy.h), dense_vals_dev(Dy.h), w, a_dev, 0, lx.pieces, &st));
      }
      check(spd_last_work(ctx.h, work.data(), lx.pieces));
      check(spd_tensor_download_vals(Ay.h, ay.data()));
      for (int64_t i = 0; i < n; i++) std::memcpy(out.data() + i * N + slab.lo, ay.data() + i * w, sizeof(double) * w);
    }
  }
  const std::vector<Task> tasks = tasks_of(plan, machine);
  std::vector<int64_t> task_work;
  for (const auto& tk : tasks) task_work.push_back(work_xy[static_cast<size_t>(tk.colors[1])][static_cast<size_t>(tk.colors[0])]);
  r.stats = make_stats(ctx.h, plan, tensors, machine, residency, tasks, task_work);
  r.stats.combines = 0;
  const SparseTensor& outstub = tensors.at(out_name);
  std::vector<LevelStorage> levels;
  for (int l = 0; l < outstub.num_levels(); l++) levels.push_back(outstub.level(l));
  r.output = SparseTensor::from_parts(od, plan.formats.at(out_name), std::move(levels), std::move(out));
  return r;
}

// 2-D grids of SDDMM / SpTTV (PAPER.md:1328-1330 shape, test_planner.cpp:
// 193-225): rows i over loop 0 (a universe split of the dense top level),
// the columns j -- the compressed level 1's coordinate -- over loop 1, the
// bucket split (level_partition.cpp:193-205; spd_partition_bucket).  The
// outputs live on B's pattern (SDDMM) or on its fibres (SpTTV), so every
// (x, y) cell writes only its own entries: one op over the row colours
// computes all cells, and each cell's work is counted on the GPU from the
// bucket split (spd_bucket_grid_work).
ExecResult execute_grid(const Plan& plan, const TensorSet& tensors, const MachineGrid& machine,
                        const Residency& residency, const std::string& kernel) {
  const PlanLoop& lx = plan.loops[0];
  const PlanLoop& ly = plan.loops[1];
  const auto& t = plan.stmt.terms[0];
  const std::string out_name = plan.stmt.lhs.tensor;
  const SparseTensor& Bt = tensors.at(t[0].tensor);
  if (lx.position_space || ly.position_space || plan.combine)
    throw ValidationError("unsupported on gpu: a 2-D " + kernel + " grid needs two universe loops and no combine");
  const int64_t Px = lx.pieces, Py = ly.pieces;
  Ctx ctx;
  DevTensor B;
  upload(ctx, Bt, B);
  std::vector<spd_color> cols(Px);
  check(spd_partition_universe(ctx.h, B.h, Px, cols.data()));
  for (int64_t c = 0; c < Px; c++) {
    const CoordRange& want = lx.color_bounds[c];
    const bool same = cols[c].color.lo == want.lo && cols[c].color.hi == want.hi;
    if (!same && !(cols[c].color.lo > cols[c].color.hi && want.empty()))
      throw std::logic_error("gpu partition differs from plan() colour bounds");
  }
  // the columns' bucket split, checked against the planner's coordinate bounds
  std::vector<int64_t> counts(Py);
  check(spd_partition_bucket(ctx.h, B.h, 1, Py, counts.data()));
  const int64_t extent = Bt.dims()[Bt.format().mode_order[1]];
  for (int64_t c = 0; c < Py; c++) {
    const int64_t block = extent / Py;
    const int64_t lo = c * block, hi = c + 1 == Py ? extent - 1 : lo + block - 1;
    const CoordRange& want = ly.color_bounds[c];
    if (!((lo == want.lo && hi == want.hi) || (lo > hi && want.empty())))
      throw std::logic_error("gpu bucket split differs from plan() colour bounds");
  }
  std::map<std::string, DevTensor> dev;
  for (const auto& a : t)
    if (a.tensor != t[0].tensor && !dev.count(a.tensor)) upload(ctx, tensors.at(a.tensor), dev[a.tensor]);
  const SparseTensor& outstub = tensors.at(out_name);
  DevTensor outbuf;
  upload(ctx, outstub, outbuf);
  double* outp = const_cast<double*>(dense_vals_dev(outbuf.h));
  spd_stats st{};
  int64_t mult = 1;
  std::vector<int64_t> spans(2 * Px);
  for (int64_t x = 0; x < Px; x++) {  // each row colour's span of level-1 positions
    const spd_range r = kernel == "sddmm" ? cols[x].q : cols[x].par;
    spans[2 * x] = r.lo, spans[2 * x + 1] = r.hi;
  }
  if (kernel == "sddmm") {
    const SparseTensor& Ct = tensors.at(t[1].tensor);
    const SparseTensor& Dt = tensors.at(t[2].tensor);
    const int64_t K = Ct.dims()[1];
    const bool jmajor = Dt.format().mode_order[0] == 1;
    check(spd_sddmm(ctx.h, B.h, dense_vals_dev(dev[t[1].tensor].h), dense_vals_dev(dev[t[2].tensor].h), K,
                    jmajor ? 1 : Dt.dims()[1], jmajor ? K : 1, outp, 0, Px, &st));
    mult = K;
  } else {
    check(spd_spttv(ctx.h, B.h, dense_vals_dev(dev[t[1].tensor].h), outp, 0, Px, &st));
  }
  std::vector<int64_t> cell(Px * Py);
  check(spd_bucket_grid_work(ctx.h, spans.data(), Px, cell.data()));
  std::vector<double> vals(outstub.leaf_count());
  check(spd_tensor_download_vals(outbuf.h, vals.data()));
  std::vector<LevelStorage> levels;
  for (int l = 0; l < outstub.num_levels(); l++) levels.push_back(outstub.level(l));
  ExecResult r{SparseTensor::from_parts(plan.dims.at(out_name), plan.formats.at(out_name), std::move(levels),
                                        std::move(vals)),
               Stats{}};
  const std::vector<Task> tasks = tasks_of(plan, machine);
  std::vector<int64_t> task_work;
  for (const auto& tk : tasks) task_work.push_back(cell[tk.colors[0] * Py + tk.colors[1]] * mult);
  r.stats = make_stats(ctx.h, plan, tensors, machine, residency, tasks, task_work);
  r.stats.combines = 0;
  return r;
}

// The GPUs a one-loop plan's colours are spread over: every visible device,
// at most one per colour, capped by DSPAR_GPUS when set.  Each GPU runs one
// contiguous block of ceil(P / G) colours, the way execute() hands colour
// tasks to its thread pool (sim.cpp:833-847, 958-980).
static int gpus_for(int64_t pieces) {
  int n = 1;
  check(spd_device_count(&n));
  if (const char* e = std::getenv("DSPAR_GPUS")) n = std::min(n, std::max(1, std::atoi(e)));
  int64_t g = std::min<int64_t>(n, std::max<int64_t>(pieces, 1));
  const int64_t cmax = (pieces + g - 1) / std::max<int64_t>(g, 1);
  return static_cast<int>(std::max<int64_t>(1, (pieces + cmax - 1) / cmax));  // every GPU gets >= 1 colour
}

// One GPU's share of execute_gpu: uploads, the partition step (checked
// against the planner's colour bounds), its block of colours -- the
// cross-GPU boundary combine and SpAdd3's offsets run over NCCL inside the
// backend -- and the copy of the output ranges it owns into `out`.
struct GpuPart {
  int device = 0, rank = 0, world = 1;
  spd_context* ctx = nullptr;  // the GPU's cached context (with its communicator when world > 1)
  int64_t first = 0, count = 0;
  std::vector<int64_t> work;
  int64_t combines = 0;
  SparseTensor spadd3_out;  // rank 0, SpAdd3 only
};

static void run_part(const Plan& plan, const TensorSet& tensors, const std::string& kernel, GpuPart& g,
                     std::vector<double>& out) {
  const PlanLoop& loop = plan.loops[0];
  const auto& terms = plan.stmt.terms;
  const std::string out_name = plan.stmt.lhs.tensor;
  const std::string b_name = terms[0][0].tensor;
  const SparseTensor& Bt = tensors.at(b_name);
  const int64_t P = loop.pieces;
  Ctx ctx(g.ctx ? g.ctx : single_context(g.device));
  DevTensor B;
  upload(ctx, Bt, B);
  std::vector<spd_color> cols(P);
  if (loop.position_space)
    check(spd_partition_nonzero(ctx.h, B.h, loop.split_level, P, cols.data()));
  else
    check(spd_partition_universe(ctx.h, B.h, P, cols.data()));
  for (int64_t c = 0; c < P; c++) {  // the GPU's partition must be the planner's
    const CoordRange& want = loop.color_bounds[c];
    bool same = cols[c].color.lo == want.lo && cols[c].color.hi == want.hi;
    bool both_empty = cols[c].color.lo > cols[c].color.hi && want.empty();
    if (!same && !both_empty) throw std::logic_error("gpu partition differs from plan() colour bounds");
  }
  spd_stats st{};
  const std::vector<int64_t>& od = plan.dims.at(out_name);
  std::map<std::string, DevTensor> dev;
  for (const auto& term : terms)
    for (const auto& a : term)
      if (a.tensor != b_name && !dev.count(a.tensor)) upload(ctx, tensors.at(a.tensor), dev[a.tensor]);
  const SparseTensor& outstub = tensors.at(out_name);
  DevTensor outbuf;
  if (kernel != "spadd3") upload(ctx, outstub, outbuf);  // dense: zeros; sparse: B's pattern reuse
  double* outp = kernel != "spadd3" ? const_cast<double*>(dense_vals_dev(outbuf.h)) : nullptr;
  const int64_t f = g.first, n = g.count;
  if (kernel == "spmv") {
    check(spd_spmv(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h), outp, f, n, &st));
  } else if (kernel == "spmm") {
    check(spd_spmm(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h), od[1], outp, f, n, &st));
  } else if (kernel == "sddmm") {
    const SparseTensor& Ct = tensors.at(terms[0][1].tensor);
    const SparseTensor& Dt = tensors.at(terms[0][2].tensor);
    const int64_t K = Ct.dims()[1];
    const bool jmajor = Dt.format().mode_order[0] == 1;
    check(spd_sddmm(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h), dense_vals_dev(dev[terms[0][2].tensor].h),
                    K, jmajor ? 1 : Dt.dims()[1], jmajor ? K : 1, outp, f, n, &st));
  } else if (kernel == "spttv") {
    check(spd_spttv(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h), outp, f, n, &st));
  } else if (kernel == "spmttkrp") {
    check(spd_spmttkrp(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h),
                       dense_vals_dev(dev[terms[0][2].tensor].h), od[1], outp, f, n, &st));
  } else {  // spadd3: two-phase assembly per GPU, the row blocks gathered on rank 0
    spd_tensor* A = nullptr;
    check(spd_spadd3(ctx.h, B.h, dev[terms[1][0].tensor].h, dev[terms[2][0].tensor].h, &A, f, n, &st));
    DevTensor Ah, Af;
    Ah.h = A;
    spd_tensor* whole = A;
    if (g.world > 1) {
      check(spd_gather_rows(ctx.h, A, 0, &Af.h));
      whole = Af.h;
    }
    if (g.rank == 0) {
      int64_t par = 0, nnz = 0;
      int k;
      check(spd_tensor_level(whole, 1, &k, &par, &nnz));
      std::vector<CoordRange> pos(par);
      std::vector<int64_t> crd(nnz);
      std::vector<double> vals(nnz);
      check(spd_tensor_download_level(whole, 1, reinterpret_cast<int64_t*>(pos.data()), crd.data()));
      check(spd_tensor_download_vals(whole, vals.data()));
      std::vector<LevelStorage> levels{std::get<DenseLevel>(Bt.level(0)),
                                       CompressedLevel{Region::ranges(IndexSpace({par}), std::move(pos), nnz),
                                                       Region::coordinates(IndexSpace({nnz}), std::move(crd))}};
      g.spadd3_out = SparseTensor::from_parts(od, plan.formats.at(out_name), std::move(levels), std::move(vals));
    }
  }
  if (kernel != "spadd3") {  // copy back the output range these colours own
    int64_t lo = 0, hi = -1, width = 1;
    if (kernel == "sddmm") {  // vals on B's pattern: the colours' positions
      lo = cols[f].q.lo, hi = cols[f + n - 1].q.hi;
      for (int64_t c = f; c < f + n; c++)
        if (cols[c].q.lo <= cols[c].q.hi) lo = std::min(lo, cols[c].q.lo), hi = std::max(hi, cols[c].q.hi);
    } else {
      check(spd_last_owned(ctx.h, f, n, &lo, &hi));
      if (kernel == "spmm" || kernel == "spmttkrp") width = od[1];
    }
    if (g.world == 1) {
      lo = 0, hi = static_cast<int64_t>(out.size()) / width - 1;
    }
    if (lo <= hi) check(spd_tensor_download_vals_range(outbuf.h, lo * width, (hi - lo + 1) * width, out.data() + lo * width));
  }
  if (g.rank == 0) {
    g.work.assign(P, 0);
    check(spd_last_work(ctx.h, g.work.data(), P));
    g.combines = st.combines;
  }
}

ExecResult execute_gpu(const Plan& plan, const TensorSet& tensors, const MachineGrid& machine,
                       const Residency& residency) {
  if (plan.loops.size() == 2) {
    const std::string k = kernel_of(plan);
    if (k == "spmm" || k == "spmttkrp") return execute_batched(plan, tensors, machine, residency, k);
    if (k == "sddmm" || k == "spttv") return execute_grid(plan, tensors, machine, residency, k);
  }
  if (plan.loops.size() != 1)
    throw ValidationError("unsupported on gpu: one distributed loop, or a two-loop grid of SpMM / SpMTTKRP "
                          "(batched) or SDDMM / SpTTV (rows x bucketed columns)");
  const PlanLoop& loop = plan.loops[0];
  const std::string kernel = kernel_of(plan);
  const std::string out_name = plan.stmt.lhs.tensor;
  const int64_t P = loop.pieces;
  const int G = gpus_for(P);
  const int64_t cmax = (P + G - 1) / G;
  std::vector<GpuPart> parts(G);
  const std::vector<spd_context*> group = G > 1 ? group_contexts(G) : std::vector<spd_context*>{};
  const SparseTensor& outstub = tensors.at(out_name);
  std::vector<double> out(kernel == "spadd3" ? 0 : static_cast<size_t>(outstub.leaf_count()), 0.0);
  for (int r = 0; r < G; r++) {
    parts[r].device = r, parts[r].rank = r, parts[r].world = G;
    parts[r].ctx = G > 1 ? group[r] : nullptr;
    parts[r].first = r * cmax;
    parts[r].count = std::min<int64_t>(cmax, P - r * cmax);
  }
  if (G == 1) {
    parts[0].first = 0, parts[0].count = P;
    run_part(plan, tensors, kernel, parts[0], out);
  } else {  // one host thread per GPU; errors are captured per thread and rethrown (sim.cpp:958-980)
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errors(G);
    for (int r = 0; r < G; r++)
      pool.emplace_back([&, r] {
        try {
          run_part(plan, tensors, kernel, parts[r], out);
        } catch (...) {
          errors[r] = std::current_exception();
          // the other GPUs may be waiting for this one in a collective:
          // abort their communicators so every thread returns
          for (int q = 0; q < G; q++)
            if (q != r) spd_context_abort(group[q]);
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errors)
      if (e) {
        drop_group(G);
        std::rethrow_exception(e);
      }
  }
  SparseTensor result;
  if (kernel == "spadd3") {
    result = std::move(parts[0].spadd3_out);
  } else {
    std::vector<LevelStorage> levels;
    for (int l = 0; l < outstub.num_levels(); l++) levels.push_back(outstub.level(l));
    result = SparseTensor::from_parts(plan.dims.at(out_name), plan.formats.at(out_name), std::move(levels),
                                      std::move(out));
  }
  ExecResult r{std::move(result), Stats{}};
  const std::vector<Task> tasks = tasks_of(plan, machine);
  std::vector<int64_t> task_work;
  for (const auto& tk : tasks) task_work.push_back(parts[0].work[static_cast<size_t>(tk.colors[0])]);
  Ctx lctx(0);  // the ledger's set counting
  r.stats = make_stats(lctx.h, plan, tensors, machine, residency, tasks, task_work);
  r.stats.combines = parts[0].combines;
  return r;
}

}  // namespace dspar_gpu
