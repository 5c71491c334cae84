// ExecMode::Gpu adapter for the reference runtime (dspar), over the C-ABI of
// include/spdistal_b200.h.  This is the code a dspar maintainer adds next to
// execute() (/root/reference/proj/core/src/sim.cpp:816) to run a Plan on the
// GPU; it compiles against the reference's own headers and the unmodified
// reference library.  See INTEGRATION.md.
//
//   dspar::ExecResult dspar_gpu::execute_gpu(const Plan&, const TensorSet&,
//                                            const MachineGrid&)
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
//   SparseTensor::from_parts, so ExecResult / Stats are drop-in.
#include <algorithm>
#include <cstring>
#include <map>
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

struct Ctx {
  spd_context* h = nullptr;
  Ctx() { check(spd_context_create(0, nullptr, &h)); }
  ~Ctx() { spd_context_destroy(h); }
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
  const auto& terms = plan.stmt.terms;
  const auto& lhs = plan.stmt.lhs;
  if (terms.size() == 3 && lhs.vars.size() == 2) {
    for (const auto& t : terms)
      if (t.size() != 1 || fmt(t[0].tensor) != "ds") throw ValidationError("unsupported on gpu: " + s);
    return "spadd3";
  }
  if (terms.size() != 1) throw ValidationError("unsupported on gpu: " + s);
  const auto& t = terms[0];
  if (t.size() == 2 && lhs.vars.size() == 1 && fmt(t[0].tensor) == "ds" && fmt(t[1].tensor) == "d")
    return "spmv";
  if (t.size() == 2 && lhs.vars.size() == 2 && fmt(t[0].tensor) == "ds" && fmt(t[1].tensor) == "dd" &&
      fmt(lhs.tensor) == "dd")
    return "spmm";
  if (t.size() == 3 && fmt(t[0].tensor) == "ds" && fmt(lhs.tensor) == "ds") return "sddmm";
  const bool csf = fmt(t[0].tensor) == "dss" || fmt(t[0].tensor) == "sss";
  if (t.size() == 2 && csf && fmt(t[1].tensor) == "d") return "spttv";
  if (t.size() == 3 && csf && fmt(lhs.tensor) == "dd") return "spmttkrp";
  throw ValidationError("unsupported on gpu: " + s);
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
                           const std::string& kernel) {
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
  r.stats.workers = machine.total_workers();
  r.stats.per_worker.resize(r.stats.workers);
  for (auto& w : r.stats.per_worker)
    for (const auto& nm : plan.stmt.tensor_names()) w.bytes_by_tensor[nm] = 0;
  const int kinds[2] = {SPD_DENSE, SPD_DENSE}, order[2] = {0, 1};
  // column slab [lo, lo + w) of a dense rows x N factor, uploaded contiguous
  auto slab_of = [&](const SparseTensor& F, int64_t lo, int64_t w, DevTensor& dst) {
    const int64_t rows = F.dims()[0];
    const std::vector<double>& fv = F.vals().scalar_values();
    std::vector<double> fy(static_cast<size_t>(rows * w));
    for (int64_t k = 0; k < rows; k++)
      for (int64_t j = 0; j < w; j++) fy[k * w + j] = fv[k * N + lo + j];
    const int64_t dims[2] = {rows, w};
    check(spd_tensor_upload(ctx.h, 2, dims, kinds, order, nullptr, nullptr, fy.data(), &dst.h));
  };
  for (int64_t y = 0; y < ly.pieces; y++) {
    const CoordRange& slab = ly.color_bounds[y];
    const int64_t w = slab.empty() ? 0 : slab.hi - slab.lo + 1;
  std::vector<int64_t> work(lx.pieces, 0);
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
      for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < w; j++) out[i * N + slab.lo + j] = ay[i * w + j];
    }
    for (int64_t x = 0; x < lx.pieces; x++) {
      std::vector<int64_t> coords(machine.rank(), 0);
      coords[machine.dim_index(lx.machine_dim)] = x;
      coords[machine.dim_index(ly.machine_dim)] = y;
      r.stats.per_worker[machine.worker_id(coords)].work = work[x];
    }
  }
  int64_t total = 0, mx = 0;
  for (const auto& w : r.stats.per_worker) total += w.work, mx = std::max(mx, w.work);
  r.stats.imbalance = total == 0 ? 1.0 : (double)mx * (double)r.stats.workers / (double)total;
  r.stats.combines = 0;
  const SparseTensor& outstub = tensors.at(out_name);
  std::vector<LevelStorage> levels;
  for (int l = 0; l < outstub.num_levels(); l++) levels.push_back(outstub.level(l));
  r.output = SparseTensor::from_parts(od, plan.formats.at(out_name), std::move(levels), std::move(out));
  return r;
}

ExecResult execute_gpu(const Plan& plan, const TensorSet& tensors, const MachineGrid& machine) {
  if (plan.loops.size() == 2) {
    const std::string k = kernel_of(plan);
    if (k == "spmm" || k == "spmttkrp") return execute_batched(plan, tensors, machine, k);
  }
  if (plan.loops.size() != 1)
    throw ValidationError("unsupported on gpu: one distributed loop, or the batched two-loop SpMM / SpMTTKRP");
  const PlanLoop& loop = plan.loops[0];
  const std::string kernel = kernel_of(plan);
  const auto& terms = plan.stmt.terms;
  const std::string out_name = plan.stmt.lhs.tensor;
  const std::string b_name = terms[0][0].tensor;
  const SparseTensor& Bt = tensors.at(b_name);

  Ctx ctx;
  DevTensor B;
  upload(ctx, Bt, B);
  std::vector<spd_color> cols(loop.pieces);
  if (loop.position_space)
    check(spd_partition_nonzero(ctx.h, B.h, loop.split_level, loop.pieces, cols.data()));
  else
    check(spd_partition_universe(ctx.h, B.h, loop.pieces, cols.data()));
  for (int64_t c = 0; c < loop.pieces; c++) {  // the GPU's partition must be the planner's
    const CoordRange& want = loop.color_bounds[c];
    bool same = cols[c].color.lo == want.lo && cols[c].color.hi == want.hi;
    bool both_empty = cols[c].color.lo > cols[c].color.hi && want.empty();
    if (!same && !both_empty) throw std::logic_error("gpu partition differs from plan() colour bounds");
  }

  spd_stats st{};
  const std::vector<int64_t>& od = plan.dims.at(out_name);
  SparseTensor out;

  // Operands and the output buffer.
  std::map<std::string, DevTensor> dev;
  for (const auto& term : terms)
    for (const auto& a : term)
      if (a.tensor != b_name && !dev.count(a.tensor)) upload(ctx, tensors.at(a.tensor), dev[a.tensor]);
  const SparseTensor& outstub = tensors.at(out_name);
  DevTensor outbuf;
  upload(ctx, outstub, outbuf);  // dense: zeros sized like the output; sparse: B's pattern reuse
  double* outp = const_cast<double*>(dense_vals_dev(outbuf.h));

  if (kernel == "spmv") {
    const std::string c = terms[0][1].tensor;
    check(spd_spmv(ctx.h, B.h, dense_vals_dev(dev[c].h), outp, 0, loop.pieces, &st));
  } else if (kernel == "spmm") {
    const std::string c = terms[0][1].tensor;
    check(spd_spmm(ctx.h, B.h, dense_vals_dev(dev[c].h), od[1], outp, 0, loop.pieces, &st));
  } else if (kernel == "sddmm") {
    const SparseTensor& Ct = tensors.at(terms[0][1].tensor);
    const SparseTensor& Dt = tensors.at(terms[0][2].tensor);
    int64_t K = Ct.dims()[1];
    bool jmajor = Dt.format().mode_order[0] == 1;
    check(spd_sddmm(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h),
                    dense_vals_dev(dev[terms[0][2].tensor].h), K, jmajor ? 1 : Dt.dims()[1],
                    jmajor ? K : 1, outp, 0, loop.pieces, &st));
  } else if (kernel == "spttv") {
    check(spd_spttv(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h), outp, 0, loop.pieces, &st));
  } else if (kernel == "spmttkrp") {
    check(spd_spmttkrp(ctx.h, B.h, dense_vals_dev(dev[terms[0][1].tensor].h),
                       dense_vals_dev(dev[terms[0][2].tensor].h), od[1], outp, 0, loop.pieces, &st));
  } else {  // spadd3: two-phase assembly on the GPU
    spd_tensor* A = nullptr;
    check(spd_spadd3(ctx.h, B.h, dev[terms[1][0].tensor].h, dev[terms[2][0].tensor].h, &A, 0,
                     loop.pieces, &st));
    DevTensor Ah;
    Ah.h = A;
    int64_t par = 0, nnz = 0;
    int k;
    check(spd_tensor_level(A, 1, &k, &par, &nnz));
    std::vector<CoordRange> pos(par);
    std::vector<int64_t> crd(nnz);
    std::vector<double> vals(nnz);
    check(spd_tensor_download_level(A, 1, reinterpret_cast<int64_t*>(pos.data()), crd.data()));
    check(spd_tensor_download_vals(A, vals.data()));
    std::vector<LevelStorage> levels{std::get<DenseLevel>(Bt.level(0)),
                                     CompressedLevel{Region::ranges(IndexSpace({par}), std::move(pos), nnz),
                                                     Region::coordinates(IndexSpace({nnz}), std::move(crd))}};
    out = SparseTensor::from_parts(od, plan.formats.at(out_name), std::move(levels), std::move(vals));
  }
  if (kernel != "spadd3") {
    std::vector<double> vals(outstub.leaf_count());
    check(spd_tensor_download_vals(outbuf.h, vals.data()));
    std::vector<LevelStorage> levels;
    for (int l = 0; l < outstub.num_levels(); l++) levels.push_back(outstub.level(l));
    out = SparseTensor::from_parts(od, plan.formats.at(out_name), std::move(levels), std::move(vals));
  }

  ExecResult r{std::move(out), Stats{}};
  r.stats.workers = machine.total_workers();
  r.stats.per_worker.resize(r.stats.workers);
  std::vector<int64_t> work(loop.pieces);
  check(spd_last_work(ctx.h, work.data(), loop.pieces));
  for (int64_t c = 0; c < loop.pieces; c++) {
    r.stats.per_worker[c].work = work[c];
    for (const auto& n : plan.stmt.tensor_names()) r.stats.per_worker[c].bytes_by_tensor[n] = 0;
  }
  r.stats.imbalance = st.imbalance;
  r.stats.combines = st.combines;
  return r;
}

}  // namespace dspar_gpu
