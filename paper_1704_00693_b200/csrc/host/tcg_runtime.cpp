#include "tcg_runtime.hpp"

#include <chrono>
#include <cstdio>

#include "../kernels/tc_bodies.h"

namespace tcg {

namespace {

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Raised when a (sub)chain's windows cannot fit in shared memory; the runtime
// then splits the chain into consecutive sub-chains (each executes exactly as
// the reference would, so results are unchanged).
struct WindowOverflow : PlanError {
  explicit WindowOverflow(const std::string& m) : PlanError(m) {}
};

LoopChain slice(const LoopChain& c, size_t a, size_t b) {
  LoopChain s;
  s.dim = c.dim;
  s.stencils = c.stencils;
  for (size_t i = a; i < b; ++i) {
    s.loops.push_back(c.loops[i]);
    s.loops.back().loop_id = static_cast<int32_t>(i - a);
  }
  return s;
}

}  // namespace

int64_t ExecutionReport::total_points() const {
  int64_t n = 0;
  for (const auto& s : loops) n += s.points;
  return n;
}
int64_t ExecutionReport::total_bytes_moved() const {
  int64_t n = 0;
  for (const auto& s : loops) n += s.bytes_moved;
  return n;
}

std::string ExecutionReport::to_text() const {
  // key=value lines, executor.cpp:321-366, plus the GPU plan shape.
  std::string o;
  char b[192];
  auto kv = [&](const char* k, const std::string& v) { o += std::string(k) + "=" + v + "\n"; };
  kv("tiled", tiled ? "1" : "0");
  kv("distributed", distributed ? "1" : "0");
  if (tiled) {
    std::string ts, sk, gr;
    for (int d = 0; d < dim; ++d) {
      ts += (d ? "," : "") + std::to_string(tile_sizes[d]);
      sk += (d ? "," : "") + std::to_string(max_skew[d]);
      gr += (d ? "," : "") + std::to_string(cta_grid[d]);
    }
    kv("tile_sizes", ts);
    kv("max_skew", sk);
    kv("plan_cache_hit", plan_cache_hit ? "1" : "0");
    kv("cta_grid", gr);
    kv("ctas", std::to_string(ctas));
    kv("subchains", std::to_string(subchains));
    kv("computed_points", std::to_string(computed_points));
  }
  kv("tiles", std::to_string(tiles_executed));
  kv("loops", std::to_string(loops.size()));
  kv("points", std::to_string(total_points()));
  kv("bytes_moved", std::to_string(total_bytes_moved()));
  kv("plan_constructions", std::to_string(plan_constructions));
  std::snprintf(b, sizeof b, "%.6f", plan_seconds);
  kv("plan_seconds", b);
  std::snprintf(b, sizeof b, "%.6f", exec_seconds);
  kv("exec_seconds", b);
  std::snprintf(b, sizeof b, "%.6f", total_seconds);
  kv("total_seconds", b);
  kv("launches", std::to_string(launches));
  if (distributed) {
    kv("halo_messages", std::to_string(halo_messages));
    kv("halo_bytes", std::to_string(halo_bytes));
    kv("halo_exchanges", std::to_string(halo_exchanges));
  }
  for (const auto& s : loops) {
    std::snprintf(b, sizeof b, "loop%d_points=%lld\nloop%d_bytes=%lld\n", s.loop_id, static_cast<long long>(s.points),
                  s.loop_id, static_cast<long long>(s.bytes_moved));
    o += b;
  }
  return o;
}

Runtime::Runtime(int dim, RuntimeConfig cfg) : dim_(dim), cfg_(cfg) {
  if (dim < 1 || dim > kMaxDims) throw InvalidArgument("Runtime: block dim must be 1, 2, or 3");
  if (cfg_.threads < 1) throw InvalidArgument("Runtime: threads must be >= 1");
  if (cfg_.skew_allowance < 0) throw InvalidArgument("Runtime: skew_allowance must be >= 0");
}

Runtime::~Runtime() = default;

DeviceExec& Runtime::device() {
  if (!dev_) dev_ = std::make_unique<DeviceExec>();
  return *dev_;
}

void Runtime::ensure_fields() {
  DeviceExec& d = device();
  for (FieldRec& f : fields_)
    if (f.dev < 0) f.dev = d.add_field(f.alloc);
}

std::vector<FieldGeom> Runtime::field_geoms() const {
  std::vector<FieldGeom> g;
  for (const FieldRec& f : fields_) g.push_back(FieldGeom{f.alloc});
  return g;
}

StencilId Runtime::declare_stencil(const std::string&, std::vector<Point> offsets) {
  Stencil s(dim_, std::move(offsets));
  max_reach_ = std::max(max_reach_, s.max_abs_offset());
  stencils_.push_back(std::move(s));
  return static_cast<StencilId>(stencils_.size() - 1);
}

DatasetId Runtime::declare_field(const std::string& name, const Range& logical, int elem_bytes) {
  if (logical.dim() != dim_) throw InvalidArgument("declare_field: range dim does not match block");
  if (logical.empty()) throw InvalidArgument("declare_field: empty logical range");
  if (elem_bytes != 8) throw InvalidArgument("declare_field: the B200 executor stores fp64 (elem_bytes = 8)");
  FieldRec f;
  f.name = name;
  f.logical = logical;
  f.pad = max_reach_ + cfg_.skew_allowance;  // runtime.cpp:30
  f.alloc = Range(dim_);
  for (int d = 0; d < dim_; ++d) f.alloc.set(d, logical.start(d) - f.pad, logical.end(d) + f.pad);
  fields_.push_back(f);
  if (dev_) fields_.back().dev = dev_->add_field(f.alloc);
  return static_cast<DatasetId>(fields_.size() - 1);
}

ReductionHandle Runtime::par_loop(KernelHandle kernel, const Range& range, std::vector<ArgSpec> args,
                                  std::optional<ReduceOp> reduction) {
  if (kernel.fn.body < 0) throw InvalidArgument("par_loop: kernel has no body");
  if (!tcb::body_known(kernel.fn.body))
    throw InvalidArgument("par_loop: kernel body " + std::to_string(kernel.fn.body) +
                          " is not in the device registry (no CPU fallback)");
  if (kernel.id < 0) throw InvalidArgument("par_loop: kernel id must be >= 0");
  if (range.dim() != dim_) throw InvalidArgument("par_loop: range dim does not match block");
  if (args.size() > static_cast<size_t>(kMaxArgs)) throw InvalidArgument("par_loop: more than 12 arguments");
  for (const ArgSpec& a : args) {
    if (a.dataset < 0 || static_cast<size_t>(a.dataset) >= fields_.size())
      throw InvalidArgument("par_loop: unknown dataset id " + std::to_string(a.dataset));
    if (a.stencil < 0 || static_cast<size_t>(a.stencil) >= stencils_.size())
      throw InvalidArgument("par_loop: unknown stencil id " + std::to_string(a.stencil));
    if (mode_writes(a.mode) && !stencils_[static_cast<size_t>(a.stencil)].is_identity())
      throw InvalidArgument("par_loop: dataset " + fields_[static_cast<size_t>(a.dataset)].name +
                            " written through a multi-point stencil; writes must land on the iteration point");
  }
  // Same-loop read at a non-zero offset of a written dataset races under
  // per-point parallelism when the shifted range meets the range
  // (runtime.cpp:56-76).
  for (const ArgSpec& r : args) {
    if (!mode_reads(r.mode)) continue;
    bool written = false;
    for (const ArgSpec& w : args) written = written || (w.dataset == r.dataset && mode_writes(w.mode));
    if (!written) continue;
    for (const Point& off : stencils_[static_cast<size_t>(r.stencil)].points()) {
      if (off == Point{0, 0, 0}) continue;
      if (!range.dilated(off, off).intersect(range).empty())
        throw InvalidArgument("par_loop: kernel reads dataset " + fields_[static_cast<size_t>(r.dataset)].name +
                              " at offset (" + std::to_string(off[0]) + "," + std::to_string(off[1]) + "," +
                              std::to_string(off[2]) +
                              ") while writing it over an overlapping range; this races under per-point parallelism");
    }
  }
  LoopRecord rec;
  rec.loop_id = static_cast<int32_t>(pending_.size());
  rec.kernel = std::move(kernel);
  rec.range = range;
  rec.args = std::move(args);
  ReductionHandle h;
  if (reduction) {
    h.id = static_cast<int32_t>(slots_.size());
    slots_.push_back(Slot{*reduction, 0.0, false, false});
    rec.reduction = ReductionSpec{*reduction, h};
  }
  pending_.push_back(std::move(rec));
  return h;
}

LoopChain Runtime::take_pending() {
  LoopChain c;
  c.dim = dim_;
  c.loops = std::move(pending_);
  c.stencils = stencils_;
  pending_.clear();
  return c;
}

ExecutionReport Runtime::flush(const ExecMode& mode) {
  if (pending_.empty()) {
    last_report_ = ExecutionReport{};
    return last_report_;
  }
  return execute_chain(take_pending(), mode);
}

DevChain Runtime::lower(const LoopChain& chain, std::vector<ReductionHandle>& handles) const {
  DevChain dc;
  dc.dim = chain.dim;
  std::vector<int> slot;
  for (const LoopRecord& lp : chain.loops) {
    DevLoop d{};
    d.body = lp.kernel.fn.body;
    d.nargs = static_cast<int32_t>(lp.args.size());
    d.red = -1;
    if (lp.reduction) {
      d.red = dc.nred++;
      d.red_op = static_cast<int32_t>(lp.reduction->op);
      dc.red_op.push_back(d.red_op);
      handles.push_back(lp.reduction->handle);
    }
    d.param_off = static_cast<int32_t>(dc.params.size());
    d.nparams = static_cast<int32_t>(lp.kernel.fn.params.size());
    dc.params.insert(dc.params.end(), lp.kernel.fn.params.begin(), lp.kernel.fn.params.end());
    for (int k = 0; k < 3; ++k) {
      d.range[k][0] = k < chain.dim ? lp.range.start(k) : 0;
      d.range[k][1] = k < chain.dim ? lp.range.end(k) : 1;
    }
    for (size_t a = 0; a < lp.args.size(); ++a) {
      const DatasetId ds = lp.args[a].dataset;
      if (ds >= static_cast<DatasetId>(slot.size())) slot.resize(static_cast<size_t>(ds) + 1, -1);
      if (slot[static_cast<size_t>(ds)] < 0) {
        slot[static_cast<size_t>(ds)] = static_cast<int>(dc.dat_ids.size());
        dc.dat_ids.push_back(ds);
      }
      d.args[a] = DevArg{slot[static_cast<size_t>(ds)], lp.args[a].stencil, static_cast<int32_t>(lp.args[a].mode), 0};
    }
    dc.loops.push_back(d);
  }
  for (const Stencil& s : chain.stencils) {
    dc.st_start.push_back(static_cast<int32_t>(dc.st_pts.size() / 3));
    dc.st_npts.push_back(static_cast<int32_t>(s.points().size()));
    for (const Point& p : s.points())
      for (int k = 0; k < 3; ++k) dc.st_pts.push_back(static_cast<int32_t>(p[k]));
  }
  // Map slots to device field indices for the executors.
  for (DatasetId& ds : dc.dat_ids) ds = fields_[static_cast<size_t>(ds)].dev;
  return dc;
}

void Runtime::store(const std::vector<ReductionHandle>& handles, const double* vals) {
  for (size_t i = 0; i < handles.size(); ++i) {
    if (!handles[i].valid() || static_cast<size_t>(handles[i].id) >= slots_.size()) continue;
    Slot& s = slots_[static_cast<size_t>(handles[i].id)];
    s.value = vals[i];
    s.ready = true;
  }
}

void Runtime::run_tiled(const LoopChain& chain, const ExecMode& mode, ExecutionReport& rep) {
  DeviceExec& dev = device();
  const int s = chain.dim - 1;
  GpuTileChoice choice;
  if (mode.kind == ExecMode::Kind::Tiled) {
    for (int d = 0; d < chain.dim; ++d) {
      if (d == s)
        choice.stream_tile = std::max<int64_t>(1, mode.tile_sizes[d]);
      else
        choice.block[d] = std::max<int64_t>(1, mode.tile_sizes[d]);
    }
  }
  choice.stream_segments = cfg_.stream_segments;
  if (const char* e = std::getenv("TCG_PREFETCH")) choice.prefetch = std::atoi(e);
  if (const char* e = std::getenv("TCG_CTAS_PER_SM")) choice.ctas_per_sm = std::atoi(e);
  const std::vector<FieldGeom> geoms = field_geoms();
  const uint64_t sig = chain.signature();
  rep.plan_cache_hit = true;

  // Plan of the sub-chain [begin, begin+len); nullptr when its windows do not
  // fit in shared memory. Cached per (signature, offset, length, mode).
  auto plan_for = [&](size_t begin, size_t len) -> std::shared_ptr<const GpuTiledPlan> {
    const auto key = std::make_tuple(sig ^ (static_cast<uint64_t>(begin) * 0x9e3779b97f4a7c15ull) ^
                                         (static_cast<uint64_t>(len) << 48),
                                     mode.tile_sizes[0] * 4 + static_cast<int64_t>(mode.kind), mode.tile_sizes[1],
                                     mode.tile_sizes[2], cfg_.stream_segments);
    auto it = gpu_plans_.find(key);
    if (it != gpu_plans_.end()) return it->second;
    rep.plan_cache_hit = false;
    const LoopChain sub = slice(chain, begin, begin + len);
    int nred = 0;
    for (const auto& l : sub.loops) nred += l.reduction ? 1 : 0;
    std::shared_ptr<const GpuTiledPlan> gp;
    try {
      const int nl = static_cast<int>(sub.size());
      const WindowBudget budget = [&](int k) { return dev.window_budget_doubles(nl, nred, k); };
      auto p = std::make_shared<GpuTiledPlan>(build_gpu_tiled_plan(sub, geoms, choice, budget, dev.info().num_sms));
      ++gpu_plan_builds_;
      ++rep.plan_constructions;
      rep.plan_seconds += p->build_seconds;
      gp = p;
    } catch (const PlanError& e) {
      const std::string m = e.what();
      if (m.find("no CTA tiling fits") == std::string::npos && m.find("more than") == std::string::npos) throw;
    }
    gpu_plans_[key] = gp;
    return gp;
  };

  size_t begin = 0;
  while (begin < chain.size()) {
    size_t len = chain.size() - begin;
    std::shared_ptr<const GpuTiledPlan> gp = plan_for(begin, len);
    if (!gp) {
      // Longest fitting prefix: fit is monotone in length for a fixed start.
      size_t lo = 0, hi = len;
      while (hi - lo > 1) {
        const size_t mid = (lo + hi) / 2;
        if (plan_for(begin, mid))
          lo = mid;
        else
          hi = mid;
      }
      if (lo == 0) throw PlanError("tiled executor: a single loop's windows do not fit in shared memory");
      len = lo;
      gp = plan_for(begin, len);
    }
    const LoopChain sub = slice(chain, begin, begin + len);
    std::vector<ReductionHandle> handles;
    DevChain dc = lower(sub, handles);
    double vals[kMaxRed] = {0};
    const uint64_t pkey = reinterpret_cast<uint64_t>(gp.get());
    dev.run_tiled(dc, *gp, pkey, vals);
    store(handles, vals);
    last_gpu_plan_ = gp;
    rep.ctas += static_cast<int64_t>(gp->ctas.size());
    rep.computed_points += gp->computed_points;
    for (const DevCta& c : gp->ctas) rep.tiles_executed += c.ntiles;
    for (int d = 0; d < chain.dim; ++d) {
      rep.max_skew[d] = std::max(rep.max_skew[d], gp->max_skew[d]);
      rep.cta_grid[d] = gp->grid[d];
      rep.tile_sizes[d] = d == s ? gp->stream_tile : gp->block[d];
    }
    ++rep.subchains;
    begin += sub.size();
  }
}

ExecutionReport Runtime::execute_chain(LoopChain chain, const ExecMode& mode) {
  const auto t0 = std::chrono::steady_clock::now();
  ExecutionReport rep;
  rep.dim = chain.dim;
  for (const LoopRecord& lp : chain.loops)
    rep.loops.push_back(LoopExecStats{lp.loop_id, lp.range.volume(), estimate_bytes_moved(lp, lp.range)});
  ensure_fields();
  DeviceExec& dev = device();
  const int64_t l0 = dev.launches();
  if (mode.kind == ExecMode::Kind::Untiled) {
    // Pad sufficiency of untiled execution: every access of the recorded
    // ranges must stay inside its allocation (the reference's checked
    // accessor would throw AccessError at run time, kernel_ctx.hpp:58-73).
    for (const LoopRecord& lp : chain.loops) {
      if (lp.range.empty()) continue;
      for (const ArgSpec& a : lp.args) {
        const Stencil& st = chain.stencil(a.stencil);
        Point lo{0, 0, 0}, hi{0, 0, 0};
        for (int d = 0; d < chain.dim; ++d) {
          lo[d] = mode_reads(a.mode) ? std::min<int64_t>(st.min_offset(d), 0) : 0;
          hi[d] = mode_reads(a.mode) ? std::max<int64_t>(st.max_offset(d), 0) : 0;
        }
        const Range touched = lp.range.dilated(lo, hi);
        if (!fields_[static_cast<size_t>(a.dataset)].alloc.contains(touched))
          throw AccessError("loop k" + std::to_string(lp.kernel.id) + " (id " + std::to_string(lp.loop_id) +
                            "), dataset " + fields_[static_cast<size_t>(a.dataset)].name + ": access over " +
                            touched.to_string() + " outside allocated extent " +
                            fields_[static_cast<size_t>(a.dataset)].alloc.to_string());
      }
    }
    std::vector<ReductionHandle> handles;
    DevChain dc = lower(chain, handles);
    std::vector<double> vals(static_cast<size_t>(std::max(1, dc.nred)));
    dev.run_untiled(dc, vals.data());
    store(handles, vals.data());
    rep.tiles_executed = 1;
  } else {
    rep.tiled = true;
    run_tiled(chain, mode, rep);
  }
  rep.launches = dev.launches() - l0;
  rep.exec_seconds = secs_since(t0) - rep.plan_seconds;
  rep.total_seconds = secs_since(t0);
  last_report_ = rep;
  return rep;
}

double Runtime::fetch_reduction(ReductionHandle h) {
  if (!h.valid() || static_cast<size_t>(h.id) >= slots_.size())
    throw InvalidArgument("fetch_reduction: unknown handle");
  Slot& slot = slots_[static_cast<size_t>(h.id)];
  if (slot.consumed) throw InvalidArgument("fetch_reduction: handle already fetched");
  if (!slot.ready) {
    size_t k = pending_.size();
    for (size_t i = 0; i < pending_.size(); ++i)
      if (pending_[i].reduction && pending_[i].reduction->handle.id == h.id) k = i;
    if (k == pending_.size()) throw InvalidArgument("fetch_reduction: reducing loop neither pending nor executed");
    if (cfg_.flush_whole_queue_on_fetch) {
      flush();
    } else {
      std::vector<LoopRecord> suffix(pending_.begin() + static_cast<std::ptrdiff_t>(k) + 1, pending_.end());
      pending_.resize(k + 1);
      execute_chain(take_pending(), default_mode_);
      for (size_t i = 0; i < suffix.size(); ++i) suffix[i].loop_id = static_cast<int32_t>(i);
      pending_ = std::move(suffix);
    }
  }
  if (!slot.ready) throw PlanError("fetch_reduction: flush did not produce the value");
  slot.consumed = true;
  return slot.value;
}

double Runtime::get(DatasetId ds, const Point& p) {
  flush();
  ensure_fields();
  return device().get_point(fields_.at(static_cast<size_t>(ds)).dev, p);
}

void Runtime::put(DatasetId ds, const Point& p, double v) {
  flush();
  ensure_fields();
  device().put_point(fields_.at(static_cast<size_t>(ds)).dev, p, v);
}

void Runtime::upload(DatasetId ds, const double* host) {
  flush();
  ensure_fields();
  device().upload(fields_.at(static_cast<size_t>(ds)).dev, host);
}

void Runtime::download(DatasetId ds, double* host) {
  flush();
  ensure_fields();
  device().download(fields_.at(static_cast<size_t>(ds)).dev, host);
}

void Runtime::fill_logical(DatasetId ds, double v) {
  flush();
  ensure_fields();
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  std::vector<double> h(static_cast<size_t>(f.alloc.volume()));
  device().download(f.dev, h.data());
  const int64_t nx = f.alloc.extent(0);
  const int64_t ny = dim_ > 1 ? f.alloc.extent(1) : 1;
  for (int64_t z = dim_ > 2 ? f.logical.start(2) : 0; z < (dim_ > 2 ? f.logical.end(2) : 1); ++z)
    for (int64_t y = dim_ > 1 ? f.logical.start(1) : 0; y < (dim_ > 1 ? f.logical.end(1) : 1); ++y)
      for (int64_t x = f.logical.start(0); x < f.logical.end(0); ++x) {
        const int64_t i = (x - f.alloc.start(0)) + nx * ((dim_ > 1 ? y - f.alloc.start(1) : 0) +
                                                          ny * (dim_ > 2 ? z - f.alloc.start(2) : 0));
        h[static_cast<size_t>(i)] = v;
      }
  device().upload(f.dev, h.data());
}

}  // namespace tcg
