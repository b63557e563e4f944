#include "tcg_runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <limits>

#include "../kernels/tc_bodies.h"
#include "tcg_jit.hpp"

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

int64_t chain_points(const LoopChain& c) {
  int64_t n = 0;
  for (const LoopRecord& lp : c.loops) n += lp.range.volume();
  return n;
}

// Host-side probe of a registered body against a loop's declared arguments:
// the body runs once on this accessor, which applies KernelCtx's checks
// (kernel_ctx.hpp:58-89: argument index, access mode, offset in the declared
// stencil, contribute() needs a reduction) and records the first violation.
// The device accessors carry no checks in the default library, so a
// mismatched declaration is refused here, at enqueue time.
struct ProbeAcc {
  const std::vector<ArgSpec>& args;
  const std::vector<Stencil>& stencils;
  bool red;
  mutable std::string err;
  void fail(int a, int dx, int dy, int dz, const char* why) const {
    if (!err.empty()) return;
    err = "arg " + std::to_string(a) + " offset (" + std::to_string(dx) + "," + std::to_string(dy) + "," +
          std::to_string(dz) + "): " + why;
  }
  bool arg_ok(int a) const {
    if (a >= 0 && static_cast<size_t>(a) < args.size()) return true;
    fail(a, 0, 0, 0, "argument index beyond the declared arguments");
    return false;
  }
  double read(int a, int dx, int dy, int dz) const {
    if (!arg_ok(a)) return 1.0;
    const ArgSpec& s = args[static_cast<size_t>(a)];
    if (!mode_reads(s.mode)) fail(a, dx, dy, dz, "read through write-only arg");
    else if (!stencils[static_cast<size_t>(s.stencil)].has_offset(dx, dy, dz)) fail(a, dx, dy, dz, "offset not in declared stencil");
    return 1.0;
  }
  void write(int a, double) const {
    if (arg_ok(a) && !mode_writes(args[static_cast<size_t>(a)].mode)) fail(a, 0, 0, 0, "write through read-only arg");
  }
  void increment(int a, double) const {
    if (!arg_ok(a)) return;
    const AccessMode m = args[static_cast<size_t>(a)].mode;
    if (!mode_writes(m) || !mode_reads(m)) fail(a, 0, 0, 0, "increment needs a readwrite/increment arg");
  }
  void contribute(double) const {
    if (!red && err.empty()) err = "contribute() without a declared reduction";
  }
  long long x() const { return 0; }
  long long y() const { return 0; }
  long long z() const { return 0; }
  int nargs() const { return static_cast<int>(args.size()); }
  int mode(int a) const { return arg_ok(a) ? static_cast<int>(args[static_cast<size_t>(a)].mode) : 0; }
  int npts(int a) const {
    return arg_ok(a) ? static_cast<int>(stencils[static_cast<size_t>(args[static_cast<size_t>(a)].stencil)].points().size()) : 0;
  }
  int pt(int a, int j, int d) const {
    return static_cast<int>(stencils[static_cast<size_t>(args[static_cast<size_t>(a)].stencil)].points()[static_cast<size_t>(j)][static_cast<size_t>(d)]);
  }
  bool reduces() const { return red; }
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
  kv("executor", executor);
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
    if (executor == "tiled") kv("grid_barriers", std::to_string(l2_syncs));
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
  if (distributed || halo_exchanges > 0) {
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
  if (const char* e = std::getenv("TCG_POISON_HALOS")) poison_ = std::atoi(e) != 0;
  if (dim < 1 || dim > kMaxDims) throw InvalidArgument("Runtime: block dim must be 1, 2, or 3");
  if (cfg_.threads < 1) throw InvalidArgument("Runtime: threads must be >= 1");
  if (cfg_.skew_allowance < 0) throw InvalidArgument("Runtime: skew_allowance must be >= 0");
  if (const char* e = std::getenv("TCG_AUTO_CANDS")) {
    auto_cands_ = 0;
    for (const char* c = e; *c; ++c)
      if (*c >= '0' && *c < '0' + kCand) auto_cands_ |= 1u << (*c - '0');
    auto_cands_ |= 2u;  // untiled always runs
  }
  // tiled_auto decisions persisted across processes (like a library autotune
  // cache): "signature ms_l2 ms_untiled ms_windowed ms_stream fits_mask" per line.
  if (const char* path = std::getenv("TCG_AUTOTUNE_FILE")) {
    autotune_file_ = path;
    if (FILE* f = std::fopen(path, "r")) {
      unsigned long long sig = 0;
      float m0 = 0, m1 = 0, m2 = 0, m3 = 0;
      int fits = 0;
      while (std::fscanf(f, "%llx %f %f %f %f %d", &sig, &m0, &m1, &m2, &m3, &fits) == 6) {
        AutoStat& a = auto_[static_cast<uint64_t>(sig)];
        const float m[kCand] = {m0, m1, m2, m3};
        for (int c = 0; c < kCand; ++c) {
          a.runs[c] = kAutoRuns;
          a.ms[c] = m[c];
          a.fits[c] = ((fits >> c) & 1) != 0;
        }
        a.saved = true;
      }
      std::fclose(f);
    }
  }
}

int Runtime::AutoStat::best() const {
  int b = 1;  // untiled always runs
  for (int c = 0; c < kCand; ++c)
    if (fits[c] && ms[c] < ms[b]) b = c;
  return b;
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
  // Body signature against the declaration (once per distinct declaration).
  {
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { key = (key ^ v) * 1099511628211ull; };
    mix(static_cast<uint64_t>(kernel.fn.body));
    mix(args.size());
    mix(reduction ? 1 : 0);
    mix(kernel.fn.params.size());
    for (const ArgSpec& a : args) mix((static_cast<uint64_t>(a.stencil) << 8) | static_cast<uint64_t>(a.mode));
    mix(stencils_.size());
    static const bool skip_probe = [] {
      const char* e = std::getenv("TCG_SKIP_BODY_PROBE");  // test hook: lets the checked device build see the fault
      return e && *e == '1';
    }();
    if (!skip_probe && !body_sig_ok_.count(key)) {
      if (args.empty()) throw InvalidArgument("par_loop: kernel " + kernel.name + " declares no arguments");
      ProbeAcc probe{args, stencils_, reduction.has_value(), {}};
      std::vector<double> prm(kernel.fn.params.begin(), kernel.fn.params.end());
      prm.resize(std::max<size_t>(prm.size(), 16), 1.0);
      tcb::run_body(kernel.fn.body, probe, prm.data());
      if (!probe.err.empty())
        throw AccessError("par_loop: kernel " + kernel.name + " (body " + std::to_string(kernel.fn.body) +
                          ") does not match its declared arguments: " + probe.err);
      body_sig_ok_.insert(key);
    }
  }
  if (recording_) {
    RecordedCall rc;
    rc.kernel = kernel;
    rc.range = range;
    rc.args = args;
    rc.reduction = reduction;
    record_cur_.push_back(std::move(rc));
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

void Runtime::set_reduction_order(int workers) {
  if (workers < 0 || workers > 1024) throw InvalidArgument("set_reduction_order: workers must be in [0, 1024]");
  flush();
  red_workers_ = workers;
  if (dev_) dev_->set_reduction_workers(workers);
}

void Runtime::set_periodic_domain(bool v) {
  flush();
  if (dist_) throw InvalidArgument("set_periodic_domain: call before the first distributed flush");
  periodic_domain_ = v;
}

void Runtime::record_begin() {
  recording_ = true;
  record_cur_.clear();
}

int Runtime::record_end() {
  if (!recording_) throw InvalidArgument("record_end: no recording in progress");
  recording_ = false;
  recorded_.push_back(std::move(record_cur_));
  record_cur_.clear();
  return static_cast<int>(recorded_.size()) - 1;
}

std::vector<ReductionHandle> Runtime::replay(int id, const double* params, size_t nparams) {
  if (id < 0 || static_cast<size_t>(id) >= recorded_.size()) throw InvalidArgument("replay: unknown recording");
  if (recording_) throw InvalidArgument("replay: a recording is in progress");
  std::vector<ReductionHandle> out;
  size_t pi = 0;
  if (params) {  // checked before anything is enqueued
    size_t need = 0;
    for (const RecordedCall& rc : recorded_[static_cast<size_t>(id)])
      if (!rc.fill) need += rc.kernel.fn.params.size();
    if (need != nparams)
      throw InvalidArgument("replay: the template holds " + std::to_string(need) + " scalar parameters, " +
                            std::to_string(nparams) + " given");
  }
  // The template is copied call by call: par_loop consumes its arguments.
  for (size_t i = 0; i < recorded_[static_cast<size_t>(id)].size(); ++i) {
    const RecordedCall& rc = recorded_[static_cast<size_t>(id)][i];
    if (rc.fill) {
      periodic_fill(rc.fill_ds, rc.fill_depth);
      continue;
    }
    KernelHandle k = rc.kernel;
    if (params) {
      if (pi + k.fn.params.size() > nparams) throw InvalidArgument("replay: too few parameter values");
      for (double& v : k.fn.params) v = params[pi++];
    }
    const ReductionHandle h = par_loop(std::move(k), rc.range, rc.args, rc.reduction);
    if (rc.reduction) out.push_back(h);
  }
  if (params && pi != nparams) throw InvalidArgument("replay: too many parameter values");
  return out;
}

LoopChain Runtime::take_pending() {
  LoopChain c;
  c.dim = dim_;
  c.loops = std::move(pending_);
  c.stencils = stencils_;
  c.fills = std::move(fill_marks_);
  pending_.clear();
  fill_marks_.clear();
  return c;
}

ExecutionReport Runtime::flush(const ExecMode& mode) {
  if (pending_.empty() && fill_marks_.empty()) {
    last_report_ = ExecutionReport{};
    return last_report_;
  }
  return execute_chain(take_pending(), mode);
}

DevChain Runtime::lower(const LoopChain& chain, const Target& t) const {
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
  // Map slots to the target's device field indices.
  for (DatasetId& ds : dc.dat_ids) ds = t.dev.at(static_cast<size_t>(ds));
  if (t.masked) {
    dc.masked = true;
    for (int k = 0; k < 3; ++k) {
      dc.mask[k][0] = k < chain.dim ? t.mask.start(k) : 0;
      dc.mask[k][1] = k < chain.dim ? t.mask.end(k) : 1;
    }
  }
  return dc;
}

namespace {
double red_identity_host(int op) { return reduce_identity(static_cast<ReduceOp>(op)); }

std::vector<ReductionHandle> reduction_handles(const LoopChain& chain) {
  std::vector<ReductionHandle> h;
  for (const LoopRecord& lp : chain.loops)
    if (lp.reduction) h.push_back(lp.reduction->handle);
  return h;
}
uint64_t mask_hash(const Runtime&, bool masked, const Range& m, int dim) {
  if (!masked) return 0;
  uint64_t h = 1469598103934665603ull;
  for (int d = 0; d < dim; ++d)
    for (int64_t v : {m.start(d), m.end(d)}) {
      h ^= static_cast<uint64_t>(v);
      h *= 1099511628211ull;
    }
  return h;
}
}  // namespace

void Runtime::store(const std::vector<ReductionHandle>& handles, const double* vals) {
  for (size_t i = 0; i < handles.size(); ++i) {
    if (!handles[i].valid() || static_cast<size_t>(handles[i].id) >= slots_.size()) continue;
    Slot& s = slots_[static_cast<size_t>(handles[i].id)];
    s.value = vals[i];
    s.ready = true;
  }
}

Runtime::Target Runtime::whole_target() const {
  Target t;
  for (const FieldRec& f : fields_) {
    t.dev.push_back(f.dev);
    t.alloc.push_back(f.alloc);
  }
  return t;
}

void Runtime::run_tiled(const LoopChain& chain, const ExecMode& mode, ExecutionReport& rep, const Target& t,
                        std::vector<double>& vals) {
  DeviceExec& dev = device();
  const int s = chain.dim - 1;
  GpuTileChoice choice;
  if (mode.kind == ExecMode::Kind::Windowed) {
    // Explicit sizes are upper bounds; 0 leaves that dimension to the sizer.
    for (int d = 0; d < chain.dim; ++d) {
      if (mode.tile_sizes[d] <= 0) continue;
      if (d == s)
        choice.stream_tile = mode.tile_sizes[d];
      else
        choice.block[d] = mode.tile_sizes[d];
    }
  }
  choice.stream_segments = cfg_.stream_segments;
  if (const char* e = std::getenv("TCG_PREFETCH")) choice.prefetch = std::atoi(e);
  if (const char* e = std::getenv("TCG_CTAS_PER_SM")) choice.ctas_per_sm = std::atoi(e);
  std::vector<FieldGeom> geoms;
  for (const Range& a : t.alloc) geoms.push_back(FieldGeom{a});
  const uint64_t sig = chain.signature() ^ mask_hash(*this, t.masked, t.mask, chain.dim);
  rep.plan_cache_hit = true;

  // Plan of the sub-chain [begin, begin+len); nullptr when its windows do not
  // fit in shared memory. Cached per (signature, offset, length, mode, mask).
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
      if (t.masked) {
        // Reductions count only the target's owned box (execute_plan's
        // reduction_mask); CTA ownership boxes are only used for that.
        for (DevCta& c : p->ctas)
          for (int d = 0; d < chain.dim; ++d) {
            c.own_lo[d] = static_cast<int32_t>(std::max<int64_t>(c.own_lo[d], t.mask.start(d)));
            c.own_hi[d] = static_cast<int32_t>(std::min<int64_t>(c.own_hi[d], t.mask.end(d)));
          }
      }
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

  // Upper bound on loops per windowed sub-chain (0 = as long as fits).
  static const size_t max_loops = [] {
    const char* e = std::getenv("TCG_WIN_MAXLOOPS");
    return e ? static_cast<size_t>(std::max(0, std::atoi(e))) : size_t{0};
  }();
  size_t begin = 0, red_base = 0;
  while (begin < chain.size()) {
    size_t len = chain.size() - begin;
    if (max_loops > 0) len = std::min(len, max_loops);
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
    DevChain dc = lower(sub, t);
    double sv[kMaxRed] = {0};
    const uint64_t pkey = reinterpret_cast<uint64_t>(gp.get());
    dev.run_tiled(dc, *gp, pkey, sv);
    for (int i = 0; i < dc.nred; ++i) vals.at(red_base + static_cast<size_t>(i)) = sv[i];
    red_base += static_cast<size_t>(dc.nred);
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

namespace {
// Access footprint of one (tile, loop) item: per dataset, the box it reads
// (range dilated by the read stencil) and the box it writes.
struct Footprint {
  std::vector<std::pair<DatasetId, Range>> reads, writes;
};
Footprint footprint(const LoopChain& chain, const LoopRecord& lp, const Range& r) {
  Footprint f;
  for (const ArgSpec& a : lp.args) {
    if (mode_reads(a.mode)) {
      const Stencil& st = chain.stencil(a.stencil);
      Point lo{0, 0, 0}, hi{0, 0, 0};
      for (int d = 0; d < chain.dim; ++d) {
        lo[d] = std::min<int64_t>(st.min_offset(d), 0);
        hi[d] = std::max<int64_t>(st.max_offset(d), 0);
      }
      f.reads.emplace_back(a.dataset, r.dilated(lo, hi));
    }
    if (mode_writes(a.mode)) f.writes.emplace_back(a.dataset, r);
  }
  return f;
}
bool overlaps(const std::vector<std::pair<DatasetId, Range>>& a, const std::vector<std::pair<DatasetId, Range>>& b) {
  for (const auto& [da, ra] : a)
    for (const auto& [db, rb] : b)
      if (da == db && !ra.intersect(rb).empty()) return true;
  return false;
}
}  // namespace

// GPU sizer of the L2 executor. Only the slowest dimension is tiled. A tile
// of sub-chain [b, e) touches (ts + skew + 2) slowest-dim slices of every
// dataset of the sub-chain; that must stay within the L2 budget. Sub-chain
// boundaries come from a cost model minimised over all split points:
//   cost(b, e) = DRAM bytes(b, e) / BW + items(b, e) * c_item,
// DRAM bytes = one read of every dataset the sub-chain reads and one write
// of every dataset it writes (the L2 holds the rest), items = tiles * loops
// (each item ends in a grid barrier at worst).
namespace {
struct SubInfo {
  int64_t slice = 0;  // bytes of one slowest-dim slice over the sub-chain's datasets
  int64_t skew = 0;   // sum of slowest-dim read reaches (upper bound of the plan skew)
  int64_t dram = 0;   // compulsory DRAM bytes
  int64_t extent = 1; // slowest-dim extent of the sub-chain's union
};
}  // namespace

std::vector<Runtime::L2Sub> Runtime::l2_split(const LoopChain& chain, const Target& t) const {
  const int s = chain.dim - 1;
  const int L = static_cast<int>(chain.size());
  int64_t budget = (device_ready() ? dev_->info().l2_bytes : int64_t{126} << 20) * 70 / 100;
  if (const char* e = std::getenv("TCG_L2_BUDGET_MB")) budget = std::atoll(e) << 20;
  double c_item = 3e-6, bw = 6.0e12;
  if (const char* e = std::getenv("TCG_L2_ITEM_US")) c_item = std::atof(e) * 1e-6;
  auto info = [&](int b, int e) {
    SubInfo si;
    std::map<DatasetId, int> use;  // bit 1 read, bit 2 written
    int64_t lo = std::numeric_limits<int64_t>::max(), hi = std::numeric_limits<int64_t>::min();
    for (int l = b; l < e; ++l) {
      const LoopRecord& lp = chain.loops[static_cast<size_t>(l)];
      int64_t reach = 0;
      for (const ArgSpec& a : lp.args) {
        use[a.dataset] |= (mode_reads(a.mode) ? 1 : 0) | (mode_writes(a.mode) ? 2 : 0);
        if (mode_reads(a.mode)) {
          const Stencil& st = chain.stencil(a.stencil);
          reach = std::max<int64_t>({reach, static_cast<int64_t>(std::llabs(st.min_offset(s))),
                                     static_cast<int64_t>(std::llabs(st.max_offset(s)))});
        }
      }
      si.skew += reach;
      lo = std::min(lo, lp.range.start(s));
      hi = std::max(hi, lp.range.end(s));
    }
    si.extent = std::max<int64_t>(1, hi - lo);
    for (const auto& [ds, u] : use) {
      const Range& al = t.alloc[static_cast<size_t>(ds)];
      int64_t b8 = 8;
      for (int d = 0; d < s; ++d) b8 *= al.extent(d);
      si.slice += b8;
      const int64_t field = b8 * al.extent(s);
      si.dram += ((u & 1) ? field : 0) + ((u & 2) ? field : 0);
    }
    return si;
  };
  // ts(b, e): deepest tile whose working set fits; a single loop needs no
  // reuse and runs as one item.
  auto tile_of = [&](int b, int e, const SubInfo& si) -> int64_t {
    if (e - b == 1) return si.extent;
    const int64_t rows = budget / std::max<int64_t>(1, si.slice);
    return rows - si.skew - 2;
  };
  std::vector<double> best(static_cast<size_t>(L) + 1, 1e300);
  std::vector<int> from(static_cast<size_t>(L) + 1, -1);
  std::vector<int64_t> tsb(static_cast<size_t>(L) + 1, 1);
  best[0] = 0;
  int max_sub = 32;  // loops per launch (descriptors in kernel parameters)
  if (const char* e = std::getenv("TCG_L2_MAXLOOPS")) max_sub = std::max(1, std::min(32, std::atoi(e)));
  for (int e = 1; e <= L; ++e)
    for (int b = e - 1; b >= std::max(0, e - max_sub); --b) {
      const SubInfo si = info(b, e);
      const int64_t ts = tile_of(b, e, si);
      if (ts < 1) break;  // longer sub-chains only get worse
      const double items = static_cast<double>((si.extent + ts - 1) / ts) * (e - b);
      const double c = best[static_cast<size_t>(b)] + static_cast<double>(si.dram) / bw + items * c_item;
      if (c < best[static_cast<size_t>(e)]) {
        best[static_cast<size_t>(e)] = c;
        from[static_cast<size_t>(e)] = b;
        tsb[static_cast<size_t>(e)] = ts;
      }
    }
  std::vector<L2Sub> subs;
  for (int e = L; e > 0; e = from[static_cast<size_t>(e)]) {
    if (from[static_cast<size_t>(e)] < 0) {  // a single loop that cannot fit: one item
      subs.push_back(L2Sub{static_cast<size_t>(e - 1), static_cast<size_t>(e), int64_t{1} << 40});
      from[static_cast<size_t>(e)] = e - 1;
      continue;
    }
    subs.push_back(L2Sub{static_cast<size_t>(from[static_cast<size_t>(e)]), static_cast<size_t>(e),
                         tsb[static_cast<size_t>(e)]});
  }
  std::reverse(subs.begin(), subs.end());
  if (const char* e = std::getenv("TCG_L2_TS")) {  // tuning: fixed depth, <= 32 loops per sub-chain
    subs.clear();
    for (size_t b = 0; b < chain.size(); b += 32)
      subs.push_back(L2Sub{b, std::min(chain.size(), b + 32), std::max<int64_t>(1, std::atoll(e))});
  }
  return subs;
}

void Runtime::run_l2(const LoopChain& chain, const ExecMode& mode, ExecutionReport& rep, const Target& t,
                     std::vector<double>& vals) {
  DeviceExec& dev = device();
  const int s = chain.dim - 1;
  bool explicit_ts = false;
  if (mode.kind == ExecMode::Kind::Tiled)
    for (int d = 0; d < chain.dim; ++d) explicit_ts = explicit_ts || mode.tile_sizes[d] > 0;
  std::vector<L2Sub> subs;
  std::array<int64_t, kMaxDims> ets{1, 1, 1};
  if (explicit_ts) {
    // The reference's tile sizes over the whole chain.
    for (int d = 0; d < chain.dim; ++d) ets[d] = std::max<int64_t>(1, mode.tile_sizes[d]);
    for (size_t b = 0; b < chain.size(); b += 32) subs.push_back(L2Sub{b, std::min(chain.size(), b + 32), 0});
  } else {
    const uint64_t key = chain.signature() ^ mask_hash(*this, t.masked, t.mask, chain.dim);
    auto sit = l2_splits_.find(key);
    if (sit == l2_splits_.end()) sit = l2_splits_.emplace(key, l2_split(chain, t)).first;
    subs = sit->second;
  }
  size_t red_base = 0;
  for (const L2Sub& sub : subs) {
    const LoopChain sc = (sub.begin == 0 && sub.end == chain.size()) ? chain : slice(chain, sub.begin, sub.end);
    std::array<int64_t, kMaxDims> ts = ets;
    if (!explicit_ts) {
      for (int d = 0; d < chain.dim; ++d) ts[d] = int64_t{1} << 40;
      ts[static_cast<size_t>(s)] = sub.ts;
    }
    bool hit = false;
    std::shared_ptr<const TilingPlan> plan = plan_cache_.get_or_build(sc, ts, &hit);
    if (!hit) {
      ++rep.plan_constructions;
      rep.plan_seconds += plan->build_seconds;
      // execute_plan's pad check (executor.cpp:209-250): every required box
      // must lie inside the (target's) allocation.
      std::vector<FieldExtent> fe;
      for (size_t i = 0; i < t.alloc.size(); ++i) fe.push_back(FieldExtent{fields_[i].name, t.alloc[i]});
      verify_plan_extents(*plan, fe);
    }
    rep.plan_cache_hit = rep.plan_cache_hit && hit;
    // Items (tile-major, loop order as in execute_plan) with a grid barrier
    // only where the next item touches what an unsynchronised earlier one
    // wrote (RAW), reads (WAR) or writes (WAW).
    auto it = l2_items_.find(plan.get());
    if (it == l2_items_.end()) {
      L2Items li;
      std::vector<DevItem>& items = li.items;
      std::vector<Footprint> open, all;
      const int32_t L = plan->num_loops;
      int32_t flag_off = 0;
      for (int64_t tt = 0; tt < plan->num_tiles(); ++tt)
        for (int32_t l = 0; l < L; ++l) {
          const Range& r = plan->range(tt, l);
          if (r.empty()) continue;
          Footprint f = footprint(sc, sc.loops[static_cast<size_t>(l)], r);
          bool conflict = false;
          for (const Footprint& o : open)
            conflict = conflict || overlaps(o.writes, f.reads) || overlaps(o.writes, f.writes) ||
                       overlaps(o.reads, f.writes);
          if (conflict && !items.empty()) {
            items.back().sync = 1;
            open.clear();
          }
          DevItem di{};
          di.loop = l;
          di.sync = 0;
          for (int d = 0; d < 3; ++d) {
            di.lo[d] = d < chain.dim ? static_cast<int32_t>(r.start(d)) : 0;
            di.hi[d] = d < chain.dim ? static_cast<int32_t>(r.end(d)) : 1;
          }
          // Chunk grid (matches k_l2tiled: 256 points in 1D, 32 x 8*kL2Run in 2D,
          // 32 x 8 x kL2Run in 3D).
          const int64_t nx = r.extent(0);
          if (chain.dim == 1) {
            di.cx = static_cast<int32_t>((nx + 255) / 256);
            di.cy = 1;
            di.nch = di.cx;
          } else if (chain.dim == 2) {
            di.cx = static_cast<int32_t>((nx + 31) / 32);
            di.cy = static_cast<int32_t>((r.extent(1) + 8 * kL2Run - 1) / (8 * kL2Run));
            di.nch = di.cx * di.cy;
          } else {
            di.cx = static_cast<int32_t>((nx + 31) / 32);
            di.cy = static_cast<int32_t>((r.extent(1) + 7) / 8);
            di.nch = di.cx * di.cy * static_cast<int32_t>((r.extent(2) + kL2Run - 1) / kL2Run);
          }
          di.flag_off = flag_off;
          flag_off += di.nch;
          // Dataflow dependencies: every earlier item it conflicts with.
          di.dep_off = static_cast<int32_t>(li.deps.size());
          for (size_t j = 0; j < all.size(); ++j)
            if (overlaps(all[j].writes, f.reads) || overlaps(all[j].writes, f.writes) ||
                overlaps(all[j].reads, f.writes))
              li.deps.push_back(static_cast<int32_t>(j));
          di.ndeps = static_cast<int32_t>(li.deps.size()) - di.dep_off;
          items.push_back(di);
          all.push_back(f);
          open.push_back(std::move(f));
        }
      // Stencil reach per dimension (dilation of the dataflow wait).
      for (const LoopRecord& lp : sc.loops)
        for (const ArgSpec& a : lp.args) {
          if (!mode_reads(a.mode)) continue;
          const Stencil& st = sc.stencil(a.stencil);
          for (int d = 0; d < chain.dim; ++d)
            li.reach[static_cast<size_t>(d)] = std::max<int32_t>(
                li.reach[static_cast<size_t>(d)],
                static_cast<int32_t>(std::max(std::llabs(st.min_offset(d)), std::llabs(st.max_offset(d)))));
        }
      it = l2_items_.emplace(plan.get(), std::move(li)).first;
    }
    DevChain dc = lower(sc, t);
    std::vector<double> out(static_cast<size_t>(std::max(1, dc.nred)));
    static const std::vector<int32_t> no_deps;
    dev.run_l2(dc, it->second.items, no_deps, it->second.reach, reinterpret_cast<uint64_t>(plan.get()), out.data());
    for (int i = 0; i < dc.nred; ++i) vals.at(red_base + static_cast<size_t>(i)) = out[static_cast<size_t>(i)];
    red_base += static_cast<size_t>(dc.nred);
    last_plan_ = plan;
    rep.tiles_executed += plan->num_tiles();
    for (const DevItem& di : it->second.items) rep.l2_syncs += di.sync;
    rep.subchains += 1;
    rep.ctas += static_cast<int64_t>(it->second.items.size());  // items
    for (int d = 0; d < chain.dim; ++d) {
      rep.tile_sizes[d] = std::max(rep.tile_sizes[d], std::min<int64_t>(ts[d], int64_t{1} << 30));
      rep.max_skew[d] = std::max(rep.max_skew[d], plan->max_skew[d]);
    }
  }
  rep.computed_points += chain_points(chain);
}

std::vector<double> Runtime::run_on(const LoopChain& full, const ExecMode& mode, ExecutionReport& rep,
                                    const Target& t) {
  DeviceExec& dev = device();
  // Loops with an empty range do nothing (a reducing one yields the
  // identity); rank-local chains have them wherever a rank computes none of a
  // loop. Execute the non-empty ones only.
  std::vector<double> all_vals;
  std::vector<int> red_src;  // per reduction of `full`: index into vals, -1 = identity
  bool any_empty = false;
  {
    int nr = 0;
    for (const LoopRecord& lp : full.loops) {
      const bool empty = lp.range.empty();
      any_empty = any_empty || empty;
      if (lp.reduction) {
        all_vals.push_back(reduce_identity(lp.reduction->op));
        red_src.push_back(empty ? -1 : nr);
        if (!empty) ++nr;
      }
    }
  }
  // The non-empty loops (a copy only when some loop is empty).
  LoopChain nonempty;
  if (any_empty) {
    nonempty.dim = full.dim;
    nonempty.stencils = full.stencils;
    for (const LoopRecord& lp : full.loops)
      if (!lp.range.empty()) nonempty.loops.push_back(lp);
  }
  const LoopChain& chain = any_empty ? nonempty : full;
  if (chain.loops.empty()) return all_vals;
  size_t nred = 0;
  for (const LoopRecord& lp : chain.loops) nred += lp.reduction ? 1 : 0;
  std::vector<double> vals(nred, 0.0);
  // Executor: 0 L2-tiled, 1 untiled, 2 windowed. tiled_auto times every
  // candidate twice per chain signature (round robin; the first run of each
  // carries plan construction and lazy module loading) and then keeps the
  // fastest -- they are all bit-exact.
  int cand = mode.kind == ExecMode::Kind::Untiled    ? 1
             : mode.kind == ExecMode::Kind::Windowed ? 2
             : mode.kind == ExecMode::Kind::Stream   ? 3
                                                     : 0;
  AutoStat* as = nullptr;
  bool measure = false;
  bool sum_ordered = false;
  if (red_workers_ > 0)
    for (const LoopRecord& lp : chain.loops) sum_ordered = sum_ordered || (lp.reduction && lp.reduction->op == ReduceOp::Sum);
  if (sum_ordered) {
    if (t.masked) throw InvalidArgument("order-matched Sum reductions are not available on a rank grid");
    dev.set_reduction_workers(red_workers_);
    cand = 1;  // the reference order is the untiled executor's (execute_untiled, executor.cpp:252-277)
  } else if (mode.kind == ExecMode::Kind::TiledAuto) {
    const uint64_t akey = chain.signature() ^ mask_hash(*this, t.masked, t.mask, chain.dim);
    auto ait = auto_.find(akey);
    if (ait == auto_.end()) {
      ait = auto_.emplace(akey, AutoStat{}).first;
      for (int c = 0; c < kCand; ++c) ait->second.fits[c] = ((auto_cands_ >> c) & 1u) != 0;
    }
    as = &ait->second;
    if (as->ev1) {
      // Resolve the pending measurement (waits for it: only while tuning).
      float ms = 0;
      dev.wait_event(as->ev1);
      if (dev.elapsed_ms(as->ev0, as->ev1, &ms)) {
        as->ms[as->pending] = std::min(as->ms[as->pending], ms);
        dev.release(as->ev0);
        dev.release(as->ev1);
        as->ev0 = as->ev1 = nullptr;
      }
    }
    cand = -1;
    if (!as->ev1) {
      for (int c = 0; c < kCand; ++c)
        if (as->fits[c] && as->runs[c] < kAutoRuns && (cand < 0 || as->runs[c] < as->runs[cand])) cand = c;
      measure = cand >= 0;
    }
    if (cand < 0) {
      cand = as->best();
      if (!as->ev1 && !as->saved) save_autotune(*as);
    }
  }
  bool use_untiled = cand == 1;
  if (measure) dev.synchronize();  // tuning only: time this chain alone, launch overhead included
  if (!use_untiled) {
    if (measure) as->ev0 = dev.record();
    try {
      rep.tiled = true;
      if (cand == 0) {
        rep.executor = "tiled";
        run_l2(chain, mode, rep, t, vals);
      } else if (cand == 3) {
        rep.executor = "stream";
        run_stream(chain, rep, t, vals);
      } else {
        rep.executor = "windowed";
        run_tiled(chain, mode, rep, t, vals);
      }
    } catch (const PlanError& e) {
      // Chains an executor cannot run at all (windows that do not fit,
      // more than 32 datasets) drop out of tiled_auto; explicit modes raise.
      if (mode.kind != ExecMode::Kind::TiledAuto) throw;
      as->fits[cand] = false;
      if (measure) {
        dev.release(as->ev0);
        as->ev0 = nullptr;
      }
      rep.tiled = false;
      use_untiled = true;
      cand = 1;
    }
  }
  if (measure && as) {
    if (use_untiled) as->ev0 = as->ev0 ? as->ev0 : dev.record();
    as->pending = cand;
    as->runs[cand]++;
  }
  if (use_untiled) {
    rep.executor = "untiled";
    check_pad(chain, t);
    DevChain dc = lower(chain, t);
    std::vector<double> out(static_cast<size_t>(std::max(1, dc.nred)));
    dev.run_untiled(dc, out.data());
    for (size_t i = 0; i < nred; ++i) vals[i] = out[i];
    rep.tiles_executed += 1;
  }
  if (measure && as) as->ev1 = dev.record();
  for (size_t i = 0; i < red_src.size(); ++i)
    if (red_src[i] >= 0) all_vals[i] = vals[static_cast<size_t>(red_src[i])];
  return all_vals;
}

// ---- streaming executor ------------------------------------------------------

std::vector<StreamGeom> Runtime::stream_geoms(const Target& t, bool from_device) {
  std::vector<StreamGeom> g(t.alloc.size());
  for (size_t ds = 0; ds < t.alloc.size(); ++ds) {
    StreamGeom& q = g[ds];
    q.alloc = t.alloc[ds];
    if (from_device && !t.dev.empty() && t.dev[ds] >= 0) {
      const DevView v = device().view(t.dev[ds], false);
      q.x0 = v.x0;
      q.y0 = v.y0;
      q.z0 = v.z0;
      q.py = v.py;
      q.pz = v.pz;
    } else {
      const Range& a = t.alloc[ds];
      int64_t lo[3], hi[3];
      for (int d = 0; d < 3; ++d) {
        lo[d] = d < a.dim() ? a.start(d) : 0;
        hi[d] = d < a.dim() ? a.end(d) : 1;
      }
      const FieldLayout fl = field_layout(a.dim(), lo, hi);
      q.x0 = fl.x0;
      q.y0 = a.dim() >= 2 ? a.start(1) : 0;
      q.z0 = a.dim() >= 3 ? a.start(2) : 0;
      q.py = a.dim() >= 2 ? fl.py : 0;
      q.pz = a.dim() >= 3 ? fl.pz : 0;
    }
  }
  return g;
}

StreamPlan Runtime::stream_plan_pending(const StreamDevice& sd) {
  LoopChain chain = take_pending();
  if (!chain.fills.empty()) {
    std::vector<Range> logical;
    for (const FieldRec& f : fields_) logical.push_back(f.logical);
    chain = apply_periodic(chain, logical).chain;
  }
  Target t;
  for (const FieldRec& f : fields_) {
    t.dev.push_back(-1);
    t.alloc.push_back(f.alloc);
  }
  return build_stream_plan(chain, stream_geoms(t, false), sd, stream_choice_, nullptr);
}

void Runtime::run_stream(const LoopChain& chain, ExecutionReport& rep, const Target& t, std::vector<double>& vals) {
  DeviceExec& dev = device();
  if (chain.dim < 2) throw PlanError("stream executor: 1D chains are not streamed");
  check_pad(chain, t);
  uint64_t key = chain.signature() ^ mask_hash(*this, t.masked, t.mask, chain.dim);
  for (int f : t.dev) key = (key ^ static_cast<uint64_t>(f + 7)) * 1099511628211ull;
  {
    const StreamChoice& c = stream_choice_;
    const int cv[8] = {c.nt, c.bx, c.by, c.ntx, c.segments, c.max_loops, c.minb, c.prefetch};
    for (int v : cv) key = (key ^ static_cast<uint64_t>(v + 1000)) * 1099511628211ull;
  }
  auto it = stream_plans_.find(key);
  if (it == stream_plans_.end()) {
    rep.plan_cache_hit = false;
    StreamDevice sd;
    sd.num_sms = dev.info().num_sms;
    sd.smem_optin = dev.info().smem_optin;
    auto plan = std::make_shared<StreamPlan>(
        build_stream_plan(chain, stream_geoms(t, true), sd, stream_choice_, t.masked ? &t.mask : nullptr));
    ++rep.plan_constructions;
    rep.plan_seconds += plan->build_seconds;
    it = stream_plans_.emplace(key, plan).first;
  } else {
    rep.plan_cache_hit = true;
  }
  const StreamPlan& plan = *it->second;
  last_stream_plan_ = it->second;
  // Every kernel of the plan is compiled / loaded before the first launch, so
  // a generated kernel NVRTC rejects is a PlanError with no side effects
  // (tiled_auto then drops the streaming candidate for this chain).
  const bool sized_plan = stream_choice_.nt == 0 && stream_choice_.bx == 0 && stream_choice_.max_loops == 0;
  for (const StreamKernel& K : plan.kernels) {
    if (K.nctas == 0) continue;
    if (sized_plan && K.end - K.begin == 1 && plan.kernels.size() > 1) continue;  // may run untiled (below)
    try {
      jit_function(K.source, K.hash, K.smem_bytes);
    } catch (const CudaError& e) {
      if (std::string(e.what()).find("NVRTC compile") != std::string::npos)
        throw PlanError(std::string("stream executor: ") + e.what());
      throw;
    }
  }
  size_t nred_total = 0;
  for (const StreamKernel& k : plan.kernels) nred_total += k.red_op.size();
  std::vector<uint64_t> buf;
  size_t red_base = 0;
  // Sub-chains of one loop have nothing to fuse: they run on the untiled
  // executor (a single streamed loop costs about twice the untiled launch,
  // measured on c3's 16th loop: 0.98 vs 0.47 ms; profiles/r5/sweeps.md).
  static const bool singleton_untiled = [] {
    const char* e = std::getenv("TCG_STREAM_SINGLETON_UNTILED");
    return !(e && *e == '0');
  }();
  std::vector<double> host_vals(nred_total, 0.0);
  std::vector<char> host_known(nred_total, 0);
  for (const StreamKernel& K : plan.kernels) {
    if (K.nctas == 0) continue;
    const bool sized = stream_choice_.nt == 0 && stream_choice_.bx == 0 && stream_choice_.max_loops == 0;  // sizer's plan
    if (singleton_untiled && sized && K.end - K.begin == 1 && plan.kernels.size() > 1) {
      const LoopChain sub = slice(chain, K.begin, K.end);
      DevChain dc = lower(sub, t);
      std::vector<double> out(static_cast<size_t>(std::max(1, dc.nred)));
      dev.run_untiled(dc, out.data());
      for (size_t i = 0; i < K.red_op.size(); ++i) {
        host_vals.at(red_base + i) = out.at(i);
        host_known.at(red_base + i) = 1;
      }
      red_base += K.red_op.size();
      rep.computed_points += sub.loops[0].range.volume();
      rep.subchains += 1;
      continue;
    }
    void* fn = jit_function(K.source, K.hash, K.smem_bytes);
    const int occ = std::max(1, jit_occupancy(fn, K.nt, K.smem_bytes));
    const int64_t ns = K.segments_for(static_cast<int64_t>(dev.info().num_sms) * occ);
    const int64_t nctas = K.tiles * ns;
    const size_t nd = K.dats.size();
    buf.assign(2 * nd + 4 + static_cast<size_t>(std::max(1, K.nparams)), 0);
    for (size_t k = 0; k < nd; ++k) {
      const int f = t.dev.at(static_cast<size_t>(K.dats[k]));
      if (K.store[k] && K.pingpong[k]) dev.sync_alt(f, K.store_box[k]);
      const DevView src = dev.view(f, false);
      buf[k] = reinterpret_cast<uint64_t>(src.base);
      buf[nd + k] = reinterpret_cast<uint64_t>(K.store[k] && K.pingpong[k] ? dev.view(f, true).base : src.base);
      if (K.store[k] && !K.pingpong[k]) dev.mark_written(f, K.store_box[k]);
    }
    double *part = nullptr, *out = nullptr;
    unsigned* ticket = nullptr;
    dev.stream_red_buffers(std::max<size_t>(1, K.red_op.size() * static_cast<size_t>(nctas)),
                           std::max<size_t>(1, nred_total), &part, &out, &ticket);
    buf[2 * nd] = reinterpret_cast<uint64_t>(part);
    buf[2 * nd + 1] = reinterpret_cast<uint64_t>(out + red_base);
    buf[2 * nd + 2] = reinterpret_cast<uint64_t>(ticket);
    buf[2 * nd + 3] = static_cast<uint64_t>(ns);
    double* prm = reinterpret_cast<double*>(buf.data() + 2 * nd + 4);
    size_t pi = 0;
    for (size_t l = K.begin; l < K.end; ++l)
      for (double v : chain.loops[l].kernel.fn.params) prm[pi++] = v;
    dev.launch_stream(fn, nctas, K.nt, K.smem_bytes, buf.data(), buf.size() * sizeof(uint64_t));
    for (size_t k = 0; k < nd; ++k)
      if (K.store[k] && K.pingpong[k]) dev.commit_alt(t.dev.at(static_cast<size_t>(K.dats[k])), K.store_box[k]);
    red_base += K.red_op.size();
    rep.ctas += nctas;
    rep.computed_points += K.computed_for(ns);
    rep.subchains += 1;
    rep.tile_sizes[0] = K.tile[0];
    if (chain.dim == 3) rep.tile_sizes[1] = K.tile[1];
    rep.cta_grid[0] = K.grid[0];
    rep.cta_grid[1] = K.grid[1];
    rep.cta_grid[2] = static_cast<int>(ns);
  }
  rep.tiles_executed += rep.ctas;
  if (nred_total > 0) {
    bool any_dev = false;
    for (char k : host_known) any_dev = any_dev || !k;
    std::vector<double> r(nred_total, 0.0);
    if (any_dev) {
      double *part = nullptr, *out = nullptr;
      unsigned* ticket = nullptr;
      dev.stream_red_buffers(1, nred_total, &part, &out, &ticket);
      dev.read_device(r.data(), out, nred_total);
    }
    for (size_t i = 0; i < nred_total; ++i) vals.at(i) = host_known[i] ? host_vals[i] : r[i];
  }
}

void Runtime::check_pad(const LoopChain& chain, const Target& t) const {
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
      const Range& alloc = t.alloc.at(static_cast<size_t>(a.dataset));
      if (!alloc.contains(touched))
        throw AccessError("loop k" + std::to_string(lp.kernel.id) + " (id " + std::to_string(lp.loop_id) +
                          "), dataset " + fields_[static_cast<size_t>(a.dataset)].name + ": access over " +
                          touched.to_string() + " outside allocated extent " + alloc.to_string());
    }
  }
}

ExecutionReport Runtime::execute_chain(LoopChain chain, const ExecMode& mode) {
  if (distributed()) {
    if (!chain.fills.empty() && !periodic_domain_)
      throw InvalidArgument("periodic_fill on a rank grid: call set_periodic_domain(true) before set_rank_grid");
    return execute_distributed(std::move(chain), mode);
  }
  const auto t0 = std::chrono::steady_clock::now();
  ExecutionReport rep;
  rep.dim = chain.dim;
  for (const LoopRecord& lp : chain.loops)
    rep.loops.push_back(LoopExecStats{lp.loop_id, lp.range.volume(), estimate_bytes_moved(lp, lp.range)});
  ensure_fields();
  DeviceExec& dev = device();
  const int64_t l0 = dev.launches();
  if (!chain.fills.empty()) {
    // Periodic marks: one wrap of the chain's inputs to the accumulated
    // depth, then the chain over extended ranges (tcg_periodic.hpp).
    std::vector<Range> logical;
    for (const FieldRec& f : fields_) logical.push_back(f.logical);
    PeriodicPlan pp = apply_periodic(chain, logical);
    std::map<std::pair<int64_t, std::vector<int64_t>>, std::vector<int>> groups;  // (depth, logical box) -> fields
    for (const auto& [ds, depth] : pp.pre_fills) {
      const FieldRec& f = fields_.at(static_cast<size_t>(ds));
      if (depth > f.pad)
        throw AccessError("periodic chain: needs " + std::to_string(depth) + " ghost layers of " + f.name +
                          " but its pad is " + std::to_string(f.pad) + " (raise skew_allowance)");
      for (int d = 0; d < dim_; ++d)
        if (depth > f.logical.extent(d)) throw InvalidArgument("periodic chain: depth exceeds the extent of " + f.name);
      std::vector<int64_t> key;
      for (int d = 0; d < dim_; ++d) {
        key.push_back(f.logical.start(d));
        key.push_back(f.logical.end(d));
      }
      groups[{depth, key}].push_back(f.dev);
    }
    for (const auto& [k, devs] : groups) {
      Range lg(dim_);
      for (int d = 0; d < dim_; ++d) lg.set_raw(d, k.second[2 * static_cast<size_t>(d)], k.second[2 * static_cast<size_t>(d) + 1]);
      dev.periodic_fill(devs, lg, k.first);
      rep.halo_exchanges += 1;
      rep.halo_messages += static_cast<int64_t>(devs.size()) * 2 * dim_;
    }
    rep.computed_points += pp.extended_points;
    chain = std::move(pp.chain);
  }
  const std::vector<double> vals = run_on(chain, mode, rep, whole_target());
  store(reduction_handles(chain), vals.data());
  rep.launches = dev.launches() - l0;
  rep.exec_seconds = secs_since(t0) - rep.plan_seconds;
  rep.total_seconds = secs_since(t0);
  last_report_ = rep;
  return rep;
}

void Runtime::save_autotune(AutoStat& as) {
  as.saved = true;
  if (autotune_file_.empty()) return;
  if (FILE* f = std::fopen(autotune_file_.c_str(), "w")) {
    for (const auto& [sig, a] : auto_)
      if (a.saved)
        std::fprintf(f, "%llx %.6f %.6f %.6f %.6f %d\n", static_cast<unsigned long long>(sig), a.ms[0], a.ms[1],
                     a.ms[2], a.ms[3], (a.fits[0] ? 1 : 0) | (a.fits[1] ? 2 : 0) | (a.fits[2] ? 4 : 0) | (a.fits[3] ? 8 : 0));
    std::fclose(f);
  }
}

// ---- distribution -------------------------------------------------------------

void Runtime::set_rank_grid(const std::array<int, kMaxDims>& grid) {
  // runtime.cpp:213-222
  for (int d = 0; d < kMaxDims; ++d) {
    if (grid[d] < 1) throw InvalidArgument("set_rank_grid: grid entries must be >= 1");
    if (d >= dim_ && grid[d] != 1) throw InvalidArgument("set_rank_grid: grid uses dimension beyond block");
  }
  flush();
  drop_dist();
  comm_.reset();
  grid_ = grid;
  grid_set_ = true;
  proc_rank_ = -1;
}

void Runtime::set_process_rank(const std::array<int, kMaxDims>& grid, int rank, const uint8_t id[kCommIdBytes]) {
  for (int d = 0; d < kMaxDims; ++d) {
    if (grid[d] < 1) throw InvalidArgument("set_process_rank: grid entries must be >= 1");
    if (d >= dim_ && grid[d] != 1) throw InvalidArgument("set_process_rank: grid uses dimension beyond block");
  }
  const int n = grid[0] * grid[1] * grid[2];
  if (rank < 0 || rank >= n) throw InvalidArgument("set_process_rank: rank out of range");
  flush();
  drop_dist();
  device();  // the communicator binds to the current device
  comm_.reset();
  comm_ = std::make_unique<Comm>(n, rank, id);
  grid_ = grid;
  grid_set_ = true;
  proc_rank_ = rank;
}

const RankLayout& Runtime::rank_layout() {
  if (!grid_set_) throw InvalidArgument("rank_layout: no rank grid set");
  if (dist_) return dist_->layout;
  static thread_local RankLayout lay;
  if (fields_.empty()) throw InvalidArgument("distributed execution requires declared fields");
  Range global = fields_[0].logical;
  int64_t pad = fields_[0].pad;
  for (const FieldRec& f : fields_) {
    global = global.hull(f.logical);
    pad = std::min(pad, f.pad);
  }
  if (periodic_domain_) {
    // the ghost layers of a periodic box are part of the decomposed domain
    Point lo{0, 0, 0}, hi{0, 0, 0};
    for (int d = 0; d < dim_; ++d) {
      lo[d] = -pad;
      hi[d] = pad;
    }
    global = global.dilated(lo, hi);
  }
  lay = decompose(global, grid_);
  return lay;
}

void Runtime::drop_dist() {
  if (!dist_) return;
  // Carry rank data back into the undistributed fields (the reference gathers
  // after every distributed flush, runtime.cpp:128-137).
  ensure_fields();
  DeviceExec& dev = device();
  for (size_t ds = 0; ds < fields_.size(); ++ds) {
    const FieldRec& f = fields_[ds];
    std::vector<double> host(static_cast<size_t>(f.alloc.volume()));
    download(static_cast<DatasetId>(ds), host.data());
    dev.upload(f.dev, host.data());
  }
  dist_.reset();
}

void Runtime::ensure_dist() {
  if (dist_ && dist_->targets.size() == static_cast<size_t>(dist_->layout.rank_count()) &&
      (dist_->local.empty() || dist_->targets[static_cast<size_t>(dist_->local[0])].dev.size() == fields_.size()))
    return;
  DeviceExec& dev = device();
  const bool fresh = !dist_;
  if (fresh) {
    auto d = std::make_unique<Dist>();
    d->layout = rank_layout();
    const int R = d->layout.rank_count();
    if (proc_rank_ >= 0) {
      if (comm_->nranks() != R) throw InvalidArgument("set_process_rank: grid and communicator size differ");
      d->local = {proc_rank_};
    } else {
      for (int r = 0; r < R; ++r) d->local.push_back(r);
    }
    d->targets.resize(static_cast<size_t>(R));
    dist_ = std::move(d);
  }
  // Rank fields: owned box +- the field's pad (dist.cpp:519-529), seeded from
  // the undistributed field when it already holds data (scatter,
  // dist.cpp:532-545).
  for (int r : dist_->local) {
    Target& t = dist_->targets[static_cast<size_t>(r)];
    t.masked = true;
    t.mask = dist_->layout.owned[static_cast<size_t>(r)];
    for (size_t ds = t.dev.size(); ds < fields_.size(); ++ds) {
      const FieldRec& f = fields_[ds];
      if (!dist_->layout.global.contains(f.logical))
        throw InvalidArgument("declare_field: field " + f.name + " lies outside the distributed domain");
      const Range a = rank_alloc(dist_->layout, r, f.pad);
      const int idx = dev.add_field(a);
      t.dev.push_back(idx);
      t.alloc.push_back(a);
      if (f.dev >= 0) {
        const Range box = a.intersect(f.alloc);
        std::vector<double> tmp(static_cast<size_t>(box.volume()));
        dev.field_to_buf(f.dev, box, tmp.data(), box);
        dev.buf_to_field(idx, box, tmp.data(), box);
        dev.synchronize();
      }
    }
  }
}

std::shared_ptr<const DistSchedule> Runtime::dist_schedule(const LoopChain& chain) {
  const auto key = std::make_pair(chain.signature(), dist_->hist_version);
  auto it = dist_->schedules.find(key);
  if (it != dist_->schedules.end()) return it->second;
  std::vector<int64_t> pads;
  for (const FieldRec& f : fields_) pads.push_back(f.pad);
  auto s = std::make_shared<const DistSchedule>(
      build_dist_schedule(chain, dist_->layout, pads, &dist_->written));
  dist_->schedules[key] = s;
  return s;
}

DistSchedule Runtime::schedule_pending() {
  if (!grid_set_) throw InvalidArgument("schedule_pending: no rank grid set");
  LoopChain chain = take_pending();
  std::vector<std::pair<DatasetId, int64_t>> wraps;
  if (!chain.fills.empty()) {
    if (!periodic_domain_)
      throw InvalidArgument("periodic_fill on a rank grid: call set_periodic_domain(true) before set_rank_grid");
    std::vector<Range> logical;
    for (const FieldRec& f : fields_) logical.push_back(f.logical);
    PeriodicPlan pp = apply_periodic(chain, logical);
    chain = std::move(pp.chain);
    wraps = std::move(pp.pre_fills);
  }
  if (!dist_) {
    // Host-only use (no device): layout and history without rank fields.
    auto d = std::make_unique<Dist>();
    d->layout = rank_layout();
    dist_ = std::move(d);
  }
  std::vector<int64_t> pads;
  for (const FieldRec& f : fields_) pads.push_back(f.pad);
  // As execute_distributed does: the wrapped points are written before the
  // schedule is built, so every rank's halo copies of them count as stale.
  for (const auto& [ds, g] : wraps) {
    Point wl{0, 0, 0}, wh{0, 0, 0};
    for (int d = 0; d < dim_; ++d) {
      wl[d] = -g;
      wh[d] = g;
    }
    dist_->written[ds].push_back(fields_.at(static_cast<size_t>(ds)).logical.dilated(wl, wh));
    ++dist_->hist_version;
  }
  DistSchedule s = build_dist_schedule(chain, dist_->layout, pads, &dist_->written);
  s.wraps = wraps;
  if (note_writes(dist_->written, chain)) ++dist_->hist_version;
  return s;
}

// DistContext::poison_stale_halos (dist.cpp:546-586): on every local rank,
// the points of each interior face strip (allocation beyond the owned box
// towards a neighbour) that this chain or an earlier one writes become NaN
// before the chain runs; their correct values can arrive only through the
// exchange or a local recompute, so a gap in the schedule shows up as NaN.
void Runtime::poison_stale_halos(const LoopChain& chain) {
  std::map<DatasetId, std::vector<Range>> writes;
  for (const LoopRecord& lp : chain.loops)
    for (const ArgSpec& a : lp.args)
      if (mode_writes(a.mode)) writes[a.dataset].push_back(lp.range);
  for (const auto& [ds, boxes] : dist_->written)
    for (const Range& b : boxes) writes[ds].push_back(b);
  DeviceExec& dev = device();
  const RankLayout& lay = dist_->layout;
  for (int r : dist_->local) {
    const Range& own = lay.owned[static_cast<size_t>(r)];
    const Target& t = dist_->targets[static_cast<size_t>(r)];
    for (const auto& [ds, boxes] : writes) {
      const Range& alloc = t.alloc[static_cast<size_t>(ds)];
      for (int d = 0; d < lay.dim; ++d)
        for (int dir : {-1, +1}) {
          if (lay.neighbor(r, d, dir) < 0) continue;
          Range strip = alloc;
          if (dir < 0)
            strip.set(d, alloc.start(d), own.start(d));
          else
            strip.set(d, own.end(d), alloc.end(d));
          for (const Range& w : boxes) {
            const Range x = strip.intersect(w);
            if (!x.empty()) dev.fill_box_bytes(t.dev[static_cast<size_t>(ds)], x, 0xFF);
          }
        }
    }
  }
}

void Runtime::exchange(const DistSchedule& s, ExecutionReport& rep) {
  DeviceExec& dev = device();
  std::vector<char> is_local(static_cast<size_t>(dist_->layout.rank_count()), 0);
  for (int r : dist_->local) is_local[static_cast<size_t>(r)] = 1;
  static const bool direct_ok = [] {
    const char* e = std::getenv("TCG_HALO_DIRECT");
    return !(e && *e == '0');
  }();
  // A message along the slowest dimension between ranks that share every
  // faster dimension's allocation (a z-split in 3D, a y-split in 2D) is a run
  // of whole planes / rows: contiguous in both fields, so it moves straight
  // from field to field -- a peer copy inside this process, ncclSend/ncclRecv
  // on the field memory between processes -- with no staging pack (the
  // reference's message, dist.cpp:463-511, widened to whole slabs: the extra
  // points are pad columns of the same slabs). The message log keeps the
  // reference's box geometry.
  auto direct = [&](const HaloMsg& m, int d) {
    if (!direct_ok || d != dim_ - 1 || dim_ < 2) return false;
    const Range as = rank_alloc(dist_->layout, m.src, fields_[static_cast<size_t>(m.ds)].pad);
    const Range ad = rank_alloc(dist_->layout, m.dst, fields_[static_cast<size_t>(m.ds)].pad);
    for (int e = 0; e + 1 < dim_; ++e)
      if (as.start(e) != ad.start(e) || as.end(e) != ad.end(e)) return false;
    const bool ls = is_local[static_cast<size_t>(m.src)], ld = is_local[static_cast<size_t>(m.dst)];
    if (ls && ld)
      return dev.same_cross_section(dist_->targets[static_cast<size_t>(m.dst)].dev[static_cast<size_t>(m.ds)],
                                    dist_->targets[static_cast<size_t>(m.src)].dev[static_cast<size_t>(m.ds)]);
    return true;  // remote peer: same declaration, same layout rule
  };
  for (int d = 0; d < kMaxDims; ++d) {
    const size_t a = s.phase[static_cast<size_t>(d)], b = s.phase[static_cast<size_t>(d) + 1];
    if (a == b) continue;
    // Staging offsets of the packed messages this process takes part in.
    std::vector<size_t> off(b - a, 0);
    std::vector<char> dir(b - a, 0);
    size_t total = 0;
    for (size_t i = a; i < b; ++i) {
      const HaloMsg& m = s.msgs[i];
      if (!is_local[static_cast<size_t>(m.src)] && !is_local[static_cast<size_t>(m.dst)]) continue;
      dir[i - a] = direct(m, d) ? 1 : 0;
      if (dir[i - a]) continue;
      off[i - a] = total;
      total += static_cast<size_t>(m.points);
    }
    double* stg = total ? dev.staging(total) : nullptr;
    // Pack every staged message whose source rank lives here.
    for (size_t i = a; i < b; ++i) {
      const HaloMsg& m = s.msgs[i];
      if (dir[i - a] || !is_local[static_cast<size_t>(m.src)]) continue;
      const Target& t = dist_->targets[static_cast<size_t>(m.src)];
      dev.field_to_buf(t.dev[static_cast<size_t>(m.ds)], m.box, stg + off[i - a], m.box);
    }
    // Carry the remote ones (one NCCL group per dimension phase).
    if (comm_) {
      bool any = false;
      for (size_t i = a; i < b && !any; ++i)
        any = is_local[static_cast<size_t>(s.msgs[i].src)] != is_local[static_cast<size_t>(s.msgs[i].dst)];
      if (any) {
        comm_->group_start();
        for (size_t i = a; i < b; ++i) {
          const HaloMsg& m = s.msgs[i];
          const bool ls = is_local[static_cast<size_t>(m.src)], ld = is_local[static_cast<size_t>(m.dst)];
          if (ls == ld) continue;
          const int64_t s0 = m.box.start(dim_ - 1), s1 = m.box.end(dim_ - 1);
          if (ls) {
            const int f = dist_->targets[static_cast<size_t>(m.src)].dev[static_cast<size_t>(m.ds)];
            if (dir[i - a])
              comm_->send(dev.slab_ptr(f, s0), dev.slab_count(f, s0, s1), m.dst, dev.stream());
            else
              comm_->send(stg + off[i - a], static_cast<size_t>(m.points), m.dst, dev.stream());
          } else {
            const int f = dist_->targets[static_cast<size_t>(m.dst)].dev[static_cast<size_t>(m.ds)];
            if (dir[i - a]) {
              comm_->recv(dev.slab_ptr(f, s0), dev.slab_count(f, s0, s1), m.src, dev.stream());
              dev.note_slab_write(f, s0, s1);
            } else {
              comm_->recv(stg + off[i - a], static_cast<size_t>(m.points), m.src, dev.stream());
            }
          }
        }
        comm_->group_end();
      }
    }
    // Local pairs: direct slab copies; staged messages unpack at their destination.
    for (size_t i = a; i < b; ++i) {
      const HaloMsg& m = s.msgs[i];
      if (!is_local[static_cast<size_t>(m.dst)]) continue;
      const Target& t = dist_->targets[static_cast<size_t>(m.dst)];
      if (dir[i - a]) {
        if (is_local[static_cast<size_t>(m.src)])
          dev.copy_slabs(t.dev[static_cast<size_t>(m.ds)],
                         dist_->targets[static_cast<size_t>(m.src)].dev[static_cast<size_t>(m.ds)],
                         m.box.start(dim_ - 1), m.box.end(dim_ - 1));
        continue;
      }
      dev.buf_to_field(t.dev[static_cast<size_t>(m.ds)], m.box, stg + off[i - a], m.box);
    }
  }
  rep.halo_messages += static_cast<int64_t>(s.msgs.size());
  rep.halo_bytes += s.message_bytes;
  rep.halo_exchanges += s.msgs.empty() ? 0 : 1;
}

void Runtime::periodic_exchange(const std::vector<std::pair<DatasetId, int64_t>>& fills, ExecutionReport& rep) {
  if (fills.empty()) return;
  DeviceExec& dev = device();
  const RankLayout& lay = dist_->layout;
  const int s = dim_ - 1;
  for (int d = 0; d < s; ++d)
    if (lay.grid[static_cast<size_t>(d)] != 1)
      throw InvalidArgument("periodic chains: the rank grid may split the slowest dimension only");
  const int lo = 0, hi = lay.rank_count() - 1;  // ranks are ordered along the split dimension
  std::vector<char> is_local(static_cast<size_t>(lay.rank_count()), 0);
  for (int r : dist_->local) is_local[static_cast<size_t>(r)] = 1;
  struct Move {
    int src, dst;
    DatasetId ds;
    int64_t src_s0, dst_s0, n;
  };
  std::vector<Move> moves;
  for (const auto& [ds, g] : fills) {
    const FieldRec& f = fields_.at(static_cast<size_t>(ds));
    if (g > f.pad)
      throw AccessError("periodic chain: needs " + std::to_string(g) + " ghost layers of " + f.name + " but its pad is " +
                        std::to_string(f.pad) + " (raise skew_allowance)");
    const int64_t L = f.logical.start(s), H = f.logical.end(s);
    if (lay.owned[static_cast<size_t>(hi)].start(s) > H - g || lay.owned[static_cast<size_t>(lo)].end(s) < L + g)
      throw PlanError("periodic chain: the wrap depth exceeds an end rank's owned width");
    // 1. faster dimensions, inside every rank, over the slabs it holds
    for (int r : dist_->local) {
      const Target& t = dist_->targets[static_cast<size_t>(r)];
      const Range& a = t.alloc[static_cast<size_t>(ds)];
      Range box = f.logical;
      box.set_raw(s, std::max(a.start(s), L), std::min(a.end(s), H));
      if (s > 0 && !box.empty()) dev.periodic_fill({t.dev[static_cast<size_t>(ds)]}, box, g, s);
    }
    // 2. the split dimension: whole slabs between the end ranks
    moves.push_back(Move{hi, lo, ds, H - g, L - g, g});
    moves.push_back(Move{lo, hi, ds, L, H, g});
    // every rank's halo copies of the wrapped points are stale now
    Point wl{0, 0, 0}, wh{0, 0, 0};
    for (int d = 0; d < dim_; ++d) {
      wl[d] = -g;
      wh[d] = g;
    }
    dist_->written[ds].push_back(f.logical.dilated(wl, wh));
    ++dist_->hist_version;
  }
  bool remote = false;
  for (const Move& m : moves) remote = remote || (is_local[static_cast<size_t>(m.src)] != is_local[static_cast<size_t>(m.dst)]);
  if (remote && !comm_) throw PlanError("periodic chain: remote end rank without a communicator");
  if (remote) comm_->group_start();
  for (const Move& m : moves) {
    const bool ls = is_local[static_cast<size_t>(m.src)], ld = is_local[static_cast<size_t>(m.dst)];
    if (ls && ld) continue;
    if (ls) {
      const int fsrc = dist_->targets[static_cast<size_t>(m.src)].dev[static_cast<size_t>(m.ds)];
      comm_->send(dev.slab_ptr(fsrc, m.src_s0), dev.slab_count(fsrc, m.src_s0, m.src_s0 + m.n), m.dst, dev.stream());
    } else if (ld) {
      const int fdst = dist_->targets[static_cast<size_t>(m.dst)].dev[static_cast<size_t>(m.ds)];
      comm_->recv(dev.slab_ptr(fdst, m.dst_s0), dev.slab_count(fdst, m.dst_s0, m.dst_s0 + m.n), m.src, dev.stream());
      dev.note_slab_write(fdst, m.dst_s0, m.dst_s0 + m.n);
    }
  }
  if (remote) comm_->group_end();
  for (const Move& m : moves) {
    if (!is_local[static_cast<size_t>(m.src)] || !is_local[static_cast<size_t>(m.dst)]) continue;
    dev.copy_slabs_shift(dist_->targets[static_cast<size_t>(m.dst)].dev[static_cast<size_t>(m.ds)], m.dst_s0,
                         dist_->targets[static_cast<size_t>(m.src)].dev[static_cast<size_t>(m.ds)], m.src_s0, m.n);
  }
  rep.halo_exchanges += 1;
  rep.halo_messages += static_cast<int64_t>(moves.size());
  for (const Move& m : moves) {
    const FieldRec& f = fields_.at(static_cast<size_t>(m.ds));
    int64_t plane = 1;
    for (int d = 0; d < s; ++d) plane *= f.logical.extent(d) + 2 * m.n;
    rep.halo_bytes += plane * m.n * 8;
  }
}

ExecutionReport Runtime::execute_distributed(LoopChain chain, const ExecMode& mode) {
  // Tiled modes: DistContext::run_tiled (dist.cpp:617-689) -- plans + halo
  // specs for every rank, ONE deep-halo exchange, per-rank execution of the
  // rank-local chain with reductions masked to the owned box, rank-order
  // fold, note_writes. Untiled: DistContext::run_untiled (dist.cpp:691-788)
  // -- per loop, an on-demand exchange of the stale faces it reads, then the
  // loop on every rank's owned part (the message-count baseline).
  const auto t0 = std::chrono::steady_clock::now();
  ExecutionReport rep;
  rep.dim = chain.dim;
  rep.distributed = true;
  for (const LoopRecord& lp : chain.loops)
    rep.loops.push_back(LoopExecStats{lp.loop_id, lp.range.volume(), estimate_bytes_moved(lp, lp.range)});
  ensure_dist();
  DeviceExec& dev = device();
  const int64_t l0 = dev.launches();
  bool on_demand = mode.kind == ExecMode::Kind::Untiled;
  if (!chain.fills.empty()) {
    // Periodic marks on a rank grid: wrap the chain's inputs once (faster
    // dimensions inside every rank, the split dimension between the end
    // ranks), then the deep-halo schedule of the rewritten chain -- whatever
    // the mode (the on-demand per-loop exchange does not own the ghost zones).
    std::vector<Range> logical;
    for (const FieldRec& f : fields_) logical.push_back(f.logical);
    PeriodicPlan pp = apply_periodic(chain, logical);
    periodic_exchange(pp.pre_fills, rep);
    chain = std::move(pp.chain);
    on_demand = false;
  }
  if (poison_) poison_stale_halos(chain);
  // Stages: (schedule, loops [begin, end) of the chain it covers).
  std::vector<std::shared_ptr<const DistSchedule>> stages;
  if (on_demand) {
    auto it = dist_->untiled_schedules.find(chain.signature());
    if (it == dist_->untiled_schedules.end()) {
      std::vector<int64_t> pads;
      for (const FieldRec& f : fields_) pads.push_back(f.pad);
      std::vector<std::shared_ptr<const DistSchedule>> v;
      for (DistSchedule& s : build_untiled_schedules(chain, dist_->layout, pads))
        v.push_back(std::make_shared<const DistSchedule>(std::move(s)));
      it = dist_->untiled_schedules.emplace(chain.signature(), std::move(v)).first;
    }
    stages = it->second;
  } else {
    stages.push_back(dist_schedule(chain));
  }
  const std::vector<ReductionHandle> handles = reduction_handles(chain);
  std::vector<ReduceOp> ops;
  for (const LoopRecord& lp : chain.loops)
    if (lp.reduction) ops.push_back(lp.reduction->op);
  const size_t nred = ops.size();
  const int R = dist_->layout.rank_count();
  std::vector<double> part(static_cast<size_t>(R) * nred, 0.0);
  std::string executor;
  size_t red_base = 0;
  for (size_t st = 0; st < stages.size(); ++st) {
    const DistSchedule& sched = *stages[st];
    // The loops this stage runs: the whole chain, or loop `st` alone.
    LoopChain sub;
    if (on_demand) {
      sub.dim = chain.dim;
      sub.stencils = chain.stencils;
      sub.loops.push_back(chain.loops[st]);
    }
    const LoopChain& sc = on_demand ? sub : chain;
    size_t sub_red = 0;
    for (const LoopRecord& lp : sc.loops) sub_red += lp.reduction ? 1 : 0;
    exchange(sched, rep);
    for (int r : dist_->local) {
      const LoopChain lc = with_ranges(sc, sched.ranks[static_cast<size_t>(r)].loop_ranges);
      ExecutionReport rr;
      rr.dim = chain.dim;
      const std::vector<double> v = run_on(lc, mode, rr, dist_->targets[static_cast<size_t>(r)]);
      for (size_t i = 0; i < sub_red; ++i) part[static_cast<size_t>(r) * nred + red_base + i] = v[i];
      rep.tiled = rep.tiled || rr.tiled;
      executor = executor.empty() || executor == rr.executor ? rr.executor : "mixed";
      rep.ctas += rr.ctas;
      rep.subchains += rr.subchains;
      rep.tiles_executed += rr.tiles_executed;
      rep.plan_constructions += rr.plan_constructions;
      rep.plan_seconds += rr.plan_seconds;
      rep.computed_points += rr.tiled ? rr.computed_points : sched.ranks[static_cast<size_t>(r)].computed_points;
      for (int d = 0; d < chain.dim; ++d) {
        rep.max_skew[d] = std::max(rep.max_skew[d], rr.max_skew[d]);
        rep.tile_sizes[d] = rr.tile_sizes[d];
        rep.cta_grid[d] = rr.cta_grid[d];
      }
    }
    red_base += sub_red;
  }
  rep.executor = executor;
  if (comm_ && nred > 0) {
    // Every rank's partials to every process, then the same rank-order fold.
    double* buf = dev.red_buffer((static_cast<size_t>(R) + 1) * nred);
    const size_t me = static_cast<size_t>(proc_rank_);
    dev.h2d(buf, part.data() + me * nred, nred);
    comm_->all_gather(buf, buf + nred, nred, dev.stream());
    dev.d2h(part.data(), buf + nred, static_cast<size_t>(R) * nred);
  }
  std::vector<double> vals(nred);
  for (size_t i = 0; i < nred; ++i) {
    double acc = reduce_identity(ops[i]);
    for (int r = 0; r < R; ++r) acc = reduce_combine(ops[i], acc, part[static_cast<size_t>(r) * nred + i]);
    vals[i] = acc;
  }
  store(handles, vals.data());
  if (note_writes(dist_->written, chain)) ++dist_->hist_version;
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
      // Periodic marks after the reducing loop stay queued with the suffix.
      std::vector<PeriodicMark> later;
      for (auto it = fill_marks_.begin(); it != fill_marks_.end();) {
        if (it->pos > k) {
          it->pos -= k + 1;
          later.push_back(std::move(*it));
          it = fill_marks_.erase(it);
        } else {
          ++it;
        }
      }
      execute_chain(take_pending(), default_mode_);
      for (size_t i = 0; i < suffix.size(); ++i) suffix[i].loop_id = static_cast<int32_t>(i);
      pending_ = std::move(suffix);
      fill_marks_ = std::move(later);
    }
  }
  if (!slot.ready) throw PlanError("fetch_reduction: flush did not produce the value");
  slot.consumed = true;
  return slot.value;
}

// Host access. Distributed: a point is read from its owning rank (padding
// points from the lowest rank whose allocation holds them); writes go to every
// local rank whose allocation holds the point, so replicated halo copies stay
// consistent (the reference re-scatters the global picture each flush,
// dist.cpp:532-545).
int Runtime::root_for(DatasetId ds, const Point& p) {
  const RankLayout& lay = dist_->layout;
  for (int r = 0; r < lay.rank_count(); ++r)
    if (lay.owned[static_cast<size_t>(r)].contains(p)) return r;
  const int64_t pad = fields_.at(static_cast<size_t>(ds)).pad;
  for (int r = 0; r < lay.rank_count(); ++r)
    if (rank_alloc(lay, r, pad).contains(p)) return r;
  throw AccessError("point outside allocated extent " + fields_.at(static_cast<size_t>(ds)).alloc.to_string());
}

double Runtime::get(DatasetId ds, const Point& p) {
  flush();
  if (!distributed()) {
    ensure_fields();
    return device().get_point(fields_.at(static_cast<size_t>(ds)).dev, p);
  }
  ensure_dist();
  const int root = root_for(ds, p);
  double v = 0;
  const Target& t = dist_->targets[static_cast<size_t>(root)];
  const bool local = !t.dev.empty();
  if (local) v = device().get_point(t.dev.at(static_cast<size_t>(ds)), p);
  if (comm_) {
    DeviceExec& dev = device();
    double* buf = dev.red_buffer(1);
    if (local) dev.h2d(buf, &v, 1);
    comm_->broadcast(buf, 1, root, dev.stream());
    dev.d2h(&v, buf, 1);
  }
  return v;
}

void Runtime::put(DatasetId ds, const Point& p, double v) {
  flush();
  if (!distributed()) {
    ensure_fields();
    device().put_point(fields_.at(static_cast<size_t>(ds)).dev, p, v);
    return;
  }
  ensure_dist();
  if (!fields_.at(static_cast<size_t>(ds)).alloc.contains(p))
    throw AccessError("point outside allocated extent " + fields_.at(static_cast<size_t>(ds)).alloc.to_string());
  for (int r : dist_->local) {
    const Target& t = dist_->targets[static_cast<size_t>(r)];
    if (t.alloc[static_cast<size_t>(ds)].contains(p)) device().put_point(t.dev[static_cast<size_t>(ds)], p, v);
  }
}

void Runtime::upload(DatasetId ds, const double* host) {
  flush();
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  if (!distributed()) {
    ensure_fields();
    device().upload(f.dev, host);
    return;
  }
  ensure_dist();
  DeviceExec& dev = device();
  for (int r : dist_->local) {
    const Target& t = dist_->targets[static_cast<size_t>(r)];
    dev.buf_to_field(t.dev[static_cast<size_t>(ds)], t.alloc[static_cast<size_t>(ds)].intersect(f.alloc), host,
                     f.alloc);
  }
  dev.synchronize();
}

void Runtime::download(DatasetId ds, double* host) {
  flush();
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  if (!distributed()) {
    ensure_fields();
    device().download(f.dev, host);
    return;
  }
  ensure_dist();
  DeviceExec& dev = device();
  // Halo/padding copies first, then every owned box (gather, dist.cpp:604-615).
  for (int r : dist_->local) {
    const Target& t = dist_->targets[static_cast<size_t>(r)];
    dev.field_to_buf(t.dev[static_cast<size_t>(ds)], t.alloc[static_cast<size_t>(ds)].intersect(f.alloc), host,
                     f.alloc);
  }
  for (int r : dist_->local) {
    const Target& t = dist_->targets[static_cast<size_t>(r)];
    dev.field_to_buf(t.dev[static_cast<size_t>(ds)], dist_->layout.owned[static_cast<size_t>(r)].intersect(f.logical),
                     host, f.alloc);
  }
  dev.synchronize();
}

void Runtime::upload_box(DatasetId ds, const double* host, const Range& box) {
  flush();
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  if (!f.alloc.contains(box)) throw AccessError("upload_box: " + box.to_string() + " outside " + f.alloc.to_string());
  DeviceExec& dev = device();
  if (!distributed()) {
    ensure_fields();
    dev.buf_to_field(f.dev, box, host, box);
  } else {
    ensure_dist();
    for (int r : dist_->local) {
      const Target& t = dist_->targets[static_cast<size_t>(r)];
      const Range part = t.alloc[static_cast<size_t>(ds)].intersect(box);
      if (!part.empty()) dev.buf_to_field(t.dev[static_cast<size_t>(ds)], part, host, box);
    }
  }
  dev.synchronize();
}

void Runtime::download_box(DatasetId ds, double* host, const Range& box) {
  flush();
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  if (!f.alloc.contains(box)) throw AccessError("download_box: " + box.to_string() + " outside " + f.alloc.to_string());
  DeviceExec& dev = device();
  if (!distributed()) {
    ensure_fields();
    dev.field_to_buf(f.dev, box, host, box);
  } else {
    ensure_dist();
    for (int pass = 0; pass < 2; ++pass)
      for (int r : dist_->local) {
        const Target& t = dist_->targets[static_cast<size_t>(r)];
        const Range part = (pass == 0 ? t.alloc[static_cast<size_t>(ds)]
                                      : dist_->layout.owned[static_cast<size_t>(r)].intersect(f.logical))
                               .intersect(box);
        if (!part.empty()) dev.field_to_buf(t.dev[static_cast<size_t>(ds)], part, host, box);
      }
  }
  dev.synchronize();
}

Range Runtime::local_box(DatasetId ds) {
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  if (!distributed()) return f.alloc;
  const RankLayout& lay = rank_layout();
  std::vector<int> local;
  if (proc_rank_ >= 0)
    local = {proc_rank_};
  else
    for (int r = 0; r < lay.rank_count(); ++r) local.push_back(r);
  Range h = rank_alloc(lay, local[0], f.pad).intersect(f.alloc);
  for (int r : local) h = h.hull(rank_alloc(lay, r, f.pad).intersect(f.alloc));
  return h;
}

void Runtime::periodic_fill(const std::vector<DatasetId>& list, int64_t depth) {
  if (distributed() && (periodic_flush_ || !periodic_domain_))
    throw InvalidArgument("periodic_fill on a rank grid: needs set_periodic_domain(true) and recorded (not eager) fills");
  if (depth < 0) throw InvalidArgument("periodic_fill: negative depth");
  if (recording_) {
    RecordedCall rc;
    rc.fill = true;
    rc.fill_ds = list;
    rc.fill_depth = depth;
    record_cur_.push_back(std::move(rc));
  }
  if (!periodic_flush_) {
    // Recorded: the flush rewrites the chain around it (tcg_periodic.hpp).
    for (DatasetId ds : list) {
      if (ds < 0 || static_cast<size_t>(ds) >= fields_.size())
        throw InvalidArgument("periodic_fill: unknown dataset id " + std::to_string(ds));
      const FieldRec& f = fields_[static_cast<size_t>(ds)];
      if (depth > f.pad) throw AccessError("periodic_fill: depth exceeds the pad of " + f.name);
      for (int d = 0; d < dim_; ++d)
        if (depth > f.logical.extent(d)) throw InvalidArgument("periodic_fill: depth exceeds the extent of " + f.name);
    }
    fill_marks_.push_back(PeriodicMark{pending_.size(), list, depth});
    return;
  }
  flush();
  ensure_fields();
  // Group fields by logical box; one kernel per dimension per group.
  std::vector<std::pair<Range, std::vector<int>>> groups;
  for (DatasetId ds : list) {
    const FieldRec& f = fields_.at(static_cast<size_t>(ds));
    if (depth > f.pad) throw AccessError("periodic_fill: depth exceeds the pad of " + f.name);
    for (int d = 0; d < dim_; ++d)
      if (depth > f.logical.extent(d)) throw InvalidArgument("periodic_fill: depth exceeds the extent of " + f.name);
    bool placed = false;
    for (auto& g : groups)
      if (g.first == f.logical) {
        g.second.push_back(f.dev);
        placed = true;
      }
    if (!placed) groups.emplace_back(f.logical, std::vector<int>{f.dev});
  }
  for (const auto& g : groups) device().periodic_fill(g.second, g.first, depth);
}

void Runtime::fill_logical(DatasetId ds, double v) {
  flush();
  const FieldRec& f = fields_.at(static_cast<size_t>(ds));
  DeviceExec& dev = device();
  auto fill = [&](int idx, const Range& box) {
    if (box.empty()) return;
    std::vector<double> h(static_cast<size_t>(box.volume()), v);
    dev.buf_to_field(idx, box, h.data(), box);
    dev.synchronize();
  };
  if (!distributed()) {
    ensure_fields();
    fill(f.dev, f.logical);
    return;
  }
  ensure_dist();
  for (int r : dist_->local) {
    const Target& t = dist_->targets[static_cast<size_t>(r)];
    fill(t.dev[static_cast<size_t>(ds)], t.alloc[static_cast<size_t>(ds)].intersect(f.logical));
  }
}

}  // namespace tcg
