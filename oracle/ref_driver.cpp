// ORACLE / TEST INFRASTRUCTURE -- not product code.
//
// C-ABI driver around the *unmodified* reference `tilechain` library
// (/root/reference/proj/core/src/*.cpp, compiled where it lies by
// oracle/Makefile into oracle/_ref/libtcref.so). Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, and only as the
// checker or the CPU baseline.
//
// Kernels: the reference runs host closures (kernel_ctx.hpp:15-19). The
// closures built here forward the reference's own checked KernelCtx to the
// shared body registry (paper_1704_00693_b200/csrc/kernels/tc_bodies.h), so
// the reference's planner, executor, lazy queue and simulated distribution
// execute exactly the same per-point expressions as the GPU.
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "tilechain/apps.hpp"
#include "tilechain/dist.hpp"
#include "tilechain/oracle.hpp"
#include "tilechain/runtime.hpp"
#include "tilechain/tile_sizer.hpp"
#include "../paper_1704_00693_b200/csrc/kernels/tc_bodies.h"

using namespace tilechain;

namespace {

thread_local std::string g_err;

struct LoopMeta {
  int nargs = 0;
  int modes[16] = {};
  std::vector<std::vector<Point>> pts;  // per arg: stencil points
  bool reduces = false;
};

// Accessor adapter: the body registry's accessor contract over KernelCtx.
struct RefAcc {
  KernelCtx& c;
  const LoopMeta* m;
  double read(int a, int dx, int dy, int dz) const { return c.read(static_cast<size_t>(a), dx, dy, dz); }
  void write(int a, double v) const { c.write(static_cast<size_t>(a), v); }
  void increment(int a, double v) const { c.increment(static_cast<size_t>(a), v); }
  void contribute(double v) const { c.contribute(v); }
  int nargs() const { return m->nargs; }
  int mode(int a) const { return m->modes[a]; }
  int npts(int a) const { return static_cast<int>(m->pts[static_cast<size_t>(a)].size()); }
  int pt(int a, int j, int d) const {
    return static_cast<int>(m->pts[static_cast<size_t>(a)][static_cast<size_t>(j)][d]);
  }
  bool reduces() const { return m->reduces; }
  int64_t x() const { return c.x(); }
  int64_t y() const { return c.y(); }
  int64_t z() const { return c.z(); }
};

struct Handle {
  std::unique_ptr<Runtime> rt;
  std::vector<std::vector<Point>> stencils;
};

Range range_from(int dim, const int64_t* r6) {
  Range r(dim);
  for (int d = 0; d < dim; ++d) r.set(d, r6[2 * d], r6[2 * d + 1]);
  return r;
}

int64_t put_text(const std::string& s, char* buf, int64_t n) {
  if (buf != nullptr && n > 0) {
    const int64_t k = std::min<int64_t>(n - 1, static_cast<int64_t>(s.size()));
    std::memcpy(buf, s.data(), static_cast<size_t>(k));
    buf[k] = 0;
  }
  return static_cast<int64_t>(s.size()) + 1;
}

template <class F>
int64_t guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// Dense copy between a Field (reference layout: alloc range, dim0 fastest,
// field.cpp:22-26) and a caller buffer of the same layout.
void copy_alloc(Field& f, double* out, const double* in) {
  const size_t n = static_cast<size_t>(f.alloc_range().volume());
  if (in)
    std::memcpy(f.raw(), in, n * sizeof(double));
  else
    std::memcpy(out, f.raw(), n * sizeof(double));
}

std::string halo_text(const HaloSpec& h, int dim) {
  std::ostringstream os;
  for (const auto& [ds, e] : h.entries) {
    os << "ds=" << ds << " needed=" << (e.needed ? 1 : 0);
    for (int d = 0; d < dim; ++d) os << " d" << d << "=" << e.faces[d].lo << "," << e.faces[d].hi;
    os << "\n";
  }
  return os.str();
}

std::string plan_text(const TilingPlan& p, int dim) {
  std::ostringstream os;
  os << p.dump();
  os << "max_skew=";
  for (int d = 0; d < dim; ++d) os << (d ? "," : "") << p.max_skew()[d];
  os << "\n";
  for (const auto& [ds, r] : p.required_extents()) os << "required ds=" << ds << " " << r.to_string() << "\n";
  return os.str();
}

}  // namespace

extern "C" {

const char* tcref_error() { return g_err.c_str(); }

void* tcref_new(int dim, int threads, int64_t skew_allowance, int64_t cache_bytes, int whole_queue) {
  try {
    RuntimeConfig cfg;
    cfg.threads = threads;
    cfg.skew_allowance = skew_allowance;
    cfg.cache_bytes = cache_bytes;
    cfg.flush_whole_queue_on_fetch = whole_queue != 0;
    auto* h = new Handle;
    h->rt = std::make_unique<Runtime>(Block{"ref", dim}, cfg);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void tcref_free(void* h) { delete static_cast<Handle*>(h); }

int64_t tcref_declare_stencil(void* hv, int npts, const int64_t* pts) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    std::vector<Point> v;
    for (int i = 0; i < npts; ++i) v.push_back(Point{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
    h->stencils.push_back(v);
    return h->rt->declare_stencil("s" + std::to_string(h->stencils.size() - 1), v);
  });
}

int64_t tcref_declare_field(void* hv, const char* name, const int64_t* logical6) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    return h->rt->declare_field(name, range_from(h->rt->block().dim, logical6));
  });
}

int64_t tcref_alloc_range(void* hv, int ds, int64_t* out6) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    const Range& a = h->rt->fields()[ds].alloc_range();
    for (int d = 0; d < 3; ++d) {
      out6[2 * d] = d < a.dim() ? a.start(d) : 0;
      out6[2 * d + 1] = d < a.dim() ? a.end(d) : 1;
    }
    return 0;
  });
}

int64_t tcref_put_alloc(void* hv, int ds, const double* data) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    h->rt->flush();
    copy_alloc(h->rt->fields()[ds], nullptr, data);
    return 0;
  });
}

int64_t tcref_get_alloc(void* hv, int ds, double* out) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    h->rt->flush();
    copy_alloc(h->rt->fields()[ds], out, nullptr);
    return 0;
  });
}

int64_t tcref_set_rank_grid(void* hv, const int* g3) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    h->rt->set_rank_grid({g3[0], g3[1], g3[2]});
    return 0;
  });
}

int64_t tcref_set_default_mode(void* hv, int kind, const int64_t* ts3) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    ExecMode m = kind == 0 ? ExecMode::untiled()
                 : kind == 1 ? ExecMode::tiled({ts3[0], ts3[1], ts3[2]})
                             : ExecMode::tiled_auto();
    h->rt->set_default_mode(m);
    return 0;
  });
}

// red: -1 none, else ReduceOp. args: 3 int32 per arg (dataset, stencil, mode).
int64_t tcref_par_loop(void* hv, int kid, int body, int red, const int64_t* range6, int nargs,
                       const int32_t* args, int nparams, const double* params) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    if (!tcb::body_known(body)) throw InvalidArgument("tcref_par_loop: unknown body id");
    auto meta = std::make_shared<LoopMeta>();
    std::vector<ArgSpec> specs;
    meta->nargs = nargs;
    for (int i = 0; i < nargs; ++i) {
      ArgSpec a;
      a.dataset = args[3 * i];
      a.stencil = args[3 * i + 1];
      a.mode = static_cast<AccessMode>(args[3 * i + 2]);
      specs.push_back(a);
      meta->modes[i] = args[3 * i + 2];
      if (a.stencil < 0 || static_cast<size_t>(a.stencil) >= h->stencils.size())
        throw InvalidArgument("par_loop: unknown stencil id " + std::to_string(a.stencil));
      meta->pts.push_back(h->stencils[static_cast<size_t>(a.stencil)]);
    }
    meta->reduces = red >= 0;
    std::vector<double> prm(params, params + nparams);
    KernelHandle k;
    k.id = kid;
    k.name = "k" + std::to_string(kid);
    k.fn = [meta, body, prm](KernelCtx& ctx) {
      RefAcc acc{ctx, meta.get()};
      tcb::run_body(body, acc, prm.data());
    };
    std::optional<ReduceOp> r;
    if (red >= 0) r = static_cast<ReduceOp>(red);
    const ReductionHandle rh =
        h->rt->par_loop(std::move(k), range_from(h->rt->block().dim, range6), specs, r);
    return rh.id;
  });
}

// kind: 0 untiled, 1 tiled(ts), 2 tiled_auto. Report = ExecutionReport::to_text.
int64_t tcref_flush(void* hv, int kind, const int64_t* ts3, char* report, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    ExecMode m = kind == 0 ? ExecMode::untiled()
                 : kind == 1 ? ExecMode::tiled({ts3[0], ts3[1], ts3[2]})
                             : ExecMode::tiled_auto();
    ExecutionReport rep = h->rt->flush(m);
    return put_text(rep.to_text(), report, n);
  });
}

int64_t tcref_fetch(void* hv, int handle, double* out) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    *out = h->rt->fetch_reduction(ReductionHandle{handle});
    return 0;
  });
}

int64_t tcref_last_plan(void* hv, char* buf, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    auto p = h->rt->last_plan();
    if (!p) return put_text("", buf, n);
    return put_text(plan_text(*p, h->rt->block().dim), buf, n);
  });
}

// Consumes the pending queue and returns construct_plan's text
// (planner.cpp:55-208, dump :234-250).
int64_t tcref_plan_pending(void* hv, const int64_t* ts3, char* buf, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    LoopChain chain = h->rt->take_pending();
    TilingPlan plan = construct_plan(chain, {ts3[0], ts3[1], ts3[2]});
    return put_text(plan_text(plan, chain.dim), buf, n);
  });
}

// Consumes the pending queue: the reference's own validators
// (validate_dependencies / validate_coverage, oracle.cpp:154-284) applied to
// an externally built plan for that chain -- ranges[(t*L + l)*6 + 2d + {0,1}]
// over the tile grid of compute_union_bounds(chain, ts). Returns the number of
// violations; their text goes to buf.
int64_t tcref_validate_plan(void* hv, const int64_t* ts3, const int64_t* ranges, int64_t ntiles, int32_t nloops,
                            char* buf, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  int64_t count = -1;
  const int64_t rc = guarded([&]() -> int64_t {
    LoopChain chain = h->rt->take_pending();
    PlanConfig cfg = compute_union_bounds(chain, {ts3[0], ts3[1], ts3[2]});
    if (cfg.total_tiles() != ntiles || static_cast<int32_t>(chain.size()) != nloops)
      throw InvalidArgument("validate_plan: plan shape does not match the chain's tile grid");
    std::vector<Range> rs;
    for (int64_t i = 0; i < ntiles * nloops; ++i) {
      Range r(chain.dim);
      for (int d = 0; d < chain.dim; ++d) r.set(d, ranges[i * 6 + 2 * d], ranges[i * 6 + 2 * d + 1]);
      rs.push_back(r);
    }
    TilingPlan plan(cfg, chain.signature(), nloops, std::move(rs), {}, 0.0);
    std::vector<oracle::Violation> v = oracle::validate_dependencies(plan, chain, 32);
    for (const oracle::Violation& x : oracle::validate_coverage(plan, chain, 32)) v.push_back(x);
    std::ostringstream os;
    for (const oracle::Violation& x : v) os << x.to_string() << "\n";
    count = static_cast<int64_t>(v.size());
    return put_text(os.str(), buf, n);
  });
  return rc < 0 ? rc : count;
}

// Consumes the pending queue: the reference's validators applied to a set of
// overlapped single-tile plans -- one per "rank", here one per CTA of the
// streaming executor (a CTA recomputes its halo like a rank of
// construct_rank_plan, dist.cpp:268-310). ranges[(r*L + l)*6 ...] is the box
// rank r computes of loop l (empty = not executed), owned[r*6 ...] its owned
// box, band[d] the replication band allowed around the owned cuts, skip[l] != 0
// marks loops the executor drops (their output is dead).
//   * validate_dependencies (oracle.cpp:154-223) per rank: every point a rank
//     reads must have been produced, inside the same rank, by the loop that
//     produces it in sequential order (nothing may come from a neighbour);
//   * validate_coverage_replicated (oracle.cpp:286-344) over the owned parts:
//     every recorded point owned exactly once.
// Returns the number of violations; text to buf.
int64_t tcref_validate_rank_plans(void* hv, int32_t nranks, int32_t nloops, const int64_t* ranges, const int64_t* owned,
                                  const int64_t* band3, const int32_t* skip, char* buf, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  int64_t count = -1;
  const int64_t rc = guarded([&]() -> int64_t {
    LoopChain chain = h->rt->take_pending();
    if (static_cast<int32_t>(chain.size()) != nloops) throw InvalidArgument("validate_rank_plans: loop count differs");
    const int64_t big = int64_t{1} << 40;
    PlanConfig cfg = compute_union_bounds(chain, {big, big, big});
    if (cfg.total_tiles() != 1) throw InvalidArgument("validate_rank_plans: expected a single-tile grid");
    auto box = [&](const int64_t* p) {
      Range r(chain.dim);
      for (int d = 0; d < chain.dim; ++d) r.set(d, p[2 * d], std::max(p[2 * d], p[2 * d + 1]));
      return r;
    };
    std::vector<oracle::Violation> v;
    std::vector<TilingPlan> exec_plans, own_plans;
    std::vector<Range> own;
    for (int32_t r = 0; r < nranks; ++r) {
      std::vector<Range> rs, os;
      const Range ob = box(owned + static_cast<size_t>(r) * 6);
      own.push_back(ob);
      for (int32_t l = 0; l < nloops; ++l) {
        const Range x = box(ranges + (static_cast<size_t>(r) * nloops + l) * 6);
        rs.push_back(x);
        os.push_back(skip[l] ? x : x.intersect(ob));
      }
      exec_plans.emplace_back(cfg, chain.signature(), nloops, std::move(rs), DependencyExtents{}, 0.0);
      own_plans.emplace_back(cfg, chain.signature(), nloops, std::move(os), DependencyExtents{}, 0.0);
    }
    for (int32_t r = 0; r < nranks && v.size() < 32; ++r)
      for (oracle::Violation& x : oracle::validate_dependencies(exec_plans[static_cast<size_t>(r)], chain, 8)) {
        x.detail += " [rank " + std::to_string(r) + "]";
        v.push_back(x);
      }
    std::vector<const TilingPlan*> ptrs;
    for (const TilingPlan& p : own_plans) ptrs.push_back(&p);
    for (const oracle::Violation& x :
         oracle::validate_coverage_replicated(ptrs, chain, own, {band3[0], band3[1], band3[2]}, 32)) {
      if (x.loop >= 0 && x.loop < nloops && skip[x.loop]) continue;
      v.push_back(x);
    }
    std::ostringstream os;
    for (const oracle::Violation& x : v) os << x.to_string() << "\n";
    count = static_cast<int64_t>(v.size());
    return put_text(os.str(), buf, n);
  });
  return rc < 0 ? rc : count;
}

// Consumes the pending queue; per rank of decompose(global, grid):
// construct_rank_plan (dist.cpp:191-390) + compute_halo_depths (:407-448).
int64_t tcref_rank_plans_pending(void* hv, const int* g3, const int64_t* ts3, char* buf, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    LoopChain chain = h->rt->take_pending();
    bool first = true;
    Range global(chain.dim);
    for (const Field& f : h->rt->fields()) {
      global = first ? f.logical_range() : global.hull(f.logical_range());
      first = false;
    }
    RankLayout layout = decompose(global, {g3[0], g3[1], g3[2]});
    std::ostringstream os;
    for (int r = 0; r < layout.rank_count(); ++r) {
      TilingPlan p = construct_rank_plan(chain, layout, r, {ts3[0], ts3[1], ts3[2]});
      os << "rank=" << r << " owned=" << layout.owned[static_cast<size_t>(r)].to_string() << "\n";
      os << plan_text(p, chain.dim);
      os << halo_text(compute_halo_depths(p, chain, layout, r), chain.dim);
    }
    return put_text(os.str(), buf, n);
  });
}

// Distributed-run introspection after a flush with a rank grid.
int64_t tcref_dist_info(void* hv, char* buf, int64_t n) {
  auto* h = static_cast<Handle*>(hv);
  return guarded([&]() -> int64_t {
    DistContext* dc = h->rt->dist();
    if (dc == nullptr) return put_text("", buf, n);
    std::ostringstream os;
    for (int r = 0; r < dc->rank_count(); ++r) {
      os << "rank=" << r << "\n" << halo_text(dc->last_rank_halos(r), h->rt->block().dim);
    }
    for (const MessageRecord& m : dc->log().messages)
      os << "msg from=" << m.from << " to=" << m.to << " ds=" << m.dataset << " dim=" << m.dim
         << " dir=" << m.dir << " points=" << m.points << " bytes=" << m.bytes << "\n";
    return put_text(os.str(), buf, n);
  });
}

// tile_sizer.cpp:27-81
int64_t tcref_auto_tile_size(int dim, int64_t cache_bytes, int threads, int64_t bpp,
                             const int64_t* extent6, int64_t* out3) {
  return guarded([&]() -> int64_t {
    SizerInput in;
    in.dim = dim;
    in.cache_bytes = cache_bytes;
    in.threads = threads;
    in.bytes_per_point = bpp;
    in.domain_extent = range_from(dim, extent6);
    const auto ts = auto_tile_size(in);
    for (int d = 0; d < 3; ++d) out3[d] = ts[d];
    return 0;
  });
}

// Reference apps end to end (apps.cpp): pins this project's copies of the
// jacobi / mini-hydro bodies against the reference's own closures.
// Outputs: logical-range values of every dataset, concatenated in id order;
// monitors for mini-hydro.
int64_t tcref_app_jacobi(int64_t nx, int64_t ny, int iters, int copy_variant, double* out) {
  return guarded([&]() -> int64_t {
    apps::AppConfig cfg;
    cfg.nx = nx;
    cfg.ny = ny;
    cfg.iters = iters;
    cfg.variant = copy_variant ? "copy" : "noncopy";
    FieldTable f = apps::jacobi_reference(cfg);
    size_t k = 0;
    for (const Field& fld : f)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) out[k++] = fld.read(pt(x, y));
    return static_cast<int64_t>(k);
  });
}

int64_t tcref_app_minihydro(int64_t nx, int64_t ny, int iters, double* out, double* monitors) {
  return guarded([&]() -> int64_t {
    apps::AppConfig cfg;
    cfg.nx = nx;
    cfg.ny = ny;
    cfg.iters = iters;
    auto [f, mon] = apps::minihydro_reference(cfg);
    size_t k = 0;
    for (const Field& fld : f)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) out[k++] = fld.read(pt(x, y));
    for (size_t i = 0; i < mon.size(); ++i) monitors[i] = mon[i];
    return static_cast<int64_t>(k);
  });
}

}  // extern "C"
