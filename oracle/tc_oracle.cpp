// ORACLE / TEST INFRASTRUCTURE -- not product code. Only tests/, smoke() and
// bench.py's cpu_baseline leg may load it, and only as the checker.
//
// A plain, strictly sequential CPU restatement of the reference's ground
// truth for the hot path:
//   * field storage: dense fp64 over logical +- pad, dim 0 fastest, zero
//     initialised (proj/core/src/field.cpp:7-28); pad = widest stencil reach
//     declared so far + skew_allowance (proj/core/src/runtime.cpp:16-33);
//   * sequential_reference: loops in chain order, points lexicographic with
//     dim 0 fastest, one thread, reduction folded in visit order from the
//     identity (proj/core/src/oracle.cpp:124-152, types.hpp:272-288);
//   * checked access like KernelCtx (kernel_ctx.hpp:58-89): mode, exact
//     stencil membership, allocation bounds.
// Laziness never changes values (the reference's lazy queue preserves the
// sequential story, runtime.hpp:40-60), so this oracle executes every loop
// eagerly at enqueue time.
//
// Pinned by tests/test_oracle.py against the reference's own known answers
// (test_oracle.cpp:73-118 sum = 42, test_apps.cpp jacobi/mini-hydro) and
// against the unmodified reference library (oracle/_ref) on the same inputs.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../paper_1704_00693_b200/csrc/kernels/tc_bodies.h"

namespace {

thread_local std::string g_err;

struct OStencil {
  std::vector<std::array<int64_t, 3>> pts;
  int64_t reach = 0;
};

struct OField {
  int64_t lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};  // allocation box
  int64_t stride[3] = {1, 0, 0};
  std::vector<double> v;
  size_t idx(int64_t x, int64_t y, int64_t z) const {
    return static_cast<size_t>((x - lo[0]) * stride[0] + (y - lo[1]) * stride[1] + (z - lo[2]) * stride[2]);
  }
  bool inside(int64_t x, int64_t y, int64_t z) const {
    return x >= lo[0] && x < hi[0] && y >= lo[1] && y < hi[1] && z >= lo[2] && z < hi[2];
  }
};

struct ORuntime {
  int dim = 1;
  int64_t skew_allowance = 16;
  int64_t max_reach = 0;
  std::vector<OStencil> stencils;
  std::vector<OField> fields;
  std::vector<double> reductions;
  std::vector<int> fetched;
  bool masked = false;            // execute_plan's reduction_mask (executor.cpp:209-250)
  int64_t mlo[3] = {0, 0, 0}, mhi[3] = {1, 1, 1};
};

struct OArg {
  OField* f;
  const OStencil* s;
  int mode;
};

struct OAcc {
  const std::vector<OArg>* args;
  int64_t p[3];
  int red_op = -1;
  double* red = nullptr;
  const ORuntime* rt = nullptr;

  [[noreturn]] void fail(const char* why) const { throw std::runtime_error(why); }
  double read(int a, int dx, int dy, int dz) const {
    const OArg& g = (*args)[static_cast<size_t>(a)];
    if (g.mode == tcb::kWrite) fail("read through write-only arg");
    bool member = false;
    for (const auto& q : g.s->pts) member = member || (q[0] == dx && q[1] == dy && q[2] == dz);
    if (!member) fail("offset not in declared stencil");
    if (!g.f->inside(p[0] + dx, p[1] + dy, p[2] + dz)) fail("outside allocated extent");
    return g.f->v[g.f->idx(p[0] + dx, p[1] + dy, p[2] + dz)];
  }
  void write(int a, double v) const {
    const OArg& g = (*args)[static_cast<size_t>(a)];
    if (g.mode == tcb::kRead) fail("write through read-only arg");
    if (!g.f->inside(p[0], p[1], p[2])) fail("outside allocated extent");
    g.f->v[g.f->idx(p[0], p[1], p[2])] = v;
  }
  void increment(int a, double v) const {
    const OArg& g = (*args)[static_cast<size_t>(a)];
    if (g.mode != tcb::kReadWrite && g.mode != tcb::kIncrement) fail("increment needs a readwrite/increment arg");
    if (!g.f->inside(p[0], p[1], p[2])) fail("outside allocated extent");
    g.f->v[g.f->idx(p[0], p[1], p[2])] += v;
  }
  void contribute(double v) const {
    if (red == nullptr) fail("contribute() without a declared reduction");
    if (rt && rt->masked)  // kernel_ctx.hpp:87: points outside the mask do not contribute
      for (int d = 0; d < 3; ++d)
        if (p[d] < rt->mlo[d] || p[d] >= rt->mhi[d]) return;
    if (red_op == tcb::kSum)
      *red = *red + v;
    else if (red_op == tcb::kMin)
      *red = *red < v ? *red : v;
    else
      *red = *red > v ? *red : v;
  }
  int nargs() const { return static_cast<int>(args->size()); }
  int mode(int a) const { return (*args)[static_cast<size_t>(a)].mode; }
  int npts(int a) const { return static_cast<int>((*args)[static_cast<size_t>(a)].s->pts.size()); }
  int pt(int a, int j, int d) const {
    return static_cast<int>((*args)[static_cast<size_t>(a)].s->pts[static_cast<size_t>(j)][d]);
  }
  bool reduces() const { return red != nullptr; }
  int64_t x() const { return p[0]; }
  int64_t y() const { return p[1]; }
  int64_t z() const { return p[2]; }
};

double identity(int op) {
  return op == tcb::kSum ? 0.0
         : op == tcb::kMin ? std::numeric_limits<double>::infinity()
                           : -std::numeric_limits<double>::infinity();
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

}  // namespace

extern "C" {

const char* tco_error() { return g_err.c_str(); }

void* tco_new(int dim, int64_t skew_allowance) {
  auto* r = new ORuntime;
  r->dim = dim;
  r->skew_allowance = skew_allowance;
  return r;
}

void tco_free(void* h) { delete static_cast<ORuntime*>(h); }

int64_t tco_declare_stencil(void* hv, int npts, const int64_t* pts) {
  auto* r = static_cast<ORuntime*>(hv);
  return guarded([&]() -> int64_t {
    if (npts <= 0) throw std::runtime_error("Stencil: empty point set");
    OStencil s;
    for (int i = 0; i < npts; ++i) {
      s.pts.push_back({pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
      for (int d = 0; d < r->dim; ++d) s.reach = std::max<int64_t>(s.reach, std::llabs(pts[3 * i + d]));
    }
    r->max_reach = std::max(r->max_reach, s.reach);
    r->stencils.push_back(s);
    return static_cast<int64_t>(r->stencils.size()) - 1;
  });
}

int64_t tco_declare_field(void* hv, const char*, const int64_t* logical6) {
  auto* r = static_cast<ORuntime*>(hv);
  return guarded([&]() -> int64_t {
    const int64_t pad = r->max_reach + r->skew_allowance;  // runtime.cpp:30
    OField f;
    int64_t stride = 1;
    for (int d = 0; d < 3; ++d) {
      if (d < r->dim) {
        f.lo[d] = logical6[2 * d] - pad;
        f.hi[d] = logical6[2 * d + 1] + pad;
        f.stride[d] = stride;
        stride *= f.hi[d] - f.lo[d];
      } else {
        f.lo[d] = 0;
        f.hi[d] = 1;
        f.stride[d] = 0;
      }
    }
    f.v.assign(static_cast<size_t>(stride), 0.0);  // field.cpp:27
    r->fields.push_back(std::move(f));
    return static_cast<int64_t>(r->fields.size()) - 1;
  });
}

int64_t tco_put_alloc(void* hv, int ds, const double* data) {
  auto* r = static_cast<ORuntime*>(hv);
  OField& f = r->fields.at(static_cast<size_t>(ds));
  std::memcpy(f.v.data(), data, f.v.size() * sizeof(double));
  return 0;
}

int64_t tco_get_alloc(void* hv, int ds, double* out) {
  auto* r = static_cast<ORuntime*>(hv);
  const OField& f = r->fields.at(static_cast<size_t>(ds));
  std::memcpy(out, f.v.data(), f.v.size() * sizeof(double));
  return 0;
}

// Executes the loop immediately (oracle.cpp:124-152). Returns the reduction
// handle (>= 0), -1 for none, -2 on error.
int64_t tco_par_loop(void* hv, int, int body, int red, const int64_t* range6, int nargs,
                     const int32_t* args, int, const double* params) {
  auto* r = static_cast<ORuntime*>(hv);
  return guarded([&]() -> int64_t {
    if (!tcb::body_known(body)) throw std::runtime_error("unknown body id");
    std::vector<OArg> a;
    for (int i = 0; i < nargs; ++i)
      a.push_back(OArg{&r->fields.at(static_cast<size_t>(args[3 * i])),
                       &r->stencils.at(static_cast<size_t>(args[3 * i + 1])), args[3 * i + 2]});
    double accum = red >= 0 ? identity(red) : 0.0;
    OAcc acc;
    acc.args = &a;
    acc.red_op = red;
    acc.red = red >= 0 ? &accum : nullptr;
    acc.rt = r;
    int64_t lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = d < r->dim ? range6[2 * d] : 0;
      hi[d] = d < r->dim ? range6[2 * d + 1] : 1;
    }
    for (int64_t z = lo[2]; z < hi[2]; ++z)
      for (int64_t y = lo[1]; y < hi[1]; ++y)
        for (int64_t x = lo[0]; x < hi[0]; ++x) {
          acc.p[0] = x;
          acc.p[1] = y;
          acc.p[2] = z;
          tcb::run_body(body, acc, params);
        }
    if (red < 0) return -1;
    r->reductions.push_back(accum);
    r->fetched.push_back(0);
    return static_cast<int64_t>(r->reductions.size()) - 1;
  });
}

// Reduction mask for the following loops (NULL clears it); a rank's owned box
// in the distributed tests.
int64_t tco_set_reduction_mask(void* hv, const int64_t* range6) {
  auto* r = static_cast<ORuntime*>(hv);
  r->masked = range6 != nullptr;
  for (int d = 0; d < 3; ++d) {
    r->mlo[d] = range6 && d < r->dim ? range6[2 * d] : 0;
    r->mhi[d] = range6 && d < r->dim ? range6[2 * d + 1] : 1;
  }
  return 0;
}

int64_t tco_fetch(void* hv, int handle, double* out) {
  auto* r = static_cast<ORuntime*>(hv);
  return guarded([&]() -> int64_t {
    if (handle < 0 || static_cast<size_t>(handle) >= r->reductions.size())
      throw std::runtime_error("fetch_reduction: unknown handle");
    if (r->fetched[static_cast<size_t>(handle)]) throw std::runtime_error("fetch_reduction: handle already fetched");
    r->fetched[static_cast<size_t>(handle)] = 1;
    *out = r->reductions[static_cast<size_t>(handle)];
    return 0;
  });
}

}  // extern "C"
