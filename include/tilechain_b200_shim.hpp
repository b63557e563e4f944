// The C++ shim a tilechain maintainer adds on the reference side: the
// reference's own types (Range, ArgSpec, ReduceOp, RuntimeConfig, ExecMode,
// exceptions; proj/core/include/tilechain/types.hpp, runtime.hpp:13-35) over
// the C-ABI of tilechain_b200.h. Error codes are rethrown as the reference's
// exception types. Compiled and run by tests/test_shim.py against the
// reference headers (in this container; the product never includes them).
//
// The one difference from tilechain::Runtime::par_loop (runtime.hpp:59-63): a
// kernel is {id, registry body, scalar parameters} instead of a host closure
// (INTEGRATION.md "Kernels").
#pragma once
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include <tilechain/runtime.hpp>  // RuntimeConfig, ExecMode
#include <tilechain/types.hpp>    // Range, ArgSpec, ReduceOp, ReductionHandle, errors

#include "tilechain_b200.h"

namespace tilechain::b200 {

inline void check(int rc) {
  if (rc == TCG_OK) return;
  char msg[1024];
  tcg_last_error(msg, sizeof msg);
  switch (rc) {
    case TCG_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
    case TCG_ERR_ACCESS: throw AccessError(msg);
    case TCG_ERR_PLAN: throw PlanError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void range6(const Range& r, int64_t o[6]) {
  for (int d = 0; d < 3; ++d) {
    o[2 * d] = d < r.dim() ? r.start(d) : 0;
    o[2 * d + 1] = d < r.dim() ? r.end(d) : 1;
  }
}

class Runtime {
 public:
  explicit Runtime(int dim, const RuntimeConfig& c = {}) {
    tcg_config cfg{c.threads, c.skew_allowance, c.cache_bytes, c.flush_whole_queue_on_fetch ? 1 : 0, 0};
    check(tcg_runtime_new(dim, &cfg, &rt_));
  }
  ~Runtime() { tcg_runtime_free(rt_); }
  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;

  StencilId declare_stencil(const std::string&, const std::vector<Point>& offsets) {
    std::vector<int64_t> p;
    for (const Point& q : offsets) p.insert(p.end(), {q[0], q[1], q[2]});
    int32_t id = -1;
    check(tcg_declare_stencil(rt_, static_cast<int>(offsets.size()), p.data(), &id));
    return id;
  }
  DatasetId declare_field(const std::string& name, const Range& logical) {
    int64_t r[6];
    range6(logical, r);
    int32_t id = -1;
    check(tcg_declare_field(rt_, name.c_str(), r, &id));
    return id;
  }
  ReductionHandle par_loop(int32_t kernel_id, int32_t body, std::span<const double> params, const Range& range,
                           const std::vector<ArgSpec>& args, std::optional<ReduceOp> red = std::nullopt) {
    int64_t r[6];
    range6(range, r);
    std::vector<int32_t> a;
    for (const ArgSpec& s : args) a.insert(a.end(), {s.dataset, s.stencil, static_cast<int32_t>(s.mode)});
    int32_t h = -1;
    check(tcg_par_loop(rt_, kernel_id, body, r, static_cast<int>(args.size()), a.data(),
                       red ? static_cast<int>(*red) : TCG_RED_NONE, static_cast<int>(params.size()), params.data(), &h));
    return ReductionHandle{h};
  }
  void flush(const ExecMode& m) {
    const int64_t ts[3] = {m.tile_sizes[0], m.tile_sizes[1], m.tile_sizes[2]};
    check(tcg_flush(rt_, static_cast<int>(m.kind), ts));
  }
  void flush() { check(tcg_flush_default(rt_)); }
  double fetch_reduction(ReductionHandle h) {
    double v = 0;
    check(tcg_fetch_reduction(rt_, h.id, &v));
    return v;
  }
  double get(DatasetId ds, const Point& p) {
    const int64_t q[3] = {p[0], p[1], p[2]};
    double v = 0;
    check(tcg_get(rt_, ds, q, &v));
    return v;
  }
  void put(DatasetId ds, const Point& p, double v) {
    const int64_t q[3] = {p[0], p[1], p[2]};
    check(tcg_put(rt_, ds, q, v));
  }
  void fill_logical(DatasetId ds, double v) { check(tcg_fill_logical(rt_, ds, v)); }
  size_t pending_loops() {
    int64_t n = 0;
    check(tcg_pending_loops(rt_, &n));
    return static_cast<size_t>(n);
  }
  tcg_runtime* handle() { return rt_; }

 private:
  tcg_runtime* rt_ = nullptr;
};

}  // namespace tilechain::b200
