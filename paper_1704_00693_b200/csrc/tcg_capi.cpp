// C-ABI boundary (include/tilechain_b200.h): plain pointers and sizes in,
// status codes out; every C++ exception is translated to its TCG_ERR_* code.
#include "../../include/tilechain_b200.h"

#include <cstring>
#include <sstream>

#include "host/tcg_jit.hpp"
#include "host/tcg_runtime.hpp"
#include "kernels/tc_bodies.h"

struct tcg_runtime {
  std::unique_ptr<tcg::Runtime> rt;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return TCG_OK;
  } catch (const tcg::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TCG_ERR_INTERNAL;
  }
}

tcg::Range range6(int dim, const int64_t* r) { return tcg::Range::box(dim, r); }

tcg::ExecMode mode_of(int mode, const int64_t* ts) {
  if (mode == TCG_UNTILED) return tcg::ExecMode::untiled();
  if (mode == TCG_TILED) return tcg::ExecMode::tiled({ts[0], ts[1], ts[2]});
  if (mode == TCG_TILED_AUTO) return tcg::ExecMode::tiled_auto();
  if (mode == TCG_WINDOWED) return tcg::ExecMode::windowed({ts[0], ts[1], ts[2]});
  if (mode == TCG_STREAM) return tcg::ExecMode::stream();
  throw tcg::InvalidArgument("unknown exec mode " + std::to_string(mode));
}

void put_text(const std::string& s, char* buf, int64_t n, int64_t* needed) {
  if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
  if (buf && n > 0) {
    const size_t k = std::min<size_t>(static_cast<size_t>(n) - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
}

std::string plan_text(const tcg::TilingPlan& p, int dim) {
  std::ostringstream os;
  os << p.dump() << "max_skew=";
  for (int d = 0; d < dim; ++d) os << (d ? "," : "") << p.max_skew[d];
  os << "\n";
  for (const auto& [ds, r] : p.required) os << "required ds=" << ds << " " << r.to_string() << "\n";
  return os.str();
}

std::string halo_text(const tcg::HaloSpec& h, int dim) {
  std::ostringstream os;
  for (const auto& [ds, e] : h.entries) {
    os << "ds=" << ds << " needed=" << (e.needed ? 1 : 0);
    for (int d = 0; d < dim; ++d) os << " d" << d << "=" << e.faces[d].lo << "," << e.faces[d].hi;
    os << "\n";
  }
  return os.str();
}

// B200 constants for plan-only calls on a machine without a GPU.
constexpr int kB200Sms = 148;
constexpr int64_t kB200SmemOptin = 232448;

}  // namespace

extern "C" {

size_t tcg_last_error(char* buf, size_t n) {
  if (buf && n > 0) {
    const size_t k = std::min(n - 1, g_err.size());
    std::memcpy(buf, g_err.data(), k);
    buf[k] = 0;
  }
  return g_err.size();
}

int tcg_abi_version(void) { return 1; }

int tcg_runtime_new(int dim, const tcg_config* cfg, tcg_runtime** out) {
  return guard([&] {
    tcg::RuntimeConfig c;
    if (cfg) {
      c.threads = cfg->threads;
      c.skew_allowance = cfg->skew_allowance;
      c.cache_bytes = cfg->cache_bytes;
      c.flush_whole_queue_on_fetch = cfg->flush_whole_queue_on_fetch != 0;
      c.stream_segments = cfg->stream_segments;
    }
    auto* h = new tcg_runtime;
    h->rt = std::make_unique<tcg::Runtime>(dim, c);
    *out = h;
  });
}

void tcg_runtime_free(tcg_runtime* rt) { delete rt; }

int tcg_declare_stencil(tcg_runtime* rt, int npts, const int64_t* pts, int32_t* out_id) {
  return guard([&] {
    std::vector<tcg::Point> v;
    for (int i = 0; i < npts; ++i) v.push_back(tcg::Point{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
    *out_id = rt->rt->declare_stencil("", std::move(v));
  });
}

int tcg_declare_field(tcg_runtime* rt, const char* name, const int64_t logical[6], int32_t* out_id) {
  return guard([&] { *out_id = rt->rt->declare_field(name ? name : "", range6(rt->rt->dim(), logical)); });
}

int tcg_alloc_range(tcg_runtime* rt, int32_t ds, int64_t out[6]) {
  return guard([&] {
    if (ds < 0 || static_cast<size_t>(ds) >= rt->rt->num_fields()) throw tcg::InvalidArgument("unknown dataset");
    const tcg::Range& a = rt->rt->alloc_range(ds);
    for (int d = 0; d < 3; ++d) {
      out[2 * d] = d < a.dim() ? a.start(d) : 0;
      out[2 * d + 1] = d < a.dim() ? a.end(d) : 1;
    }
  });
}

int tcg_par_loop(tcg_runtime* rt, int32_t kernel_id, int32_t body, const int64_t range[6], int nargs,
                 const int32_t* args, int red_op, int nparams, const double* params, int32_t* out_handle) {
  return guard([&] {
    tcg::KernelHandle k;
    k.id = kernel_id;
    k.name = "k" + std::to_string(kernel_id);
    k.fn.body = body;
    if (nparams > 0) k.fn.params.assign(params, params + nparams);
    std::vector<tcg::ArgSpec> a;
    for (int i = 0; i < nargs; ++i) {
      if (args[3 * i + 2] < 0 || args[3 * i + 2] > 3) throw tcg::InvalidArgument("par_loop: bad access mode");
      a.push_back(tcg::ArgSpec{args[3 * i], args[3 * i + 1], static_cast<tcg::AccessMode>(args[3 * i + 2])});
    }
    std::optional<tcg::ReduceOp> r;
    if (red_op >= 0) {
      if (red_op > 2) throw tcg::InvalidArgument("par_loop: bad reduction op");
      r = static_cast<tcg::ReduceOp>(red_op);
    }
    const tcg::ReductionHandle h = rt->rt->par_loop(std::move(k), range6(rt->rt->dim(), range), std::move(a), r);
    if (out_handle) *out_handle = h.id;
  });
}

int tcg_flush(tcg_runtime* rt, int mode, const int64_t ts[3]) {
  return guard([&] {
    const int64_t z[3] = {0, 0, 0};
    rt->rt->flush(mode_of(mode, ts ? ts : z));
  });
}

int tcg_flush_default(tcg_runtime* rt) {
  return guard([&] { rt->rt->flush(); });
}

int tcg_set_default_mode(tcg_runtime* rt, int mode, const int64_t ts[3]) {
  return guard([&] {
    const int64_t z[3] = {0, 0, 0};
    rt->rt->set_default_mode(mode_of(mode, ts ? ts : z));
  });
}

int tcg_fetch_reduction(tcg_runtime* rt, int32_t handle, double* out) {
  return guard([&] { *out = rt->rt->fetch_reduction(tcg::ReductionHandle{handle}); });
}

int tcg_pending_loops(tcg_runtime* rt, int64_t* out) {
  return guard([&] { *out = static_cast<int64_t>(rt->rt->pending_loops()); });
}

int tcg_get(tcg_runtime* rt, int32_t ds, const int64_t p[3], double* out) {
  return guard([&] { *out = rt->rt->get(ds, tcg::Point{p[0], p[1], p[2]}); });
}

int tcg_put(tcg_runtime* rt, int32_t ds, const int64_t p[3], double v) {
  return guard([&] { rt->rt->put(ds, tcg::Point{p[0], p[1], p[2]}, v); });
}

int tcg_fill_logical(tcg_runtime* rt, int32_t ds, double v) {
  return guard([&] { rt->rt->fill_logical(ds, v); });
}

int tcg_upload(tcg_runtime* rt, int32_t ds, const double* host) {
  return guard([&] {
    if (ds < 0 || static_cast<size_t>(ds) >= rt->rt->num_fields()) throw tcg::InvalidArgument("unknown dataset");
    rt->rt->upload(ds, host);
  });
}

int tcg_download(tcg_runtime* rt, int32_t ds, double* host) {
  return guard([&] {
    if (ds < 0 || static_cast<size_t>(ds) >= rt->rt->num_fields()) throw tcg::InvalidArgument("unknown dataset");
    rt->rt->download(ds, host);
  });
}

int tcg_synchronize(tcg_runtime* rt) {
  return guard([&] {
    if (rt->rt->device_ready()) rt->rt->device().synchronize();
  });
}

int tcg_report_text(tcg_runtime* rt, char* buf, int64_t n, int64_t* needed) {
  return guard([&] { put_text(rt->rt->last_report().to_text(), buf, n, needed); });
}

int tcg_set_stream_choice(tcg_runtime* rt, const int32_t cfg[8]) {
  return guard([&] {
    tcg::StreamChoice c;
    c.nt = cfg[0];
    c.bx = cfg[1];
    c.by = cfg[2];
    c.ntx = cfg[3];
    c.segments = cfg[4];
    c.max_loops = cfg[5];
    c.minb = cfg[6];
    c.prefetch = cfg[7];
    rt->rt->set_stream_choice(c);
  });
}

int tcg_stream_plan_pending(tcg_runtime* rt, int what, char* buf, int64_t n, int64_t* needed) {
  return guard([&] {
    tcg::StreamDevice sd;  // B200: 148 SMs, 227 KB opt-in shared memory per CTA
    const tcg::StreamPlan p = rt->rt->stream_plan_pending(sd);
    std::string out = p.summary();
    for (size_t i = 0; i < p.kernels.size(); ++i) {
      const tcg::StreamKernel& k = p.kernels[i];
      if (what & 1) {
        std::string log;
        const std::string cubin = k.nctas ? tcg::jit_compile_cubin(k.source, &log) : std::string();
        out += "compiled kernel " + std::to_string(i) + " cubin_bytes=" + std::to_string(cubin.size()) + "\n";
        if (!log.empty()) out += log + "\n";
      }
      if (what & 2) out += "----- source kernel " + std::to_string(i) + "\n" + k.source;
      if ((what & 4) && k.nctas) out += "----- ctas kernel " + std::to_string(i) + "\n" + k.cta_text(k.grid[2]);
    }
    put_text(out, buf, n, needed);
  });
}

int tcg_periodic_plan_pending(tcg_runtime* rt, char* buf, int64_t n, int64_t* needed) {
  return guard([&] {
    tcg::LoopChain c = rt->rt->take_pending();
    std::vector<tcg::Range> logical;
    for (size_t i = 0; i < rt->rt->num_fields(); ++i) logical.push_back(rt->rt->logical_range(static_cast<tcg::DatasetId>(i)));
    const tcg::PeriodicPlan p = tcg::apply_periodic(c, logical);
    std::ostringstream os;
    os << "loops=" << p.chain.size() << " marks=" << c.fills.size() << " max_extension=" << p.max_extension
       << " extended_points=" << p.extended_points << "\n";
    for (size_t l = 0; l < p.chain.size(); ++l)
      os << "loop=" << l << " " << c.loops[l].kernel.name << " range=" << p.chain.loops[l].range.to_string() << "\n";
    for (const auto& [ds, depth] : p.pre_fills) os << "wrap ds=" << ds << " depth=" << depth << "\n";
    put_text(os.str(), buf, n, needed);
  });
}

int tcg_plan_pending(tcg_runtime* rt, const int64_t ts[3], char* buf, int64_t n, int64_t* needed) {
  return guard([&] {
    tcg::LoopChain c = rt->rt->take_pending();
    const tcg::TilingPlan p = tcg::construct_plan(c, {ts[0], ts[1], ts[2]});
    put_text(plan_text(p, c.dim), buf, n, needed);
  });
}

int tcg_rank_plans_pending(tcg_runtime* rt, const int32_t grid[3], const int64_t ts[3], char* buf, int64_t n,
                           int64_t* needed) {
  return guard([&] {
    tcg::LoopChain c = rt->rt->take_pending();
    bool first = true;
    tcg::Range global(c.dim);
    for (size_t i = 0; i < rt->rt->num_fields(); ++i) {
      const tcg::Range& l = rt->rt->logical_range(static_cast<tcg::DatasetId>(i));
      global = first ? l : global.hull(l);
      first = false;
    }
    const tcg::RankLayout lay = tcg::decompose(global, {grid[0], grid[1], grid[2]});
    std::ostringstream os;
    for (int r = 0; r < lay.rank_count(); ++r) {
      const tcg::TilingPlan p = tcg::construct_rank_plan(c, lay, r, {ts[0], ts[1], ts[2]});
      os << "rank=" << r << " owned=" << lay.owned[static_cast<size_t>(r)].to_string() << "\n";
      os << plan_text(p, c.dim) << halo_text(tcg::compute_halo_depths(p, c, lay, r), c.dim);
    }
    put_text(os.str(), buf, n, needed);
  });
}

int tcg_gpu_plan_pending(tcg_runtime* rt, int mode, const int64_t ts[3], char* buf, int64_t n, int64_t* needed) {
  return guard([&] {
    tcg::LoopChain c = rt->rt->take_pending();
    const int s = c.dim - 1;
    tcg::GpuTileChoice choice;
    if (mode == TCG_WINDOWED)
      for (int d = 0; d < c.dim; ++d) {
        if (d == s)
          choice.stream_tile = std::max<int64_t>(1, ts[d]);
        else
          choice.block[d] = std::max<int64_t>(1, ts[d]);
      }
    choice.stream_segments = rt->rt->config().stream_segments;
    int nred = 0;
    for (const auto& l : c.loops) nred += l.reduction ? 1 : 0;
    const int nl = static_cast<int>(c.size());
    const tcg::WindowBudget budget = [&](int k) {
      const int64_t per_block = std::min<int64_t>(kB200SmemOptin, 233472 / k - 1024);
      const int64_t fixed = 6144 + nl * (static_cast<int64_t>(sizeof(tcg::DevLoop)) + 12 * 16 + 24) +
                            static_cast<int64_t>(nred) * (512 / k) * 8;
      return (per_block - fixed) / 8;
    };
    if (const char* e = std::getenv("TCG_CTAS_PER_SM")) choice.ctas_per_sm = std::atoi(e);
    const tcg::GpuTiledPlan gp = tcg::build_gpu_tiled_plan(c, rt->rt->field_geoms(), choice, budget, kB200Sms);
    std::ostringstream os;
    os << "grid=" << gp.grid[0] << "," << gp.grid[1] << "," << gp.grid[2] << " block=" << gp.block[0] << ","
       << gp.block[1] << " stream_tile=" << gp.stream_tile << " ctas=" << gp.ctas.size()
       << " smem_doubles=" << gp.smem_doubles << " computed_points=" << gp.computed_points
       << " recorded_points=" << gp.recorded_points << " max_skew=";
    for (int d = 0; d < c.dim; ++d) os << (d ? "," : "") << gp.max_skew[d];
    os << "\n";
    for (int k = 0; k < gp.ndat; ++k)
      os << "dat slot=" << k << " ds=" << gp.dat_ids[static_cast<size_t>(k)] << " load=" << gp.dats[static_cast<size_t>(k)].load
         << " written=" << gp.dats[static_cast<size_t>(k)].written
         << " pingpong=" << gp.dats[static_cast<size_t>(k)].pingpong << "\n";
    for (size_t i = 0; i < gp.ctas.size(); ++i) {
      const tcg::DevCta& ct = gp.ctas[i];
      os << "cta=" << i << " ntiles=" << ct.ntiles << " own=";
      for (int d = 0; d < c.dim; ++d) os << "[" << ct.own_lo[d] << "," << ct.own_hi[d] << ")";
      os << " wb=";
      for (int d = 0; d < c.dim; ++d) os << "[" << ct.wb_lo[d] << "," << ct.wb_hi[d] << ")";
      os << " cols=[" << ct.col_lo[0] << "," << ct.col_hi[0] << ")[" << ct.col_lo[1] << "," << ct.col_hi[1] << ") W=";
      for (int k = 0; k < gp.ndat; ++k) os << (k ? "," : "") << ct.W[k];
      os << "\n";
      for (int t = 0; t < ct.ntiles; ++t)
        for (int l = 0; l < gp.nloops; ++l) {
          const int32_t* b = &gp.boxes[static_cast<size_t>(ct.box_off) + (static_cast<size_t>(t) * gp.nloops + l) * 6];
          os << "box cta=" << i << " tile=" << t << " loop=" << l;
          for (int d = 0; d < c.dim; ++d) os << " [" << b[2 * d] << "," << b[2 * d + 1] << ")";
          os << "\n";
        }
    }
    put_text(os.str(), buf, n, needed);
  });
}

int tcg_set_rank_grid(tcg_runtime* rt, const int32_t grid[3]) {
  return guard([&] { rt->rt->set_rank_grid({grid[0], grid[1], grid[2]}); });
}

int tcg_upload_box(tcg_runtime* rt, int32_t ds, const double* host, const int64_t box[6]) {
  return guard([&] { rt->rt->upload_box(ds, host, range6(rt->rt->dim(), box)); });
}

int tcg_download_box(tcg_runtime* rt, int32_t ds, double* host, const int64_t box[6]) {
  return guard([&] { rt->rt->download_box(ds, host, range6(rt->rt->dim(), box)); });
}

int tcg_local_box(tcg_runtime* rt, int32_t ds, int64_t out[6]) {
  return guard([&] {
    const tcg::Range b = rt->rt->local_box(ds);
    for (int d = 0; d < 3; ++d) {
      out[2 * d] = d < b.dim() ? b.start(d) : 0;
      out[2 * d + 1] = d < b.dim() ? b.end(d) : 1;
    }
  });
}

int tcg_set_reduction_order(tcg_runtime* rt, int workers) {
  return guard([&] { rt->rt->set_reduction_order(workers); });
}
int tcg_record_begin(tcg_runtime* rt) {
  return guard([&] { rt->rt->record_begin(); });
}
int tcg_record_end(tcg_runtime* rt, int32_t* id) {
  return guard([&] { *id = rt->rt->record_end(); });
}
int tcg_replay(tcg_runtime* rt, int32_t id, const double* params, int64_t nparams, int32_t* handles, int64_t max_handles,
               int64_t* nhandles) {
  return guard([&] {
    const std::vector<tcg::ReductionHandle> hs = rt->rt->replay(id, params, params ? static_cast<size_t>(nparams) : 0);
    if (nhandles) *nhandles = static_cast<int64_t>(hs.size());
    for (size_t i = 0; i < hs.size() && static_cast<int64_t>(i) < max_handles; ++i) handles[i] = hs[i].id;
  });
}

int tcg_set_periodic_domain(tcg_runtime* rt, int on) {
  return guard([&] { rt->rt->set_periodic_domain(on != 0); });
}

int tcg_set_periodic_flush(tcg_runtime* rt, int flush_each) {
  return guard([&] { rt->rt->set_periodic_flush(flush_each != 0); });
}

int tcg_periodic_fill(tcg_runtime* rt, int n, const int32_t* ds, int64_t depth) {
  return guard([&] { rt->rt->periodic_fill(std::vector<tcg::DatasetId>(ds, ds + n), depth); });
}

int tcg_rank_owned(tcg_runtime* rt, int32_t rank, int64_t out[6]) {
  return guard([&] {
    const tcg::RankLayout& lay = rt->rt->rank_layout();
    if (rank < 0 || rank >= lay.rank_count()) throw tcg::InvalidArgument("rank_owned: rank out of range");
    const tcg::Range& o = lay.owned[static_cast<size_t>(rank)];
    for (int d = 0; d < 3; ++d) {
      out[2 * d] = d < o.dim() ? o.start(d) : 0;
      out[2 * d + 1] = d < o.dim() ? o.end(d) : 1;
    }
  });
}

int tcg_comm_unique_id(uint8_t out[128]) {
  return guard([&] { tcg::Comm::unique_id(out); });
}

int tcg_set_process_rank(tcg_runtime* rt, const int32_t grid[3], int32_t rank, const uint8_t id[128]) {
  return guard([&] { rt->rt->set_process_rank({grid[0], grid[1], grid[2]}, rank, id); });
}

int tcg_dist_schedule_pending(tcg_runtime* rt, char* buf, int64_t n, int64_t* needed) {
  return guard([&] {
    const tcg::DistSchedule s = rt->rt->schedule_pending();
    put_text(tcg::schedule_text(s, rt->rt->dim()), buf, n, needed);
  });
}

int tcg_signature_pending(tcg_runtime* rt, uint64_t* out) {
  return guard([&] {
    tcg::LoopChain c = rt->rt->take_pending();
    *out = c.signature();
  });
}

int tcg_auto_tile_size(int dim, int64_t cache_bytes, int32_t threads, int64_t bpp, const int64_t extent[6],
                       int64_t out[3]) {
  return guard([&] {
    tcg::SizerInput in;
    in.dim = dim;
    in.cache_bytes = cache_bytes;
    in.threads = threads;
    in.bytes_per_point = bpp;
    in.domain_extent = tcg::Range::box(dim, extent);
    const auto ts = tcg::auto_tile_size(in);
    for (int d = 0; d < 3; ++d) out[d] = ts[d];
  });
}

int tcg_device_info(char* name, size_t n, int32_t* num_sms, int64_t* smem_optin, int64_t* l2_bytes) {
  return guard([&] {
    tcg::DeviceExec ex;
    const tcg::DeviceInfo& i = ex.info();
    if (name && n > 0) {
      const size_t k = std::min(n - 1, i.name.size());
      std::memcpy(name, i.name.data(), k);
      name[k] = 0;
    }
    if (num_sms) *num_sms = i.num_sms;
    if (smem_optin) *smem_optin = i.smem_optin;
    if (l2_bytes) *l2_bytes = i.l2_bytes;
  });
}

int tcg_launches(tcg_runtime* rt, int64_t* out) {
  return guard([&] { *out = rt->rt->device_ready() ? rt->rt->device().launches() : 0; });
}

int tcg_stream(tcg_runtime* rt, void** out) {
  return guard([&] { *out = rt->rt->device().stream(); });
}

int tcg_body_known(int32_t body) { return tcb::body_known(body) ? 1 : 0; }

int tcg_select_device(int device) {
  return guard([&] { tcg::select_device(device); });
}

int tcg_set_timing(tcg_runtime* rt, int on) {
  return guard([&] { rt->rt->device().set_timing(on != 0); });
}

int tcg_kernel_timing(tcg_runtime* rt, double* tiled_ms, int64_t* tiled_n, double* untiled_ms, int64_t* untiled_n) {
  return guard([&] { rt->rt->device().kernel_ms(tiled_ms, tiled_n, untiled_ms, untiled_n); });
}

}  // extern "C"
