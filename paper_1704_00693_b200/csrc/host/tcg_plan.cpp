#include "tcg_plan.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <set>

namespace tcg {

namespace {

constexpr int64_t kNone = std::numeric_limits<int64_t>::min();

struct Slab {
  int64_t s = 0, e = 0;
};

// Per-rank planning frame. A shared-memory plan is the frame of one rank that
// owns the union bounds and has no neighbours (see header comment).
struct Frame {
  Range owned;
  bool rank_mode = false;
  std::array<bool, kMaxDims> has_left{false, false, false};
};

DatasetDeps& deps_for(std::map<DatasetId, DatasetDeps>& deps, DatasetId ds, const PlanConfig& cfg) {
  auto it = deps.find(ds);
  if (it != deps.end()) return it->second;
  DatasetDeps dd;
  for (int d = 0; d < cfg.dim; ++d) {
    dd.read[d].assign(static_cast<size_t>(cfg.num_tiles[d]), DepExtent{});
    dd.write[d].assign(static_cast<size_t>(cfg.num_tiles[d]), DepExtent{});
  }
  return deps.emplace(ds, std::move(dd)).first->second;
}

// The backward per-dimension sweep (planner.cpp:55-155 / dist.cpp:232-340).
// Loops are visited last to first; for each tile slab t of dimension d:
//   end  = loop end on the last non-empty slab of the rank owning the loop end;
//          otherwise the furthest read of this loop's outputs by the same slab of
//          later loops (read-after-write), clamped at the loop end;
//        = pushed further right so later writes of this slab do not clobber
//          what the next slab of this loop still reads (write-after-read/write,
//          not on the final slab);
//        = nominal slab boundary when no dependency applies;
//   start = previous slab's end (slab 0: loop start, or in rank mode the
//          leftmost read of its outputs by slab 0 of later loops), so an
//          overshooting slab empties its successor.
// Then the loop's arguments widen the running read/write extents.
void sweep_dim(const LoopChain& chain, const PlanConfig& cfg, const Frame& fr, int d,
               std::map<DatasetId, DatasetDeps>& deps, std::vector<Slab>& out, int64_t& skew) {
  const int32_t L = static_cast<int32_t>(chain.size());
  const int64_t T = cfg.num_tiles[d];
  const int64_t ts = cfg.tile_sizes[d];
  const int64_t u0 = cfg.union_bounds.start(d);
  const int64_t own_s = fr.owned.start(d), own_e = fr.owned.end(d);
  out.assign(static_cast<size_t>(L) * static_cast<size_t>(T), Slab{});
  std::vector<int64_t> ends(static_cast<size_t>(T));
  auto nominal = [&](int64_t t, int64_t cap) { return std::min(cap, u0 + (t + 1) * ts); };

  for (int32_t l = L - 1; l >= 0; --l) {
    const LoopRecord& lp = chain.loops[static_cast<size_t>(l)];
    const int64_t gs = lp.range.start(d), ge = lp.range.end(d);
    const int64_t rs = std::max(gs, own_s), re = std::min(ge, own_e);
    const bool owns_end = own_e >= ge;

    int64_t last = -1;
    for (int64_t t = T - 1; t >= 0 && last < 0; --t)
      if (u0 + t * ts < re) last = t;

    for (int64_t t = 0; t < T; ++t) {
      const size_t ti = static_cast<size_t>(t);
      int64_t end = kNone;
      if (t == last && owns_end) {
        end = ge;
      } else {
        for (const ArgSpec& a : lp.args) {
          if (!mode_writes(a.mode)) continue;
          const DepExtent& rd = deps_for(deps, a.dataset, cfg).read[d][ti];
          if (rd.set()) end = std::max(end, rd.end);
        }
        if (end != kNone) end = std::min(end, ge);
      }
      if (t != T - 1) {
        int64_t war = kNone;
        for (const ArgSpec& a : lp.args) {
          const DepExtent& wd = deps_for(deps, a.dataset, cfg).write[d][ti];
          if (wd.set()) war = std::max(war, wd.end - chain.stencil(a.stencil).min_offset(d));
        }
        if (war != kNone) end = std::max(end, std::min(war, ge));
      }
      if (end == kNone) end = nominal(t, re);
      if (fr.rank_mode && t == last) end = std::max(end, re);
      ends[ti] = end;
    }

    int64_t start = rs;
    if (fr.has_left[d]) {
      int64_t left = std::numeric_limits<int64_t>::max();
      for (const ArgSpec& a : lp.args) {
        if (!mode_writes(a.mode)) continue;
        const DepExtent& rd = deps_for(deps, a.dataset, cfg).read[d][0];
        if (rd.set()) left = std::min(left, rd.start);
      }
      if (left != std::numeric_limits<int64_t>::max()) start = std::max(gs, std::min(start, left));
    }
    for (int64_t t = 0; t < T; ++t) {
      const int64_t e = std::max(ends[static_cast<size_t>(t)], start);
      out[static_cast<size_t>(l) * static_cast<size_t>(T) + static_cast<size_t>(t)] = {start, e};
      skew = std::max(skew, e - nominal(t, re));
      start = e;
    }

    for (int64_t t = 0; t < T; ++t) {
      const Slab sl = out[static_cast<size_t>(l) * static_cast<size_t>(T) + static_cast<size_t>(t)];
      if (sl.e <= sl.s) continue;
      for (const ArgSpec& a : lp.args) {
        DatasetDeps& dd = deps_for(deps, a.dataset, cfg);
        const Stencil& st = chain.stencil(a.stencil);
        if (mode_reads(a.mode)) {
          DepExtent& x = dd.read[d][static_cast<size_t>(t)];
          x.end = std::max(x.end, sl.e + st.max_offset(d));
          x.start = std::min(x.start, sl.s + st.min_offset(d));
        }
        if (mode_writes(a.mode)) {
          DepExtent& x = dd.write[d][static_cast<size_t>(t)];
          x.end = std::max(x.end, sl.e);
          x.start = std::min(x.start, sl.s);
        }
      }
    }
  }
}

TilingPlan sweep_chain(const LoopChain& chain, const PlanConfig& cfg, const Frame& fr) {
  const auto t0 = std::chrono::steady_clock::now();
  const int dim = cfg.dim;
  const int32_t L = static_cast<int32_t>(chain.size());
  TilingPlan plan;
  plan.config = cfg;
  plan.signature = chain.signature();
  plan.num_loops = L;

  std::array<std::vector<Slab>, kMaxDims> slabs;
  for (int d = 0; d < dim; ++d) sweep_dim(chain, cfg, fr, d, plan.deps, slabs[d], plan.max_skew[d]);

  // Cartesian product of per-dimension slabs, tiles lexicographic with t0
  // slowest (planner.cpp:158-201), plus the required-extent hull.
  const int64_t total = cfg.total_tiles();
  plan.ranges.reserve(static_cast<size_t>(total) * static_cast<size_t>(L));
  for (int64_t tile = 0; tile < total; ++tile) {
    const auto tc = plan.tile_coords(tile);
    for (int32_t l = 0; l < L; ++l) {
      Range r(dim);
      for (int d = 0; d < dim; ++d) {
        const Slab sl = slabs[d][static_cast<size_t>(l) * static_cast<size_t>(cfg.num_tiles[d]) +
                                 static_cast<size_t>(tc[d])];
        r.set(d, sl.s, std::max(sl.s, sl.e));
      }
      if (!r.empty()) {
        for (const ArgSpec& a : chain.loops[static_cast<size_t>(l)].args) {
          const Stencil& st = chain.stencil(a.stencil);
          Point lo{0, 0, 0}, hi{0, 0, 0};
          for (int d = 0; d < dim; ++d) {
            if (a.mode == AccessMode::Read) {
              lo[d] = st.min_offset(d);
              hi[d] = st.max_offset(d);
            } else if (mode_reads(a.mode)) {
              lo[d] = std::min<int64_t>(st.min_offset(d), 0);
              hi[d] = std::max<int64_t>(st.max_offset(d), 0);
            }
          }
          const Range touched = r.dilated(lo, hi);
          auto it = plan.required.find(a.dataset);
          if (it == plan.required.end())
            plan.required.emplace(a.dataset, touched);
          else
            it->second = it->second.hull(touched);
        }
      }
      plan.ranges.push_back(r);
    }
  }
  plan.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return plan;
}

void fill_grid(PlanConfig& cfg, const std::array<int64_t, kMaxDims>& ts) {
  for (int d = 0; d < cfg.dim; ++d) {
    cfg.tile_sizes[d] = std::max<int64_t>(1, ts[d]);
    const int64_t ext = cfg.union_bounds.extent(d);
    cfg.num_tiles[d] = ext > 0 ? (ext - 1) / cfg.tile_sizes[d] + 1 : 1;
  }
}

}  // namespace

std::array<int64_t, kMaxDims> TilingPlan::tile_coords(int64_t tile) const {
  std::array<int64_t, kMaxDims> tc{0, 0, 0};
  for (int d = config.dim - 1; d >= 0; --d) {
    tc[d] = tile % config.num_tiles[d];
    tile /= config.num_tiles[d];
  }
  return tc;
}

std::string TilingPlan::dump() const {
  std::string s;
  char buf[128];
  for (int64_t t = 0; t < num_tiles(); ++t)
    for (int32_t l = 0; l < num_loops; ++l) {
      const Range& r = range(t, l);
      for (int d = 0; d < config.dim; ++d) {
        std::snprintf(buf, sizeof buf, "tile=%lld loop=%d d=%d [%lld,%lld)\n", static_cast<long long>(t), l, d,
                      static_cast<long long>(r.start(d)), static_cast<long long>(r.end(d)));
        s += buf;
      }
    }
  return s;
}

PlanConfig compute_union_bounds(const LoopChain& chain, const std::array<int64_t, kMaxDims>& ts) {
  if (chain.empty()) throw PlanError("compute_union_bounds: empty chain");
  PlanConfig cfg;
  cfg.dim = chain.dim;
  cfg.union_bounds = chain.loops.front().range;
  for (const LoopRecord& l : chain.loops) cfg.union_bounds = cfg.union_bounds.hull(l.range);
  fill_grid(cfg, ts);
  return cfg;
}

TilingPlan construct_plan(const LoopChain& chain, const std::array<int64_t, kMaxDims>& ts) {
  if (chain.empty()) throw PlanError("construct_plan: empty chain");
  const PlanConfig cfg = compute_union_bounds(chain, ts);
  Frame fr;
  fr.owned = cfg.union_bounds;
  return sweep_chain(chain, cfg, fr);
}

TilingPlan construct_rank_plan(const LoopChain& chain, const RankLayout& layout, int rank,
                               const std::array<int64_t, kMaxDims>& ts) {
  if (chain.empty()) throw PlanError("construct_rank_plan: empty chain");
  const Range& owned = layout.owned.at(static_cast<size_t>(rank));
  PlanConfig cfg;
  cfg.dim = chain.dim;
  bool have = false;
  for (const LoopRecord& l : chain.loops) {
    const Range c = l.range.intersect(owned);
    if (c.empty()) continue;
    cfg.union_bounds = have ? cfg.union_bounds.hull(c) : c;
    have = true;
  }
  if (!have) {
    cfg.union_bounds = Range(chain.dim);
    for (int d = 0; d < chain.dim; ++d) cfg.union_bounds.set(d, owned.start(d), owned.start(d));
  }
  fill_grid(cfg, ts);
  Frame fr;
  fr.owned = owned;
  fr.rank_mode = true;
  for (int d = 0; d < chain.dim; ++d) fr.has_left[d] = layout.neighbor(rank, d, -1) >= 0;
  return sweep_chain(chain, cfg, fr);
}

void verify_plan_extents(const TilingPlan& plan, const std::vector<FieldExtent>& fields) {
  for (const auto& [ds, req] : plan.required) {
    const FieldExtent& f = fields.at(static_cast<size_t>(ds));
    if (f.alloc.contains(req)) continue;
    std::string msg = "plan requires dataset " + f.name + " over " + req.to_string() + " but allocation is " +
                      f.alloc.to_string() + " (per-face shortfall:";
    for (int d = 0; d < f.alloc.dim(); ++d)
      msg += " d" + std::to_string(d) + "=-" + std::to_string(std::max<int64_t>(0, f.alloc.start(d) - req.start(d))) +
             "/+" + std::to_string(std::max<int64_t>(0, req.end(d) - f.alloc.end(d)));
    msg += "); declare wider stencils first or raise the skew allowance";
    throw PlanError(msg);
  }
}

std::shared_ptr<const TilingPlan> PlanCache::get_or_build(const LoopChain& chain,
                                                          const std::array<int64_t, kMaxDims>& ts, bool* hit) {
  return get_or_build(chain.signature(), ts, [&] { return construct_plan(chain, ts); }, hit);
}

std::shared_ptr<const TilingPlan> PlanCache::get_or_build(uint64_t sig, const std::array<int64_t, kMaxDims>& ts,
                                                          const std::function<TilingPlan()>& build, bool* hit) {
  const auto key = std::make_tuple(sig, ts[0], ts[1], ts[2]);
  auto it = entries_.find(key);
  if (it != entries_.end()) {
    ++hits_;
    if (hit) *hit = true;
    return it->second;
  }
  if (hit) *hit = false;
  ++constructions_;
  auto p = std::make_shared<const TilingPlan>(build());
  entries_.emplace(key, p);
  return p;
}

// ---- distribution -------------------------------------------------------------

std::array<int, kMaxDims> RankLayout::coords_of(int rank) const {
  std::array<int, kMaxDims> c{0, 0, 0};
  for (int d = dim - 1; d >= 0; --d) {
    c[d] = rank % grid[d];
    rank /= grid[d];
  }
  return c;
}

int RankLayout::rank_of(const std::array<int, kMaxDims>& c) const {
  int r = 0;
  for (int d = 0; d < dim; ++d) r = r * grid[d] + c[d];
  return r;
}

int RankLayout::neighbor(int rank, int d, int dir) const {
  auto c = coords_of(rank);
  c[d] += dir;
  if (c[d] < 0 || c[d] >= grid[d]) return -1;
  return rank_of(c);
}

RankLayout decompose(const Range& global, const std::array<int, kMaxDims>& grid) {
  RankLayout lay;
  lay.dim = global.dim();
  lay.grid = grid;
  lay.global = global;
  int total = 1;
  for (int d = 0; d < kMaxDims; ++d) {
    if (grid[d] < 1) throw InvalidArgument("decompose: rank counts must be >= 1");
    if (d >= lay.dim) {
      if (grid[d] != 1) throw InvalidArgument("decompose: grid uses dimension beyond domain");
      continue;
    }
    if (grid[d] > global.extent(d))
      throw InvalidArgument("decompose: more ranks than points in dim " + std::to_string(d));
    total *= grid[d];
  }
  lay.owned.assign(static_cast<size_t>(total), Range(lay.dim));
  for (int r = 0; r < total; ++r) {
    const auto c = lay.coords_of(r);
    Range own(lay.dim);
    for (int d = 0; d < lay.dim; ++d) {
      const int64_t ext = global.extent(d), q = ext / grid[d], rem = ext % grid[d];
      const int64_t s = global.start(d) + c[d] * q + std::min<int64_t>(c[d], rem);
      own.set(d, s, s + q + (c[d] < rem ? 1 : 0));
    }
    lay.owned[static_cast<size_t>(r)] = own;
  }
  return lay;
}

int64_t HaloSpec::depth_lo(DatasetId ds, int d) const {
  auto it = entries.find(ds);
  return it == entries.end() ? 0 : it->second.faces[d].lo;
}
int64_t HaloSpec::depth_hi(DatasetId ds, int d) const {
  auto it = entries.find(ds);
  return it == entries.end() ? 0 : it->second.faces[d].hi;
}
bool HaloSpec::needed(DatasetId ds) const {
  auto it = entries.find(ds);
  return it != entries.end() && it->second.needed;
}

bool covered_by(const Range& box, const std::vector<Range>& covers) {
  // Repeatedly carve each cover out of the still-uncovered fragments.
  std::vector<Range> left{box};
  const int dim = box.dim();
  for (const Range& c : covers) {
    std::vector<Range> next;
    for (Range f : left) {
      if (f.intersect(c).empty()) {
        next.push_back(f);
        continue;
      }
      for (int d = 0; d < dim; ++d) {
        if (f.start(d) < c.start(d)) {
          Range piece = f;
          piece.set(d, f.start(d), c.start(d));
          next.push_back(piece);
          f.set(d, c.start(d), f.end(d));
        }
        if (f.end(d) > c.end(d)) {
          Range piece = f;
          piece.set(d, c.end(d), f.end(d));
          next.push_back(piece);
          f.set(d, f.start(d), c.end(d));
        }
      }
    }
    left.swap(next);
    if (left.empty()) return true;
  }
  return left.empty();
}

std::map<DatasetId, bool> exchange_flags(const LoopChain& chain, const WriteHistory* prior) {
  WriteHistory dirty;
  if (prior) dirty = *prior;
  for (const LoopRecord& lp : chain.loops)
    for (const ArgSpec& a : lp.args)
      if (mode_writes(a.mode)) dirty[a.dataset].push_back(lp.range);
  std::map<DatasetId, bool> needed;
  WriteHistory covered;
  for (const LoopRecord& lp : chain.loops) {
    for (const ArgSpec& a : lp.args) {
      if (!mode_reads(a.mode)) continue;
      bool& flag = needed[a.dataset];
      if (flag) continue;
      const Stencil& st = chain.stencil(a.stencil);
      Range reads = lp.range;
      for (int d = 0; d < chain.dim; ++d)
        reads.set(d, reads.start(d) + st.min_offset(d), reads.end(d) + st.max_offset(d));
      auto it = dirty.find(a.dataset);
      if (it == dirty.end()) continue;
      for (const Range& w : it->second) {
        const Range hz = reads.intersect(w);
        if (!hz.empty() && !covered_by(hz, covered[a.dataset])) {
          flag = true;
          break;
        }
      }
    }
    for (const ArgSpec& a : lp.args)
      if (mode_writes(a.mode)) covered[a.dataset].push_back(lp.range);
  }
  return needed;
}

HaloSpec compute_halo_depths(const TilingPlan& plan, const LoopChain& chain, const RankLayout& layout, int rank,
                             const WriteHistory* prior) {
  HaloSpec spec;
  const Range& own = layout.owned.at(static_cast<size_t>(rank));
  const auto flags = exchange_flags(chain, prior);
  std::map<DatasetId, AccessMode> first;
  for (const LoopRecord& lp : chain.loops)
    for (const ArgSpec& a : lp.args) first.emplace(a.dataset, a.mode);
  for (const auto& [ds, m] : first) {
    HaloSpec::Entry e;
    auto f = flags.find(ds);
    e.needed = mode_reads(m) || (f != flags.end() && f->second);
    if (e.needed) {
      auto it = plan.deps.find(ds);
      if (it != plan.deps.end())
        for (int d = 0; d < chain.dim; ++d)
          for (const DepExtent& x : it->second.read[d]) {
            if (!x.set()) continue;
            e.faces[d].lo = std::max(e.faces[d].lo, own.start(d) - x.start);
            e.faces[d].hi = std::max(e.faces[d].hi, x.end - own.end(d));
          }
    }
    spec.entries.emplace(ds, e);
  }
  return spec;
}

// ---- reference sizer ------------------------------------------------------------

namespace {
int64_t int_sqrt(int64_t v) {
  if (v <= 0) return 0;
  int64_t r = static_cast<int64_t>(std::sqrt(static_cast<double>(v)));
  while ((r + 1) * (r + 1) <= v) ++r;
  while (r * r > v) --r;
  return r;
}
}  // namespace

std::array<int64_t, kMaxDims> auto_tile_size(const SizerInput& in) {
  if (in.dim < 1 || in.dim > kMaxDims) throw SizerError("auto_tile_size: dim must be in [1,3]");
  if (in.cache_bytes <= 0 || in.threads <= 0 || in.bytes_per_point <= 0)
    throw SizerError("auto_tile_size: cache_bytes, threads, bytes_per_point must be positive");
  if (in.domain_extent.empty()) throw SizerError("auto_tile_size: empty domain extent");
  const int64_t cap = in.cache_bytes / in.bytes_per_point;
  const int64_t T = in.threads;
  if (cap < T) throw SizerError("auto_tile_size: cache cannot hold one point per thread");
  std::array<int64_t, kMaxDims> ext{1, 1, 1}, ts{1, 1, 1};
  for (int d = 0; d < in.dim; ++d) ext[d] = in.domain_extent.extent(d);
  if (in.dim == 1) {
    ts[0] = std::min(ext[0], cap);
    return ts;
  }
  if (in.dim == 2) {
    int64_t y = int_sqrt(cap / 2) / T * T;
    if (y < T) y = T;
    if (ext[1] < y) {
      y = ext[1] / T * T;
      if (y < T) y = std::min<int64_t>(T, ext[1]);
    }
    ts[1] = y;
    ts[0] = std::min(ext[0], std::max(2 * y, cap / y));
    return ts;
  }
  const int64_t x = ext[0];
  const int64_t bound = std::min({int_sqrt(cap / x), ext[1], ext[2], std::max<int64_t>(1, x / 2)});
  int64_t y = 0;
  for (int64_t c = bound; c >= 1 && y == 0; --c)
    if ((c * c) % T == 0) y = c;
  if (y == 0) {
    y = T;
    for (int64_t c = 1; c < T; ++c)
      if ((c * c) % T == 0) {
        y = c;
        break;
      }
  }
  ts[0] = x;
  ts[1] = y;
  ts[2] = y;
  return ts;
}

// ---- chain -----------------------------------------------------------------------

uint64_t LoopChain::signature() const {
  // FNV-1a 64 over bytes of (dim, #loops, per loop: kernel id, range, #args,
  // arg (ds, stencil, mode), reduction tag) -- loop.cpp:20-41.
  uint64_t h = 14695981039346656037ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix(static_cast<uint64_t>(dim));
  mix(loops.size());
  for (const LoopRecord& l : loops) {
    mix(static_cast<uint64_t>(l.kernel.id));
    for (int d = 0; d < dim; ++d) {
      mix(static_cast<uint64_t>(l.range.start(d)));
      mix(static_cast<uint64_t>(l.range.end(d)));
    }
    mix(l.args.size());
    for (const ArgSpec& a : l.args) {
      mix(static_cast<uint64_t>(a.dataset));
      mix(static_cast<uint64_t>(a.stencil));
      mix(static_cast<uint64_t>(a.mode));
    }
    mix(l.reduction ? 0x9e3779b9u + static_cast<uint64_t>(l.reduction->op) : 0ull);
  }
  return h;
}

int64_t estimate_bytes_moved(const LoopRecord& loop, const Range& executed) {
  const int64_t pts = executed.volume();
  int64_t b = 0;
  for (const ArgSpec& a : loop.args)
    b += pts * 8 * ((a.mode == AccessMode::ReadWrite || a.mode == AccessMode::Increment) ? 2 : 1);
  return b;
}

}  // namespace tcg
