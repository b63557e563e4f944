#include "tcg_gpuplan.hpp"

#include <chrono>

#include "../kernels/tc_bodies.h"

namespace tcg {

namespace {

constexpr int64_t kHuge = int64_t{1} << 40;

int64_t floor_even(int64_t v) { return v - (((v % 2) + 2) % 2); }
int64_t ceil_even(int64_t v) { return floor_even(v + 1); }

struct DatInfo {
  DatasetId id;
  bool load = false, written = false, pingpong = false;
  int64_t reach = 0;  // max |stream-dim offset| of reads (mirror rows per side)
  std::vector<Range> wboxes;
};

// Chain-level dataset classification.
//   load:    some read may observe a value this chain has not produced yet (the
//            read box is not covered by chain-earlier write ranges), so the
//            window must be seeded from global memory. Mirrors the coverage
//            logic of exchange_flags (dist.cpp:79-115) without prior history:
//            global memory is always current on the device.
//   pingpong: loaded AND written -- other CTAs may still read the chain-start
//            values of points this CTA overwrites, so owned results go to the
//            dataset's second buffer (the reference hides the same hazard
//            behind rank-private storage, dist.cpp:520-530).
std::vector<DatInfo> classify(const LoopChain& chain, std::vector<int>& slot_of) {
  std::vector<DatInfo> out;
  auto slot = [&](DatasetId ds) {
    if (ds >= static_cast<DatasetId>(slot_of.size())) slot_of.resize(static_cast<size_t>(ds) + 1, -1);
    int& s = slot_of[static_cast<size_t>(ds)];
    if (s < 0) {
      s = static_cast<int>(out.size());
      DatInfo di;
      di.id = ds;
      out.push_back(di);
    }
    return s;
  };
  std::map<DatasetId, std::vector<Range>> covered;
  for (const LoopRecord& lp : chain.loops) {
    for (const ArgSpec& a : lp.args) {
      DatInfo& di = out[static_cast<size_t>(slot(a.dataset))];
      if (mode_reads(a.mode)) {
        const Stencil& st = chain.stencil(a.stencil);
        const int s = chain.dim - 1;
        di.reach = std::max({di.reach, static_cast<int64_t>(std::llabs(st.min_offset(s))),
                             static_cast<int64_t>(std::llabs(st.max_offset(s)))});
      }
      if (!mode_reads(a.mode) || di.load) continue;
      const Stencil& st = chain.stencil(a.stencil);
      Range rb = lp.range;
      if (rb.empty()) continue;
      for (int d = 0; d < chain.dim; ++d) rb.set(d, rb.start(d) + st.min_offset(d), rb.end(d) + st.max_offset(d));
      if (!covered_by(rb, covered[a.dataset])) di.load = true;
    }
    for (const ArgSpec& a : lp.args)
      if (mode_writes(a.mode)) {
        DatInfo& di = out[static_cast<size_t>(slot(a.dataset))];
        di.written = true;
        if (!lp.range.empty()) {
          covered[a.dataset].push_back(lp.range);
          di.wboxes.push_back(lp.range);
        }
      }
  }
  for (DatInfo& di : out) di.pingpong = di.load && di.written;
  return out;
}

struct Layout {
  RankLayout ranks;
  std::array<int64_t, kMaxDims> block{0, 0, 0};
  int64_t stream_tile = 1;
  bool prefetch = false;
};

int64_t floor_div(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// CTA decomposition of the union bounds. Column dims are cut at multiples of
// an even block width in ABSOLUTE coordinates, so interior ownership
// boundaries are 16-byte aligned in every dataset (bulk-copy evictions); the
// stream dim is split into near-equal segments like the reference's
// decompose (dist.cpp:142-177). Ranks are lexicographic, dim 0 slowest.
Layout make_layout(const Range& U, int dim, const std::array<int64_t, kMaxDims>& block, int64_t stile, int nseg) {
  Layout L;
  const int s = dim - 1;
  Range Ug = U;  // an empty union (all loops empty) still needs one CTA
  for (int d = 0; d < dim; ++d)
    if (Ug.extent(d) <= 0) Ug.set(d, U.start(d), U.start(d) + 1);
  std::array<std::vector<int64_t>, kMaxDims> cuts;
  for (int d = 0; d < dim; ++d) {
    const int64_t lo = Ug.start(d), hi = Ug.end(d), ext = hi - lo;
    std::vector<int64_t>& c = cuts[d];
    c.push_back(lo);
    if (d == s) {
      const int64_t g = std::max<int64_t>(1, std::min<int64_t>(nseg, ext));
      const int64_t q = ext / g, rem = ext % g;
      int64_t p = lo;
      for (int64_t i = 0; i < g; ++i) {
        p += q + (i < rem ? 1 : 0);
        c.push_back(p);
      }
    } else {
      int64_t b = std::max<int64_t>(2, block[d]);
      b += b & 1;
      for (int64_t p = floor_div(lo, b) * b + b; p < hi; p += b) c.push_back(p);
      c.push_back(hi);
    }
  }
  RankLayout& R = L.ranks;
  R.dim = dim;
  R.global = Ug;
  for (int d = 0; d < kMaxDims; ++d) R.grid[d] = d < dim ? static_cast<int>(cuts[d].size()) - 1 : 1;
  const int total = R.grid[0] * R.grid[1] * R.grid[2];
  R.owned.assign(static_cast<size_t>(total), Range(dim));
  for (int r = 0; r < total; ++r) {
    const auto co = R.coords_of(r);
    Range own(dim);
    for (int d = 0; d < dim; ++d)
      own.set(d, cuts[d][static_cast<size_t>(co[d])], cuts[d][static_cast<size_t>(co[d]) + 1]);
    R.owned[static_cast<size_t>(r)] = own;
  }
  L.block = block;
  L.stream_tile = std::max<int64_t>(1, stile);
  return L;
}

struct CtaBuild {
  DevCta cta{};
  std::vector<int32_t> boxes, win;
  int64_t smem = 0;
  int64_t computed = 0;
  std::array<int64_t, kMaxDims> skew{0, 0, 0};
};

int32_t clamp32(int64_t v) {
  return static_cast<int32_t>(std::max<int64_t>(std::numeric_limits<int32_t>::min() / 2,
                                                std::min<int64_t>(std::numeric_limits<int32_t>::max() / 2, v)));
}

CtaBuild build_cta(const LoopChain& chain, const std::vector<DatInfo>& dats, const std::vector<int>& slot_of,
                   const std::vector<FieldGeom>& fields, const Layout& lay, int rank) {
  const int dim = chain.dim, s = dim - 1;
  const int L = static_cast<int>(chain.size());
  const int nd = static_cast<int>(dats.size());
  const Range& own = lay.ranks.owned[static_cast<size_t>(rank)];
  std::array<int64_t, kMaxDims> ts{1, 1, 1};
  for (int d = 0; d < dim; ++d) ts[d] = d == s ? lay.stream_tile : kHuge;
  const TilingPlan plan = construct_rank_plan(chain, lay.ranks, rank, ts);
  const int64_t T = plan.config.num_tiles[s];
  // Every access of this CTA's plan must stay inside the allocation
  // (verify_plan_extents, planner.cpp:252-269, applied per CTA).
  for (const auto& [ds, req] : plan.required) {
    const Range& alloc = fields.at(static_cast<size_t>(ds)).alloc;
    if (!alloc.contains(req))
      throw PlanError("tiled plan (CTA " + std::to_string(rank) + ") requires dataset " + std::to_string(ds) +
                      " over " + req.to_string() + " but allocation is " + alloc.to_string() +
                      "; declare wider stencils first or raise the skew allowance");
  }

  CtaBuild cb;
  DevCta& c = cb.cta;
  c.ntiles = static_cast<int32_t>(T);
  cb.skew = plan.max_skew;

  // Allocation hull of the chain's datasets (write-back ownership at edges).
  Range ahull = fields[static_cast<size_t>(dats[0].id)].alloc;
  for (const DatInfo& di : dats) ahull = ahull.hull(fields[static_cast<size_t>(di.id)].alloc);
  const auto coords = lay.ranks.coords_of(rank);
  for (int d = 0; d < 3; ++d) {
    c.own_lo[d] = d < dim ? clamp32(own.start(d)) : 0;
    c.own_hi[d] = d < dim ? clamp32(own.end(d)) : 1;
    c.wb_lo[d] = c.own_lo[d];
    c.wb_hi[d] = c.own_hi[d];
    if (d < dim) {
      if (coords[d] == 0) c.wb_lo[d] = clamp32(std::min(own.start(d), ahull.start(d)));
      if (coords[d] == lay.ranks.grid[d] - 1) c.wb_hi[d] = clamp32(std::max(own.end(d), ahull.end(d)));
    }
  }

  // Boxes [t][l][d][2] and per-dataset access hulls.
  cb.boxes.resize(static_cast<size_t>(T) * L * 6, 0);
  std::vector<int64_t> acc_lo(static_cast<size_t>(T) * nd, kHuge), acc_hi(static_cast<size_t>(T) * nd, -kHuge);
  int64_t col_lo[2] = {kHuge, kHuge}, col_hi[2] = {-kHuge, -kHuge};
  bool any_pp = false;
  for (const DatInfo& di : dats) any_pp = any_pp || di.pingpong;
  for (int64_t t = 0; t < T; ++t)
    for (int l = 0; l < L; ++l) {
      const Range& r = plan.range(t, l);
      int32_t* b = &cb.boxes[(static_cast<size_t>(t) * L + l) * 6];
      for (int d = 0; d < 3; ++d) {
        b[2 * d] = d < dim ? clamp32(r.start(d)) : 0;
        b[2 * d + 1] = d < dim ? clamp32(r.end(d)) : 1;
      }
      if (r.empty()) continue;
      cb.computed += r.volume();
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
        const Range tb = r.dilated(lo, hi);
        const int k = slot_of[static_cast<size_t>(a.dataset)];
        const size_t ix = static_cast<size_t>(t) * nd + k;
        acc_lo[ix] = std::min(acc_lo[ix], tb.start(s));
        acc_hi[ix] = std::max(acc_hi[ix], tb.end(s));
        for (int d = 0; d < s; ++d) {
          col_lo[d] = std::min(col_lo[d], tb.start(d));
          col_hi[d] = std::max(col_hi[d], tb.end(d));
        }
      }
    }
  // Window columns: every access of this CTA's plan. Write-back points of a
  // ping-ponged dataset outside the window are never written by the chain
  // (they lie outside the union bounds), so the kernel copies them
  // global-to-global instead of staging them.
  (void)any_pp;
  for (int d = 0; d < s; ++d)
    if (col_lo[d] > col_hi[d]) col_lo[d] = col_hi[d] = own.start(d);
  if (s >= 1) {
    col_lo[0] = floor_even(col_lo[0]);
    col_hi[0] = ceil_even(col_hi[0]);
  }
  for (int d = 0; d < 2; ++d) {
    c.col_lo[d] = d < s ? clamp32(col_lo[d]) : 0;
    c.col_hi[d] = d < s ? clamp32(col_hi[d]) : 1;
  }
  const int64_t P = static_cast<int64_t>(c.col_hi[0] - c.col_lo[0]) * (c.col_hi[1] - c.col_lo[1]);

  // Sliding windows along the stream dim:
  //   rows loaded at tile t:  [hi(t-1), hi(t)), hi(-1) = lo(0)
  //   rows evicted after t:   [lo(t), lo(t+1)), lo(T) = hi(T-1)
  //   present during tile t:  [lo(t), hi(t)) which contains every access of t.
  cb.win.assign(static_cast<size_t>(T + 1) * nd * 2, 0);
  int64_t sm = 0;
  for (int k = 0; k < nd; ++k) {
    int64_t first = -1;
    for (int64_t t = 0; t < T && first < 0; ++t)
      if (acc_lo[static_cast<size_t>(t) * nd + k] <= acc_hi[static_cast<size_t>(t) * nd + k]) first = t;
    if (first < 0) {
      c.W[k] = 0;
      c.sbase[k] = 0;
      continue;
    }
    std::vector<int64_t> lo(static_cast<size_t>(T) + 1), hi(static_cast<size_t>(T));
    int64_t suffix = kHuge;
    for (int64_t t = T - 1; t >= 0; --t) {
      const size_t ix = static_cast<size_t>(t) * nd + k;
      if (acc_lo[ix] <= acc_hi[ix]) suffix = std::min(suffix, acc_lo[ix]);
      lo[static_cast<size_t>(t)] = suffix;
    }
    int64_t run = lo[0];
    for (int64_t t = 0; t < T; ++t) {
      const size_t ix = static_cast<size_t>(t) * nd + k;
      if (acc_lo[ix] <= acc_hi[ix]) run = std::max(run, acc_hi[ix]);
      hi[static_cast<size_t>(t)] = run;
    }
    for (int64_t t = 1; t < T; ++t)
      lo[static_cast<size_t>(t)] = std::min(lo[static_cast<size_t>(t)], hi[static_cast<size_t>(t) - 1]);
    for (int64_t t = 0; t < T; ++t) lo[static_cast<size_t>(t)] = std::min(lo[static_cast<size_t>(t)], hi[static_cast<size_t>(t)]);
    lo[static_cast<size_t>(T)] = hi[static_cast<size_t>(T) - 1];
    // Depth covers the rows of slab t, plus (prefetch) those loaded for slab
    // t+1 while t computes: rows [lo(t), hi(t+1)).
    int64_t W = 0;
    for (int64_t t = 0; t < T; ++t)
      W = std::max(W, hi[static_cast<size_t>(lay.prefetch ? std::min(t + 1, T - 1) : t)] - lo[static_cast<size_t>(t)]);
    W = std::max<int64_t>(W, 1);
    for (int64_t t = 0; t <= T; ++t) {
      int32_t* w = &cb.win[(static_cast<size_t>(t) * nd + k) * 2];
      w[0] = clamp32(lo[static_cast<size_t>(t)]);
      w[1] = clamp32(t < T ? hi[static_cast<size_t>(t)] : hi[static_cast<size_t>(T) - 1]);
    }
    c.W[k] = static_cast<int32_t>(W);
    c.sbase[k] = static_cast<int32_t>(sm);
    sm += W * P;
  }
  cb.smem = sm;
  return cb;
}

struct Candidate {
  std::array<int64_t, kMaxDims> block{0, 0, 0};
  int64_t stile = 1;
  int nseg = 1;
  int k = 1;  // CTAs per SM
};

}  // namespace

GpuTiledPlan build_gpu_tiled_plan(const LoopChain& chain, const std::vector<FieldGeom>& fields,
                                  const GpuTileChoice& choice, const WindowBudget& budget_fn, int num_sms) {
  const auto t0 = std::chrono::steady_clock::now();
  if (chain.empty()) throw PlanError("build_gpu_tiled_plan: empty chain");
  const int dim = chain.dim, s = dim - 1;
  GpuTiledPlan gp;
  gp.dim = dim;
  gp.nloops = static_cast<int>(chain.size());
  std::vector<int> slot_of;
  const std::vector<DatInfo> dats = classify(chain, slot_of);
  if (dats.size() > static_cast<size_t>(kMaxChainDats))
    throw PlanError("tiled executor: chain touches more than 32 datasets");
  gp.ndat = static_cast<int>(dats.size());
  for (const DatInfo& di : dats) gp.dat_ids.push_back(di.id);
  for (const LoopRecord& lp : chain.loops) {
    if (lp.reduction) ++gp.nred;
    if (lp.args.size() > static_cast<size_t>(kMaxArgs)) throw PlanError("tiled executor: too many args in a loop");
  }
  if (gp.nred > kMaxRed) throw PlanError("tiled executor: more than 8 reducing loops in one chain");

  Range U = chain.loops.front().range;
  for (const LoopRecord& lp : chain.loops) U = U.hull(lp.range);

  // Candidate list: explicit fields are fixed; auto fields are searched from
  // the least redundant (widest block) downwards.
  std::vector<Candidate> cands;
  {
    std::vector<int64_t> bx_list, by_list, st_list;
    // An explicit size is the first choice; when its windows do not fit in
    // shared memory, smaller defaults are tried (the explicit size acts as an
    // upper bound rather than an error, unlike a CPU cache that only slows).
    auto pick = [](int64_t v, std::initializer_list<int64_t> dflt) {
      if (v <= 0) return std::vector<int64_t>(dflt);
      std::vector<int64_t> out{v};
      for (int64_t d : dflt)
        if (d < v) out.push_back(d);
      return out;
    };
    if (dim == 1) {
      bx_list = {1};
      by_list = {1};
      st_list = pick(choice.stream_tile, {64, 16, 4, 1});
    } else if (dim == 2) {
      bx_list = pick(choice.block[0], {384, 256, 192, 128, 96, 64, 32, 16, 8});
      by_list = {1};
      st_list = pick(choice.stream_tile, {8, 4, 2, 1});
    } else {
      bx_list = pick(choice.block[0], {64, 48, 32, 16, 8});
      by_list = pick(choice.block[1], {32, 16, 8, 4});
      st_list = pick(choice.stream_tile, {4, 2, 1});
    }
    // 1 or 2 CTAs per SM (512 / 256 threads; the kernels built).
    const std::vector<int> k_list = choice.ctas_per_sm == 1 || choice.ctas_per_sm == 2
                                        ? std::vector<int>{choice.ctas_per_sm}
                                        : std::vector<int>{2, 1};
    for (int k : k_list)
    for (int64_t st : st_list)
      for (int64_t bx : bx_list)
        for (int64_t by : by_list) {
          Candidate c;
          if (dim >= 2) c.block[0] = bx;
          if (dim == 3) c.block[1] = by;
          c.stile = st;
          c.k = k;
          const int64_t slots = static_cast<int64_t>(num_sms) * k;
          // Stream segments: fill the SMs when the column grid alone cannot.
          int64_t cols = 1;
          for (int d = 0; d < s; ++d) cols *= (std::max<int64_t>(1, U.extent(d)) + c.block[d] - 1) / c.block[d];
          if (choice.stream_segments > 0) {
            c.nseg = choice.stream_segments;
          } else {
            // Wave-aware: one CTA per SM, so the critical path is
            // waves * (rows per segment + per-segment warm-up skew).
            const int64_t ext = std::max<int64_t>(1, U.extent(s));
            const int64_t max_seg = std::max<int64_t>(1, ext / 32);
            const int64_t warm = 2 * st + 8;
            int64_t best = 1;
            double best_cost = 1e300;
            for (int64_t g = 1; g <= max_seg; ++g) {
              const int64_t waves = (cols * g + slots - 1) / slots;
              const double cost = static_cast<double>(waves) * (static_cast<double>(ext) / g + warm);
              if (cost < best_cost * 0.999) {
                best_cost = cost;
                best = g;
              }
            }
            c.nseg = static_cast<int>(best);
          }
          cands.push_back(c);
        }
  }

  std::string last_err = "no candidate";
  for (const Candidate& cand : cands) {
    Layout lay = make_layout(U, dim, cand.block, cand.stile, cand.nseg);
    lay.prefetch = choice.prefetch != 0;
    const int64_t budget = budget_fn(cand.k);
    // Cheap probe with the middle CTA before building all of them.
    const int probe = lay.ranks.rank_count() / 2;
    if (build_cta(chain, dats, slot_of, fields, lay, probe).smem > budget) {
      last_err = "window storage exceeds the shared-memory budget";
      continue;
    }
    std::vector<CtaBuild> builds;
    builds.reserve(static_cast<size_t>(lay.ranks.rank_count()));
    bool ok = true;
    for (int r = 0; r < lay.ranks.rank_count() && ok; ++r) {
      builds.push_back(build_cta(chain, dats, slot_of, fields, lay, r));
      ok = builds.back().smem <= budget;
    }
    if (!ok) {
      last_err = "edge CTA window storage exceeds the shared-memory budget";
      continue;
    }
    // Verify every CTA plan stays inside the allocations (planner.cpp:252-269
    // semantics, checked on the hull the window loader will touch).
    gp.grid = lay.ranks.grid;
    gp.block = cand.block;
    gp.stream_tile = cand.stile;
    gp.prefetch = lay.prefetch;
    gp.ctas_per_sm = cand.k;
    gp.threads = 512 / cand.k;
    for (CtaBuild& cb : builds) {
      cb.cta.box_off = static_cast<int32_t>(gp.boxes.size());
      cb.cta.win_off = static_cast<int32_t>(gp.win.size());
      gp.boxes.insert(gp.boxes.end(), cb.boxes.begin(), cb.boxes.end());
      gp.win.insert(gp.win.end(), cb.win.begin(), cb.win.end());
      gp.ctas.push_back(cb.cta);
      gp.smem_doubles = std::max(gp.smem_doubles, cb.smem);
      gp.computed_points += cb.computed;
      for (int d = 0; d < dim; ++d) gp.max_skew[d] = std::max(gp.max_skew[d], cb.skew[d]);
    }
    for (const LoopRecord& lp : chain.loops) gp.recorded_points += lp.range.volume();
    for (const DatInfo& di : dats) {
      DevDat dd{};
      dd.load = di.load;
      dd.written = di.written;
      dd.pingpong = di.pingpong;
      dd.wbox_off = static_cast<int32_t>(gp.wboxes.size() / 6);
      dd.nwbox = di.pingpong ? 0 : static_cast<int32_t>(di.wboxes.size());
      dd.reach = static_cast<int32_t>(di.reach);
      if (!di.pingpong)
        for (const Range& r : di.wboxes)
          for (int d = 0; d < 3; ++d) {
            gp.wboxes.push_back(d < dim ? clamp32(r.start(d)) : 0);
            gp.wboxes.push_back(d < dim ? clamp32(r.end(d)) : 1);
          }
      gp.dats.push_back(dd);
    }
    gp.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return gp;
  }
  throw PlanError("tiled executor: no CTA tiling fits (" + last_err + ")");
}

}  // namespace tcg
