// Deep-halo distribution schedule; see tcg_dist.hpp for the reference map.
#include "tcg_dist.hpp"

#include <sstream>

namespace tcg {

Range rank_alloc(const RankLayout& layout, int rank, int64_t pad) {
  const Range& own = layout.owned.at(static_cast<size_t>(rank));
  Range a(layout.dim);
  for (int d = 0; d < layout.dim; ++d) a.set(d, own.start(d) - pad, own.end(d) + pad);
  return a;
}

LoopChain with_ranges(const LoopChain& chain, const std::vector<Range>& ranges) {
  LoopChain c;
  c.dim = chain.dim;
  c.stencils = chain.stencils;
  c.loops = chain.loops;
  for (size_t l = 0; l < c.loops.size(); ++l) c.loops[l].range = ranges.at(l);
  return c;
}

DistSchedule build_dist_schedule(const LoopChain& chain, const RankLayout& layout,
                                 const std::vector<int64_t>& pads, const WriteHistory* prior) {
  DistSchedule s;
  const int R = layout.rank_count();
  const int dim = chain.dim;
  const int32_t L = static_cast<int32_t>(chain.size());
  // One slab per rank and dimension: the rank-local overlapped range of each
  // loop is then the plan's single tile (the union over any finer tiling of
  // the same rank plan is the same box).
  std::array<int64_t, kMaxDims> whole{1, 1, 1};
  for (int d = 0; d < dim; ++d) whole[d] = int64_t{1} << 40;
  s.ranks.resize(static_cast<size_t>(R));
  for (int r = 0; r < R; ++r) {
    RankWork& w = s.ranks[static_cast<size_t>(r)];
    w.owned = layout.owned[static_cast<size_t>(r)];
    const TilingPlan plan = construct_rank_plan(chain, layout, r, whole);
    w.loop_ranges.reserve(static_cast<size_t>(L));
    for (int32_t l = 0; l < L; ++l) {
      w.loop_ranges.push_back(plan.range(0, l));
      w.computed_points += plan.range(0, l).volume();
    }
    w.spec = compute_halo_depths(plan, chain, layout, r, prior);
  }
  build_messages(s, layout, pads);
  return s;
}

void build_messages(DistSchedule& s, const RankLayout& layout, const std::vector<int64_t>& pads) {
  const int R = layout.rank_count();
  s.msgs.clear();
  s.message_bytes = 0;
  // exchange_halos (dist.cpp:463-511): dimension-ordered; strips of dims
  // already exchanged are widened by the receiver's depth there, so corners
  // arrive through the neighbour.
  for (int d = 0; d < layout.dim; ++d) {
    s.phase[static_cast<size_t>(d)] = s.msgs.size();
    for (int r = 0; r < R; ++r) {
      const Range& own = layout.owned[static_cast<size_t>(r)];
      for (int dir : {-1, +1}) {
        const int src = layout.neighbor(r, d, dir);
        if (src < 0) continue;
        for (const auto& [ds, e] : s.ranks[static_cast<size_t>(r)].spec.entries) {
          if (!e.needed) continue;
          const int64_t depth = dir < 0 ? e.faces[static_cast<size_t>(d)].lo : e.faces[static_cast<size_t>(d)].hi;
          if (depth <= 0) continue;
          Range strip(layout.dim);
          for (int dd = 0; dd < layout.dim; ++dd) {
            if (dd == d) {
              if (dir < 0)
                strip.set(dd, own.start(dd) - depth, own.start(dd));
              else
                strip.set(dd, own.end(dd), own.end(dd) + depth);
            } else if (dd < d) {
              int64_t lo = own.start(dd), hi = own.end(dd);
              if (layout.neighbor(r, dd, -1) >= 0) lo -= e.faces[static_cast<size_t>(dd)].lo;
              if (layout.neighbor(r, dd, +1) >= 0) hi += e.faces[static_cast<size_t>(dd)].hi;
              strip.set(dd, lo, hi);
            } else {
              strip.set(dd, own.start(dd), own.end(dd));
            }
          }
          const int64_t pad = pads.at(static_cast<size_t>(ds));
          const Range box =
              strip.intersect(rank_alloc(layout, r, pad)).intersect(rank_alloc(layout, src, pad));
          if (box.empty()) continue;
          const Range& sown = layout.owned[static_cast<size_t>(src)];
          if (box.start(d) < sown.start(d) || box.end(d) > sown.end(d))
            throw PlanError("distributed chain: halo depth " + std::to_string(depth) + " of dataset " +
                            std::to_string(ds) + " in dim " + std::to_string(d) + " exceeds the owned width " +
                            std::to_string(sown.extent(d)) + " of neighbour rank " + std::to_string(src) +
                            "; use fewer ranks or shorter chains");
          HaloMsg m;
          m.src = src;
          m.dst = r;
          m.ds = ds;
          m.dim = d;
          m.dir = dir;
          m.box = box;
          m.points = box.volume();
          s.message_bytes += m.points * 8;
          s.msgs.push_back(m);
        }
      }
    }
  }
  for (int d = layout.dim; d <= kMaxDims; ++d) s.phase[static_cast<size_t>(d)] = s.msgs.size();
}

std::vector<DistSchedule> build_untiled_schedules(const LoopChain& chain, const RankLayout& layout,
                                                  const std::vector<int64_t>& pads) {
  // DistContext::run_untiled (dist.cpp:691-788): per loop, exchange exactly
  // the faces this loop reads that are stale (every face of a dataset goes
  // stale when any loop writes it; nothing is fresh at chain start), then
  // every rank runs the loop over its owned part.
  const int R = layout.rank_count();
  std::vector<DistSchedule> out;
  out.reserve(chain.size());
  std::map<DatasetId, std::array<HaloSpec::Faces, kMaxDims>> valid;
  for (const LoopRecord& loop : chain.loops) {
    HaloSpec spec;
    for (const ArgSpec& a : loop.args) {
      if (!mode_reads(a.mode)) continue;
      const Stencil& st = chain.stencil(a.stencil);
      auto& have = valid[a.dataset];
      HaloSpec::Entry e;
      bool stale = false;
      for (int d = 0; d < chain.dim; ++d) {
        e.faces[static_cast<size_t>(d)].lo = std::max<int64_t>(0, -st.min_offset(d));
        e.faces[static_cast<size_t>(d)].hi = std::max<int64_t>(0, st.max_offset(d));
        stale = stale || e.faces[static_cast<size_t>(d)].lo > have[static_cast<size_t>(d)].lo ||
                e.faces[static_cast<size_t>(d)].hi > have[static_cast<size_t>(d)].hi;
      }
      if (!stale) continue;
      e.needed = true;
      auto [it, inserted] = spec.entries.emplace(a.dataset, e);
      if (!inserted)
        for (int d = 0; d < chain.dim; ++d) {
          auto& f = it->second.faces[static_cast<size_t>(d)];
          f.lo = std::max(f.lo, e.faces[static_cast<size_t>(d)].lo);
          f.hi = std::max(f.hi, e.faces[static_cast<size_t>(d)].hi);
        }
    }
    for (const auto& [ds, e] : spec.entries) {
      auto& have = valid[ds];
      for (int d = 0; d < chain.dim; ++d) {
        have[static_cast<size_t>(d)].lo = std::max(have[static_cast<size_t>(d)].lo, e.faces[static_cast<size_t>(d)].lo);
        have[static_cast<size_t>(d)].hi = std::max(have[static_cast<size_t>(d)].hi, e.faces[static_cast<size_t>(d)].hi);
      }
    }
    DistSchedule s;
    s.ranks.resize(static_cast<size_t>(R));
    for (int r = 0; r < R; ++r) {
      RankWork& w = s.ranks[static_cast<size_t>(r)];
      w.owned = layout.owned[static_cast<size_t>(r)];
      w.loop_ranges.push_back(loop.range.intersect(w.owned));
      w.computed_points = w.loop_ranges.back().volume();
      w.spec = spec;
    }
    build_messages(s, layout, pads);
    out.push_back(std::move(s));
    for (const ArgSpec& a : loop.args)
      if (mode_writes(a.mode)) valid[a.dataset] = {};
  }
  return out;
}

bool note_writes(WriteHistory& hist, const LoopChain& chain) {
  bool changed = false;
  for (const LoopRecord& lp : chain.loops)
    for (const ArgSpec& a : lp.args) {
      if (!mode_writes(a.mode)) continue;
      std::vector<Range>& boxes = hist[a.dataset];
      bool held = false;
      for (const Range& b : boxes) held = held || b.contains(lp.range);
      if (!held) {
        boxes.push_back(lp.range);
        changed = true;
      }
    }
  return changed;
}

std::string schedule_text(const DistSchedule& s, int dim) {
  std::ostringstream os;
  for (size_t r = 0; r < s.ranks.size(); ++r) {
    const RankWork& w = s.ranks[r];
    os << "rank=" << r << " owned=" << w.owned.to_string() << " computed=" << w.computed_points << "\n";
    for (size_t l = 0; l < w.loop_ranges.size(); ++l) {
      os << "loop rank=" << r << " l=" << l;
      for (int d = 0; d < dim; ++d) os << " " << w.loop_ranges[l].start(d) << " " << w.loop_ranges[l].end(d);
      os << "\n";
    }
  }
  for (const auto& [ds, depth] : s.wraps) os << "wrap ds=" << ds << " depth=" << depth << "\n";
  for (const HaloMsg& m : s.msgs) {
    os << "msg src=" << m.src << " dst=" << m.dst << " ds=" << m.ds << " dim=" << m.dim << " dir=" << m.dir
       << " box";
    for (int d = 0; d < dim; ++d) os << " " << m.box.start(d) << " " << m.box.end(d);
    os << "\n";
  }
  return os.str();
}

}  // namespace tcg
