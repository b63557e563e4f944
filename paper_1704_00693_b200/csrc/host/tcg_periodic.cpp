#include "tcg_periodic.hpp"

#include <algorithm>

namespace tcg {

namespace {
struct Need {
  int64_t v[kMaxDims][2] = {{0, 0}, {0, 0}, {0, 0}};
  bool any() const {
    for (int d = 0; d < kMaxDims; ++d)
      if (v[d][0] > 0 || v[d][1] > 0) return true;
    return false;
  }
  int64_t max() const {
    int64_t m = 0;
    for (int d = 0; d < kMaxDims; ++d) m = std::max({m, v[d][0], v[d][1]});
    return m;
  }
};
}  // namespace

PeriodicPlan apply_periodic(const LoopChain& chain, const std::vector<Range>& logical) {
  PeriodicPlan out;
  out.chain.dim = chain.dim;
  out.chain.stencils = chain.stencils;
  out.chain.loops = chain.loops;
  const int dim = chain.dim;
  const size_t L = chain.loops.size();
  const size_t nd = logical.size();
  // need[ds]: ghost depth (per dim / side) to which the version of ds live at
  // the walk's position must hold periodic images. tent[ds]: ghost reads of
  // unextended loops, periodic only if a mark covers them further back.
  std::vector<Need> need(nd), tent(nd);
  auto commit_marks = [&](size_t pos) {
    for (const PeriodicMark& m : chain.fills) {
      if (m.pos != pos) continue;
      for (DatasetId ds : m.ds) {
        Need& t = tent.at(static_cast<size_t>(ds));
        Need& g = need.at(static_cast<size_t>(ds));
        if (pos == L) {
          // Trailing mark: the ghosts must be valid after the chain.
          for (int d = 0; d < dim; ++d)
            for (int e = 0; e < 2; ++e) g.v[d][e] = std::max(g.v[d][e], m.depth);
          continue;
        }
        for (int d = 0; d < dim; ++d)
          for (int e = 0; e < 2; ++e) {
            if (t.v[d][e] > m.depth)
              throw PlanError("periodic chain: a loop reads " + std::to_string(t.v[d][e]) +
                              " ghost layers of a dataset filled to depth " + std::to_string(m.depth));
            g.v[d][e] = std::max(g.v[d][e], t.v[d][e]);
            t.v[d][e] = 0;
          }
      }
    }
  };
  commit_marks(L);
  for (size_t li = L; li-- > 0;) {
    if (li + 1 < L) commit_marks(li + 1);
    const LoopRecord& lp = chain.loops[li];
    if (lp.range.empty()) continue;
    // Extension: the deepest need among the datasets the loop writes, on the
    // sides where the loop reaches the dataset's logical edge.
    Need ext;
    for (const ArgSpec& a : lp.args) {
      if (!mode_writes(a.mode)) continue;
      const Range& lg = logical.at(static_cast<size_t>(a.dataset));
      const Need& g = need[static_cast<size_t>(a.dataset)];
      for (int d = 0; d < dim; ++d) {
        if (lp.range.start(d) == lg.start(d)) ext.v[d][0] = std::max(ext.v[d][0], g.v[d][0]);
        if (lp.range.end(d) == lg.end(d)) ext.v[d][1] = std::max(ext.v[d][1], g.v[d][1]);
      }
    }
    if (ext.any() && lp.reduction)
      throw PlanError("periodic chain: a reducing loop writes a dataset whose ghost layers are needed");
    // Versions before this loop.
    for (const ArgSpec& a : lp.args) {
      if (!mode_writes(a.mode)) continue;
      const Range& lg = logical.at(static_cast<size_t>(a.dataset));
      Need& g = need[static_cast<size_t>(a.dataset)];
      Need& t = tent[static_cast<size_t>(a.dataset)];
      for (int d = 0; d < dim; ++d) {
        const bool edge[2] = {lp.range.start(d) == lg.start(d), lp.range.end(d) == lg.end(d)};
        for (int e = 0; e < 2; ++e) {
          if (!edge[e]) continue;  // ghosts on this side pass through from the earlier version
          g.v[d][e] = mode_reads(a.mode) ? ext.v[d][e] : 0;
          t.v[d][e] = 0;  // unmarked ghost reads of the new version see whatever is there
        }
      }
    }
    Range r = lp.range;
    for (int d = 0; d < dim; ++d) r.set_raw(d, lp.range.start(d) - ext.v[d][0], lp.range.end(d) + ext.v[d][1]);
    out.chain.loops[li].range = r;
    out.extended_points += r.volume() - lp.range.volume();
    out.max_extension = std::max(out.max_extension, ext.max());
    // Reads.
    for (const ArgSpec& a : lp.args) {
      if (!mode_reads(a.mode)) continue;
      const Stencil& st = chain.stencil(a.stencil);
      const Range& lg = logical.at(static_cast<size_t>(a.dataset));
      Need& g = need[static_cast<size_t>(a.dataset)];
      Need& t = tent[static_cast<size_t>(a.dataset)];
      for (int d = 0; d < dim; ++d) {
        const int64_t reach[2] = {std::max<int64_t>(0, -st.min_offset(d)), std::max<int64_t>(0, st.max_offset(d))};
        const int64_t beyond[2] = {lg.start(d) - (r.start(d) - reach[0]), (r.end(d) + reach[1]) - lg.end(d)};
        for (int e = 0; e < 2; ++e) {
          if (beyond[e] <= 0) continue;
          if (ext.v[d][e] > 0 || (mode_writes(a.mode) && beyond[e] > 0))
            g.v[d][e] = std::max(g.v[d][e], beyond[e]);
          else
            t.v[d][e] = std::max(t.v[d][e], beyond[e]);
        }
      }
    }
  }
  commit_marks(0);
  for (size_t ds = 0; ds < nd; ++ds)
    if (need[ds].any()) out.pre_fills.emplace_back(static_cast<DatasetId>(ds), need[ds].max());
  return out;
}

}  // namespace tcg
