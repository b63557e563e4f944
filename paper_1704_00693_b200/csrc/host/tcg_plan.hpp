// Run-time dependency analysis and tile planning (host C++).
//
// Semantics follow the reference planner exactly so plans are comparable
// line for line with its golden dumps:
//   compute_union_bounds / construct_plan      planner.cpp:24-208
//   TilingPlan + dump + verify_plan_extents   planner.hpp:45-93, planner.cpp:234-269
//   PlanCache (signature, ts0, ts1, ts2)      planner.cpp:271-294
//   decompose / RankLayout                    dist.cpp:119-177
//   construct_rank_plan                       dist.cpp:191-390
//   exchange_flags / compute_halo_depths      dist.cpp:79-115, :407-448
//   auto_tile_size                            tile_sizer.cpp:27-109
// The shared-memory and per-rank analyses are one backward sweep here
// (`sweep_chain`): the shared-memory plan is the rank plan of a lone rank that
// owns the union bounds. On the GPU the same per-rank plan is built for every
// CTA of the windowed executor ("rank = CTA").
#pragma once
#include <functional>
#include <map>
#include <memory>
#include <tuple>

#include "tcg_types.hpp"

namespace tcg {

struct PlanConfig {
  int dim = 1;
  Range union_bounds;
  std::array<int64_t, kMaxDims> tile_sizes{1, 1, 1};
  std::array<int64_t, kMaxDims> num_tiles{1, 1, 1};
  int64_t total_tiles() const {
    int64_t n = 1;
    for (int d = 0; d < dim; ++d) n *= num_tiles[d];
    return n;
  }
};

struct DepExtent {
  int64_t start = std::numeric_limits<int64_t>::max();
  int64_t end = std::numeric_limits<int64_t>::min();
  bool set() const { return end != std::numeric_limits<int64_t>::min(); }
};

struct DatasetDeps {
  std::array<std::vector<DepExtent>, kMaxDims> read, write;  // [dim][slab]
};

class TilingPlan {
 public:
  PlanConfig config;
  uint64_t signature = 0;
  int32_t num_loops = 0;
  std::vector<Range> ranges;  // [tile * L + loop]
  std::map<DatasetId, DatasetDeps> deps;
  std::map<DatasetId, Range> required;
  std::array<int64_t, kMaxDims> max_skew{0, 0, 0};
  double build_seconds = 0;

  int64_t num_tiles() const { return config.total_tiles(); }
  const Range& range(int64_t tile, int32_t loop) const {
    return ranges[static_cast<size_t>(tile) * static_cast<size_t>(num_loops) + static_cast<size_t>(loop)];
  }
  std::array<int64_t, kMaxDims> tile_coords(int64_t tile) const;
  // "tile=<t> loop=<l> d=<d> [s,e)\n" per (tile, loop, dim), planner.cpp:234-250
  std::string dump() const;
};

PlanConfig compute_union_bounds(const LoopChain& chain, const std::array<int64_t, kMaxDims>& ts);
TilingPlan construct_plan(const LoopChain& chain, const std::array<int64_t, kMaxDims>& ts);

struct FieldExtent {
  std::string name;
  Range alloc;
};
// Throws PlanError naming the dataset and per-face shortfall.
void verify_plan_extents(const TilingPlan& plan, const std::vector<FieldExtent>& fields);

class PlanCache {
 public:
  std::shared_ptr<const TilingPlan> get_or_build(const LoopChain& chain,
                                                 const std::array<int64_t, kMaxDims>& ts,
                                                 bool* hit = nullptr);
  std::shared_ptr<const TilingPlan> get_or_build(uint64_t sig, const std::array<int64_t, kMaxDims>& ts,
                                                 const std::function<TilingPlan()>& build,
                                                 bool* hit = nullptr);
  int64_t constructions() const { return constructions_; }
  int64_t hits() const { return hits_; }
  void clear() { entries_.clear(); }

 private:
  std::map<std::tuple<uint64_t, int64_t, int64_t, int64_t>, std::shared_ptr<const TilingPlan>> entries_;
  int64_t constructions_ = 0;
  int64_t hits_ = 0;
};

// ---- distribution -----------------------------------------------------------
struct RankLayout {
  int dim = 1;
  std::array<int, kMaxDims> grid{1, 1, 1};
  Range global;
  std::vector<Range> owned;
  int rank_count() const { return static_cast<int>(owned.size()); }
  std::array<int, kMaxDims> coords_of(int rank) const;
  int rank_of(const std::array<int, kMaxDims>& c) const;
  int neighbor(int rank, int d, int dir) const;  // -1 at domain edges
};

RankLayout decompose(const Range& global, const std::array<int, kMaxDims>& grid);

TilingPlan construct_rank_plan(const LoopChain& chain, const RankLayout& layout, int rank,
                               const std::array<int64_t, kMaxDims>& ts);

struct HaloSpec {
  struct Faces {
    int64_t lo = 0, hi = 0;
  };
  struct Entry {
    bool needed = false;
    std::array<Faces, kMaxDims> faces{};
  };
  std::map<DatasetId, Entry> entries;
  int64_t depth_lo(DatasetId ds, int d) const;
  int64_t depth_hi(DatasetId ds, int d) const;
  bool needed(DatasetId ds) const;
};

using WriteHistory = std::map<DatasetId, std::vector<Range>>;

// True per dataset when some read touches points dirtied (prior history or any
// write of this chain) that no chain-earlier write recomputes first.
std::map<DatasetId, bool> exchange_flags(const LoopChain& chain, const WriteHistory* prior);

HaloSpec compute_halo_depths(const TilingPlan& rank_plan, const LoopChain& chain, const RankLayout& layout,
                             int rank, const WriteHistory* prior = nullptr);

// Box algebra helper: is `box` inside the union of `covers`?
bool covered_by(const Range& box, const std::vector<Range>& covers);

// ---- reference cache-footprint sizer (tile_sizer.cpp:27-109) -----------------
struct SizerInput {
  int dim = 2;
  int64_t cache_bytes = 0;
  int threads = 1;
  int64_t bytes_per_point = 0;
  Range domain_extent;
};
std::array<int64_t, kMaxDims> auto_tile_size(const SizerInput& in);

}  // namespace tcg
