// Windowed tiled-executor plan builder: the reference's two planning
// algorithms composed with "rank = CTA".
//   * Across CTAs: overlapped tiling = construct_rank_plan (dist.cpp:191-390)
//     over a CTA grid that decomposes the chain's union bounds. Boundary
//     iterations are recomputed redundantly, so CTAs never talk to each other.
//   * Inside a CTA: the rank plan's skewed slabs along the slowest ("stream")
//     dimension are executed in order (planner.cpp:55-208 semantics,
//     executor.cpp:232-244 order), on CTA-private shared-memory windows that
//     slide along the stream dimension -- the B200 analogue of the reference's
//     rank-private FieldTable (dist.cpp:520-530).
#pragma once
#include <vector>

#include "tcg_device.hpp"
#include "tcg_plan.hpp"

namespace tcg {

struct FieldGeom {
  Range alloc;
};

struct GpuTileChoice {
  std::array<int64_t, kMaxDims> block{0, 0, 0};  // owned CTA extent per non-stream dim (0 = auto)
  int64_t stream_tile = 0;                        // skewed slab height along the stream dim (0 = auto)
  int stream_segments = 0;                        // CTA segments along the stream dim (0 = auto)
  int prefetch = 0;                               // 1: deepen windows to overlap slab loads with compute
  int ctas_per_sm = 0;                            // 1, 2 or 4 resident CTAs per SM (0 = auto)
};

// Window storage (doubles) available to one CTA when `ctas_per_sm` CTAs of
// 512 / ctas_per_sm threads share an SM.
using WindowBudget = std::function<int64_t(int ctas_per_sm)>;

struct GpuTiledPlan {
  int dim = 1;
  int nloops = 0;
  int ndat = 0;
  int nred = 0;
  std::vector<DatasetId> dat_ids;   // chain-local slot -> dataset id
  std::vector<DevCta> ctas;
  std::vector<int32_t> boxes, win, wboxes;
  std::vector<DevDat> dats;
  int64_t smem_doubles = 0;
  std::array<int, kMaxDims> grid{1, 1, 1};
  std::array<int64_t, kMaxDims> block{0, 0, 0};
  int64_t stream_tile = 1;
  bool prefetch = false;
  int ctas_per_sm = 1;
  int threads = 512;
  std::array<int64_t, kMaxDims> max_skew{0, 0, 0};
  // Accounting: points computed (incl. redundant) vs recorded.
  int64_t computed_points = 0;
  int64_t recorded_points = 0;
  double build_seconds = 0;
};

// budget(k): per-CTA window storage with k CTAs per SM. Throws PlanError
// ("no CTA tiling fits") when nothing fits; auto fields are searched.
GpuTiledPlan build_gpu_tiled_plan(const LoopChain& chain, const std::vector<FieldGeom>& fields,
                                  const GpuTileChoice& choice, const WindowBudget& budget, int num_sms);

}  // namespace tcg
