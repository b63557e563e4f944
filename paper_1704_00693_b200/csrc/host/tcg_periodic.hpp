// Periodic boundaries inside a chain: the deep-halo scheme of the distributed
// path (one exchange per chain, depth = the chain's accumulated stencil reach,
// redundant computation in the halo; dist.cpp:191-390, :617-689) applied to
// the wrap-around neighbour. The reference has no periodic support
// (dist.cpp:135-140: neighbor() returns -1 at the domain edge); BASELINE
// config c5 needs it with the RK step kept as one chain.
//
// A chain carrying PeriodicMarks is rewritten before execution:
//   * a backward walk over the loops finds, per dataset version, how deep into
//     the ghost layers it must hold periodic images for the marked reads that
//     follow (a mark makes the ghost reads of the loops after it periodic);
//   * the loop that produces such a version runs over its range extended by
//     that depth (the ghost points are recomputed from periodic images, which
//     is bit-identical to copying the opposite side);
//   * datasets the chain starts from are wrapped ONCE, before the chain, to
//     the accumulated depth (the "self-exchange" of a single rank).
// The rewritten chain has no marks and runs on any executor.
#pragma once
#include <vector>

#include "tcg_types.hpp"

namespace tcg {

struct PeriodicPlan {
  LoopChain chain;  // extended ranges, no marks
  // Datasets wrapped before the chain and the depth of each wrap.
  std::vector<std::pair<DatasetId, int64_t>> pre_fills;
  int64_t max_extension = 0;
  int64_t extended_points = 0;  // loop points added by the extensions
};

// logical[ds] = logical box of each declared dataset. Throws PlanError when a
// loop after a mark reads deeper than the mark's depth, or a reducing loop
// would have to be extended.
PeriodicPlan apply_periodic(const LoopChain& chain, const std::vector<Range>& logical);

}  // namespace tcg
