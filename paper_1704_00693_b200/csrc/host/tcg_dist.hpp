// Deep-halo distribution of a chain over a rank grid.
//
// The reference simulates ranks inside one process (DistContext,
// proj/core/include/tilechain/dist.hpp:96-156): per rank an overlapped plan
// (construct_rank_plan, dist.cpp:191-390), a halo spec (compute_halo_depths,
// dist.cpp:407-448), ONE dimension-ordered exchange per chain
// (exchange_halos, dist.cpp:463-511), then per-rank execution with the
// reduction masked to the owned box and a rank-order fold (run_tiled,
// dist.cpp:617-689).
//
// Here the same analysis produces a DistSchedule that the device runtime
// executes: either every rank on one GPU (the reference's simulation,
// Runtime::set_rank_grid) or one rank per process/GPU with the messages
// carried by NCCL over NVLink (Runtime::set_process_rank). Each rank's work is
// a *rank-local chain*: the chain with every loop's range replaced by the
// rank's overlapped range for it; any executor (untiled, windowed tiled) runs
// it unchanged.
#pragma once
#include <memory>
#include <vector>

#include "tcg_plan.hpp"

namespace tcg {

struct HaloMsg {
  int src = -1, dst = -1;
  DatasetId ds = -1;
  int dim = 0, dir = 0;
  Range box;            // global coordinates, inside both ranks' allocations
  int64_t points = 0;
};

struct RankWork {
  Range owned;
  std::vector<Range> loop_ranges;  // rank-local overlapped range per loop (may be empty)
  HaloSpec spec;
  int64_t computed_points = 0;
};

struct DistSchedule {
  std::vector<RankWork> ranks;          // every rank of the layout
  std::vector<HaloMsg> msgs;            // global exchange order (dist.cpp:463-511)
  // Periodic chains: datasets wrapped before the exchange and their depth
  // (faster dimensions inside every rank, the split one between the end ranks).
  std::vector<std::pair<DatasetId, int64_t>> wraps;
  std::array<size_t, kMaxDims + 1> phase{0, 0, 0, 0};  // msgs[phase[d], phase[d+1]) exchange along dim d
  int64_t message_bytes = 0;
};

// Allocation of dataset ds on rank r: owned box +- the field's pad, exactly
// as DistContext allocates rank fields (dist.cpp:519-529).
Range rank_alloc(const RankLayout& layout, int rank, int64_t pad);

// Builds the schedule. pads[ds] is the pad of each declared field. Throws
// PlanError when a face's halo depth exceeds the neighbour's owned width (the
// neighbour would have to forward data it does not own; the reference
// silently reads stale values there).
DistSchedule build_dist_schedule(const LoopChain& chain, const RankLayout& layout,
                                 const std::vector<int64_t>& pads, const WriteHistory* prior);

// Halo messages of s.ranks[*].spec (exchange_halos order, dist.cpp:463-511).
void build_messages(DistSchedule& s, const RankLayout& layout, const std::vector<int64_t>& pads);

// On-demand untiled distribution (DistContext::run_untiled, dist.cpp:691-788):
// one schedule per loop -- the stale faces that loop reads, exchanged just
// before it; every rank then runs the loop over its owned part. The baseline
// that the deep-halo schedule's "fewer, larger messages" is measured against.
std::vector<DistSchedule> build_untiled_schedules(const LoopChain& chain, const RankLayout& layout,
                                                  const std::vector<int64_t>& pads);

// note_writes (dist.cpp:590-602): remember every written loop range that is
// not already held by a recorded box. Returns true when the history changed.
bool note_writes(WriteHistory& hist, const LoopChain& chain);

// The chain with loop ranges replaced (rank-local chain).
LoopChain with_ranges(const LoopChain& chain, const std::vector<Range>& ranges);

std::string schedule_text(const DistSchedule& s, int dim);

}  // namespace tcg
