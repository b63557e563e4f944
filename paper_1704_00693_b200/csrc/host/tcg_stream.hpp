// Streaming fused-chain executor: planner and CUDA code generator.
//
// The reference executes a chain tile by tile over a skewed plan so that a
// tile's data stays in cache from loop to loop (execute_plan,
// proj/core/src/executor.cpp:209-250, over construct_plan,
// proj/core/src/planner.cpp:55-208; overlapped per-rank tiles,
// proj/core/src/dist.cpp:191-390). On B200 the same idea becomes a
// *streaming pipeline* per CTA:
//
//   * the CTA owns a box of the cross-section (x in 2D, x-y in 3D) widened by
//     the chain's accumulated in-plane stencil reach E (overlapped tiling:
//     halo points are recomputed redundantly, as the reference's ranks do,
//     dist.cpp:268-310), and walks the slowest dimension (y / z) row by row;
//   * every loop of the (sub-)chain is a pipeline stage that lags the
//     previous ones by its stream-direction read reach (the skew of
//     planner.cpp:103-135, per row instead of per tile);
//   * every dataset *version* (the state after a loop writes it) lives in a
//     per-thread register ring along the stream dimension; in-plane
//     neighbours cross threads through a double-buffered shared-memory
//     plane; inputs are read from HBM once, live outputs written once;
//   * bodies are compiled into the kernel: one kernel per chain signature is
//     generated here and compiled by NVRTC for sm_100a (tcg_jit.cpp), the way
//     OPS generates code per loop chain.
//
// Datasets a chain both reads and rewrites are written to their second
// buffer (ping-pong) so no CTA can observe another CTA's writes.
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "tcg_plan.hpp"

namespace tcg {

// Device geometry of one dataset's buffers (both ping-pong buffers share it):
// element (x, y, z) at base[(z - z0) * pz + (y - y0) * py + (x - x0)].
struct StreamGeom {
  Range alloc;
  int64_t x0 = 0, y0 = 0, z0 = 0, py = 0, pz = 0;
};

// Tuning knobs; 0 / -1 = chosen by the sizer.
struct StreamChoice {
  int nt = 0;         // threads per CTA
  int bx = 0;         // points per thread along x
  int by = 0;         // points per thread along y (3D)
  int ntx = 0;        // threads along x (3D)
  int segments = 0;   // CTA segments along the stream dimension
  int max_loops = 0;  // loops per sub-chain (kernel)
  int minb = 0;       // __launch_bounds__ minimum CTAs per SM
  int prefetch = -1;  // L2 prefetch distance (rows) of HBM inputs, 0 = off
};

struct StreamDevice {
  int num_sms = 148;
  int64_t smem_optin = 232448;
  int64_t regs_per_sm = 65536;
};

// One generated kernel: a sub-chain [begin, end) of the flushed chain.
struct StreamKernel {
  size_t begin = 0, end = 0;
  std::string source;
  uint64_t hash = 0;  // of the source (JIT cache key)
  int dim = 2;
  int nt = 0, minb = 1;
  int smem_bytes = 0;
  int64_t nctas = 0;
  // Chain datasets of this kernel, in slot order (kernel argument arrays).
  std::vector<DatasetId> dats;
  std::vector<uint8_t> load;      // input version read from HBM
  std::vector<uint8_t> store;     // final version written to HBM
  std::vector<uint8_t> pingpong;  // stored into the second buffer (then swapped)
  std::vector<Range> store_box;   // write hull of each stored dataset
  std::vector<int32_t> param_off; // per loop of the sub-chain
  int nparams = 0;
  std::vector<int32_t> red_op;    // per reducing loop, chain order
  // Shape (reported).
  int tile[2] = {1, 1};      // computed cross-section tile (points)
  int owned[2] = {1, 1};     // owned cross-section per CTA (interior tiles)
  int grid[3] = {1, 1, 1};   // CTAs along x, y (3D), stream segments
  int bx = 1, by = 1, ntx = 1;
  int64_t ext[3][2] = {};    // overlapped-tile extension per dim / side
  int lag_max = 0;           // pipeline depth in rows
  int ring_doubles = 0;      // register-ring doubles per point
  int smem_stages = 0;       // stages staging a plane through shared memory
  int64_t computed_points = 0;  // loop-point evaluations per launch (incl. redundancy)
  int64_t recorded_points = 0;  // loop points of the recorded ranges
  // Launch-time segment choice: CTAs = tiles x segments, segments from the
  // compiled kernel's occupancy (whole waves), each at least min_seg rows.
  int64_t tiles = 1;
  int64_t stream_extent = 1;
  int64_t min_seg = 8;
  int64_t warm_rows = 0;          // pipeline warm-up rows per segment
  int64_t tile_points = 1;        // computed cross-section points per CTA
  int live_loops = 0;
  int forced_segments = 0;        // StreamChoice::segments
  // Schedule export (validators): the owned hull, the per-loop ranges and the
  // extension each live loop is computed over beyond a CTA's owned box.
  Range hull;
  std::vector<Range> loop_range;
  std::vector<uint8_t> loop_live;
  std::vector<std::array<int64_t, 6>> loop_need;  // [d * 2 + side]
  // CTA plans as text, one line per (CTA, loop): "cta=<i> loop=<l> owned=<box> range=<box>"
  // (range empty for loops the kernel does not execute), for ns stream segments.
  std::string cta_text(int64_t ns) const;
  int64_t segments_for(int64_t slots) const;
  int64_t computed_for(int64_t ns) const { return live_loops * tiles * tile_points * (stream_extent + ns * warm_rows); }
};

struct StreamPlan {
  std::vector<StreamKernel> kernels;
  double build_seconds = 0;
  std::string summary() const;
};

// Plans and generates the kernels of a chain. geoms is indexed by dataset id.
// live_after[ds] == false lets the planner skip storing a dataset's final
// version (none of the product paths do today: every dataset stays live).
// red_mask (optional): reductions only count points inside it (a rank's
// owned box). Throws PlanError when the chain cannot be streamed (1D, a
// loop writing one dataset through two arguments, ...).
StreamPlan build_stream_plan(const LoopChain& chain, const std::vector<StreamGeom>& geoms,
                             const StreamDevice& dev, const StreamChoice& choice, const Range* red_mask);

}  // namespace tcg
