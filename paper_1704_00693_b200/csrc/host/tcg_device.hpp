// Plain-old-data descriptors that cross from the host planner to the CUDA
// executors (csrc/cuda/tcg_exec.cu). No torch or STL types: these are the
// "chain descriptor" and "plan descriptor" of the C-ABI boundary
// (SURVEY.md §8(b)).
#pragma once
#include <cstdint>

namespace tcg {

constexpr int kMaxArgs = 12;        // arguments per loop
constexpr int kMaxChainDats = 32;   // distinct datasets per chain (tiled executor)
constexpr int kMaxRed = 8;          // reducing loops per tiled chain
// Rows (2D) / planes (3D) each thread of the L2-tiled executor walks per
// chunk; chunks are 32 x 8*kL2Run (2D) and 32 x 8 x kL2Run (3D) points.
constexpr int kL2Run = 4;  // 8 measured: c1 -7%, c3 -9%, c2 +18% (tools/ab_l2run.sh)

// One dataset buffer on the device. Element (x, y, z) lives at
// base[(z - z0) * pz + (y - y0) * py + (x - x0)], where x0 is a multiple of 16
// (so even x is 16-byte aligned, x % 16 == 0 is 128-byte aligned) and py is a
// multiple of 16 elements. The buffer has >= 16 elements of slack before the
// allocation's first point and after its last point in x.
// Layout of a field buffer over allocation box [lo, hi) (dim 0 fastest):
// x origin a multiple of 16 at least 16 elements before the allocation, row
// pitch a multiple of 16 elements.
struct FieldLayout {
  int64_t x0, py, ny, nz, pz;
};
inline FieldLayout field_layout(int dim, const int64_t lo[3], const int64_t hi[3]) {
  auto fl16 = [](int64_t v) { return v >= 0 ? v / 16 * 16 : -((-v + 15) / 16) * 16; };
  FieldLayout L;
  L.x0 = fl16(lo[0]) - 16;
  L.py = ((hi[0] + 16 - L.x0) + 15) / 16 * 16;
  L.ny = dim >= 2 ? hi[1] - lo[1] : 1;
  L.nz = dim >= 3 ? hi[2] - lo[2] : 1;
  L.pz = L.py * L.ny;
  return L;
}

struct DevView {
  double* base;
  int64_t x0, y0, z0;
  int64_t py, pz;
  int64_t alo[3], ahi[3];  // allocation box (global coordinates)
};

struct DevArg {
  int32_t dat;      // chain-local dataset slot
  int32_t stencil;  // index into the chain stencil table
  int32_t mode;     // tcb::Mode
  int32_t pad;
};

struct DevLoop {
  int32_t body;
  int32_t nargs;
  int32_t red;      // chain-local reduction index, -1 if none
  int32_t red_op;   // tcb::RedOp
  int32_t param_off;
  int32_t nparams;
  int32_t pad[2];
  int64_t range[3][2];
  DevArg args[kMaxArgs];
};

// One (tile, loop) work item of the L2-resident tiled executor: the loop's
// range inside the tile (TilingPlan::range(t, l), planner.cpp:158-201).
struct DevItem {
  int32_t loop;
  int32_t sync;        // 1: grid barrier after this item (barrier mode)
  int32_t lo[3], hi[3];
  int32_t cx, cy, nch; // chunk grid of the item (x chunks, y chunks, total)
  int32_t flag_off;    // dataflow mode: first completion flag of this item's chunks
  int32_t dep_off;     // dataflow mode: deps[dep_off, dep_off + ndeps) = earlier items it conflicts with
  int32_t ndeps;
  int32_t pad[2];
};

// Stencil table: points of stencil s are pts[3*start[s] ..].
struct DevStencils {
  const int32_t* start;
  const int32_t* npts;
  const int32_t* pts;
};

// ---- windowed tiled executor plan (one "rank" per CTA) ----------------------
// Coordinates are global int32. Stream dimension = chain dim - 1 (y in 2D,
// z in 3D, x in 1D); "columns" are the remaining dims.
struct DevCta {
  int32_t ntiles;
  int32_t box_off;   // boxes[box_off + (t*L + l)*6 + 2*d + {0,1}]
  int32_t win_off;   // win[win_off + (t*ndat + k)*2 + {0 lo, 1 hi}] for t in [0, ntiles]
  int32_t pad0;
  int32_t col_lo[2], col_hi[2];  // window columns (x even-aligned)
  int32_t own_lo[3], own_hi[3];  // reduction mask (decomposition of the union bounds)
  int32_t wb_lo[3], wb_hi[3];    // write-back ownership (owned, widened to the allocation at edges)
  int32_t W[kMaxChainDats];      // window depth (rows) per chain dataset, 0 = absent
  int32_t sbase[kMaxChainDats];  // shared-memory offset (doubles) of each window
};

// Per chain dataset, same for every CTA.
struct DevDat {
  int32_t load;       // window rows are loaded from `src`
  int32_t written;    // some loop writes it
  int32_t pingpong;   // src != dst: read old, write owned points to the other buffer
  int32_t wbox_off;   // in-place write-back boxes: wboxes[(wbox_off + i)*6 ..]
  int32_t nwbox;
  int32_t reach;      // R: largest |stream offset| of any read; windows keep R
                      // mirror rows on each side so reads never wrap
};

struct DevTiledPlan {
  int32_t dim;
  int32_t nloops;
  int32_t ndat;
  int32_t nred;
  int32_t nctas;
  int32_t smem_doubles;  // max over CTAs (window storage only)
  int32_t prefetch;      // windows are deep enough to load slab t+1 while slab t computes
  const DevCta* ctas;
  const int32_t* boxes;
  const int32_t* win;
  const int32_t* wboxes;
  const DevLoop* loops;
  const double* params;
  DevStencils stencils;
  DevDat dats[kMaxChainDats];
  DevView src[kMaxChainDats];
  DevView dst[kMaxChainDats];
  int32_t red_op[kMaxRed];
  double* red_partials;  // [nred][nctas]
  double* red_out;       // [nred]
};

}  // namespace tcg
