// L2-resident tiled executor: the reference's execute_plan (for tile, for
// loop: execute_loop_range, proj/core/src/executor.cpp:209-250) run by ONE
// persistent cooperative kernel per chain. The host lowers the reference
// tile plan (construct_plan, planner.cpp:55-208) to a list of (tile, loop)
// items in execution order; every CTA of the grid takes a share of each
// item's points and a grid-wide barrier separates dependent items. Tiles are
// sized so a tile's working set stays in the 126 MB L2 across its loops:
// intermediate values of the chain are written and re-read in L2, and DRAM
// sees roughly one read and one write of each field per chain.
//
// In-place execution is exactly the reference's: the tile plan's
// dependency analysis (RAW / WAR extents) is what makes tile-by-tile order
// equal to loop-by-loop order, so no ping-pong buffers are needed.
// Loads are ordinary (coherent) global loads -- data written by an earlier
// item on another SM must be seen after the barrier, which rules out the
// non-coherent __ldg path.
#include <cooperative_groups.h>

#include "tcg_common.cuh"

namespace tcg {

namespace {

namespace cg = cooperative_groups;

// Per-loop descriptor (built on the host for the current field buffers),
// staged into shared memory at the start of each item.
struct LArg {
  double* base;
  int64_t x0, y0, z0, py, pz;
};

struct __align__(16) LoopDesc {
  int32_t body, nargs, red, red_op, param_off, pad[3];
  int32_t mode[kMaxArgs], stencil[kMaxArgs];
  LArg a[kMaxArgs];
};

// Global load the compiler may reorder against this item's stores: within
// one item no point reads a location another point writes (par_loop's race
// rule, runtime.cpp:56-76), and every address depends on the item fetched
// after the last grid barrier, so the load cannot move above that barrier.
// Same instruction (coherent ld.global) as a plain load; only the C++
// aliasing constraint is dropped, which lets a thread's loads for its whole
// run of points issue together.
template <int LM>
__device__ __forceinline__ double ld_item(const double* p) {
  double v;
  if (LM == 1) return __ldg(p);
  if (LM == 2) return __ldcg(p);
  asm("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

constexpr int kL2MaxLoops = 32;  // loop descriptors live in the kernel parameters

struct L2Launch {
  int32_t nitems, nred, masked, dataflow;
  const DevItem* items;
  const int32_t* deps;
  uint32_t* flags;
  uint32_t epoch;
  int32_t reach[3];
  const double* params;
  DevStencils st;
  int32_t red_op[kMaxRed];
  int64_t mlo[3], mhi[3];
  double* partials;  // [nred][gridDim.x]
  LoopDesc loops[kL2MaxLoops];
};

// Accessor for the current point; the loop's argument table is in shared
// memory, the body (and so every argument index it uses) is compile-time.
template <int LM>
struct LAcc {
  const L2Launch& P;
  const LoopDesc& L;  // kernel-parameter space: read-only, never reloaded after stores
  double* c[kMaxArgs];
  int64_t px, py, pz;
  double acc;
  __device__ __forceinline__ double* at(int a, int dx, int dy, int dz) const {
    return c[a] + (dz * L.a[a].pz + dy * L.a[a].py + dx);
  }
  __device__ __forceinline__ void locate() {
#pragma unroll
    for (int a = 0; a < kMaxArgs; ++a)
      if (a < L.nargs) {
        const LArg& g = L.a[a];
        c[a] = g.base + ((pz - g.z0) * g.pz + (py - g.y0) * g.py + (px - g.x0));
      }
  }
  template <int DIM>
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int a = 0; a < kMaxArgs; ++a)
      if (a < L.nargs) c[a] += DIM == 3 ? L.a[a].pz : L.a[a].py;
  }
  __device__ __forceinline__ int64_t x() const { return px; }
  __device__ __forceinline__ int64_t y() const { return py; }
  __device__ __forceinline__ int64_t z() const { return pz; }
  __device__ __forceinline__ double read(int a, int dx, int dy, int dz) const { return ld_item<LM>(at(a, dx, dy, dz)); }
  __device__ __forceinline__ void write(int a, double v) const { *c[a] = v; }
  __device__ __forceinline__ void increment(int a, double v) const { *c[a] = ld_item<LM>(c[a]) + v; }
  __device__ __forceinline__ void contribute(double v) {
    if (P.masked && (px < P.mlo[0] || px >= P.mhi[0] || py < P.mlo[1] || py >= P.mhi[1] || pz < P.mlo[2] ||
                     pz >= P.mhi[2]))
      return;
    acc = red_combine(L.red_op, acc, v);
  }
  __device__ __forceinline__ int nargs() const { return L.nargs; }
  __device__ __forceinline__ int mode(int a) const { return L.mode[a]; }
  __device__ __forceinline__ int npts(int a) const { return P.st.npts[L.stencil[a]]; }
  __device__ __forceinline__ int pt(int a, int j, int d) const {
    return P.st.pts[3 * (P.st.start[L.stencil[a]] + j) + d];
  }
  __device__ __forceinline__ bool reduces() const { return L.red >= 0; }
};

constexpr int kRun = kL2Run;  // rows (2D) / planes (3D) per thread

// Points of one item handled by this CTA: chunks of 32 x (8*kRun) (2D),
// 32 x 8 x kRun (3D) or 256 (1D), grid-strided over the CTAs.
template <int DIM, int BODY, int LM>
__device__ __forceinline__ double run_item(const L2Launch& P, const LoopDesc& L, const DevItem& I) {
  LAcc<LM> a{P, L, {}, 0, 0, 0, red_identity(L.red_op)};
  const double* prm = P.params + L.param_off;
  const uint32_t nch = static_cast<uint32_t>(I.nch);
  if (DIM == 1) {
    for (uint32_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
      a.px = I.lo[0] + static_cast<int64_t>(ch) * 256 + threadIdx.x + 32 * threadIdx.y;
      if (a.px < I.hi[0]) {
        a.locate();
        tcb::run_body(BODY, a, prm);
      }
    }
    return a.acc;
  }
  const uint32_t cx = static_cast<uint32_t>(I.cx), cy = static_cast<uint32_t>(I.cy);
  for (uint32_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const uint32_t ix = ch % cx, rest = ch / cx;
    const uint32_t iy = DIM == 2 ? rest : rest % cy, iz = DIM == 2 ? 0 : rest / cy;
    a.px = I.lo[0] + static_cast<int32_t>(ix * 32 + threadIdx.x);
    int r0, rend;
    if (DIM == 2) {
      r0 = I.lo[1] + static_cast<int32_t>((iy * 8 + threadIdx.y) * kRun);
      rend = I.hi[1];
      a.py = r0;
      a.pz = 0;
    } else {
      a.py = I.lo[1] + static_cast<int32_t>(iy * 8 + threadIdx.y);
      r0 = I.lo[2] + static_cast<int32_t>(iz * kRun);
      rend = I.hi[2];
      a.pz = r0;
    }
    const bool active = a.px < I.hi[0] && (DIM == 2 || a.py < I.hi[1]) && r0 < rend;
    if (active) {
      a.locate();
      if (r0 + kRun <= rend) {
#pragma unroll
        for (int k = 0; k < kRun; ++k) {
          tcb::run_body(BODY, a, prm);
          a.template advance<DIM>();
          if (DIM == 2) ++a.py; else ++a.pz;
        }
      } else {
        for (int k = r0; k < rend; ++k) {
          tcb::run_body(BODY, a, prm);
          a.template advance<DIM>();
          if (DIM == 2) ++a.py; else ++a.pz;
        }
      }
    }
  }
  return a.acc;
}

template <int DIM, int LM>
__global__ void __launch_bounds__(256, 4) k_l2tiled(const __grid_constant__ L2Launch P) {
  __shared__ double red_cta[kMaxRed];
  const int tid = threadIdx.x + 32 * threadIdx.y;
  if (tid < kMaxRed) red_cta[tid] = red_identity(tid < P.nred ? P.red_op[tid] : 0);
  cg::grid_group grid = cg::this_grid();
  for (int it = 0; it < P.nitems; ++it) {
    const DevItem I = P.items[it];
    const LoopDesc& L = P.loops[I.loop];
    double v = red_identity(L.red >= 0 ? L.red_op : 0);
    tcb::dispatch(L.body, [&](auto tag) {
      constexpr int B = decltype(tag)::value;
      v = run_item<DIM, B, LM>(P, L, I);
    });
    if (L.red >= 0) {
      // Deterministic: fixed chunk -> thread assignment, fixed fold order.
      v = block_reduce(v, L.red_op);
      if (tid == 0) red_cta[L.red] = red_combine(L.red_op, red_cta[L.red], v);
    }
    if (I.sync) grid.sync();
  }
  __syncthreads();
  if (tid < P.nred) P.partials[static_cast<int64_t>(tid) * gridDim.x + blockIdx.x] = red_cta[tid];
}

static_assert(sizeof(LoopDesc) % 16 == 0, "LoopDesc is copied as int4 words");

template <int DIM, int LM>
int l2_grid(const DeviceInfo& info) {
  static int blocks = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_l2tiled<DIM, LM>, 256, 0);
    return b;
  }();
  return std::max(1, blocks) * info.num_sms;
}

}  // namespace

void DeviceExec::run_l2(const DevChain& ch, const std::vector<DevItem>& items, const std::vector<int32_t>& deps,
                        const std::array<int32_t, 3>& reach, uint64_t key, double* red_out) {
  mark_chain_writes(ch);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  if (ch.dat_ids.size() > static_cast<size_t>(kMaxChainDats))
    throw PlanError("tiled executor: chain touches more than 32 datasets");
  if (ch.nred > kMaxRed) throw PlanError("tiled executor: more than 8 reducing loops in one chain");
  // Item list, dependency lists and completion flags: cached per plan key.
  ItemBufs* ib = nullptr;
  for (auto& ic : item_cache_)
    if (ic.key == key && ic.nitems == items.size()) ib = &ic;
  if (!ib) {
    ItemBufs nb;
    nb.key = key;
    nb.nitems = items.size();
    size_t nflags = 0;
    for (const DevItem& it : items) nflags = std::max(nflags, static_cast<size_t>(it.flag_off + it.nch));
    TCG_CK(cudaMalloc(&nb.items, std::max<size_t>(1, items.size()) * sizeof(DevItem)));
    TCG_CK(cudaMalloc(&nb.deps, std::max<size_t>(1, deps.size()) * sizeof(int32_t)));
    TCG_CK(cudaMalloc(&nb.flags, std::max<size_t>(1, nflags) * sizeof(uint32_t)));
    TCG_CK(cudaMemsetAsync(nb.flags, 0, std::max<size_t>(1, nflags) * sizeof(uint32_t), st));
    TCG_CK(cudaMemcpyAsync(nb.items, items.data(), items.size() * sizeof(DevItem), cudaMemcpyHostToDevice, st));
    if (!deps.empty())
      TCG_CK(cudaMemcpyAsync(nb.deps, deps.data(), deps.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    if (item_cache_.size() >= 256) {
      TCG_CK(cudaStreamSynchronize(st));
      cudaFree(item_cache_.front().items);
      cudaFree(item_cache_.front().deps);
      cudaFree(item_cache_.front().flags);
      item_cache_.erase(item_cache_.begin());
    }
    item_cache_.push_back(nb);
    ib = &item_cache_.back();
  }
  // Chain tables + per-loop descriptors (into the kernel parameters) for
  // the current field buffers.
  if (ch.loops.size() > static_cast<size_t>(kL2MaxLoops))
    throw PlanError("L2 tiled executor: more than 32 loops in one launch");
  void* scratch = ensure_scratch(chain_bytes(ch));
  const ChainDev cd = upload_chain(ch, scratch, st, &scratch_hash_);
  static L2Launch P;  // large (kernel parameters); host copy reused
  std::memset(&P, 0, sizeof P);
  for (size_t l = 0; l < ch.loops.size(); ++l) {
    const DevLoop& lp = ch.loops[l];
    LoopDesc& d = P.loops[l];
    d.body = lp.body;
    d.nargs = lp.nargs;
    d.red = lp.red;
    d.red_op = lp.red >= 0 ? lp.red_op : 0;
    d.param_off = lp.param_off;
    for (int a = 0; a < lp.nargs; ++a) {
      const DevView v = view(ch.dat_ids[static_cast<size_t>(lp.args[a].dat)], false);
      d.a[a] = LArg{v.base, v.x0, v.y0, v.z0, v.py, v.pz};
      d.mode[a] = lp.args[a].mode;
      d.stencil[a] = lp.args[a].stencil;
    }
  }
  P.nitems = static_cast<int32_t>(items.size());
  P.nred = ch.nred;
  P.items = ib->items;
  P.deps = ib->deps;
  P.flags = ib->flags;
  P.dataflow = 0;
  P.epoch = ++epoch_;
  for (int d = 0; d < 3; ++d) P.reach[d] = reach[static_cast<size_t>(d)];
  P.params = cd.params;
  P.st = cd.st;
  for (int r = 0; r < ch.nred; ++r) P.red_op[r] = ch.red_op[static_cast<size_t>(r)];
  P.masked = ch.masked ? 1 : 0;
  for (int d = 0; d < 3; ++d) {
    P.mlo[d] = ch.mask[d][0];
    P.mhi[d] = ch.mask[d][1];
  }
  static const int lm = [] {
    const char* e = std::getenv("TCG_L2_LOADS");
    return e ? std::atoi(e) : 0;
  }();
  const int grid = lm == 1 ? (ch.dim == 1 ? l2_grid<1, 1>(info_) : ch.dim == 2 ? l2_grid<2, 1>(info_) : l2_grid<3, 1>(info_))
                 : lm == 2 ? (ch.dim == 1 ? l2_grid<1, 2>(info_) : ch.dim == 2 ? l2_grid<2, 2>(info_) : l2_grid<3, 2>(info_))
                           : (ch.dim == 1 ? l2_grid<1, 0>(info_) : ch.dim == 2 ? l2_grid<2, 0>(info_) : l2_grid<3, 0>(info_));
  if (ch.nred > 0) P.partials = ensure_partials(static_cast<size_t>(ch.nred) * grid);
  void* args[] = {&P};
  void* e0 = nullptr;
  if (timing_) {
    e0 = take_event();
    TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e0), st));
  }
  const void* fns[3][3] = {{reinterpret_cast<const void*>(k_l2tiled<1, 0>), reinterpret_cast<const void*>(k_l2tiled<1, 1>),
                            reinterpret_cast<const void*>(k_l2tiled<1, 2>)},
                           {reinterpret_cast<const void*>(k_l2tiled<2, 0>), reinterpret_cast<const void*>(k_l2tiled<2, 1>),
                            reinterpret_cast<const void*>(k_l2tiled<2, 2>)},
                           {reinterpret_cast<const void*>(k_l2tiled<3, 0>), reinterpret_cast<const void*>(k_l2tiled<3, 1>),
                            reinterpret_cast<const void*>(k_l2tiled<3, 2>)}};
  const void* fn = fns[ch.dim - 1][lm < 0 || lm > 2 ? 0 : lm];
  TCG_CK(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(32, 8), args, 0, st));
  if (timing_) {
    void* e1 = take_event();
    TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e1), st));
    ev_tiled_.emplace_back(e0, e1);
  }
  ++launches_;
  for (int r = 0; r < ch.nred; ++r) {
    k_fold<<<1, 1024, 0, st>>>(P.partials + static_cast<int64_t>(r) * grid, grid, P.red_op[r], red_dev_ + r);
    TCG_CK(cudaGetLastError());
    ++launches_;
  }
  if (ch.nred > 0) {
    read_reductions(red_out, ch.nred);
  }
}

}  // namespace tcg
