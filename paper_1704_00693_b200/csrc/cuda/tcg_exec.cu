// CUDA executors for sm_100a (B200) -- the replacement of the reference's
// CPU execute_untiled / execute_plan (proj/core/src/executor.cpp:124-277).
//
//   k_untiled<DIM>   one launch per loop over its recorded range, in place in
//                    HBM (the "untiled" baseline, executor.cpp:252-277). Each
//                    thread runs the loop's registered body at one point;
//                    coalesced along x (dim 0 is fastest in memory).
//   k_tiled<DIM>     the windowed tiled executor: one CTA per "rank" of an
//                    overlapped CTA decomposition; each CTA executes its own
//                    reference-style skewed rank plan on
//                    shared-memory windows that slide along the slowest
//                    dimension, so intermediate values of the chain never
//                    leave the SM.
//   k_fold           deterministic fixed-order fold of per-block reduction
//                    partials (the reference folds worker partials in worker
//                    order, executor.cpp:175-176).
// All arithmetic is fp64 and compiled with -fmad=false so every per-point
// expression rounds exactly like the reference's (FMA-free) host build.
#include "tcg_common.cuh"

namespace tcg {

namespace {

// ---------------------------------------------------------------------------
// Untiled per-loop executor.

struct UArg {
  double* base;
  int64_t x0, y0, z0, py, pz;
  int32_t mode, stencil;
};

struct ULaunch {
  int32_t body, nargs, red_op, has_red;
  int64_t lo[3], n[3];
  int32_t masked, pad_;
  int64_t mlo[3], mhi[3];  // reduction mask (rank-owned box) when masked
  UArg a[kMaxArgs];
  double prm[kMaxParams];
  DevStencils st;
  double* partials;
  // Order-matched Sum (DeviceExec::set_reduction_workers): every point's
  // contribution is stored here at its memory-order index within the loop
  // range instead of being folded by the thread.
  double* capture;
  // L2 prefetch of the block's read footprint (0 = off): union of the read
  // stencils' offsets per dimension, and the mask of arguments that read.
  int32_t pf, rmask;
  int32_t rlo[3], rhi[3];
  int32_t pad3_[3];
  int32_t band;  // 3D: y-blocks per rasterisation band (block_yz), 0 = hardware order
#ifdef TCG_CHECKED
  int64_t alo[kMaxArgs][3], ahi[kMaxArgs][3];  // allocation of each argument
#endif
};

#ifdef TCG_CHECKED
// Checked build (libtcg_checked.so): the reference's KernelCtx checks
// (kernel_ctx.hpp:58-89) on the device -- access mode, stencil membership of
// every read offset, allocation bounds -- reported and trapped.
__device__ __noinline__ void checked_fail(const ULaunch& L, int a, int dx, int dy, int dz, int64_t x, int64_t y,
                                          int64_t z, const char* what) {
  printf("tcg checked: body %d arg %d offset (%d,%d,%d) at point (%lld,%lld,%lld): %s\n", L.body, a, dx, dy, dz,
         static_cast<long long>(x), static_cast<long long>(y), static_cast<long long>(z), what);
  __trap();
}
__device__ __noinline__ void checked_access(const ULaunch& L, int a, int dx, int dy, int dz, int64_t x, int64_t y,
                                            int64_t z, bool rd, bool wr) {
  if (a < 0 || a >= L.nargs) checked_fail(L, a, dx, dy, dz, x, y, z, "argument index out of range");
  const int m = L.a[a].mode;
  if (rd && m == tcb::kWrite) checked_fail(L, a, dx, dy, dz, x, y, z, "read of a Write-mode argument");
  if (wr && m == tcb::kRead) checked_fail(L, a, dx, dy, dz, x, y, z, "write of a Read-mode argument");
  if (rd) {
    const int s = L.a[a].stencil, n = L.st.npts[s], b = L.st.start[s];
    bool found = false;
    for (int j = 0; j < n && !found; ++j)
      found = L.st.pts[3 * (b + j)] == dx && L.st.pts[3 * (b + j) + 1] == dy && L.st.pts[3 * (b + j) + 2] == dz;
    if (!found) checked_fail(L, a, dx, dy, dz, x, y, z, "offset is not a point of the argument's stencil");
  }
  const int64_t p[3] = {x + dx, y + dy, z + dz};
  for (int d = 0; d < 3; ++d)
    if (p[d] < L.alo[a][d] || p[d] >= L.ahi[a][d])
      checked_fail(L, a, dx, dy, dz, x, y, z, "access outside the allocated extent");
}
#define TCG_CHECK_ACCESS(a, dx, dy, dz, rd, wr) checked_access(L, a, dx, dy, dz, px, py, pz, rd, wr)
#else
#define TCG_CHECK_ACCESS(a, dx, dy, dz, rd, wr) ((void)0)
#endif

// Issues one bulk L2 prefetch (cp.async.bulk.prefetch.L2) per row segment of
// the block's read footprint, for every reading argument, before any point
// is computed: the block's DRAM misses are then all in flight at once
// instead of one plane / row at a time behind the dependent loads (the 3D
// walk was measured long-scoreboard bound at 46% occupancy).
// 3D block order. The hardware walks blockIdx x-fastest, then y, then z: two
// z-chunks of the same column run a whole plane-chunk apart (c5: 6 fields x
// 4 planes x 4.7 MB = 113 MB, the size of L2), so the z-halo planes of the
// radius-2 stars were re-read from HBM (2.09x read amplification on the
// energy RHS, profiles/r3/c5_untiled.md). With a band of L.band y-blocks the
// linear (y, z) index is re-read as (y inside the band, z-chunk, band): a
// column's z-chunks follow each other within one band, and only the band's
// edge rows are fetched twice.
__device__ __forceinline__ void block_yz(const ULaunch& L, unsigned& by, unsigned& bz) {
  by = blockIdx.y;
  bz = blockIdx.z;
  const unsigned band = static_cast<unsigned>(L.band);
  if (band == 0 || band >= gridDim.y) return;
  const unsigned ny = gridDim.y, nz = gridDim.z;
  const unsigned lin = blockIdx.y + ny * blockIdx.z;
  const unsigned full = (ny / band) * band * nz;  // blocks in whole bands
  if (lin < full) {
    const unsigned b = lin / (band * nz), r = lin - b * band * nz;
    bz = r / band;
    by = b * band + (r - bz * band);
  } else {
    const unsigned w = ny % band, r = lin - full;
    bz = r / w;
    by = (ny / band) * band + (r - bz * w);
  }
}

template <int DIM, int RUN>
__device__ __forceinline__ void prefetch_footprint(const ULaunch& L) {
  const int64_t xe = L.lo[0] + L.n[0], ye = L.lo[1] + L.n[1], ze = L.lo[2] + L.n[2];
  const int64_t x0 = L.lo[0] + static_cast<int64_t>(blockIdx.x) * blockDim.x;
  const int64_t x1 = min(x0 + static_cast<int64_t>(blockDim.x), xe);
  int64_t y0, y1, z0, z1;
  if (DIM == 2) {
    y0 = L.lo[1] + static_cast<int64_t>(blockIdx.y) * blockDim.y * RUN;
    y1 = min(y0 + static_cast<int64_t>(blockDim.y) * RUN, ye);
    z0 = 0;
    z1 = 1;
  } else {
    unsigned by, bz;
    block_yz(L, by, bz);
    y0 = L.lo[1] + static_cast<int64_t>(by) * blockDim.y;
    y1 = min(y0 + static_cast<int64_t>(blockDim.y), ye);
    z0 = L.lo[2] + static_cast<int64_t>(bz) * RUN;
    z1 = min(z0 + static_cast<int64_t>(RUN), ze);
  }
  if (x0 >= x1 || y0 >= y1 || z0 >= z1) return;
  const int64_t ex0 = x0 + L.rlo[0], ex1 = x1 + L.rhi[0];
  const int64_t ey0 = y0 + L.rlo[1], ny = (y1 + L.rhi[1]) - ey0;
  const int64_t ez0 = DIM == 3 ? z0 + L.rlo[2] : 0, nz = DIM == 3 ? (z1 + L.rhi[2]) - ez0 : 1;
  const int rows = static_cast<int>(ny * nz);
  const int nread = __popc(static_cast<unsigned>(L.rmask));
  const int tid = threadIdx.x + blockDim.x * threadIdx.y, nth = blockDim.x * blockDim.y;
  for (int i = tid; i < nread * rows; i += nth) {
    const int k = i / rows, row = i - k * rows;
    unsigned m = static_cast<unsigned>(L.rmask);
    for (int j = 0; j < k; ++j) m &= m - 1;  // k-th reading argument
    const UArg& g = L.a[__ffs(m) - 1];
    const int64_t yy = ey0 + row % ny, zz = ez0 + row / ny;
    const char* p0 = reinterpret_cast<const char*>(g.base + ((zz - g.z0) * g.pz + (yy - g.y0) * g.py + (ex0 - g.x0)));
    const char* p1 = reinterpret_cast<const char*>(g.base + ((zz - g.z0) * g.pz + (yy - g.y0) * g.py + (ex1 - g.x0)));
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p0) & ~uintptr_t{15};
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p1) + 15) & ~uintptr_t{15};
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(static_cast<unsigned>(a1 - a0)) : "memory");
  }
}

// Accessor over HBM. c[a] points at argument a's element for the current
// point; a thread walks a short run of rows, advancing every pointer by one
// row pitch. All reads use the read-only (non-coherent) path: legal because
// a loop never reads a point another point of the same loop writes
// (runtime.cpp:56-76), and it lets the compiler keep overlapping stencil
// rows of consecutive points in registers.
struct GAcc {
  const ULaunch& L;
  double* c[kMaxArgs];
  int64_t px, py, pz;
  double acc;
  __device__ __forceinline__ double* at(int a, int dx, int dy, int dz) const {
    const UArg& g = L.a[a];
    return c[a] + (dz * g.pz + dy * g.py + dx);
  }
  __device__ __forceinline__ void locate() {
#pragma unroll
    for (int a = 0; a < kMaxArgs; ++a) {
      const UArg& g = L.a[a];
      c[a] = g.base + ((pz - g.z0) * g.pz + (py - g.y0) * g.py + (px - g.x0));
    }
  }
  template <int DIM>
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int a = 0; a < kMaxArgs; ++a) c[a] += DIM == 3 ? L.a[a].pz : L.a[a].py;
  }
  __device__ __forceinline__ int64_t x() const { return px; }
  __device__ __forceinline__ int64_t y() const { return py; }
  __device__ __forceinline__ int64_t z() const { return pz; }
  __device__ __forceinline__ double read(int a, int dx, int dy, int dz) const {
    TCG_CHECK_ACCESS(a, dx, dy, dz, true, false);
    return __ldg(at(a, dx, dy, dz));
  }
  __device__ __forceinline__ void write(int a, double v) const {
    TCG_CHECK_ACCESS(a, 0, 0, 0, false, true);
    *c[a] = v;
  }
  __device__ __forceinline__ void increment(int a, double v) const {
    TCG_CHECK_ACCESS(a, 0, 0, 0, true, true);
    *c[a] = __ldg(c[a]) + v;
  }
  __device__ __forceinline__ void contribute(double v) {
    if (L.masked && (px < L.mlo[0] || px >= L.mhi[0] || py < L.mlo[1] || py >= L.mhi[1] || pz < L.mlo[2] ||
                     pz >= L.mhi[2]))
      return;
    if (L.capture) {
      L.capture[((pz - L.lo[2]) * L.n[1] + (py - L.lo[1])) * L.n[0] + (px - L.lo[0])] = v;
      return;
    }
    acc = red_combine(L.red_op, acc, v);
  }
  __device__ __forceinline__ int nargs() const { return L.nargs; }
  __device__ __forceinline__ int mode(int a) const { return L.a[a].mode; }
  __device__ __forceinline__ int npts(int a) const { return L.st.npts[L.a[a].stencil]; }
  __device__ __forceinline__ int pt(int a, int j, int d) const {
    return L.st.pts[3 * (L.st.start[L.a[a].stencil] + j) + d];
  }
  __device__ __forceinline__ bool reduces() const { return L.has_red != 0; }
};

// Order-matched Sum, the reference's fold (executor.cpp:55-61 slice,
// :141-144 per-worker partials from the identity, :175-176 worker-order
// fold): block w sums span w of the captured contributions sequentially --
// the block stages chunks through shared memory, thread 0 adds them in index
// order -- and the last block to finish folds the T partials in worker order.
__global__ void __launch_bounds__(256) k_ordered_sum(const double* __restrict__ vals, int64_t n, int workers, double* part,
                                                     unsigned* ticket, double* out) {
  constexpr int kChunk = 2048;
  __shared__ double buf[kChunk];
  const int64_t T = workers, w = blockIdx.x;
  const int64_t base = n / T, rem = n % T;
  const int64_t begin = w * base + (w < rem ? w : rem);
  const int64_t end = begin + base + (w < rem ? 1 : 0);
  double acc = 0.0;  // reduce_identity(Sum)
  for (int64_t c = begin; c < end; c += kChunk) {
    const int m = static_cast<int>(end - c < kChunk ? end - c : kChunk);
    for (int i = threadIdx.x; i < m; i += blockDim.x) buf[i] = __ldg(vals + c + i);
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 8
      for (int i = 0; i < m; ++i) acc = acc + buf[i];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[w] = acc;
    __threadfence();
    if (atomicAdd(ticket, 1u) == static_cast<unsigned>(workers) - 1) {
      __threadfence();
      double r = 0.0;
      for (int i = 0; i < workers; ++i) r = r + __ldcg(part + i);
      *out = r;
      *ticket = 0u;
    }
  }
}

// Two-pass run for bodies whose reads are few and in a data-independent order
// but whose arithmetic holds a branchy IEEE division (c2's CFL min-reduction,
// 0.5 / (rho + p * c)): the division's slow-path call fences the compiler's
// load scheduling, so a plain run keeps only one row's reads in flight
// (measured 4.4 TB/s against 6.4 for point loops). Pass 1 issues every read
// of the whole run into registers (the body's arithmetic is dead there and
// removed); pass 2 replays the body on the buffered values in the same order,
// so the results are the plain run's bit for bit.
template <int BODY>
struct BatchReads {
  static constexpr int kReads = BODY == tcb::kHydroCfl ? 3 : 0;
};

constexpr int kBatchRows = 2;

template <int N>
struct PreAcc {
  const GAcc& g;
  double* buf;
  mutable int i;
  __device__ __forceinline__ double read(int a, int dx, int dy, int dz) const {
    const double v = g.read(a, dx, dy, dz);
    if (i < N) buf[i] = v;
    ++i;
    return v;
  }
  __device__ __forceinline__ void write(int, double) const {}
  __device__ __forceinline__ void increment(int, double) const {}
  __device__ __forceinline__ void contribute(double) const {}
  __device__ __forceinline__ int64_t x() const { return g.x(); }
  __device__ __forceinline__ int64_t y() const { return g.y(); }
  __device__ __forceinline__ int64_t z() const { return g.z(); }
  __device__ __forceinline__ int nargs() const { return g.nargs(); }
  __device__ __forceinline__ int mode(int a) const { return g.mode(a); }
  __device__ __forceinline__ int npts(int a) const { return g.npts(a); }
  __device__ __forceinline__ int pt(int a, int j, int d) const { return g.pt(a, j, d); }
  __device__ __forceinline__ bool reduces() const { return g.reduces(); }
};

template <int N>
struct ReplayAcc {
  GAcc& g;
  const double* buf;
  mutable int i;
  __device__ __forceinline__ double read(int, int, int, int) const { return buf[i++]; }
  __device__ __forceinline__ void write(int a, double v) const { g.write(a, v); }
  __device__ __forceinline__ void increment(int a, double v) const { g.increment(a, v); }
  __device__ __forceinline__ void contribute(double v) const { g.contribute(v); }
  __device__ __forceinline__ int64_t x() const { return g.x(); }
  __device__ __forceinline__ int64_t y() const { return g.y(); }
  __device__ __forceinline__ int64_t z() const { return g.z(); }
  __device__ __forceinline__ int nargs() const { return g.nargs(); }
  __device__ __forceinline__ int mode(int a) const { return g.mode(a); }
  __device__ __forceinline__ int npts(int a) const { return g.npts(a); }
  __device__ __forceinline__ int pt(int a, int j, int d) const { return g.pt(a, j, d); }
  __device__ __forceinline__ bool reduces() const { return g.reduces(); }
};

// Rows (2D: y, 3D: z) walked by one thread of the untiled executor
// (template parameter kUntiledRun of k_untiled; 4 unless tuned).

template <int DIM, int BODY, int kUntiledRun>
__device__ __forceinline__ void untiled_block(const ULaunch& L) {
  if (DIM >= 2 && L.pf) prefetch_footprint<DIM, kUntiledRun>(L);
  GAcc acc{L, {}, 0, 0, 0, red_identity(L.red_op)};
  if (DIM == 1) {
    acc.px = L.lo[0] + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (acc.px < L.lo[0] + L.n[0]) {
      acc.locate();
      tcb::run_body(BODY, acc, L.prm);
    }
  } else {
    acc.px = L.lo[0] + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t r0, rend;
    if (DIM == 2) {
      r0 = L.lo[1] + (static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y) * kUntiledRun;
      rend = L.lo[1] + L.n[1];
      acc.py = r0;
    } else {
      unsigned by, bz;
      block_yz(L, by, bz);
      acc.py = L.lo[1] + static_cast<int64_t>(by) * blockDim.y + threadIdx.y;
      r0 = L.lo[2] + static_cast<int64_t>(bz) * kUntiledRun;
      rend = L.lo[2] + L.n[2];
      acc.pz = r0;
    }
    const bool active = acc.px < L.lo[0] + L.n[0] && (DIM == 2 || acc.py < L.lo[1] + L.n[1]);
    if (active) {
      acc.locate();
      const int nr = static_cast<int>(min(static_cast<int64_t>(kUntiledRun), rend - r0));
      constexpr int kNR = BatchReads<BODY>::kReads;
      if (kNR > 0 && nr == kUntiledRun) {
        // Chunks of kBatchRows rows: 2D runs sit under a 6-blocks/SM
        // register budget. Measured on c2's CFL loop (plain 91.7 us):
        // 2-row chunks 76.3, 4-row 82.6, the whole 8-row run 100 (spills).
        constexpr int kChunk = kUntiledRun < kBatchRows ? kUntiledRun : kBatchRows;
        static_assert(kUntiledRun % kChunk == 0, "a run is a whole number of read batches");
#pragma unroll
        for (int c0 = 0; c0 < kUntiledRun; c0 += kChunk) {
          double buf[kNR > 0 ? kNR * kChunk : 1];
          GAcc g1 = acc;
#pragma unroll
          for (int k = 0; k < kChunk; ++k) {
            PreAcc<kNR> pa{g1, buf + k * kNR, 0};
            tcb::run_body(BODY, pa, L.prm);
            g1.advance<DIM>();
            if (DIM == 2)  // the checked build reports / bounds-checks against the point's coordinates
              ++g1.py;
            else
              ++g1.pz;
          }
#pragma unroll
          for (int k = 0; k < kChunk; ++k) {
            ReplayAcc<kNR> ra{acc, buf + k * kNR, 0};
            tcb::run_body(BODY, ra, L.prm);
            acc.advance<DIM>();
            if (DIM == 2)
              ++acc.py;
            else
              ++acc.pz;
          }
        }
      } else if (nr == kUntiledRun) {
#pragma unroll
        for (int k = 0; k < kUntiledRun; ++k) {
          tcb::run_body(BODY, acc, L.prm);
          acc.advance<DIM>();
          if (DIM == 2)
            ++acc.py;
          else
            ++acc.pz;
        }
      } else {
        for (int k = 0; k < nr; ++k) {
          tcb::run_body(BODY, acc, L.prm);
          acc.advance<DIM>();
          if (DIM == 2)
            ++acc.py;
          else
            ++acc.pz;
        }
      }
    }
  }
  if (L.has_red) {
    const double v = block_reduce(acc.acc, L.red_op);
    if (threadIdx.x == 0 && threadIdx.y == 0)
      L.partials[blockIdx.x + static_cast<int64_t>(gridDim.x) * (blockIdx.y + static_cast<int64_t>(gridDim.y) * blockIdx.z)] = v;
  }
}

// Register budget per dimension, measured on B200 (tools/ab_minb2.sh): the 2D
// walk is DRAM-latency bound and gains from 6 resident blocks per SM (c2
// -4%); the 3D walk spills and slows under any cap (c5 +20% at 4 blocks).
template <int DIM, int BODY, int kUntiledRun = 4>
__global__ void __launch_bounds__(256) k_untiled(const __grid_constant__ ULaunch L) {
  untiled_block<DIM, BODY, kUntiledRun>(L);
}
template <int BODY, int kUntiledRun = 4>
__global__ void __launch_bounds__(256, 6) k_untiled2(const __grid_constant__ ULaunch L) {
  untiled_block<2, BODY, kUntiledRun>(L);
}

// Periodic ghost fill along dimension D: for every field, the ghost layers
// [L-depth, L) and [H, H+depth) in dim D take the values at +-N, over the
// logical box in later dims and the ghost-extended box in earlier dims.
constexpr int kMaxPeriodic = 16;
struct PLaunch {
  int32_t nf, depth;
  int64_t L[3], H[3];
  UArg f[kMaxPeriodic];
};

template <int D>
__global__ void __launch_bounds__(256) k_periodic(const __grid_constant__ PLaunch P) {
  // Point grid over (2*depth) x ext(other dims), field index in blockIdx.y.
  int64_t ext[3], org[3];
  for (int d = 0; d < 3; ++d) {
    if (d == D) {
      ext[d] = 2 * P.depth;
      org[d] = 0;
    } else if (d < D) {
      ext[d] = P.H[d] - P.L[d] + 2 * P.depth;
      org[d] = P.L[d] - P.depth;
    } else {
      ext[d] = P.H[d] - P.L[d];
      org[d] = P.L[d];
    }
  }
  const int64_t total = ext[0] * ext[1] * ext[2];
  const UArg& g = P.f[blockIdx.y];
  const int64_t N = P.H[D] - P.L[D];
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t c[3];
    c[0] = i % ext[0];
    c[1] = (i / ext[0]) % ext[1];
    c[2] = i / (ext[0] * ext[1]);
    int64_t p[3];
    for (int d = 0; d < 3; ++d) p[d] = org[d] + c[d];
    int64_t s[3] = {p[0], p[1], p[2]};
    if (c[D] < P.depth) {
      p[D] = P.L[D] - P.depth + c[D];
      s[D] = p[D] + N;
    } else {
      p[D] = P.H[D] + (c[D] - P.depth);
      s[D] = p[D] - N;
    }
    double* dst = g.base + ((p[2] - g.z0) * g.pz + (p[1] - g.y0) * g.py + (p[0] - g.x0));
    const double* src = g.base + ((s[2] - g.z0) * g.pz + (s[1] - g.y0) * g.py + (s[0] - g.x0));
    *dst = *src;
  }
}

}  // namespace


// ---------------------------------------------------------------------------
// Host side.

void select_device(int device) {
  int ndev = 0;
  TCG_CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    throw InvalidArgument("select_device: device " + std::to_string(device) + " of " + std::to_string(ndev));
  TCG_CK(cudaSetDevice(device));
}

DeviceExec::DeviceExec() {
  int ndev = 0;
  TCG_CK(cudaGetDeviceCount(&ndev));
  if (ndev <= 0) throw CudaError("no CUDA device visible: the B200 executor has no CPU fallback");
  TCG_CK(cudaGetDevice(&info_.device));
  device_ = info_.device;
  cudaDeviceProp prop;
  TCG_CK(cudaGetDeviceProperties(&prop, info_.device));
  info_.num_sms = prop.multiProcessorCount;
  info_.smem_optin = static_cast<int64_t>(prop.sharedMemPerBlockOptin);
  info_.smem_per_sm = static_cast<int64_t>(prop.sharedMemPerMultiprocessor);
  info_.l2_bytes = prop.l2CacheSize;
  info_.name = prop.name;
  if (prop.major < 10) throw CudaError("executor is built for sm_100a (B200); found " + info_.name);
  cudaStream_t st;
  TCG_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  stream_ = st;
  ensure_red(64);
}

DeviceExec::~DeviceExec() {
  for (Buf* b : fields_) {
    if (b->mem[0]) cudaFree(b->mem[0]);
    if (b->mem[1]) cudaFree(b->mem[1]);
    delete b;
  }
  for (auto& pb : plan_cache_) {
    cudaFree(pb.second->mem);
    delete pb.second;
  }
  for (auto& ic : item_cache_) {
    cudaFree(ic.items);
    cudaFree(ic.deps);
    cudaFree(ic.flags);
  }
  if (scratch_) cudaFree(scratch_);
  if (partials_) cudaFree(partials_);
  if (red_dev_) cudaFree(red_dev_);
  if (red_host_) cudaFreeHost(red_host_);
  if (staging_) cudaFree(staging_);
  if (redbuf_) cudaFree(redbuf_);
  if (st_part_) cudaFree(st_part_);
  if (st_out_) cudaFree(st_out_);
  if (st_ticket_) cudaFree(st_ticket_);
  if (capture_) cudaFree(capture_);
  if (ord_part_) cudaFree(ord_part_);
  if (ord_ticket_) cudaFree(ord_ticket_);
  if (host_stage_) cudaFreeHost(host_stage_);
  drop_graphs();
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

int DeviceExec::add_field(const Range& alloc) {
  auto* b = new Buf;
  b->alloc = alloc;
  const int dim = alloc.dim();
  int64_t lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = d < dim ? alloc.start(d) : 0;
    hi[d] = d < dim ? alloc.end(d) : 1;
  }
  const FieldLayout fl = field_layout(dim, lo, hi);
  b->x0 = fl.x0;
  b->py = fl.py;
  b->ny = fl.ny;
  b->nz = fl.nz;
  b->pz = fl.pz;
  b->bytes = static_cast<size_t>(b->pz * b->nz) * sizeof(double);
  TCG_CK(cudaMalloc(&b->mem[0], b->bytes));
  TCG_CK(cudaMemsetAsync(b->mem[0], 0, b->bytes, static_cast<cudaStream_t>(stream_)));
  fields_.push_back(b);
  return static_cast<int>(fields_.size()) - 1;
}

int64_t DeviceExec::field_bytes(int f) const { return static_cast<int64_t>(fields_.at(static_cast<size_t>(f))->bytes); }

DevView DeviceExec::view(int f, bool alt) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  const int which = alt ? 1 - b->cur : b->cur;
  if (!b->mem[which]) {
    TCG_CK(cudaMalloc(&b->mem[which], b->bytes));
    TCG_CK(cudaMemsetAsync(b->mem[which], 0, b->bytes, static_cast<cudaStream_t>(stream_)));
  }
  DevView v{};
  const int dim = b->alloc.dim();
  v.base = b->mem[which];
  v.x0 = b->x0;
  v.y0 = dim >= 2 ? b->alloc.start(1) : 0;
  v.z0 = dim >= 3 ? b->alloc.start(2) : 0;
  v.py = b->py;
  v.pz = dim >= 3 ? b->pz : 0;
  if (dim < 2) v.py = 0;
  for (int d = 0; d < 3; ++d) {
    v.alo[d] = d < dim ? b->alloc.start(d) : 0;
    v.ahi[d] = d < dim ? b->alloc.end(d) : 1;
  }
  return v;
}

void DeviceExec::swap(int f) { fields_.at(static_cast<size_t>(f))->cur ^= 1; }

namespace {
double* point_addr(const DevView& v, const Range& alloc, const Point& p) {
  if (!alloc.contains(p)) throw AccessError("point outside allocated extent " + alloc.to_string());
  return v.base + ((p[2] - v.z0) * v.pz + (p[1] - v.y0) * v.py + (p[0] - v.x0));
}
}  // namespace

double DeviceExec::get_point(int f, const Point& p) {
  const DevView v = view(f, false);
  double out = 0;
  read_device(&out, point_addr(v, fields_.at(static_cast<size_t>(f))->alloc, p), 1);
  return out;
}

void DeviceExec::put_point(int f, const Point& p, double val) {
  const DevView v = view(f, false);
  double* dst = point_addr(v, fields_.at(static_cast<size_t>(f))->alloc, p);
  // Stream-ordered through the pinned staging buffer (a pageable source may
  // return before the copy lands, and the executor stream is non-blocking).
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  TCG_CK(cudaStreamSynchronize(st));
  red_host_[0] = val;
  TCG_CK(cudaMemcpyAsync(dst, red_host_, 8, cudaMemcpyHostToDevice, st));
  TCG_CK(cudaStreamSynchronize(st));
  Range box(fields_.at(static_cast<size_t>(f))->alloc.dim());
  for (int d = 0; d < box.dim(); ++d) box.set(d, p[d], p[d] + 1);
  mark_written(f, box);
}

namespace {
// A dense or pitched buffer: element (ox, oy, oz) at base, `pitch` elements
// per row, `rows` rows per plane.
struct BoxBuf {
  double* base;
  int64_t ox, oy, oz, pitch, rows;
};

int64_t lo_of(const Range& r, int d) { return d < r.dim() ? r.start(d) : 0; }
int64_t ext_of(const Range& r, int d) { return d < r.dim() ? r.extent(d) : 1; }

BoxBuf dense_buf(double* p, const Range& over) {
  return BoxBuf{p, lo_of(over, 0), lo_of(over, 1), lo_of(over, 2), ext_of(over, 0), ext_of(over, 1)};
}

void copy_box(const BoxBuf& dst, const BoxBuf& src, const Range& box, cudaStream_t st) {
  if (box.empty()) return;
  cudaMemcpy3DParms p{};
  p.srcPtr = make_cudaPitchedPtr(src.base, static_cast<size_t>(src.pitch) * 8, static_cast<size_t>(src.pitch) * 8,
                                 static_cast<size_t>(src.rows));
  p.dstPtr = make_cudaPitchedPtr(dst.base, static_cast<size_t>(dst.pitch) * 8, static_cast<size_t>(dst.pitch) * 8,
                                 static_cast<size_t>(dst.rows));
  p.srcPos = make_cudaPos(static_cast<size_t>(lo_of(box, 0) - src.ox) * 8, static_cast<size_t>(lo_of(box, 1) - src.oy),
                          static_cast<size_t>(lo_of(box, 2) - src.oz));
  p.dstPos = make_cudaPos(static_cast<size_t>(lo_of(box, 0) - dst.ox) * 8, static_cast<size_t>(lo_of(box, 1) - dst.oy),
                          static_cast<size_t>(lo_of(box, 2) - dst.oz));
  p.extent = make_cudaExtent(static_cast<size_t>(ext_of(box, 0)) * 8, static_cast<size_t>(ext_of(box, 1)),
                             static_cast<size_t>(ext_of(box, 2)));
  p.kind = cudaMemcpyDefault;
  TCG_CK(cudaMemcpy3DAsync(&p, st));
}
}  // namespace

void DeviceExec::field_to_buf(int f, const Range& box, double* buf, const Range& buf_box) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  if (!b->alloc.contains(box) || !buf_box.contains(box))
    throw AccessError("field_to_buf: box " + box.to_string() + " outside " + b->alloc.to_string() + " or " +
                      buf_box.to_string());
  const BoxBuf fb{b->mem[b->cur], b->x0, lo_of(b->alloc, 1), lo_of(b->alloc, 2), b->py, b->ny};
  copy_box(dense_buf(buf, buf_box), fb, box, static_cast<cudaStream_t>(stream_));
}

void DeviceExec::buf_to_field(int f, const Range& box, const double* buf, const Range& buf_box) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  if (!b->alloc.contains(box) || !buf_box.contains(box))
    throw AccessError("buf_to_field: box " + box.to_string() + " outside " + b->alloc.to_string() + " or " +
                      buf_box.to_string());
  const BoxBuf fb{b->mem[b->cur], b->x0, lo_of(b->alloc, 1), lo_of(b->alloc, 2), b->py, b->ny};
  copy_box(fb, dense_buf(const_cast<double*>(buf), buf_box), box, static_cast<cudaStream_t>(stream_));
  mark_written(f, box);
}

void DeviceExec::fill_box_bytes(int f, const Range& box, int byte) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  if (!b->alloc.contains(box)) throw AccessError("fill_box_bytes: " + box.to_string() + " outside " + b->alloc.to_string());
  if (box.empty()) return;
  double* base = b->mem[b->cur] + ((lo_of(box, 2) - lo_of(b->alloc, 2)) * b->pz + (lo_of(box, 1) - lo_of(b->alloc, 1)) * b->py +
                                   (lo_of(box, 0) - b->x0));
  const cudaPitchedPtr pp = make_cudaPitchedPtr(base, static_cast<size_t>(b->py) * 8, static_cast<size_t>(b->py) * 8,
                                                static_cast<size_t>(b->ny));
  const cudaExtent ext = make_cudaExtent(static_cast<size_t>(ext_of(box, 0)) * 8, static_cast<size_t>(ext_of(box, 1)),
                                         static_cast<size_t>(ext_of(box, 2)));
  TCG_CK(cudaMemset3DAsync(pp, byte, ext, static_cast<cudaStream_t>(stream_)));
  mark_written(f, box);
}

void DeviceExec::copy_within(int f, const Range& box, const Point& shift) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  Range src(box.dim());
  for (int d = 0; d < box.dim(); ++d) src.set(d, box.start(d) + shift[d], box.end(d) + shift[d]);
  if (!b->alloc.contains(box) || !b->alloc.contains(src))
    throw AccessError("copy_within: " + box.to_string() + " / " + src.to_string() + " outside " + b->alloc.to_string());
  if (box.empty()) return;
  const BoxBuf fb{b->mem[b->cur], b->x0, lo_of(b->alloc, 1), lo_of(b->alloc, 2), b->py, b->ny};
  cudaMemcpy3DParms p{};
  p.srcPtr = p.dstPtr = make_cudaPitchedPtr(fb.base, static_cast<size_t>(fb.pitch) * 8, static_cast<size_t>(fb.pitch) * 8,
                                            static_cast<size_t>(fb.rows));
  p.srcPos = make_cudaPos(static_cast<size_t>(lo_of(src, 0) - fb.ox) * 8, static_cast<size_t>(lo_of(src, 1) - fb.oy),
                          static_cast<size_t>(lo_of(src, 2) - fb.oz));
  p.dstPos = make_cudaPos(static_cast<size_t>(lo_of(box, 0) - fb.ox) * 8, static_cast<size_t>(lo_of(box, 1) - fb.oy),
                          static_cast<size_t>(lo_of(box, 2) - fb.oz));
  p.extent = make_cudaExtent(static_cast<size_t>(ext_of(box, 0)) * 8, static_cast<size_t>(ext_of(box, 1)),
                             static_cast<size_t>(ext_of(box, 2)));
  p.kind = cudaMemcpyDeviceToDevice;
  TCG_CK(cudaMemcpy3DAsync(&p, static_cast<cudaStream_t>(stream_)));
  mark_written(f, box);
}

void DeviceExec::periodic_fill(const std::vector<int>& fields, const Range& logical, int64_t depth, int ndims) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  const int dim = logical.dim();
  const int nd = ndims < 0 ? dim : std::min(ndims, dim);
  for (size_t b = 0; b < fields.size(); b += kMaxPeriodic) {
    PLaunch P{};
    P.nf = static_cast<int32_t>(std::min<size_t>(kMaxPeriodic, fields.size() - b));
    P.depth = static_cast<int32_t>(depth);
    for (int d = 0; d < 3; ++d) {
      P.L[d] = d < dim ? logical.start(d) : 0;
      P.H[d] = d < dim ? logical.end(d) : 1;
    }
    for (int k = 0; k < P.nf; ++k) {
      const DevView v = view(fields[b + static_cast<size_t>(k)], false);
      P.f[k] = UArg{v.base, v.x0, v.y0, v.z0, v.py, v.pz, 0, 0};
    }
    for (int d = 0; d < nd; ++d) {
      int64_t total = 2 * depth;
      for (int e = 0; e < dim; ++e)
        if (e != d) total *= (logical.extent(e) + (e < d ? 2 * depth : 0));
      const dim3 grid(static_cast<unsigned>(std::min<int64_t>(4096, (total + 255) / 256)),
                      static_cast<unsigned>(P.nf));
      if (d == 0)
        k_periodic<0><<<grid, 256, 0, st>>>(P);
      else if (d == 1)
        k_periodic<1><<<grid, 256, 0, st>>>(P);
      else
        k_periodic<2><<<grid, 256, 0, st>>>(P);
      TCG_CK(cudaGetLastError());
      ++launches_;
    }
  }
  // Ghost layers written: the slabs outside the logical box, every dimension.
  for (int f : fields) {
    const Range& al = fields_.at(static_cast<size_t>(f))->alloc;
    for (int d = 0; d < nd; ++d)
      for (int side = 0; side < 2; ++side) {
        Range g(dim);
        for (int e = 0; e < dim; ++e) {
          const int64_t w = e < d ? depth : 0;
          g.set_raw(e, logical.start(e) - w, logical.end(e) + w);
        }
        if (side == 0)
          g.set_raw(d, logical.start(d) - depth, logical.start(d));
        else
          g.set_raw(d, logical.end(d), logical.end(d) + depth);
        mark_written(f, g.intersect(al));
      }
  }
}

double* DeviceExec::staging(size_t n) {
  if (n > staging_n_) {
    if (staging_) TCG_CK(cudaFree(staging_));
    staging_n_ = std::max(n, staging_n_ * 2);
    TCG_CK(cudaMalloc(&staging_, staging_n_ * sizeof(double)));
  }
  return staging_;
}

void DeviceExec::h2d(double* dev, const double* host, size_t n) {
  TCG_CK(cudaMemcpyAsync(dev, host, n * sizeof(double), cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream_)));
}

void DeviceExec::d2h(double* host, const double* dev, size_t n) {
  TCG_CK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)));
  TCG_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
}

double* DeviceExec::red_buffer(size_t n) {
  if (n > redbuf_n_) {
    if (redbuf_) TCG_CK(cudaFree(redbuf_));
    redbuf_n_ = std::max<size_t>(n, 64);
    TCG_CK(cudaMalloc(&redbuf_, redbuf_n_ * sizeof(double)));
  }
  return redbuf_;
}

namespace {
void copy2d(DeviceExec& ex, int f, double* dev, int64_t x0, int64_t py, const Range& alloc, double* host, bool up,
            bool async, cudaStream_t st) {
  const int64_t nx = alloc.extent(0);
  const int64_t rows = alloc.volume() / std::max<int64_t>(1, nx);
  double* d = dev + (alloc.start(0) - x0);
  const size_t w = static_cast<size_t>(nx) * sizeof(double);
  (void)ex;
  (void)f;
  if (up)
    TCG_CK(cudaMemcpy2DAsync(d, static_cast<size_t>(py) * sizeof(double), host, w, w, static_cast<size_t>(rows),
                             cudaMemcpyHostToDevice, st));
  else
    TCG_CK(cudaMemcpy2DAsync(host, w, d, static_cast<size_t>(py) * sizeof(double), w, static_cast<size_t>(rows),
                             cudaMemcpyDeviceToHost, st));
  if (!async) TCG_CK(cudaStreamSynchronize(st));
}
}  // namespace

void DeviceExec::upload(int f, const double* host) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  mark_written(f, b->alloc);
  copy2d(*this, f, b->mem[b->cur], b->x0, b->alloc.dim() >= 2 ? b->py : b->py, b->alloc, const_cast<double*>(host),
         true, false, static_cast<cudaStream_t>(stream_));
}
void DeviceExec::download(int f, double* host) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  copy2d(*this, f, b->mem[b->cur], b->x0, b->py, b->alloc, host, false, false, static_cast<cudaStream_t>(stream_));
}
void DeviceExec::upload_async(int f, const double* host) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  mark_written(f, b->alloc);
  copy2d(*this, f, b->mem[b->cur], b->x0, b->py, b->alloc, const_cast<double*>(host), true, true,
         static_cast<cudaStream_t>(stream_));
}
void DeviceExec::download_async(int f, double* host) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  copy2d(*this, f, b->mem[b->cur], b->x0, b->py, b->alloc, host, false, true, static_cast<cudaStream_t>(stream_));
}

// Chain reductions to the host through a pinned buffer (a pageable
// destination would take the driver's staged copy path on every flush).
void DeviceExec::read_reductions(double* out, int n) {
  if (static_cast<size_t>(n) > red_n_) throw CudaError("read_reductions: more results than the reduction buffer holds");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  TCG_CK(cudaMemcpyAsync(red_host_, red_dev_, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, st));
  TCG_CK(cudaStreamSynchronize(st));
  std::memcpy(out, red_host_, sizeof(double) * static_cast<size_t>(n));
}

void DeviceExec::synchronize() { TCG_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_))); }

void* DeviceExec::take_event() {
  if (!ev_pool_.empty()) {
    void* e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  TCG_CK(cudaEventCreate(&e));
  return e;
}

void* DeviceExec::record() {
  void* e = take_event();
  TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e), static_cast<cudaStream_t>(stream_)));
  return e;
}

bool DeviceExec::elapsed_ms(void* a, void* b, float* ms) {
  if (cudaEventQuery(static_cast<cudaEvent_t>(b)) != cudaSuccess) return false;
  TCG_CK(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
  return true;
}

void DeviceExec::release(void* ev) { ev_pool_.push_back(ev); }

void DeviceExec::wait_event(void* ev) { TCG_CK(cudaEventSynchronize(static_cast<cudaEvent_t>(ev))); }

void DeviceExec::set_timing(bool on) {
  timing_ = on;
  double a, b;
  int64_t c, d;
  kernel_ms(&a, &c, &b, &d);  // drain and reset
}

void DeviceExec::kernel_ms(double* tiled_ms, int64_t* tiled_n, double* untiled_ms, int64_t* untiled_n) {
  TCG_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
  auto drain = [&](std::vector<std::pair<void*, void*>>& v, double* ms, int64_t* n) {
    double acc = 0;
    for (auto& p : v) {
      float f = 0;
      TCG_CK(cudaEventElapsedTime(&f, static_cast<cudaEvent_t>(p.first), static_cast<cudaEvent_t>(p.second)));
      acc += f;
      ev_pool_.push_back(p.first);
      ev_pool_.push_back(p.second);
    }
    *ms = acc;
    *n = static_cast<int64_t>(v.size());
    v.clear();
  };
  drain(ev_tiled_, tiled_ms, tiled_n);
  drain(ev_untiled_, untiled_ms, untiled_n);
}

void* DeviceExec::ensure_scratch(size_t bytes) {
  if (bytes > scratch_bytes_) {
    if (scratch_) {
      TCG_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
      TCG_CK(cudaFree(scratch_));
    }
    scratch_bytes_ = std::max(bytes, scratch_bytes_ * 2);
    TCG_CK(cudaMalloc(&scratch_, scratch_bytes_));
    scratch_hash_ = 0;
  }
  return scratch_;
}

// Chain reduction results (device) and their pinned host mirror: one double
// per reducing loop of a chain, grown to the chain's count (a flush may hold
// any number of reducing loops, runtime.cpp:94-151).
void DeviceExec::ensure_red(size_t n) {
  if (n <= red_n_) return;
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  TCG_CK(cudaStreamSynchronize(st));
  if (red_dev_) TCG_CK(cudaFree(red_dev_));
  if (red_host_) TCG_CK(cudaFreeHost(red_host_));
  red_dev_ = nullptr;
  red_host_ = nullptr;
  red_n_ = std::max<size_t>({n, red_n_ * 2, 64});
  TCG_CK(cudaMalloc(&red_dev_, sizeof(double) * red_n_));
  TCG_CK(cudaMallocHost(&red_host_, sizeof(double) * red_n_));
}

double* DeviceExec::ensure_partials(size_t n) {
  if (n > partials_n_) {
    if (partials_) {
      TCG_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
      TCG_CK(cudaFree(partials_));
    }
    partials_n_ = std::max(n, partials_n_ * 2);
    TCG_CK(cudaMalloc(&partials_, partials_n_ * sizeof(double)));
  }
  return partials_;
}

namespace {
// One untiled launch (a loop, or the fold of a reducing loop's partials).
struct ULaunchRec {
  ULaunch L;
  const void* fn;
  dim3 grid, block;
  unsigned smem;  // dynamic shared memory (none today)
  int64_t nblocks;
  int red;  // >= 0: followed by k_fold into red_dev_[red]
  bool ordered = false;  // Sum folded by k_ordered_sum over the captured contributions
  int64_t volume = 0;
};

uint64_t launch_key(const std::vector<ULaunchRec>& recs, int dim) {
  // Structure of the launch sequence; loop parameters excluded (they are
  // updated in place on a cached graph).
  uint64_t h = fnv_bytes(1469598103934665603ull, &dim, sizeof dim);
  for (const ULaunchRec& r : recs) {
    ULaunch L = r.L;
    std::memset(L.prm, 0, sizeof L.prm);
    h = fnv_bytes(h, &L, sizeof L);
    h = fnv_bytes(h, &r.fn, sizeof r.fn);
    h = fnv_bytes(h, &r.grid, sizeof r.grid);
    h = fnv_bytes(h, &r.block, sizeof r.block);
    h = fnv_bytes(h, &r.red, sizeof r.red);
    h = fnv_bytes(h, &r.smem, sizeof r.smem);
  }
  return h ^ recs.size();
}
}  // namespace

// A chain's untiled launch sequence as one CUDA graph (built explicitly,
// kernel nodes in loop order, k_fold after each reducing loop), replayed on
// later flushes of the same structure; changed loop parameters (CG's alpha /
// beta) are patched into the executable graph node by node.
struct DeviceExec::UGraph {
  uint64_t key = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> nodes;  // kernel node per record
  std::vector<ULaunch> launched;       // parameters the exec graph holds
  int64_t kernels = 0;
};

void DeviceExec::drop_graphs() {
  for (UGraph* g : graphs_) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
  }
  graphs_.clear();
}

void DeviceExec::run_untiled(const DevChain& ch, double* red_out) {
  ensure_red(static_cast<size_t>(ch.nred));
  mark_chain_writes(ch);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  void* scratch = ensure_scratch(chain_bytes(ch));
  const ChainDev cd = upload_chain(ch, scratch, st, &scratch_hash_);
  // Block shape and rows per thread: TCG_UNTILED_CFG="bx,by,run" (2D) /
  // TCG_UNTILED_CFG3 (3D) override the measured defaults (tuning).
  static const int3 ucfg = [] {
    // Measured on B200 (tools/ab_run.sh): 256x1 threads, 8 rows each (c2 -2%, c1 -4% vs 4 rows).
    int3 c{256, 1, 8};
    if (const char* e = std::getenv("TCG_UNTILED_CFG")) std::sscanf(e, "%d,%d,%d", &c.x, &c.y, &c.z);
    if (c.x * c.y > 256 || c.x * c.y < 32 || (c.z != 2 && c.z != 4 && c.z != 8)) c = int3{256, 1, 8};
    return c;
  }();
  // 3D: 64x2 threads; planes per thread chosen per loop (below) unless
  // TCG_UNTILED_CFG3="bx,by,run" fixes them.
  static const bool cfg3_env = std::getenv("TCG_UNTILED_CFG3") != nullptr;
  static const int3 ucfg3 = [] {
    int3 c{64, 2, 8};
    if (const char* e = std::getenv("TCG_UNTILED_CFG3")) std::sscanf(e, "%d,%d,%d", &c.x, &c.y, &c.z);
    if (c.x * c.y > 256 || c.x * c.y < 32 || (c.z != 4 && c.z != 8)) c = int3{64, 2, 8};
    return c;
  }();
  static const bool use_graphs = [] {
    const char* e = std::getenv("TCG_GRAPHS");
    return !e || std::atoi(e) != 0;
  }();
  static const bool prefetch = [] {
    const char* e = std::getenv("TCG_PREFETCH_L2");
    return !e || std::atoi(e) != 0;
  }();
  const int run_dim = ch.dim == 2 ? ucfg.z : ch.dim == 3 ? ucfg3.z : 4;

  // Lower every loop to a launch record.
  std::vector<ULaunchRec> recs;
  recs.reserve(ch.loops.size());
  int64_t max_blocks = 0;
  bool empty_red = false;
  for (const DevLoop& lp : ch.loops) {
    ULaunchRec R{};
    ULaunch& L = R.L;
    L.body = lp.body;
    L.nargs = lp.nargs;
    L.red_op = lp.red >= 0 ? lp.red_op : 0;
    L.has_red = lp.red >= 0;
    L.masked = ch.masked && L.has_red;
    for (int d = 0; d < 3; ++d) {
      L.mlo[d] = ch.mask[d][0];
      L.mhi[d] = ch.mask[d][1];
    }
    int64_t n[3];
    bool empty = false;
    for (int d = 0; d < 3; ++d) {
      L.lo[d] = lp.range[d][0];
      n[d] = lp.range[d][1] - lp.range[d][0];
      L.n[d] = n[d];
      if (n[d] <= 0) empty = true;
    }
    if (lp.nparams > kMaxParams) throw InvalidArgument("untiled executor: more than 16 scalar params in one loop");
    for (int i = 0; i < lp.nparams; ++i) L.prm[i] = ch.params[static_cast<size_t>(lp.param_off + i)];
    for (int a = 0; a < lp.nargs; ++a) {
      const DevView v = view(ch.dat_ids.empty() ? lp.args[a].dat : ch.dat_ids[static_cast<size_t>(lp.args[a].dat)], false);
      L.a[a] = UArg{v.base, v.x0, v.y0, v.z0, v.py, v.pz, lp.args[a].mode, lp.args[a].stencil};
#ifdef TCG_CHECKED
      for (int d = 0; d < 3; ++d) {
        L.alo[a][d] = v.alo[d];
        L.ahi[a][d] = v.ahi[d];
      }
#endif
    }
    L.st = cd.st;
    L.pf = prefetch ? 1 : 0;

    // Planes per thread in 3D: 8 for small stencils (c3's 7 points: the
    // z-neighbours of 8 planes stay in registers), 4 when the loop reads
    // more than 8 stencil points in total (c5's radius-2 RHS loops: 8 planes
    // took 246-255 registers, 11% occupancy; measured c5 277 -> 257 ms).
    int run2 = run_dim;
    if (ch.dim == 3 && !cfg3_env) {
      int pts = 0;
      for (int a = 0; a < lp.nargs; ++a)
        if (lp.args[a].mode != tcb::kWrite) pts += ch.st_npts[static_cast<size_t>(lp.args[a].stencil)];
      run2 = pts <= 8 ? 8 : 4;
    }
    for (int a = 0; a < lp.nargs; ++a) {
      if (lp.args[a].mode == tcb::kWrite) continue;
      L.rmask |= 1 << a;
      const int sid = lp.args[a].stencil;
      const int s0 = ch.st_start[static_cast<size_t>(sid)], np = ch.st_npts[static_cast<size_t>(sid)];
      for (int j = 0; j < np; ++j)
        for (int d = 0; d < 3; ++d) {
          L.rlo[d] = std::min(L.rlo[d], ch.st_pts[static_cast<size_t>(3 * (s0 + j) + d)]);
          L.rhi[d] = std::max(L.rhi[d], ch.st_pts[static_cast<size_t>(3 * (s0 + j) + d)]);
        }
    }
    // Rasterisation band (block_yz): measured on B200 (profiles/r5/sweeps.md) -- c5's radius-2 loops
    // 283.9 ms/step in hardware order, 275.1 with 64-block bands (-3%); c3's 7-point sweeps (8 planes
    // per thread, reach 1) lose 11% with any band, so only loops reaching >= 2 planes are banded.
    // TCG_UNTILED_BAND overrides (0 = hardware order everywhere).
    static const int band_env = [] {
      const char* e = std::getenv("TCG_UNTILED_BAND");
      return e && *e ? std::atoi(e) : -1;
    }();
    L.band = ch.dim == 3 ? (band_env >= 0 ? band_env : (L.rhi[2] - L.rlo[2] >= 4 ? 64 : 0)) : 0;
    if (ch.dim == 1) {
      R.block = dim3(256, 1, 1);
      R.grid = dim3(static_cast<unsigned>(std::max<int64_t>(1, (n[0] + 255) / 256)), 1, 1);
    } else if (ch.dim == 2) {
      R.block = dim3(static_cast<unsigned>(ucfg.x), static_cast<unsigned>(ucfg.y), 1);
      const int64_t ry = static_cast<int64_t>(ucfg.y) * run2;  // rows of y per block
      R.grid = dim3(static_cast<unsigned>(std::max<int64_t>(1, (n[0] + ucfg.x - 1) / ucfg.x)),
                    static_cast<unsigned>(std::max<int64_t>(1, (n[1] + ry - 1) / ry)), 1);
    } else {
      R.block = dim3(static_cast<unsigned>(ucfg3.x), static_cast<unsigned>(ucfg3.y), 1);
      R.grid = dim3(static_cast<unsigned>(std::max<int64_t>(1, (n[0] + ucfg3.x - 1) / ucfg3.x)),
                    static_cast<unsigned>(std::max<int64_t>(1, (n[1] + ucfg3.y - 1) / ucfg3.y)),
                    static_cast<unsigned>(std::max<int64_t>(1, (n[2] + run2 - 1) / run2)));
    }
    R.nblocks = static_cast<int64_t>(R.grid.x) * R.grid.y * R.grid.z;
    R.red = L.has_red ? lp.red : -1;
    if (L.has_red && red_workers_ > 0 && L.red_op == tcb::kSum && !empty) {
      if (L.masked) throw InvalidArgument("order-matched Sum: not available for rank-masked reductions");
      R.ordered = true;
      R.volume = n[0] * n[1] * n[2];
    }
    if (empty) {
      if (L.has_red) {
        // Empty reducing loop: the result is the identity.
        const double idv = red_identity(L.red_op);
        TCG_CK(cudaMemcpyAsync(red_dev_ + lp.red, &idv, 8, cudaMemcpyHostToDevice, st));
        TCG_CK(cudaStreamSynchronize(st));
        empty_red = true;
      }
      continue;
    }
    // One kernel instantiation per (dim, body): the body is a compile-time
    // constant inside the kernel.
    const bool known = tcb::dispatch(L.body, [&](auto tag) {
      constexpr int B = decltype(tag)::value;
      if (ch.dim == 1)
        R.fn = reinterpret_cast<const void*>(k_untiled<1, B>);
      else if (ch.dim == 2 && run2 == 2)
        R.fn = reinterpret_cast<const void*>(k_untiled2<B, 2>);
      else if (ch.dim == 2 && run2 == 8)
        R.fn = reinterpret_cast<const void*>(k_untiled2<B, 8>);
      else if (ch.dim == 2)
        R.fn = reinterpret_cast<const void*>(k_untiled2<B>);
      else if (run2 == 8)
        R.fn = reinterpret_cast<const void*>(k_untiled<3, B, 8>);
      else
        R.fn = reinterpret_cast<const void*>(k_untiled<3, B>);
    });
    if (!known) throw InvalidArgument("untiled executor: body " + std::to_string(L.body) + " not in the registry");
    if (L.has_red) max_blocks = std::max(max_blocks, R.nblocks);
    recs.push_back(R);
  }
  // Reduction partials: one buffer region per reducing loop (a graph replays
  // the loops back to back, so they must not share one).
  if (max_blocks > 0) {
    int64_t nr = 0;
    for (const ULaunchRec& r : recs) nr += r.red >= 0 ? 1 : 0;
    double* part = ensure_partials(static_cast<size_t>(max_blocks * nr));
    int64_t i = 0;
    for (ULaunchRec& r : recs)
      if (r.red >= 0) r.L.partials = part + (i++) * max_blocks;
  }

  // Order-matched Sums: one capture region per such loop, then the
  // reference's span partition and worker-order fold (k_ordered_sum).
  bool any_ordered = false;
  {
    size_t total = 0;
    for (const ULaunchRec& r : recs) total += r.ordered ? static_cast<size_t>(r.volume) : 0;
    if (total > 0) {
      any_ordered = true;
      if (total > capture_n_) {
        TCG_CK(cudaStreamSynchronize(st));
        if (capture_) TCG_CK(cudaFree(capture_));
        capture_n_ = total;
        TCG_CK(cudaMalloc(&capture_, capture_n_ * sizeof(double)));
      }
      if (!ord_part_) {
        TCG_CK(cudaMalloc(&ord_part_, sizeof(double) * 1024));
        TCG_CK(cudaMalloc(&ord_ticket_, sizeof(unsigned)));
        TCG_CK(cudaMemsetAsync(ord_ticket_, 0, sizeof(unsigned), st));
      }
      size_t off = 0;
      for (ULaunchRec& r : recs)
        if (r.ordered) {
          r.L.capture = capture_ + off;
          off += static_cast<size_t>(r.volume);
        }
    }
  }
  const bool graph_ok = use_graphs && !timing_ && !empty_red && !recs.empty() && !any_ordered;
  if (graph_ok) {
    const uint64_t key = launch_key(recs, ch.dim);
    UGraph* g = nullptr;
    for (UGraph* c : graphs_)
      if (c->key == key) g = c;
    if (!g) {
      if (graphs_.size() >= 64) {
        TCG_CK(cudaStreamSynchronize(st));
        UGraph* old = graphs_.front();
        cudaGraphExecDestroy(old->exec);
        cudaGraphDestroy(old->graph);
        delete old;
        graphs_.erase(graphs_.begin());
      }
      g = new UGraph;
      g->key = key;
      TCG_CK(cudaGraphCreate(&g->graph, 0));
      cudaGraphNode_t prev = nullptr;
      for (ULaunchRec& r : recs) {
        cudaKernelNodeParams kp{};
        void* args[] = {&r.L};
        kp.func = const_cast<void*>(r.fn);
        kp.gridDim = r.grid;
        kp.blockDim = r.block;
        kp.sharedMemBytes = r.smem;
        kp.kernelParams = args;
        cudaGraphNode_t node;
        TCG_CK(cudaGraphAddKernelNode(&node, g->graph, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
        g->nodes.push_back(node);
        g->launched.push_back(r.L);
        prev = node;
        ++g->kernels;
        if (r.red >= 0) {
          const double* pp = r.L.partials;
          int64_t nb = r.nblocks;
          int op = r.L.red_op;
          double* out = red_dev_ + r.red;
          void* fargs[] = {&pp, &nb, &op, &out};
          cudaKernelNodeParams fp{};
          fp.func = reinterpret_cast<void*>(k_fold);
          fp.gridDim = dim3(1);
          fp.blockDim = dim3(1024);
          fp.kernelParams = fargs;
          cudaGraphNode_t fnode;
          TCG_CK(cudaGraphAddKernelNode(&fnode, g->graph, &prev, 1, &fp));
          prev = fnode;
          ++g->kernels;
        }
      }
      TCG_CK(cudaGraphInstantiate(&g->exec, g->graph, 0));
      graphs_.push_back(g);
    } else {
      // Same structure: patch parameters that changed.
      for (size_t i = 0; i < recs.size(); ++i) {
        if (std::memcmp(recs[i].L.prm, g->launched[i].prm, sizeof recs[i].L.prm) == 0) continue;
        cudaKernelNodeParams kp{};
        void* args[] = {&recs[i].L};
        kp.func = const_cast<void*>(recs[i].fn);
        kp.gridDim = recs[i].grid;
        kp.blockDim = recs[i].block;
        kp.sharedMemBytes = recs[i].smem;
        kp.kernelParams = args;
        TCG_CK(cudaGraphExecKernelNodeSetParams(g->exec, g->nodes[i], &kp));
        g->launched[i] = recs[i].L;
      }
    }
    TCG_CK(cudaGraphLaunch(g->exec, st));
    launches_ += g->kernels;
  } else {
    for (ULaunchRec& r : recs) {
      void* e0 = nullptr;
      if (timing_) {
        e0 = take_event();
        TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e0), st));
      }
      void* args[] = {&r.L};
      TCG_CK(cudaLaunchKernel(r.fn, r.grid, r.block, args, r.smem, st));
      if (timing_) {
        void* e1 = take_event();
        TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e1), st));
        ev_untiled_.emplace_back(e0, e1);
      }
      ++launches_;
      if (r.ordered) {
        k_ordered_sum<<<red_workers_, 256, 0, st>>>(r.L.capture, r.volume, red_workers_, ord_part_, ord_ticket_,
                                                    red_dev_ + r.red);
        TCG_CK(cudaGetLastError());
        ++launches_;
      } else if (r.red >= 0) {
        k_fold<<<1, 1024, 0, st>>>(r.L.partials, r.nblocks, r.L.red_op, red_dev_ + r.red);
        TCG_CK(cudaGetLastError());
        ++launches_;
      }
    }
  }
  if (ch.nred > 0) {
    read_reductions(red_out, ch.nred);
  }
}

}  // namespace tcg
