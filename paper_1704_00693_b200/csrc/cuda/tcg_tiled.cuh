// Windowed tiled executor (included by tcg_exec.cu).
//
// One CTA = one "rank" of an overlapped decomposition of the chain's union
// bounds (construct_rank_plan, dist.cpp:191-390). Each CTA runs its rank plan:
// skewed slabs along the slowest ("stream") dimension, executed slab by slab
// and loop by loop (executor.cpp:232-244 order) on CTA-private shared-memory
// windows -- the device analogue of the reference's rank-private FieldTable.
//
// Per slab t:  async-load rows [hi(t-1), hi(t)) of every seeded dataset
//              (cp.async 16 B, all datasets in flight at once) -> wait -> bar
//              for each loop l: run its box of slab t on the window -> bar
//              evict rows [lo(t), lo(t+1)) of written datasets to HBM -> bar
// Reads/writes inside a slab never touch HBM; each dataset crosses HBM once in
// (seeded datasets) and once out (written datasets) per chain, plus the
// overlapped halo columns.
#pragma once

namespace tiled {

__device__ __forceinline__ int pmod(int r, int w) {
  const int m = r % w;
  return m < 0 ? m + w : m;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Maps (row, col) pairs of an nrows x per grid onto the CTA without a
// division per element: if a row is narrower than the CTA, several rows are
// covered per pass.
template <class F>
__device__ __forceinline__ void for_grid(int nrows, int per, int tid, int nth, F&& f) {
  if (nrows <= 0 || per <= 0) return;
  if (per >= nth) {
    for (int rr = 0; rr < nrows; ++rr)
      for (int c = tid; c < per; c += nth) f(rr, c);
  } else {
    const int rstep = nth / per;
    const int rid = tid / per;
    const int c = tid - rid * per;
    if (rid < rstep)
      for (int rr = rid; rr < nrows; rr += rstep) f(rr, c);
  }
}

struct Shared {
  DevCta C;
  int32_t wso[kMaxChainDats];  // slot(r) = r + wso (wrapped by W) during the current slab
};

// Per-(loop, arg) window descriptor, refreshed each slab: {sbase, slot offset, W}.
struct ArgWin {
  int32_t sb, so, W, pad;
};

template <int DIM>
struct WAcc {
  double* sm;
  const ArgWin* aw;
  const DevLoop* lp;
  const Shared* S;
  DevStencils st;
  double* red;
  int px, py, pz, ctr, wx, pn, tid, nth;
  __device__ __forceinline__ int slot(int a, int r) const {
    const int s = r + aw[a].so;
    return s >= aw[a].W ? s - aw[a].W : s;
  }
  __device__ __forceinline__ double* at(int a, int dx, int dy, int dz) const {
    if (DIM == 1) return sm + aw[a].sb + slot(a, px + dx);
    if (DIM == 2) return sm + aw[a].sb + slot(a, py + dy) * wx + ctr + dx;
    return sm + aw[a].sb + slot(a, pz + dz) * pn + ctr + dy * wx + dx;
  }
  __device__ __forceinline__ int64_t x() const { return px; }
  __device__ __forceinline__ int64_t y() const { return py; }
  __device__ __forceinline__ int64_t z() const { return pz; }
  __device__ __forceinline__ double read(int a, int dx, int dy, int dz) const { return *at(a, dx, dy, dz); }
  __device__ __forceinline__ void write(int a, double v) const { *at(a, 0, 0, 0) = v; }
  __device__ __forceinline__ void increment(int a, double v) const {
    double* p = at(a, 0, 0, 0);
    *p = *p + v;
  }
  __device__ __forceinline__ void contribute(double v) const {
    const DevCta& C = S->C;
    if (px < C.own_lo[0] || px >= C.own_hi[0]) return;
    if (DIM >= 2 && (py < C.own_lo[1] || py >= C.own_hi[1])) return;
    if (DIM == 3 && (pz < C.own_lo[2] || pz >= C.own_hi[2])) return;
    double& r = red[lp->red * nth + tid];
    r = red_combine(lp->red_op, r, v);
  }
  __device__ __forceinline__ int nargs() const { return lp->nargs; }
  __device__ __forceinline__ int mode(int a) const { return lp->args[a].mode; }
  __device__ __forceinline__ int npts(int a) const { return st.npts[lp->args[a].stencil]; }
  __device__ __forceinline__ int pt(int a, int j, int d) const {
    return st.pts[3 * (st.start[lp->args[a].stencil] + j) + d];
  }
  __device__ __forceinline__ bool reduces() const { return lp->red >= 0; }
};

// Issues async loads of window rows [r0, r1) of chain dataset k.
template <int DIM>
__device__ void win_load(double* sm, const DevCta& C, int k, const DevView& v, int r0, int r1, int tid, int nth) {
  constexpr int s = DIM - 1;
  r0 = max(r0, static_cast<int>(v.alo[s]));
  r1 = min(r1, static_cast<int>(v.ahi[s]));
  if (r0 >= r1) return;
  const int W = C.W[k];
  double* win = sm + C.sbase[k];
  if (DIM == 1) {
    for (int r = r0 + tid; r < r1; r += nth) cp_async8(win + pmod(r, W), v.base + (r - v.x0));
    return;
  }
  const int cx0 = C.col_lo[0], wx = C.col_hi[0] - C.col_lo[0];
  const int xa = max(cx0, static_cast<int>(v.x0));
  const int xb = min(C.col_hi[0], static_cast<int>(v.x0 + v.py));
  if (xa >= xb) return;
  const int nv = (xb - xa) >> 1;  // 16-byte chunks per row (xa, xb even)
  if (DIM == 2) {
    const double* g0 = v.base + (xa - v.x0);
    double* s0 = win + (xa - cx0);
    for_grid(r1 - r0, nv, tid, nth, [&](int rr, int c) {
      const int r = r0 + rr;
      cp_async16(s0 + pmod(r, W) * wx + 2 * c, g0 + static_cast<int64_t>(r - v.y0) * v.py + 2 * c);
    });
  } else {
    const int cy0 = C.col_lo[1];
    const int ya = max(cy0, static_cast<int>(v.alo[1])), yb = min(C.col_hi[1], static_cast<int>(v.ahi[1]));
    if (ya >= yb) return;
    const int pn = wx * (C.col_hi[1] - cy0);
    const int ny = yb - ya;
    const double* g0 = v.base + (xa - v.x0);
    double* s0 = win + (xa - cx0);
    // rows of the grid = (plane, y) pairs
    for_grid((r1 - r0) * ny, nv, tid, nth, [&](int rr, int c) {
      const int q = rr / ny, r = r0 + q, y = ya + (rr - q * ny);
      cp_async16(s0 + pmod(r, W) * pn + (y - cy0) * wx + 2 * c,
                 g0 + static_cast<int64_t>(r - v.z0) * v.pz + static_cast<int64_t>(y - v.y0) * v.py + 2 * c);
    });
  }
}

// Stores window rows [r0, r1) x columns [xl, xh) x [yl, yh) of dataset k.
template <int DIM>
__device__ void win_store(const double* sm, const DevCta& C, int k, const DevView& v, int r0, int r1, int xl, int xh,
                          int yl, int yh, int tid, int nth) {
  constexpr int s = DIM - 1;
  r0 = max(r0, static_cast<int>(v.alo[s]));
  r1 = min(r1, static_cast<int>(v.ahi[s]));
  if (r0 >= r1) return;
  const int W = C.W[k];
  const double* win = sm + C.sbase[k];
  if (DIM == 1) {
    for (int r = r0 + tid; r < r1; r += nth) v.base[r - v.x0] = win[pmod(r, W)];
    return;
  }
  xl = max(max(xl, C.col_lo[0]), static_cast<int>(v.alo[0]));
  xh = min(min(xh, C.col_hi[0]), static_cast<int>(v.ahi[0]));
  if (xl >= xh) return;
  const int cx0 = C.col_lo[0], wx = C.col_hi[0] - C.col_lo[0], nx = xh - xl;
  if (DIM == 2) {
    for_grid(r1 - r0, nx, tid, nth, [&](int rr, int c) {
      const int r = r0 + rr, x = xl + c;
      v.base[static_cast<int64_t>(r - v.y0) * v.py + (x - v.x0)] = win[pmod(r, W) * wx + (x - cx0)];
    });
  } else {
    yl = max(max(yl, C.col_lo[1]), static_cast<int>(v.alo[1]));
    yh = min(min(yh, C.col_hi[1]), static_cast<int>(v.ahi[1]));
    if (yl >= yh) return;
    const int cy0 = C.col_lo[1], pn = wx * (C.col_hi[1] - cy0), ny = yh - yl;
    for_grid((r1 - r0) * ny, nx, tid, nth, [&](int rr, int c) {
      const int q = rr / ny, r = r0 + q, y = yl + (rr - q * ny), x = xl + c;
      v.base[static_cast<int64_t>(r - v.z0) * v.pz + static_cast<int64_t>(y - v.y0) * v.py + (x - v.x0)] =
          win[pmod(r, W) * pn + (y - cy0) * wx + (x - cx0)];
    });
  }
}

// Global-to-global copy of rows [r0, r1) x cols: ping-pong rows a CTA owns
// but never holds in a window.
template <int DIM>
__device__ void g2g_copy(const DevView& a, const DevView& b, int r0, int r1, int xl, int xh, int yl, int yh, int tid,
                         int nth) {
  constexpr int s = DIM - 1;
  r0 = max(r0, static_cast<int>(a.alo[s]));
  r1 = min(r1, static_cast<int>(a.ahi[s]));
  if (r0 >= r1) return;
  if (DIM == 1) {
    for (int r = r0 + tid; r < r1; r += nth) b.base[r - b.x0] = a.base[r - a.x0];
    return;
  }
  xl = max(xl, static_cast<int>(a.alo[0]));
  xh = min(xh, static_cast<int>(a.ahi[0]));
  if (xl >= xh) return;
  const int nx = xh - xl;
  if (DIM == 2) {
    for_grid(r1 - r0, nx, tid, nth, [&](int rr, int c) {
      const int r = r0 + rr, x = xl + c;
      b.base[static_cast<int64_t>(r - b.y0) * b.py + (x - b.x0)] = a.base[static_cast<int64_t>(r - a.y0) * a.py + (x - a.x0)];
    });
  } else {
    yl = max(yl, static_cast<int>(a.alo[1]));
    yh = min(yh, static_cast<int>(a.ahi[1]));
    if (yl >= yh) return;
    const int ny = yh - yl;
    for_grid((r1 - r0) * ny, nx, tid, nth, [&](int rr, int c) {
      const int q = rr / ny, r = r0 + q, y = yl + (rr - q * ny), x = xl + c;
      b.base[static_cast<int64_t>(r - b.z0) * b.pz + static_cast<int64_t>(y - b.y0) * b.py + (x - b.x0)] =
          a.base[static_cast<int64_t>(r - a.z0) * a.pz + static_cast<int64_t>(y - a.y0) * a.py + (x - a.x0)];
    });
  }
}

template <int DIM>
__global__ void __launch_bounds__(kTiledThreads, 1) k_tiled(const __grid_constant__ DevTiledPlan P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Shared S;
  constexpr int s = DIM - 1;
  const int tid = threadIdx.x, nth = blockDim.x;
  if (tid == 0) S.C = P.ctas[blockIdx.x];
  const int L = P.nloops;
  DevLoop* lsm = reinterpret_cast<DevLoop*>(sm + P.smem_doubles);
  ArgWin* aw = reinterpret_cast<ArgWin*>(lsm + L);
  double* red = reinterpret_cast<double*>(aw + L * kMaxArgs);
  {
    const int nwords = L * static_cast<int>(sizeof(DevLoop) / 4);
    const int* src = reinterpret_cast<const int*>(P.loops);
    int* dst = reinterpret_cast<int*>(lsm);
    for (int i = tid; i < nwords; i += nth) dst[i] = src[i];
    for (int r = 0; r < P.nred; ++r) red[r * nth + tid] = red_identity(P.red_op[r]);
  }
  __syncthreads();
  const DevCta& C = S.C;
  const int nd = P.ndat, T = C.ntiles;
  const int cx0 = C.col_lo[0], cy0 = C.col_lo[1];
  const int wx = C.col_hi[0] - cx0;
  const int pn = wx * (C.col_hi[1] - cy0);
  const int32_t* win = P.win + C.win_off;
  const int wbs0 = C.wb_lo[s], wbs1 = C.wb_hi[s];

  // Ping-pong rows this CTA owns outside its windows.
  for (int k = 0; k < nd; ++k) {
    if (!P.dats[k].pingpong) continue;
    const int first = C.W[k] ? win[k * 2] : wbs1;
    const int last = C.W[k] ? win[(T * nd + k) * 2 + 1] : wbs1;
    g2g_copy<DIM>(P.src[k], P.dst[k], wbs0, min(first, wbs1), C.wb_lo[0], C.wb_hi[0], C.wb_lo[1], C.wb_hi[1], tid, nth);
    if (C.W[k]) g2g_copy<DIM>(P.src[k], P.dst[k], max(last, wbs0), wbs1, C.wb_lo[0], C.wb_hi[0], C.wb_lo[1], C.wb_hi[1], tid, nth);
  }

  for (int t = 0; t < T; ++t) {
    const int32_t* w = win + t * nd * 2;
    for (int k = 0; k < nd; ++k) {
      if (!C.W[k] || !P.dats[k].load) continue;
      const int r0 = t == 0 ? w[2 * k] : w[2 * k - 2 * nd + 1];
      win_load<DIM>(sm, C, k, P.src[k], r0, w[2 * k + 1], tid, nth);
    }
    if (tid < nd && C.W[tid]) S.wso[tid] = pmod(w[2 * tid], C.W[tid]) - w[2 * tid];
    cp_async_wait_all();
    __syncthreads();
    // Per-(loop, arg) window table for this slab.
    for (int i = tid; i < L * kMaxArgs; i += nth) {
      const int l = i / kMaxArgs, a = i - l * kMaxArgs;
      if (a < lsm[l].nargs) {
        const int k = lsm[l].args[a].dat;
        aw[i] = ArgWin{C.sbase[k], S.wso[k], C.W[k] > 0 ? C.W[k] : 1, 0};
      }
    }
    __syncthreads();

    for (int l = 0; l < L; ++l) {
      const int32_t* b = P.boxes + C.box_off + (t * L + l) * 6;
      const int bx0 = b[0], nx = b[1] - b[0];
      const int by0 = b[2], ny = b[3] - b[2];
      const int bz0 = b[4], nz = b[5] - b[4];
      if (nx <= 0 || ny <= 0 || nz <= 0) continue;
      const DevLoop& lp = lsm[l];
      WAcc<DIM> acc;
      acc.sm = sm;
      acc.aw = aw + l * kMaxArgs;
      acc.lp = &lp;
      acc.S = &S;
      acc.st = P.stencils;
      acc.red = red;
      acc.wx = wx;
      acc.pn = pn;
      acc.tid = tid;
      acc.nth = nth;
      const double* prm = P.params + lp.param_off;
      const int body = lp.body;
      for_grid(ny * nz, nx, tid, nth, [&](int rr, int c) {
        acc.px = bx0 + c;
        if (DIM == 1) {
          acc.py = acc.pz = 0;
          acc.ctr = 0;
        } else if (DIM == 2) {
          acc.py = by0 + rr;
          acc.pz = 0;
          acc.ctr = acc.px - cx0;
        } else {
          const int q = rr / ny;
          acc.pz = bz0 + q;
          acc.py = by0 + (rr - q * ny);
          acc.ctr = (acc.py - cy0) * wx + (acc.px - cx0);
        }
        tcb::run_body(body, acc, prm);
      });
      __syncthreads();
    }

    // Evict rows [lo(t), lo(t+1)) of written datasets to global memory.
    const int32_t* wn = w + nd * 2;
    for (int k = 0; k < nd; ++k) {
      if (!C.W[k] || !P.dats[k].written) continue;
      const int r0 = max(w[2 * k], wbs0), r1 = min(wn[2 * k], wbs1);
      if (r0 >= r1) continue;
      if (P.dats[k].pingpong) {
        win_store<DIM>(sm, C, k, P.dst[k], r0, r1, C.wb_lo[0], C.wb_hi[0], C.wb_lo[1], C.wb_hi[1], tid, nth);
      } else {
        for (int i = 0; i < P.dats[k].nwbox; ++i) {
          const int32_t* bb = P.wboxes + (P.dats[k].wbox_off + i) * 6;
          const int q0 = max(r0, bb[2 * s]), q1 = min(r1, bb[2 * s + 1]);
          if (q0 >= q1) continue;
          int xl = 0, xh = 1, yl = 0, yh = 1;
          if (DIM >= 2) {
            xl = max(bb[0], C.wb_lo[0]);
            xh = min(bb[1], C.wb_hi[0]);
          }
          if (DIM == 3) {
            yl = max(bb[2], C.wb_lo[1]);
            yh = min(bb[3], C.wb_hi[1]);
          }
          win_store<DIM>(sm, C, k, P.dst[k], q0, q1, xl, xh, yl, yh, tid, nth);
        }
      }
    }
    __syncthreads();
  }

  for (int r = 0; r < P.nred; ++r) {
    const double v = block_reduce(red[r * nth + tid], P.red_op[r]);
    if (tid == 0) P.red_partials[r * P.nctas + blockIdx.x] = v;
    __syncthreads();
  }
}

}  // namespace tiled
