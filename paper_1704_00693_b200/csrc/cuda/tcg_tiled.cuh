// Windowed tiled executor (included by tcg_exec.cu).
//
// One CTA = one "rank" of an overlapped decomposition of the chain's union
// bounds (construct_rank_plan, dist.cpp:191-390). Each CTA runs its rank plan:
// skewed slabs along the slowest ("stream") dimension, executed slab by slab
// and loop by loop (executor.cpp:232-244 order) on CTA-private shared-memory
// windows -- the device analogue of the reference's rank-private FieldTable.
//
// Windows are LINEAR: during slab t, dataset k's rows [lo_k(t), hi_k(t)) sit
// at window rows 0 .. hi-lo, so every stencil access is `centre + constant`.
// Per slab t:
//   wait for slab t's rows (bulk-copy engine, mbarrier)            -> bar
//   for each loop l: run its box of slab t on the windows            -> bar
//   evict rows [lo(t), lo(t+1)) of written datasets (bulk stores)   -> bar
//   compact: move rows [lo(t+1), hi(t)) to the window front          -> bar(s)
//   issue bulk loads of rows [hi(t), hi(t+1)) behind them
// Reads/writes inside a slab never touch HBM; each dataset crosses HBM once
// in (seeded datasets) and once out (written datasets) per chain, plus the
// overlapped halo columns.
#pragma once

namespace tiled {

// ---- bulk-copy engine (TMA, cp.async.bulk) --------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(m)),
      "r"(parity)
      : "memory");
}
// global -> shared, completion counted in bytes on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
// shared -> global, tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// a / b for 0 <= a < 2^22, b > 0 through the fast reciprocal: (a + 0.5) / b
// is never within float rounding of an integer, so truncation is exact.
__device__ __forceinline__ int fdivi(int a, int b) {
  return __float2int_rz(__fdividef(static_cast<float>(a) + 0.5f, static_cast<float>(b)));
}

// Maps (row, col) pairs of an nrows x per grid onto the CTA: flat index
// i = rr*per + c advanced by nth without dividing.
template <class F>
__device__ __forceinline__ void for_grid(int nrows, int per, int tid, int nth, F&& f) {
  if (nrows <= 0 || per <= 0) return;
  const int dr = nth / per, dc = nth - dr * per;
  int rr = tid / per, c = tid - rr * per;
  while (rr < nrows) {
    f(rr, c);
    rr += dr;
    c += dc;
    if (c >= per) {
      c -= per;
      ++rr;
    }
  }
}

// Per-dataset copy descriptor, built once per CTA so that a slab's loads,
// evictions and compaction are pure row arithmetic. Global addresses are
// base + element offset; window addresses are sbase + position.
struct DatCopy {
  const double* lsrc;  // load source base
  double* sdst;        // eviction destination base
  int64_t lofs;        // element offset of (load x0, load y0, stream row 0)
  int64_t sofs;        // element offset of (store x0, store y0, stream row 0)
  int64_t rp;          // stream-row pitch (elements)
  int64_t yp;          // y pitch (3D)
  int W, sbase;
  int lrlo, lrhi;      // loadable stream rows (allocation)
  int nvl, lny;        // 16-byte chunks per load row, y rows per load plane (3D)
  int lwin;            // window offset of the first loaded element in a row/plane
  int srlo, srhi;      // storable stream rows
  int snx, sny;        // stored columns (x), y rows per plane (3D)
  int swin;            // window offset of the first stored element in a row/plane
  int sx0;             // absolute x of the first stored column (bulk-store alignment)
  int mode;            // bit 1 load, bit 2 fast store, bit 4 generic store
};

struct Shared {
  DevCta C;
  int32_t lo[kMaxChainDats];  // stream row held at window row 0, per dataset
  DatCopy dc[kMaxChainDats];
  uint64_t mbar;              // bulk-load completion barrier (one phase per slab)
};

template <int DIM>
__device__ void make_copy(DatCopy& d, const DevTiledPlan& P, const DevCta& C, int k) {
  constexpr int s = DIM - 1;
  const DevView& v = P.src[k];
  const DevView& o = P.dst[k];
  const DevDat& dd = P.dats[k];
  d.W = C.W[k];
  d.sbase = C.sbase[k];
  d.mode = 0;
  if (!d.W) return;
  const int cx0 = C.col_lo[0], cy0 = C.col_lo[1], wx = C.col_hi[0] - cx0;
  d.rp = DIM == 1 ? 1 : (DIM == 2 ? v.py : v.pz);
  d.yp = v.py;
  d.lsrc = v.base;
  d.sdst = o.base;
  const int64_t row0 = DIM == 1 ? v.x0 : (DIM == 2 ? v.y0 : v.z0);  // stream origin of the layout
  if (dd.load) {
    d.lrlo = static_cast<int>(v.alo[s]);
    d.lrhi = static_cast<int>(v.ahi[s]);
    if (DIM == 1) {
      d.nvl = d.lny = 1;
      d.lwin = 0;
      d.lofs = -row0;
    } else {
      const int xa = max(cx0, static_cast<int>(v.x0)), xb = min(C.col_hi[0], static_cast<int>(v.x0 + v.py));
      int ya = 0, yb = 1;
      if (DIM == 3) {
        ya = max(cy0, static_cast<int>(v.alo[1]));
        yb = min(C.col_hi[1], static_cast<int>(v.ahi[1]));
      }
      d.nvl = max(0, (xb - xa) >> 1);
      d.lny = max(0, yb - ya);
      d.lwin = (DIM == 3 ? (ya - cy0) * wx : 0) + (xa - cx0);
      d.lofs = (xa - v.x0) + (DIM == 3 ? static_cast<int64_t>(ya - v.y0) * v.py : 0) - row0 * d.rp;
    }
    if (d.nvl > 0 && d.lny > 0) d.mode |= 1;
  }
  if (dd.written) {
    int xl = C.wb_lo[0], xh = C.wb_hi[0], yl = C.wb_lo[1], yh = C.wb_hi[1];
    int rlo = C.wb_lo[s], rhi = C.wb_hi[s];
    if (!dd.pingpong) {
      if (dd.nwbox != 1) {
        d.mode |= 4;  // several write boxes: generic eviction path
        return;
      }
      const int32_t* b = P.wboxes + dd.wbox_off * 6;
      rlo = max(rlo, b[2 * s]);
      rhi = min(rhi, b[2 * s + 1]);
      if (DIM >= 2) {
        xl = max(xl, b[0]);
        xh = min(xh, b[1]);
      }
      if (DIM == 3) {
        yl = max(yl, b[2]);
        yh = min(yh, b[3]);
      }
    }
    rlo = max(rlo, static_cast<int>(o.alo[s]));
    rhi = min(rhi, static_cast<int>(o.ahi[s]));
    d.srlo = rlo;
    d.srhi = rhi;
    if (DIM == 1) {
      d.snx = d.sny = 1;
      d.swin = 0;
      d.sx0 = 0;
      d.sofs = -row0;
    } else {
      xl = max(max(xl, cx0), static_cast<int>(o.alo[0]));
      xh = min(min(xh, C.col_hi[0]), static_cast<int>(o.ahi[0]));
      if (DIM == 3) {
        yl = max(max(yl, cy0), static_cast<int>(o.alo[1]));
        yh = min(min(yh, C.col_hi[1]), static_cast<int>(o.ahi[1]));
      } else {
        yl = 0;
        yh = 1;
      }
      d.snx = max(0, xh - xl);
      d.sny = max(0, yh - yl);
      d.sx0 = xl;
      d.swin = (DIM == 3 ? (yl - cy0) * wx : 0) + (xl - cx0);
      d.sofs = (xl - o.x0) + (DIM == 3 ? static_cast<int64_t>(yl - o.y0) * o.py : 0) - row0 * d.rp;
    }
    if (d.snx > 0 && d.sny > 0 && rlo < rhi) d.mode |= 2;
  }
}

// Loads stream rows [r0, r1) of a dataset whose window row 0 holds row `lo`.
// 2D/3D: one cp.async.bulk per row segment (window columns are even and
// 16-byte aligned in global and shared memory). 1D: plain loads.
template <int DIM>
__device__ __forceinline__ void load_rows(double* sm, const DatCopy& d, int lo, int r0, int r1, int stride, int wx,
                                          int tid, int nth, uint64_t* mbar) {
  r0 = max(r0, d.lrlo);
  r1 = min(r1, d.lrhi);
  if (r0 >= r1) return;
  double* win = sm + d.sbase + d.lwin + (r0 - lo) * stride;
  const double* g0 = d.lsrc + d.lofs + static_cast<int64_t>(r0) * d.rp;
  if (DIM == 1) {
    for (int rr = tid; rr < r1 - r0; rr += nth) win[rr] = g0[rr];
    return;
  }
  const unsigned bytes = static_cast<unsigned>(d.nvl) * 16u;
  const int ny = DIM == 3 ? d.lny : 1;
  const int nitems = (r1 - r0) * ny;
  for (int it = tid; it < nitems; it += nth) {
    int q = it, yy = 0;
    if (DIM == 3) {
      q = it / ny;
      yy = it - q * ny;
    }
    mbar_expect_tx(mbar, bytes);
    bulk_g2s(win + q * stride + yy * wx, g0 + static_cast<int64_t>(q) * d.rp + static_cast<int64_t>(yy) * d.yp, bytes,
             mbar);
  }
}

// Evicts stream rows [r0, r1): the 16-byte aligned middle of each row segment
// as one cp.async.bulk store, an odd first / last element by plain stores.
template <int DIM>
__device__ __forceinline__ void store_rows(const double* sm, const DatCopy& d, int lo, int r0, int r1, int stride,
                                           int wx, int tid, int nth) {
  r0 = max(r0, d.srlo);
  r1 = min(r1, d.srhi);
  if (r0 >= r1) return;
  const double* win = sm + d.sbase + d.swin + (r0 - lo) * stride;
  double* g0 = d.sdst + d.sofs + static_cast<int64_t>(r0) * d.rp;
  if (DIM == 1) {
    for (int rr = tid; rr < r1 - r0; rr += nth) g0[rr] = win[rr];
    return;
  }
  const int head = d.sx0 & 1, tail = (d.sx0 + d.snx) & 1;
  const int mid = d.snx - head - tail;
  const int ny = DIM == 3 ? d.sny : 1;
  const int nitems = (r1 - r0) * ny;
  for (int it = tid; it < nitems; it += nth) {
    int q = it, yy = 0;
    if (DIM == 3) {
      q = it / ny;
      yy = it - q * ny;
    }
    double* g = g0 + static_cast<int64_t>(q) * d.rp + static_cast<int64_t>(yy) * d.yp;
    const double* w = win + q * stride + yy * wx;
    if (head) g[0] = w[0];
    if (tail) g[d.snx - 1] = w[d.snx - 1];
    if (mid > 0) bulk_s2g(g + head, w + head, static_cast<unsigned>(mid) * 8u);
  }
}

// Generic eviction (in-place datasets written through several boxes).
template <int DIM>
__device__ void store_box(const double* sm, const DevCta& C, const DatCopy& d, const DevView& v, int lo, int r0,
                          int r1, int xl, int xh, int yl, int yh, int stride, int tid, int nth) {
  constexpr int s = DIM - 1;
  r0 = max(r0, static_cast<int>(v.alo[s]));
  r1 = min(r1, static_cast<int>(v.ahi[s]));
  if (r0 >= r1) return;
  const double* win = sm + d.sbase + (r0 - lo) * stride;
  if (DIM == 1) {
    for (int rr = tid; rr < r1 - r0; rr += nth) v.base[r0 + rr - v.x0] = win[rr];
    return;
  }
  const int cx0 = C.col_lo[0], wx = C.col_hi[0] - cx0;
  xl = max(max(xl, cx0), static_cast<int>(v.alo[0]));
  xh = min(min(xh, C.col_hi[0]), static_cast<int>(v.ahi[0]));
  if (xl >= xh) return;
  if (DIM == 3) {
    yl = max(max(yl, C.col_lo[1]), static_cast<int>(v.alo[1]));
    yh = min(min(yh, C.col_hi[1]), static_cast<int>(v.ahi[1]));
    if (yl >= yh) return;
  } else {
    yl = 0;
    yh = 1;
  }
  const int nx = xh - xl, ny = yh - yl;
  for_grid((r1 - r0) * ny, nx, tid, nth, [&](int rr, int c) {
    const int q = rr / ny, yy = rr - q * ny, r = r0 + q, x = xl + c, y = yl + yy;
    const int64_t gi = DIM == 2 ? static_cast<int64_t>(r - v.y0) * v.py + (x - v.x0)
                                : static_cast<int64_t>(r - v.z0) * v.pz + static_cast<int64_t>(y - v.y0) * v.py + (x - v.x0);
    v.base[gi] = win[q * stride + (DIM == 3 ? (y - C.col_lo[1]) * wx : 0) + (x - cx0)];
  });
}

// Global-to-global copy of a box (stream rows [r0, r1) x cols): ping-pong
// points a CTA owns that never pass through its windows.
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
  if (DIM == 3) {
    yl = max(yl, static_cast<int>(a.alo[1]));
    yh = min(yh, static_cast<int>(a.ahi[1]));
    if (yl >= yh) return;
  } else {
    yl = 0;
    yh = 1;
  }
  const int nx = xh - xl, ny = yh - yl;
  for_grid((r1 - r0) * ny, nx, tid, nth, [&](int rr, int c) {
    const int q = rr / ny, r = r0 + q, y = yl + (rr - q * ny), x = xl + c;
    if (DIM == 2)
      b.base[static_cast<int64_t>(r - b.y0) * b.py + (x - b.x0)] = a.base[static_cast<int64_t>(r - a.y0) * a.py + (x - a.x0)];
    else
      b.base[static_cast<int64_t>(r - b.z0) * b.pz + static_cast<int64_t>(y - b.y0) * b.py + (x - b.x0)] =
          a.base[static_cast<int64_t>(r - a.z0) * a.pz + static_cast<int64_t>(y - a.y0) * a.py + (x - a.x0)];
  });
}

// Accessor over the windows. Bodies are dispatched once per (slab, loop)
// with a compile-time id, so argument indices are constants and the
// per-argument positions live in registers (only the generic GEN_SUM body
// indexes them dynamically). A thread walks a column of the box: positions
// advance by one window row per point, reads are centre + constant.
// With DEFER, writes are held in registers until commit(): several points of
// one loop can then be evaluated with interleaved loads. Legal because a
// loop never reads another point's write (par_loop race rule,
// runtime.cpp:56-76); a centre read-modify-write reads before it writes.
template <int DIM, bool DEFER = false>
struct WAcc {
  double* sm;
  const DevLoop* lp;
  const Shared* S;
  DevStencils st;
  double* red;
  int wb[kMaxArgs];  // window position of (stream row 0, column origin) per argument
  int pb[kMaxArgs];  // centre position of the current point per argument
  double wv[DEFER ? kMaxArgs : 1];
  bool wf[DEFER ? kMaxArgs : 1];
  int px, py, pz, ctr, wx, pn, tid, nth;
  __device__ __forceinline__ void clear_pending() {
    if (DEFER) {
#pragma unroll
      for (int a = 0; a < kMaxArgs; ++a) wf[a] = false;
    }
  }
  __device__ __forceinline__ void commit() {
    if (DEFER) {
#pragma unroll
      for (int a = 0; a < kMaxArgs; ++a)
        if (wf[a]) sm[pb[a]] = wv[a];
    }
  }
  __device__ __forceinline__ int stride() const { return DIM == 1 ? 1 : (DIM == 2 ? wx : pn); }
  __device__ __forceinline__ void locate() {
    const int r = DIM == 1 ? px : (DIM == 2 ? py : pz);
#pragma unroll
    for (int a = 0; a < kMaxArgs; ++a) pb[a] = wb[a] + r * stride() + ctr;
  }
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int a = 0; a < kMaxArgs; ++a) pb[a] += stride();
  }
  __device__ __forceinline__ double* at(int a, int dx, int dy, int dz) const {
    if (DIM == 1) return sm + pb[a] + dx;
    if (DIM == 2) return sm + pb[a] + dy * wx + dx;
    return sm + pb[a] + dz * pn + dy * wx + dx;
  }
  __device__ __forceinline__ int64_t x() const { return px; }
  __device__ __forceinline__ int64_t y() const { return py; }
  __device__ __forceinline__ int64_t z() const { return pz; }
  __device__ __forceinline__ double read(int a, int dx, int dy, int dz) const { return *at(a, dx, dy, dz); }
  __device__ __forceinline__ void write(int a, double v) {
    if (DEFER) {
      wv[a] = v;
      wf[a] = true;
    } else {
      sm[pb[a]] = v;
    }
  }
  __device__ __forceinline__ void increment(int a, double v) { write(a, sm[pb[a]] + v); }
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

// NT threads per CTA, 512 / NT CTAs resident per SM (same register budget).
template <int DIM, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_tiled(const __grid_constant__ DevTiledPlan P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Shared S;
  constexpr int s = DIM - 1;
  const int tid = threadIdx.x, nth = blockDim.x;
  if (tid == 0) S.C = P.ctas[blockIdx.x];
  const int L = P.nloops;
  DevLoop* lsm = reinterpret_cast<DevLoop*>(sm + P.smem_doubles);
  int32_t* aw = reinterpret_cast<int32_t*>(lsm + L);               // [L][kMaxArgs] window bases
  double* red = reinterpret_cast<double*>(aw + L * kMaxArgs * 4);  // (keeps 16-byte ArgWin footprint)
  int32_t* bxs = reinterpret_cast<int32_t*>(red + P.nred * nth);  // boxes of the current slab [L][6]
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
  const int stride = DIM == 1 ? 1 : (DIM == 2 ? wx : pn);
  const int32_t* win = P.win + C.win_off;
  const int wbs0 = C.wb_lo[s], wbs1 = C.wb_hi[s];
  if (tid < nd) {
    make_copy<DIM>(S.dc[tid], P, C, tid);
    S.lo[tid] = win[2 * tid];
  }
  if (tid == 0) {
    mbar_init(&S.mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0;

  // Ping-pong points this CTA owns that never pass through its windows (rows
  // outside the window's span, padding columns outside its column box) are
  // unmodified by the chain: copy them old -> new buffer directly.
  for (int k = 0; k < nd; ++k) {
    if (!P.dats[k].pingpong) continue;
    int x0 = C.wb_lo[0], x1 = C.wb_hi[0], y0 = C.wb_lo[1], y1 = C.wb_hi[1];
    const int s0 = wbs0, s1 = wbs1;
    const int is0 = C.W[k] ? win[k * 2] : wbs1;
    const int is1 = C.W[k] ? win[(T * nd + k) * 2 + 1] : wbs1;
    const DevView& A = P.src[k];
    const DevView& B = P.dst[k];
    bool rest = true;
    if (DIM >= 2) {
      const int ix0 = C.col_lo[0], ix1 = C.col_hi[0];
      if (x0 < ix0) {
        g2g_copy<DIM>(A, B, s0, s1, x0, min(x1, ix0), y0, y1, tid, nth);
        x0 = ix0;
      }
      if (x1 > ix1 && x0 < x1) {
        g2g_copy<DIM>(A, B, s0, s1, max(x0, ix1), x1, y0, y1, tid, nth);
        x1 = ix1;
      }
      rest = x0 < x1;
    }
    if (DIM == 3 && rest) {
      const int iy0 = C.col_lo[1], iy1 = C.col_hi[1];
      if (y0 < iy0) {
        g2g_copy<DIM>(A, B, s0, s1, x0, x1, y0, min(y1, iy0), tid, nth);
        y0 = iy0;
      }
      if (y1 > iy1 && y0 < y1) {
        g2g_copy<DIM>(A, B, s0, s1, x0, x1, max(y0, iy1), y1, tid, nth);
        y1 = iy1;
      }
      rest = y0 < y1;
    }
    if (rest) {
      if (s0 < is0) g2g_copy<DIM>(A, B, s0, min(s1, is0), x0, x1, y0, y1, tid, nth);
      if (s1 > is1) g2g_copy<DIM>(A, B, max(s0, is1), s1, x0, x1, y0, y1, tid, nth);
    }
  }

  // Slab 0 rows [lo(0), hi(0)).
  for (int k = 0; k < nd; ++k)
    if (S.dc[k].mode & 1) load_rows<DIM>(sm, S.dc[k], win[2 * k], win[2 * k], win[2 * k + 1], stride, wx, tid, nth, &S.mbar);
  __syncthreads();
  if (tid == 0) mbar_arrive(&S.mbar);

  for (int t = 0; t < T; ++t) {
    const int32_t* w = win + t * nd * 2;
    const int32_t* wn = w + nd * 2;  // entry t+1 (entry T: lo = hi(T-1))
    mbar_wait(&S.mbar, phase);       // slab t rows have landed
    phase ^= 1u;
    for (int i = tid; i < L * 6; i += nth) bxs[i] = P.boxes[C.box_off + t * L * 6 + i];
    for (int i = tid; i < L * kMaxArgs; i += nth) {
      const int l = i / kMaxArgs, a = i - l * kMaxArgs;
      if (a < lsm[l].nargs) {
        const int k = lsm[l].args[a].dat;
        aw[i] = C.sbase[k] - S.lo[k] * stride;
      }
    }
    __syncthreads();

    for (int l = 0; l < L; ++l) {
      const int32_t* b = bxs + l * 6;
      const int bx0 = b[0], nx = b[1] - b[0];
      const int by0 = b[2], ny = b[3] - b[2];
      const int bz0 = b[4], nz = b[5] - b[4];
      if (nx <= 0 || ny <= 0 || nz <= 0) continue;
      const DevLoop& lp = lsm[l];
      const double* prm = P.params + lp.param_off;
      const int32_t* law = aw + l * kMaxArgs;
      const int nargs = lp.nargs;
      tcb::dispatch(lp.body, [&](auto tag) {
        constexpr int B = decltype(tag)::value;
        constexpr bool kDefer = B != tcb::kGenSum;  // GEN_SUM indexes args dynamically
        WAcc<DIM, kDefer> acc;
        acc.sm = sm;
        acc.lp = &lp;
        acc.S = &S;
        acc.st = P.stencils;
        acc.red = red;
        acc.wx = wx;
        acc.pn = pn;
        acc.tid = tid;
        acc.nth = nth;
#pragma unroll
        for (int a = 0; a < kMaxArgs; ++a) acc.wb[a] = a < nargs ? law[a] : 0;
        acc.clear_pending();
        if (DIM == 1) {
          for (int c = tid; c < nx; c += nth) {
            acc.px = bx0 + c;
            acc.py = acc.pz = 0;
            acc.ctr = 0;
            acc.locate();
            acc.clear_pending();
            tcb::run_body(B, acc, prm);
            acc.commit();
          }
        } else {
          // Column runs: a thread owns one column of the box and walks a
          // contiguous run of its rows, two rows per step (deferred writes let
          // the two points' loads interleave).
          const int ncol = DIM == 2 ? nx : nx * ny;
          const int nrow = DIM == 2 ? ny : nz;
          auto run_col = [&](int col, int a0, int a1) {
            if (DIM == 2) {
              acc.px = bx0 + col;
              acc.py = by0 + a0;
              acc.pz = 0;
              acc.ctr = acc.px - cx0;
            } else {
              const int q = fdivi(col, nx);
              acc.px = bx0 + (col - q * nx);
              acc.py = by0 + q;
              acc.pz = bz0 + a0;
              acc.ctr = (acc.py - cy0) * wx + (acc.px - cx0);
            }
            acc.locate();
            int rr = a0;
            if (kDefer) {
              WAcc<DIM, kDefer> acc2 = acc;
              acc2.advance();
              if (DIM == 2)
                ++acc2.py;
              else
                ++acc2.pz;
              for (; rr + 1 < a1; rr += 2) {
                acc.clear_pending();
                acc2.clear_pending();
                tcb::run_body(B, acc, prm);
                tcb::run_body(B, acc2, prm);
                acc.commit();
                acc2.commit();
                acc.advance();
                acc.advance();
                acc2.advance();
                acc2.advance();
                if (DIM == 2) {
                  acc.py += 2;
                  acc2.py += 2;
                } else {
                  acc.pz += 2;
                  acc2.pz += 2;
                }
              }
            }
            for (; rr < a1; ++rr) {
              acc.clear_pending();
              tcb::run_body(B, acc, prm);
              acc.commit();
              acc.advance();
              if (DIM == 2)
                ++acc.py;
              else
                ++acc.pz;
            }
          };
          if (ncol >= nth) {
            for (int col = tid; col < ncol; col += nth) run_col(col, 0, nrow);
          } else {
            const int ng = fdivi(nth, ncol), g = fdivi(tid, ncol), col = tid - g * ncol;
            const int chunk = fdivi(nrow + ng - 1, ng);
            const int a0 = g * chunk, a1 = min(nrow, a0 + chunk);
            if (g < ng && a0 < a1) run_col(col, a0, a1);
          }
        }
      });
      __syncthreads();
    }

    // Evict rows [lo(t), lo(t+1)) of written datasets.
    if (DIM >= 2) {
      fence_proxy_async();  // generic-proxy window writes -> bulk-copy reads
      __syncthreads();
    }
    for (int k = 0; k < nd; ++k) {
      const DatCopy& d = S.dc[k];
      if (d.mode & 2) {
        store_rows<DIM>(sm, d, S.lo[k], w[2 * k], wn[2 * k], stride, wx, tid, nth);
      } else if (d.mode & 4) {
        const int r0 = max(w[2 * k], wbs0), r1 = min(wn[2 * k], wbs1);
        for (int i = 0; i < P.dats[k].nwbox && r0 < r1; ++i) {
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
          store_box<DIM>(sm, C, d, P.dst[k], S.lo[k], q0, q1, xl, xh, yl, yh, stride, tid, nth);
        }
      }
    }
    if (DIM >= 2) {
      bulk_commit();
      bulk_wait_read0();  // evicted rows have been read out of the windows
    }
    if (t + 1 == T) break;

    // Compaction: rows [lo(t+1), hi(t)) move to the window front, in chunks
    // of `delta` rows so source and destination never overlap within a pass.
    __syncthreads();
    int passes = 0;
    for (int k = 0; k < nd; ++k) {
      if (!C.W[k]) continue;
      const int delta = wn[2 * k] - S.lo[k], keep = w[2 * k + 1] - wn[2 * k];
      if (delta > 0 && keep > 0) passes = max(passes, (keep + delta - 1) / delta);
    }
    for (int p = 0; p < passes; ++p) {
      for (int k = 0; k < nd; ++k) {
        if (!C.W[k]) continue;
        const int delta = wn[2 * k] - S.lo[k], keep = w[2 * k + 1] - wn[2 * k];
        if (delta <= 0 || keep <= 0) continue;
        const int r_a = p * delta, r_b = min(keep, (p + 1) * delta);  // destination rows of this pass
        if (r_a >= r_b) continue;
        double* base = sm + C.sbase[k];
        const int n = (r_b - r_a) * stride;  // even: stride is even in 2D/3D
        if (DIM == 1) {
          for (int i = tid; i < n; i += nth) base[r_a + i] = base[r_a + delta + i];
        } else {
          double2* dst = reinterpret_cast<double2*>(base + r_a * stride);
          const double2* src = reinterpret_cast<const double2*>(base + (r_a + delta) * stride);
          for (int i = tid; i < n / 2; i += nth) dst[i] = src[i];
        }
      }
      __syncthreads();
    }
    if (tid < nd && C.W[tid]) S.lo[tid] = wn[2 * tid];
    if (DIM >= 2) fence_proxy_async();  // generic window accesses before async-proxy refills
    __syncthreads();
    // Refill: rows [hi(t), hi(t+1)) behind the retained ones.
    for (int k = 0; k < nd; ++k)
      if (S.dc[k].mode & 1) load_rows<DIM>(sm, S.dc[k], S.lo[k], w[2 * k + 1], wn[2 * k + 1], stride, wx, tid, nth, &S.mbar);
    __syncthreads();
    if (tid == 0) mbar_arrive(&S.mbar);
  }
  if (DIM >= 2) bulk_wait0();
  __syncthreads();

  for (int r = 0; r < P.nred; ++r) {
    const double v = block_reduce(red[r * nth + tid], P.red_op[r]);
    if (tid == 0) P.red_partials[r * P.nctas + blockIdx.x] = v;
    __syncthreads();
  }
}

}  // namespace tiled
