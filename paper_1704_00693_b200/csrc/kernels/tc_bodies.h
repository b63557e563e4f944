// Per-point kernel bodies ("user kernels") of the B200 stencil-chain executor.
//
// The reference dispatches a per-point std::function<void(KernelCtx&)>
// (proj/core/include/tilechain/kernel_ctx.hpp:15-19) through a checked accessor
// (kernel_ctx.hpp:58-89). Host closures cannot run on the device, so this
// project replaces them with a *registry of bodies*: each body is written once
// as a template over an accessor type and compiled twice -- by nvcc into the
// device executors (untiled, windowed-tiled) and by g++ into the CPU oracle
// drivers (oracle/). One source means one expression tree on both sides, which
// together with `-fmad=false` (device) and no FMA contraction (host) gives
// bit-identical per-point arithmetic.
//
// Accessor contract (mirrors KernelCtx):
//   double read(int arg, int dx, int dy, int dz)   -- stencil read
//   void   write(int arg, double v)                 -- centre write
//   void   increment(int arg, double v)             -- centre +=
//   void   contribute(double v)                     -- reduction (masked)
//   long   x(), y(), z()                            -- iteration point
//   int    nargs(), mode(arg), npts(arg), pt(arg, j, d), reduces()
//                                                   -- introspection (gen body)
// A body id not in the registry is an error at enqueue time: there is no
// CPU fallback.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define TC_HD __host__ __device__ __forceinline__
#else
#define TC_HD inline
#endif

namespace tcb {

// AccessMode numbering follows proj/core/include/tilechain/types.hpp:185.
enum Mode : int { kRead = 0, kWrite = 1, kReadWrite = 2, kIncrement = 3 };
// ReduceOp numbering follows types.hpp:270.
enum RedOp : int { kSum = 0, kMin = 1, kMax = 2 };

enum Body : int32_t {
  // Generic contracting dyadic combination of every declared read, the kernel
  // shape of the reference's random-chain generator
  // (proj/tests/support/chain_gen.cpp:168-196). Params: [0] = scale.
  kGenSum = 1,
  // Reference app kernels (proj/core/src/apps.cpp:43-57, :142-254).
  kJacobiStencil = 2,
  kJacobiCopy = 3,
  kMhEos = 10,
  kMhBcX = 11,
  kMhBcY = 12,
  kMhAccelX = 13,
  kMhAccelY = 14,
  kMhFluxX = 15,
  kMhFluxY = 16,
  kMhAdvectRho = 17,
  kMhAdvectE = 18,
  kMhSmooth = 19,
  kMhBlend = 20,
  kMhMonitor = 21,
  // Reference unit-test kernels (test_executor.cpp:29-33, test_dist.cpp:27-60).
  kSmooth2D = 30,   // 0.5*c + 0.125*(W+E+S+N)
  kSmooth1D = 31,   // 0.5*c + 0.25*(W+E)
  kConsume1D = 32,  // 0.25*(W+c+E)
  kCopy = 33,       // write(1, read(0))
  kSumRead = 34,    // contribute(read(0))
  kIota = 35,       // write(0, x)                       test_oracle.cpp:80-83
  kNbrSum = 36,     // write(1, read(0,-1) + read(0,+1))  test_oracle.cpp:86-90
  // BASELINE config c1: 2D heat chain.
  kHeatLap = 100,   // v = u + 0.1*lap(u)
  kHeatCopy = 101,  // u = v
  // BASELINE config c2: 2D hydro-like chain. 200 + 2*stencil_kind + has_r3.
  kHydroBase = 200,  // .. 209
  kHydroCfl = 220,   // min-reduction closing each step
  // BASELINE config c3: 3D 7-point Jacobi.
  kJacobi3D = 300,
  // BASELINE config c4: CG on a variable-coefficient 5-point operator.
  kCgPUpdate = 400,  // p = r + beta*p         params [beta]
  kCgMatvec = 401,   // q = A p ; sum p*q
  kCgXUpdate = 402,  // x = x + alpha*p        params [alpha]
  kCgRUpdate = 403,  // r = r - alpha*q ; sum r*r   params [alpha]
  kCgDot = 404,      // sum r*r
  // BASELINE config c5: 3D compressible NS (Taylor-Green), see tc_ns.h.
  kNsFirst = 500,
  kNsLast = 539,
};

// ---------------------------------------------------------------------------
// Generic body (chain_gen.cpp:168-196): s = sum of every Read-arg stencil point
// in declaration order; out = s*scale + 1/16; write / blend / increment the
// last arg; contribute(out) when the loop reduces.
template <class A>
TC_HD void gen_sum(A& a, const double* p) {
  double s = 0;
  const int n = a.nargs();
  for (int i = 0; i < n; ++i) {
    if (a.mode(i) != kRead) continue;
    const int np = a.npts(i);
    for (int j = 0; j < np; ++j) s += a.read(i, a.pt(i, j, 0), a.pt(i, j, 1), a.pt(i, j, 2));
  }
  const double out = s * p[0] + 0.0625;
  const int wi = n - 1;
  const int wm = a.mode(wi);
  if (wm == kWrite)
    a.write(wi, out);
  else if (wm == kReadWrite)
    a.write(wi, 0.5 * a.read(wi, 0, 0, 0) + 0.5 * out);
  else
    a.increment(wi, 0.25 * out);
  if (a.reduces()) a.contribute(out);
}

// ---------------------------------------------------------------------------
// c2 hydro loop bodies. Arg 0 = r1 read through the cycling stencil, arg 1 =
// r2 (point), [arg 2 = r3 (point)], last arg = written dat.
//   out = 0.25 + 0.5*mean(r1 over stencil) + 0.125*r2 + 0.125*(r1c*r2)
//   out = 0.25 + 0.5*mean(...) + 0.0625*r2 + 0.0625*r3 + 0.125*(r1c*r2)
// Stencil kinds: 0 point, 1 star5, 2 box9, 3 one-sided {(0,0),(1,0),(0,1)},
// 4 radius-2 star.
template <class A>
TC_HD double hydro_stencil_sum(A& a, int kind) {
  if (kind == 0) return a.read(0, 0, 0, 0);
  if (kind == 1)
    return (((a.read(0, 0, 0, 0) + a.read(0, 1, 0, 0)) + a.read(0, -1, 0, 0)) + a.read(0, 0, 1, 0)) +
           a.read(0, 0, -1, 0);
  if (kind == 2) {
    double s = a.read(0, -1, -1, 0);
    s += a.read(0, 0, -1, 0);
    s += a.read(0, 1, -1, 0);
    s += a.read(0, -1, 0, 0);
    s += a.read(0, 0, 0, 0);
    s += a.read(0, 1, 0, 0);
    s += a.read(0, -1, 1, 0);
    s += a.read(0, 0, 1, 0);
    s += a.read(0, 1, 1, 0);
    return s;
  }
  if (kind == 3) return (a.read(0, 0, 0, 0) + a.read(0, 1, 0, 0)) + a.read(0, 0, 1, 0);
  double s = a.read(0, 0, 0, 0);
  s += a.read(0, 1, 0, 0);
  s += a.read(0, -1, 0, 0);
  s += a.read(0, 2, 0, 0);
  s += a.read(0, -2, 0, 0);
  s += a.read(0, 0, 1, 0);
  s += a.read(0, 0, -1, 0);
  s += a.read(0, 0, 2, 0);
  s += a.read(0, 0, -2, 0);
  return s;
}

TC_HD double hydro_inv_npts(int kind) {
  return kind == 0 ? 1.0 : kind == 1 ? 0.2 : kind == 2 ? (1.0 / 9.0) : kind == 3 ? (1.0 / 3.0) : (1.0 / 9.0);
}

template <class A>
TC_HD void hydro_loop(A& a, int kind, bool r3) {
  const double m = hydro_stencil_sum(a, kind) * hydro_inv_npts(kind);
  const double c = a.read(0, 0, 0, 0);
  const double r2 = a.read(1, 0, 0, 0);
  double out;
  if (r3) {
    const double r3v = a.read(2, 0, 0, 0);
    out = (((0.25 + 0.5 * m) + 0.0625 * r2) + 0.0625 * r3v) + 0.125 * (c * r2);
    a.write(3, out);
  } else {
    out = ((0.25 + 0.5 * m) + 0.125 * r2) + 0.125 * (c * r2);
    a.write(2, out);
  }
}

// Compile-time body tag (dispatch hands one to the executors' lambdas).
template <int B>
struct BodyTag {
  static constexpr int value = B;
};

// ---------------------------------------------------------------------------
// c5 compressible Navier-Stokes bodies live in their own header.
}  // namespace tcb

#include "tc_ns.h"

namespace tcb {

TC_HD bool body_known(int32_t b) {
  switch (b) {
    case kGenSum: case kJacobiStencil: case kJacobiCopy:
    case kMhEos: case kMhBcX: case kMhBcY: case kMhAccelX: case kMhAccelY: case kMhFluxX:
    case kMhFluxY: case kMhAdvectRho: case kMhAdvectE: case kMhSmooth: case kMhBlend:
    case kMhMonitor:
    case kSmooth2D: case kSmooth1D: case kConsume1D: case kCopy: case kSumRead: case kIota: case kNbrSum:
    case kHeatLap: case kHeatCopy: case kHydroCfl: case kJacobi3D:
    case kCgPUpdate: case kCgMatvec: case kCgXUpdate: case kCgRUpdate: case kCgDot:
      return true;
    default:
      if (b >= kHydroBase && b < kHydroBase + 10) return true;
      return ns_body_known(b);
  }
}

// Compile-time body list for executors that hoist the dispatch out of the
// per-point loop (one specialised point loop per body).
#define TCB_CORE_BODIES(X)                                                                              \
  X(kGenSum) X(kJacobiStencil) X(kJacobiCopy) X(kMhEos) X(kMhBcX) X(kMhBcY) X(kMhAccelX) X(kMhAccelY)    \
  X(kMhFluxX) X(kMhFluxY) X(kMhAdvectRho) X(kMhAdvectE) X(kMhSmooth) X(kMhBlend) X(kMhMonitor)          \
  X(kSmooth2D) X(kSmooth1D) X(kConsume1D) X(kCopy) X(kSumRead) X(kIota) X(kNbrSum) X(kHeatLap)         \
  X(kHeatCopy) X(kHydroBase + 0) X(kHydroBase + 1) X(kHydroBase + 2) X(kHydroBase + 3)                 \
  X(kHydroBase + 4) X(kHydroBase + 5) X(kHydroBase + 6) X(kHydroBase + 7) X(kHydroBase + 8)             \
  X(kHydroBase + 9) X(kHydroCfl) X(kJacobi3D) X(kCgPUpdate) X(kCgMatvec) X(kCgXUpdate) X(kCgRUpdate)    \
  X(kCgDot)

// Calls f(BodyTag<body>{}) for a registered body; false if unknown.
template <class F>
TC_HD bool dispatch(int32_t body, F&& f) {
  switch (body) {
#define TCB_CASE(B) \
  case B:           \
    f(BodyTag<B>{}); \
    return true;
    TCB_CORE_BODIES(TCB_CASE)
#undef TCB_CASE
    default:
      return ns_dispatch(body, f);
  }
}

// One body, selected at compile time: only the matching branch is
// instantiated (the generated streaming kernels call body_t<B> directly).
template <int B, class A>
TC_HD void body_t(A& a, const double* p) {
  (void)p;
  if constexpr (B == kGenSum) {
    gen_sum(a, p);
  } else if constexpr (B == kJacobiStencil) {  // proj/core/src/apps.cpp:43-57
    a.write(1, 0.5 * a.read(0, 0, 0, 0) +
                   0.125 * (a.read(0, 1, 0, 0) + a.read(0, -1, 0, 0) + a.read(0, 0, 1, 0) + a.read(0, 0, -1, 0)));
  } else if constexpr (B == kJacobiCopy) {
    a.write(1, a.read(0, 0, 0, 0));
  } else if constexpr (B == kMhEos) {  // proj/core/src/apps.cpp:163-254 (mini-hydro)
    a.write(2, 0.4 * a.read(0, 0, 0, 0) * a.read(1, 0, 0, 0));
  } else if constexpr (B == kMhBcX) {
    a.write(1, a.read(0, 1, 0, 0));
  } else if constexpr (B == kMhBcY) {
    a.write(1, a.read(0, 0, 1, 0));
  } else if constexpr (B == kMhAccelX) {
    a.increment(1, 0.01 * (a.read(0, 1, 0, 0) - a.read(0, 0, 0, 0)));
  } else if constexpr (B == kMhAccelY) {
    a.increment(1, 0.01 * (a.read(0, 0, 1, 0) - a.read(0, 0, 0, 0)));
  } else if constexpr (B == kMhFluxX) {
    a.write(2, 0.5 * (a.read(0, 0, 0, 0) * a.read(1, 0, 0, 0) + a.read(0, 1, 0, 0) * a.read(1, 1, 0, 0)));
  } else if constexpr (B == kMhFluxY) {
    a.write(2, 0.5 * (a.read(0, 0, 0, 0) * a.read(1, 0, 0, 0) + a.read(0, 0, 1, 0) * a.read(1, 0, 1, 0)));
  } else if constexpr (B == kMhAdvectRho) {
    a.increment(2, 0.01 * (a.read(0, -1, 0, 0) - a.read(0, 0, 0, 0) + a.read(1, 0, -1, 0) - a.read(1, 0, 0, 0)));
  } else if constexpr (B == kMhAdvectE) {
    a.increment(2, 0.005 * (a.read(0, -1, 0, 0) - a.read(0, 0, 0, 0) + a.read(1, 0, -1, 0) - a.read(1, 0, 0, 0)));
  } else if constexpr (B == kMhSmooth) {
    a.write(1, 0.25 * (a.read(0, 1, 0, 0) + a.read(0, -1, 0, 0) + a.read(0, 0, 1, 0) + a.read(0, 0, -1, 0)));
  } else if constexpr (B == kMhBlend) {
    a.write(0, 0.9 * a.read(0, 0, 0, 0) + 0.1 * a.read(1, 0, 0, 0));
  } else if constexpr (B == kMhMonitor) {
    a.contribute(a.read(0, 0, 0, 0));
  } else if constexpr (B == kSmooth2D) {  // proj/tests/test_executor.cpp:29-33, test_dist.cpp:27-60
    a.write(1, 0.5 * a.read(0, 0, 0, 0) +
                   0.125 * (a.read(0, -1, 0, 0) + a.read(0, 1, 0, 0) + a.read(0, 0, -1, 0) + a.read(0, 0, 1, 0)));
  } else if constexpr (B == kSmooth1D) {
    a.write(1, 0.5 * a.read(0, 0, 0, 0) + 0.25 * (a.read(0, -1, 0, 0) + a.read(0, 1, 0, 0)));
  } else if constexpr (B == kConsume1D) {
    a.write(1, 0.25 * (a.read(0, -1, 0, 0) + a.read(0, 0, 0, 0) + a.read(0, 1, 0, 0)));
  } else if constexpr (B == kCopy) {
    a.write(1, a.read(0, 0, 0, 0));
  } else if constexpr (B == kSumRead) {
    a.contribute(a.read(0, 0, 0, 0));
  } else if constexpr (B == kIota) {
    a.write(0, static_cast<double>(a.x()));
  } else if constexpr (B == kNbrSum) {
    a.write(1, a.read(0, -1, 0, 0) + a.read(0, 1, 0, 0));
  } else if constexpr (B == kHeatLap) {  // c1 heat: v = u + 0.1 * (E + W + N + S - 4u)
    const double c = a.read(0, 0, 0, 0);
    const double lap =
        (((a.read(0, 1, 0, 0) + a.read(0, -1, 0, 0)) + a.read(0, 0, 1, 0)) + a.read(0, 0, -1, 0)) - 4.0 * c;
    a.write(1, c + 0.1 * lap);
  } else if constexpr (B == kHeatCopy) {
    a.write(1, a.read(0, 0, 0, 0));
  } else if constexpr (B == kHydroCfl) {  // c2: cell-wise CFL-like expression, min-reduced
    // Named reads: the three loads are sequenced (rho, p, c) in every
    // instantiation, whatever the accessor.
    const double rho = a.read(0, 0, 0, 0);
    const double pr = a.read(1, 0, 0, 0);
    const double cs = a.read(2, 0, 0, 0);
    a.contribute(0.5 / (rho + pr * cs));
  } else if constexpr (B == kJacobi3D) {
    // c3: b = 0.5*a + 0.5*(sum of 6 neighbours * 1/6) -- the 1/6 averaging
    // coefficient is a constant product (no per-point IEEE division).
    const double s = ((((a.read(0, 1, 0, 0) + a.read(0, -1, 0, 0)) + a.read(0, 0, 1, 0)) + a.read(0, 0, -1, 0)) +
                      a.read(0, 0, 0, 1)) +
                     a.read(0, 0, 0, -1);
    a.write(1, 0.5 * a.read(0, 0, 0, 0) + 0.5 * (s * (1.0 / 6.0)));
  } else if constexpr (B == kCgPUpdate) {  // c4 CG: p (RW), r (R); params [beta]
    a.write(0, a.read(1, 0, 0, 0) + p[0] * a.read(0, 0, 0, 0));
  } else if constexpr (B == kCgMatvec) {  // p (R star5), kx (R {0,-x}), ky (R {0,-y}), q (W)
    const double pc = a.read(0, 0, 0, 0);
    const double kxe = a.read(1, 0, 0, 0), kxw = a.read(1, -1, 0, 0);
    const double kyn = a.read(2, 0, 0, 0), kys = a.read(2, 0, -1, 0);
    const double diag = (((1.0 + kxe) + kxw) + kyn) + kys;
    const double q = ((((diag * pc - kxe * a.read(0, 1, 0, 0)) - kxw * a.read(0, -1, 0, 0)) - kyn * a.read(0, 0, 1, 0)) -
                      kys * a.read(0, 0, -1, 0));
    a.write(3, q);
    a.contribute(pc * q);
  } else if constexpr (B == kCgXUpdate) {  // x (RW), p (R); params [alpha]
    a.write(0, a.read(0, 0, 0, 0) + p[0] * a.read(1, 0, 0, 0));
  } else if constexpr (B == kCgRUpdate) {  // r (RW), q (R); params [alpha]
    const double r = a.read(0, 0, 0, 0) - p[0] * a.read(1, 0, 0, 0);
    a.write(0, r);
    a.contribute(r * r);
  } else if constexpr (B == kCgDot) {
    const double r = a.read(0, 0, 0, 0);
    a.contribute(r * r);
  } else if constexpr (B >= kHydroBase && B < kHydroBase + 10) {
    hydro_loop(a, (B - kHydroBase) >> 1, ((B - kHydroBase) & 1) != 0);
  } else {
    static_assert(ns_body_known(B), "body id not in the registry");
    ns_body_t<B>(a, p);
  }
}

// Dispatch one body at one point (run-time id). Returns false for an unknown id.
template <class A>
TC_HD bool run_body(int32_t body, A& a, const double* p) {
  switch (body) {
#define TCB_RUN(B)        \
  case B:                 \
    body_t<B>(a, p);      \
    return true;
    TCB_CORE_BODIES(TCB_RUN)
    TCB_NS_BODIES(TCB_RUN)
#undef TCB_RUN
    default:
      return false;
  }
}

}  // namespace tcb
