// BASELINE config c5: 3D compressible Navier-Stokes-like chain on a periodic
// 2*pi box (Taylor-Green vortex), 4th-order central differences (radius-2
// star per axis), 3-stage low-storage Runge-Kutta (Williamson 2N):
//   dU = a_s * dU + dt * RHS(U);   U = U + b_s * dU.
// The chain shape is this project's (the reference has no NS app); the
// expressions below are the single source both the device executors and the
// CPU oracle evaluate, in this exact order.
//
// Fields: conserved U = (rho, mx, my, mz, E), stage accumulators dU (5),
// primitives (u, v, w, p, T). Per RK stage: one primitive loop, five RHS
// loops (each accumulates into its dU), one update loop; the step ends with
// a kinetic-energy sum. Periodicity is a ghost copy between loops
// (Runtime::periodic_fill), as the reference would need too.
#pragma once

namespace tcb {

enum NsBody : int32_t {
  kNsPrim = 500,     // args rho,mx,my,mz,E (R) ; u,v,w,p,T (W)            params [gamma-1]
  kNsRhsMass = 501,  // args mx,my,mz (R star2) ; dRho (RW)                 params [1/12h, a, dt]
  kNsRhsMomX = 502,  // args m_c,u,v,w,p (R star2) ; dM_c (RW)              params [1/12h, 1/12h^2, mu, a, dt]
  kNsRhsMomY = 503,
  kNsRhsMomZ = 504,
  kNsRhsEnergy = 505,  // args E,p,u,v,w,T (R star2) ; dE (RW)  params [1/12h, 1/12h^2, mu, kappa, a, dt]
  kNsUpdate = 506,     // args U0..U4 (RW) ; dU0..dU4 (R)       params [b]
  kNsKinetic = 507,    // args rho,mx,my,mz (R) ; Sum reduction of 0.5*|m|^2/rho
};

// 4th-order first derivative along `axis` of f(k) = value at offset k:
// (8 (f[+1] - f[-1]) - (f[+2] - f[-2])) / (12 h).
template <class F>
TC_HD double ns_d1(F&& f, double inv12h) {
  return (8.0 * (f(1) - f(-1)) - (f(2) - f(-2))) * inv12h;
}

// 4th-order second derivative: (-f[+2] + 16 f[+1] - 30 f[0] + 16 f[-1] - f[-2]) / (12 h^2).
template <class F>
TC_HD double ns_d2(F&& f, double inv12h2) {
  return ((((-f(2) + 16.0 * f(1)) - 30.0 * f(0)) + 16.0 * f(-1)) - f(-2)) * inv12h2;
}

// Value of argument `arg` at offset k along `axis`.
template <class A>
TC_HD double ns_at(const A& a, int arg, int axis, int k) {
  return a.read(arg, axis == 0 ? k : 0, axis == 1 ? k : 0, axis == 2 ? k : 0);
}

template <class A>
TC_HD void ns_prim(A& a, const double* p) {
  // One IEEE division per point (1/rho), products elsewhere.
  const double rho = a.read(0, 0, 0, 0);
  const double rinv = 1.0 / rho;
  const double u = a.read(1, 0, 0, 0) * rinv;
  const double v = a.read(2, 0, 0, 0) * rinv;
  const double w = a.read(3, 0, 0, 0) * rinv;
  const double pr = p[0] * (a.read(4, 0, 0, 0) - 0.5 * rho * ((u * u + v * v) + w * w));
  a.write(5, u);
  a.write(6, v);
  a.write(7, w);
  a.write(8, pr);
  a.write(9, pr * rinv);
}

template <class A>
TC_HD void ns_rhs_mass(A& a, const double* p) {
  double conv = 0.0;
  for (int ax = 0; ax < 3; ++ax) conv = conv + ns_d1([&](int k) { return ns_at(a, ax, ax, k); }, p[0]);
  a.write(3, p[1] * a.read(3, 0, 0, 0) + p[2] * (-conv));
}

// Momentum component c: flux along axis ax is m_c * vel_ax (+ p when ax == c);
// viscous term mu * Laplacian(vel_c).
template <class A>
TC_HD void ns_rhs_mom(A& a, const double* p, int c) {
  double conv = 0.0;
  for (int ax = 0; ax < 3; ++ax)
    conv = conv + ns_d1(
                      [&](int k) {
                        const double f = ns_at(a, 0, ax, k) * ns_at(a, 1 + ax, ax, k);
                        return ax == c ? f + ns_at(a, 4, ax, k) : f;
                      },
                      p[0]);
  double lap = 0.0;
  for (int ax = 0; ax < 3; ++ax) lap = lap + ns_d2([&](int k) { return ns_at(a, 1 + c, ax, k); }, p[1]);
  a.write(5, p[3] * a.read(5, 0, 0, 0) + p[4] * (p[2] * lap - conv));
}

// Energy: flux (E + p) vel_ax; viscous mu * Laplacian(|u|^2 / 2) + kappa * Laplacian(T).
template <class A>
TC_HD void ns_rhs_energy(A& a, const double* p) {
  double conv = 0.0;
  for (int ax = 0; ax < 3; ++ax)
    conv = conv + ns_d1([&](int k) { return (ns_at(a, 0, ax, k) + ns_at(a, 1, ax, k)) * ns_at(a, 2 + ax, ax, k); },
                        p[0]);
  double lk = 0.0, lt = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    lk = lk + ns_d2(
                  [&](int k) {
                    const double u = ns_at(a, 2, ax, k), v = ns_at(a, 3, ax, k), w = ns_at(a, 4, ax, k);
                    return 0.5 * ((u * u + v * v) + w * w);
                  },
                  p[1]);
    lt = lt + ns_d2([&](int k) { return ns_at(a, 5, ax, k); }, p[1]);
  }
  a.write(6, p[4] * a.read(6, 0, 0, 0) + p[5] * ((p[2] * lk + p[3] * lt) - conv));
}

template <class A>
TC_HD void ns_update(A& a, const double* p) {
  for (int c = 0; c < 5; ++c) a.write(c, a.read(c, 0, 0, 0) + p[0] * a.read(5 + c, 0, 0, 0));
}

template <class A>
TC_HD void ns_kinetic(A& a) {
  const double mx = a.read(1, 0, 0, 0), my = a.read(2, 0, 0, 0), mz = a.read(3, 0, 0, 0);
  a.contribute(0.5 * ((mx * mx + my * my) + mz * mz) / a.read(0, 0, 0, 0));
}

#if defined(__CUDACC__)
__host__ __device__ constexpr bool ns_body_known(int32_t b) { return b >= kNsPrim && b <= kNsKinetic; }
#else
constexpr bool ns_body_known(int32_t b) { return b >= kNsPrim && b <= kNsKinetic; }
#endif

#define TCB_NS_BODIES(X) \
  X(kNsPrim) X(kNsRhsMass) X(kNsRhsMomX) X(kNsRhsMomY) X(kNsRhsMomZ) X(kNsRhsEnergy) X(kNsUpdate) X(kNsKinetic)

template <int B, class A>
TC_HD void ns_body_t(A& a, const double* p) {
  if constexpr (B == kNsPrim) ns_prim(a, p);
  else if constexpr (B == kNsRhsMass) ns_rhs_mass(a, p);
  else if constexpr (B == kNsRhsMomX) ns_rhs_mom(a, p, 0);
  else if constexpr (B == kNsRhsMomY) ns_rhs_mom(a, p, 1);
  else if constexpr (B == kNsRhsMomZ) ns_rhs_mom(a, p, 2);
  else if constexpr (B == kNsRhsEnergy) ns_rhs_energy(a, p);
  else if constexpr (B == kNsUpdate) ns_update(a, p);
  else ns_kinetic(a);
}

template <class F>
TC_HD bool ns_dispatch(int32_t body, F&& f) {
  switch (body) {
    case kNsPrim: f(BodyTag<kNsPrim>{}); return true;
    case kNsRhsMass: f(BodyTag<kNsRhsMass>{}); return true;
    case kNsRhsMomX: f(BodyTag<kNsRhsMomX>{}); return true;
    case kNsRhsMomY: f(BodyTag<kNsRhsMomY>{}); return true;
    case kNsRhsMomZ: f(BodyTag<kNsRhsMomZ>{}); return true;
    case kNsRhsEnergy: f(BodyTag<kNsRhsEnergy>{}); return true;
    case kNsUpdate: f(BodyTag<kNsUpdate>{}); return true;
    case kNsKinetic: f(BodyTag<kNsKinetic>{}); return true;
    default: return false;
  }
}

}  // namespace tcb
