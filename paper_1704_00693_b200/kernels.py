"""Body ids of the device kernel registry (csrc/kernels/tc_bodies.h).

A reference KernelHandle carries a host closure (kernel_ctx.hpp:15-19); here a
loop names a registered body and passes its scalars as a parameter block.
"""
GEN_SUM = 1            # chain_gen.cpp:168-196 contracting dyadic combination; params [scale]
JACOBI_STENCIL = 2     # apps.cpp:43-53
JACOBI_COPY = 3        # apps.cpp:55-57
MH_EOS, MH_BC_X, MH_BC_Y, MH_ACCEL_X, MH_ACCEL_Y, MH_FLUX_X, MH_FLUX_Y = 10, 11, 12, 13, 14, 15, 16
MH_ADVECT_RHO, MH_ADVECT_E, MH_SMOOTH, MH_BLEND, MH_MONITOR = 17, 18, 19, 20, 21
SMOOTH_2D = 30         # test_executor.cpp:29-33
SMOOTH_1D = 31         # test_dist.cpp:52-56
CONSUME_1D = 32        # test_dist.cpp:31-35
COPY = 33              # write(1, read(0))
SUM_READ = 34          # contribute(read(0))
IOTA = 35              # write(0, x)  test_oracle.cpp:80-83
NBR_SUM = 36           # write(1, read(0,-1) + read(0,+1))  test_oracle.cpp:86-90
HEAT_LAP = 100         # c1
HEAT_COPY = 101        # c1
HYDRO_BASE = 200       # c2: 200 + 2*stencil_kind + has_r3
HYDRO_CFL = 220        # c2 min-reduction
JACOBI_3D = 300        # c3
CG_P_UPDATE = 400      # c4 p = r + beta*p
CG_MATVEC = 401        # c4 q = A p, sum p.q
CG_X_UPDATE = 402      # c4 x += alpha p
CG_R_UPDATE = 403      # c4 r -= alpha q, sum r.r
CG_DOT = 404           # c4 sum r.r
NS_FIRST = 500         # c5 (3D compressible NS), csrc/kernels/tc_ns.h
NS_PRIM = 500          # rho,mx,my,mz,E -> u,v,w,p,T        params [gamma-1]
NS_RHS_MASS = 501      # dRho = a dRho + dt * RHS           params [1/12h, a, dt]
NS_RHS_MOM = 502       # + component (0..2)                 params [1/12h, 1/12h^2, mu, a, dt]
NS_RHS_ENERGY = 505    #                                    params [1/12h, 1/12h^2, mu, kappa, a, dt]
NS_UPDATE = 506        # U += b dU                          params [b]
NS_KINETIC = 507       # Sum 0.5 |m|^2 / rho


def hydro_body(stencil_kind: int, has_r3: bool) -> int:
    return HYDRO_BASE + 2 * stencil_kind + (1 if has_r3 else 0)
