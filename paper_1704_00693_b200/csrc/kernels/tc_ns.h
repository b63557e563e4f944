// BASELINE config c5 (3D compressible Navier-Stokes, Taylor-Green vortex)
// kernel bodies. Filled in with the c5 chain; until then no id in
// [kNsFirst, kNsLast] is registered.
#pragma once

namespace tcb {

TC_HD bool ns_body_known(int32_t) { return false; }

template <class A>
TC_HD bool ns_run_body(int32_t, A&, const double*) {
  return false;
}

template <class F>
TC_HD bool ns_dispatch(int32_t, F&&) {
  return false;
}

}  // namespace tcb
