// Compiles the reference-side shim (include/tilechain_b200_shim.hpp) against
// the reference's headers and drives the host-only part of the C-ABI through
// it: declarations, the lazy queue, par_loop validation rethrown as the
// reference's exception types. No GPU needed.
#include <cstdio>

#include "tilechain_b200_shim.hpp"

using namespace tilechain;

int main() {
  b200::Runtime rt(2, RuntimeConfig{});
  const StencilId ident = rt.declare_stencil("id", {Point{0, 0, 0}});
  const StencilId star = rt.declare_stencil("star", {Point{0, 0, 0}, Point{1, 0, 0}, Point{-1, 0, 0}, Point{0, 1, 0}, Point{0, -1, 0}});
  const DatasetId u = rt.declare_field("u", Range::d2(0, 32, 0, 32));
  const DatasetId v = rt.declare_field("v", Range::d2(0, 32, 0, 32));
  const double none[1] = {0};
  // c1's two loops (body ids of tc_bodies.h: kHeatLap = 100, kHeatCopy = 101)
  rt.par_loop(0, 100, std::span<const double>(none, 0), Range::d2(0, 32, 0, 32),
              {ArgSpec{u, star, AccessMode::Read}, ArgSpec{v, ident, AccessMode::Write}});
  rt.par_loop(1, 101, std::span<const double>(none, 0), Range::d2(0, 32, 0, 32),
              {ArgSpec{v, ident, AccessMode::Read}, ArgSpec{u, ident, AccessMode::Write}});
  if (rt.pending_loops() != 2) return 1;
  bool threw = false;
  try {  // write through a multi-point stencil: the reference's InvalidArgument (runtime.cpp:45-52)
    rt.par_loop(2, 101, std::span<const double>(none, 0), Range::d2(0, 32, 0, 32),
                {ArgSpec{v, ident, AccessMode::Read}, ArgSpec{u, star, AccessMode::Write}});
  } catch (const InvalidArgument&) {
    threw = true;
  }
  if (!threw) return 2;
  threw = false;
  try {  // body reads outside its declared stencil: the reference's AccessError (kernel_ctx.hpp:58-73)
    rt.par_loop(3, 100, std::span<const double>(none, 0), Range::d2(0, 32, 0, 32),
                {ArgSpec{u, ident, AccessMode::Read}, ArgSpec{v, ident, AccessMode::Write}});
  } catch (const AccessError&) {
    threw = true;
  }
  if (!threw) return 3;
  if (rt.pending_loops() != 2) return 4;
  std::puts("shim ok");
  return 0;
}
