// Shared pieces of the CUDA executors (one copy per translation unit).
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../host/tcg_exec.hpp"
#include "../kernels/tc_bodies.h"

namespace tcg {

namespace {

#define TCG_CK(x)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kTiledThreads = 512;
constexpr int kMaxParams = 16;

__host__ __device__ __forceinline__ double red_identity(int op) {
  return op == 0 ? 0.0 : (op == 1 ? HUGE_VAL : -HUGE_VAL);
}
__device__ __forceinline__ double red_combine(int op, double a, double b) {
  return op == 0 ? a + b : (op == 1 ? (a < b ? a : b) : (a > b ? a : b));
}

// Block-wide reduction, deterministic for a fixed block shape: xor-shuffle
// tree inside each warp, then warp results in warp order. Result on thread 0.
__device__ double block_reduce(double v, int op) {
  __shared__ double ws[32];
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  for (int o = 16; o > 0; o >>= 1) v = red_combine(op, v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((tid & 31) == 0) ws[tid >> 5] = v;
  __syncthreads();
  if (tid < 32) {
    const int nw = (nthr + 31) >> 5;
    v = tid < nw ? ws[tid] : red_identity(op);
    for (int o = 16; o > 0; o >>= 1) v = red_combine(op, v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;
}

__global__ void __launch_bounds__(1024) k_fold(const double* __restrict__ p, int64_t n, int op, double* out) {
  const int64_t chunk = (n + blockDim.x - 1) / blockDim.x;
  const int64_t a = static_cast<int64_t>(threadIdx.x) * chunk;
  const int64_t b = a + chunk < n ? a + chunk : n;
  double v = red_identity(op);
  for (int64_t i = a; i < b; ++i) v = red_combine(op, v, p[i]);
  v = block_reduce(v, op);
  if (threadIdx.x == 0) *out = v;
}

// Uploads the chain tables into scratch; returns device pointers.
struct ChainDev {
  DevLoop* loops;
  double* params;
  DevStencils st;
};

template <class T>
size_t align_up(size_t v) {
  return (v + 255) / 256 * 256 + 0 * sizeof(T);
}

// Hash of a byte range, 8 bytes per step (keys of per-flush caches: cheap
// enough to run on every flush of a launch-bound chain).
uint64_t fnv_bytes(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h = (h ^ w) * 1099511628211ull;
    h ^= h >> 29;
  }
  for (; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// Content hash of the chain tables upload_chain writes (loops, params,
// stencil tables) plus the scratch address they go to.
uint64_t chain_tables_hash(const DevChain& ch, const void* scratch) {
  uint64_t h = 1469598103934665603ull;
  h = fnv_bytes(h, &scratch, sizeof scratch);
  h = fnv_bytes(h, ch.loops.data(), ch.loops.size() * sizeof(DevLoop));
  h = fnv_bytes(h, ch.params.data(), ch.params.size() * sizeof(double));
  h = fnv_bytes(h, ch.st_start.data(), ch.st_start.size() * 4);
  h = fnv_bytes(h, ch.st_npts.data(), ch.st_npts.size() * 4);
  h = fnv_bytes(h, ch.st_pts.data(), ch.st_pts.size() * 4);
  return (h ^ ch.loops.size() * 31 ^ ch.params.size() * 131 ^ ch.st_pts.size() * 1031) | 1;
}

// Uploads the chain tables into scratch (skipped when *last_hash says the
// scratch already holds identical tables: repeated flushes of one chain then
// cost no host-to-device copies). Returns the device pointers.
ChainDev upload_chain(const DevChain& ch, void* scratch, cudaStream_t st, uint64_t* last_hash = nullptr) {
  const uint64_t hh = last_hash ? chain_tables_hash(ch, scratch) : 0;
  const bool skip = last_hash && *last_hash == hh;
  if (last_hash) *last_hash = hh;
  const size_t nl = ch.loops.size() * sizeof(DevLoop);
  const size_t np = std::max<size_t>(1, ch.params.size()) * sizeof(double);
  const size_t ns = std::max<size_t>(1, ch.st_start.size()) * 4;
  const size_t nq = std::max<size_t>(1, ch.st_pts.size()) * 4;
  char* base = static_cast<char*>(scratch);
  size_t off = 0;
  ChainDev cd;
  cd.loops = reinterpret_cast<DevLoop*>(base + off);
  if (nl && !skip) TCG_CK(cudaMemcpyAsync(base + off, ch.loops.data(), nl, cudaMemcpyHostToDevice, st));
  off += align_up<char>(nl);
  cd.params = reinterpret_cast<double*>(base + off);
  if (!ch.params.empty() && !skip)
    TCG_CK(cudaMemcpyAsync(base + off, ch.params.data(), ch.params.size() * 8, cudaMemcpyHostToDevice, st));
  off += align_up<char>(np);
  int32_t* s0 = reinterpret_cast<int32_t*>(base + off);
  if (!ch.st_start.empty() && !skip) TCG_CK(cudaMemcpyAsync(s0, ch.st_start.data(), ch.st_start.size() * 4, cudaMemcpyHostToDevice, st));
  off += align_up<char>(ns);
  int32_t* s1 = reinterpret_cast<int32_t*>(base + off);
  if (!ch.st_npts.empty() && !skip) TCG_CK(cudaMemcpyAsync(s1, ch.st_npts.data(), ch.st_npts.size() * 4, cudaMemcpyHostToDevice, st));
  off += align_up<char>(ns);
  int32_t* s2 = reinterpret_cast<int32_t*>(base + off);
  if (!ch.st_pts.empty() && !skip) TCG_CK(cudaMemcpyAsync(s2, ch.st_pts.data(), ch.st_pts.size() * 4, cudaMemcpyHostToDevice, st));
  cd.st = DevStencils{s0, s1, s2};
  return cd;
}

size_t chain_bytes(const DevChain& ch) {
  return align_up<char>(ch.loops.size() * sizeof(DevLoop)) + align_up<char>(std::max<size_t>(1, ch.params.size()) * 8) +
         2 * align_up<char>(std::max<size_t>(1, ch.st_start.size()) * 4) +
         align_up<char>(std::max<size_t>(1, ch.st_pts.size()) * 4) + 256;
}
}  // namespace

struct DeviceExec::Buf {
  Range alloc;
  int64_t x0 = 0, nxp = 0, py = 0, pz = 0, ny = 1, nz = 1;
  double* mem[2] = {nullptr, nullptr};
  size_t bytes = 0;
  int cur = 0;
  // Streaming executor bookkeeping: boxes where the second buffer may differ
  // from the current one (alt_synced false: anywhere).
  std::vector<Range> dirty;
  bool alt_synced = false;
};

struct DeviceExec::PlanBufs {
  void* mem = nullptr;
  DevCta* ctas = nullptr;
  int32_t* boxes = nullptr;
  int32_t* win = nullptr;
  int32_t* wboxes = nullptr;
};

}  // namespace tcg
