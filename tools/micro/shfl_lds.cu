// Does SHFL share the shared-memory crossbar with LDS on B200? Times three
// loops per SM-filling grid: LDS.64 only, SHFL (64-bit = 2 x SHFL.32) only,
// and both interleaved. If the mixed loop costs max(a, b) the pipes are
// separate; if a + b they share one.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512) k(double* out, int iters) {
  __shared__ double sm[4 * 512 + 64];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * 512 + 64; i += 512) sm[i] = i * 0.5;
  __syncthreads();
  double a0 = tid, a1 = tid * 2.0, a2 = 1.0, a3 = 3.0;
  const double* p = sm + tid + 1;
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
      a0 += p[0];
      a1 += p[512 + 1];
      a2 += p[1024 + 2];
      a3 += p[1536 + 3];
    }
    if (MODE & 2) {
      a0 += __shfl_up_sync(0xffffffffu, a1, 1);
      a1 += __shfl_down_sync(0xffffffffu, a2, 1);
      a2 += __shfl_up_sync(0xffffffffu, a3, 2);
      a3 += __shfl_down_sync(0xffffffffu, a0, 2);
    }
    p += (it & 1) ? -1 : 1;
  }
  out[blockIdx.x * 512 + tid] = a0 + a1 + a2 + a3;
}

template <int MODE>
float run(double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<148 * 2, 512>>>(out, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<MODE><<<148 * 2, 512>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 2 * 512);
  const int iters = 200000;
  const float a = run<1>(out, iters), b = run<2>(out, iters), c = run<3>(out, iters), d = run<0>(out, iters);
  // per SM per iteration: 32 warps x 4 ops
  const double ops = 32.0 * 4 * iters;
  std::printf("lds64 %.3f ms (%.2f clk/warp-op @1.9GHz)\nshfl64 %.3f ms (%.2f)\nboth %.3f ms\nempty %.3f ms\n", a,
              a * 1e-3 * 1.9e9 / ops, b, b * 1e-3 * 1.9e9 / ops, c, d);
  return 0;
}
