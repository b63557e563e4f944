// Run-time compilation of generated chain kernels (NVRTC, sm_100a) and their
// launch through the CUDA driver API. Kernels are cached in memory by source
// hash and on disk as cubins (TCG_JIT_CACHE, default <library dir>/jit), so a
// chain signature is compiled once per machine.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

namespace tcg {

// Compiles `src` (kernel `tcg_stream`) to an sm_100a cubin. Throws CudaError
// with the NVRTC log on failure. Needs no GPU.
std::string jit_compile_cubin(const std::string& src, std::string* log = nullptr);

// Loaded kernel for the current device context (compiles on a cache miss).
void* jit_function(const std::string& src, uint64_t hash, int smem_bytes);

// Launch: grid x 1 x 1 CTAs of nt threads, dynamic shared memory, the kernel
// argument block passed by value.
void jit_launch(void* func, int64_t grid, int nt, int smem_bytes, void* stream, const void* args, size_t arg_bytes);

// Resident CTAs per SM of a loaded kernel at nt threads and smem bytes.
int jit_occupancy(void* func, int nt, int smem_bytes);

// Registers and local memory of a loaded kernel (tests, reports).
void jit_attributes(void* func, int* regs, int* local_bytes);

}  // namespace tcg
