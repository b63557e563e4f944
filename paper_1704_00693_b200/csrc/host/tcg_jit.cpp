// NVRTC compilation and driver-API launch of generated chain kernels.
#include "tcg_jit.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <tuple>
#include <vector>

#include "tcg_types.hpp"

namespace tcg {
namespace {

// tc_bodies.h / tc_ns.h, embedded at build time (build.py writes this file).
#include "tcb_sources.inc"

const char* kStdint =
    "#pragma once\n"
    "typedef signed char int8_t; typedef short int16_t; typedef int int32_t; typedef long long int64_t;\n"
    "typedef unsigned char uint8_t; typedef unsigned short uint16_t; typedef unsigned int uint32_t;\n"
    "typedef unsigned long long uint64_t;\n";

void nv_check(nvrtcResult r, const char* what) {
  if (r != NVRTC_SUCCESS) throw CudaError(std::string("NVRTC ") + what + ": " + nvrtcGetErrorString(r));
}

void cu_check(cudaError_t r, const char* what) {
  if (r != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(r));
}

std::string cache_dir() {
  if (const char* e = std::getenv("TCG_JIT_CACHE")) return e;
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&cache_dir), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const size_t k = p.rfind('/');
    if (k != std::string::npos) return p.substr(0, k) + "/jit";
  }
  return "";
}

std::string hex(uint64_t h) {
  char b[32];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(h));
  return b;
}

struct Loaded {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
  int smem = 0;
};

std::mutex g_mu;
std::map<std::pair<uint64_t, int>, Loaded> g_loaded;

}  // namespace

std::string jit_compile_cubin(const std::string& src, std::string* log) {
  nvrtcProgram prog;
  const char* hdrs[] = {kTcbBodiesSrc, kTcbNsSrc, kStdint};
  const char* names[] = {"tc_bodies.h", "tc_ns.h", "stdint.h"};
  nv_check(nvrtcCreateProgram(&prog, src.c_str(), "tcg_stream.cu", 3, hdrs, names), "create");
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17", "-lineinfo",
                                   "-default-device", "--extra-device-vectorization"};
  if (std::getenv("TCG_JIT_VERBOSE")) opts.push_back("--ptxas-options=-v");
  if (const char* e = std::getenv("TCG_JIT_MAXRREG")) {
    static std::string m;
    m = std::string("--maxrregcount=") + e;
    opts.push_back(m.c_str());
  }
  const nvrtcResult r = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
  size_t n = 0;
  nvrtcGetProgramLogSize(prog, &n);
  std::string lg(n, '\0');
  if (n) nvrtcGetProgramLog(prog, lg.data());
  while (!lg.empty() && lg.back() == '\0') lg.pop_back();
  if (log) *log = lg;
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    throw CudaError("NVRTC compile of a generated chain kernel failed: " + lg.substr(0, 4000));
  }
  size_t cn = 0;
  nv_check(nvrtcGetCUBINSize(prog, &cn), "cubin size");
  std::string cubin(cn, '\0');
  nv_check(nvrtcGetCUBIN(prog, cubin.data()), "cubin");
  nvrtcDestroyProgram(&prog);
  return cubin;
}

void* jit_function(const std::string& src, uint64_t hash, int smem_bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  cu_check(cudaGetDevice(&dev), "cudaGetDevice");
  auto key = std::make_pair(hash, dev);
  auto it = g_loaded.find(key);
  if (it == g_loaded.end()) {
    std::string cubin;
    const std::string dir = cache_dir();
    // The cache key covers the generated source AND the body registry headers
    // it includes (a cubin cached before a body changed must not be reused).
    static const uint64_t headers_hash = [] {
      uint64_t h = 1469598103934665603ull;
      for (const char* t : {kTcbBodiesSrc, kTcbNsSrc})
        for (const char* c = t; *c; ++c) h = (h ^ static_cast<unsigned char>(*c)) * 1099511628211ull;
      return h;
    }();
    const std::string path = dir.empty() ? "" : dir + "/" + hex(hash ^ (headers_hash * 0x9E3779B97F4A7C15ull)) + ".cubin";
    if (!path.empty()) {
      std::ifstream f(path, std::ios::binary);
      if (f) {
        std::ostringstream ss;
        ss << f.rdbuf();
        cubin = ss.str();
      }
    }
    if (cubin.empty()) {
      cubin = jit_compile_cubin(src);
      if (!path.empty()) {
        ::mkdir(dir.c_str(), 0755);
        const std::string tmp = path + ".tmp" + std::to_string(::getpid());
        {
          std::ofstream f(tmp, std::ios::binary);
          f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
        }
        std::rename(tmp.c_str(), path.c_str());
      }
    }
    Loaded L;
    cu_check(cudaLibraryLoadData(&L.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
             "cudaLibraryLoadData(generated chain kernel)");
    cu_check(cudaLibraryGetKernel(&L.fn, L.lib, "tcg_stream"), "cudaLibraryGetKernel");
    it = g_loaded.emplace(key, L).first;
  }
  Loaded& L = it->second;
  if (smem_bytes > L.smem) {
    cu_check(cudaFuncSetAttribute(reinterpret_cast<const void*>(L.fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_bytes),
             "cudaFuncSetAttribute(max dynamic smem)");
    L.smem = smem_bytes;
  }
  return reinterpret_cast<void*>(L.fn);
}

void jit_launch(void* func, int64_t grid, int nt, int smem_bytes, void* stream, const void* args, size_t arg_bytes) {
  (void)arg_bytes;  // the kernel's single by-value parameter block
  void* params[] = {const_cast<void*>(args)};
  cu_check(cudaLaunchKernel(reinterpret_cast<const void*>(func), dim3(static_cast<unsigned>(grid)),
                            dim3(static_cast<unsigned>(nt)), params, static_cast<size_t>(smem_bytes),
                            static_cast<cudaStream_t>(stream)),
           "cudaLaunchKernel(generated chain kernel)");
}

int jit_occupancy(void* func, int nt, int smem_bytes) {
  static std::mutex mu;
  static std::map<std::tuple<void*, int, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(func, nt, smem_bytes);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  cu_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reinterpret_cast<const void*>(func), nt,
                                                         static_cast<size_t>(smem_bytes)),
           "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  cache[key] = n;
  return n;
}

void jit_attributes(void* func, int* regs, int* local_bytes) {
  cudaFuncAttributes fa{};
  cu_check(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(func)), "cudaFuncGetAttributes");
  if (regs) *regs = fa.numRegs;
  if (local_bytes) *local_bytes = static_cast<int>(fa.localSizeBytes);
}

}  // namespace tcg
