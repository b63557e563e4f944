// Host-side interface of the CUDA executors (implemented in
// csrc/cuda/tcg_exec.cu). Host code includes this without CUDA headers.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "tcg_device.hpp"
#include "tcg_gpuplan.hpp"
#include "tcg_types.hpp"

namespace tcg {

// One chain lowered for the device: loops with chain-local dataset slots,
// the parameter blob and the stencil table.
struct DevChain {
  int dim = 1;
  std::vector<DevLoop> loops;
  std::vector<double> params;
  std::vector<int32_t> st_start, st_npts, st_pts;
  std::vector<DatasetId> dat_ids;  // slot -> dataset
  int nred = 0;
  std::vector<int32_t> red_op;     // per reduction index
};

struct DeviceInfo {
  int device = 0;
  int num_sms = 0;
  int64_t smem_optin = 0;
  int64_t smem_per_sm = 0;
  int64_t l2_bytes = 0;
  std::string name;
};

// Timing of the last executed chain on the executor stream (CUDA events).
struct ExecTiming {
  int launches = 0;
  double gpu_ms = 0;
};

// cudaSetDevice in this library's CUDA runtime (one process per GPU).
void select_device(int device);

class DeviceExec {
 public:
  DeviceExec();
  ~DeviceExec();
  DeviceExec(const DeviceExec&) = delete;
  DeviceExec& operator=(const DeviceExec&) = delete;

  const DeviceInfo& info() const { return info_; }

  // Field storage. The second buffer of a dataset is allocated on first use
  // by a ping-ponged tiled chain.
  int add_field(const Range& alloc);
  void upload(int f, const double* host_dense);
  void download(int f, double* host_dense);
  void upload_async(int f, const double* host_dense);     // host buffer must be pinned and live
  void download_async(int f, double* host_dense);
  DevView view(int f, bool alt);
  void swap(int f);
  int64_t field_bytes(int f) const;
  double get_point(int f, const Point& p);
  void put_point(int f, const Point& p, double v);

  // Execute a lowered chain loop by loop (reference execute_untiled,
  // executor.cpp:252-277). Reductions land in red_out (host) when the call
  // returns if sync_reductions is true.
  void run_untiled(const DevChain& ch, double* red_out);
  // Execute with the windowed tiled executor.
  void run_tiled(const DevChain& ch, const GpuTiledPlan& gp, uint64_t plan_key, double* red_out);

  void synchronize();
  void* stream() const { return stream_; }
  int64_t launches() const { return launches_; }
  // Kernel timing: when enabled, CUDA events bracket every main executor
  // kernel (k_tiled, k_untiled) on the executor stream; kernel_ms() syncs and
  // returns the accumulated device time and launch count since the last reset.
  void set_timing(bool on);
  void kernel_ms(double* tiled_ms, int64_t* tiled_n, double* untiled_ms, int64_t* untiled_n);
  // Bytes of dynamic shared memory available for windows for a chain shape.
  int64_t window_budget_doubles(int nloops, int nred, int ctas_per_sm) const;

 private:
  struct Buf;
  struct PlanBufs;
  DeviceInfo info_;
  void* stream_ = nullptr;
  std::vector<Buf*> fields_;
  // scratch
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  double* partials_ = nullptr;
  size_t partials_n_ = 0;
  double* red_dev_ = nullptr;
  std::vector<std::pair<uint64_t, PlanBufs*>> plan_cache_;
  int64_t launches_ = 0;
  bool timing_ = false;
  std::vector<std::pair<void*, void*>> ev_tiled_, ev_untiled_;  // (start, stop) event pairs
  std::vector<void*> ev_pool_;
  void* take_event();
  void* ensure_scratch(size_t bytes);
  double* ensure_partials(size_t n);
  PlanBufs* plan_bufs(const GpuTiledPlan& gp, uint64_t key);
};

}  // namespace tcg
