// Host-side interface of the CUDA executors (implemented in
// csrc/cuda/tcg_exec.cu). Host code includes this without CUDA headers.
#pragma once
#include <array>
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
  // Reduction mask (execute_plan's reduction_mask, executor.cpp:209-250):
  // when set, only points inside contribute (a rank's owned box).
  bool masked = false;
  int64_t mask[3][2] = {{0, 1}, {0, 1}, {0, 1}};
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
  // Box copies (stream-ordered) between field f's current buffer and a dense
  // buffer laid out over buf_box (dim 0 fastest), host or device memory.
  void field_to_buf(int f, const Range& box, double* buf, const Range& buf_box);
  void buf_to_field(int f, const Range& box, const double* buf, const Range& buf_box);
  // Copy box + shift -> box inside field f (periodic ghost layers).
  void copy_within(int f, const Range& dst_box, const Point& shift);
  // Sets every byte of box (inside field f's allocation) to `byte`
  // (0xFF: every double a NaN -- the halo-poisoning tripwire).
  void fill_box_bytes(int f, const Range& box, int byte);
  // Periodic ghost fill of fields (all with the same logical box), all
  // dimensions in order (edges/corners wrap), one kernel launch per dimension.
  // ndims >= 0: wrap only dimensions [0, ndims) (a rank of a grid split along
  // the slowest dimension wraps the faster ones itself; the slowest one is
  // carried between the end ranks as whole slabs).
  void periodic_fill(const std::vector<int>& fields, const Range& logical, int64_t depth, int ndims = -1);
  // Device staging for halo messages: >= n doubles, valid until the next
  // call that needs more.
  double* staging(size_t n);
  // Contiguous slabs along the slowest dimension (whole rows in 2D, whole
  // planes in 3D, pitch padding included): the halo messages of a domain
  // split along that dimension need no packing.
  //   slab_ptr   first element of slab coordinate s of field f
  //   slab_count doubles in slabs [s0, s1)
  //   same_cross_section  both fields share every faster dimension's range
  //                       and pitch, so slab s of one maps onto slab s of the other
  //   copy_slabs f_dst[s0, s1) <- f_src[s0, s1) (cudaMemcpyPeerAsync: the same
  //              call carries a rank pair hosted on two devices of one process)
  double* slab_ptr(int f, int64_t s);
  size_t slab_count(int f, int64_t s0, int64_t s1);
  bool same_cross_section(int fa, int fb) const;
  void copy_slabs(int f_dst, int f_src, int64_t s0, int64_t s1);
  // f_dst[dst_s0, dst_s0 + n) <- f_src[src_s0, src_s0 + n): the periodic wrap along the slowest dimension.
  void copy_slabs_shift(int f_dst, int64_t dst_s0, int f_src, int64_t src_s0, int64_t n);
  void note_slab_write(int f, int64_t s0, int64_t s1);
  int device_index() const { return device_; }
  // Device buffer for reduction partials exchanged between processes.
  double* red_buffer(size_t n);
  // Stream-ordered small copies; d2h synchronizes the stream.
  void h2d(double* dev, const double* host, size_t n);
  void d2h(double* host, const double* dev, size_t n);

  // Execute a lowered chain loop by loop (reference execute_untiled,
  // executor.cpp:252-277). Reductions land in red_out (host) when the call
  // returns if sync_reductions is true.
  void run_untiled(const DevChain& ch, double* red_out);
  // Execute with the windowed tiled executor.
  void run_tiled(const DevChain& ch, const GpuTiledPlan& gp, uint64_t plan_key, double* red_out);
  // Execute a reference tile plan (the (tile, loop) items in order, as
  // execute_plan does, executor.cpp:209-250) in one persistent cooperative
  // launch: every CTA works on each item, a grid barrier separates items, so
  // a tile's data stays in the 126 MB L2 from loop to loop.
  // Dataflow mode (deps non-empty): no grid barriers; a CTA waits, chunk by
  // chunk, for the chunks of the conflicting earlier items within `reach` of
  // its chunk (completion flags in global memory).
  void run_l2(const DevChain& ch, const std::vector<DevItem>& items, const std::vector<int32_t>& deps,
              const std::array<int32_t, 3>& reach, uint64_t plan_key, double* red_out);

  // ---- streaming executor support (csrc/cuda/tcg_stream_exec.cu) ----
  // Box of field f's current buffer written by anything but a streaming
  // kernel: the second buffer may differ there from now on.
  void mark_written(int f, const Range& box);
  // Makes field f's second buffer equal to its current one outside `keep`
  // (allocating and copying it whole on first use).
  void sync_alt(int f, const Range& keep);
  // A streaming kernel stored `box` into f's second buffer: swap the buffers;
  // the new second buffer differs from the new current one inside `box`.
  void commit_alt(int f, const Range& box);
  // mark_written for every write of a lowered chain (untiled / L2 / windowed).
  void mark_chain_writes(const DevChain& ch);
  // Reduction scratch of a streaming launch: CTA partials, results, ticket.
  void stream_red_buffers(size_t npart, size_t nout, double** part, double** out, unsigned** ticket);
  void launch_stream(void* fn, int64_t grid, int nt, int smem, const void* args, size_t bytes);
  // Device -> host through the pinned staging buffer (syncs the stream).
  void read_device(double* host, const double* dev, size_t n);

  void synchronize();
  // Copies the first n chain-reduction slots to `out` (syncs the stream).
  void read_reductions(double* out, int n);
  void* stream() const { return stream_; }
  int64_t launches() const { return launches_; }
  // Kernel timing: when enabled, CUDA events bracket every main executor
  // kernel (k_tiled, k_untiled) on the executor stream; kernel_ms() syncs and
  // returns the accumulated device time and launch count since the last reset.
  void set_timing(bool on);
  // Chain-level interval timing for the auto executor choice: record() returns
  // an event recorded on the stream; elapsed_ms(a, b) is valid once b completed.
  void* record();
  bool elapsed_ms(void* a, void* b, float* ms);
  void wait_event(void* ev);
  void release(void* ev);
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
  size_t red_n_ = 0;  // doubles in red_dev_ / red_host_
  double* st_part_ = nullptr;
  size_t st_part_n_ = 0;
  double* st_out_ = nullptr;
  size_t st_out_n_ = 0;
  unsigned* st_ticket_ = nullptr;
  int device_ = 0;
  // Order-matched Sum reductions (set_reduction_workers).
  int red_workers_ = 0;
  double* capture_ = nullptr;
  size_t capture_n_ = 0;
  double* ord_part_ = nullptr;
  unsigned* ord_ticket_ = nullptr;
  double* host_stage_ = nullptr;  // pinned
  size_t host_stage_n_ = 0;
  double* red_host_ = nullptr;  // pinned
  double* staging_ = nullptr;
  size_t staging_n_ = 0;
  double* redbuf_ = nullptr;
  size_t redbuf_n_ = 0;
  std::vector<std::pair<uint64_t, PlanBufs*>> plan_cache_;
  struct ItemBufs {
    uint64_t key = 0;
    size_t nitems = 0;
    DevItem* items = nullptr;
    int32_t* deps = nullptr;
    uint32_t* flags = nullptr;
  };
  std::vector<ItemBufs> item_cache_;
  uint32_t epoch_ = 0;
  int64_t launches_ = 0;
  uint64_t scratch_hash_ = 0;  // content hash of the chain tables in scratch_
  struct UGraph;
  std::vector<UGraph*> graphs_;  // untiled launch sequences as CUDA graphs
  void drop_graphs();
  bool timing_ = false;
  std::vector<std::pair<void*, void*>> ev_tiled_, ev_untiled_;  // (start, stop) event pairs (k_l2tiled counts as tiled)
  std::vector<void*> ev_pool_;
  void* take_event();
  void* ensure_scratch(size_t bytes);
  double* ensure_partials(size_t n);
 public:
  // Sum reductions of untiled chains folded in the reference's order for a
  // pool of `workers` threads (executor.cpp:55-61, :141-144, :175-176):
  // sequential sums over the static memory-order spans, then a worker-order
  // fold. 0 (default): warp/block tree fold. At most 1024 workers.
  void set_reduction_workers(int workers) { red_workers_ = workers < 0 ? 0 : (workers > 1024 ? 1024 : workers); }
  int reduction_workers() const { return red_workers_; }
 private:
  void ensure_red(size_t n);
  PlanBufs* plan_bufs(const GpuTiledPlan& gp, uint64_t key);
};

}  // namespace tcg
