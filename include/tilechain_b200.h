/*
 * tilechain_b200.h -- C-ABI of the B200-native lazy stencil-chain executor.
 *
 * The reference (`tilechain`, arXiv 1704.00693 restated in C++20) exposes its
 * hot path through the C++ class tilechain::Runtime
 * (proj/core/include/tilechain/runtime.hpp:44-135). It has no foreign-function
 * interface of its own; each entry point below is the plain-C form of one
 * reference member, with the same argument meaning, validation and error
 * behaviour (an error code + message instead of a C++ exception):
 *
 *   tcg_runtime_new        Runtime::Runtime(Block, RuntimeConfig)   runtime.hpp:46, runtime.cpp:7-14
 *   tcg_declare_stencil    Runtime::declare_stencil                 runtime.hpp:48, runtime.cpp:16-22
 *   tcg_declare_field      Runtime::declare_field                   runtime.hpp:49-50, runtime.cpp:24-33
 *   tcg_par_loop           Runtime::par_loop                        runtime.hpp:56-58, runtime.cpp:35-92
 *   tcg_flush              Runtime::flush(ExecMode)                 runtime.hpp:61-64, runtime.cpp:103-151
 *   tcg_set_default_mode   Runtime::set_default_mode                runtime.hpp:63
 *   tcg_fetch_reduction    Runtime::fetch_reduction                 runtime.hpp:69, runtime.cpp:164-197
 *   tcg_get / tcg_put      Runtime::get / put                       runtime.hpp:73-74, runtime.cpp:199-207
 *   tcg_fill_logical       Runtime::fill_logical                    runtime.hpp:75, runtime.cpp:209-212
 *   tcg_upload/download    bulk form of put/get over a whole allocation (Field layout, field.cpp:7-28)
 *   tcg_plan_pending       take_pending + construct_plan + TilingPlan::dump   runtime.cpp:94-101, planner.cpp:55-250
 *   tcg_rank_plans_pending construct_rank_plan + compute_halo_depths          dist.cpp:191-448
 *   tcg_auto_tile_size     auto_tile_size                           tile_sizer.cpp:27-81
 *   tcg_report_text        ExecutionReport::to_text                 executor.cpp:321-366
 *   tcg_set_rank_grid      Runtime::set_rank_grid (ranks simulated in one process)  runtime.hpp:77-81, runtime.cpp:213-222
 *   tcg_set_process_rank   one rank per process (DistContext's ranks as processes, NCCL transport)  dist.hpp:96-156
 *   tcg_dist_schedule_pending  construct_rank_plan + compute_halo_depths + exchange_halos message list
 *                          for the pending chain (host only)        dist.cpp:191-511
 *
 * Kernels: the reference's KernelHandle{id, name, std::function} becomes
 * (kernel_id, body, params): `body` selects a per-point body compiled into the
 * device registry (csrc/kernels/tc_bodies.h); a body not in the registry is an
 * error. There is no CPU fallback: flush, get and put fail with TCG_ERR_CUDA
 * when no B200 is visible.
 *
 * Conventions: every call returns 0 on success or one of the TCG_ERR_* codes;
 * tcg_last_error() describes the last failure on the calling thread. Calls on
 * one runtime come from one host thread (SPEC: one control thread owns the
 * queue). Ranges are half-open [lo, hi) per dimension, 6 int64 values
 * {lo0, hi0, lo1, hi1, lo2, hi2}; unused dimensions are ignored.
 */
#ifndef TILECHAIN_B200_H
#define TILECHAIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TCG_OK = 0,
  TCG_ERR_INVALID_ARGUMENT = 1, /* tilechain::InvalidArgument */
  TCG_ERR_ACCESS = 2,           /* tilechain::AccessError */
  TCG_ERR_PLAN = 3,             /* tilechain::PlanError */
  TCG_ERR_CUDA = 4,             /* device missing or CUDA failure */
  TCG_ERR_SIZER = 5,            /* tilechain::SizerError */
  TCG_ERR_INTERNAL = 6
};

/* AccessMode (types.hpp:185) and ReduceOp (types.hpp:270) numbering. */
enum { TCG_READ = 0, TCG_WRITE = 1, TCG_READ_WRITE = 2, TCG_INCREMENT = 3 };
enum { TCG_RED_NONE = -1, TCG_RED_SUM = 0, TCG_RED_MIN = 1, TCG_RED_MAX = 2 };
/* ExecMode kinds (runtime.hpp:25-35). TCG_TILED runs the reference tile
 * plan (tile_sizes as in the reference, 0 = GPU sizer) on the L2-resident
 * executor; TCG_WINDOWED selects the shared-memory windowed executor
 * (tile_sizes = column block / stream tile bounds, 0 = sizer); TCG_TILED_AUTO
 * times the executors per chain and keeps the fastest. TCG_STREAM runs the
 * fused streaming executor: one kernel per chain signature, generated and
 * compiled for sm_100a at run time. */
enum { TCG_UNTILED = 0, TCG_TILED = 1, TCG_TILED_AUTO = 2, TCG_WINDOWED = 3, TCG_STREAM = 4 };

typedef struct tcg_runtime tcg_runtime;

typedef struct tcg_config {
  int32_t threads;                    /* RuntimeConfig::threads (reference sizer input) */
  int64_t skew_allowance;             /* RuntimeConfig::skew_allowance, default 16 */
  int64_t cache_bytes;                /* RuntimeConfig::cache_bytes, default 8 MiB */
  int32_t flush_whole_queue_on_fetch; /* RuntimeConfig::flush_whole_queue_on_fetch */
  int32_t stream_segments;            /* B200: CTA segments along the slowest dim, 0 = auto */
} tcg_config;

size_t tcg_last_error(char* buf, size_t n);
int tcg_abi_version(void);

int tcg_runtime_new(int dim, const tcg_config* cfg /* NULL = defaults */, tcg_runtime** out);
void tcg_runtime_free(tcg_runtime* rt);

/* pts: 3 int64 per point (unused coordinates 0). */
int tcg_declare_stencil(tcg_runtime* rt, int npts, const int64_t* pts, int32_t* out_id);
int tcg_declare_field(tcg_runtime* rt, const char* name, const int64_t logical[6], int32_t* out_id);
int tcg_alloc_range(tcg_runtime* rt, int32_t ds, int64_t out[6]);

/* args: 3 int32 per argument {dataset, stencil, access mode}.
 * red_op: TCG_RED_NONE or a ReduceOp; out_handle receives the reduction
 * handle (-1 when none). params: scalar parameter block of the body. */
int tcg_par_loop(tcg_runtime* rt, int32_t kernel_id, int32_t body, const int64_t range[6], int nargs,
                 const int32_t* args, int red_op, int nparams, const double* params, int32_t* out_handle);

/* mode: TCG_UNTILED, TCG_TILED / TCG_WINDOWED (tile_sizes used), TCG_TILED_AUTO. */
int tcg_flush(tcg_runtime* rt, int mode, const int64_t tile_sizes[3]);
int tcg_flush_default(tcg_runtime* rt);
int tcg_set_default_mode(tcg_runtime* rt, int mode, const int64_t tile_sizes[3]);
int tcg_fetch_reduction(tcg_runtime* rt, int32_t handle, double* out);
int tcg_pending_loops(tcg_runtime* rt, int64_t* out);
/* Step templates: the par_loop / periodic_fill calls made between
 * tcg_record_begin and tcg_record_end are kept (they are enqueued normally
 * too); tcg_replay issues the same calls again through par_loop, as the
 * reference's C++ apps do every step (apps.cpp:59-130, :163-254), in one
 * crossing of the binding. params (may be NULL) replaces the kernels' scalar
 * parameters in call order. Returns the new reduction handles in call order. */
/* Sum reductions folded in the reference's order for RuntimeConfig::threads =
 * workers (executor.cpp:55-61, :141-144, :175-176): such chains run untiled,
 * every point's contribution is captured and summed sequentially over the
 * reference's static spans, partials folded in worker order. 0 = fast fold. */
int tcg_set_reduction_order(tcg_runtime* rt, int workers);
int tcg_record_begin(tcg_runtime* rt);
int tcg_record_end(tcg_runtime* rt, int32_t* id);
int tcg_replay(tcg_runtime* rt, int32_t id, const double* params, int64_t nparams, int32_t* handles,
               int64_t max_handles, int64_t* nhandles);

int tcg_get(tcg_runtime* rt, int32_t ds, const int64_t p[3], double* out);
int tcg_put(tcg_runtime* rt, int32_t ds, const int64_t p[3], double v);
int tcg_fill_logical(tcg_runtime* rt, int32_t ds, double v);
/* Periodic ghost layers (depth <= pad) of n fields, all dimensions. No
 * reference counterpart (the reference has no periodic neighbours,
 * dist.cpp:135-140); c5 needs it. The call is
 * RECORDED in the lazy queue like a loop: at flush the chain is rewritten so
 * its inputs are wrapped once, to the chain's accumulated stencil reach, and
 * the producing loops run over ranges extended into the ghost layers (the
 * deep-halo scheme of dist.cpp:617-689 applied to the wrap-around neighbour).
 * The RK step of c5 stays one chain. After such a chain only the logical box
 * of a field is defined. tcg_set_periodic_flush(rt, 1) restores the eager
 * form: flush, then copy the opposite side into the ghost layers. */
int tcg_periodic_fill(tcg_runtime* rt, int n, const int32_t* ds, int64_t depth);
int tcg_set_periodic_flush(tcg_runtime* rt, int flush_each);
/* Periodic box on a rank grid (before tcg_set_rank_grid / tcg_set_process_rank):
 * the ghost layers join the decomposed domain (owned by the end ranks) and the
 * wrap along the split (slowest) dimension is one slab message between the
 * end ranks per chain -- a self-exchange at one rank. */
int tcg_set_periodic_domain(tcg_runtime* rt, int on);
/* Host-only: the rewrite of the pending chain around its periodic marks
 * (extended loop ranges, datasets wrapped before the chain); consumed. */
int tcg_periodic_plan_pending(tcg_runtime* rt, char* buf, int64_t n, int64_t* needed);
/* host: dense fp64 over the allocation range, dim 0 fastest. */
int tcg_upload(tcg_runtime* rt, int32_t ds, const double* host);
int tcg_download(tcg_runtime* rt, int32_t ds, double* host);
int tcg_synchronize(tcg_runtime* rt);
/* Box forms: host dense over box (inside the allocation); in a distributed
 * runtime only the parts this process's ranks hold move. tcg_local_box: the
 * part of the allocation this process holds (what it must upload). */
int tcg_upload_box(tcg_runtime* rt, int32_t ds, const double* host, const int64_t box[6]);
int tcg_download_box(tcg_runtime* rt, int32_t ds, double* host, const int64_t box[6]);
int tcg_local_box(tcg_runtime* rt, int32_t ds, int64_t out[6]);

/* Text outputs: write up to n bytes (NUL-terminated) and store the full
 * length + 1 in *needed. */
int tcg_report_text(tcg_runtime* rt, char* buf, int64_t n, int64_t* needed);
int tcg_plan_pending(tcg_runtime* rt, const int64_t tile_sizes[3], char* buf, int64_t n, int64_t* needed);
int tcg_rank_plans_pending(tcg_runtime* rt, const int32_t grid[3], const int64_t tile_sizes[3], char* buf,
                           int64_t n, int64_t* needed);
/* GPU windowed plan of the pending chain (consumed), summary text. */
int tcg_gpu_plan_pending(tcg_runtime* rt, int mode, const int64_t tile_sizes[3], char* buf, int64_t n,
                         int64_t* needed);
int tcg_signature_pending(tcg_runtime* rt, uint64_t* out);
/* Streaming executor (the B200 form of execute_plan over the skewed tile
 * plan, executor.cpp:209-250 / planner.cpp:55-208). cfg: {threads per CTA,
 * points per thread x, points per thread y, threads along x, stream segments,
 * loops per kernel, min CTAs per SM, L2 prefetch rows}; 0 (prefetch -1) =
 * sizer. tcg_stream_plan_pending consumes the pending chain and returns the
 * plan summary; what & 1: also compile every kernel with NVRTC (no GPU
 * needed) and append the compiler log; what & 2: append the sources. */
int tcg_set_stream_choice(tcg_runtime* rt, const int32_t cfg[8]);
int tcg_stream_plan_pending(tcg_runtime* rt, int what, char* buf, int64_t n, int64_t* needed);

/* Distribution. grid: ranks per dimension (slabs: {1,P,1}
 * in 2D, {1,1,P} in 3D). tcg_set_rank_grid hosts every rank in this process
 * on the current GPU; tcg_set_process_rank hosts rank `rank` here and reaches
 * the others through NCCL: rank 0 calls tcg_comm_unique_id and shares the 128
 * bytes with every process (e.g. torch.distributed broadcast) before all call
 * tcg_set_process_rank. Data already uploaded is carried into the rank fields.
 * In a multi-process job, get() is collective (every process calls it) and
 * download() fills the regions this process's rank holds. */
int tcg_set_rank_grid(tcg_runtime* rt, const int32_t grid[3]);
int tcg_comm_unique_id(uint8_t out[128]);
/* Owned box of a rank (decompose, dist.cpp:142-177, over the fields' hull). */
int tcg_rank_owned(tcg_runtime* rt, int32_t rank, int64_t out[6]);
int tcg_set_process_rank(tcg_runtime* rt, const int32_t grid[3], int32_t rank, const uint8_t id[128]);
/* Text: "rank=", "loop rank= l= lo hi ...", "msg src= dst= ds= dim= dir= box lo hi ..." lines. */
int tcg_dist_schedule_pending(tcg_runtime* rt, char* buf, int64_t n, int64_t* needed);
int tcg_auto_tile_size(int dim, int64_t cache_bytes, int32_t threads, int64_t bytes_per_point,
                       const int64_t extent[6], int64_t out[3]);
/* Selects the CUDA device for runtimes created afterwards on this thread
 * (one process per GPU: pass LOCAL_RANK). */
int tcg_select_device(int device);
/* Name, SM count, shared memory, L2 of the executor device (initialises CUDA). */
int tcg_device_info(char* name, size_t n, int32_t* num_sms, int64_t* smem_optin, int64_t* l2_bytes);
/* Launch count and the CUDA stream of a runtime's executor (for timing). */
int tcg_launches(tcg_runtime* rt, int64_t* out);
int tcg_stream(tcg_runtime* rt, void** out);
int tcg_body_known(int32_t body);
/* Device-time instrumentation of the executor kernels (CUDA events on the
 * executor stream). tcg_kernel_timing synchronizes, returns the accumulated
 * milliseconds and launch counts of k_tiled and k_untiled since the last call,
 * and resets them. */
int tcg_set_timing(tcg_runtime* rt, int on);
int tcg_kernel_timing(tcg_runtime* rt, double* tiled_ms, int64_t* tiled_launches, double* untiled_ms,
                      int64_t* untiled_launches);

#ifdef __cplusplus
}
#endif
#endif /* TILECHAIN_B200_H */
