// Front door of the B200 stencil-chain executor: the reference's Runtime API
// (proj/core/include/tilechain/runtime.hpp:44-135) with the same lazy-queue
// semantics, rebuilt over device-resident fields and the CUDA executors.
//   declare_stencil / declare_field        runtime.cpp:16-33 (pad rule kept)
//   par_loop (validation, lazy enqueue)    runtime.cpp:35-92
//   take_pending / flush / execute_chain   runtime.cpp:94-151
//   fetch_reduction (prefix flush)         runtime.cpp:164-197
//   get / put / fill_logical               runtime.cpp:199-212
// Differences by design: fields live in HBM (the host never holds a copy),
// kernels are registry bodies, and ExecMode::tiled / tiled_auto run the
// windowed CTA executor.
#pragma once
#include <map>
#include <memory>
#include <unordered_set>

#include "tcg_comm.hpp"
#include "tcg_dist.hpp"
#include "tcg_exec.hpp"
#include "tcg_gpuplan.hpp"
#include "tcg_periodic.hpp"
#include "tcg_plan.hpp"
#include "tcg_stream.hpp"

namespace tcg {

struct RuntimeConfig {
  int threads = 1;                          // kept for API parity (CPU sizer input)
  int64_t skew_allowance = 16;              // runtime.hpp:17
  int64_t cache_bytes = int64_t{8} << 20;   // runtime.hpp:19 (reference sizer only)
  bool flush_whole_queue_on_fetch = false;  // runtime.hpp:22
  int stream_segments = 0;                  // GPU: CTA segments along the stream dim (0 = auto)
};

struct ExecMode {
  // Untiled / Tiled / TiledAuto are the reference's modes (runtime.hpp:25-35).
  // Tiled runs the reference tile plan with the L2-resident executor
  // (tile_sizes as in the reference; 0 = GPU sizer). Windowed is the
  // shared-memory windowed executor (tile_sizes = column block / stream tile
  // upper bounds; 0 = sizer).
  // Stream is the fused streaming executor (generated per chain, DESIGN.md
  // §3.2); TiledAuto times untiled and stream per chain signature.
  enum class Kind : uint8_t { Untiled = 0, Tiled = 1, TiledAuto = 2, Windowed = 3, Stream = 4 };
  Kind kind = Kind::Untiled;
  std::array<int64_t, kMaxDims> tile_sizes{0, 0, 0};
  static ExecMode untiled() { return {}; }
  static ExecMode tiled(const std::array<int64_t, kMaxDims>& ts) { return {Kind::Tiled, ts}; }
  static ExecMode tiled_auto() { return {Kind::TiledAuto, {0, 0, 0}}; }
  static ExecMode windowed(const std::array<int64_t, kMaxDims>& ts) { return {Kind::Windowed, ts}; }
  static ExecMode stream() { return {Kind::Stream, {0, 0, 0}}; }
};

struct LoopExecStats {
  int32_t loop_id = 0;
  int64_t points = 0;
  int64_t bytes_moved = 0;
};

// executor.hpp:57-80 plus the GPU plan shape.
struct ExecutionReport {
  bool tiled = false;
  bool distributed = false;
  bool plan_cache_hit = false;
  int dim = 1;
  std::array<int64_t, kMaxDims> tile_sizes{0, 0, 0};
  std::array<int64_t, kMaxDims> max_skew{0, 0, 0};
  int64_t tiles_executed = 0;
  int64_t plan_constructions = 0;
  double plan_seconds = 0;
  double exec_seconds = 0;
  double total_seconds = 0;
  std::vector<LoopExecStats> loops;
  int64_t halo_messages = 0, halo_bytes = 0, halo_exchanges = 0;
  // GPU specifics
  int64_t launches = 0;
  int64_t ctas = 0;
  int64_t subchains = 0;
  int64_t computed_points = 0;
  int64_t l2_syncs = 0;  // grid barriers of the L2-tiled executor
  std::string executor = "untiled";  // executor that ran the chain (tiled_auto may pick either)
  std::array<int, kMaxDims> cta_grid{1, 1, 1};
  int64_t total_points() const;
  int64_t total_bytes_moved() const;
  std::string to_text() const;
};

class Runtime {
 public:
  Runtime(int dim, RuntimeConfig cfg = {});
  ~Runtime();

  StencilId declare_stencil(const std::string& name, std::vector<Point> offsets);
  DatasetId declare_field(const std::string& name, const Range& logical, int elem_bytes = 8);

  ReductionHandle par_loop(KernelHandle kernel, const Range& range, std::vector<ArgSpec> args,
                           std::optional<ReduceOp> reduction = std::nullopt);

  ExecutionReport flush(const ExecMode& mode);
  ExecutionReport flush() { return flush(default_mode_); }
  void set_default_mode(const ExecMode& m) { default_mode_ = m; }
  const ExecMode& default_mode() const { return default_mode_; }

  double fetch_reduction(ReductionHandle h);

  double get(DatasetId ds, const Point& p);
  void put(DatasetId ds, const Point& p, double v);
  void fill_logical(DatasetId ds, double v);
  // Periodic boundary: copy the opposite side of the logical box into the
  // ghost layers (depth <= pad) of every listed field, dimension by
  // dimension so edges and corners wrap too. Flushes first. (The reference
  // has no periodic support; c5 needs it.)
  void periodic_fill(const std::vector<DatasetId>& ds, int64_t depth);
  // true: periodic_fill flushes and wraps at once (the round-1 behaviour);
  // false (default): it records a PeriodicMark in the queue and the chain is
  // rewritten at flush (tcg_periodic.hpp) -- one wrap per chain.
  void set_periodic_flush(bool v) { periodic_flush_ = v; }
  // Periodic box on a rank grid (call before set_rank_grid / set_process_rank):
  // the decomposed domain is the fields' logical hull dilated by the smallest
  // field pad, so the ghost layers belong to the end ranks, the rewritten
  // chain's extended loops stay inside the domain, and the wrap along the
  // split (slowest) dimension is a slab message between the end ranks -- the
  // "self-exchange" at one rank. The grid may split the slowest dimension only.
  void set_periodic_domain(bool v);
  bool periodic_domain() const { return periodic_domain_; }
  // Order-matched Sum reductions: chains with a Sum reduction run on the
  // untiled executor and fold in the reference's order for a pool of
  // `workers` threads (executor.cpp:55-61 static spans, :141-144 sequential
  // per-worker partials, :175-176 worker-order fold), so a c4 residual
  // history follows RefRuntime(threads = workers, untiled) bit for bit.
  // 0 (default): the fast tree fold.
  void set_reduction_order(int workers);
  int reduction_order() const { return red_workers_; }
  // Bulk host <-> device copies of a whole allocation (dense, dim 0 fastest,
  // the reference Field layout, field.cpp:22-26). Flush first.
  void upload(DatasetId ds, const double* host);
  void download(DatasetId ds, double* host);
  // Box forms: `host` is dense over `box` (inside the allocation). In a
  // distributed runtime only the parts held by this process's ranks move.
  void upload_box(DatasetId ds, const double* host, const Range& box);
  void download_box(DatasetId ds, double* host, const Range& box);
  // The part of ds's allocation this process holds: the whole allocation,
  // or the hull of its ranks' allocations (clipped to the field's).
  Range local_box(DatasetId ds);

  // Distribution over a rank grid (reference Runtime::set_rank_grid,
  // runtime.hpp:77-81, runtime.cpp:213-222). set_rank_grid hosts every rank
  // in this process on this GPU (the reference's simulated ranks);
  // set_process_rank hosts one rank per process, messages over NCCL. Data
  // already on the device is carried over into the rank fields.
  void set_rank_grid(const std::array<int, kMaxDims>& grid);
  void set_process_rank(const std::array<int, kMaxDims>& grid, int rank, const uint8_t id[kCommIdBytes]);
  bool distributed() const { return grid_set_; }
  const RankLayout& rank_layout();
  // Host-only: the distribution schedule of the pending chain (consumed; its
  // writes are recorded as if it had run). Needs a rank grid, no GPU.
  DistSchedule schedule_pending();

  // Host-side step recording (the role of the reference's C++ apps,
  // apps.cpp:59-130 / :163-254, which re-issue the same par_loop calls every
  // step): between record_begin and record_end every par_loop / periodic_fill
  // call is also kept as a template; replay(id) issues the same calls again
  // through par_loop (validation, lazy queue, new reduction handles) without
  // crossing the language binding once per loop. `params`, if given, replaces
  // the kernels' scalar parameters in call order (nparams values).
  void record_begin();
  int record_end();
  std::vector<ReductionHandle> replay(int id, const double* params = nullptr, size_t nparams = 0);

  size_t pending_loops() const { return pending_.size(); }
  LoopChain take_pending();
  const Range& alloc_range(DatasetId ds) const { return fields_.at(static_cast<size_t>(ds)).alloc; }
  const Range& logical_range(DatasetId ds) const { return fields_.at(static_cast<size_t>(ds)).logical; }
  size_t num_fields() const { return fields_.size(); }
  int dim() const { return dim_; }
  const RuntimeConfig& config() const { return cfg_; }
  const std::vector<Stencil>& stencils() const { return stencils_; }
  const ExecutionReport& last_report() const { return last_report_; }
  std::shared_ptr<const GpuTiledPlan> last_gpu_plan() const { return last_gpu_plan_; }
  std::shared_ptr<const StreamPlan> last_stream_plan() const { return last_stream_plan_; }
  void set_stream_choice(const StreamChoice& c) { stream_choice_ = c; }
  const StreamChoice& stream_choice() const { return stream_choice_; }
  // Host-only: the streaming plan (with generated sources) of the pending
  // chain, consumed; field geometry from the device layout rule.
  StreamPlan stream_plan_pending(const StreamDevice& sd);
  PlanCache& plan_cache() { return plan_cache_; }
  int64_t gpu_plan_constructions() const { return gpu_plan_builds_; }
  DeviceExec& device();
  bool device_ready() const { return dev_ != nullptr; }
  std::vector<FieldGeom> field_geoms() const;

 private:
  struct FieldRec {
    std::string name;
    Range logical, alloc;
    int64_t pad = 0;
    int dev = -1;
  };
  struct Slot {
    ReduceOp op = ReduceOp::Sum;
    double value = 0;
    bool ready = false;
    bool consumed = false;
  };

  // Where a chain executes: the undistributed fields or one rank's fields.
  struct Target {
    std::vector<int> dev;      // dataset -> device field index
    std::vector<Range> alloc;  // dataset -> allocation
    bool masked = false;       // reductions only over `mask` (the rank's owned box)
    Range mask;
  };
  struct Dist {
    RankLayout layout;
    std::vector<int> local;            // ranks hosted by this process
    std::vector<Target> targets;       // [rank]; filled for local ranks
    WriteHistory written;              // note_writes history (dist.cpp:590-602)
    uint64_t hist_version = 0;
    std::map<std::pair<uint64_t, uint64_t>, std::shared_ptr<const DistSchedule>> schedules;
    // Untiled (on-demand) per-loop schedules, per chain signature.
    std::map<uint64_t, std::vector<std::shared_ptr<const DistSchedule>>> untiled_schedules;
  };

  ExecutionReport execute_chain(LoopChain chain, const ExecMode& mode);
  ExecutionReport execute_distributed(LoopChain chain, const ExecMode& mode);
  std::vector<double> run_on(const LoopChain& chain, const ExecMode& mode, ExecutionReport& rep, const Target& t);
  void ensure_fields();
  Target whole_target() const;
  void ensure_dist();
  void drop_dist();
  std::shared_ptr<const DistSchedule> dist_schedule(const LoopChain& chain);
  void exchange(const DistSchedule& s, ExecutionReport& rep);
  void periodic_exchange(const std::vector<std::pair<DatasetId, int64_t>>& fills, ExecutionReport& rep);
  void poison_stale_halos(const LoopChain& chain);
  bool poison_ = false;  // TCG_POISON_HALOS=1 (debug tripwire, dist.cpp:546-586)
  int root_for(DatasetId ds, const Point& p);
  DevChain lower(const LoopChain& chain, const Target& t) const;
  void run_tiled(const LoopChain& chain, const ExecMode& mode, ExecutionReport& rep, const Target& t,
                 std::vector<double>& vals);
  void run_l2(const LoopChain& chain, const ExecMode& mode, ExecutionReport& rep, const Target& t,
              std::vector<double>& vals);
  void run_stream(const LoopChain& chain, ExecutionReport& rep, const Target& t, std::vector<double>& vals);
  void check_pad(const LoopChain& chain, const Target& t) const;
  std::vector<StreamGeom> stream_geoms(const Target& t, bool from_device);
  StreamChoice stream_choice_;
  std::map<uint64_t, std::shared_ptr<const StreamPlan>> stream_plans_;
  std::shared_ptr<const StreamPlan> last_stream_plan_;
  struct L2Sub {
    size_t begin, end;  // loops [begin, end)
    int64_t ts;         // slowest-dim tile size
  };
  std::vector<L2Sub> l2_split(const LoopChain& chain, const Target& t) const;
  void store(const std::vector<ReductionHandle>& handles, const double* vals);

  int dim_;
  RuntimeConfig cfg_;
  std::vector<Stencil> stencils_;
  int64_t max_reach_ = 0;
  std::vector<FieldRec> fields_;
  std::vector<LoopRecord> pending_;
  std::vector<PeriodicMark> fill_marks_;  // recorded periodic fills of the pending loops
  struct RecordedCall {
    bool fill = false;
    KernelHandle kernel;
    Range range;
    std::vector<ArgSpec> args;
    std::optional<ReduceOp> reduction;
    std::vector<DatasetId> fill_ds;
    int64_t fill_depth = 0;
  };
  bool recording_ = false;
  std::vector<RecordedCall> record_cur_;
  std::vector<std::vector<RecordedCall>> recorded_;
  bool periodic_flush_ = false;
  bool periodic_domain_ = false;
  int red_workers_ = 0;
  std::unordered_set<uint64_t> body_sig_ok_;  // (body, declaration) pairs the probe accepted
  ExecMode default_mode_;
  std::vector<Slot> slots_;
  PlanCache plan_cache_;
  std::map<std::tuple<uint64_t, int64_t, int64_t, int64_t, int>, std::shared_ptr<const GpuTiledPlan>> gpu_plans_;
  int64_t gpu_plan_builds_ = 0;
  std::shared_ptr<const GpuTiledPlan> last_gpu_plan_;
  std::shared_ptr<const TilingPlan> last_plan_;
  struct L2Items {
    std::vector<DevItem> items;
    std::vector<int32_t> deps;
    std::array<int32_t, 3> reach{0, 0, 0};
  };
  std::map<const TilingPlan*, L2Items> l2_items_;
  std::map<uint64_t, std::vector<L2Sub>> l2_splits_;
  ExecutionReport last_report_;
  // tiled_auto: per chain signature, device time of the windowed-tiled and the
  // untiled executor (both bit-exact); later flushes use the faster one.
  // tiled_auto: per chain signature, device time of each executor candidate
  // (0 L2-tiled, 1 untiled, 2 windowed); all bit-exact, the fastest is kept.
  // Candidates: 0 L2-tiled, 1 untiled, 2 windowed, 3 stream; enabled by
  // auto_cands_ (default untiled + stream; TCG_AUTO_CANDS=0,1,2,3).
  static constexpr int kCand = 4;
  static constexpr int kAutoRuns = 3;  // timed runs per candidate (min kept)
  unsigned auto_cands_ = 0xA;
  struct AutoStat {
    int runs[kCand] = {0, 0, 0, 0};
    float ms[kCand] = {1e30f, 1e30f, 1e30f, 1e30f};
    bool fits[kCand] = {true, true, true, true};
    void* ev0 = nullptr;
    void* ev1 = nullptr;
    int pending = -1;    // candidate being timed
    bool saved = false;  // decision final (and written to TCG_AUTOTUNE_FILE)
    int best() const;
  };
  void save_autotune(AutoStat& as);
  std::map<uint64_t, AutoStat> auto_;
  std::string autotune_file_;
  std::array<int, kMaxDims> grid_{1, 1, 1};
  bool grid_set_ = false;
  int proc_rank_ = -1;  // >= 0: one rank per process
  std::unique_ptr<Dist> dist_;
  std::unique_ptr<DeviceExec> dev_;
  std::unique_ptr<Comm> comm_;  // destroyed before dev_ (declared after it)
};

}  // namespace tcg
