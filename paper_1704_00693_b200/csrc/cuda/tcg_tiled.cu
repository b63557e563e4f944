// Launch glue of the windowed tiled executor (kernel: tcg_tiled.cuh).
#include "tcg_common.cuh"

namespace tcg {

namespace {

// ---------------------------------------------------------------------------
// Windowed tiled executor.
#include "tcg_tiled.cuh"


// Launch of k_tiled<DIM, NT>: NT = 512 / (CTAs per SM) threads.
template <int DIM, int NT>
void launch_tiled_nt(const DevTiledPlan& P, int64_t smem, cudaStream_t st) {
  TCG_CK(cudaFuncSetAttribute(tiled::k_tiled<DIM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem)));
  tiled::k_tiled<DIM, NT><<<dim3(static_cast<unsigned>(P.nctas)), dim3(NT), smem, st>>>(P);
}

template <int DIM>
void launch_tiled(const DevTiledPlan& P, int threads, int64_t smem, cudaStream_t st) {
  if (threads == 512)
    launch_tiled_nt<DIM, 512>(P, smem, st);
  else if (threads == 256)
    launch_tiled_nt<DIM, 256>(P, smem, st);
  else
    throw InvalidArgument("tiled executor: " + std::to_string(threads) + " threads per CTA not built");
}

}  // namespace

int64_t DeviceExec::window_budget_doubles(int nloops, int nred, int ctas_per_sm) const {
  const int k = std::max(1, ctas_per_sm);
  const int threads = kTiledThreads / k;
  // Per-CTA share of the SM (1 KB of every CTA's share is reserved by the driver).
  const int64_t per_block = std::min<int64_t>(info_.smem_optin, info_.smem_per_sm / k - 1024);
  const int64_t fixed = static_cast<int64_t>(sizeof(tiled::Shared)) + 512 + 256 +
                        static_cast<int64_t>(nloops) * (kMaxArgs * 16 + 6 * 4 + static_cast<int64_t>(sizeof(DevLoop))) +
                        static_cast<int64_t>(nred) * threads * 8;
  return std::max<int64_t>(0, (per_block - fixed) / 8);
}

DeviceExec::PlanBufs* DeviceExec::plan_bufs(const GpuTiledPlan& gp, uint64_t key) {
  for (auto& pb : plan_cache_)
    if (pb.first == key) return pb.second;
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  auto* pb = new PlanBufs;
  const size_t a = align_up<char>(gp.ctas.size() * sizeof(DevCta));
  const size_t b = align_up<char>(std::max<size_t>(1, gp.boxes.size()) * 4);
  const size_t c = align_up<char>(std::max<size_t>(1, gp.win.size()) * 4);
  const size_t d = align_up<char>(std::max<size_t>(1, gp.wboxes.size()) * 4);
  TCG_CK(cudaMalloc(&pb->mem, a + b + c + d));
  char* m = static_cast<char*>(pb->mem);
  pb->ctas = reinterpret_cast<DevCta*>(m);
  pb->boxes = reinterpret_cast<int32_t*>(m + a);
  pb->win = reinterpret_cast<int32_t*>(m + a + b);
  pb->wboxes = reinterpret_cast<int32_t*>(m + a + b + c);
  TCG_CK(cudaMemcpyAsync(pb->ctas, gp.ctas.data(), gp.ctas.size() * sizeof(DevCta), cudaMemcpyHostToDevice, st));
  if (!gp.boxes.empty()) TCG_CK(cudaMemcpyAsync(pb->boxes, gp.boxes.data(), gp.boxes.size() * 4, cudaMemcpyHostToDevice, st));
  if (!gp.win.empty()) TCG_CK(cudaMemcpyAsync(pb->win, gp.win.data(), gp.win.size() * 4, cudaMemcpyHostToDevice, st));
  if (!gp.wboxes.empty())
    TCG_CK(cudaMemcpyAsync(pb->wboxes, gp.wboxes.data(), gp.wboxes.size() * 4, cudaMemcpyHostToDevice, st));
  TCG_CK(cudaStreamSynchronize(st));
  plan_cache_.emplace_back(key, pb);
  if (plan_cache_.size() > 64) {
    cudaFree(plan_cache_.front().second->mem);
    delete plan_cache_.front().second;
    plan_cache_.erase(plan_cache_.begin());
  }
  return pb;
}

void DeviceExec::run_tiled(const DevChain& ch, const GpuTiledPlan& gp, uint64_t key, double* red_out) {
  mark_chain_writes(ch);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  PlanBufs* pb = plan_bufs(gp, key);
  void* scratch = ensure_scratch(chain_bytes(ch));
  const ChainDev cd = upload_chain(ch, scratch, st, &scratch_hash_);
  DevTiledPlan P{};
  P.dim = gp.dim;
  P.nloops = gp.nloops;
  P.ndat = gp.ndat;
  P.nred = gp.nred;
  P.nctas = static_cast<int32_t>(gp.ctas.size());
  P.smem_doubles = static_cast<int32_t>((gp.smem_doubles + 1) / 2 * 2);
  P.prefetch = gp.prefetch ? 1 : 0;
  P.ctas = pb->ctas;
  P.boxes = pb->boxes;
  P.win = pb->win;
  P.wboxes = pb->wboxes;
  P.loops = cd.loops;
  P.params = cd.params;
  P.stencils = cd.st;
  // Device fields come from the lowered chain (the target's field map: the
  // undistributed fields or one rank's); the plan only knows chain slots.
  if (ch.dat_ids.size() != static_cast<size_t>(gp.ndat))
    throw PlanError("tiled executor: chain and plan disagree on the dataset count");
  for (int k = 0; k < gp.ndat; ++k) {
    P.dats[k] = gp.dats[static_cast<size_t>(k)];
    const int f = ch.dat_ids[static_cast<size_t>(k)];
    P.src[k] = view(f, false);
    P.dst[k] = gp.dats[static_cast<size_t>(k)].pingpong ? view(f, true) : P.src[k];
  }
  for (int r = 0; r < gp.nred && r < kMaxRed; ++r) P.red_op[r] = ch.red_op[static_cast<size_t>(r)];
  if (gp.nred > 0) P.red_partials = ensure_partials(static_cast<size_t>(gp.nred) * gp.ctas.size());
  P.red_out = red_dev_;
  const int64_t smem = static_cast<int64_t>(P.smem_doubles) * 8 +
                       static_cast<int64_t>(gp.nloops) * (sizeof(DevLoop) + kMaxArgs * 16 + 6 * 4) +
                       static_cast<int64_t>(gp.nred) * gp.threads * 8;
  if (smem > info_.smem_optin) throw PlanError("tiled executor: shared memory request exceeds the device limit");
  void* e0 = nullptr;
  if (timing_) {
    e0 = take_event();
    TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e0), st));
  }
  if (gp.dim == 1)
    launch_tiled<1>(P, gp.threads, smem, st);
  else if (gp.dim == 2)
    launch_tiled<2>(P, gp.threads, smem, st);
  else
    launch_tiled<3>(P, gp.threads, smem, st);
  TCG_CK(cudaGetLastError());
  if (timing_) {
    void* e1 = take_event();
    TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e1), st));
    ev_tiled_.emplace_back(e0, e1);
  }
  ++launches_;
  for (int k = 0; k < gp.ndat; ++k)
    if (gp.dats[static_cast<size_t>(k)].pingpong) swap(ch.dat_ids[static_cast<size_t>(k)]);
  for (int r = 0; r < gp.nred; ++r) {
    k_fold<<<1, 1024, 0, st>>>(P.red_partials + static_cast<int64_t>(r) * P.nctas, P.nctas, P.red_op[r], red_dev_ + r);
    TCG_CK(cudaGetLastError());
    ++launches_;
  }
  if (gp.nred > 0) {
    read_reductions(red_out, gp.nred);
  }
}

}  // namespace tcg
