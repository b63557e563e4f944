// Device-side support of the streaming executor (kernels are generated and
// compiled at run time, tcg_stream.cpp / tcg_jit.cpp): second-buffer
// bookkeeping for ping-ponged datasets, reduction scratch, launches.
#include "../host/tcg_jit.hpp"
#include "tcg_common.cuh"

namespace tcg {

namespace {
int64_t lo3(const Range& r, int d) { return d < r.dim() ? r.start(d) : 0; }
int64_t ext3(const Range& r, int d) { return d < r.dim() ? r.extent(d) : 1; }

}  // namespace

void DeviceExec::mark_written(int f, const Range& box) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  if (!b->alt_synced || box.empty()) return;
  const Range c = box.intersect(b->alloc);
  if (c.empty()) return;
  for (const Range& r : b->dirty)
    if (r.contains(c)) return;
  b->dirty.push_back(c);
  if (b->dirty.size() > 24) {
    Range h = b->dirty[0];
    for (const Range& r : b->dirty) h = h.hull(r);
    b->dirty.assign(1, h);
  }
}

void DeviceExec::mark_chain_writes(const DevChain& ch) {
  for (const DevLoop& L : ch.loops)
    for (int a = 0; a < L.nargs; ++a) {
      if (L.args[a].mode == 0) continue;  // read
      const int f = ch.dat_ids.at(static_cast<size_t>(L.args[a].dat));
      Range r(ch.dim);
      for (int d = 0; d < ch.dim; ++d) r.set_raw(d, L.range[d][0], L.range[d][1]);
      mark_written(f, r);
    }
}

void DeviceExec::sync_alt(int f, const Range& keep) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  double* cur = b->mem[b->cur];
  double*& alt = b->mem[1 - b->cur];
  if (!alt) TCG_CK(cudaMalloc(&alt, b->bytes));
  if (!b->alt_synced) {
    TCG_CK(cudaMemcpyAsync(alt, cur, b->bytes, cudaMemcpyDeviceToDevice, st));
    b->alt_synced = true;
    b->dirty.clear();
    return;
  }
  const size_t pitch = static_cast<size_t>(b->py) * 8;
  for (const Range& box : b->dirty) {
    if (keep.contains(box) || box.empty()) continue;
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(cur, pitch, pitch, static_cast<size_t>(b->ny));
    p.dstPtr = make_cudaPitchedPtr(alt, pitch, pitch, static_cast<size_t>(b->ny));
    const cudaPos pos = make_cudaPos(static_cast<size_t>(lo3(box, 0) - b->x0) * 8,
                                     static_cast<size_t>(lo3(box, 1) - lo3(b->alloc, 1)),
                                     static_cast<size_t>(lo3(box, 2) - lo3(b->alloc, 2)));
    p.srcPos = pos;
    p.dstPos = pos;
    p.extent = make_cudaExtent(static_cast<size_t>(ext3(box, 0)) * 8, static_cast<size_t>(ext3(box, 1)),
                               static_cast<size_t>(ext3(box, 2)));
    p.kind = cudaMemcpyDeviceToDevice;
    TCG_CK(cudaMemcpy3DAsync(&p, st));
  }
  b->dirty.clear();
}

void DeviceExec::commit_alt(int f, const Range& box) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  b->cur ^= 1;
  b->dirty.assign(1, box.intersect(b->alloc));
  b->alt_synced = true;
}

void DeviceExec::stream_red_buffers(size_t npart, size_t nout, double** part, double** out, unsigned** ticket) {
  if (npart > st_part_n_) {
    if (st_part_) TCG_CK(cudaFree(st_part_));
    st_part_n_ = std::max(npart, st_part_n_ * 2);
    TCG_CK(cudaMalloc(&st_part_, st_part_n_ * sizeof(double)));
  }
  if (nout > st_out_n_) {
    if (st_out_) {
      TCG_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
      TCG_CK(cudaFree(st_out_));
    }
    st_out_n_ = std::max<size_t>(std::max(nout, st_out_n_ * 2), 64);
    TCG_CK(cudaMalloc(&st_out_, st_out_n_ * sizeof(double)));
  }
  if (!st_ticket_) {
    TCG_CK(cudaMalloc(&st_ticket_, sizeof(unsigned) * 64));
    TCG_CK(cudaMemsetAsync(st_ticket_, 0, sizeof(unsigned) * 64, static_cast<cudaStream_t>(stream_)));
  }
  *part = st_part_;
  *out = st_out_;
  *ticket = st_ticket_;
}

void DeviceExec::launch_stream(void* fn, int64_t grid, int nt, int smem, const void* args, size_t bytes) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  void* e0 = nullptr;
  if (timing_) {
    e0 = take_event();
    TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e0), st));
  }
  jit_launch(fn, grid, nt, smem, stream_, args, bytes);
  if (timing_) {
    void* e1 = take_event();
    TCG_CK(cudaEventRecord(static_cast<cudaEvent_t>(e1), st));
    ev_tiled_.emplace_back(e0, e1);
  }
  ++launches_;
}

double* DeviceExec::slab_ptr(int f, int64_t s) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  const int d = b->alloc.dim() - 1;
  if (s < b->alloc.start(d) || s > b->alloc.end(d)) throw AccessError("slab_ptr: slab outside the allocation");
  const int64_t pitch = d == 2 ? b->pz : (d == 1 ? b->py : 1);
  return b->mem[b->cur] + (s - b->alloc.start(d)) * pitch;
}

size_t DeviceExec::slab_count(int f, int64_t s0, int64_t s1) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  const int d = b->alloc.dim() - 1;
  const int64_t pitch = d == 2 ? b->pz : (d == 1 ? b->py : 1);
  return static_cast<size_t>(std::max<int64_t>(0, s1 - s0) * pitch);
}

bool DeviceExec::same_cross_section(int fa, int fb) const {
  const Buf* a = fields_.at(static_cast<size_t>(fa));
  const Buf* b = fields_.at(static_cast<size_t>(fb));
  if (a->alloc.dim() != b->alloc.dim() || a->alloc.dim() < 2) return false;
  for (int d = 0; d + 1 < a->alloc.dim(); ++d)
    if (a->alloc.start(d) != b->alloc.start(d) || a->alloc.end(d) != b->alloc.end(d)) return false;
  return a->x0 == b->x0 && a->py == b->py && (a->alloc.dim() < 3 || a->pz == b->pz);
}

void DeviceExec::note_slab_write(int f, int64_t s0, int64_t s1) {
  Buf* b = fields_.at(static_cast<size_t>(f));
  Range box = b->alloc;
  box.set_raw(b->alloc.dim() - 1, s0, s1);
  mark_written(f, box);
}

void DeviceExec::copy_slabs(int f_dst, int f_src, int64_t s0, int64_t s1) {
  if (s1 <= s0) return;
  if (!same_cross_section(f_dst, f_src)) throw AccessError("copy_slabs: the fields differ in a faster dimension");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  // Rank r of a single-process multi-device run lives on device r % ndev;
  // here both ranks share this executor's device, and the peer copy is a
  // device-to-device copy.
  TCG_CK(cudaMemcpyPeerAsync(slab_ptr(f_dst, s0), device_, slab_ptr(f_src, s0), device_, slab_count(f_src, s0, s1) * sizeof(double), st));
  note_slab_write(f_dst, s0, s1);
}

void DeviceExec::copy_slabs_shift(int f_dst, int64_t dst_s0, int f_src, int64_t src_s0, int64_t n) {
  if (n <= 0) return;
  if (!same_cross_section(f_dst, f_src)) throw AccessError("copy_slabs_shift: the fields differ in a faster dimension");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  TCG_CK(cudaMemcpyPeerAsync(slab_ptr(f_dst, dst_s0), device_, slab_ptr(f_src, src_s0), device_,
                             slab_count(f_src, src_s0, src_s0 + n) * sizeof(double), st));
  note_slab_write(f_dst, dst_s0, dst_s0 + n);
}

void DeviceExec::read_device(double* host, const double* dev, size_t n) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  if (n > host_stage_n_) {
    if (host_stage_) {
      TCG_CK(cudaStreamSynchronize(st));
      TCG_CK(cudaFreeHost(host_stage_));
    }
    host_stage_n_ = std::max<size_t>(n, 64);
    TCG_CK(cudaMallocHost(&host_stage_, host_stage_n_ * sizeof(double)));
  }
  TCG_CK(cudaMemcpyAsync(host_stage_, dev, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  TCG_CK(cudaStreamSynchronize(st));
  std::memcpy(host, host_stage_, n * sizeof(double));
}

}  // namespace tcg
