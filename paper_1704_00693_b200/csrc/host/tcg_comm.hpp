// Inter-process transport of the distributed executor: one NCCL communicator
// per runtime (one process per GPU), driven from the runtime's single control
// thread on the executor stream. Halo messages are grouped ncclSend/ncclRecv
// (point-to-point over NVLink/NVSwitch); reduction partials are all-gathered
// and folded in rank order on the host, as DistContext folds ranks in rank-id
// order (dist.cpp:657-672).
//
// NCCL is loaded with dlopen("libnccl.so.2") when the first communicator is
// created, so a process that already imported torch reuses torch's NCCL.
#pragma once
#include <cstddef>
#include <cstdint>

namespace tcg {

constexpr int kCommIdBytes = 128;  // NCCL_UNIQUE_ID_BYTES

class Comm {
 public:
  static void unique_id(uint8_t out[kCommIdBytes]);
  Comm(int nranks, int rank, const uint8_t id[kCommIdBytes]);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;

  int nranks() const { return nranks_; }
  int rank() const { return rank_; }
  void group_start();
  void group_end();
  void send(const double* dev, size_t n, int peer, void* stream);
  void recv(double* dev, size_t n, int peer, void* stream);
  void all_gather(const double* dev_send, double* dev_recv, size_t n, void* stream);
  void broadcast(double* dev, size_t n, int root, void* stream);

 private:
  void* comm_ = nullptr;
  int nranks_ = 1, rank_ = 0;
};

}  // namespace tcg
