// NCCL transport (see host/tcg_comm.hpp).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../host/tcg_comm.hpp"
#include "../host/tcg_types.hpp"

namespace tcg {

namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(sym("ncclBroadcast"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw CudaError(err);
  return n;
}

void ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

void Comm::unique_id(uint8_t out[kCommIdBytes]) {
  ncclUniqueId id;
  ck(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, kCommIdBytes);
}

Comm::Comm(int nranks, int rank, const uint8_t idb[kCommIdBytes]) : nranks_(nranks), rank_(rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("Comm: rank out of range");
  ncclUniqueId id;
  std::memcpy(id.internal, idb, kCommIdBytes);
  ncclComm_t c = nullptr;
  ck(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
  comm_ = c;
}

Comm::~Comm() {
  if (comm_) nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void Comm::group_start() { ck(nccl().group_start(), "ncclGroupStart"); }
void Comm::group_end() { ck(nccl().group_end(), "ncclGroupEnd"); }

void Comm::send(const double* dev, size_t n, int peer, void* stream) {
  ck(nccl().send(dev, n, ncclFloat64, peer, static_cast<ncclComm_t>(comm_), static_cast<cudaStream_t>(stream)),
     "ncclSend");
}

void Comm::recv(double* dev, size_t n, int peer, void* stream) {
  ck(nccl().recv(dev, n, ncclFloat64, peer, static_cast<ncclComm_t>(comm_), static_cast<cudaStream_t>(stream)),
     "ncclRecv");
}

void Comm::all_gather(const double* s, double* r, size_t n, void* stream) {
  ck(nccl().all_gather(s, r, n, ncclFloat64, static_cast<ncclComm_t>(comm_), static_cast<cudaStream_t>(stream)),
     "ncclAllGather");
}

void Comm::broadcast(double* dev, size_t n, int root, void* stream) {
  ck(nccl().broadcast(dev, dev, n, ncclFloat64, root, static_cast<ncclComm_t>(comm_),
                      static_cast<cudaStream_t>(stream)),
     "ncclBroadcast");
}

}  // namespace tcg
