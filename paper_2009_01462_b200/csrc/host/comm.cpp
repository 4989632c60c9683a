// NCCL point-to-point transport (comm.hpp), opened with dlopen.
#include "comm.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "respar_b200.hpp"

namespace respar::b200 {

namespace {
// the public nccl.h ABI (nccl 2.x): ncclResult_t is an int enum, ncclComm_t a pointer,
// ncclUniqueId 128 bytes, ncclFloat32 == 7
struct UniqueId {
  char internal[kNcclUniqueIdBytes];
};
constexpr int kNcclSuccess = 0;
constexpr int kNcclInProgress = 7;
constexpr int kNcclFloat32 = 7;
}  // namespace

struct NcclApi {
  void* handle = nullptr;
  std::string path;
  int (*get_unique_id)(UniqueId*) = nullptr;
  int (*comm_init_rank)(void**, int, UniqueId, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*comm_get_async_error)(void*, int*) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*error_string)(int) = nullptr;
};

namespace {

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // prefer the NCCL already in the process (torch's), then RP_NCCL_LIBRARY, then the soname
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    std::string path = "libnccl.so.2 (already loaded)";
    if (!h) {
      if (const char* e = std::getenv("RP_NCCL_LIBRARY")) {
        h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
        path = e;
      }
    }
    if (!h) {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      path = "libnccl.so.2";
    }
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) err = std::string("libnccl: missing symbol ") + name;
      return p;
    };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.comm_get_async_error = reinterpret_cast<decltype(a.comm_get_async_error)>(sym("ncclCommGetAsyncError"));
    a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    a.path = path;
    if (err.empty()) a.handle = h;
  });
  if (!a.handle) throw DeviceError(RP_ERR_NCCL, err.empty() ? "libnccl unavailable" : err);
  return a;
}

void nccl_check(const NcclApi& a, int r, const char* what) {
  if (r != kNcclSuccess && r != kNcclInProgress)
    throw DeviceError(RP_ERR_NCCL, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
}

}  // namespace

std::string nccl_library_in_use() { return api().path; }

void NcclComm::unique_id(uint8_t out[kNcclUniqueIdBytes]) {
  const NcclApi& a = api();
  UniqueId id{};
  nccl_check(a, a.get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, kNcclUniqueIdBytes);
}

NcclComm::NcclComm(const uint8_t id[kNcclUniqueIdBytes], int nranks, int rank, int device)
    : api_(&api()), nranks_(nranks), rank_(rank), device_(device) {
  if (nranks < 1 || rank < 0 || rank >= nranks)
    throw std::invalid_argument("NcclComm: rank " + std::to_string(rank) + " of " + std::to_string(nranks));
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) throw DeviceError(RP_ERR_CUDA, "NcclComm: cudaSetDevice failed");
  UniqueId u{};
  std::memcpy(u.internal, id, kNcclUniqueIdBytes);
  const int r = api_->comm_init_rank(&comm_, nranks, u, rank);
  cudaSetDevice(prev);
  nccl_check(*api_, r, "ncclCommInitRank");
}

NcclComm::~NcclComm() {
  if (comm_) api_->comm_destroy(comm_);
}

void NcclComm::group_start() { nccl_check(*api_, api_->group_start(), "ncclGroupStart"); }
void NcclComm::group_end() { nccl_check(*api_, api_->group_end(), "ncclGroupEnd"); }

void NcclComm::send(const float* buf, size_t count, int peer, cudaStream_t s) {
  nccl_check(*api_, api_->send(buf, count, kNcclFloat32, peer, comm_, s), "ncclSend");
}

void NcclComm::recv(float* buf, size_t count, int peer, cudaStream_t s) {
  nccl_check(*api_, api_->recv(buf, count, kNcclFloat32, peer, comm_, s), "ncclRecv");
}

void NcclComm::check_async() const {
  int e = kNcclSuccess;
  nccl_check(*api_, api_->comm_get_async_error(comm_, &e), "ncclCommGetAsyncError");
  nccl_check(*api_, e, "NCCL asynchronous error");
}

}  // namespace respar::b200
