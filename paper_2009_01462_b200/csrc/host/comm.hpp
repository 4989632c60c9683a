// NCCL point-to-point transport for the stage pipeline (the neighbour exchange
// of p_k and lambda_k between the ranks holding stages k-1 and k).
//
// libnccl is opened at run time (dlopen), so the library has no link-time NCCL dependency
// and loads the NCCL the process already has (torch's bundled one when torch is imported
// first; RP_NCCL_LIBRARY names another).  Only the stable public C ABI of nccl.h is used.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace respar::b200 {

constexpr int kNcclUniqueIdBytes = 128;   // NCCL_UNIQUE_ID_BYTES

struct NcclApi;   // dlopen'd entry points

// One NCCL communicator (nranks ranks, this process = rank) on one device.
class NcclComm {
 public:
  // ncclGetUniqueId: rank 0 creates it, the caller ships the bytes to every rank
  static void unique_id(uint8_t out[kNcclUniqueIdBytes]);
  NcclComm(const uint8_t id[kNcclUniqueIdBytes], int nranks, int rank, int device);
  ~NcclComm();
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;

  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  int device() const { return device_; }

  // point-to-point fp32 transfers; calls between group_start / group_end are matched as
  // one group (a send to this rank's own rank must be in the group of its receive)
  void group_start();
  void group_end();
  void send(const float* buf, size_t count, int peer, cudaStream_t s);
  void recv(float* buf, size_t count, int peer, cudaStream_t s);
  void check_async() const;   // ncclCommGetAsyncError

 private:
  const NcclApi* api_ = nullptr;
  void* comm_ = nullptr;   // ncclComm_t
  int nranks_ = 0, rank_ = 0, device_ = 0;
};

std::string nccl_library_in_use();

}  // namespace respar::b200
