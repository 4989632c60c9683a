// Stage pipeline: DecoupledTrainer::step (decoupled.cpp:172-194) across processes, one per
// B200, replacing the reference's StagePool (runtime.cpp:41-88) for multi-GPU runs
// (SURVEY §8e).  Each process holds one (or, in the single-process loopback used by the
// tests, several) stage-sharded trainers; the neighbour exchange runs over NCCL from here
// (C++ host), on dedicated communication streams, overlapped with compute:
//
//   stage streams    forward / synthetic-phi backward / SGD of the local stages, and the
//                    corrections of the boundaries inside a trainer (DecoupledTrainer::step_local)
//   stream A (commA) p_lo -> prev rank  ||  p_hi <- next rank, in C row chunks; chunk j is
//                    posted as soon as stage lo's backward is done
//   stage hi-1       ghost correction (correct_aux + correct_multiplier of boundary hi) of
//                    chunk j as soon as chunk j of p_hi has arrived
//   stream B (commB) lambda_hi -> next rank  ||  lambda_lo <- prev rank, chunk j as soon as
//                    its correction is done
//
// so the downstream transfer of lambda overlaps the upstream transfer of p and the
// corrections.  Ordering across iterations is carried by events only (no host sync): stage lo
// waits for this iteration's lambda_lo (and for its p_lo to be sent before the next backward
// overwrites it), the next correction waits for the previous lambda send, the next p receive
// for the previous correction.  The boundaries' corrections read only their own state, so the
// result equals the single-process trainer's bit for bit, for any chunk count.
//
// The whole step (kernels, events and NCCL calls) can be captured into one CUDA graph and
// replayed (set_graphs), like DecoupledTrainer::step.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "comm.hpp"
#include "respar_b200.hpp"

namespace respar::b200 {

class StagePipeline {
 public:
  struct Member {
    DecoupledTrainer* trainer;
    int prev_peer;   // rank (in both communicators) holding stage lo - 1, -1 if lo == 0
    int next_peer;   // rank holding stage hi, -1 if hi == K
  };
  // comm_a carries the adjoints p, comm_b the corrected lambdas (two communicators over the
  // same ranks, so the two directions progress independently).  members: this process's
  // trainers in stage order, all on comm_a's device.
  StagePipeline(NcclComm* comm_a, NcclComm* comm_b, std::vector<Member> members, int chunks);
  ~StagePipeline();
  StagePipeline(const StagePipeline&) = delete;
  StagePipeline& operator=(const StagePipeline&) = delete;

  // reset_lambda_from_forward (decoupled.cpp:44-63) as a chained forward over the ranks:
  // x_full (device, all num_samples raw inputs) is read by the member holding stage 0.
  void reset_lambda_from_forward(const float* x_full);
  // one iteration; x / labels are device pointers (read by the members holding stage 0 / K-1)
  void step(const float* x, const int32_t* labels, int nrows, int row0, const StepParams& p);
  // the last stage's pre-update loss (only on the process holding stage K-1)
  double loss();
  bool has_last_stage() const;
  void set_graphs(bool on);
  int chunks() const { return chunks_; }
  // device-timed region over many steps (every stream of the process joined)
  void region_begin();
  float region_end();
  void sync();

 private:
  void step_eager(const float* x, const int32_t* labels, int nrows, int row0, const StepParams& p);
  int effective_chunks(int nrows, const StepParams& p) const;

  NcclComm* ca_;
  NcclComm* cb_;
  std::vector<Member> m_;
  int chunks_;
  int device_;
  cudaStream_t sa_ = nullptr, sb_ = nullptr, ctl_ = nullptr;
  std::vector<cudaEvent_t> ev_a_, ev_c_;   // [chunk]: p chunk received / corrected
  cudaEvent_t ev_a_end_ = nullptr, ev_b_end_ = nullptr, ev_c_end_ = nullptr, ev_fork_ = nullptr;
  std::vector<cudaEvent_t> ev_join_;        // per member: its control stream joined back
  cudaEvent_t ev_rb_ = nullptr, ev_re_ = nullptr;
  bool first_ = true;                       // no previous iteration to wait for

  // CUDA graph of one step (key: pointers, rows, parameters, multiplier flags, buffers)
  struct Key {
    const void* x = nullptr;
    const void* y = nullptr;
    int nrows = -1, row0 = -1, chunks = 0;
    double beta = 0, tau = 0, lr = 0, lambda_lr = 0, kappa_lr = 0, momentum = 0;
    int max_corrections = 0;
    std::vector<uint64_t> masks;   // per member: kappa_zero_mask, alloc_epoch
    bool operator==(const Key& o) const;
  };
  Key make_key(const float* x, const int32_t* y, int nrows, int row0, const StepParams& p) const;
  bool graphs_ = false;
  bool graph_valid_ = false;
  Key key_;
  cudaGraphExec_t exec_ = nullptr;
  uint64_t graph_kernels_ = 0;
};

}  // namespace respar::b200
