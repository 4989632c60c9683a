// C++ host mirror of the reference library's model/stage/trainer API for the
// layer-parallel training step (reference include/respar/decoupled.hpp:17-137,
// network.hpp:29-117, runtime.hpp:15-74), re-designed for B200: device-resident NHWC
// state, one CUDA stream per stage, events instead of the StagePool barrier, and every
// GPU operation issued through the C ABI in include/respar_b200.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "respar_b200.h"

namespace respar::b200 {

// ---- the reference's exception types (tensor.hpp:11-13, config.hpp:13-15, runtime.hpp:15-20)
struct ShapeError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct StageError : std::runtime_error {
  int stage;
  StageError(int s, const std::string& what) : std::runtime_error("stage " + std::to_string(s) + ": " + what), stage(s) {}
};
// CUDA / NCCL / internal failures.
struct DeviceError : std::runtime_error {
  int code;
  DeviceError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Throws the exception type the reference would throw for an rp status code.
[[noreturn]] void throw_status(int code, const std::string& msg);
// Status code for an exception thrown by this library (inverse of throw_status).
int status_of(const std::exception& e);
inline void check(int rc) {
  if (rc != RP_OK) throw_status(rc, rp_last_error());
}

enum class TrainMode { Serial = RP_MODE_SERIAL, Penalty = RP_MODE_PENALTY, Alm = RP_MODE_ALM };
enum class PenaltyKind { SquaredL2 = RP_PSI_SQUARED_L2, L1 = RP_PSI_L1, LInf = RP_PSI_LINF };

// Owning device allocation (RAII), pinned to one device.
class DeviceArray {
 public:
  DeviceArray() = default;
  ~DeviceArray();
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  DeviceArray(DeviceArray&& o) noexcept { swap(o); }
  DeviceArray& operator=(DeviceArray&& o) noexcept {
    swap(o);
    return *this;
  }
  // no-op when already at least that big; returns true when it (re)allocated, which moves
  // the buffer (a captured CUDA graph holding the old pointer must be re-captured)
  bool allocate(int device, int64_t bytes);
  void zero(cudaStream_t s);
  template <class T = float>
  T* get() const {
    return static_cast<T*>(ptr_);
  }
  int64_t bytes() const { return bytes_; }
  int device() const { return device_; }

 private:
  void swap(DeviceArray& o) noexcept {
    std::swap(ptr_, o.ptr_);
    std::swap(bytes_, o.bytes_);
    std::swap(device_, o.device_);
  }
  void* ptr_ = nullptr;
  int64_t bytes_ = 0;
  int device_ = 0;
};

// StepParams (decoupled.hpp:45-52) + momentum (0 == the reference's plain GD).
struct StepParams {
  double beta = 1.0;
  double tau = -1.0;
  double lr = 0.1;
  double lambda_lr = 0.1;
  double kappa_lr = 1e-9;
  int max_corrections = 1;
  double momentum = 0.0;
};

// NetGrads (network.hpp:81-87) of one stage: its contiguous slice [begin, begin + size) of the
// flat parameter layout (S when k = 0, the stage's blocks, T when k = K-1), copied to the host.
struct NetGrads {
  int64_t begin = 0;
  std::vector<float> values;
};

struct ViolationReport {
  std::vector<double> per_stage;
  double max_violation = 0.0;
  long normalizer = 0;
};

// partition (decoupled.cpp:10-21): K equal ranges; ConfigError unless K divides L.
std::vector<std::pair<int, int>> partition(int num_blocks, int stages);

// StagePool replacement (runtime.hpp:33-67): stage k runs on devices[floor(k*G/K)],
// on its own stream; the iteration barrier is a control stream waiting on every stage's
// completion event, so nothing host-side blocks unless a result is read back.
class StageScheduler {
 public:
  StageScheduler(int stages, std::vector<int> devices);
  ~StageScheduler();
  StageScheduler(const StageScheduler&) = delete;
  StageScheduler& operator=(const StageScheduler&) = delete;

  int stages() const { return static_cast<int>(streams_.size()); }
  int device_of(int k) const { return devices_.at(k); }
  cudaStream_t stream(int k) const { return streams_.at(k); }
  // stages of device_of(k) issuing on streams of their own (1 when they share one stream)
  int concurrent_ways(int k) const;
  cudaStream_t control() const { return ctl_; }
  int control_device() const { return devices_.at(0); }
  // iteration bracket: begin() fans out from the control stream, end() joins.
  void begin();
  void end();
  // stream `k` waits for the last record of `what` on stream `j`
  enum Mark { kBackwardDone = 0, kCorrectionDone = 1, kStageDone = 2, kNumMarks = 3 };
  void record(int j, Mark what);
  void wait(int k, int j, Mark what);
  cudaEvent_t mark_event(int j, Mark what) const { return marks_.at((size_t)j * kNumMarks + what); }
  float last_ms() const;  // device time between begin() and end() (control stream)
  // device-timed region over many iterations on the control stream
  void region_begin();
  float region_end();
  void sync();

 private:
  std::vector<int> devices_;
  std::vector<cudaStream_t> streams_;
  std::vector<bool> owned_;
  std::vector<cudaEvent_t> marks_;  // [stage][Mark]
  cudaStream_t ctl_ = nullptr;
  cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr, ev_rb_ = nullptr, ev_re_ = nullptr;
  bool timed_ = false;
};

// DecoupledTrainer (decoupled.hpp:56-120) on device.  Parameters are fp32 in the flat
// layout of include/respar_b200.h; lambda/kappa/boundary state is N_train x (H W C) fp32.
//
// Stage-sharded form (one process per GPU): a trainer may materialise only
// the stages [stage_lo, stage_hi) of the K-stage net.  When stage_hi < K it also holds a
// "ghost" of stage stage_hi -- lambda, kappa and the received boundary adjoint p of the
// boundary it corrects -- because boundary k is corrected by the owner of stage k-1
// (which holds X^{k-1}_end and, for its own backward, lambda_k / kappa_k).  The neighbour
// exchange (p_k upstream, the corrected lambda_k downstream) is done by the caller
// (paper_2009_01462_b200/distributed.py) on the stage streams.
class DecoupledTrainer {
 public:
  DecoupledTrainer(const rp_geometry& g, int stages, TrainMode mode, PenaltyKind kind, int num_samples,
                   int math = RP_MATH_FP32, std::vector<int> devices = {}, int stage_lo = 0, int stage_hi = -1);
  ~DecoupledTrainer();

  // ---- parameters (ResidualNet, network.hpp:29-41) ----
  void init_params(uint64_t& rng_state);  // make_net draw order (network.cpp:49-68)
  void set_params(const float* host);
  void get_params(float* host) const;
  void get_grads(float* host) const;
  int64_t param_count() const { return param_total_; }

  // ---- reference methods; x / labels are device pointers ----
  // full_x: raw inputs of all num_samples rows (stage_lo == 0); ignored when stage_lo > 0
  // (stage_lo's lambda must already hold the upstream rank's boundary output).
  void reset_lambda_from_forward(const float* full_x);
  double step(const float* batch_x, const int32_t* labels, int nrows, int row0, const StepParams& p,
              bool read_loss = true);
  void take_snapshot(int k, int row0, int nrows);
  void stage_forward(int k, const float* batch_x, int nrows, int row0);
  // returns the stage's gradients, as the reference does (decoupled.hpp:78-79)
  NetGrads stage_backward_update(int k, const int32_t* labels, double beta, double lr, int row0,
                                 double momentum = 0.0);
  NetGrads stage_grads(int k) const;   // the last backward's gradients of stage k
  void correct_aux(int k, const StepParams& p, int row0, int nrows);
  void correct_multiplier(int k, double beta, double kappa_lr, int row0, int nrows);
  void correction_gradient(int k, double beta, int row0, int nrows, float* out) const;
  // ---- stage-sharded iteration: the parallel phase of the local stages plus the
  // corrections of the boundaries inside [stage_lo, stage_hi) (step() == this + the loss
  // read on a trainer that owns every stage); then, once the downstream rank's p has been
  // received into the ghost's boundary adjoint, the ghost boundary's correction.
  void step_local(const float* batch_x, const int32_t* labels, int nrows, int row0, const StepParams& p);
  // CUDA graphs: step() captures the iteration (all stage streams) into one graph the first
  // time it sees a (pointers, rows, StepParams, multiplier state) key and replays it after
  // that.  Only for trainers that own every stage and single-pass corrections (tau < 0).
  void set_graphs(bool on);
  bool graphs() const { return graphs_; }
  void correct_ghost(const StepParams& p, int row0, int nrows);
  // the ghost boundary's correction on rows [row0 + sub0, row0 + sub0 + subn) of the batch
  // [row0, row0 + nrows) (normaliser of the whole batch): the chunked exchange of the stage
  // pipeline corrects each chunk as its adjoint rows arrive.  Elementwise kinds, one pass.
  void correct_ghost_rows(const StepParams& p, int row0, int nrows, int sub0, int subn);
  // ---- for the stage pipeline (pipeline.hpp), which drives step_local / correct_ghost_rows
  // and may capture them into its own CUDA graph
  void prepare(int nrows, const StepParams& p);          // buffers the step will use (no capture)
  void note_replayed_step(int nrows, int row0);          // host bookkeeping of a replayed step
  uint64_t kappa_zero_mask() const;
  uint64_t alloc_epoch() const { return alloc_epoch_; }
  int stage_lo() const { return stage_lo_; }
  int stage_hi() const { return stage_hi_; }
  bool is_local(int k) const { return k >= stage_lo_ && k < stage_hi_; }
  bool has_ghost() const { return stage_hi_ < static_cast<int>(stages_.size()); }
  float* state_device(int k, int which);     // start of the [num_samples][feat] buffer
  double* loss_device();                      // last stage's loss (device fp64)
  ViolationReport violation_report() const;
  double last_loss() const;
  // full serial forward of the current net (eval): logits [nrows, classes] device
  void forward(const float* x, int nrows, float* logits);
  // evaluation forward of the local stages [stage_lo, stage_hi) only (no tape kept):
  // `in` = raw inputs (stage_lo == 0) or the upstream boundary features; `out` = the
  // boundary features after stage_hi - 1, or the logits when the last stage is local.
  void forward_local(const float* in, int nrows, float* out);

  static long normalizer(int nrows, int feature_size) { return static_cast<long>(nrows) * feature_size; }

  // ---- state access (decoupled.hpp:29-32): 0 lambda, 1 kappa, 2 boundary_out, 3 boundary_adjoint
  int64_t state_elems(int k, int which) const;
  void get_state(int k, int which, float* host) const;
  void set_state(int k, int which, const float* host);

  int stages() const { return static_cast<int>(stages_.size()); }
  int blocks_per_stage() const { return blocks_per_stage_; }
  long iteration() const { return iteration_; }
  long stage_version(int k) const { return stages_.at(k).version; }
  int num_samples() const { return num_samples_; }
  const rp_geometry& geometry() const { return geo_; }
  TrainMode mode() const { return mode_; }
  PenaltyKind penalty_kind() const { return kind_; }
  void set_kappa_rule(int rule) { kappa_rule_ = rule; }
  StageScheduler& scheduler() { return *sched_; }
  float last_step_ms() const { return sched_->last_ms(); }
  // device staging for host inputs (used by the C ABI host-buffer entry points)
  float* input_staging(int nrows);
  int32_t* label_staging(int nrows);

 private:
  struct Stage {
    int index = 0, begin = 0, end = 0, device = 0;
    DeviceArray lam, kappa, bout, badj;  // [num_samples][feat]
    bool kappa_zero = true;
    std::vector<DeviceArray> xs;  // tape inputs x_1..x_{n-1}
    std::vector<DeviceArray> as;  // tape activations a_0..a_{n-1}
    // plane-pair tape (fp32 math on tcgen05 shapes): bf16 [2][elements] pairs of the block
    // inputs x_0..x_{n-1} and of a_0..a_{n-1}; dpre_p / g_p are backward scratch
    std::vector<DeviceArray> xps, aps;
    DeviceArray dpre_p, g_p;
    DeviceArray gscale;   // plane path: the cotangent planes' power-of-two scale (+ max partials)
    DeviceArray filters;  // plane path: the blocks' prepared filter pairs (forward, then reused for dgrad)
    bool tape_planes = false;
    bool tape_bf16 = false;  // bf16 math: xps / aps / dpre_p / g_p hold single bf16 copies
    std::vector<DeviceArray> dps;  // bf16 tape: bf16(1 - a^2) per block (as / dpre fp32 unused)
    DeviceArray x0, dpre, ws, red_ws, pooled, logits, loss;
    DeviceArray snap_lam, snap_kappa;
    int snap_rows = -1;
    bool snap_has_kappa = false;
    int cap_rows = 0;
    long version = -1;
    int fwd_rows = 0, fwd_row0 = 0;
    const float* input0 = nullptr;  // x_0 of the last forward
    const float* raw = nullptr;     // raw input of the last forward (stage 0)
  };

  void ensure_capacity(int nrows);
  const float* params_for(int k) const;
  float* params_for(int k);
  float* grads_for(int k);
  void run_forward(Stage& st, const float* input, int nrows, float* out_features, cudaStream_t s);
  void run_backward(Stage& st, const int32_t* labels, int nrows, int row0, double beta, double lr, double momentum,
                    bool use_snapshot, cudaStream_t s);
  void run_correction(int k, const StepParams& p, int row0, int nrows, bool fuse_kappa, cudaStream_t s,
                      int sub0 = 0, int subn = -1);
  void check_rows(int row0, int nrows, const char* where) const;
  void need_local(int k, const char* where) const;
  bool owns_state(int k) const { return is_local(k) || k == stage_hi_; }
  int64_t feat() const { return (int64_t)geo_.height * geo_.width * geo_.channels; }
  int64_t hid() const { return (int64_t)geo_.height * geo_.width * geo_.hidden; }
  int64_t raw_feat() const { return (int64_t)geo_.height * geo_.width * geo_.in_channels; }

  rp_geometry geo_;
  TrainMode mode_;
  PenaltyKind kind_;
  int num_samples_;
  int math_;
  int kappa_rule_ = RP_KAPPA_RULE_REFERENCE;
  int blocks_per_stage_ = 0;
  int64_t param_total_ = 0;
  std::vector<int> devices_;               // per stage
  std::vector<int> unique_devices_;
  std::vector<DeviceArray> params_, grads_, mom_;  // per unique device
  std::vector<Stage> stages_;
  std::unique_ptr<StageScheduler> sched_;
  DeviceArray in_stage_, lab_stage_, eval_a_, eval_b_;
  long iteration_ = 0;
  bool has_forward_ = false;
  int stage_lo_ = 0, stage_hi_ = 0;

  struct GraphKey {
    const void* x = nullptr;
    const void* y = nullptr;
    int nrows = -1, row0 = -1;
    double beta = 0, tau = 0, lr = 0, lambda_lr = 0, kappa_lr = 0, momentum = 0;
    int max_corrections = 0;
    uint64_t kappa_zero_mask = 0;
    uint64_t alloc_epoch = 0;   // buffer generation: any reallocation invalidates the graph
    bool operator==(const GraphKey& o) const {
      return alloc_epoch == o.alloc_epoch && x == o.x && y == o.y && nrows == o.nrows && row0 == o.row0 && beta == o.beta && tau == o.tau &&
             lr == o.lr && lambda_lr == o.lambda_lr && kappa_lr == o.kappa_lr && momentum == o.momentum &&
             max_corrections == o.max_corrections && kappa_zero_mask == o.kappa_zero_mask;
    }
  };
  bool graphs_ = false;
  bool graph_valid_ = false;
  GraphKey graph_key_;
  cudaGraphExec_t graph_exec_ = nullptr;
  uint64_t graph_kernels_ = 0;   // kernel nodes of the captured iteration (launch accounting)
  void step_graphed(const float* batch_x, const int32_t* labels, int nrows, int row0, const StepParams& p);
  uint64_t alloc_epoch_ = 0;       // bumped whenever a buffer the step reads or writes moves
  void ensure_momentum();          // velocity buffers, allocated and zeroed synchronously
  void enable_peer_access();       // in-process multi-device: neighbouring stages read each other
};

}  // namespace respar::b200
