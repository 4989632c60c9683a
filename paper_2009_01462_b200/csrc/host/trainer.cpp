// DecoupledTrainer / StageScheduler on device (reference decoupled.cpp:10-205,
// runtime.cpp:9-110).  Every GPU operation goes through the C ABI (rp_op_*).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "respar_b200.hpp"

namespace rp {
void note_launches(uint64_t n);   // capi_trainer.cpp: kernels launched through a graph replay
}

namespace respar::b200 {

namespace {

void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(RP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (d != prev) cu(cudaSetDevice(d), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

struct Layout {
  int64_t s_w, s_b, block0, block_stride, t_w, t_b, total;
  explicit Layout(const rp_geometry& g) {
    s_w = 0;
    block0 = rp_param_offset_block(&g, 0);
    block_stride = g.blocks > 1 ? rp_param_offset_block(&g, 1) - block0 : rp_param_offset_head(&g) - block0;
    s_b = block0 - g.channels;
    t_w = rp_param_offset_head(&g);
    t_b = t_w + (int64_t)g.channels * g.classes;
    total = rp_param_count(&g);
  }
};

}  // namespace

[[noreturn]] void throw_status(int code, const std::string& msg) {
  switch (code) {
    case RP_ERR_SHAPE: throw ShapeError(msg);
    case RP_ERR_CONFIG: throw ConfigError(msg);
    case RP_ERR_STATE: throw std::logic_error(msg);
    case RP_ERR_RANGE: throw std::invalid_argument(msg);
    case RP_ERR_STAGE: throw StageError(-1, msg);
    case RP_ERR_DIVERGED: throw std::runtime_error(msg);
    default: throw DeviceError(code, msg);
  }
}

int status_of(const std::exception& e) {
  if (dynamic_cast<const ShapeError*>(&e)) return RP_ERR_SHAPE;
  if (dynamic_cast<const ConfigError*>(&e)) return RP_ERR_CONFIG;
  if (dynamic_cast<const StageError*>(&e)) return RP_ERR_STAGE;
  if (auto* d = dynamic_cast<const DeviceError*>(&e)) return d->code;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return RP_ERR_RANGE;
  if (dynamic_cast<const std::logic_error*>(&e)) return RP_ERR_STATE;
  return RP_ERR_INTERNAL;
}

// ------------------------------------------------------------- DeviceArray
DeviceArray::~DeviceArray() {
  if (ptr_) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    cudaFree(ptr_);
    cudaSetDevice(prev);
  }
}

bool DeviceArray::allocate(int device, int64_t bytes) {
  if (ptr_ && bytes <= bytes_ && device == device_) return false;
  if (ptr_) {
    DeviceGuard g(device_);
    cudaFree(ptr_);
    ptr_ = nullptr;
    bytes_ = 0;
  }
  if (bytes <= 0) return true;
  DeviceGuard g(device);
  cu(cudaMalloc(&ptr_, static_cast<size_t>(bytes)), "cudaMalloc");
  bytes_ = bytes;
  device_ = device;
  return true;
}

void DeviceArray::zero(cudaStream_t s) {
  if (ptr_) {
    DeviceGuard g(device_);
    cu(cudaMemsetAsync(ptr_, 0, static_cast<size_t>(bytes_), s), "cudaMemsetAsync");
  }
}

// --------------------------------------------------------------- partition
std::vector<std::pair<int, int>> partition(int num_blocks, int stages) {
  if (stages < 1) throw ConfigError("partition: need at least one stage");
  if (num_blocks < 1 || num_blocks % stages != 0)
    throw ConfigError("partition: " + std::to_string(stages) + " stages do not divide " + std::to_string(num_blocks) +
                      " blocks evenly");
  const int n = num_blocks / stages;
  std::vector<std::pair<int, int>> r;
  for (int k = 0; k < stages; ++k) r.emplace_back(k * n, (k + 1) * n);
  return r;
}

// ---------------------------------------------------------- StageScheduler
StageScheduler::StageScheduler(int stages, std::vector<int> devices) {
  if (stages < 1) throw std::invalid_argument("StageScheduler: need at least one stage");
  if (devices.empty()) {
    int d = 0;
    cu(cudaGetDevice(&d), "cudaGetDevice");
    devices.push_back(d);
  }
  const int G = static_cast<int>(devices.size());
  for (int k = 0; k < stages; ++k) devices_.push_back(devices[(int64_t)k * G / stages]);
  streams_.resize(stages);
  owned_.assign(stages, false);
  marks_.resize((size_t)stages * kNumMarks);
  // Stages that share a GPU share its stream unless RP_CONCURRENT_STAGES=1: at the
  // benchmark sizes every conv launch fills the 148 SMs on its own, and serialising
  // keeps each kernel's event-timed duration clean for the roofline.
  const char* env = std::getenv("RP_CONCURRENT_STAGES");
  const bool concurrent = env && std::string(env) == "1";
  for (int k = 0; k < stages; ++k) {
    DeviceGuard g(devices_[k]);
    int share = -1;
    for (int j = 0; j < k && !concurrent; ++j)
      if (devices_[j] == devices_[k]) {
        share = j;
        break;
      }
    if (share >= 0) {
      streams_[k] = streams_[share];
    } else {
      cu(cudaStreamCreateWithFlags(&streams_[k], cudaStreamNonBlocking), "cudaStreamCreate");
      owned_[k] = true;
    }
    for (int m = 0; m < kNumMarks; ++m)
      cu(cudaEventCreateWithFlags(&marks_[(size_t)k * kNumMarks + m], cudaEventDisableTiming), "cudaEventCreate");
  }
  DeviceGuard g(devices_[0]);
  cu(cudaStreamCreateWithFlags(&ctl_, cudaStreamNonBlocking), "cudaStreamCreate");
  cu(cudaEventCreate(&ev_begin_), "cudaEventCreate");
  cu(cudaEventCreate(&ev_end_), "cudaEventCreate");
  cu(cudaEventCreate(&ev_rb_), "cudaEventCreate");
  cu(cudaEventCreate(&ev_re_), "cudaEventCreate");
}

// the calling thread's "stages issuing concurrently" setting for the ops, restored on exit
struct ConcurrentStagesScope {
  int prev;
  explicit ConcurrentStagesScope(int ways) : prev(rp_op_concurrent_stages()) { rp_op_set_concurrent_stages(ways); }
  ~ConcurrentStagesScope() { rp_op_set_concurrent_stages(prev); }
  ConcurrentStagesScope(const ConcurrentStagesScope&) = delete;
  ConcurrentStagesScope& operator=(const ConcurrentStagesScope&) = delete;
};

int StageScheduler::concurrent_ways(int k) const {
  std::vector<cudaStream_t> seen;
  for (size_t j = 0; j < streams_.size(); ++j)
    if (devices_[j] == devices_.at(k) && std::find(seen.begin(), seen.end(), streams_[j]) == seen.end())
      seen.push_back(streams_[j]);
  return static_cast<int>(seen.size());
}

StageScheduler::~StageScheduler() {
  for (size_t k = 0; k < streams_.size(); ++k) {
    cudaSetDevice(devices_[k]);
    cudaStreamSynchronize(streams_[k]);
  }
  for (size_t k = 0; k < streams_.size(); ++k) {
    cudaSetDevice(devices_[k]);
    if (owned_[k]) cudaStreamDestroy(streams_[k]);
    for (int m = 0; m < kNumMarks; ++m) cudaEventDestroy(marks_[k * kNumMarks + m]);
  }
  cudaSetDevice(devices_[0]);
  cudaStreamSynchronize(ctl_);
  cudaStreamDestroy(ctl_);
  cudaEventDestroy(ev_begin_);
  cudaEventDestroy(ev_end_);
  cudaEventDestroy(ev_rb_);
  cudaEventDestroy(ev_re_);
}

void StageScheduler::region_begin() {
  DeviceGuard g(devices_[0]);
  cu(cudaEventRecord(ev_rb_, ctl_), "cudaEventRecord");
}

float StageScheduler::region_end() {
  // join every stage stream (work enqueued after end(), e.g. the neighbour exchange and
  // the ghost correction of a stage-sharded step, belongs to the region)
  for (int k = 0; k < stages(); ++k) {
    record(k, kStageDone);
    DeviceGuard g(devices_[0]);
    cu(cudaStreamWaitEvent(ctl_, marks_[(size_t)k * kNumMarks + kStageDone], 0), "cudaStreamWaitEvent");
  }
  DeviceGuard g(devices_[0]);
  cu(cudaEventRecord(ev_re_, ctl_), "cudaEventRecord");
  cu(cudaEventSynchronize(ev_re_), "cudaEventSynchronize");
  float ms = 0.f;
  cu(cudaEventElapsedTime(&ms, ev_rb_, ev_re_), "cudaEventElapsedTime");
  return ms;
}

void StageScheduler::begin() {
  DeviceGuard g(devices_[0]);
  cu(cudaEventRecord(ev_begin_, ctl_), "cudaEventRecord");
  for (int k = 0; k < stages(); ++k) {
    DeviceGuard gk(devices_[k]);
    cu(cudaStreamWaitEvent(streams_[k], ev_begin_, 0), "cudaStreamWaitEvent");
  }
}

void StageScheduler::end() {
  for (int k = 0; k < stages(); ++k) {
    record(k, kStageDone);
    DeviceGuard g(devices_[0]);
    cu(cudaStreamWaitEvent(ctl_, marks_[(size_t)k * kNumMarks + kStageDone], 0), "cudaStreamWaitEvent");
  }
  DeviceGuard g(devices_[0]);
  cu(cudaEventRecord(ev_end_, ctl_), "cudaEventRecord");
  timed_ = true;
}

void StageScheduler::record(int j, Mark what) {
  DeviceGuard g(devices_[j]);
  cu(cudaEventRecord(marks_[(size_t)j * kNumMarks + what], streams_[j]), "cudaEventRecord");
}

void StageScheduler::wait(int k, int j, Mark what) {
  DeviceGuard g(devices_[k]);
  cu(cudaStreamWaitEvent(streams_[k], marks_[(size_t)j * kNumMarks + what], 0), "cudaStreamWaitEvent");
}

float StageScheduler::last_ms() const {
  if (!timed_) return 0.f;
  float ms = 0.f;
  cu(cudaEventSynchronize(ev_end_), "cudaEventSynchronize");
  cu(cudaEventElapsedTime(&ms, ev_begin_, ev_end_), "cudaEventElapsedTime");
  return ms;
}

void StageScheduler::sync() {
  for (int k = 0; k < stages(); ++k) {
    DeviceGuard g(devices_[k]);
    cu(cudaStreamSynchronize(streams_[k]), "cudaStreamSynchronize");
  }
  DeviceGuard g(devices_[0]);
  cu(cudaStreamSynchronize(ctl_), "cudaStreamSynchronize");
}

// --------------------------------------------------------- DecoupledTrainer
DecoupledTrainer::DecoupledTrainer(const rp_geometry& g, int stages, TrainMode mode, PenaltyKind kind,
                                   int num_samples, int math, std::vector<int> devices, int stage_lo, int stage_hi)
    : geo_(g), mode_(mode), kind_(kind), num_samples_(num_samples), math_(math) {
  if (rp_param_count(&g) < 0) check(RP_ERR_CONFIG);
  if (num_samples < 1) throw ConfigError("DecoupledTrainer: need at least one sample");
  const auto ranges = partition(g.blocks, stages);
  stage_lo_ = stage_lo;
  stage_hi_ = stage_hi < 0 ? stages : stage_hi;
  if (stage_lo_ < 0 || stage_lo_ >= stage_hi_ || stage_hi_ > stages)
    throw std::invalid_argument("DecoupledTrainer: local stage range [" + std::to_string(stage_lo_) + ", " +
                                std::to_string(stage_hi_) + ") is not inside [0, " + std::to_string(stages) + ")");
  blocks_per_stage_ = ranges[0].second - ranges[0].first;
  sched_ = std::make_unique<StageScheduler>(stages, devices);
  param_total_ = rp_param_count(&g);
  for (int k = 0; k < stages; ++k) {
    devices_.push_back(sched_->device_of(k));
    if (std::find(unique_devices_.begin(), unique_devices_.end(), devices_[k]) == unique_devices_.end())
      unique_devices_.push_back(devices_[k]);
  }
  if (unique_devices_.size() > 1) enable_peer_access();
  params_.resize(unique_devices_.size());
  grads_.resize(unique_devices_.size());
  mom_.resize(unique_devices_.size());
  for (size_t i = 0; i < unique_devices_.size(); ++i) {
    params_[i].allocate(unique_devices_[i], param_total_ * 4);
    grads_[i].allocate(unique_devices_[i], param_total_ * 4);
    params_[i].zero(nullptr);
    grads_[i].zero(nullptr);
  }
  stages_.resize(stages);
  const int64_t state_bytes = (int64_t)num_samples * feat() * 4;
  for (int k = 0; k < stages; ++k) {
    Stage& st = stages_[k];
    st.index = k;
    st.begin = ranges[k].first;
    st.end = ranges[k].second;
    st.device = devices_[k];
    if (!owns_state(k)) continue;               // another rank's stage
    const bool ghost = !is_local(k);
    if (ghost) st.device = devices_[k - 1];     // lives with the stage that corrects it
    if (k > 0) {
      st.lam.allocate(st.device, state_bytes);
      st.kappa.allocate(st.device, state_bytes);
      st.lam.zero(nullptr);
      st.kappa.zero(nullptr);
    }
    st.badj.allocate(st.device, state_bytes);
    st.badj.zero(nullptr);
    st.red_ws.allocate(st.device, rp_op_reduce_workspace_bytes());   // psi / correction reductions
    if (ghost) continue;
    st.bout.allocate(st.device, state_bytes);
    st.bout.zero(nullptr);
    st.loss.allocate(st.device, 8);
    st.loss.zero(nullptr);
  }
  cu(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
}

DecoupledTrainer::~DecoupledTrainer() {
  try {
    if (sched_) sched_->sync();
  } catch (...) {
    // a sticky CUDA error was already reported by the call that raised it
  }
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
}

static size_t dev_index(const std::vector<int>& u, int d) {
  return static_cast<size_t>(std::find(u.begin(), u.end(), d) - u.begin());
}

const float* DecoupledTrainer::params_for(int k) const {
  return params_[dev_index(unique_devices_, devices_[k])].get();
}
float* DecoupledTrainer::params_for(int k) { return params_[dev_index(unique_devices_, devices_[k])].get(); }
float* DecoupledTrainer::grads_for(int k) { return grads_[dev_index(unique_devices_, devices_[k])].get(); }

void DecoupledTrainer::init_params(uint64_t& rng_state) {
  uint64_t s0 = rng_state;
  for (size_t i = 0; i < unique_devices_.size(); ++i) {
    DeviceGuard g(unique_devices_[i]);
    uint64_t s = s0;
    check(rp_op_init_params(&geo_, params_[i].get(), &s, nullptr));
    rng_state = s;
  }
  cu(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
}

void DecoupledTrainer::set_params(const float* host) {
  sched_->sync();
  for (size_t i = 0; i < unique_devices_.size(); ++i) {
    DeviceGuard g(unique_devices_[i]);
    cu(cudaMemcpy(params_[i].get(), host, param_total_ * 4, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
}

void DecoupledTrainer::get_params(float* host) const {
  sched_->sync();
  // each stage's device owns its parameter slice (stage 0 owns S, stage K-1 owns T)
  const Layout L(geo_);
  for (int k = stage_lo_; k < stage_hi_; ++k) {
    const Stage& st = stages_[k];
    int64_t beg = L.block0 + (int64_t)st.begin * L.block_stride;
    int64_t end = L.block0 + (int64_t)st.end * L.block_stride;
    if (k == 0) beg = 0;
    if (k == stages() - 1) end = L.total;
    DeviceGuard g(st.device);
    cu(cudaMemcpy(host + beg, params_for(k) + beg, (end - beg) * 4, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  }
}

void DecoupledTrainer::get_grads(float* host) const {
  sched_->sync();
  const Layout L(geo_);
  for (int k = stage_lo_; k < stage_hi_; ++k) {
    const Stage& st = stages_[k];
    int64_t beg = L.block0 + (int64_t)st.begin * L.block_stride;
    int64_t end = L.block0 + (int64_t)st.end * L.block_stride;
    if (k == 0) beg = 0;
    if (k == stages() - 1) end = L.total;
    DeviceGuard g(st.device);
    const float* src = grads_[dev_index(unique_devices_, st.device)].get();
    cu(cudaMemcpy(host + beg, src + beg, (end - beg) * 4, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  }
}

void DecoupledTrainer::ensure_capacity(int nrows) {
  for (int k = stage_lo_; k < stage_hi_; ++k) {
    Stage& st = stages_[k];
    if (st.cap_rows >= nrows) continue;
    const int n = st.end - st.begin;
    const bool planes = rp_op_block_planes_supported(&geo_, nrows, math_) != 0;
    const bool bf16t = rp_op_block_bf16_tape_supported(&geo_, nrows, math_) != 0;
    // on the tape paths the backward reads the bf16 copies of the block inputs, so the fp32
    // block inputs x_1.. only roll through two buffers (x_i feeds block i's forward alone)
    const bool rolling = planes || bf16t;
    st.xs.resize(n);
    st.as.resize(n);
    for (int i = 0; i < n; ++i) {
      if (i > 0 && (!rolling || i <= 2)) st.xs[i].allocate(st.device, (int64_t)nrows * feat() * 4);
      if (!bf16t) st.as[i].allocate(st.device, (int64_t)nrows * hid() * 4);   // bf16 tape: a16 / d16 only
    }
    if (k == 0) st.x0.allocate(st.device, (int64_t)nrows * feat() * 4);
    if (!bf16t) st.dpre.allocate(st.device, (int64_t)nrows * hid() * 4);
    if (bf16t) {
      st.dps.resize(n);
      for (int i = 0; i < n; ++i) st.dps[i].allocate(st.device, (int64_t)nrows * hid() * 2);
    }
    if (rolling) {
      const int64_t eb = planes ? 4 : 2;   // bytes per element: a bf16 plane pair, or one bf16 copy
      st.xps.resize(n);
      st.aps.resize(n);
      for (int i = 0; i < n; ++i) {
        st.xps[i].allocate(st.device, (int64_t)nrows * feat() * eb);
        st.aps[i].allocate(st.device, (int64_t)nrows * hid() * eb);
      }
      st.dpre_p.allocate(st.device, (int64_t)nrows * hid() * eb);
      st.g_p.allocate(st.device, (int64_t)nrows * feat() * eb);
      st.filters.allocate(st.device, std::max<int64_t>(256, rp_op_planes_filters_bytes(&geo_, n)));
      st.gscale.allocate(st.device, rp_op_plane_scale_bytes());   // the cotangent planes' scale
    }
    st.ws.allocate(st.device, rp_op_workspace_bytes(&geo_, nrows, math_));
    if (k == stages() - 1) {
      st.pooled.allocate(st.device, (int64_t)nrows * geo_.channels * 4);
      st.logits.allocate(st.device, (int64_t)nrows * geo_.classes * 4);
    }
    st.cap_rows = nrows;
    ++alloc_epoch_;   // the tape / workspace pointers moved
  }
}

float* DecoupledTrainer::input_staging(int nrows) {
  if (in_stage_.allocate(stages_[stage_lo_].device, std::max<int64_t>(1, (int64_t)nrows * raw_feat() * 4)))
    ++alloc_epoch_;
  return in_stage_.get();
}

int32_t* DecoupledTrainer::label_staging(int nrows) {
  if (lab_stage_.allocate(stages_[stage_hi_ - 1].device, std::max<int64_t>(4, (int64_t)nrows * 4))) ++alloc_epoch_;
  return lab_stage_.get<int32_t>();
}

void DecoupledTrainer::ensure_momentum() {
  for (size_t i = 0; i < unique_devices_.size(); ++i) {
    if (mom_[i].bytes() != 0) continue;
    DeviceGuard g(unique_devices_[i]);
    mom_[i].allocate(unique_devices_[i], param_total_ * 4);
    cu(cudaMemset(mom_[i].get(), 0, (size_t)param_total_ * 4), "cudaMemset");
    cu(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    ++alloc_epoch_;
  }
}

void DecoupledTrainer::enable_peer_access() {
  // stage k's kernels read lambda / kappa of stage k+1 and the correction of boundary k
  // reads X^{k-1}_end of stage k-1, so every pair of neighbouring devices needs peer access
  for (size_t k = 1; k < devices_.size(); ++k) {
    const int a = devices_[k - 1], b = devices_[k];
    if (a == b) continue;
    for (auto [from, to] : {std::pair<int, int>{a, b}, std::pair<int, int>{b, a}}) {
      int ok = 0;
      cu(cudaDeviceCanAccessPeer(&ok, from, to), "cudaDeviceCanAccessPeer");
      if (!ok)
        throw ConfigError("DecoupledTrainer: devices " + std::to_string(from) + " and " + std::to_string(to) +
                          " have no peer access; run one process per GPU instead");
      DeviceGuard g(from);
      const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();   // clear the non-sticky status
      else
        cu(e, "cudaDeviceEnablePeerAccess");
    }
  }
}

void DecoupledTrainer::need_local(int k, const char* where) const {
  if (k >= 0 && k < stages() && !is_local(k))
    throw std::invalid_argument(std::string(where) + ": stage " + std::to_string(k) + " is not local to this rank");
}

void DecoupledTrainer::check_rows(int row0, int nrows, const char* where) const {
  if (row0 < 0 || nrows < 0 || (int64_t)row0 + nrows > num_samples_)
    throw ShapeError(std::string(where) + ": rows [" + std::to_string(row0) + ", " + std::to_string(row0 + nrows) +
                     ") out of " + std::to_string(num_samples_) + " samples");
}

// net_forward over the stage's block range (network.cpp:112-143).  The stage output
// (X^k_end) is written to out_features; the tape keeps x_1..x_{n-1} and every a.
void DecoupledTrainer::run_forward(Stage& st, const float* input, int nrows, float* out_features, cudaStream_t s) {
  const ConcurrentStagesScope share(sched_->concurrent_ways(st.index));
  const Layout L(geo_);
  const float* P = params_for(st.index);
  const float* cur = input;
  const int n = st.end - st.begin;
  st.tape_planes = n > 0 && rp_op_block_planes_supported(&geo_, nrows, math_);
  st.tape_bf16 = n > 0 && rp_op_block_bf16_tape_supported(&geo_, nrows, math_);
  // the first block's input planes: written by the stem in its pass, else split here
  bool in_planes = false;
  if (st.index == 0) {
    if (st.tape_planes || st.tape_bf16) {
      auto* p = st.xps[0].get<uint16_t>();
      check(rp_op_stem_fwd_planes(&geo_, nrows, input, P, st.x0.get(), p,
                                  st.tape_bf16 ? nullptr : p + (int64_t)nrows * feat(), s));
      in_planes = true;
    } else {
      check(rp_op_stem_fwd(&geo_, nrows, input, P, st.x0.get(), math_, st.ws.get(), st.ws.bytes(), s));
    }
    st.raw = input;
    cur = st.x0.get();
  }
  st.input0 = cur;
  if (st.tape_bf16) {
    // bf16 copies of every block input and activation for the TMA-fed bf16 wgrad
    if (!in_planes) check(rp_op_split_planes(cur, (int64_t)nrows * feat(), st.xps[0].get(), nullptr, nullptr, s));
    for (int i = 0; i < n; ++i) {
      const int l = st.begin + i;
      float* out = i == n - 1 ? out_features : st.xs[1 + (i & 1)].get();
      check(rp_op_block_fwd_bf16t(&geo_, nrows, cur, st.xps[i].get(), P + L.block0 + (int64_t)l * L.block_stride,
                                  st.aps[i].get(), st.dps[i].get(), out,
                                  i == n - 1 ? nullptr : st.xps[i + 1].get(), st.ws.get(), st.ws.bytes(), s));
      cur = out;
    }
    if (st.index == stages() - 1)
      check(rp_op_head_fwd(&geo_, nrows, out_features, P + L.t_w, st.pooled.get(), st.logits.get(), s));
    return;
  }
  if (st.tape_planes) {
    const int64_t e = (int64_t)nrows * feat();
    auto* p = st.xps[0].get<uint16_t>();
    if (!in_planes) check(rp_op_split_planes(cur, e, p, p + e, nullptr, s));
    // every block's forward filters in one launch (not one per conv)
    const int64_t fpair = rp_op_planes_filters_bytes(&geo_, 1);
    check(rp_op_prep_planes_filters(&geo_, P + L.block0 + (int64_t)st.begin * L.block_stride, n, 0,
                                    st.filters.get(), s));
    for (int i = 0; i < n; ++i) {
      const int l = st.begin + i;
      float* out = i == n - 1 ? out_features : st.xs[1 + (i & 1)].get();
      check(rp_op_block_fwd_planes(&geo_, nrows, cur, st.xps[i].get(), P + L.block0 + (int64_t)l * L.block_stride,
                                   st.as[i].get(), out, st.aps[i].get(), i == n - 1 ? nullptr : st.xps[i + 1].get(),
                                   st.filters.get<char>() + i * fpair, st.ws.get(), st.ws.bytes(), s));
      cur = out;
    }
    if (st.index == stages() - 1)
      check(rp_op_head_fwd(&geo_, nrows, out_features, P + L.t_w, st.pooled.get(), st.logits.get(), s));
    return;
  }
  for (int i = 0; i < n; ++i) {
    const int l = st.begin + i;
    float* out = i == n - 1 ? out_features : st.xs[i + 1].get();
    check(rp_op_block_fwd(&geo_, nrows, cur, P + L.block0 + (int64_t)l * L.block_stride, st.as[i].get(), out, math_,
                          st.ws.get(), st.ws.bytes(), s));
    cur = out;
  }
  if (st.index == stages() - 1)
    check(rp_op_head_fwd(&geo_, nrows, out_features, P + L.t_w, st.pooled.get(), st.logits.get(), s));
}

// stage_backward_update body (decoupled.cpp:85-115): upstream, net_vjp, apply_updates,
// boundary_adjoint.  The cotangent lives in the boundary_adjoint rows and is updated
// block by block in place, so p^k lands where correct_aux reads it.
void DecoupledTrainer::run_backward(Stage& st, const int32_t* labels, int nrows, int row0, double beta, double lr,
                                    double momentum, bool use_snapshot, cudaStream_t s) {
  const ConcurrentStagesScope share(sched_->concurrent_ways(st.index));
  const Layout L(geo_);
  const int k = st.index;
  float* P = params_for(k);
  float* G = grads_for(k);
  float* g = st.badj.get() + (int64_t)row0 * feat();
  const float* x_end = st.bout.get() + (int64_t)st.fwd_row0 * feat();
  const int64_t n = (int64_t)nrows * feat();
  // the tape paths' first backward conv reads g as bf16 planes: the synthetic upstream writes
  // them in the same pass (planes_done), the head's cotangent is split afterwards
  const bool tape = (st.tape_bf16 || st.tape_planes) && st.fwd_rows == nrows;
  uint16_t* gp16 = tape ? st.g_p.get<uint16_t>() : nullptr;
  bool planes_done = false;
  if (k == stages() - 1) {
    if (tape) {
      check(rp_op_head_loss_bwd_planes(&geo_, nrows, st.pooled.get(), st.logits.get(), P + L.t_w, labels,
                                       st.loss.get<double>(), G + L.t_w, g, gp16, st.tape_bf16 ? nullptr : gp16 + n,
                                       st.tape_bf16 ? nullptr : st.gscale.get(), st.ws.get(), st.ws.bytes(), s));
      planes_done = true;
    } else {
      check(rp_op_head_loss_bwd(&geo_, nrows, st.pooled.get(), st.logits.get(), P + L.t_w, labels,
                                st.loss.get<double>(), G + L.t_w, g, st.ws.get(), st.ws.bytes(), s));
    }
  } else {
    const Stage& nx = stages_[k + 1];
    const float* lam_next;
    const float* kap_next;
    if (use_snapshot) {
      lam_next = st.snap_lam.get();
      kap_next = st.snap_has_kappa ? st.snap_kappa.get() : nullptr;
    } else {
      lam_next = nx.lam.get() + (int64_t)row0 * feat();
      kap_next = nx.kappa_zero ? nullptr : nx.kappa.get() + (int64_t)row0 * feat();
    }
    const double w = beta / static_cast<double>(normalizer(nrows, (int)feat()));
    if (tape) {
      check(rp_op_synthetic_grad_planes((int)kind_, lam_next, x_end, kap_next, n, w, g, gp16,
                                        st.tape_bf16 ? nullptr : gp16 + n, st.tape_bf16 ? nullptr : st.gscale.get(),
                                        st.red_ws.get(), s));
      planes_done = true;
    } else {
      check(rp_op_synthetic_grad((int)kind_, lam_next, x_end, kap_next, n, w, g, st.red_ws.get(), s));
    }
  }
  const int nb = st.end - st.begin;
  if (st.tape_bf16 && st.fwd_rows == nrows) {
    auto* gp = st.g_p.get<uint16_t>();
    if (!planes_done) check(rp_op_split_planes(g, n, gp, nullptr, nullptr, s));
    for (int i = nb - 1; i >= 0; --i) {
      const int l = st.begin + i;
      const int64_t off = L.block0 + (int64_t)l * L.block_stride;
      check(rp_op_block_bwd_bf16t(&geo_, nrows, st.xps[i].get(), st.aps[i].get(), st.dps[i].get(), P + off, g, gp,
                                  st.dpre_p.get(), G + off, st.ws.get(), st.ws.bytes(), s));
    }
  } else if (st.tape_planes && st.fwd_rows == nrows) {
    auto* gp = st.g_p.get<uint16_t>();
    if (!planes_done) check(rp_op_split_planes(g, n, gp, gp + n, st.gscale.get(), s));
    // every block's input-gradient filters in one launch, from the current parameters
    const int64_t fpair = rp_op_planes_filters_bytes(&geo_, 1);
    check(rp_op_prep_planes_filters(&geo_, P + L.block0 + (int64_t)st.begin * L.block_stride, nb, 1,
                                    st.filters.get(), s));
    for (int i = nb - 1; i >= 0; --i) {
      const int l = st.begin + i;
      const int64_t off = L.block0 + (int64_t)l * L.block_stride;
      check(rp_op_block_bwd_planes(&geo_, nrows, st.xps[i].get(), st.as[i].get(), st.aps[i].get(), P + off, g, gp,
                                   st.gscale.get(),
                                   st.dpre.get(), st.dpre_p.get(), G + off, st.filters.get<char>() + i * fpair,
                                   st.ws.get(), st.ws.bytes(), s));
    }
  } else {
    if ((st.tape_planes && nb > 1) || st.tape_bf16)   // the fp32 block inputs / activations were not kept
      throw std::logic_error("stage_backward_update: rows differ from the stage's forward");
  for (int i = nb - 1; i >= 0; --i) {
    const int l = st.begin + i;
    const float* xin = i == 0 ? st.input0 : st.xs[i].get();
    const int64_t off = L.block0 + (int64_t)l * L.block_stride;
    check(rp_op_block_bwd(&geo_, nrows, xin, st.as[i].get(), P + off, g, st.dpre.get(), G + off, math_, st.ws.get(),
                          st.ws.bytes(), s));
  }
  }
  if (k == 0) check(rp_op_stem_bwd(&geo_, nrows, st.raw, g, G, st.ws.get(), st.ws.bytes(), s));
  // apply_updates (network.cpp:174-191): the stage's parameter range is contiguous
  int64_t beg = L.block0 + (int64_t)st.begin * L.block_stride;
  int64_t end = L.block0 + (int64_t)st.end * L.block_stride;
  if (k == 0) beg = 0;
  if (k == stages() - 1) end = L.total;
  float* v = nullptr;
  if (momentum != 0.0) {
    const size_t di = dev_index(unique_devices_, st.device);
    if (mom_[di].bytes() == 0) throw std::logic_error("stage_backward_update: momentum buffers not allocated");
    v = mom_[di].get() + beg;
  }
  check(rp_op_sgd(P + beg, G + beg, v, end - beg, lr, momentum, s));
}

// correct_aux + correct_multiplier (decoupled.cpp:135-170) for boundary k.
void DecoupledTrainer::run_correction(int k, const StepParams& p, int row0, int nrows, bool fuse_kappa,
                                      cudaStream_t s, int sub0, int subn) {
  Stage& st = stages_[k];
  const Stage& prev = stages_[k - 1];
  if (subn < 0) subn = nrows - sub0;
  const bool part = sub0 != 0 || subn != nrows;
  if (part && (kind_ == PenaltyKind::LInf || (p.max_corrections > 1 && p.tau >= 0.0)))
    throw std::logic_error("correction: a row sub-range needs an elementwise penalty and a single pass");
  const int64_t off = (int64_t)(row0 + sub0) * feat();
  const int64_t n = (int64_t)subn * feat();
  const long norm = normalizer(nrows, (int)feat());   // # of the whole mini-batch slice
  const double w = p.beta / static_cast<double>(norm);
  float* lam = st.lam.get() + off;
  const float* xp = prev.bout.get() + off;
  const float* pk = st.badj.get() + off;
  const bool alm = fuse_kappa && mode_ == TrainMode::Alm;
  if (alm && kind_ != PenaltyKind::SquaredL2)
    throw std::logic_error("correct_multiplier: the multiplier update is only derived for the squared_l2 penalty");
  const double coef = kappa_rule_ == RP_KAPPA_RULE_TEXTBOOK ? -p.beta : p.kappa_lr * (double)norm / (2.0 * p.beta);
  float* kap = (alm || !st.kappa_zero) ? st.kappa.get() + off : nullptr;
  const bool single = p.max_corrections <= 1 || p.tau < 0.0;
  if (single) {
    check(rp_op_correct((int)kind_, lam, xp, pk, kap, n, w, p.lambda_lr, 1, coef, alm ? 1 : 0, st.red_ws.get(), s));
  } else {
    for (int pass = 0; pass < p.max_corrections; ++pass) {
      if (pass >= 1) {
        double v = 0.0;
        check(rp_op_psi((int)kind_, lam, xp, n, &v, st.red_ws.get(), s));
        if (v <= p.tau) break;
      }
      check(rp_op_correct((int)kind_, lam, xp, pk, kap, n, w, p.lambda_lr, 1, 0.0, 0, st.red_ws.get(), s));
    }
    if (alm) check(rp_op_correct((int)kind_, lam, xp, pk, kap, n, w, 0.0, 0, coef, 1, st.red_ws.get(), s));
  }
  if (alm && !part) st.kappa_zero = false;
}

void DecoupledTrainer::reset_lambda_from_forward(const float* full_x) {
  sched_->sync();
  if (stage_lo_ == 0 && !full_x) throw std::invalid_argument("reset_lambda_from_forward: null input");
  const int chunk = std::min(num_samples_, std::max(256, stages_[stage_lo_].cap_rows));
  ensure_capacity(chunk);
  for (int r0 = 0; r0 < num_samples_; r0 += chunk) {
    const int nr = std::min(chunk, num_samples_ - r0);
    const float* in = stage_lo_ == 0 ? full_x + (int64_t)r0 * raw_feat()
                                     : stages_[stage_lo_].lam.get() + (int64_t)r0 * feat();
    for (int k = stage_lo_; k < stage_hi_; ++k) {
      Stage& st = stages_[k];
      DeviceGuard g(st.device);
      cudaStream_t s = sched_->stream(k);
      if (k > stage_lo_) {
        // lambda_k := X_{kn} (the previous stage's output rows)
        const Stage& pv = stages_[k - 1];
        sched_->record(k - 1, StageScheduler::kStageDone);
        sched_->wait(k, k - 1, StageScheduler::kStageDone);
        cu(cudaMemcpyPeerAsync(st.lam.get() + (int64_t)r0 * feat(), st.device, pv.bout.get() + (int64_t)r0 * feat(),
                               pv.device, (size_t)nr * feat() * 4, s),
           "cudaMemcpyPeerAsync");
        in = st.lam.get() + (int64_t)r0 * feat();
      }
      run_forward(st, in, nr, st.bout.get() + (int64_t)r0 * feat(), s);
    }
  }
  if (has_ghost()) {
    // the ghost's lambda starts as this rank's boundary output (the downstream rank
    // receives the same rows as its stage input)
    Stage& gh = stages_[stage_hi_];
    const Stage& pv = stages_[stage_hi_ - 1];
    DeviceGuard g(gh.device);
    cudaStream_t s = sched_->stream(stage_hi_ - 1);
    cu(cudaMemcpyAsync(gh.lam.get(), pv.bout.get(), (size_t)num_samples_ * feat() * 4, cudaMemcpyDeviceToDevice, s),
       "cudaMemcpyAsync");
    gh.kappa.zero(s);
    gh.badj.zero(s);
    gh.kappa_zero = true;
  }
  for (int k = stage_lo_; k < stage_hi_; ++k) {
    Stage& st = stages_[k];
    DeviceGuard g(st.device);
    if (k > 0) st.kappa.zero(sched_->stream(k));
    st.badj.zero(sched_->stream(k));
    st.kappa_zero = true;
    st.version = iteration_;
    st.fwd_rows = 0;
  }
  sched_->sync();
  has_forward_ = true;
}

double DecoupledTrainer::step(const float* batch_x, const int32_t* labels, int nrows, int row0, const StepParams& p,
                              bool read_loss) {
  if (has_ghost() || stage_lo_ > 0)
    throw std::logic_error("step: this trainer holds stages [" + std::to_string(stage_lo_) + ", " +
                           std::to_string(stage_hi_) + ") only; use the distributed step");
  const bool single_pass = p.max_corrections <= 1 || p.tau < 0.0;   // no host-side psi test
  if (graphs_ && single_pass)
    step_graphed(batch_x, labels, nrows, row0, p);
  else
    step_local(batch_x, labels, nrows, row0, p);
  if (!read_loss) return 0.0;
  return last_loss();
}

void DecoupledTrainer::step_local(const float* batch_x, const int32_t* labels, int nrows, int row0,
                                  const StepParams& p) {
  check_rows(row0, nrows, "step");
  if (nrows < 1) throw ShapeError("step: empty batch");
  ensure_capacity(nrows);
  if (p.momentum != 0.0) ensure_momentum();
  ++iteration_;
  sched_->begin();
  // parallel phase: every stage's forward, synthetic/phi backward and update
  // (pool.run_iteration, decoupled.cpp:184-187).  Stage k reads lambda_{k+1}/kappa_{k+1}
  // directly: nothing writes them before the correction phase, so the iteration-start
  // snapshot of decoupled.cpp:65-73 is implicit.
  for (int k = stage_lo_; k < stage_hi_; ++k) {
    Stage& st = stages_[k];
    DeviceGuard g(st.device);
    cudaStream_t s = sched_->stream(k);
    const float* in = k == 0 ? batch_x : st.lam.get() + (int64_t)row0 * feat();
    run_forward(st, in, nrows, st.bout.get() + (int64_t)row0 * feat(), s);
    st.version = iteration_;
    st.fwd_rows = nrows;
    st.fwd_row0 = row0;
    run_backward(st, labels, nrows, row0, p.beta, p.lr, p.momentum, false, s);
    sched_->record(k, StageScheduler::kBackwardDone);
  }
  has_forward_ = true;
  // serial correction sweep (decoupled.cpp:189-192): boundaries are independent, so
  // boundary k runs on stage k's stream once stage k-1 is done.
  for (int k = stage_lo_ + 1; k < stage_hi_; ++k) {
    DeviceGuard g(stages_[k].device);
    sched_->wait(k, k - 1, StageScheduler::kBackwardDone);
    run_correction(k, p, row0, nrows, true, sched_->stream(k));
  }
  sched_->end();
}

void DecoupledTrainer::set_graphs(bool on) {
  graphs_ = on;
  if (!on && graph_exec_) {
    sched_->sync();
    cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
    graph_valid_ = false;
  }
}

uint64_t DecoupledTrainer::kappa_zero_mask() const {
  uint64_t m = 0;
  for (int k = 0; k < stages() && k < 64; ++k)
    if (owns_state(k) && stages_[k].kappa_zero) m |= 1ull << k;
  return m;
}

// One CUDA graph per iteration shape.  Capturing runs step_local's host logic (so the host
// bookkeeping -- iteration, versions, multiplier flags -- advances exactly as for an eager
// step) while the device work is recorded instead of executed; the graph is then launched
// once for this step.  Replays repeat the bookkeeping by hand and launch the graph.
void DecoupledTrainer::step_graphed(const float* batch_x, const int32_t* labels, int nrows, int row0,
                                    const StepParams& p) {
  check_rows(row0, nrows, "step");
  if (nrows < 1) throw ShapeError("step: empty batch");
  if (unique_devices_.size() > 1) {   // multi-device capture is not attempted
    step_local(batch_x, labels, nrows, row0, p);
    return;
  }
  ensure_capacity(nrows);
  if (p.momentum != 0.0) ensure_momentum();   // before the capture: no allocation inside it
  GraphKey key;
  key.x = batch_x;
  key.y = labels;
  key.nrows = nrows;
  key.row0 = row0;
  key.beta = p.beta;
  key.tau = p.tau;
  key.lr = p.lr;
  key.lambda_lr = p.lambda_lr;
  key.kappa_lr = p.kappa_lr;
  key.momentum = p.momentum;
  key.max_corrections = p.max_corrections;
  key.kappa_zero_mask = kappa_zero_mask();
  key.alloc_epoch = alloc_epoch_;
  cudaStream_t ctl = sched_->control();
  DeviceGuard g(sched_->control_device());
  if (graph_valid_ && key == graph_key_) {
    ++iteration_;
    for (int k = stage_lo_; k < stage_hi_; ++k) {
      Stage& st = stages_[k];
      st.version = iteration_;
      st.fwd_rows = nrows;
      st.fwd_row0 = row0;
    }
    has_forward_ = true;
    cu(cudaGraphLaunch(graph_exec_, ctl), "cudaGraphLaunch");
    rp::note_launches(graph_kernels_);
    return;
  }
  if (graph_exec_) {
    cu(cudaStreamSynchronize(ctl), "cudaStreamSynchronize");
    cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
  }
  graph_valid_ = false;
  cudaGraph_t graph = nullptr;
  cu(cudaStreamBeginCapture(ctl, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  try {
    step_local(batch_x, labels, nrows, row0, p);
  } catch (...) {
    cudaStreamEndCapture(ctl, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  cu(cudaStreamEndCapture(ctl, &graph), "cudaStreamEndCapture");
  size_t nnodes = 0;
  cu(cudaGraphGetNodes(graph, nullptr, &nnodes), "cudaGraphGetNodes");
  std::vector<cudaGraphNode_t> nodes(nnodes);
  if (nnodes) cu(cudaGraphGetNodes(graph, nodes.data(), &nnodes), "cudaGraphGetNodes");
  graph_kernels_ = 0;
  for (cudaGraphNode_t n : nodes) {
    cudaGraphNodeType t;
    cu(cudaGraphNodeGetType(n, &t), "cudaGraphNodeGetType");
    if (t == cudaGraphNodeTypeKernel) ++graph_kernels_;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  cu(e, "cudaGraphInstantiate");
  graph_exec_ = exec;
  // the key is taken after the captured step: its multiplier flags are the replay's
  graph_key_ = key;
  graph_key_.kappa_zero_mask = kappa_zero_mask();
  graph_valid_ = graph_key_.kappa_zero_mask == key.kappa_zero_mask;   // replayable as is
  cu(cudaGraphLaunch(graph_exec_, ctl), "cudaGraphLaunch");
}

void DecoupledTrainer::correct_ghost_rows(const StepParams& p, int row0, int nrows, int sub0, int subn) {
  if (!has_ghost()) throw std::logic_error("correct_ghost: this trainer owns the last stage");
  check_rows(row0, nrows, "correct_ghost");
  if (sub0 < 0 || subn < 0 || sub0 + subn > nrows) throw std::invalid_argument("correct_ghost: bad row sub-range");
  DeviceGuard g(stages_[stage_hi_ - 1].device);
  run_correction(stage_hi_, p, row0, nrows, true, sched_->stream(stage_hi_ - 1), sub0, subn);
  // the multiplier state is non-zero once the last chunk of an ALM correction ran
  if (mode_ == TrainMode::Alm && sub0 + subn == nrows) stages_[stage_hi_].kappa_zero = false;
}

void DecoupledTrainer::prepare(int nrows, const StepParams& p) {
  check_rows(0, nrows, "prepare");
  ensure_capacity(nrows);
  if (p.momentum != 0.0) ensure_momentum();
}

void DecoupledTrainer::note_replayed_step(int nrows, int row0) {
  ++iteration_;
  for (int k = stage_lo_; k < stage_hi_; ++k) {
    Stage& st = stages_[k];
    st.version = iteration_;
    st.fwd_rows = nrows;
    st.fwd_row0 = row0;
  }
  has_forward_ = true;
}

void DecoupledTrainer::correct_ghost(const StepParams& p, int row0, int nrows) {
  if (!has_ghost()) throw std::logic_error("correct_ghost: this trainer owns the last stage");
  check_rows(row0, nrows, "correct_ghost");
  // runs on the stream of stage_hi - 1, after its backward and the receive of p
  DeviceGuard g(stages_[stage_hi_ - 1].device);
  run_correction(stage_hi_, p, row0, nrows, true, sched_->stream(stage_hi_ - 1));
}

float* DecoupledTrainer::state_device(int k, int which) {
  if (k < 0 || k >= stages()) throw std::out_of_range("state: bad stage index");
  if (which < 0 || which > 3) throw std::invalid_argument("state: which must be 0..3");
  if (!owns_state(k)) throw std::invalid_argument("state: stage " + std::to_string(k) + " is not held by this rank");
  Stage& st = stages_[k];
  DeviceArray* arr[4] = {&st.lam, &st.kappa, &st.bout, &st.badj};
  if (arr[which]->bytes() == 0) throw std::invalid_argument("state: stage " + std::to_string(k) + " has no such buffer");
  return arr[which]->get();
}

double* DecoupledTrainer::loss_device() {
  if (stage_hi_ != stages()) throw std::logic_error("loss: the last stage is not local");
  return stages_.back().loss.get<double>();
}

double DecoupledTrainer::last_loss() const {
  if (stage_hi_ != stages()) throw std::logic_error("last_loss: the last stage is not local");
  const Stage& st = stages_.back();
  double v = 0.0;
  DeviceGuard g(sched_->control_device());
  cu(cudaMemcpyAsync(&v, st.loss.get(), 8, cudaMemcpyDeviceToHost, sched_->control()), "cudaMemcpyAsync D2H");
  cu(cudaStreamSynchronize(sched_->control()), "cudaStreamSynchronize");
  return v;
}

void DecoupledTrainer::take_snapshot(int k, int row0, int nrows) {
  if (k < 0 || k >= stages() - 1)
    throw std::invalid_argument("take_snapshot: stage " + std::to_string(k) + " has no downstream neighbour");
  need_local(k, "take_snapshot");
  check_rows(row0, nrows, "take_snapshot");
  Stage& st = stages_[k];
  const Stage& nx = stages_[k + 1];
  const int64_t bytes = std::max<int64_t>(4, (int64_t)nrows * feat() * 4);
  st.snap_lam.allocate(st.device, bytes);
  st.snap_kappa.allocate(st.device, bytes);
  sched_->sync();
  DeviceGuard g(st.device);
  cu(cudaMemcpyPeer(st.snap_lam.get(), st.device, nx.lam.get() + (int64_t)row0 * feat(), nx.device,
                    (size_t)nrows * feat() * 4),
     "cudaMemcpyPeer");
  cu(cudaMemcpyPeer(st.snap_kappa.get(), st.device, nx.kappa.get() + (int64_t)row0 * feat(), nx.device,
                    (size_t)nrows * feat() * 4),
     "cudaMemcpyPeer");
  st.snap_has_kappa = !nx.kappa_zero;
  st.snap_rows = nrows;
}

void DecoupledTrainer::stage_forward(int k, const float* batch_x, int nrows, int row0) {
  if (k < 0 || k >= stages()) throw std::out_of_range("stage_forward: bad stage index");
  need_local(k, "stage_forward");
  check_rows(row0, nrows, "stage_forward");
  ensure_capacity(std::max(nrows, 1));
  Stage& st = stages_[k];
  DeviceGuard g(st.device);
  cudaStream_t s = sched_->stream(k);
  const float* in = k == 0 ? batch_x : st.lam.get() + (int64_t)row0 * feat();
  run_forward(st, in, nrows, st.bout.get() + (int64_t)row0 * feat(), s);
  st.version = iteration_;
  st.fwd_rows = nrows;
  st.fwd_row0 = row0;
  has_forward_ = true;
  cu(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

NetGrads DecoupledTrainer::stage_grads(int k) const {
  if (k < 0 || k >= stages()) throw std::out_of_range("stage_grads: bad stage index");
  need_local(k, "stage_grads");
  sched_->sync();
  const Layout L(geo_);
  const Stage& st = stages_[k];
  int64_t beg = L.block0 + (int64_t)st.begin * L.block_stride;
  int64_t end = L.block0 + (int64_t)st.end * L.block_stride;
  if (k == 0) beg = 0;
  if (k == stages() - 1) end = L.total;
  NetGrads g;
  g.begin = beg;
  g.values.resize((size_t)(end - beg));
  DeviceGuard dg(st.device);
  const float* src = grads_[dev_index(unique_devices_, st.device)].get();
  cu(cudaMemcpy(g.values.data(), src + beg, (size_t)(end - beg) * 4, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  return g;
}

NetGrads DecoupledTrainer::stage_backward_update(int k, const int32_t* labels, double beta, double lr, int row0,
                                                 double momentum) {
  if (k < 0 || k >= stages()) throw std::out_of_range("stage_backward_update: bad stage index");
  need_local(k, "stage_backward_update");
  Stage& st = stages_[k];
  if (st.version != iteration_ || st.fwd_rows == 0)
    throw std::logic_error("stage_backward_update: stage " + std::to_string(k) +
                           " has no forward pass for this iteration");
  const int nrows = st.fwd_rows;
  check_rows(row0, nrows, "stage_backward_update");
  if (k < stages() - 1) {
    if (st.snap_rows < 0)
      throw std::invalid_argument("stage_backward_update: stage " + std::to_string(k) +
                                  " needs the (lambda, kappa) snapshot of stage " + std::to_string(k + 1));
    if (st.snap_rows != nrows) throw ShapeError("stage_backward_update: snapshot rows do not match the batch");
  }
  if (momentum != 0.0) ensure_momentum();
  {
    DeviceGuard g(st.device);
    cudaStream_t s = sched_->stream(k);
    run_backward(st, labels, nrows, row0, beta, lr, momentum, true, s);
    cu(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  }
  return stage_grads(k);
}

void DecoupledTrainer::correct_aux(int k, const StepParams& p, int row0, int nrows) {
  if (k < 1 || k >= stages())
    throw std::invalid_argument("correction: stage " + std::to_string(k) +
                                " out of range (lambda_0 is fixed to the true input)");
  if (!has_forward_) throw std::logic_error("correct_aux before any forward pass");
  need_local(k - 1, "correct_aux");
  check_rows(row0, nrows, "correct_aux");
  sched_->sync();
  DeviceGuard g(stages_[k].device);
  run_correction(k, p, row0, nrows, false, sched_->stream(k));
  sched_->sync();
}

void DecoupledTrainer::correct_multiplier(int k, double beta, double kappa_lr, int row0, int nrows) {
  if (k < 1 || k >= stages())
    throw std::invalid_argument("correction: stage " + std::to_string(k) +
                                " out of range (lambda_0 is fixed to the true input)");
  if (kind_ != PenaltyKind::SquaredL2)
    throw std::logic_error("correct_multiplier: the multiplier update is only derived for the squared_l2 penalty");
  need_local(k - 1, "correct_multiplier");
  check_rows(row0, nrows, "correct_multiplier");
  sched_->sync();
  Stage& st = stages_[k];
  const int64_t off = (int64_t)row0 * feat();
  const long norm = normalizer(nrows, (int)feat());
  const double coef = kappa_rule_ == RP_KAPPA_RULE_TEXTBOOK ? -beta : kappa_lr * (double)norm / (2.0 * beta);
  DeviceGuard g(st.device);
  check(rp_op_correct((int)kind_, st.lam.get() + off, stages_[k - 1].bout.get() + off, nullptr, st.kappa.get() + off,
                      (int64_t)nrows * feat(), 0.0, 0.0, 0, coef, 1, st.red_ws.get(), sched_->stream(k)));
  st.kappa_zero = false;
  sched_->sync();
}

void DecoupledTrainer::correction_gradient(int k, double beta, int row0, int nrows, float* out) const {
  if (k < 1 || k >= stages())
    throw std::invalid_argument("correction: stage " + std::to_string(k) +
                                " out of range (lambda_0 is fixed to the true input)");
  need_local(k - 1, "correction_gradient");
  check_rows(row0, nrows, "correction_gradient");
  sched_->sync();
  const Stage& st = stages_[k];
  const int64_t off = (int64_t)row0 * feat();
  const int64_t n = (int64_t)nrows * feat();
  const double w = beta / static_cast<double>(normalizer(nrows, (int)feat()));
  DeviceGuard g(st.device);
  cudaStream_t s = sched_->stream(k);
  // g = w d_lambda psi + p - kappa   (decoupled.cpp:124-133)
  check(rp_op_psi_grad((int)kind_, st.lam.get() + off, stages_[k - 1].bout.get() + off, n, w, out, st.red_ws.get(), s));
  check(rp_op_sgd(out, st.badj.get() + off, nullptr, n, -1.0, 0.0, s));   // out += p
  check(rp_op_sgd(out, st.kappa.get() + off, nullptr, n, 1.0, 0.0, s));   // out -= kappa
  cu(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

ViolationReport DecoupledTrainer::violation_report() const {
  if (!has_forward_) throw std::logic_error("violation_report: no forward pass has cached boundary states yet");
  sched_->sync();
  ViolationReport r;
  r.normalizer = normalizer(num_samples_, (int)feat());
  r.per_stage.push_back(0.0);
  for (int k = 1; k < stages(); ++k) {
    // boundary k is reported by the holder of stage k-1 (0 for the other ranks' boundaries)
    if (!is_local(k - 1)) {
      r.per_stage.push_back(0.0);
      continue;
    }
    const Stage& st = stages_[k];
    DeviceGuard g(st.device);
    double v = 0.0;
    check(rp_op_psi((int)kind_, st.lam.get(), stages_[k - 1].bout.get(), (int64_t)num_samples_ * feat(), &v,
                    st.red_ws.get(), sched_->stream(k)));
    r.per_stage.push_back(v);
  }
  for (double v : r.per_stage) r.max_violation = std::max(r.max_violation, v);
  return r;
}

void DecoupledTrainer::forward(const float* x, int nrows, float* logits) {
  if (stage_lo_ != 0 || stage_hi_ != stages()) throw std::logic_error("forward: needs every stage on this trainer");
  forward_local(x, nrows, logits);
}

void DecoupledTrainer::forward_local(const float* x, int nrows, float* out) {
  sched_->sync();
  if (nrows <= 0) return;
  if (unique_devices_.size() > 1) throw std::logic_error("forward: eval on multi-device trainers is not supported");
  const int chunk = std::max(1, std::min(nrows, std::max(256, stages_[stage_lo_].cap_rows)));
  ensure_capacity(chunk);
  eval_a_.allocate(stages_[stage_lo_].device, (int64_t)chunk * feat() * 4);
  eval_b_.allocate(stages_[stage_lo_].device, (int64_t)chunk * feat() * 4);
  cudaStream_t s = sched_->stream(stage_lo_);
  DeviceGuard g(stages_[stage_lo_].device);
  const bool last = stage_hi_ == stages();
  const int64_t in_stride = stage_lo_ == 0 ? raw_feat() : feat();
  for (int r0 = 0; r0 < nrows; r0 += chunk) {
    const int nr = std::min(chunk, nrows - r0);
    const float* in = x + (int64_t)r0 * in_stride;
    float* bufs[2] = {eval_a_.get(), eval_b_.get()};
    for (int k = stage_lo_; k < stage_hi_; ++k) {
      Stage& st = stages_[k];
      float* o = (!last && k == stage_hi_ - 1) ? out + (int64_t)r0 * feat() : bufs[(k - stage_lo_) & 1];
      // run_forward records tape pointers; eval does not touch trainer state otherwise
      const float* saved_in0 = st.input0;
      const float* saved_raw = st.raw;
      run_forward(st, in, nr, o, s);
      st.input0 = saved_in0;
      st.raw = saved_raw;
      in = o;
    }
    if (last) {
      const Stage& lst = stages_.back();
      cu(cudaMemcpyAsync(out + (int64_t)r0 * geo_.classes, lst.logits.get(), (size_t)nr * geo_.classes * 4,
                         cudaMemcpyDeviceToDevice, s),
         "cudaMemcpyAsync");
    }
  }
  cu(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  // eval clobbered the tapes: a following stage_backward_update needs a fresh forward
  for (int k = stage_lo_; k < stage_hi_; ++k) stages_[k].version = -1;
}

int64_t DecoupledTrainer::state_elems(int k, int which) const {
  if (k < 0 || k >= stages()) throw std::out_of_range("state: bad stage index");
  if (which < 0 || which > 3) throw std::invalid_argument("state: which must be 0..3");
  if (k == 0 && which < 2) return 0;
  if (!owns_state(k)) throw std::invalid_argument("state: stage " + std::to_string(k) + " is not held by this rank");
  if (!is_local(k) && which == 2) throw std::invalid_argument("state: the ghost stage has no boundary_out");
  return (int64_t)num_samples_ * feat();
}

void DecoupledTrainer::get_state(int k, int which, float* host) const {
  const int64_t n = state_elems(k, which);
  if (n == 0) return;
  sched_->sync();
  const Stage& st = stages_[k];
  const DeviceArray* arr[4] = {&st.lam, &st.kappa, &st.bout, &st.badj};
  DeviceGuard g(st.device);
  cu(cudaMemcpy(host, arr[which]->get(), n * 4, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
}

void DecoupledTrainer::set_state(int k, int which, const float* host) {
  const int64_t n = state_elems(k, which);
  if (n == 0) throw ShapeError("set_state: stage 0 has no lambda/kappa");
  sched_->sync();
  Stage& st = stages_[k];
  DeviceArray* arr[4] = {&st.lam, &st.kappa, &st.bout, &st.badj};
  DeviceGuard g(st.device);
  cu(cudaMemcpy(arr[which]->get(), host, n * 4, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  if (which == 1) st.kappa_zero = false;
}

}  // namespace respar::b200
