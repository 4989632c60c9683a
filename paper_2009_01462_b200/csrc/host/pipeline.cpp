// StagePipeline (pipeline.hpp): the stage-sharded training iteration over NCCL.
#include "pipeline.hpp"

#include <algorithm>
#include <string>

namespace rp {
void note_launches(uint64_t n);
}

namespace respar::b200 {

namespace {

void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(RP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaEvent_t make_event() {
  cudaEvent_t e = nullptr;
  cu(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  return e;
}

constexpr int kMaxChunks = 16;

}  // namespace

bool StagePipeline::Key::operator==(const Key& o) const {
  return x == o.x && y == o.y && nrows == o.nrows && row0 == o.row0 && chunks == o.chunks && beta == o.beta &&
         tau == o.tau && lr == o.lr && lambda_lr == o.lambda_lr && kappa_lr == o.kappa_lr &&
         momentum == o.momentum && max_corrections == o.max_corrections && masks == o.masks;
}

StagePipeline::StagePipeline(NcclComm* comm_a, NcclComm* comm_b, std::vector<Member> members, int chunks)
    : ca_(comm_a), cb_(comm_b), m_(std::move(members)), chunks_(std::max(1, std::min(chunks, kMaxChunks))) {
  if (!ca_ || !cb_) throw std::invalid_argument("StagePipeline: needs two communicators");
  if (ca_->rank() != cb_->rank() || ca_->nranks() != cb_->nranks() || ca_->device() != cb_->device())
    throw std::invalid_argument("StagePipeline: the two communicators must span the same ranks and device");
  if (m_.empty()) throw std::invalid_argument("StagePipeline: no local stages");
  device_ = ca_->device();
  const int K = m_[0].trainer->stages();
  for (size_t e = 0; e < m_.size(); ++e) {
    const Member& mb = m_[e];
    DecoupledTrainer& t = *mb.trainer;
    if (t.stages() != K) throw std::invalid_argument("StagePipeline: members disagree on the stage count");
    if (t.scheduler().device_of(t.stage_lo()) != device_)
      throw std::invalid_argument("StagePipeline: a member lives on another device than its communicator");
    if ((t.stage_lo() > 0) != (mb.prev_peer >= 0) || (t.stage_hi() < K) != (mb.next_peer >= 0))
      throw std::invalid_argument("StagePipeline: peers do not match the members' stage ranges");
    if (e > 0 && m_[e - 1].trainer->stage_hi() != t.stage_lo())
      throw std::invalid_argument("StagePipeline: members must hold consecutive stage ranges");
    for (int p : {mb.prev_peer, mb.next_peer})
      if (p >= ca_->nranks()) throw std::invalid_argument("StagePipeline: peer rank out of range");
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cu(cudaSetDevice(device_), "cudaSetDevice");
  cu(cudaStreamCreateWithFlags(&sa_, cudaStreamNonBlocking), "cudaStreamCreate");
  cu(cudaStreamCreateWithFlags(&sb_, cudaStreamNonBlocking), "cudaStreamCreate");
  cu(cudaStreamCreateWithFlags(&ctl_, cudaStreamNonBlocking), "cudaStreamCreate");
  ev_a_.resize(kMaxChunks);
  ev_c_.resize(m_.size() * kMaxChunks);
  for (auto& e : ev_a_) e = make_event();
  for (auto& e : ev_c_) e = make_event();
  ev_a_end_ = make_event();
  ev_b_end_ = make_event();
  ev_c_end_ = make_event();
  ev_fork_ = make_event();
  ev_join_.resize(m_.size());
  for (auto& e : ev_join_) e = make_event();
  cu(cudaEventCreate(&ev_rb_), "cudaEventCreate");
  cu(cudaEventCreate(&ev_re_), "cudaEventCreate");
  cudaSetDevice(prev);
}

StagePipeline::~StagePipeline() {
  cudaSetDevice(device_);
  cudaStreamSynchronize(sa_);
  cudaStreamSynchronize(sb_);
  cudaStreamSynchronize(ctl_);
  if (exec_) cudaGraphExecDestroy(exec_);
  for (auto e : ev_a_) cudaEventDestroy(e);
  for (auto e : ev_c_) cudaEventDestroy(e);
  for (auto e : ev_join_) cudaEventDestroy(e);
  for (auto e : {ev_a_end_, ev_b_end_, ev_c_end_, ev_fork_, ev_rb_, ev_re_}) cudaEventDestroy(e);
  cudaStreamDestroy(sa_);
  cudaStreamDestroy(sb_);
  cudaStreamDestroy(ctl_);
}

bool StagePipeline::has_last_stage() const { return m_.back().next_peer < 0; }

double StagePipeline::loss() {
  if (!has_last_stage()) throw std::logic_error("loss: the last stage is not on this process");
  sync();   // a replayed graph runs on the pipeline's stream, not the trainer's
  return m_.back().trainer->last_loss();
}

int StagePipeline::effective_chunks(int nrows, const StepParams& p) const {
  // the chunked correction is elementwise: the L-inf penalty (an argmax over the batch) and
  // the tau-loop (psi over the batch) correct the whole boundary at once
  if (m_[0].trainer->penalty_kind() == PenaltyKind::LInf || (p.max_corrections > 1 && p.tau >= 0.0)) return 1;
  return std::max(1, std::min(chunks_, nrows));
}

void StagePipeline::sync() {
  cudaSetDevice(device_);
  for (const Member& mb : m_) mb.trainer->scheduler().sync();
  cu(cudaStreamSynchronize(sa_), "cudaStreamSynchronize");
  cu(cudaStreamSynchronize(sb_), "cudaStreamSynchronize");
  cu(cudaStreamSynchronize(ctl_), "cudaStreamSynchronize");
}

void StagePipeline::reset_lambda_from_forward(const float* x_full) {
  sync();
  const int64_t feat = (int64_t)m_[0].trainer->geometry().height * m_[0].trainer->geometry().width *
                       m_[0].trainer->geometry().channels;
  const int N = m_[0].trainer->num_samples();
  const size_t count = (size_t)N * feat;
  for (size_t e = 0; e < m_.size(); ++e) {
    DecoupledTrainer& t = *m_[e].trainer;
    const bool local_prev = e > 0;   // the previous member already handed its boundary over below
    if (m_[e].prev_peer >= 0 && !local_prev) {
      ca_->group_start();
      ca_->recv(t.state_device(t.stage_lo(), 0), count, m_[e].prev_peer, sa_);
      ca_->group_end();
      cu(cudaStreamSynchronize(sa_), "cudaStreamSynchronize");
    }
    t.reset_lambda_from_forward(t.stage_lo() == 0 ? x_full : nullptr);   // synchronous
    if (m_[e].next_peer >= 0) {
      // the ghost's lambda now holds this member's boundary output: it is the next stage's input
      ca_->group_start();
      ca_->send(t.state_device(t.stage_hi(), 0), count, m_[e].next_peer, sa_);
      if (e + 1 < m_.size()) {
        DecoupledTrainer& u = *m_[e + 1].trainer;
        ca_->recv(u.state_device(u.stage_lo(), 0), count, m_[e + 1].prev_peer, sa_);
      }
      ca_->group_end();
      cu(cudaStreamSynchronize(sa_), "cudaStreamSynchronize");
    }
  }
  ca_->check_async();
  first_ = true;
}

StagePipeline::Key StagePipeline::make_key(const float* x, const int32_t* y, int nrows, int row0,
                                           const StepParams& p) const {
  Key k;
  k.x = x;
  k.y = y;
  k.nrows = nrows;
  k.row0 = row0;
  k.chunks = effective_chunks(nrows, p);
  k.beta = p.beta;
  k.tau = p.tau;
  k.lr = p.lr;
  k.lambda_lr = p.lambda_lr;
  k.kappa_lr = p.kappa_lr;
  k.momentum = p.momentum;
  k.max_corrections = p.max_corrections;
  for (const Member& mb : m_) {
    k.masks.push_back(mb.trainer->kappa_zero_mask());
    k.masks.push_back(mb.trainer->alloc_epoch());
  }
  return k;
}

void StagePipeline::set_graphs(bool on) {
  graphs_ = on;
  if (!on && exec_) {
    sync();
    cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
    graph_valid_ = false;
    first_ = true;
  }
}

void StagePipeline::step(const float* x, const int32_t* labels, int nrows, int row0, const StepParams& p) {
  if (nrows < 1) throw ShapeError("step: empty batch");
  cudaSetDevice(device_);
  for (const Member& mb : m_) mb.trainer->prepare(nrows, p);   // every allocation before any capture
  const bool single_pass = p.max_corrections <= 1 || p.tau < 0.0;
  if (!graphs_ || !single_pass) {
    step_eager(x, labels, nrows, row0, p);
    return;
  }
  const Key key = make_key(x, labels, nrows, row0, p);
  if (graph_valid_ && key == key_) {
    for (const Member& mb : m_) mb.trainer->note_replayed_step(nrows, row0);
    cu(cudaGraphLaunch(exec_, ctl_), "cudaGraphLaunch");
    rp::note_launches(graph_kernels_);
    return;
  }
  if (exec_) {
    sync();
    cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
  }
  graph_valid_ = false;
  // eager work enqueued before (and the previous iteration's events) completes first: a
  // captured step carries its iteration-to-iteration order through the graph launches
  sync();
  first_ = true;
  cudaGraph_t graph = nullptr;
  cu(cudaStreamBeginCapture(ctl_, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  try {
    cu(cudaEventRecord(ev_fork_, ctl_), "cudaEventRecord");
    for (const Member& mb : m_)
      cu(cudaStreamWaitEvent(mb.trainer->scheduler().control(), ev_fork_, 0), "cudaStreamWaitEvent");
    cu(cudaStreamWaitEvent(sa_, ev_fork_, 0), "cudaStreamWaitEvent");
    cu(cudaStreamWaitEvent(sb_, ev_fork_, 0), "cudaStreamWaitEvent");
    step_eager(x, labels, nrows, row0, p);
    for (size_t e = 0; e < m_.size(); ++e) {
      cu(cudaEventRecord(ev_join_[e], m_[e].trainer->scheduler().control()), "cudaEventRecord");
      cu(cudaStreamWaitEvent(ctl_, ev_join_[e], 0), "cudaStreamWaitEvent");
    }
    cu(cudaStreamWaitEvent(ctl_, ev_a_end_, 0), "cudaStreamWaitEvent");
    cu(cudaStreamWaitEvent(ctl_, ev_b_end_, 0), "cudaStreamWaitEvent");
    cu(cudaStreamWaitEvent(ctl_, ev_c_end_, 0), "cudaStreamWaitEvent");
  } catch (...) {
    cudaStreamEndCapture(ctl_, &graph);
    if (graph) cudaGraphDestroy(graph);
    first_ = true;
    throw;
  }
  cu(cudaStreamEndCapture(ctl_, &graph), "cudaStreamEndCapture");
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
  exec_ = exec;
  // the key after the captured step: its multiplier flags are the ones a replay starts from
  key_ = make_key(x, labels, nrows, row0, p);
  graph_valid_ = key_.masks == key.masks;
  cu(cudaGraphLaunch(exec_, ctl_), "cudaGraphLaunch");
  first_ = true;   // the next eager step (if any) must not wait on events recorded inside the capture
}

void StagePipeline::step_eager(const float* x, const int32_t* labels, int nrows, int row0, const StepParams& p) {
  const int C = effective_chunks(nrows, p);
  const int K = m_[0].trainer->stages();
  const int64_t feat = (int64_t)m_[0].trainer->geometry().height * m_[0].trainer->geometry().width *
                       m_[0].trainer->geometry().channels;
  auto rows = [&](int j) { return std::make_pair(j * nrows / C, (j + 1) * nrows / C - j * nrows / C); };
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cu(cudaStreamIsCapturing(ctl_, &cs), "cudaStreamIsCapturing");
  const bool capturing = cs == cudaStreamCaptureStatusActive;
  const bool chain = !first_ && !capturing;   // order after the previous (eager) iteration's events

  // 1. every member's local stages: forward, synthetic / phi backward, SGD, inner corrections
  for (const Member& mb : m_) {
    DecoupledTrainer& t = *mb.trainer;
    const int lo = t.stage_lo();
    if (chain && mb.prev_peer >= 0) {
      // lambda_lo of this iteration has arrived, and p_lo of the last one has left
      cu(cudaStreamWaitEvent(t.scheduler().stream(lo), ev_b_end_, 0), "cudaStreamWaitEvent");
      cu(cudaStreamWaitEvent(t.scheduler().stream(lo), ev_a_end_, 0), "cudaStreamWaitEvent");
    }
    t.step_local(lo == 0 ? x : nullptr, t.stage_hi() == K ? labels : nullptr, nrows, row0, p);
  }
  // 2. exchange A: p_lo upstream, p_hi into the ghost's adjoint rows, chunk by chunk
  if (chain) cu(cudaStreamWaitEvent(sa_, ev_c_end_, 0), "cudaStreamWaitEvent");   // ghost adjoints read
  for (const Member& mb : m_)
    if (mb.prev_peer >= 0)
      cu(cudaStreamWaitEvent(sa_, mb.trainer->scheduler().mark_event(mb.trainer->stage_lo(),
                                                                      StageScheduler::kBackwardDone), 0),
         "cudaStreamWaitEvent");
  for (int j = 0; j < C; ++j) {
    const auto [r0, rn] = rows(j);
    const size_t off = (size_t)(row0 + r0) * feat, cnt = (size_t)rn * feat;
    ca_->group_start();
    for (const Member& mb : m_) {
      DecoupledTrainer& t = *mb.trainer;
      if (mb.prev_peer >= 0) ca_->send(t.state_device(t.stage_lo(), 3) + off, cnt, mb.prev_peer, sa_);
      if (mb.next_peer >= 0) ca_->recv(t.state_device(t.stage_hi(), 3) + off, cnt, mb.next_peer, sa_);
    }
    ca_->group_end();
    cu(cudaEventRecord(ev_a_[j], sa_), "cudaEventRecord");
  }
  cu(cudaEventRecord(ev_a_end_, sa_), "cudaEventRecord");
  // 3. the ghost boundaries' corrections, chunk j once its adjoint rows are in
  for (size_t e = 0; e < m_.size(); ++e) {
    const Member& mb = m_[e];
    if (mb.next_peer < 0) continue;
    DecoupledTrainer& t = *mb.trainer;
    cudaStream_t s = t.scheduler().stream(t.stage_hi() - 1);
    if (chain) cu(cudaStreamWaitEvent(s, ev_b_end_, 0), "cudaStreamWaitEvent");   // lambda_hi sent
    for (int j = 0; j < C; ++j) {
      const auto [r0, rn] = rows(j);
      cu(cudaStreamWaitEvent(s, ev_a_[j], 0), "cudaStreamWaitEvent");
      t.correct_ghost_rows(p, row0, nrows, r0, rn);
      cu(cudaEventRecord(ev_c_[e * kMaxChunks + j], s), "cudaEventRecord");
    }
  }
  // 4. exchange B: the corrected lambda_hi downstream, lambda_lo from upstream
  for (const Member& mb : m_)
    if (mb.prev_peer >= 0)
      cu(cudaStreamWaitEvent(sb_, mb.trainer->scheduler().mark_event(mb.trainer->stage_lo(),
                                                                      StageScheduler::kBackwardDone), 0),
         "cudaStreamWaitEvent");
  for (int j = 0; j < C; ++j) {
    const auto [r0, rn] = rows(j);
    const size_t off = (size_t)(row0 + r0) * feat, cnt = (size_t)rn * feat;
    for (size_t e = 0; e < m_.size(); ++e)
      if (m_[e].next_peer >= 0) cu(cudaStreamWaitEvent(sb_, ev_c_[e * kMaxChunks + j], 0), "cudaStreamWaitEvent");
    cb_->group_start();
    for (const Member& mb : m_) {
      DecoupledTrainer& t = *mb.trainer;
      if (mb.next_peer >= 0) cb_->send(t.state_device(t.stage_hi(), 0) + off, cnt, mb.next_peer, sb_);
      if (mb.prev_peer >= 0) cb_->recv(t.state_device(t.stage_lo(), 0) + off, cnt, mb.prev_peer, sb_);
    }
    cb_->group_end();
  }
  cu(cudaEventRecord(ev_b_end_, sb_), "cudaEventRecord");
  // every correction done (the next exchange A may overwrite the ghost adjoints)
  cu(cudaEventRecord(ev_c_end_, sb_), "cudaEventRecord");
  first_ = false;
}

void StagePipeline::region_begin() {
  cudaSetDevice(device_);
  cu(cudaEventRecord(ev_rb_, ctl_), "cudaEventRecord");
}

float StagePipeline::region_end() {
  cudaSetDevice(device_);
  for (size_t e = 0; e < m_.size(); ++e) {
    StageScheduler& s = m_[e].trainer->scheduler();
    for (int k = m_[e].trainer->stage_lo(); k < m_[e].trainer->stage_hi(); ++k) {
      s.record(k, StageScheduler::kStageDone);
      cu(cudaStreamWaitEvent(ctl_, s.mark_event(k, StageScheduler::kStageDone), 0), "cudaStreamWaitEvent");
    }
    cu(cudaEventRecord(ev_join_[e], s.control()), "cudaEventRecord");
    cu(cudaStreamWaitEvent(ctl_, ev_join_[e], 0), "cudaStreamWaitEvent");
  }
  cudaEvent_t ea = make_event(), eb = make_event();
  cu(cudaEventRecord(ea, sa_), "cudaEventRecord");
  cu(cudaEventRecord(eb, sb_), "cudaEventRecord");
  cu(cudaStreamWaitEvent(ctl_, ea, 0), "cudaStreamWaitEvent");
  cu(cudaStreamWaitEvent(ctl_, eb, 0), "cudaStreamWaitEvent");
  cu(cudaEventRecord(ev_re_, ctl_), "cudaEventRecord");
  cu(cudaEventSynchronize(ev_re_), "cudaEventSynchronize");
  cudaEventDestroy(ea);
  cudaEventDestroy(eb);
  float ms = 0.f;
  cu(cudaEventElapsedTime(&ms, ev_rb_, ev_re_), "cudaEventElapsedTime");
  ca_->check_async();
  cb_->check_async();
  return ms;
}

}  // namespace respar::b200
