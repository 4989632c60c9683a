// C ABI, trainer layer (include/respar_b200.h "rp_trainer_*"): an opaque handle on
// respar::b200::DecoupledTrainer with one entry point per reference method
// (decoupled.hpp:56-120).  Host-buffer entry points stage inputs through device
// buffers owned by the trainer (the H2D copy is part of the call).
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "host/comm.hpp"
#include "host/pipeline.hpp"
#include "host/respar_b200.hpp"

namespace rp {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void note_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace rp

using respar::b200::DecoupledTrainer;
using respar::b200::StepParams;

struct rp_trainer {
  std::unique_ptr<DecoupledTrainer> tr;
  bool serial = false;
  respar::b200::DeviceArray eval_logits, eval_ws;   // rp_trainer_evaluate scratch
};

struct rp_comm {
  std::unique_ptr<respar::b200::NcclComm> c;
};

struct rp_pipeline {
  std::unique_ptr<respar::b200::StagePipeline> p;
};

namespace {

template <class F>
int tguard(F&& f) {
  try {
    f();
    return RP_OK;
  } catch (const rp::Error& e) {
    rp::set_last_error(e.what());
    return e.code;
  } catch (const std::out_of_range& e) {
    rp::set_last_error(e.what());
    return RP_ERR_RANGE;
  } catch (const std::exception& e) {
    rp::set_last_error(e.what());
    return respar::b200::status_of(e);
  } catch (...) {
    rp::set_last_error("unknown error");
    return RP_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

StepParams to_params(const rp_step_params* p) {
  StepParams s;
  if (p) {
    s.beta = p->beta;
    s.tau = p->tau;
    s.lr = p->lr;
    s.lambda_lr = p->lambda_lr;
    s.kappa_lr = p->kappa_lr;
    s.max_corrections = p->max_corrections;
    s.momentum = p->momentum;
  }
  if (s.lr < 0.0) throw std::invalid_argument("step: lr must be >= 0");
  return s;
}

void h2d(void* dst, const void* src, int64_t bytes) {
  if (bytes <= 0) return;
  cudaError_t e = cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) throw respar::b200::DeviceError(RP_ERR_CUDA, cudaGetErrorString(e));
}

void d2h(void* dst, const void* src, int64_t bytes) {
  if (bytes <= 0) return;
  cudaError_t e = cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) throw respar::b200::DeviceError(RP_ERR_CUDA, cudaGetErrorString(e));
}

int64_t raw_feat(const rp_geometry& g) { return (int64_t)g.height * g.width * g.in_channels; }

// loss_phi rejects labels outside [0, classes) (network.cpp:201-205)
void check_labels(const int32_t* y, int n, int classes) {
  for (int i = 0; i < n; ++i)
    if (y[i] < 0 || y[i] >= classes)
      throw std::invalid_argument("loss_phi: label " + std::to_string(y[i]) + " out of range for " +
                                  std::to_string(classes) + " classes");
}

const int32_t* stage_labels(DecoupledTrainer& tr, const int32_t* host, int n) {
  if (!host) return nullptr;
  check_labels(host, n, tr.geometry().classes);
  int32_t* dev = tr.label_staging(n);
  h2d(dev, host, (int64_t)n * 4);
  return dev;
}

const float* stage_input(DecoupledTrainer& tr, const float* host, int n) {
  float* dev = tr.input_staging(n);
  h2d(dev, host, (int64_t)n * raw_feat(tr.geometry()) * 4);
  return dev;
}

}  // namespace

extern "C" {

const char* rp_last_error(void) { return rp::g_last_error.c_str(); }
int rp_version(void) { return 1; }
uint64_t rp_launch_count(void) { return rp::g_launches.load(); }

int64_t rp_param_count(const rp_geometry* g) {
  if (!g) return -1;
  try {
    rp::validate_geometry(*g);
  } catch (const rp::Error& e) {
    rp::set_last_error(e.what());
    return -1;
  }
  return rp::ParamLayout::of(*g).total;
}

int64_t rp_param_offset_block(const rp_geometry* g, int32_t block) {
  if (!g || block < 0 || block > g->blocks) return -1;
  const rp::ParamLayout L = rp::ParamLayout::of(*g);
  return L.block0 + (int64_t)block * L.block_stride;
}

int64_t rp_param_offset_head(const rp_geometry* g) {
  if (!g) return -1;
  return rp::ParamLayout::of(*g).t_w;
}

int rp_trainer_create(const rp_geometry* g, int32_t stages, int32_t mode, int32_t penalty, int32_t num_samples,
                      const float* params_host, uint64_t* seed_state, int32_t math, const int32_t* devices,
                      int32_t ndev, rp_trainer** out) {
  return tguard([&] {
    need(g, "geometry");
    need(out, "out");
    *out = nullptr;
    if (rp_param_count(g) < 0) throw respar::b200::ConfigError(rp_last_error());
    if (mode < RP_MODE_SERIAL || mode > RP_MODE_ALM) throw respar::b200::ConfigError("unknown train mode");
    if (penalty < 0 || penalty > 2) throw respar::b200::ConfigError("unknown penalty kind");
    if (math < RP_MATH_FP32 || math > RP_MATH_SIMT) throw respar::b200::ConfigError("unknown math mode");
    if (mode == RP_MODE_SERIAL && stages != 1) throw respar::b200::ConfigError("serial mode runs exactly one stage");
    std::vector<int> devs;
    for (int i = 0; i < ndev; ++i) devs.push_back(devices[i]);
    auto h = std::make_unique<rp_trainer>();
    h->serial = mode == RP_MODE_SERIAL;
    h->tr = std::make_unique<DecoupledTrainer>(
        *g, stages, mode == RP_MODE_ALM ? respar::b200::TrainMode::Alm : respar::b200::TrainMode::Penalty,
        static_cast<respar::b200::PenaltyKind>(penalty), num_samples, math, devs);
    if (params_host) {
      h->tr->set_params(params_host);
    } else {
      need(seed_state, "seed_state");
      h->tr->init_params(*seed_state);
    }
    *out = h.release();
  });
}

int rp_trainer_create_local(const rp_geometry* g, int32_t stages, int32_t mode, int32_t penalty, int32_t num_samples,
                            const float* params_host, uint64_t* seed_state, int32_t math, int32_t device,
                            int32_t stage_lo, int32_t stage_hi, rp_trainer** out) {
  return tguard([&] {
    need(g, "geometry");
    need(out, "out");
    *out = nullptr;
    if (rp_param_count(g) < 0) throw respar::b200::ConfigError(rp_last_error());
    if (mode != RP_MODE_PENALTY && mode != RP_MODE_ALM)
      throw respar::b200::ConfigError("stage-sharded trainers run the penalty or ALM mode");
    if (penalty < 0 || penalty > 2) throw respar::b200::ConfigError("unknown penalty kind");
    if (math < RP_MATH_FP32 || math > RP_MATH_SIMT) throw respar::b200::ConfigError("unknown math mode");
    auto h = std::make_unique<rp_trainer>();
    h->tr = std::make_unique<DecoupledTrainer>(
        *g, stages, mode == RP_MODE_ALM ? respar::b200::TrainMode::Alm : respar::b200::TrainMode::Penalty,
        static_cast<respar::b200::PenaltyKind>(penalty), num_samples, math, std::vector<int>{device}, stage_lo,
        stage_hi);
    if (params_host) {
      h->tr->set_params(params_host);
    } else {
      need(seed_state, "seed_state");
      h->tr->init_params(*seed_state);
    }
    *out = h.release();
  });
}

int rp_trainer_local_range(rp_trainer* t, int32_t* stage_lo, int32_t* stage_hi) {
  return tguard([&] {
    need(t, "trainer");
    if (stage_lo) *stage_lo = t->tr->stage_lo();
    if (stage_hi) *stage_hi = t->tr->stage_hi();
  });
}

int rp_trainer_reset_local(rp_trainer* t, const float* x_dev) {
  return tguard([&] {
    need(t, "trainer");
    t->tr->reset_lambda_from_forward(x_dev);
  });
}

int rp_trainer_step_local(rp_trainer* t, const float* x_dev, const int32_t* labels_dev, int32_t nrows, int32_t row0,
                          const rp_step_params* p) {
  return tguard([&] {
    need(t, "trainer");
    DecoupledTrainer& tr = *t->tr;
    if (tr.stage_lo() == 0) need(x_dev, "x");
    if (tr.stage_hi() == tr.stages()) need(labels_dev, "labels");
    tr.step_local(x_dev, labels_dev, nrows, row0, to_params(p));
  });
}

int rp_trainer_correct_ghost(rp_trainer* t, const rp_step_params* p, int32_t row0, int32_t nrows) {
  return tguard([&] {
    need(t, "trainer");
    t->tr->correct_ghost(to_params(p), row0, nrows);
  });
}

int rp_trainer_state_device(rp_trainer* t, int32_t k, int32_t which, float** ptr) {
  return tguard([&] {
    need(t, "trainer");
    need(ptr, "ptr");
    *ptr = t->tr->state_device(k, which);
  });
}

int rp_trainer_stage_stream(rp_trainer* t, int32_t k, void** stream) {
  return tguard([&] {
    need(t, "trainer");
    need(stream, "stream");
    if (k < 0 || k >= t->tr->stages()) throw std::out_of_range("stage_stream: bad stage index");
    *stream = static_cast<void*>(t->tr->scheduler().stream(k));
  });
}

int rp_trainer_forward_local(rp_trainer* t, const float* in_dev, int32_t nrows, float* out_dev) {
  return tguard([&] {
    need(t, "trainer");
    if (nrows > 0) {
      need(in_dev, "in");
      need(out_dev, "out");
    }
    t->tr->forward_local(in_dev, nrows, out_dev);
  });
}

int rp_trainer_loss_device(rp_trainer* t, double** ptr) {
  return tguard([&] {
    need(t, "trainer");
    need(ptr, "ptr");
    *ptr = t->tr->loss_device();
  });
}

int rp_trainer_set_graphs(rp_trainer* t, int32_t on) {
  return tguard([&] {
    need(t, "trainer");
    t->tr->set_graphs(on != 0);
  });
}

int rp_trainer_destroy(rp_trainer* t) {
  return tguard([&] { delete t; });
}

int rp_trainer_set_kappa_rule(rp_trainer* t, int32_t rule) {
  return tguard([&] {
    need(t, "trainer");
    if (rule != RP_KAPPA_RULE_REFERENCE && rule != RP_KAPPA_RULE_TEXTBOOK)
      throw std::invalid_argument("unknown multiplier rule");
    t->tr->set_kappa_rule(rule);
  });
}

int rp_trainer_get_params(rp_trainer* t, float* host) {
  return tguard([&] {
    need(t, "trainer");
    need(host, "host");
    t->tr->get_params(host);
  });
}

int rp_trainer_set_params(rp_trainer* t, const float* host) {
  return tguard([&] {
    need(t, "trainer");
    need(host, "host");
    t->tr->set_params(host);
  });
}

int rp_trainer_get_grads(rp_trainer* t, float* host) {
  return tguard([&] {
    need(t, "trainer");
    need(host, "host");
    t->tr->get_grads(host);
  });
}

int rp_trainer_reset_lambda_from_forward(rp_trainer* t, const float* x_host) {
  return tguard([&] {
    need(t, "trainer");
    need(x_host, "x");
    DecoupledTrainer& tr = *t->tr;
    const float* x = stage_input(tr, x_host, tr.num_samples());
    tr.reset_lambda_from_forward(x);
  });
}

int rp_trainer_step(rp_trainer* t, const float* x_host, const int32_t* labels_host, int32_t nrows, int32_t row0,
                    const rp_step_params* p, double* loss_out) {
  return tguard([&] {
    need(t, "trainer");
    need(x_host, "x");
    need(labels_host, "labels");
    DecoupledTrainer& tr = *t->tr;
    const StepParams sp = to_params(p);
    const int32_t* y = stage_labels(tr, labels_host, nrows);
    const float* x = stage_input(tr, x_host, nrows);
    const double loss = tr.step(x, y, nrows, row0, sp, true);
    if (loss_out) *loss_out = loss;
  });
}

int rp_trainer_step_device(rp_trainer* t, const float* x_dev, const int32_t* labels_dev, int32_t nrows, int32_t row0,
                           const rp_step_params* p, double* loss_out) {
  return tguard([&] {
    need(t, "trainer");
    need(x_dev, "x");
    need(labels_dev, "labels");
    const double loss = t->tr->step(x_dev, labels_dev, nrows, row0, to_params(p), loss_out != nullptr);
    if (loss_out) *loss_out = loss;
  });
}

int rp_trainer_last_loss(rp_trainer* t, double* loss_out) {
  return tguard([&] {
    need(t, "trainer");
    need(loss_out, "loss_out");
    *loss_out = t->tr->last_loss();
  });
}

int rp_trainer_take_snapshot(rp_trainer* t, int32_t k, int32_t row0, int32_t nrows) {
  return tguard([&] {
    need(t, "trainer");
    t->tr->take_snapshot(k, row0, nrows);
  });
}

int rp_trainer_stage_forward(rp_trainer* t, int32_t k, const float* x_host, int32_t nrows, int32_t row0) {
  return tguard([&] {
    need(t, "trainer");
    DecoupledTrainer& tr = *t->tr;
    const float* x = nullptr;
    if (k == 0) {
      need(x_host, "x");
      x = stage_input(tr, x_host, nrows);
    }
    tr.stage_forward(k, x, nrows, row0);
  });
}

int rp_trainer_stage_backward_update(rp_trainer* t, int32_t k, const int32_t* labels_host, int32_t nrows, double beta,
                                     double lr, int32_t row0) {
  return tguard([&] {
    need(t, "trainer");
    DecoupledTrainer& tr = *t->tr;
    const int32_t* y = nullptr;
    if (k == tr.stages() - 1) {
      need(labels_host, "labels");
      y = stage_labels(tr, labels_host, nrows);
    }
    tr.stage_backward_update(k, y, beta, lr, row0);
  });
}

int rp_trainer_correct_aux(rp_trainer* t, int32_t k, const rp_step_params* p, int32_t row0, int32_t nrows) {
  return tguard([&] {
    need(t, "trainer");
    StepParams sp;
    if (p) {
      sp.beta = p->beta;
      sp.tau = p->tau;
      sp.lambda_lr = p->lambda_lr;
      sp.max_corrections = p->max_corrections;
    }
    t->tr->correct_aux(k, sp, row0, nrows);
  });
}

int rp_trainer_correct_multiplier(rp_trainer* t, int32_t k, double beta, double kappa_lr, int32_t row0,
                                  int32_t nrows) {
  return tguard([&] {
    need(t, "trainer");
    t->tr->correct_multiplier(k, beta, kappa_lr, row0, nrows);
  });
}

int rp_trainer_correction_gradient(rp_trainer* t, int32_t k, double beta, int32_t row0, int32_t nrows,
                                   float* out_host) {
  return tguard([&] {
    need(t, "trainer");
    need(out_host, "out");
    DecoupledTrainer& tr = *t->tr;
    const rp_geometry& g = tr.geometry();
    const int64_t n = (int64_t)nrows * g.height * g.width * g.channels;
    float* dev = nullptr;
    if (cudaMalloc(&dev, std::max<int64_t>(4, n * 4)) != cudaSuccess)
      throw respar::b200::DeviceError(RP_ERR_CUDA, "cudaMalloc");
    try {
      tr.correction_gradient(k, beta, row0, nrows, dev);
      d2h(out_host, dev, n * 4);
    } catch (...) {
      cudaFree(dev);
      throw;
    }
    cudaFree(dev);
  });
}

int rp_trainer_violation_report(rp_trainer* t, double* per_stage, double* max_violation, int64_t* normalizer) {
  return tguard([&] {
    need(t, "trainer");
    const respar::b200::ViolationReport r = t->tr->violation_report();
    if (per_stage)
      for (size_t i = 0; i < r.per_stage.size(); ++i) per_stage[i] = r.per_stage[i];
    if (max_violation) *max_violation = r.max_violation;
    if (normalizer) *normalizer = r.normalizer;
  });
}

int rp_trainer_get_state(rp_trainer* t, int32_t k, int32_t which, float* host) {
  return tguard([&] {
    need(t, "trainer");
    need(host, "host");
    t->tr->get_state(k, which, host);
  });
}

int rp_trainer_set_state(rp_trainer* t, int32_t k, int32_t which, const float* host) {
  return tguard([&] {
    need(t, "trainer");
    need(host, "host");
    t->tr->set_state(k, which, host);
  });
}

int rp_trainer_forward(rp_trainer* t, const float* x_host, int32_t nrows, float* logits_host) {
  return tguard([&] {
    need(t, "trainer");
    need(x_host, "x");
    need(logits_host, "logits");
    DecoupledTrainer& tr = *t->tr;
    const float* x = stage_input(tr, x_host, nrows);
    float* dev = nullptr;
    const int64_t bytes = std::max<int64_t>(4, (int64_t)nrows * tr.geometry().classes * 4);
    if (cudaMalloc(&dev, bytes) != cudaSuccess) throw respar::b200::DeviceError(RP_ERR_CUDA, "cudaMalloc");
    try {
      tr.forward(x, nrows, dev);
      d2h(logits_host, dev, (int64_t)nrows * tr.geometry().classes * 4);
    } catch (...) {
      cudaFree(dev);
      throw;
    }
    cudaFree(dev);
  });
}

int rp_trainer_evaluate(rp_trainer* t, const float* x_host, const int32_t* labels_host, int32_t nrows,
                        double* loss_out, double* accuracy_out) {
  return tguard([&] {
    need(t, "trainer");
    DecoupledTrainer& tr = *t->tr;
    if (nrows < 0) throw respar::b200::ShapeError("evaluate: negative row count");
    if (nrows == 0) {   // accuracy of nothing (network.cpp:226)
      if (loss_out) *loss_out = 0.0;
      if (accuracy_out) *accuracy_out = 0.0;
      return;
    }
    need(x_host, "x");
    need(labels_host, "labels");
    check_labels(labels_host, nrows, tr.geometry().classes);
    const float* x = stage_input(tr, x_host, nrows);
    const int32_t* y = stage_labels(tr, labels_host, nrows);
    const int dev = tr.scheduler().device_of(0);
    t->eval_logits.allocate(dev, std::max<int64_t>(4, (int64_t)nrows * tr.geometry().classes * 4));
    const int64_t wsb = rp_op_eval_workspace_bytes(nrows);
    t->eval_ws.allocate(dev, wsb);
    tr.forward(x, nrows, t->eval_logits.get());   // the full serial forward (synchronous)
    double loss = 0.0;
    int64_t hits = 0;
    const int rc = rp_op_eval_loss_accuracy(t->eval_logits.get(), y, nrows, tr.geometry().classes, &loss, &hits,
                                            nullptr, t->eval_ws.get(), wsb, nullptr);
    if (rc != RP_OK) respar::b200::throw_status(rc, rp_last_error());
    if (loss_out) *loss_out = loss;
    if (accuracy_out) *accuracy_out = (double)hits / (double)nrows;
  });
}

int64_t rp_trainer_iteration(rp_trainer* t) { return t ? t->tr->iteration() : -1; }
int32_t rp_trainer_stages(rp_trainer* t) { return t ? t->tr->stages() : -1; }

int rp_trainer_last_step_ms(rp_trainer* t, float* ms) {
  return tguard([&] {
    need(t, "trainer");
    need(ms, "ms");
    *ms = t->tr->last_step_ms();
  });
}

int rp_trainer_region(rp_trainer* t, int32_t which, float* ms) {
  return tguard([&] {
    need(t, "trainer");
    if (which == 0) {
      t->tr->scheduler().region_begin();
      if (ms) *ms = 0.f;
    } else {
      const float v = t->tr->scheduler().region_end();
      if (ms) *ms = v;
    }
  });
}

int rp_serial_train_step(rp_trainer* t, const float* x_host, const int32_t* labels_host, int32_t nrows, double lr,
                         double* loss_out) {
  return tguard([&] {
    need(t, "trainer");
    if (t->tr->stages() != 1) throw std::invalid_argument("serial_train_step: needs a one-stage (serial) trainer");
    if (lr < 0.0) throw std::invalid_argument("serial_train_step: lr must be >= 0");
    if (nrows > t->tr->num_samples()) throw respar::b200::ShapeError("serial_train_step: batch larger than the trainer");
    rp_step_params p{1.0, -1.0, lr, 0.0, 0.0, 1, 0.0};
    DecoupledTrainer& tr = *t->tr;
    const int32_t* y = stage_labels(tr, labels_host, nrows);
    const float* x = stage_input(tr, x_host, nrows);
    const double loss = tr.step(x, y, nrows, 0, to_params(&p), true);
    if (loss_out) *loss_out = loss;
  });
}

// ---- stage pipeline over NCCL (host/pipeline.hpp) ------------------------------------
int rp_comm_unique_id(uint8_t* id) {
  return tguard([&] {
    need(id, "id");
    respar::b200::NcclComm::unique_id(id);
  });
}

int rp_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, rp_comm** out) {
  return tguard([&] {
    need(id, "id");
    need(out, "out");
    *out = nullptr;
    auto h = std::make_unique<rp_comm>();
    h->c = std::make_unique<respar::b200::NcclComm>(id, nranks, rank, device);
    *out = h.release();
  });
}

int rp_comm_destroy(rp_comm* c) {
  return tguard([&] { delete c; });
}

int rp_pipeline_create(rp_comm* comm_a, rp_comm* comm_b, rp_trainer* const* trainers, const int32_t* prev_peer,
                       const int32_t* next_peer, int32_t n, int32_t chunks, rp_pipeline** out) {
  return tguard([&] {
    need(comm_a, "comm_a");
    need(comm_b, "comm_b");
    need(trainers, "trainers");
    need(prev_peer, "prev_peer");
    need(next_peer, "next_peer");
    need(out, "out");
    *out = nullptr;
    if (n < 1) throw std::invalid_argument("pipeline: no trainers");
    std::vector<respar::b200::StagePipeline::Member> m;
    for (int i = 0; i < n; ++i) {
      need(trainers[i], "trainer");
      m.push_back({trainers[i]->tr.get(), prev_peer[i], next_peer[i]});
    }
    auto h = std::make_unique<rp_pipeline>();
    h->p = std::make_unique<respar::b200::StagePipeline>(comm_a->c.get(), comm_b->c.get(), std::move(m), chunks);
    *out = h.release();
  });
}

int rp_pipeline_reset_lambda_from_forward(rp_pipeline* p, const float* x_full_dev) {
  return tguard([&] {
    need(p, "pipeline");
    p->p->reset_lambda_from_forward(x_full_dev);
  });
}

int rp_pipeline_step(rp_pipeline* p, const float* x_dev, const int32_t* labels_dev, int32_t nrows, int32_t row0,
                     const rp_step_params* sp, double* loss_out) {
  return tguard([&] {
    need(p, "pipeline");
    p->p->step(x_dev, labels_dev, nrows, row0, to_params(sp));
    if (loss_out) *loss_out = p->p->loss();
  });
}

int rp_pipeline_loss(rp_pipeline* p, double* loss_out) {
  return tguard([&] {
    need(p, "pipeline");
    need(loss_out, "loss_out");
    *loss_out = p->p->loss();
  });
}

int rp_pipeline_set_graphs(rp_pipeline* p, int32_t on) {
  return tguard([&] {
    need(p, "pipeline");
    p->p->set_graphs(on != 0);
  });
}

int rp_pipeline_region(rp_pipeline* p, int32_t which, float* ms) {
  return tguard([&] {
    need(p, "pipeline");
    if (which == 0) {
      p->p->region_begin();
    } else {
      const float v = p->p->region_end();
      if (ms) *ms = v;
    }
  });
}

int rp_pipeline_sync(rp_pipeline* p) {
  return tguard([&] {
    need(p, "pipeline");
    p->p->sync();
  });
}

int rp_pipeline_destroy(rp_pipeline* p) {
  return tguard([&] { delete p; });
}

}  // extern "C"
