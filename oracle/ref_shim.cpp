// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A flat extern "C" shim over the *unmodified* reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/build_ref.sh into
// oracle/_ref/librespar_ref.so).  It lets the Python tests, the golden-vector
// generator and bench.py's `--impl reference` arm drive the reference's own
// DecoupledTrainer / serial_train_step through ctypes.  Nothing here re-implements
// reference arithmetic: every call forwards to the reference symbol named in the
// comment.
//
// Flat parameter layout (the reference's make_net draw order, network.hpp:43-45):
//   s.w (in_dim*d)  s.b (d)  { w1 (d*h) b1 (h) w2 (h*d) b2 (d) } x L  t.w (d*classes) t.b (classes)
// Per-stage state selectors: 0 lambda, 1 kappa, 2 boundary_out, 3 boundary_adjoint
// (decoupled.hpp:29-32).

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "respar/decoupled.hpp"
#include "respar/gradcheck.hpp"

using namespace respar;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const StageError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 4;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

void copy_in(Tensor& t, const double* src) { std::memcpy(t.data.data(), src, sizeof(double) * t.data.size()); }
void copy_out(const Tensor& t, double* dst) { std::memcpy(dst, t.data.data(), sizeof(double) * t.data.size()); }

long flat_size(const ResidualNet& n) { return n.param_count(); }

void net_to_flat(const ResidualNet& n, double* p) {
  auto put = [&](const Tensor& t) { copy_out(t, p); p += t.size(); };
  put(n.s.w); put(n.s.b);
  for (const auto& b : n.blocks) { put(b.w1); put(b.b1); put(b.w2); put(b.b2); }
  put(n.t.w); put(n.t.b);
}

void flat_to_net(ResidualNet& n, const double* p) {
  auto get = [&](Tensor& t) { copy_in(t, p); p += t.size(); };
  get(n.s.w); get(n.s.b);
  for (auto& b : n.blocks) { get(b.w1); get(b.b1); get(b.w2); get(b.b2); }
  get(n.t.w); get(n.t.b);
}

void grads_to_flat(const NetGrads& g, const ResidualNet& n, double* p) {
  // Same layout as net_to_flat for the covered parameters; absent S/T are zeros.
  auto put = [&](const Tensor* t, long size) {
    if (t && t->size() == size) copy_out(*t, p); else std::memset(p, 0, sizeof(double) * size);
    p += size;
  };
  put(g.has_s ? &g.s.w : nullptr, n.s.w.size());
  put(g.has_s ? &g.s.b : nullptr, n.s.b.size());
  for (const auto& b : g.blocks) {
    put(&b.w1, n.blocks[0].w1.size()); put(&b.b1, n.blocks[0].b1.size());
    put(&b.w2, n.blocks[0].w2.size()); put(&b.b2, n.blocks[0].b2.size());
  }
  put(g.has_t ? &g.t.w : nullptr, n.t.w.size());
  put(g.has_t ? &g.t.b : nullptr, n.t.b.size());
}

ResidualNet shape_net(int in_dim, int d, int h, int L, int classes, int act) {
  ResidualNet n = make_zero_net(in_dim, d, h, L, classes);
  n.activation = act == 0 ? Activation::Tanh : Activation::Identity;
  return n;
}

struct Handle {
  std::unique_ptr<DecoupledTrainer> tr;
  std::unique_ptr<StagePool> pool;
  std::vector<NeighborSnapshot> snaps;
  NetGrads last_grads;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- RNG (tensor.cpp:163-197) -------------------------------------------
int ref_rng_uniform(uint64_t* state, int rows, int cols, double lo, double hi, double* out) {
  return guard([&] {
    Rng r(*state);
    copy_out(rng_uniform(r, rows, cols, lo, hi), out);
    *state = r.state;
  });
}
int ref_rng_normal(uint64_t* state, int rows, int cols, double mean, double sigma, double* out) {
  return guard([&] {
    Rng r(*state);
    copy_out(rng_normal(r, rows, cols, mean, sigma), out);
    *state = r.state;
  });
}
uint64_t ref_rng_next_u64(uint64_t* state) { Rng r(*state); uint64_t v = r.next_u64(); *state = r.state; return v; }
uint64_t ref_rng_split(uint64_t* state) { Rng r(*state); Rng s = r.split(); *state = r.state; return s.state; }

// ---- model (network.cpp) --------------------------------------------------
long ref_param_count(int in_dim, int d, int h, int L, int classes) {
  return make_zero_net(in_dim, d, h, L, classes).param_count();
}
int ref_make_net(uint64_t* state, int in_dim, int d, int h, int L, int classes, double* params) {
  return guard([&] {
    Rng r(*state);
    net_to_flat(make_net(in_dim, d, h, L, classes, r), params);
    *state = r.state;
  });
}
int ref_net_forward(int in_dim, int d, int h, int L, int classes, int act, const double* params,
                    const double* x, int rows, int from, int to, double* features, double* logits) {
  return guard([&] {
    ResidualNet n = shape_net(in_dim, d, h, L, classes, act);
    flat_to_net(n, params);
    Tensor xt(rows, from == 0 ? in_dim : d);
    copy_in(xt, x);
    ForwardTape tape = net_forward(n, xt, from, to);
    copy_out(tape.features, features);
    if (tape.has_output_layer && logits) copy_out(tape.logits, logits);
  });
}
int ref_serial_train_step(int in_dim, int d, int h, int L, int classes, int act, double* params,
                          const double* x, const int* labels, int rows, double lr, double* loss) {
  return guard([&] {
    ResidualNet n = shape_net(in_dim, d, h, L, classes, act);
    flat_to_net(n, params);
    Tensor xt(rows, in_dim);
    copy_in(xt, x);
    std::vector<int> y(labels, labels + rows);
    *loss = serial_train_step(n, xt, y, lr);
    net_to_flat(n, params);
  });
}
// build_initial_net (decoupled.cpp:207-245).  mode: TrainMode (0 serial, 1 penalty, 2 alm);
// init: InitScheme (0 multilevel, 1 warmstart, 2 random), config.hpp:17-18.  The reference
// hard-codes in_dim = 2 (the toy input).  lr schedule = (epoch, value) steps.
int ref_build_initial_net(int mode, int init, int d, int h, int L, int K, int classes, int coarse_epochs,
                          int warm_epochs, const int* lr_epochs, const double* lr_values, int n_lr,
                          const double* x, const int* labels, int rows, uint64_t* state, double* params) {
  return guard([&] {
    TrainConfig cfg;
    cfg.mode = static_cast<TrainMode>(mode);
    cfg.init = static_cast<InitScheme>(init);
    cfg.feature_dim = d;
    cfg.hidden_dim = h;
    cfg.num_blocks = L;
    cfg.stages = K;
    cfg.classes = classes;
    cfg.coarse_epochs = coarse_epochs;
    cfg.warmstart_epochs = warm_epochs;
    cfg.schedules.lr_steps.clear();
    for (int i = 0; i < n_lr; ++i) cfg.schedules.lr_steps.emplace_back(lr_epochs[i], lr_values[i]);
    Tensor xt(rows, 2);
    copy_in(xt, x);
    std::vector<int> y(labels, labels + rows);
    Rng r(*state);
    ResidualNet n = build_initial_net(cfg, xt, y, r);
    net_to_flat(n, params);
    *state = r.state;
  });
}

int ref_loss_phi(const double* logits, const int* labels, int rows, int classes, double* value,
                 double* grad) {
  return guard([&] {
    Tensor l(rows, classes);
    copy_in(l, logits);
    LossResult r = loss_phi(l, std::vector<int>(labels, labels + rows));
    *value = r.value;
    if (grad) copy_out(r.grad_logits, grad);
  });
}
int ref_accuracy(int in_dim, int d, int h, int L, int classes, int act, const double* params,
                 const double* x, const int* labels, int rows, double* acc) {
  return guard([&] {
    ResidualNet n = shape_net(in_dim, d, h, L, classes, act);
    flat_to_net(n, params);
    Tensor xt(rows, in_dim);
    copy_in(xt, x);
    *acc = accuracy(n, xt, std::vector<int>(labels, labels + rows));
  });
}

// ---- penalty (penalty.cpp) ----------------------------------------------
int ref_psi(int kind, const double* lam, const double* x, int rows, int cols, double* out) {
  return guard([&] {
    Tensor a(rows, cols), b(rows, cols);
    copy_in(a, lam); copy_in(b, x);
    *out = psi(static_cast<PenaltyKind>(kind), a, b);
  });
}
int ref_psi_grads(int kind, const double* lam, const double* x, int rows, int cols, double* d_lambda,
                  double* d_x) {
  return guard([&] {
    Tensor a(rows, cols), b(rows, cols);
    copy_in(a, lam); copy_in(b, x);
    PsiGrads g = psi_grads(static_cast<PenaltyKind>(kind), a, b);
    copy_out(g.d_lambda, d_lambda);
    copy_out(g.d_x, d_x);
  });
}

// ---- decoupled trainer (decoupled.cpp) ----------------------------------
void* ref_trainer_create(int in_dim, int d, int h, int L, int classes, int act, const double* params,
                         int stages, int mode, int penalty, int num_samples, int workers) {
  Handle* hd = nullptr;
  int rc = guard([&] {
    ResidualNet n = shape_net(in_dim, d, h, L, classes, act);
    flat_to_net(n, params);
    auto tr = std::make_unique<DecoupledTrainer>(std::move(n), stages, static_cast<TrainMode>(mode),
                                                 static_cast<PenaltyKind>(penalty), num_samples);
    hd = new Handle;
    hd->tr = std::move(tr);
    hd->pool = std::make_unique<StagePool>(stages, workers <= 0 ? stages : workers);
    hd->snaps.resize(stages);
  });
  return rc == 0 ? hd : nullptr;
}
void ref_trainer_destroy(void* h) { delete static_cast<Handle*>(h); }

int ref_trainer_get_params(void* h, double* params) {
  return guard([&] { net_to_flat(static_cast<Handle*>(h)->tr->net(), params); });
}
int ref_trainer_set_params(void* h, const double* params) {
  return guard([&] { flat_to_net(static_cast<Handle*>(h)->tr->net(), params); });
}
int ref_trainer_reset_lambda(void* h, const double* x, int rows, int cols) {
  return guard([&] {
    Tensor t(rows, cols);
    copy_in(t, x);
    static_cast<Handle*>(h)->tr->reset_lambda_from_forward(t);
  });
}
static Tensor& state_ref(DecoupledTrainer& tr, int k, int which) {
  StageState& st = tr.stage(k);
  switch (which) {
    case 0: return st.lambda;
    case 1: return st.kappa;
    case 2: return st.boundary_out;
    default: return st.boundary_adjoint;
  }
}
long ref_trainer_state_size(void* h, int k, int which) {
  return state_ref(*static_cast<Handle*>(h)->tr, k, which).size();
}
int ref_trainer_get_state(void* h, int k, int which, double* out) {
  return guard([&] { copy_out(state_ref(*static_cast<Handle*>(h)->tr, k, which), out); });
}
int ref_trainer_set_state(void* h, int k, int which, const double* in, int rows, int cols) {
  return guard([&] {
    Tensor t(rows, cols);
    copy_in(t, in);
    state_ref(*static_cast<Handle*>(h)->tr, k, which) = t;
  });
}
int ref_trainer_step(void* h, const double* x, int rows, int cols, const int* labels, int row0,
                     double beta, double tau, double lr, double lambda_lr, double kappa_lr,
                     int max_corrections, double* loss) {
  return guard([&] {
    Handle* hd = static_cast<Handle*>(h);
    Tensor t(rows, cols);
    copy_in(t, x);
    StepParams sp;
    sp.beta = beta; sp.tau = tau; sp.lr = lr; sp.lambda_lr = lambda_lr; sp.kappa_lr = kappa_lr;
    sp.max_corrections = max_corrections;
    *loss = hd->tr->step(t, std::vector<int>(labels, labels + rows), row0, sp, *hd->pool);
  });
}
int ref_trainer_take_snapshot(void* h, int k, int row0, int nrows) {
  return guard([&] {
    Handle* hd = static_cast<Handle*>(h);
    hd->tr->take_snapshot(k, row0, nrows, hd->snaps.at(k));
  });
}
int ref_trainer_stage_forward(void* h, int k, const double* x, int rows, int cols, int row0) {
  return guard([&] {
    Tensor t(rows, cols);
    copy_in(t, x);
    static_cast<Handle*>(h)->tr->stage_forward(k, t, row0);
  });
}
// grads_out: full flat layout (zeros outside stage k); may be null.
int ref_trainer_stage_backward_update(void* h, int k, const int* labels, int nrows, double beta,
                                      double lr, int row0, double* grads_out) {
  return guard([&] {
    Handle* hd = static_cast<Handle*>(h);
    DecoupledTrainer& tr = *hd->tr;
    NetGrads g = tr.stage_backward_update(k, std::vector<int>(labels, labels + nrows),
                                          hd->snaps.at(k), beta, lr, row0);
    if (grads_out) {
      const ResidualNet& n = tr.net();
      std::memset(grads_out, 0, sizeof(double) * flat_size(n));
      const long s_sz = n.s.w.size() + n.s.b.size();
      const long blk = n.blocks[0].w1.size() + n.blocks[0].b1.size() + n.blocks[0].w2.size() + n.blocks[0].b2.size();
      double* p = grads_out;
      if (g.has_s) { copy_out(g.s.w, p); copy_out(g.s.b, p + n.s.w.size()); }
      p = grads_out + s_sz + static_cast<long>(tr.stage(k).begin) * blk;
      for (const auto& b : g.blocks) {
        copy_out(b.w1, p); p += b.w1.size();
        copy_out(b.b1, p); p += b.b1.size();
        copy_out(b.w2, p); p += b.w2.size();
        copy_out(b.b2, p); p += b.b2.size();
      }
      if (g.has_t) {
        double* t = grads_out + s_sz + static_cast<long>(n.depth()) * blk;
        copy_out(g.t.w, t); copy_out(g.t.b, t + n.t.w.size());
      }
    }
  });
}
int ref_trainer_correct_aux(void* h, int k, double beta, double tau, double lambda_lr,
                            int max_corrections, int row0, int nrows) {
  return guard([&] {
    StepParams sp;
    sp.beta = beta; sp.tau = tau; sp.lambda_lr = lambda_lr; sp.max_corrections = max_corrections;
    static_cast<Handle*>(h)->tr->correct_aux(k, sp, row0, nrows);
  });
}
int ref_trainer_correct_multiplier(void* h, int k, double beta, double kappa_lr, int row0, int nrows) {
  return guard([&] { static_cast<Handle*>(h)->tr->correct_multiplier(k, beta, kappa_lr, row0, nrows); });
}
int ref_trainer_correction_gradient(void* h, int k, double beta, int row0, int nrows, double* out) {
  return guard([&] { copy_out(static_cast<Handle*>(h)->tr->correction_gradient(k, beta, row0, nrows), out); });
}
int ref_trainer_violation_report(void* h, double* per_stage, double* max_violation, long* normalizer) {
  return guard([&] {
    ViolationReport r = static_cast<Handle*>(h)->tr->violation_report();
    for (std::size_t i = 0; i < r.per_stage.size(); ++i) per_stage[i] = r.per_stage[i];
    *max_violation = r.max_violation;
    *normalizer = r.normalizer;
  });
}
long ref_trainer_iteration(void* h) { return static_cast<Handle*>(h)->tr->iteration(); }
int ref_partition(int num_blocks, int stages, int* ranges) {
  return guard([&] {
    auto r = partition(num_blocks, stages);
    for (int k = 0; k < stages; ++k) { ranges[2 * k] = r[k].first; ranges[2 * k + 1] = r[k].second; }
  });
}
int ref_gradcheck(uint64_t seed, double eps, double* max_rel_err) {
  return guard([&] { *max_rel_err = fd_gradcheck(seed, eps).max_rel_err; });
}

}  // extern "C"
