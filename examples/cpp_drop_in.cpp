// A compiled C++ caller of the B200 step through the C++ mirror of the reference API
// (csrc/host/respar_b200.hpp) -- the pattern of INTEGRATION.md §2: what respar's train()
// (decoupled.cpp:282-314) does with DecoupledTrainer, on device.  tests/test_gpu_cpp_example.py
// builds it against librespar_b200.so, runs it on a B200 and checks its losses against the
// Python front end bit for bit, and that the reference's exception types come through.
//
//   nvcc -std=c++17 -I include -I paper_2009_01462_b200/csrc examples/cpp_drop_in.cpp \
//        -L paper_2009_01462_b200 -lrespar_b200 -Xlinker -rpath=... -o cpp_drop_in
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <vector>

#include "host/respar_b200.hpp"
#include "respar_b200.h"

using namespace respar::b200;

int main() {
  // the conv network (3x8x8 inputs, C = hidden = 64: the tcgen05 plane path), 4 blocks, 2 stages
  const rp_geometry geo{3, 8, 8, 64, 64, 4, 10, RP_ACT_TANH, 1.0};
  const int K = 2, N = 8;
  DecoupledTrainer gpu(geo, K, TrainMode::Alm, PenaltyKind::SquaredL2, N);
  uint64_t seed = 12345;   // make_net draw order on device (network.cpp:49-68)
  gpu.init_params(seed);

  // the batch: rng_uniform(-1, 1) from Rng(777) (tensor.cpp:177-185) on device, labels i % 10
  float* x = nullptr;
  int32_t* y = nullptr;
  const int64_t nx = (int64_t)N * geo.height * geo.width * geo.in_channels;
  cudaMalloc(&x, nx * sizeof(float));
  cudaMalloc(&y, N * sizeof(int32_t));
  uint64_t st = 777;
  check(rp_op_fill_uniform(x, nx, &st, -1.0, 1.0, 1.0, nullptr));
  std::vector<int32_t> labels(N);
  for (int i = 0; i < N; ++i) labels[i] = i % 10;
  cudaMemcpy(y, labels.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaDeviceSynchronize();

  gpu.reset_lambda_from_forward(x);                          // decoupled.cpp:285
  StepParams sp;
  sp.beta = 0.5;
  sp.lr = 0.05;
  sp.lambda_lr = 0.05;
  sp.kappa_lr = 1e-6;
  for (int it = 0; it < 3; ++it) {                            // decoupled.cpp:314
    const double loss = gpu.step(x, y, N, 0, sp);
    std::printf("loss %d %.17g\n", it, loss);
  }

  // the piecewise API keeps the reference's signatures and exceptions
  gpu.take_snapshot(0, 0, N);
  gpu.stage_forward(0, x, N, 0);
  const NetGrads g0 = gpu.stage_backward_update(0, nullptr, sp.beta, 0.0, 0);
  std::printf("stage0 grads begin %lld size %zu\n", (long long)g0.begin, g0.values.size());
  try {
    gpu.correct_aux(0, sp, 0, N);                             // lambda_0 is pinned to the input
    std::printf("no exception\n");
  } catch (const std::invalid_argument&) {
    std::printf("invalid_argument ok\n");
  }
  try {
    DecoupledTrainer bad(geo, 3, TrainMode::Penalty, PenaltyKind::SquaredL2, N);   // 3 does not divide 4
    std::printf("no exception\n");
  } catch (const ConfigError&) {
    std::printf("ConfigError ok\n");
  }
  const ViolationReport r = gpu.violation_report();
  std::printf("violation %.17g normalizer %ld\n", r.max_violation, r.normalizer);
  cudaFree(x);
  cudaFree(y);
  return 0;
}
