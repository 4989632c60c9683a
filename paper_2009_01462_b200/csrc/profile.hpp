// Live per-kernel-class device timing (CUDA events on the launching stream), used by
// bench.py for the roofline line.  Disabled by default; zero cost when off.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include "respar_b200.h"

namespace rp::prof {

extern std::atomic<bool> g_enabled;

void begin(int cls, cudaStream_t s, double flops, double bytes, void** token);
void end(void* token, cudaStream_t s);

struct Scope {
  void* token = nullptr;
  cudaStream_t s;
  Scope(int cls, cudaStream_t st, double flops, double bytes) : s(st) {
    if (g_enabled.load(std::memory_order_relaxed)) begin(cls, st, flops, bytes, &token);
  }
  ~Scope() {
    if (token) end(token, s);
  }
};

}  // namespace rp::prof
