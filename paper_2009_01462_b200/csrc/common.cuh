// Shared helpers for the sm_100a kernels and the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>
#include <stdexcept>
#include <string>

#include "respar_b200.h"

namespace rp {

// Status-carrying exception used inside the library; converted to an int status at
// the C ABI (capi.cpp) and back to the reference's exception types by the wrappers.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    fail(RP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                          std::to_string(line));
  }
}

#define RP_CUDA(x) ::rp::cuda_check((x), #x, __FILE__, __LINE__)
#define RP_LAUNCHED() \
  do {                \
    ::rp::note_launch(); \
    RP_CUDA(cudaGetLastError()); \
  } while (0)

void note_launch();
void note_launches(uint64_t n);   // kernels launched through a CUDA graph replay

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

constexpr int kNumSMs = 148;

// splitmix64, tensor.cpp:163-169.  Draw i of a stream at state s = mix(s + (i+1)*gamma).
__host__ __device__ inline uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

// Flat parameter layout (network.hpp:43-45 draw order).
struct ParamLayout {
  int64_t s_w, s_b, block0, block_stride, w1, b1, w2, b2, t_w, t_b, total;
  static ParamLayout of(const rp_geometry& g) {
    ParamLayout p{};
    const int64_t Ci = g.in_channels, C = g.channels, Ch = g.hidden;
    p.s_w = 0;
    p.s_b = 9 * Ci * C;
    p.block0 = p.s_b + C;
    p.w1 = 0;
    p.b1 = 9 * C * Ch;
    p.w2 = p.b1 + Ch;
    p.b2 = p.w2 + 9 * Ch * C;
    p.block_stride = p.b2 + C;
    p.t_w = p.block0 + p.block_stride * g.blocks;
    p.t_b = p.t_w + C * g.classes;
    p.total = p.t_b + g.classes;
    return p;
  }
};

// Launch with programmatic stream serialization (PDL): the kernel may start while the
// previous kernel of the stream finishes; it must call pdl_wait() (umma.cuh) before touching
// that kernel's outputs.  RP_PDL=0 launches plainly.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class Kernel, class... Args>
inline void launch_pdl(Kernel k, int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  if (e != cudaSuccess) fail(RP_ERR_CUDA, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));
}

// The same with a 1-D thread-block cluster of `cluster` CTAs (grid % cluster == 0).
template <class Kernel, class... Args>
inline void launch_pdl_cluster(Kernel k, int grid, int block, size_t smem, cudaStream_t st, int cluster,
                               Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  if (e != cudaSuccess) fail(RP_ERR_CUDA, std::string("cudaLaunchKernelEx (cluster): ") + cudaGetErrorString(e));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute
// belongs to the device's context, so a multi-device trainer needs it on every device.
inline void ensure_max_dynamic_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) fail(RP_ERR_CUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({fn, dev})) return;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) fail(RP_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  done.insert({fn, dev});
}

inline void validate_geometry(const rp_geometry& g) {
  if (g.in_channels < 1 || g.height < 1 || g.width < 1 || g.channels < 1 || g.hidden < 1 ||
      g.blocks < 1 || g.classes < 2)
    fail(RP_ERR_CONFIG, "geometry: all sizes must be >= 1 (classes >= 2)");
  if (g.activation != RP_ACT_TANH && g.activation != RP_ACT_IDENTITY)
    fail(RP_ERR_CONFIG, "geometry: unknown activation");
  if (g.classes > 1024) fail(RP_ERR_CONFIG, "geometry: at most 1024 classes");
}

}  // namespace rp
