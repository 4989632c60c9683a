// HBM-bound kernels of the hot path: synthetic-loss upstream, fused lambda/kappa
// correction, SGD, psi reductions, counter-based RNG fills.
//
// All are grid-stride, float4-vectorised, one read + one write per element (the
// algorithmic minimum: DESIGN.md §kernels).  Reductions are deterministic two-pass
// (fixed partition, fixed combine order; no float atomics), so results do not depend
// on stage placement or launch timing (runtime.hpp:28-32).
#include <cmath>

#include <cuda_bf16.h>

#include "../common.cuh"
#include "kernels.cuh"
#include "planes.cuh"

namespace rp::k {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxReduceBlocks = 1024;

struct ArgMax {
  float v;
  long long i;
};

__device__ __forceinline__ ArgMax argmax_combine(ArgMax a, ArgMax b) {
  // larger |d| wins; ties go to the lowest flat index (penalty.cpp:79-84)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ __forceinline__ float sign0(float v) { return v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f); }

int grid_for(int64_t n, int per_thread = 4) {
  int64_t blocks = (n + (int64_t)kThreads * per_thread - 1) / ((int64_t)kThreads * per_thread);
  if (blocks < 1) blocks = 1;
  if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
  return static_cast<int>(blocks);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ----------------------------------------------------------------- RNG fills
__global__ void fill_uniform_kernel(float* __restrict__ dst, int64_t n, uint64_t state, double lo, double span,
                                    double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z = splitmix_mix(state + (uint64_t)(i + 1) * kGamma);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    dst[i] = (float)((lo + span * u) * scale);
  }
}

__global__ void fill_normal_kernel(float* __restrict__ dst, int64_t n, uint64_t state, double mean, double sigma,
                                   int accumulate) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z1 = splitmix_mix(state + (uint64_t)(2 * i + 1) * kGamma);
    const uint64_t z2 = splitmix_mix(state + (uint64_t)(2 * i + 2) * kGamma);
    const double u1 = 1.0 - (double)(z1 >> 11) * 0x1.0p-53;
    const double u2 = (double)(z2 >> 11) * 0x1.0p-53;
    const double v = mean + sigma * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    if (accumulate)
      dst[i] = (float)((double)dst[i] + v);
    else
      dst[i] = (float)v;
  }
}

// ------------------------------------------------------------- reductions
// kind 0: sum d^2, 1: sum |d|, 2: max |d| (penalty.cpp:38-58), fp64 accumulation.
__global__ void psi_partial_kernel(int kind, const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                   double* __restrict__ partial) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  // fixed contiguous chunk per block -> result independent of scheduling
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t beg = blockIdx.x * chunk;
  const int64_t end = min(n, beg + chunk);
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    if (kind == 0) acc += d * d;
    else if (kind == 1) acc += fabs(d);
    else acc = fmax(acc, fabs(d));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = kind == 2 ? fmax(sh[threadIdx.x], sh[threadIdx.x + s])
                                                      : sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void psi_final_kernel(int kind, const double* __restrict__ partial, int nblocks, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < nblocks; ++i) acc = kind == 2 ? fmax(acc, partial[i]) : acc + partial[i];
    *out = acc;
  }
}

__global__ void argmax_partial_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                      ArgMax* __restrict__ partial) {
  __shared__ ArgMax sh[kThreads];
  ArgMax best{-1.f, (long long)n};
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t beg = blockIdx.x * chunk;
  const int64_t end = min(n, beg + chunk);
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    ArgMax c{fabsf(a[i] - b[i]), (long long)i};
    best = argmax_combine(best, c);
  }
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = argmax_combine(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void argmax_final_kernel(const ArgMax* __restrict__ partial, int nblocks, ArgMax* __restrict__ out) {
  if (threadIdx.x == 0) {
    ArgMax best = partial[0];
    for (int i = 1; i < nblocks; ++i) best = argmax_combine(best, partial[i]);
    *out = best;
  }
}

// ------------------------------------------------------- elementwise bodies
// d_lambda psi for one element (penalty.cpp:60-87); LInf handled via `arg`.
__device__ __forceinline__ float dlam(int kind, float d, int64_t i, long long arg) {
  if (kind == 0) return 2.f * d;
  if (kind == 1) return sign0(d);
  return i == arg ? sign0(d) : 0.f;
}

// g = w * d_x + kappa,  d_x = -d_lambda   (decoupled.cpp:105-110)
// p0 (p1 null, optional): the bf16 single plane of g for the bf16 tape path, same pass.
// bmax (optional): per-CTA max |g| (the plane-pair scale is formed from these afterwards).
__global__ void synthetic_grad_vec4(int kind, const float4* __restrict__ lam, const float4* __restrict__ x,
                                    const float4* __restrict__ kap, int64_t n4, float w, float4* __restrict__ g,
                                    uint2* __restrict__ p0, float* __restrict__ bmax) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 l = lam[i], xe = x[i];
    float4 k4 = kap ? kap[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 o;
    o.x = -dlam(kind, l.x - xe.x, 0, -1) * w + k4.x;
    o.y = -dlam(kind, l.y - xe.y, 0, -1) * w + k4.y;
    o.z = -dlam(kind, l.z - xe.z, 0, -1) * w + k4.z;
    o.w = -dlam(kind, l.w - xe.w, 0, -1) * w + k4.w;
    g[i] = o;
    m = fmaxf(m, fmaxf(fmaxf(fabsf(o.x), fabsf(o.y)), fmaxf(fabsf(o.z), fabsf(o.w))));
    if (p0) {
      const float v[4] = {o.x, o.y, o.z, o.w};
      p0[i] = pack_single4(v);
    }
  }
  if (bmax) {
    __shared__ float sh[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int wi = 1; wi < kThreads / 32; ++wi) m = fmaxf(m, sh[wi]);
      bmax[blockIdx.x] = fmaxf(m, sh[0]);
    }
  }
}

__global__ void synthetic_grad_scalar(int kind, const float* __restrict__ lam, const float* __restrict__ x,
                                      const float* __restrict__ kap, int64_t n, float w, const ArgMax* am,
                                      float* __restrict__ g) {
  const long long arg = am ? am->i : -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float k = kap ? kap[i] : 0.f;
    g[i] = -dlam(kind, lam[i] - x[i], i, arg) * w + k;
  }
}

// lam' = lam - eta (w d_lambda + p - kappa);  kappa' = kappa - c (lam' - x)   (decoupled.cpp:135-170)
__device__ __forceinline__ void correct_one(int kind, float& l, float xp, float p, float& k, int64_t i,
                                            long long arg, float w, float eta, bool ul, float kc, bool uk) {
  if (ul) {
    float g = dlam(kind, l - xp, i, arg) * w;
    g = g + p;
    g = g - k;
    l = l + (-eta) * g;
  }
  if (uk) k = k + (-kc) * (l - xp);
}

__global__ void correct_vec4(int kind, float4* __restrict__ lam, const float4* __restrict__ xp,
                             const float4* __restrict__ p, float4* __restrict__ kap, int64_t n4, float w, float eta,
                             int ul, float kc, int uk) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 l = lam[i];
    const float4 x4 = xp[i];
    const float4 p4 = ul ? p[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 k4 = kap ? kap[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    correct_one(kind, l.x, x4.x, p4.x, k4.x, 0, -1, w, eta, ul, kc, uk);
    correct_one(kind, l.y, x4.y, p4.y, k4.y, 0, -1, w, eta, ul, kc, uk);
    correct_one(kind, l.z, x4.z, p4.z, k4.z, 0, -1, w, eta, ul, kc, uk);
    correct_one(kind, l.w, x4.w, p4.w, k4.w, 0, -1, w, eta, ul, kc, uk);
    if (ul) lam[i] = l;
    if (uk) kap[i] = k4;
  }
}

__global__ void correct_scalar(int kind, float* __restrict__ lam, const float* __restrict__ xp,
                               const float* __restrict__ p, float* __restrict__ kap, int64_t n, float w, float eta,
                               int ul, float kc, int uk, const ArgMax* am) {
  const long long arg = am ? am->i : -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float l = lam[i];
    float k = kap ? kap[i] : 0.f;
    correct_one(kind, l, xp[i], ul ? p[i] : 0.f, k, i, arg, w, eta, ul, kc, uk);
    if (ul) lam[i] = l;
    if (uk) kap[i] = k;
  }
}

__global__ void psi_grad_scalar(int kind, const float* __restrict__ lam, const float* __restrict__ x, int64_t n,
                                float scale, const ArgMax* am, float* __restrict__ out) {
  const long long arg = am ? am->i : -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = dlam(kind, lam[i] - x[i], i, arg) * scale;
}

// W -= lr g  (axpy_inplace, tensor.cpp:122-125); momentum: v = mu v + g, W -= lr v
__global__ void sgd_vec4(float4* __restrict__ w, const float4* __restrict__ g, float4* __restrict__ v, int64_t n4,
                         float lr, float mu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 w4 = w[i];
    float4 g4 = g[i];
    if (v) {
      float4 v4 = v[i];
      v4.x = mu * v4.x + g4.x; v4.y = mu * v4.y + g4.y; v4.z = mu * v4.z + g4.z; v4.w = mu * v4.w + g4.w;
      v[i] = v4;
      g4 = v4;
    }
    w4.x += -lr * g4.x; w4.y += -lr * g4.y; w4.z += -lr * g4.z; w4.w += -lr * g4.w;
    w[i] = w4;
  }
}

__global__ void sgd_scalar(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v, int64_t n,
                           float lr, float mu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float gi = g[i];
    if (v) {
      const float vi = mu * v[i] + gi;
      v[i] = vi;
      gi = vi;
    }
    w[i] += -lr * gi;
  }
}

int reduce_blocks(int64_t n) {
  int64_t b = (n + 4095) / 4096;
  if (b < 1) b = 1;
  if (b > kMaxReduceBlocks) b = kMaxReduceBlocks;
  return static_cast<int>(b);
}

}  // namespace

int64_t reduce_workspace_bytes() { return (kMaxReduceBlocks + 2) * 16; }

void fill_uniform(float* dst, int64_t n, uint64_t state, double lo, double hi, double scale, cudaStream_t s) {
  if (n <= 0) return;
  fill_uniform_kernel<<<grid_for(n, 1), kThreads, 0, s>>>(dst, n, state, lo, hi - lo, scale);
  RP_LAUNCHED();
}

void fill_normal(float* dst, int64_t n, uint64_t state, double mean, double sigma, bool accumulate, cudaStream_t s) {
  if (n <= 0) return;
  fill_normal_kernel<<<grid_for(n, 1), kThreads, 0, s>>>(dst, n, state, mean, sigma, accumulate ? 1 : 0);
  RP_LAUNCHED();
}

void psi_device(int kind, const float* a, const float* b, int64_t n, void* ws, double* out_dev, cudaStream_t s) {
  double* partial = static_cast<double*>(ws);
  const int nb = reduce_blocks(n);
  psi_partial_kernel<<<nb, kThreads, 0, s>>>(kind, a, b, n, partial);
  RP_LAUNCHED();
  psi_final_kernel<<<1, 32, 0, s>>>(kind, partial, nb, out_dev);
  RP_LAUNCHED();
}

static const ArgMax* linf_argmax(const float* a, const float* b, int64_t n, void* ws, cudaStream_t s) {
  ArgMax* partial = static_cast<ArgMax*>(ws);
  ArgMax* fin = partial + kMaxReduceBlocks;
  const int nb = reduce_blocks(n);
  argmax_partial_kernel<<<nb, kThreads, 0, s>>>(a, b, n, partial);
  RP_LAUNCHED();
  argmax_final_kernel<<<1, 32, 0, s>>>(partial, nb, fin);
  RP_LAUNCHED();
  return fin;
}

void psi_grad(int kind, const float* lam, const float* x, int64_t n, double scale, float* out, void* ws,
              cudaStream_t s) {
  if (n <= 0) return;
  const ArgMax* am = kind == RP_PSI_LINF ? linf_argmax(lam, x, n, ws, s) : nullptr;
  psi_grad_scalar<<<grid_for(n), kThreads, 0, s>>>(kind, lam, x, n, (float)scale, am, out);
  RP_LAUNCHED();
}

void synthetic_grad(int kind, const float* lam_next, const float* x_end, const float* kappa, int64_t n, double w,
                    float* g, void* ws, cudaStream_t s, void* p0, void* p1, float* scale) {
  if (n <= 0) return;
  if (p1 && !scale) fail(RP_ERR_INTERNAL, "synthetic_grad: the cotangent plane pair needs a scale buffer");
  if (kind != RP_PSI_LINF && n % 4 == 0 && aligned16(lam_next) && aligned16(x_end) && aligned16(g) &&
      (!kappa || aligned16(kappa)) && (!p0 || aligned16(p0)) && (!p1 || aligned16(p1))) {
    const int grid = grid_for(n / 4);
    float* part = p1 ? scale + kPlaneScalePartOffset : nullptr;   // grid <= 8 x 148 partials
    synthetic_grad_vec4<<<grid, kThreads, 0, s>>>(
        kind, reinterpret_cast<const float4*>(lam_next), reinterpret_cast<const float4*>(x_end),
        reinterpret_cast<const float4*>(kappa), n / 4, (float)w, reinterpret_cast<float4*>(g),
        p1 ? nullptr : static_cast<uint2*>(p0), part);
    RP_LAUNCHED();
    if (p1) split_planes_from_parts(g, n, p0, p1, part, grid, scale, s);
    return;
  }
  const ArgMax* am = kind == RP_PSI_LINF ? linf_argmax(lam_next, x_end, n, ws, s) : nullptr;
  synthetic_grad_scalar<<<grid_for(n), kThreads, 0, s>>>(kind, lam_next, x_end, kappa, n, (float)w, am, g);
  RP_LAUNCHED();
  if (p0) split_planes(g, n, p0, p1, s, p1 ? scale : nullptr);   // the planes in a second pass (LInf / unaligned)
}

void correct(int kind, float* lam, const float* x_prev, const float* p, float* kappa, int64_t n, double w,
             double eta, bool update_lambda, double kappa_coef, bool update_kappa, void* ws, cudaStream_t s) {
  if (n <= 0 || (!update_lambda && !update_kappa)) return;
  if (update_kappa && !kappa) fail(RP_ERR_INTERNAL, "correct: kappa update without kappa storage");
  const bool linf = update_lambda && kind == RP_PSI_LINF;
  if (!linf && n % 4 == 0 && aligned16(lam) && aligned16(x_prev) && (!p || aligned16(p)) &&
      (!kappa || aligned16(kappa))) {
    correct_vec4<<<grid_for(n / 4), kThreads, 0, s>>>(
        kind, reinterpret_cast<float4*>(lam), reinterpret_cast<const float4*>(x_prev),
        reinterpret_cast<const float4*>(p), reinterpret_cast<float4*>(kappa), n / 4, (float)w, (float)eta,
        update_lambda ? 1 : 0, (float)kappa_coef, update_kappa ? 1 : 0);
  } else {
    const ArgMax* am = linf ? linf_argmax(lam, x_prev, n, ws, s) : nullptr;
    correct_scalar<<<grid_for(n), kThreads, 0, s>>>(kind, lam, x_prev, p, kappa, n, (float)w, (float)eta,
                                                    update_lambda ? 1 : 0, (float)kappa_coef,
                                                    update_kappa ? 1 : 0, am);
  }
  RP_LAUNCHED();
}

void sgd(float* w, const float* g, float* v, int64_t n, double lr, double momentum, cudaStream_t s) {
  if (n <= 0) return;
  if (n % 4 == 0 && aligned16(w) && aligned16(g) && (!v || aligned16(v))) {
    sgd_vec4<<<grid_for(n / 4), kThreads, 0, s>>>(reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g),
                                                   reinterpret_cast<float4*>(v), n / 4, (float)lr, (float)momentum);
  } else {
    sgd_scalar<<<grid_for(n), kThreads, 0, s>>>(w, g, v, n, (float)lr, (float)momentum);
  }
  RP_LAUNCHED();
}

}  // namespace rp::k
