// Output map T and the task loss (network.cpp:108-110, 193-221), conv form:
// global average pool -> affine C->classes -> mean softmax-CE, and its backward.
// All reductions run in a fixed order (deterministic).
#include <cuda_bf16.h>
#include <algorithm>
#include <cfloat>

#include "../common.cuh"
#include "kernels.cuh"
#include "planes.cuh"

namespace rp::k {

namespace {

// pooled[b][c] = mean_p x[b][p][c]; one CTA per sample.
// pooled[b][c] = mean_p x[b][p][c].  One CTA per image; thread (group g, float4 lane q)
// sums positions g, g + G, ... (8 loads in flight), groups combined in fixed order.
constexpr int kGapThreads = 512;
__global__ __launch_bounds__(kGapThreads) void gap_kernel_vec4(const float4* __restrict__ x, int hw, int C4,
                                                              float* __restrict__ pooled) {
  extern __shared__ float4 sh4[];
  const int b = blockIdx.x;
  const float4* xb = x + (int64_t)b * hw * C4;
  const int groups = kGapThreads / C4;     // C4 divides kGapThreads (host check)
  const int g = threadIdx.x / C4, q = threadIdx.x % C4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int p = g;
  for (; p + 7 * groups < hw; p += 8 * groups) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(xb + (int64_t)(p + u * groups) * C4 + q);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc.x += v[u].x, acc.y += v[u].y, acc.z += v[u].z, acc.w += v[u].w;
  }
  for (; p < hw; p += groups) {
    const float4 v = __ldg(xb + (int64_t)p * C4 + q);
    acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
  }
  sh4[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < C4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int gg = 0; gg < groups; ++gg) {
      const float4 v = sh4[gg * C4 + threadIdx.x];
      s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
    }
    const float inv = 1.f / (float)hw;
    reinterpret_cast<float4*>(pooled)[(int64_t)b * C4 + threadIdx.x] =
        make_float4(s.x * inv, s.y * inv, s.z * inv, s.w * inv);
  }
}

__global__ __launch_bounds__(256) void gap_kernel(const float* __restrict__ x, int hw, int C,
                                                 float* __restrict__ pooled) {
  extern __shared__ float sh[];
  const int b = blockIdx.x;
  const float* xb = x + (int64_t)b * hw * C;
  const int groups = C <= 256 ? max(1, 256 / C) : 1;
  const float inv = 1.f / (float)hw;
  for (int cbase = 0; cbase < C; cbase += 256) {
    const int cw = min(256, C - cbase);
    const int g = threadIdx.x / cw;
    const int c = cbase + threadIdx.x % cw;
    float acc = 0.f;
    if (g < groups && threadIdx.x < groups * cw)
      for (int p = g; p < hw; p += groups) acc += xb[(int64_t)p * C + c];
    if (threadIdx.x < groups * cw) sh[g * cw + (c - cbase)] = acc;
    __syncthreads();
    if (threadIdx.x < cw) {
      float s = 0.f;
      for (int gg = 0; gg < groups; ++gg) s += sh[gg * cw + threadIdx.x];
      pooled[(int64_t)b * C + cbase + threadIdx.x] = s * inv;
    }
    __syncthreads();
  }
}

// logits[b][j] = sum_c pooled[b][c] t_w[c][j] + t_b[j]   (affine_forward)
__global__ void fc_kernel(const float* __restrict__ pooled, const float* __restrict__ t_w,
                          const float* __restrict__ t_b, int C, int classes, float* __restrict__ logits) {
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < C; ++c) s = fmaf(pooled[(int64_t)b * C + c], t_w[(int64_t)c * classes + j], s);
    logits[(int64_t)b * classes + j] = s + t_b[j];
  }
}

// Per sample: softmax-CE (max-shifted, network.cpp:207-217) in fp64, grad_logits /B,
// and the pooled-feature cotangent gpool = grad_logits . t_w^T.
__global__ void loss_grad_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels,
                                 const float* __restrict__ t_w, int nrows, int C, int classes,
                                 float* __restrict__ glog, double* __restrict__ loss_b, float* __restrict__ gpool) {
  const int b = blockIdx.x;
  const float* l = logits + (int64_t)b * classes;
  __shared__ double s_lse;
  __shared__ float s_g[1024];
  if (threadIdx.x == 0) {
    double m = l[0];
    for (int c = 1; c < classes; ++c) m = fmax(m, (double)l[c]);
    double z = 0.0;
    for (int c = 0; c < classes; ++c) z += exp((double)l[c] - m);
    const double lse = m + log(z);
    const int y = labels[b];
    loss_b[b] = (y >= 0 && y < classes) ? lse - (double)l[y] : __longlong_as_double(0x7ff8000000000000LL);
    s_lse = lse;
  }
  __syncthreads();
  const int y = labels[b];
  for (int c = threadIdx.x; c < classes; c += blockDim.x) {
    const double sm = exp((double)l[c] - s_lse);
    const float g = (float)((sm - (c == y ? 1.0 : 0.0)) / (double)nrows);
    glog[(int64_t)b * classes + c] = g;
    s_g[c] = g;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < classes; ++j) s = fmaf(s_g[j], t_w[(int64_t)c * classes + j], s);
    gpool[(int64_t)b * C + c] = s;
  }
}

// gt_w[c][j] = sum_b pooled[b][c] glog[b][j]; gt_b[j] = sum_b glog[b][j]; loss = mean loss_b.
// gt_w[c][j] = sum_b pooled[b][c] glog[b][j], gt_b[j] = sum_b glog[b][j], loss = mean_b
// loss_b: one warp per output, lanes stride the rows, fixed shuffle order (fp64).
__global__ void head_param_grad_kernel(const float* __restrict__ pooled, const float* __restrict__ glog,
                                       const double* __restrict__ loss_b, int nrows, int C, int classes,
                                       float* __restrict__ gt_w, float* __restrict__ gt_b, double* __restrict__ loss) {
  const int total = C * classes + classes + 1;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (w >= total) return;
  double s = 0.0;
  if (w < C * classes) {
    const int c = w / classes, j = w % classes;
    for (int b = lane; b < nrows; b += 32) s += (double)pooled[(int64_t)b * C + c] * (double)glog[(int64_t)b * classes + j];
  } else if (w < C * classes + classes) {
    const int j = w - C * classes;
    for (int b = lane; b < nrows; b += 32) s += (double)glog[(int64_t)b * classes + j];
  } else {
    for (int b = lane; b < nrows; b += 32) s += loss_b[b];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane != 0) return;
  if (w < C * classes)
    gt_w[w] = (float)s;
  else if (w < C * classes + classes)
    gt_b[w - C * classes] = (float)s;
  else if (loss)
    *loss = s / (double)nrows;
}

// g[b][p][c] = gpool[b][c] / hw  (d mean / d x)
__global__ void broadcast_kernel(const float* __restrict__ gpool, int64_t hw, int C, int64_t total,
                                 float inv_hw, float* __restrict__ g) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t b = i / ((int64_t)C * hw);
    g[i] = gpool[b * C + c] * inv_hw;
  }
}

// p0 (nullable): the cotangent's bf16 single plane (bf16 tape path), same pass; bmax (nullable):
// per-CTA max |g| for the fp16 pair's scale (planes.cuh), split afterwards
__global__ void broadcast_kernel_vec4(const float* __restrict__ gpool, int64_t hw, int C, int64_t total4,
                                      float inv_hw, float4* __restrict__ g, uint2* __restrict__ p0,
                                      float* __restrict__ bmax) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 4;
    const int c = (int)(e % C);
    const int64_t b = e / ((int64_t)C * hw);
    const float* gp = gpool + b * C + c;
    const float4 v = make_float4(gp[0] * inv_hw, gp[1] * inv_hw, gp[2] * inv_hw, gp[3] * inv_hw);
    g[i] = v;
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    if (p0) {
      const float vv[4] = {v.x, v.y, v.z, v.w};
      p0[i] = pack_single4(vv);
    }
  }
  if (bmax) {
    __shared__ float sh[8];
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, sh[w]);
      bmax[blockIdx.x] = fmaxf(m, sh[0]);
    }
  }
}

__global__ void argmax_hits_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels, int nrows,
                                   int classes, unsigned long long* hits) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nrows; b += gridDim.x * blockDim.x) {
    const float* l = logits + (int64_t)b * classes;
    int best = 0;
    for (int c = 1; c < classes; ++c)
      if (l[c] > l[best]) best = c;  // strict: ties -> lowest class (network.cpp:229)
    if (best == labels[b]) atomicAdd(hits, 1ULL);  // integer: order-independent
  }
}

int64_t align256(int64_t v) { return (v + 255) / 256 * 256; }

// Evaluation (network.cpp:193-234): per row the softmax-CE term lse - logit[y] (fp64, max-shifted,
// as loss_grad_kernel) and the argmax (strict '>': ties to the lowest class), one warp per row;
// per-CTA fp64 partial sums of the loss terms and hit counts in fixed order.
constexpr int kEvalRows = 8;   // rows (warps) per CTA
__global__ void eval_rows_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels, int nrows,
                                 int classes, double* __restrict__ part_loss, unsigned long long* __restrict__ part_hits,
                                 int32_t* __restrict__ pred) {
  __shared__ double sl[kEvalRows];
  __shared__ unsigned long long sh[kEvalRows];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kEvalRows + w;
  double term = 0.0;
  unsigned long long hit = 0;
  if (b < nrows) {
    const float* l = logits + (int64_t)b * classes;
    // argmax, lowest index on ties: per-lane best, then a fixed-order butterfly on (value, index)
    float bv = -INFINITY;
    int bi = classes;
    double m = -INFINITY;
    for (int c = lane; c < classes; c += 32) {
      const float v = l[c];
      if (v > bv) bv = v, bi = c;
      m = fmax(m, (double)v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    double z = 0.0;
    for (int c = lane; c < classes; c += 32) z += exp((double)l[c] - m);
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    const int y = labels[b];
    term = (y >= 0 && y < classes) ? m + log(z) - (double)l[y] : __longlong_as_double(0x7ff8000000000000LL);
    hit = bi == y ? 1ull : 0ull;
    if (pred && lane == 0) pred[b] = bi;
  }
  if (lane == 0) {
    sl[w] = term;
    sh[w] = hit;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    unsigned long long h = 0;
    for (int i = 0; i < kEvalRows; ++i) s += sl[i], h += sh[i];
    part_loss[blockIdx.x] = s;
    part_hits[blockIdx.x] = h;
  }
}

__global__ void eval_final_kernel(const double* __restrict__ part_loss, const unsigned long long* __restrict__ part_hits,
                                  int nparts, int nrows, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    unsigned long long h = 0;
    for (int i = 0; i < nparts; ++i) s += part_loss[i], h += part_hits[i];
    out[0] = nrows ? s / (double)nrows : 0.0;
    out[1] = (double)h;
  }
}

}  // namespace

int64_t eval_ws_bytes(int nrows) {
  const int64_t parts = (nrows + kEvalRows - 1) / kEvalRows;
  return align256(parts * 8) * 2 + 256;
}

void eval_loss_hits(const float* logits, const int32_t* labels, int nrows, int classes, double* out2, int32_t* pred,
                    void* ws, cudaStream_t st) {
  const int parts = std::max(1, (nrows + kEvalRows - 1) / kEvalRows);
  double* pl = static_cast<double*>(ws);
  auto* ph = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + align256((int64_t)parts * 8));
  if (nrows > 0) {
    eval_rows_kernel<<<parts, 32 * kEvalRows, 0, st>>>(logits, labels, nrows, classes, pl, ph, pred);
    RP_LAUNCHED();
  }
  eval_final_kernel<<<1, 32, 0, st>>>(pl, ph, nrows > 0 ? parts : 0, nrows, out2);
  RP_LAUNCHED();
}

int64_t head_ws_bytes(int nrows, int channels, int classes) {
  return align256((int64_t)nrows * classes * 4) + align256((int64_t)nrows * 8) + align256((int64_t)nrows * channels * 4);
}

void head_forward(int nrows, int hw, int C, int classes, const float* x_end, const float* t_w, const float* t_b,
                  float* pooled, float* logits, cudaStream_t st) {
  if (nrows <= 0) return;
  const int cw = C < 256 ? C : 256;
  const int groups = C <= 256 ? (256 / C > 0 ? 256 / C : 1) : 1;
  if (C % 4 == 0 && kGapThreads % (C / 4) == 0 && (reinterpret_cast<uintptr_t>(x_end) & 15u) == 0) {
    gap_kernel_vec4<<<nrows, kGapThreads, kGapThreads * sizeof(float4), st>>>(
        reinterpret_cast<const float4*>(x_end), hw, C / 4, pooled);
  } else {
    gap_kernel<<<nrows, 256, groups * cw * sizeof(float), st>>>(x_end, hw, C, pooled);
  }
  RP_LAUNCHED();
  fc_kernel<<<nrows, 32, 0, st>>>(pooled, t_w, t_b, C, classes, logits);
  RP_LAUNCHED();
}

void head_loss_backward(int nrows, int hw, int C, int classes, const float* pooled, const float* logits,
                        const float* t_w, const int32_t* labels, double* loss_dev, float* gt_w, float* gt_b,
                        float* g_out, void* ws, cudaStream_t st, void* p0, void* p1, float* scale) {
  if (nrows <= 0) return;
  if (p1 && !scale) fail(RP_ERR_INTERNAL, "head_loss_backward: the cotangent plane pair needs a scale buffer");
  char* w = static_cast<char*>(ws);
  float* glog = reinterpret_cast<float*>(w);
  double* loss_b = reinterpret_cast<double*>(w + align256((int64_t)nrows * classes * 4));
  float* gpool = reinterpret_cast<float*>(w + align256((int64_t)nrows * classes * 4) + align256((int64_t)nrows * 8));
  loss_grad_kernel<<<nrows, 128, 0, st>>>(logits, labels, t_w, nrows, C, classes, glog, loss_b, gpool);
  RP_LAUNCHED();
  const int total = C * classes + classes + 1;
  head_param_grad_kernel<<<ceil_div((int64_t)total * 32, 256), 256, 0, st>>>(pooled, glog, loss_b, nrows, C, classes,
                                                                            gt_w, gt_b, loss_dev);
  RP_LAUNCHED();
  const int64_t n = (int64_t)nrows * hw * C;
  const float inv = 1.f / (float)hw;
  const int grid = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, 2 * kPlaneScaleMaxParts);
  if (C % 4 == 0 && (reinterpret_cast<uintptr_t>(g_out) & 15u) == 0) {
    float* part = p1 ? scale + kPlaneScalePartOffset : nullptr;
    broadcast_kernel_vec4<<<grid, 256, 0, st>>>(gpool, hw, C, n / 4, inv, reinterpret_cast<float4*>(g_out),
                                                p1 ? nullptr : static_cast<uint2*>(p0), part);
    RP_LAUNCHED();
    if (p1) split_planes_from_parts(g_out, n, p0, p1, part, grid, scale, st);
    return;
  }
  broadcast_kernel<<<grid, 256, 0, st>>>(gpool, hw, C, n, inv, g_out);
  RP_LAUNCHED();
  if (p0) split_planes(g_out, n, p0, p1, st, p1 ? scale : nullptr);
}

void argmax_hits(const float* logits, const int32_t* labels, int nrows, int classes, unsigned long long* hits_dev,
                 cudaStream_t st) {
  RP_CUDA(cudaMemsetAsync(hits_dev, 0, sizeof(unsigned long long), st));
  if (nrows <= 0) return;
  argmax_hits_kernel<<<ceil_div(nrows, 128), 128, 0, st>>>(logits, labels, nrows, classes, hits_dev);
  RP_LAUNCHED();
}

}  // namespace rp::k
