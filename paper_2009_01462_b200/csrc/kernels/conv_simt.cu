// SIMT-FFMA fp32 implicit-GEMM 3x3 convolutions (NHWC, zero pad 1, stride 1).
//
// This is the CUDA-core path: exact fp32 products, fixed accumulation order.  It
// is kept (RP_MATH_SIMT) as the on-device cross-check of the tcgen05 kernels and
// for shapes the tensor-core kernels do not take.  The hot path is conv_tc.cu.
//
//   fprop : out[m][co] = sum_{tap,ci} in[m + off(tap)][ci] * w[tap][ci][co]
//           (matmul(x, W1) / matmul(a, W2), network.cpp:85,87, generalised)
//   dgrad : fprop of the cotangent with wd[tap'][co][ci] = w[8-tap'][ci][co]
//           (matmul(upstream, W2^T), matmul(dpre, W1^T), network.cpp:100,104)
//   wgrad : gw[tap][ci][co] = sum_m in[m + off(tap)][ci] * g[m][co]   + bias sums
//           (matmul(a^T, upstream), matmul(x^T, dpre), col_sum, network.cpp:98-103)
//           deterministic split-K: fixed pixel ranges, fixed-order final sum.
#include "../common.cuh"
#include "kernels.cuh"

namespace rp::k {

namespace {

struct FwdArgs {
  const float* in;
  const float* w;
  const float* bias;
  const float* aux;
  float* out;
  int N, H, W, Ci, Co, M, K;
  float h;
};

template <int EPI>
__device__ __forceinline__ float epi_apply(float v, int64_t idx, int co, const FwdArgs& a) {
  if constexpr (EPI == EPI_BIAS) return v + a.bias[co];
  if constexpr (EPI == EPI_BIAS_TANH) return tanhf(v + a.bias[co]);
  if constexpr (EPI == EPI_RESID) return a.aux[idx] + a.h * (v + a.bias[co]);
  if constexpr (EPI == EPI_TANH_BWD) {
    const float t = a.aux[idx];
    return (a.h * v) * (1.f - t * t);
  }
  if constexpr (EPI == EPI_ADD) return a.aux[idx] + v;
  return a.h * v;  // EPI_SCALE
}

constexpr int BM = 128, BN = 64, BK = 16, APAD = 4;

template <int EPI>
__global__ __launch_bounds__(256) void conv3x3_fwd_simt_kernel(FwdArgs a) {
  __shared__ __align__(16) float As[2][BK][BM + APAD];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int HW = a.H * a.W;

  // A loads: fixed k lane, 8 pixel rows per thread
  const int a_kk = tid & 15;
  const int a_r0 = tid >> 4;
  int pn[8], py[8], px[8];
  bool pv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + a_r0 + 16 * i;
    pv[i] = m < a.M;
    const int mm = pv[i] ? m : 0;
    pn[i] = mm / HW;
    const int rem = mm - pn[i] * HW;
    py[i] = rem / a.W;
    px[i] = rem - py[i] * a.W;
  }
  const int b_c = tid & 63, b_k0 = tid >> 6;
  float ra[8], rb[4];

  auto load_tile = [&](int k0) {
    const int kg = k0 + a_kk;
    const bool kv = kg < a.K;
    const int tap = kv ? kg / a.Ci : 0;
    const int ci = kg - tap * a.Ci;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int y = py[i] + dy, x = px[i] + dx;
      const bool ok = kv && pv[i] && y >= 0 && y < a.H && x >= 0 && x < a.W;
      ra[i] = ok ? __ldg(a.in + (((int64_t)pn[i] * a.H + y) * a.W + x) * a.Ci + ci) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kr = k0 + b_k0 + 4 * i;
      const int c = n0 + b_c;
      rb[i] = (kr < a.K && c < a.Co) ? __ldg(a.w + (int64_t)kr * a.Co + c) : 0.f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) As[buf][a_kk][a_r0 + 16 * i] = ra[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) Bs[buf][b_k0 + 4 * i][b_c] = rb[i];
  };

  const int tx = tid & 15, ty = tid >> 4;
  float acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;

  const int nk = (a.K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    if (t + 1 < nk) load_tile((t + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * 8 + 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[cur][kk][tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
    }
    if (t + 1 < nk) store_tile(cur ^ 1);
    __syncthreads();
  }

  const int co0 = n0 + tx * 4;
  const bool vec = (a.Co % 4 == 0) && (co0 + 3 < a.Co);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int m = m0 + ty * 8 + r;
    if (m >= a.M) continue;
    const int64_t base = (int64_t)m * a.Co;
    if (vec) {
      float4 o;
      o.x = epi_apply<EPI>(acc[r][0], base + co0 + 0, co0 + 0, a);
      o.y = epi_apply<EPI>(acc[r][1], base + co0 + 1, co0 + 1, a);
      o.z = epi_apply<EPI>(acc[r][2], base + co0 + 2, co0 + 2, a);
      o.w = epi_apply<EPI>(acc[r][3], base + co0 + 3, co0 + 3, a);
      *reinterpret_cast<float4*>(a.out + base + co0) = o;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (co0 + c < a.Co) a.out[base + co0 + c] = epi_apply<EPI>(acc[r][c], base + co0 + c, co0 + c, a);
    }
  }
}

__global__ void dgrad_weights_kernel(const float* __restrict__ w, int ci, int co, float* __restrict__ wd) {
  const int total = 9 * ci * co;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    // idx enumerates wd[tap'][o][i]
    const int i = idx % ci;
    const int o = (idx / ci) % co;
    const int tap = idx / (ci * co);
    const int src_tap = 8 - tap;
    wd[idx] = w[((int64_t)src_tap * ci + i) * co + o];
  }
}

// ---------------------------------------------------------------- wgrad
struct WgArgs {
  const float* in;
  const float* g;
  float* ws;   // float [splits][K][Co], then double [splits][Co] (bias)
  int N, H, W, Ci, Co, M, K;
  int pix_per_split;
  int splits;
};

constexpr int WT = 64, WP = 16, WPAD = 4;

// float offset of the fp64 bias partials: after the weight partials, 64-byte aligned
__host__ __device__ inline int64_t bias_offset(int splits, int K, int Co) {
  return ((int64_t)splits * K * Co + 15) / 16 * 16;
}

__global__ __launch_bounds__(256) void conv3x3_wgrad_simt_kernel(WgArgs a) {
  __shared__ __align__(16) float As[2][WP][WT + WPAD];
  __shared__ __align__(16) float Gs[2][WP][WT + WPAD];
  const int tid = threadIdx.x;
  const int k0 = blockIdx.x * WT;
  const int c0 = blockIdx.y * WT;
  const int split = blockIdx.z;
  const int p_beg = split * a.pix_per_split;
  const int p_end = min(a.M, p_beg + a.pix_per_split);
  const int HW = a.H * a.W;

  const int lane_k = tid & 63;  // k (for A) / co (for G) column of this thread's loads
  const int prow0 = tid >> 6;   // pixel rows prow0 + 4 i
  const int kg = k0 + lane_k;
  const bool kv = kg < a.K;
  const int tap = kv ? kg / a.Ci : 0;
  const int ci = kg - tap * a.Ci;
  const int dy = tap / 3 - 1, dx = tap % 3 - 1;
  const int cg = c0 + lane_k;
  const bool cv = cg < a.Co;

  float ra[4], rg[4];
  auto load_chunk = [&](int pb) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = pb + prow0 + 4 * i;
      float va = 0.f, vg = 0.f;
      if (m < p_end) {
        const int n = m / HW;
        const int rem = m - n * HW;
        const int y = rem / a.W + dy, x = rem % a.W + dx;
        if (kv && y >= 0 && y < a.H && x >= 0 && x < a.W)
          va = __ldg(a.in + (((int64_t)n * a.H + y) * a.W + x) * a.Ci + ci);
        if (cv) vg = __ldg(a.g + (int64_t)m * a.Co + cg);
      }
      ra[i] = va;
      rg[i] = vg;
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[buf][prow0 + 4 * i][lane_k] = ra[i];
      Gs[buf][prow0 + 4 * i][lane_k] = rg[i];
    }
  };

  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
  double bacc[4] = {0.0, 0.0, 0.0, 0.0};  // bias sums in fp64: col_sum over up to 10^6 pixels
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const bool do_bias = blockIdx.x == 0 && ty == 0;

  const int nchunks = p_end > p_beg ? (p_end - p_beg + WP - 1) / WP : 0;
  if (nchunks > 0) {
    load_chunk(p_beg);
    store_chunk(0);
  }
  __syncthreads();
  for (int t = 0; t < nchunks; ++t) {
    const int cur = t & 1;
    if (t + 1 < nchunks) load_chunk(p_beg + (t + 1) * WP);
#pragma unroll
    for (int p = 0; p < WP; ++p) {
      const float4 av = *reinterpret_cast<const float4*>(&As[cur][p][ty * 4]);
      const float4 gv = *reinterpret_cast<const float4*>(&Gs[cur][p][tx * 4]);
      const float aa[4] = {av.x, av.y, av.z, av.w};
      const float gg[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(aa[i], gg[j], acc[i][j]);
      if (do_bias) {
#pragma unroll
        for (int j = 0; j < 4; ++j) bacc[j] += (double)gg[j];
      }
    }
    if (t + 1 < nchunks) store_chunk(cur ^ 1);
    __syncthreads();
  }

  float* part = a.ws + (int64_t)split * a.K * a.Co;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty * 4 + i;
    if (k >= a.K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c < a.Co) part[(int64_t)k * a.Co + c] = acc[i][j];
    }
  }
  if (do_bias) {
    double* pb = reinterpret_cast<double*>(a.ws + bias_offset(a.splits, a.K, a.Co)) + (int64_t)split * a.Co;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c < a.Co) pb[c] = bacc[j];
    }
  }
}

// fixed-order fp64 combine of the split-K partials
template <class T>
__global__ void splitk_reduce_kernel(const T* __restrict__ ws, int splits, int64_t n, double scale,
                                     float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += (double)ws[(int64_t)k * n + i];
    out[i] = (float)(scale * s);
  }
}

struct SplitPlan {
  int splits, pix_per_split;
};

SplitPlan plan_wgrad(const ConvShape& s) {
  const int64_t M = s.pixels();
  const int tiles = ceil_div(9 * s.ci, WT) * ceil_div(s.co, WT);
  int64_t splits = (4 * kNumSMs + tiles - 1) / tiles;
  const int64_t max_splits = (M + 255) / 256;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int64_t pps = (M + splits - 1) / splits;
  pps = (pps + WP - 1) / WP * WP;
  splits = (M + pps - 1) / pps;
  if (splits < 1) splits = 1;
  return {static_cast<int>(splits), static_cast<int>(pps)};
}

}  // namespace

void conv3x3_fwd_simt(const ConvShape& s, const float* in, const float* w, const float* bias, const float* aux,
                      float h, int epi, float* out, cudaStream_t st) {
  FwdArgs a{in, w, bias, aux, out, s.n, s.h, s.w, s.ci, s.co, (int)s.pixels(), 9 * s.ci, h};
  if (a.M == 0) return;
  dim3 grid(ceil_div(a.M, BM), ceil_div(s.co, BN));
  switch (epi) {
    case EPI_BIAS: conv3x3_fwd_simt_kernel<EPI_BIAS><<<grid, 256, 0, st>>>(a); break;
    case EPI_BIAS_TANH: conv3x3_fwd_simt_kernel<EPI_BIAS_TANH><<<grid, 256, 0, st>>>(a); break;
    case EPI_RESID: conv3x3_fwd_simt_kernel<EPI_RESID><<<grid, 256, 0, st>>>(a); break;
    case EPI_TANH_BWD: conv3x3_fwd_simt_kernel<EPI_TANH_BWD><<<grid, 256, 0, st>>>(a); break;
    case EPI_ADD: conv3x3_fwd_simt_kernel<EPI_ADD><<<grid, 256, 0, st>>>(a); break;
    default: conv3x3_fwd_simt_kernel<EPI_SCALE><<<grid, 256, 0, st>>>(a); break;
  }
  RP_LAUNCHED();
}

void conv3x3_dgrad_weights(const float* w, int ci, int co, float* wd, cudaStream_t st) {
  const int total = 9 * ci * co;
  dgrad_weights_kernel<<<ceil_div(total, 256), 256, 0, st>>>(w, ci, co, wd);
  RP_LAUNCHED();
}

int64_t conv3x3_wgrad_ws_bytes(const ConvShape& s) {
  const SplitPlan p = plan_wgrad(s);
  return bias_offset(p.splits, 9 * s.ci, s.co) * 4 + (int64_t)p.splits * s.co * 8;
}

void conv3x3_wgrad_simt(const ConvShape& s, const float* in, const float* g, float scale, float* gw, float* gb,
                        void* ws, cudaStream_t st) {
  const SplitPlan p = plan_wgrad(s);
  WgArgs a{in, g, static_cast<float*>(ws), s.n, s.h, s.w, s.ci, s.co, (int)s.pixels(), 9 * s.ci,
           p.pix_per_split, p.splits};
  dim3 grid(ceil_div(a.K, WT), ceil_div(s.co, WT), p.splits);
  conv3x3_wgrad_simt_kernel<<<grid, 256, 0, st>>>(a);
  RP_LAUNCHED();
  const int64_t nw = (int64_t)a.K * s.co;
  splitk_reduce_kernel<float><<<ceil_div(nw, 256), 256, 0, st>>>(a.ws, p.splits, nw, scale, gw);
  RP_LAUNCHED();
  if (gb) {
    const double* pb = reinterpret_cast<const double*>(a.ws + bias_offset(p.splits, a.K, s.co));
    splitk_reduce_kernel<double><<<ceil_div(s.co, 256), 256, 0, st>>>(pb, p.splits, s.co, scale, gb);
    RP_LAUNCHED();
  }
}

}  // namespace rp::k
