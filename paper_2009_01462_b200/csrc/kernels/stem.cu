// The stem S: a 3x3 conv from the raw image channels (Cin <= 4) to C channels
// (affine_forward S, network.cpp:108-110, as a conv) and its weight gradient
// (net_vjp's S grads, network.cpp:165-170).  With Cin = 3 the conv is 27 MACs per
// output: the cost is writing / reading the C-channel activation, so these kernels
// are plain CUDA-core streaming kernels sized for HBM, not implicit GEMMs.
//
//   fwd  : x0[p][co] = s_b[co] + sum_{tap, ci} x[p + off(tap)][ci] * s_w[tap][ci][co]
//   wgrad: gw[tap][ci][co] = scale * sum_p x[p + off(tap)][ci] * g[p][co],
//          gb[co] = scale * sum_p g[p][co]   (deterministic: fixed position ranges per
//          CTA, fixed-order lane / CTA reductions)
#include <cuda_bf16.h>

#include "../common.cuh"
#include "kernels.cuh"
#include "planes.cuh"

namespace rp::k {

namespace {

constexpr int kStemMaxCin = 4;
constexpr int kStemTilesMax = 3;
constexpr int kStemXItems = 3;         // wgrad im2col (position, tap) items per thread and chunk
constexpr int kStemGItems = 6;         // wgrad g float4s per thread and chunk       // wgrad register tiles per thread ((9 Cin + 1) / 4 x C / 8 <= 768)
constexpr int kStemGrid = 8 * kNumSMs;   // wgrad partials (8 CTAs / SM hide the gather latency)

template <int Cin>
__global__ __launch_bounds__(256) void stem_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                       const float* __restrict__ b, int N, int H, int W, int C,
                                                       float* __restrict__ out) {
  extern __shared__ float ws[];   // [9 * Cin * C] weights then [C] bias
  const int nw = 9 * Cin * C;
  for (int i = threadIdx.x; i < nw + C; i += blockDim.x) ws[i] = i < nw ? w[i] : b[i - nw];
  __syncthreads();
  const int groups = C / 16;
  const int64_t items = (int64_t)N * H * W * groups;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(it % groups);
    const int64_t p = it / groups;
    const int xq = (int)(p % W);
    const int yq = (int)((p / W) % H);
    const int64_t n = p / ((int64_t)W * H);
    const int c0 = cg * 16;
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = ws[nw + c0 + j];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int yy = yq + tap / 3 - 1, xx = xq + tap % 3 - 1;
      if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
      const float* xp = x + ((n * H + yy) * W + xx) * Cin;
#pragma unroll
      for (int ci = 0; ci < Cin; ++ci) {
        const float v = __ldg(xp + ci);
        const float4* wr = reinterpret_cast<const float4*>(ws + (tap * Cin + ci) * C + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 wv = wr[q];
          acc[4 * q + 0] = fmaf(v, wv.x, acc[4 * q + 0]);
          acc[4 * q + 1] = fmaf(v, wv.y, acc[4 * q + 1]);
          acc[4 * q + 2] = fmaf(v, wv.z, acc[4 * q + 2]);
          acc[4 * q + 3] = fmaf(v, wv.w, acc[4 * q + 3]);
        }
      }
    }
    float4* o = reinterpret_cast<float4*>(out + p * C + c0);
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
}

// Register-blocked variant for W % 4 == 0: a thread computes 4 consecutive positions
// of one row x CG channels, so every weight float4 read from smem feeds 16 FMAs.  CG = 8
// keeps the accumulators at 32 registers: 3 CTAs / SM instead of 2 hide the smem latency.
template <int Cin, int CG>
__global__ __launch_bounds__(256, CG == 8 ? 3 : 2) void stem_fwd4_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                        const float* __restrict__ b, int N, int H, int W, int C,
                                                        float* __restrict__ out, uint2* __restrict__ p0,
                                                        uint2* __restrict__ p1) {
  extern __shared__ float ws[];
  const int nw = 9 * Cin * C;
  for (int i = threadIdx.x; i < nw + C; i += blockDim.x) ws[i] = i < nw ? w[i] : b[i - nw];
  __syncthreads();
  const int groups = C / CG;
  const int64_t items = (int64_t)N * H * (W / 4) * groups;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(it % groups);
    const int64_t q = it / groups;                     // quad of positions
    const int x0 = (int)(q % (W / 4)) * 4;
    const int yq = (int)((q / (W / 4)) % H);
    const int64_t n = q / ((int64_t)(W / 4) * H);
    const int c0 = cg * CG;
    float acc[4][CG];
#pragma unroll
    for (int j = 0; j < CG; ++j) {
      const float bj = ws[nw + c0 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][j] = bj;
    }
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const int yy = yq + dy - 1;
      if (yy < 0 || yy >= H) continue;
      const float* row = x + (n * H + yy) * (int64_t)W * Cin;
      // the 6 input columns x0-1 .. x0+4 of this row (zero outside)
      float xv[6][Cin];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int xx = x0 + k - 1;
#pragma unroll
        for (int ci = 0; ci < Cin; ++ci) xv[k][ci] = (xx >= 0 && xx < W) ? __ldg(row + (int64_t)xx * Cin + ci) : 0.f;
      }
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
        for (int ci = 0; ci < Cin; ++ci) {
          const float4* wr = reinterpret_cast<const float4*>(ws + ((dy * 3 + dx) * Cin + ci) * C + c0);
#pragma unroll
          for (int qq = 0; qq < CG / 4; ++qq) {
            const float4 wv = wr[qq];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float v = xv[i + dx][ci];
              acc[i][4 * qq + 0] = fmaf(v, wv.x, acc[i][4 * qq + 0]);
              acc[i][4 * qq + 1] = fmaf(v, wv.y, acc[i][4 * qq + 1]);
              acc[i][4 * qq + 2] = fmaf(v, wv.z, acc[i][4 * qq + 2]);
              acc[i][4 * qq + 3] = fmaf(v, wv.w, acc[i][4 * qq + 3]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float4* o = reinterpret_cast<float4*>(out + ((n * H + yq) * (int64_t)W + x0 + i) * C + c0);
#pragma unroll
      for (int qq = 0; qq < CG / 4; ++qq)
        o[qq] = make_float4(acc[i][4 * qq], acc[i][4 * qq + 1], acc[i][4 * qq + 2], acc[i][4 * qq + 3]);
      if (p0) {   // the first block's input planes (planes.cuh), as split_planes makes them
        const int64_t e4 = (((n * H + yq) * (int64_t)W + x0 + i) * C + c0) / 4;
#pragma unroll
        for (int qq = 0; qq < CG / 4; ++qq) {
          const float v[4] = {acc[i][4 * qq], acc[i][4 * qq + 1], acc[i][4 * qq + 2], acc[i][4 * qq + 3]};
          if (p1)
            pack_pair4(v, kActPlaneScale, p0[e4 + qq], p1[e4 + qq]);   // fp32 path: the fp16 pair
          else
            p0[e4 + qq] = pack_single4(v);                  // bf16 tape path: the bf16 copy
        }
      }
    }
  }
}

// Weight gradient as a small GEMM gW[r][co] = sum_p X[p][r] g[p][co] over the im2col
// rows r = (tap, ci) plus a ones row (r = 9 Cin: the bias).  CTA b owns positions
// [b P / G, (b+1) P / G), staged PC at a time into smem; thread (half h, row quad rb,
// channel octet cb) accumulates a 4 x 8 register tile over the positions pp = h mod halves
// (3 smem float4 loads per 32 FMAs).
// When the tiles outnumber the threads (Cin = 4, C = 256: 10 x 32 = 320 tiles), every
// thread owns up to kStemTiles tiles (t, t + 256, ...) and halves = 1.
template <int Cin, int kStemTiles>
__global__ __launch_bounds__(256) void stem_wgrad_gemm_kernel(const float* __restrict__ x,
                                                              const float* __restrict__ g, int N, int H, int W,
                                                              int C, int PC, float* __restrict__ part) {
  constexpr int R = 9 * Cin + 1;
  constexpr int RP = (R + 3) / 4 * 4;
  extern __shared__ __align__(16) float sm[];
  float* X = sm;                   // [PC][RP]
  float* G = sm + PC * RP;         // [PC][C]
  const int C4 = C / 4, C8 = C / 8, nt = (RP / 4) * C8;   // 4 rows x 8 channels per tile
  const int halves = max(1, 256 / nt);
  const int t = threadIdx.x;
  const int h = nt >= 256 ? 0 : t / nt;
  const bool active = h < halves;
  int rbs[kStemTiles], cbs[kStemTiles];
  bool own[kStemTiles];
#pragma unroll
  for (int j = 0; j < kStemTiles; ++j) {
    const int q = nt >= 256 ? t + 256 * j : (j == 0 ? t % nt : nt);
    own[j] = active && q < nt;
    rbs[j] = own[j] ? q / C8 : 0;
    cbs[j] = own[j] ? q % C8 : 0;
  }
  const int64_t P = (int64_t)N * H * W;
  const int64_t p0 = blockIdx.x * P / gridDim.x, p1 = (blockIdx.x + 1) * P / gridDim.x;
  float acc[kStemTiles][4][8] = {};
  // the next chunk's im2col items and g float4s wait in registers while this chunk is
  // multiplied (kStemXItems * 256 >= PC * 9, kStemGItems * 256 >= PC * C / 4: host-checked)
  float xr[kStemXItems][Cin];
  float4 gr[kStemGItems];
  auto fetch = [&](int64_t c0, int np) {
#pragma unroll
    for (int j = 0; j < kStemXItems; ++j) {
      const int i = t + 256 * j;
      const int pp = i / 9, tap = i - pp * 9;
#pragma unroll
      for (int ci = 0; ci < Cin; ++ci) xr[j][ci] = 0.f;
      if (pp < np) {
        // the position's (n, y, x) from 32-bit divisions (P < 2^32, checked on the host)
        const uint32_t p = (uint32_t)(c0 + pp);
        const uint32_t r1 = p / (uint32_t)W, xq = p - r1 * (uint32_t)W;
        const uint32_t n = r1 / (uint32_t)H, yq = r1 - n * (uint32_t)H;
        const int yy = (int)yq + tap / 3 - 1, xx = (int)xq + tap % 3 - 1;
        if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
          const float* src = x + (((int64_t)n * H + yy) * W + xx) * Cin;
#pragma unroll
          for (int ci = 0; ci < Cin; ++ci) xr[j][ci] = __ldg(src + ci);
        }
      }
    }
    const float4* g4 = reinterpret_cast<const float4*>(g + c0 * C);
#pragma unroll
    for (int j = 0; j < kStemGItems; ++j) {
      const int i = t + 256 * j;
      gr[j] = i < np * C4 ? __ldg(g4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  const float4* X4 = reinterpret_cast<const float4*>(X);
  float4* G4 = reinterpret_cast<float4*>(G);
  if (p0 < p1) fetch(p0, (int)(p1 - p0 < (int64_t)PC ? p1 - p0 : (int64_t)PC));
  for (int64_t c0 = p0; c0 < p1; c0 += PC) {
    const int np = (int)(p1 - c0 < (int64_t)PC ? p1 - c0 : (int64_t)PC);
    __syncthreads();   // the previous chunk's products have read X and G
#pragma unroll
    for (int j = 0; j < kStemXItems; ++j) {
      const int i = t + 256 * j;
      if (i < PC * 9) {
        const int pp = i / 9, tap = i - pp * 9;
#pragma unroll
        for (int ci = 0; ci < Cin; ++ci) X[pp * RP + tap * Cin + ci] = xr[j][ci];
      }
    }
    // the ones row (bias) and the padding rows
    for (int i = t; i < PC * (RP - 9 * Cin); i += blockDim.x) {
      const int pp = i / (RP - 9 * Cin), j = i - pp * (RP - 9 * Cin);
      X[pp * RP + 9 * Cin + j] = (j == 0 && pp < np) ? 1.f : 0.f;
    }
#pragma unroll
    for (int j = 0; j < kStemGItems; ++j) {
      const int i = t + 256 * j;
      if (i < PC * C4) G4[i] = gr[j];
    }
    __syncthreads();
    if (c0 + PC < p1) fetch(c0 + PC, (int)(p1 - c0 - PC < (int64_t)PC ? p1 - c0 - PC : (int64_t)PC));
    if (kStemTiles == 1) {
      if (active) {   // one tile: no per-tile branch, two positions in flight
        const float4* xp = X4 + rbs[0];
        const float4* gp = G4 + 2 * cbs[0];
#pragma unroll 2
        for (int pp = h; pp < np; pp += halves) {
          const float4 xv = xp[pp * (RP / 4)];
          const float4 gv = gp[pp * C4], gv2 = gp[pp * C4 + 1];
          const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
          const float ga[8] = {gv.x, gv.y, gv.z, gv.w, gv2.x, gv2.y, gv2.z, gv2.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[0][i][j] = fmaf(xa[i], ga[j], acc[0][i][j]);
        }
      }
    } else if (active) {
      for (int pp = h; pp < np; pp += halves) {
#pragma unroll
        for (int q = 0; q < kStemTiles; ++q) {
          if (!own[q]) continue;
          const float4 xv = X4[pp * (RP / 4) + rbs[q]];
          const float4 gv = G4[pp * C4 + 2 * cbs[q]], gv2 = G4[pp * C4 + 2 * cbs[q] + 1];
          const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
          const float ga[8] = {gv.x, gv.y, gv.z, gv.w, gv2.x, gv2.y, gv2.z, gv2.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[q][i][j] = fmaf(xa[i], ga[j], acc[q][i][j]);
        }
      }
    }
  }
  // fixed-order combine of the halves, then the CTA partial [RP][C]
  __syncthreads();
  float* red = sm;                 // [halves][RP][C]
#pragma unroll
  for (int q = 0; q < kStemTiles; ++q)
    if (own[q])
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) red[((size_t)h * RP + rbs[q] * 4 + i) * C + cbs[q] * 8 + j] = acc[q][i][j];
  __syncthreads();
  for (int i = t; i < RP * C; i += blockDim.x) {
    float s = 0.f;
    for (int hh = 0; hh < halves; ++hh) s += red[(size_t)hh * RP * C + i];
    part[(int64_t)blockIdx.x * RP * C + i] = s;
  }
}

// out[i] = scale * sum_b part[b][i], one warp per output, fixed lane striding and
// shuffle order.  i < 9 Cin C -> gw (HWIO == [tap][ci][co]); the next C -> gb.
// Partials have `rows` rows of C per CTA (rows >= 9 Cin + 1; padding rows ignored).
__global__ void stem_wgrad_reduce_kernel(const float* __restrict__ part, int grid, int Cin, int C, int rows,
                                         double scale, float* __restrict__ gw, float* __restrict__ gb) {
  const int R = 9 * Cin + 1;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (warp >= R * C) return;
  double s = 0.0;
  for (int b = lane; b < grid; b += 32) s += (double)part[(int64_t)b * rows * C + warp];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const int r = warp / C;
    if (r < 9 * Cin)
      gw[warp] = (float)(scale * s);
    else if (gb)
      gb[warp - 9 * Cin * C] = (float)(scale * s);
  }
}

}  // namespace

bool stem_supported(const ConvShape& s) {
  return s.ci >= 1 && s.ci <= kStemMaxCin && s.co % 16 == 0 && s.co <= 256 && 256 % s.co == 0;
}

int64_t stem_wgrad_ws_bytes(const ConvShape& s) {
  return (int64_t)kStemGrid * ((9 * s.ci + 1 + 3) / 4 * 4) * s.co * 4 + 256;
}

void stem_fwd(const ConvShape& s, const float* x, const float* w, const float* b, float* out, cudaStream_t st,
              void* p0, void* p1) {
  const int64_t items = s.pixels() * (s.co / 16);
  const int grid = (int)std::min<int64_t>((items + 255) / 256, 32 * kNumSMs);
  const size_t smem = (size_t)(9 * s.ci * s.co + s.co) * 4;
  const dim3 gr(std::max(grid, 1));
  if (s.w % 4 == 0) {
    constexpr int CG = 8;
    auto* u0 = static_cast<uint2*>(p0);
    auto* u1 = static_cast<uint2*>(p1);
    const int64_t items4 = s.pixels() / 4 * (s.co / CG);
    const dim3 gr4((unsigned)std::max<int64_t>(1, std::min<int64_t>((items4 + 255) / 256, 32 * kNumSMs)));
    switch (s.ci) {
      case 1: stem_fwd4_kernel<1, CG><<<gr4, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out, u0, u1); break;
      case 2: stem_fwd4_kernel<2, CG><<<gr4, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out, u0, u1); break;
      case 3: stem_fwd4_kernel<3, CG><<<gr4, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out, u0, u1); break;
      default: stem_fwd4_kernel<4, CG><<<gr4, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out, u0, u1); break;
    }
    RP_LAUNCHED();
    return;
  }
  switch (s.ci) {
    case 1: stem_fwd_kernel<1><<<gr, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out); break;
    case 2: stem_fwd_kernel<2><<<gr, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out); break;
    case 3: stem_fwd_kernel<3><<<gr, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out); break;
    default: stem_fwd_kernel<4><<<gr, 256, smem, st>>>(x, w, b, s.n, s.h, s.w, s.co, out); break;
  }
  RP_LAUNCHED();
  if (p0) split_planes(out, s.pixels() * s.co, p0, p1, st);
}

// One wave: the grid is what fits the SMs at once (<= kStemGrid partials), so no CTA
// waits for a second wave (the 4 x 8 tile kernel holds 4 CTAs / SM, not 8).
template <typename Kernel>
int one_wave_grid(Kernel k, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem) != cudaSuccess || occ < 1) occ = 1;
  return std::min(kStemGrid, occ * kNumSMs);
}

template <int Cin>
int launch_wgrad_gemm(const ConvShape& s, const float* x, const float* g, float* part, cudaStream_t st) {
  constexpr int RP = (9 * Cin + 1 + 3) / 4 * 4;
  const int PC = std::max(16, std::min(64, 24 * 1024 / ((RP + s.co) * 4)));
  const size_t smem = std::max<size_t>((size_t)PC * (RP + s.co) * 4,
                                       (size_t)std::max(1, 256 / ((RP / 4) * (s.co / 8))) * RP * s.co * 4);
  if (s.pixels() >= (int64_t)1 << 32) fail(RP_ERR_SHAPE, "stem_wgrad: more than 2^32 positions");
  if (PC * 9 > kStemXItems * 256 || PC * s.co / 4 > kStemGItems * 256)
    fail(RP_ERR_INTERNAL, "stem_wgrad: chunk exceeds the register prefetch");
  // one register tile per thread while the tiles fit the 256 threads (registers -> occupancy)
  const int nt = (RP / 4) * (s.co / 8);
  if (nt <= 256) {
    const int grid = one_wave_grid(stem_wgrad_gemm_kernel<Cin, 1>, smem);
    stem_wgrad_gemm_kernel<Cin, 1><<<grid, 256, smem, st>>>(x, g, s.n, s.h, s.w, s.co, PC, part);
    return grid;
  }
  const int grid = one_wave_grid(stem_wgrad_gemm_kernel<Cin, kStemTilesMax>, smem);
  stem_wgrad_gemm_kernel<Cin, kStemTilesMax><<<grid, 256, smem, st>>>(x, g, s.n, s.h, s.w, s.co, PC, part);
  return grid;
}

void stem_wgrad(const ConvShape& s, const float* x, const float* g, float scale, float* gw, float* gb, void* ws,
                cudaStream_t st) {
  float* part = static_cast<float*>(ws);
  int grid;
  switch (s.ci) {
    case 1: grid = launch_wgrad_gemm<1>(s, x, g, part, st); break;
    case 2: grid = launch_wgrad_gemm<2>(s, x, g, part, st); break;
    case 3: grid = launch_wgrad_gemm<3>(s, x, g, part, st); break;
    default: grid = launch_wgrad_gemm<4>(s, x, g, part, st); break;
  }
  RP_LAUNCHED();
  const int rows = (9 * s.ci + 1 + 3) / 4 * 4;
  const int outs = (9 * s.ci + 1) * s.co;
  stem_wgrad_reduce_kernel<<<ceil_div((int64_t)outs * 32, 256), 256, 0, st>>>(part, grid, s.ci, s.co, rows,
                                                                              (double)scale, gw, gb);
  RP_LAUNCHED();
}

}  // namespace rp::k
