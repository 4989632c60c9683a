// tcgen05 weight-gradient kernel for the 3x3 convs (block_vjp's matmul(a^T, upstream)
// and matmul(x^T, dpre) + col_sum, network.cpp:98-103, generalised to 3x3 taps):
//
//   gW[tap][ci][co] = scale * sum_p x[p + off(tap)][ci] * g[p][co],   gb[co] = scale * sum_p g[p][co]
//
// The reduction (GEMM K) runs over output positions p.  As in conv_tc.cu, positions live
// in the zero-padded interior frame (rows x (W+2) columns) of one image, so a tap is a
// constant shift of the x slab; g is zero at the two padding columns (TMA out-of-bounds
// fill), so padded positions contribute nothing.
//
// Operands are MN-major (channels contiguous, K = positions): TMA loads 32 channels x
// positions as 128-byte rows with the 128B/32B-atom swizzle, the only MN-major smem
// layout tf32 UMMA accepts.  The swizzle is a function of absolute shared-memory
// address bits (verified on device by rp_debug_umma_probe_sw32), so a tap shift of s
// positions is simply +128*s bytes of descriptor start address with base_offset 0.
//
//   D[r][(tap, ci)] += sum_p A[r][p] * X_tap[ci][p]
//     3xTF32: A = [g_hi ; g_lo] stacked along M (M = 128 for Co = 64) so one MMA per split
//     of x (hi, lo) yields hi*hi, lo*hi, hi*lo (and lo*lo); the reduce sums the row halves.
//     N = 32 channels of x per MMA; 9 taps in two tap groups (TMEM: 5 x 64 fp32 columns).
//
// Persistent CTAs (1/SM) are split between the tap groups; each accumulates a contiguous
// range of pixel blocks in TMEM and writes one fp32 partial; a fixed-order fp64 reduce
// combines them (deterministic: no atomics).
#include <cuda.h>

#include <map>
#include <mutex>
#include <tuple>

#include "../common.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace rp::k {

namespace {

using namespace rp::umma;

constexpr int kThreads = 320;
constexpr int kXStages = 2;
constexpr int kMaxSmem = 220 * 1024;
constexpr int kPad = 1024;          // zero rows around every x slab (shifted reads)

struct WgArgs {
  int N, H, W, Ci, Co, Wp, rg, P, Pp, nchunks, rowsA, three;
  int tg;                        // taps per group (group 1 holds the rest)
  int ctas_g0;                   // CTAs assigned to tap group 0
  int blocks_per_img, num_blocks;
  uint32_t slab;                 // bytes per 32-channel g slab (Pp rows of 128 B, 1 KB aligned)
  uint32_t xb;                   // bytes per x slab body ((rg+2)*Wp rows, 1 KB aligned)
  uint32_t g_stride;             // bytes per g slot (rowsA/32 slabs)
  uint32_t x_stride;             // bytes per x stage (pad hi pad pad lo pad)
  float* part;                   // [grid][rowsA][tg * Ci]
  double* part_bias;             // [grid][Co]
};

__device__ __forceinline__ float rna_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

__device__ __forceinline__ void split_inplace(float4* hi, float4* lo, int n16, int tid) {
  for (int i = tid; i < n16; i += 128) {
    const float4 v = hi[i];
    float4 h, l;
    h.x = rna_tf32(v.x); h.y = rna_tf32(v.y); h.z = rna_tf32(v.z); h.w = rna_tf32(v.w);
    l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
    hi[i] = h;
    lo[i] = l;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_x,
                    const WgArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nslab = a.rowsA / 32;
  const int nslab_hi = a.Co / 32;

  uint8_t* g_base = smem;
  uint8_t* x_base = smem + 2 * a.g_stride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(x_base + kXStages * a.x_stride);
  uint64_t* g_full = bars;                // [2]
  uint64_t* g_conv = bars + 2;            // [2]
  uint64_t* g_empty = bars + 4;           // [2]
  uint64_t* x_full = bars + 6;            // [kXStages]
  uint64_t* x_conv = bars + 6 + kXStages;
  uint64_t* x_empty = bars + 6 + 2 * kXStages;
  uint64_t* acc_full = bars + 6 + 3 * kXStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 3 * kXStages);
  double* bsum = reinterpret_cast<double*>(bars + 10 + 3 * kXStages);   // [128]

  auto g_slab = [&](int s, int j) { return g_base + s * a.g_stride + j * a.slab; };
  auto x_hi = [&](int s) { return x_base + s * a.x_stride + kPad; };
  auto x_lo = [&](int s) { return x_base + s * a.x_stride + 3 * kPad + a.xb; };

  // CTA -> (tap group, contiguous block range)
  const bool g0 = (int)blockIdx.x < a.ctas_g0;
  const int jg = g0 ? blockIdx.x : blockIdx.x - a.ctas_g0;
  const int ng = g0 ? a.ctas_g0 : gridDim.x - a.ctas_g0;
  const int blk_beg = (int)((int64_t)jg * a.num_blocks / ng);
  const int blk_end = (int)((int64_t)(jg + 1) * a.num_blocks / ng);
  const int t0 = g0 ? 0 : a.tg;
  const int ntaps = g0 ? min(a.tg, 9) : 9 - a.tg;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&g_full[i], 1);
      mbar_init(&g_conv[i], 128);
      mbar_init(&g_empty[i], 1);
    }
    for (int i = 0; i < kXStages; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_conv[i], 128);
      mbar_init(&x_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tmap_g);
    prefetch_tmap(&tmap_x);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  // Zero everything once: the x pads and the g rows P..Pp-1 are read (against zero g)
  // but never written, so they must hold finite values.
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const int n16 = (int)((2 * (size_t)a.g_stride + kXStages * (size_t)a.x_stride) / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int Wp = a.Wp;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int gs = 0, xs = 0;
      uint32_t gph = 0, xph = 0;
      for (int b = blk_beg; b < blk_end; ++b) {
        const int n = b / a.blocks_per_img;
        const int y0 = (b % a.blocks_per_img) * a.rg;
        mbar_wait(&g_empty[gs], gph ^ 1);
        mbar_arrive_expect_tx(&g_full[gs], (uint32_t)nslab_hi * a.P * 128u);
        for (int j = 0; j < nslab_hi; ++j) tma_load_4d(&tmap_g, &g_full[gs], g_slab(gs, j), 32 * j, -1, y0, n);
        if (++gs == 2) gs = 0, gph ^= 1;
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&x_empty[xs], xph ^ 1);
          mbar_arrive_expect_tx(&x_full[xs], (uint32_t)(a.rg + 2) * Wp * 128u);
          tma_load_4d(&tmap_x, &x_full[xs], x_hi(xs), 32 * c, -1, y0 - 1, n);
          if (++xs == kXStages) xs = 0, xph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t id = idesc(2, 128, 32, 1, 1);
      int gs = 0, xs = 0;
      uint32_t gph = 0, xph = 0;
      const int ksteps = a.Pp / 8;
      for (int b = blk_beg; b < blk_end; ++b) {
        mbar_wait(&g_conv[gs], gph);
        tc_fence_after();
        const uint64_t da0 = desc_general(smem_u32(g_slab(gs, 0)), a.slab, 512, 1, 0);
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(a.three ? &x_conv[xs] : &x_full[xs], xph);
          tc_fence_after();
          const uint32_t xh = smem_u32(x_hi(xs)), xl = smem_u32(x_lo(xs));
          for (int ti = 0; ti < ntaps; ++ti) {
            const int t = t0 + ti;
            const int shift = (t / 3) * Wp + (t % 3) - 1;
            const uint64_t dbh0 = desc_general(xh + (uint32_t)(shift * 128), a.xb, 512, 1, 0);
            const uint64_t dbl0 = desc_general(xl + (uint32_t)(shift * 128), a.xb, 512, 1, 0);
            const uint32_t d = tmem_base + (uint32_t)(ti * a.Ci + c * 32);
            for (int k = 0; k < ksteps; ++k) {
              const uint64_t kadv = (uint64_t)(k * 64);     // 8 rows x 128 B, in 16-byte units
              const uint32_t accum = (b > blk_beg || k > 0) ? 1u : 0u;
              mma_tf32(d, da0 + kadv, dbh0 + kadv, id, accum);
              if (a.three) mma_tf32(d, da0 + kadv, dbl0 + kadv, id, 1u);
            }
          }
          mma_commit(&x_empty[xs]);
          if (++xs == kXStages) xs = 0, xph ^= 1;
        }
        mma_commit(&g_empty[gs]);
        if (++gs == 2) gs = 0, gph ^= 1;
      }
      mma_commit(acc_full);
    }
  } else if (warp < 6) {
    // ===================== converters: bias sums + 3xTF32 split =====================
    const int tid = threadIdx.x - 64;
    const int npar = 128 / a.Co;               // threads per bias channel (Co <= 128)
    const int bco = tid % a.Co, bpar = tid / a.Co;
    double bacc = 0.0;
    int gs = 0, xs = 0;
    uint32_t gph = 0, xph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      mbar_wait(&g_full[gs], gph);
      if (g0) {
        // raw g element (p, co): slab co/32, row p, 32-byte granule swizzled by (p & 3)
        const uint8_t* sl = g_slab(gs, bco / 32);
        const int c = bco % 32;
        for (int p = bpar; p < a.P; p += npar) {
          const int gran = (c >> 3) ^ (p & 3);
          bacc += (double)*reinterpret_cast<const float*>(sl + p * 128 + gran * 32 + (c & 7) * 4);
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");   // bias reads finish before hi overwrites
      if (a.three)
        for (int j = 0; j < nslab_hi; ++j)
          split_inplace(reinterpret_cast<float4*>(g_slab(gs, j)), reinterpret_cast<float4*>(g_slab(gs, nslab_hi + j)),
                        a.P * 8, tid);
      fence_proxy_async_smem();
      mbar_arrive(&g_conv[gs]);
      if (++gs == 2) gs = 0, gph ^= 1;
      if (a.three) {
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&x_full[xs], xph);
          split_inplace(reinterpret_cast<float4*>(x_hi(xs)), reinterpret_cast<float4*>(x_lo(xs)),
                        (a.rg + 2) * Wp * 8, tid);
          fence_proxy_async_smem();
          mbar_arrive(&x_conv[xs]);
          if (++xs == kXStages) xs = 0, xph ^= 1;
        }
      }
    }
    if (g0) {
      bsum[tid] = bacc;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid < a.Co) {
        double s = 0.0;
        for (int k = 0; k < npar; ++k) s += bsum[tid + k * a.Co];
        a.part_bias[(size_t)blockIdx.x * a.Co + tid] = s;
      }
    }
    (void)nslab;
  } else {
    // ===================== epilogue: TMEM accumulator -> fp32 partial =====================
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int cols = ntaps * a.Ci;
    float* dst = a.part + ((size_t)blockIdx.x * a.rowsA + row) * (size_t)(a.tg * a.Ci);
    const bool any = blk_end > blk_beg;
    if (any) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    for (int cc = 0; cc < cols; cc += 16) {
      uint32_t r[16];
      tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)cc, r);
      tmem_wait_ld();
      float4* d4 = reinterpret_cast<float4*>(dst + cc);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        d4[v] = any ? make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                  __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// gW[tap][ci][co] (HWIO) = scale * sum over the tap group's CTAs of D[co][col] (+ D[Co+co][col])
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, const double* __restrict__ part_bias, int grid,
                                    int ctas_g0, int tg, int Ci, int Co, int rowsA, int three, double scale,
                                    float* __restrict__ gw, float* __restrict__ gb) {
  const int total = 9 * Ci * Co;
  const int64_t pstride = (int64_t)rowsA * tg * Ci;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total + Co; idx += gridDim.x * blockDim.x) {
    if (idx < total) {
      const int co = idx % Co;
      const int ci = (idx / Co) % Ci;
      const int tap = idx / (Co * Ci);
      const bool grp0 = tap < tg;
      const int ti = grp0 ? tap : tap - tg;
      const int b0 = grp0 ? 0 : ctas_g0;
      const int b1 = grp0 ? ctas_g0 : grid;
      const int64_t col = (int64_t)ti * Ci + ci;
      double s = 0.0;
      for (int b = b0; b < b1; ++b) {
        const float* p = part + b * pstride;
        s += (double)p[(int64_t)co * tg * Ci + col];
        if (three) s += (double)p[(int64_t)(Co + co) * tg * Ci + col];
      }
      gw[idx] = (float)(scale * s);
    } else if (gb) {
      const int co = idx - total;
      double s = 0.0;
      for (int b = 0; b < ctas_g0; ++b) s += part_bias[(int64_t)b * Co + co];
      gb[co] = (float)(scale * s);
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// NHWC as (C, W, H, N); box = 32 channels x (W+2) columns (from x = -1) x rows x 1,
// 128B swizzle with 32-byte atoms.
CUtensorMap make_map(const float* t, int n, int h, int w, int c, int rows) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)c * 4, (cuuint64_t)w * c * 4, (cuuint64_t)h * w * c * 4};
  const cuuint32_t box[4] = {32, (cuuint32_t)(w + 2), (cuuint32_t)rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(t), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled (sw32) failed (" + std::to_string((int)r) + ")");
  return m;
}

std::mutex g_mu;
std::map<std::tuple<const void*, int, int, int, int, int>, CUtensorMap> g_maps;

const CUtensorMap& cached(const float* t, int n, int h, int w, int c, int rows) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple((const void*)t, n, h, w, c, rows);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();
    it = g_maps.emplace(key, make_map(t, n, h, w, c, rows)).first;
  }
  return it->second;
}

uint32_t round1k(uint64_t v) { return (uint32_t)((v + 1023) / 1024 * 1024); }

struct WgPlan {
  bool ok = false;
  int rg, P, Pp, tg, ctas_g0, grid, rowsA;
  uint32_t slab, xb, g_stride, x_stride;
  size_t smem;
};

WgPlan plan(const ConvShape& s, bool three) {
  WgPlan p;
  p.rowsA = (three ? 2 : 1) * s.co;
  if (p.rowsA != 128 || s.ci % 32 != 0 || s.co % 32 != 0 || s.w + 2 > 256) return p;
  const int Wp = s.w + 2;
  const int ngroups = (9 * s.ci + 511) / 512;
  if (ngroups > 2) return p;
  p.tg = (9 + ngroups - 1) / ngroups;
  // largest block (whole padded rows) whose double-buffered g and x stages fit
  for (int rg = std::min(s.h, 8); rg >= 1; --rg) {
    WgPlan q = p;
    q.rg = rg;
    q.P = rg * Wp;
    q.Pp = (q.P + 7) / 8 * 8;
    q.slab = round1k((uint64_t)q.Pp * 128);
    q.xb = round1k((uint64_t)(rg + 2) * Wp * 128 + (q.Pp - q.P) * 128);
    q.g_stride = (uint32_t)(q.rowsA / 32) * q.slab;
    q.x_stride = 2 * (kPad + q.xb + kPad);
    q.smem = 2 * (size_t)q.g_stride + kXStages * (size_t)q.x_stride + 2048 + 1024;
    if (q.smem > (size_t)kMaxSmem || q.rg + 2 > 256) continue;
    q.grid = kNumSMs;
    q.ctas_g0 = ngroups == 1 ? q.grid : (int)((int64_t)q.grid * q.tg / 9);
    q.ok = true;
    return q;
  }
  return p;
}

}  // namespace

bool conv3x3_wgrad_tc_supported(const ConvShape& s, bool three) { return plan(s, three).ok; }

int64_t conv3x3_wgrad_tc_ws_bytes(const ConvShape& s, bool three) {
  const WgPlan p = plan(s, three);
  if (!p.ok) return 0;
  return ((int64_t)p.grid * p.rowsA * p.tg * s.ci * 4 + 255) / 256 * 256 + (int64_t)p.grid * s.co * 8 + 256;
}

void conv3x3_wgrad_tc(const ConvShape& s, const float* in, const float* g, float scale, float* gw, float* gb,
                      bool three, void* ws, cudaStream_t st) {
  const WgPlan p = plan(s, three);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_wgrad_tc: unsupported shape");
  WgArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = s.w + 2;
  a.rg = p.rg;
  a.P = p.P;
  a.Pp = p.Pp;
  a.nchunks = s.ci / 32;
  a.rowsA = p.rowsA;
  a.three = three ? 1 : 0;
  a.tg = p.tg;
  a.ctas_g0 = p.ctas_g0;
  a.blocks_per_img = (s.h + p.rg - 1) / p.rg;
  a.num_blocks = s.n * a.blocks_per_img;
  a.slab = p.slab;
  a.xb = p.xb;
  a.g_stride = p.g_stride;
  a.x_stride = p.x_stride;
  a.part = static_cast<float*>(ws);
  a.part_bias = reinterpret_cast<double*>(static_cast<char*>(ws) +
                                          ((int64_t)p.grid * p.rowsA * p.tg * s.ci * 4 + 255) / 256 * 256);
  const CUtensorMap& mg = cached(g, s.n, s.h, s.w, s.co, p.rg);
  const CUtensorMap& mx = cached(in, s.n, s.h, s.w, s.ci, p.rg + 2);
  static bool configured = false;
  if (!configured) {
    RP_CUDA(cudaFuncSetAttribute(wgrad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    configured = true;
  }
  wgrad_tc_kernel<<<p.grid, kThreads, p.smem, st>>>(mg, mx, a);
  RP_LAUNCHED();
  const int total = 9 * s.ci * s.co + s.co;
  wgrad_reduce_kernel<<<ceil_div(total, 256), 256, 0, st>>>(a.part, a.part_bias, p.grid, p.ctas_g0, p.tg, s.ci,
                                                            s.co, p.rowsA, a.three, (double)scale, gw, gb);
  RP_LAUNCHED();
}

}  // namespace rp::k
