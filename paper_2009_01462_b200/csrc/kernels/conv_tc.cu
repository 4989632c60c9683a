// tcgen05 implicit-GEMM 3x3 convolution (fprop and dgrad), NHWC fp32, sm_100a.
//
//   out[p][co] = epi( sum_{tap, ci} in[p + off(tap)][ci] * w[tap][ci][co] )
//
// (block_forward's matmul(x, W1) / matmul(a, W2) and block_vjp's matmul(upstream,
// W2^T) / matmul(dpre, W1^T), network.cpp:85-104, generalised to 3x3 taps.)
//
// Design:
//  * M = output positions in the zero-padded "interior frame" of one image (H rows x
//    (W+2) columns, flattened): tap (dy,dx) is then a constant shift of
//    dy*(W+2)+dx positions, so one halo slab per 16-channel chunk, loaded once by TMA
//    (out-of-bounds rows/columns zero-filled by the TMA unit), serves all 9 taps as 9
//    shifted UMMA descriptors.  The 2 padding columns per row are computed and
//    discarded (6% of the MMA work at W = 32).
//  * operands are K-major "interleaved" (no swizzle): for each group of 4 channels
//    every position is 16 contiguous bytes, so a shift by one position is +16 B of
//    descriptor start address.  The TMA box is (4 ch, W+2, rows, 4 kgroups, 1) over a
//    5-D view of NHWC whose 4th dim is the channel group (stride 16 B).
//  * a unit = S consecutive 128-position tiles sharing one weight pass (S
//    accumulators of 128 x Co fp32 in TMEM, double-buffered across units).
//  * fp32 accuracy with tensor cores: 3xTF32.  Each operand v = hi + lo with
//    hi = rna_tf32(v) and lo = v - hi (exact); D += Ahi Bhi + Ahi Blo + Alo Bhi.
//    Weights are split once per call into global memory; the activation halo is split
//    in shared memory by 4 converter warps.  RP_MATH_TF32 issues only Ahi Bhi.
//  * warp roles (320 threads, persistent, 1 CTA/SM): w0 TMA producer, w1 MMA issuer
//    (one thread), w2-5 converters, w6-9 epilogue (TMEM -> registers -> fused
//    bias / tanh / skip / step-size -> global).
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
constexpr int kWStages = 4;
constexpr int kChunk = 16;           // input channels per halo chunk
constexpr int kMaxSmem = 220 * 1024;

struct TcArgs {
  int N, H, W, Ci, Co, Wp, rows_h, S, units_per_img, num_units, halo_pos, nchunks;
  uint32_t halo_bytes;  // one raw (or lo) halo buffer
  uint32_t w_bytes;     // one hi (or lo) weight stage
  uint32_t halo_stride; // bytes per halo stage slot (raw + lo + pads)
  int three;            // 1: 3xTF32, 0: plain TF32
  int epi;
  float h;
  const float* w_hi;    // [tap][chunk][kg][co][4]
  const float* w_lo;
  const float* bias;
  const float* aux;
  float* out;
};

__device__ __forceinline__ float rna_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

template <int EPI>
__device__ __forceinline__ float epi_value(float acc, int co, int64_t idx, const TcArgs& a) {
  if constexpr (EPI == EPI_BIAS) return acc + __ldg(a.bias + co);
  if constexpr (EPI == EPI_BIAS_TANH) return tanhf(acc + __ldg(a.bias + co));
  if constexpr (EPI == EPI_RESID) return __ldg(a.aux + idx) + a.h * (acc + __ldg(a.bias + co));
  if constexpr (EPI == EPI_TANH_BWD) {
    const float t = __ldg(a.aux + idx);
    return (a.h * acc) * (1.f - t * t);
  }
  if constexpr (EPI == EPI_ADD) return a.aux[idx] + acc;
  return a.h * acc;
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tmap, const TcArgs a, int tmem_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- shared memory carve-up
  uint8_t* halo_base = smem;                                      // 2 slots
  uint8_t* w_base = smem + 2 * a.halo_stride;                     // kWStages x (hi, lo)
  uint64_t* bars = reinterpret_cast<uint64_t*>(w_base + kWStages * 2 * a.w_bytes);
  uint64_t* halo_full = bars;        // [2]
  uint64_t* halo_conv = bars + 2;    // [2]
  uint64_t* halo_empty = bars + 4;   // [2]
  uint64_t* w_full = bars + 6;       // [kWStages]
  uint64_t* w_empty = bars + 6 + kWStages;
  uint64_t* acc_full = bars + 6 + 2 * kWStages;   // [2]
  uint64_t* acc_empty = bars + 8 + 2 * kWStages;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10 + 2 * kWStages);

  auto halo_raw = [&](int s) { return halo_base + s * a.halo_stride + 128; };
  auto halo_lo = [&](int s) { return halo_base + s * a.halo_stride + 128 + a.halo_bytes + 128; };
  auto w_hi_s = [&](int s) { return w_base + s * 2 * a.w_bytes; };
  auto w_lo_s = [&](int s) { return w_base + s * 2 * a.w_bytes + a.w_bytes; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&halo_full[i], 1);
      mbar_init(&halo_conv[i], 128);
      mbar_init(&halo_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    for (int i = 0; i < kWStages; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);  // column count fixed at the max; see host
  // zero the 128-byte pads around the halo buffers (read only by discarded rows)
  for (int i = threadIdx.x; i < 2 * 3 * 32; i += blockDim.x) {
    const int s = i / 96, part = (i / 32) % 3, w = i % 32;
    uint8_t* base = halo_base + s * a.halo_stride +
                    (part == 0 ? 0 : part == 1 ? 128 + a.halo_bytes : 256 + 2 * a.halo_bytes);
    reinterpret_cast<uint32_t*>(base)[w] = 0u;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  (void)tmem_cols;

  const int Wp = a.Wp;
  const uint32_t kg_stride_a = (uint32_t)a.halo_pos * 16u;     // bytes between channel groups (halo)
  const uint32_t kg_stride_b = (uint32_t)a.Co * 16u;           // bytes between channel groups (weights)

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int hs = 0, ws = 0;
      uint32_t hph = 0, wph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        const int n = u / a.units_per_img;
        const int f0 = (u % a.units_per_img) * a.S * 128;
        const int y0 = f0 / Wp;
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&halo_empty[hs], hph ^ 1);
          mbar_arrive_expect_tx(&halo_full[hs], a.halo_bytes);
          tma_load_5d(&tmap, &halo_full[hs], halo_raw(hs), 0, -1, y0 - 1, 4 * c, n);
          if (++hs == 2) hs = 0, hph ^= 1;
          for (int t = 0; t < 9; ++t) {
            mbar_wait(&w_empty[ws], wph ^ 1);
            mbar_arrive_expect_tx(&w_full[ws], a.three ? 2 * a.w_bytes : a.w_bytes);
            const int64_t off = ((int64_t)t * a.nchunks + c) * (a.w_bytes / 4);
            bulk_load(w_hi_s(ws), a.w_hi + off, a.w_bytes, &w_full[ws]);
            if (a.three) bulk_load(w_lo_s(ws), a.w_lo + off, a.w_bytes, &w_full[ws]);
            if (++ws == kWStages) ws = 0, wph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t id = idesc(2, 128, a.Co);
      int hs = 0, ws = 0, ab = 0;
      uint32_t hph = 0, wph = 0, aph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        const int f0 = (u % a.units_per_img) * a.S * 128;
        const int c0 = f0 % Wp;
        mbar_wait(&acc_empty[ab], aph ^ 1);
        tc_fence_after();
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(a.three ? &halo_conv[hs] : &halo_full[hs], hph);
          tc_fence_after();
          const uint32_t raw = smem_u32(halo_raw(hs));
          const uint32_t lo = smem_u32(halo_lo(hs));
          for (int t = 0; t < 9; ++t) {
            mbar_wait(&w_full[ws], wph);
            tc_fence_after();
            const int shift = c0 + (t / 3) * Wp + (t % 3) - 1;
            const uint32_t bh = smem_u32(w_hi_s(ws));
            const uint32_t bl = smem_u32(w_lo_s(ws));
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint64_t db_hi = desc_kmajor_interleave(bh + 2 * j * kg_stride_b, kg_stride_b, 128);
              const uint64_t db_lo = desc_kmajor_interleave(bl + 2 * j * kg_stride_b, kg_stride_b, 128);
              for (int s = 0; s < a.S; ++s) {
                const uint32_t pos = (uint32_t)(shift + s * 128);
                const uint32_t aoff = 2 * j * kg_stride_a + pos * 16u;
                const uint64_t da_hi = desc_kmajor_interleave(raw + aoff, kg_stride_a, 128);
                const uint32_t d = tmem_base + (uint32_t)((ab * a.S + s) * a.Co);
                const uint32_t accum = (c | t | j) ? 1u : 0u;
                mma_tf32(d, da_hi, db_hi, id, accum);
                if (a.three) {
                  const uint64_t da_lo = desc_kmajor_interleave(lo + aoff, kg_stride_a, 128);
                  mma_tf32(d, da_hi, db_lo, id, 1u);
                  mma_tf32(d, da_lo, db_hi, id, 1u);
                }
              }
            }
            mma_commit(&w_empty[ws]);
            if (++ws == kWStages) ws = 0, wph ^= 1;
          }
          mma_commit(&halo_empty[hs]);
          if (++hs == 2) hs = 0, hph ^= 1;
        }
        mma_commit(&acc_full[ab]);
        if (++ab == 2) ab = 0, aph ^= 1;
      }
    }
  } else if (warp < 6) {
    // ===================== converters (3xTF32 split of the halo) =====================
    if (a.three) {
      const int tid = threadIdx.x - 64;
      int hs = 0;
      uint32_t hph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&halo_full[hs], hph);
          float4* raw = reinterpret_cast<float4*>(halo_raw(hs));
          float4* lo = reinterpret_cast<float4*>(halo_lo(hs));
          const int n16 = (int)(a.halo_bytes / 16);
          for (int i = tid; i < n16; i += 128) {
            float4 v = raw[i];
            float4 hi, l;
            hi.x = rna_tf32(v.x); hi.y = rna_tf32(v.y); hi.z = rna_tf32(v.z); hi.w = rna_tf32(v.w);
            l.x = v.x - hi.x; l.y = v.y - hi.y; l.z = v.z - hi.z; l.w = v.w - hi.w;
            raw[i] = hi;
            lo[i] = l;
          }
          fence_proxy_async_smem();
          mbar_arrive(&halo_conv[hs]);
          if (++hs == 2) hs = 0, hph ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue =====================
    const int q = warp & 3;         // TMEM lane quadrant this warp may access
    const int m = q * 32 + lane;    // accumulator row == position within the tile
    int ab = 0;
    uint32_t aph = 0;
    for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
      const int n = u / a.units_per_img;
      const int f0 = (u % a.units_per_img) * a.S * 128;
      mbar_wait(&acc_full[ab], aph);
      tc_fence_after();
      for (int s = 0; s < a.S; ++s) {
        const int f = f0 + s * 128 + m;
        const int y = f / Wp, X = f - (f / Wp) * Wp;
        const bool valid = y < a.H && X >= 1 && X <= a.W;
        const int64_t base = valid ? ((((int64_t)n * a.H + y) * a.W) + (X - 1)) * a.Co : 0;
        for (int cc = 0; cc < a.Co; cc += 16) {
          uint32_t r[16];
          tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * a.S + s) * a.Co + cc), r);
          tmem_wait_ld();
          if (valid) {
            float4* dst = reinterpret_cast<float4*>(a.out + base + cc);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float4 o;
              o.x = epi_value<EPI>(__uint_as_float(r[4 * v + 0]), cc + 4 * v + 0, base + cc + 4 * v + 0, a);
              o.y = epi_value<EPI>(__uint_as_float(r[4 * v + 1]), cc + 4 * v + 1, base + cc + 4 * v + 1, a);
              o.z = epi_value<EPI>(__uint_as_float(r[4 * v + 2]), cc + 4 * v + 2, base + cc + 4 * v + 2, a);
              o.w = epi_value<EPI>(__uint_as_float(r[4 * v + 3]), cc + 4 * v + 3, base + cc + 4 * v + 3, a);
              dst[v] = o;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
      if (++ab == 2) ab = 0, aph ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// weights HWIO src[tap][ci][co] -> prepped [tap'][chunk][kg][co'][4] (hi, lo) for an
// fprop (flip = 0: ci' = ci, co' = co) or dgrad (flip = 1: tap' = 8 - tap, ci' = co, co' = ci)
__global__ void prep_weights_kernel(const float* __restrict__ w, int ci_src, int co_src, int flip, int three,
                                    float* __restrict__ hi, float* __restrict__ lo) {
  const int Ci = flip ? co_src : ci_src;
  const int Co = flip ? ci_src : co_src;
  const int nchunks = Ci / kChunk;
  const int total = 9 * Ci * Co;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int e = idx & 3;
    const int co = (idx >> 2) % Co;
    const int rest = (idx >> 2) / Co;        // (tap, chunk, kg)
    const int kg = rest % 4;
    const int chunk = (rest / 4) % nchunks;
    const int tap = rest / (4 * nchunks);
    const int ci = chunk * kChunk + kg * 4 + e;
    float v;
    if (!flip)
      v = w[((int64_t)tap * ci_src + ci) * co_src + co];
    else
      v = w[((int64_t)(8 - tap) * ci_src + co) * co_src + ci];
    if (three) {
      const float h = rna_tf32(v);
      hi[idx] = h;
      lo[idx] = v - h;
    } else {
      hi[idx] = v;
    }
  }
}

// ---------------------------------------------------------------- host side
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

CUtensorMap make_halo_map(const float* in, const ConvShape& s, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {4, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)(s.ci / 4), (cuuint64_t)s.n};
  const cuuint64_t strides[4] = {(cuuint64_t)s.ci * 4, (cuuint64_t)s.w * s.ci * 4, 16,
                                 (cuuint64_t)s.h * s.w * s.ci * 4};
  const cuuint32_t box[5] = {4, (cuuint32_t)Wp, (cuuint32_t)rows_h, 4, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

struct Plan {
  int S, Wp, rows_h, halo_pos, T, units_per_img;
  uint32_t halo_bytes, w_bytes, halo_stride;
  size_t smem;
};

Plan plan_for(const ConvShape& s) {
  Plan best{};
  double best_eff = -1.0;
  for (int S = 4; S >= 1; --S) {
    if (2 * S * s.co > 512) continue;
    Plan p{};
    p.S = S;
    p.Wp = s.w + 2;
    p.rows_h = (3 * p.Wp + 128 * S + p.Wp - 1) / p.Wp;
    p.halo_pos = p.rows_h * p.Wp;
    p.T = (s.h * p.Wp + 127) / 128;
    p.units_per_img = (p.T + S - 1) / S;
    p.halo_bytes = (uint32_t)p.halo_pos * 64u;
    p.w_bytes = (uint32_t)s.co * kChunk * 4u;
    p.halo_stride = (128 + p.halo_bytes + 128 + p.halo_bytes + 128 + 1023) / 1024 * 1024;
    p.smem = 2 * (size_t)p.halo_stride + kWStages * 2 * (size_t)p.w_bytes + 256 + 1024;
    if (p.smem > (size_t)kMaxSmem || p.rows_h > 256) continue;
    const double eff = (double)p.T / (double)(p.units_per_img * S);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = p;
    }
  }
  return best;
}

std::mutex g_map_mu;
std::map<std::tuple<const void*, int, int, int, int, int>, CUtensorMap> g_maps;

const CUtensorMap& cached_map(const float* in, const ConvShape& s, int Wp, int rows_h) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto key = std::make_tuple((const void*)in, s.n, s.h, s.w, s.ci, rows_h);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();
    it = g_maps.emplace(key, make_halo_map(in, s, Wp, rows_h)).first;
  }
  return it->second;
}

template <int EPI>
void launch_epi(const CUtensorMap& m, const TcArgs& a, size_t smem, int grid, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    RP_CUDA(cudaFuncSetAttribute(conv3x3_tc_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    configured = true;
  }
  conv3x3_tc_kernel<EPI><<<grid, kThreads, smem, st>>>(m, a, 512);
}

}  // namespace

bool conv3x3_tc_supported(const ConvShape& s) {
  if (s.ci % kChunk != 0 || s.co % 16 != 0 || s.co > 256 || s.co < 16) return false;
  if (s.w + 2 > 256) return false;
  return plan_for(s).S > 0;
}

int64_t conv3x3_tc_ws_bytes(const ConvShape& s) { return 2 * (9LL * s.ci * s.co * 4 + 256); }

void conv3x3_fwd_tc(const ConvShape& s, const float* in, const float* w_hwio, bool dgrad_weights, const float* bias,
                    const float* aux, float h, int epi, float* out, bool three, void* ws, cudaStream_t st) {
  if (s.pixels() == 0) return;
  const Plan p = plan_for(s);
  if (p.S == 0) fail(RP_ERR_INTERNAL, "conv3x3_fwd_tc: unsupported shape");
  float* w_hi = static_cast<float*>(ws);
  float* w_lo = w_hi + (9LL * s.ci * s.co + 63) / 64 * 64;
  // the weight tensor handed in is HWIO of the *forward* conv; for dgrad it has
  // (ci_src, co_src) = (s.co, s.ci)
  const int ci_src = dgrad_weights ? s.co : s.ci;
  const int co_src = dgrad_weights ? s.ci : s.co;
  const int total = 9 * s.ci * s.co;
  prep_weights_kernel<<<ceil_div(total, 256), 256, 0, st>>>(w_hwio, ci_src, co_src, dgrad_weights ? 1 : 0,
                                                             three ? 1 : 0, w_hi, w_lo);
  RP_LAUNCHED();
  TcArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = p.Wp;
  a.rows_h = p.rows_h;
  a.S = p.S;
  a.units_per_img = p.units_per_img;
  a.num_units = s.n * p.units_per_img;
  a.halo_pos = p.halo_pos;
  a.nchunks = s.ci / kChunk;
  a.halo_bytes = p.halo_bytes;
  a.w_bytes = p.w_bytes;
  a.halo_stride = p.halo_stride;
  a.three = three ? 1 : 0;
  a.epi = epi;
  a.h = h;
  a.w_hi = w_hi;
  a.w_lo = w_lo;
  a.bias = bias;
  a.aux = aux;
  a.out = out;
  const CUtensorMap& m = cached_map(in, s, p.Wp, p.rows_h);
  const int grid = std::min(a.num_units, kNumSMs);
  switch (epi) {
    case EPI_BIAS: launch_epi<EPI_BIAS>(m, a, p.smem, grid, st); break;
    case EPI_BIAS_TANH: launch_epi<EPI_BIAS_TANH>(m, a, p.smem, grid, st); break;
    case EPI_RESID: launch_epi<EPI_RESID>(m, a, p.smem, grid, st); break;
    case EPI_TANH_BWD: launch_epi<EPI_TANH_BWD>(m, a, p.smem, grid, st); break;
    case EPI_ADD: launch_epi<EPI_ADD>(m, a, p.smem, grid, st); break;
    default: launch_epi<EPI_SCALE>(m, a, p.smem, grid, st); break;
  }
  RP_LAUNCHED();
}

}  // namespace rp::k
