// tcgen05 weight gradient with bf16 operands and fp32 accumulation (RP_MATH_BF16):
//
//   gW[tap][ci][co] = scale * sum_p bf16(x[p + off(tap)][ci]) * bf16(g[p][co]),
//   gb[co] = scale * sum_p g[p][co]   (fp32 values, Kahan-compensated)
//
// Structure of conv_wgrad_tc.cu (positions of the padded interior frame as the GEMM K,
// taps as shifted B descriptors, TMEM accumulation over a CTA's pixel blocks, per-CTA
// partials + fixed-order fp64 reduce) re-tiled for kind::f16:
//   A = g^T  (M = 128 output channels, MN-major bf16, 128B swizzle: 64 channels per row)
//   B = x^T  (N = 128 input channels, MN-major bf16, 128B swizzle)
//   K = 16 positions per MMA; TMEM: 3 taps x 128 columns per tap group.
// TMA brings each block's fp32 g / x in 32-channel pieces (unswizzled) into a 2-slot
// staging ring; converter warps round them to bf16 (RNE) into the swizzled operand
// stage (16-byte chunk c of row r stored at c ^ (absolute row & 7)), and sum g for the
// bias.  CTAs split into (co block, ci block, tap group) work groups.
#include <cuda.h>
#include <cuda_bf16.h>

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
constexpr int kStages = 2;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kLead = 128;          // zero row before the x slabs (tap shift -1)
constexpr int kTrail = 2048;        // zero rows after them (K padding reads up to 15 rows)
constexpr int kTg = 3;              // taps per group (3 x 128 TMEM columns)
constexpr int kConvThreads = 256;   // warps 2..9
constexpr int kPiece = 64;          // channels per TMA piece (one bf16 slab row: 256-byte fp32 rows)
constexpr int kPieces = 128 / kPiece; // pieces per operand per block
constexpr int kMaxSlots = 8;        // fp32 staging ring depth (as many as shared memory allows)

struct BwArgs {
  int N, H, W, Ci, Co, Wp, rg, P, Pp;
  int mo, mi;                    // 128-channel co blocks, 128-channel ci blocks
  int blocks_per_img, num_blocks;
  uint32_t g_slab;               // bytes per 64-channel bf16 g slab (Pp rows of 128 B)
  uint32_t x_slab;               // bytes per 64-channel bf16 x slab ((rg+2)*Wp rows, packed)
  uint32_t x_off;                // offset of x slab 0 in a stage
  uint32_t stage;                // bytes per operand stage
  uint32_t piece;                // bytes per staging slot (largest fp32 piece)
  int nslots;                    // staging ring depth
  unsigned long long* trace;     // per-block timestamps (tools/trace_wgrad.py), null = off
  float* part;                   // [grid][kTg * 128 (ci)][128 (co)]
  double* part_bias;             // [grid][128]
};

__device__ __forceinline__ int grp_start(int gid, int grid, const BwArgs& a) {
  // 3 tap groups of 3 taps per (co block, ci block) pair: CTAs split evenly
  return (int)((int64_t)grid * gid / (3 * a.mo * a.mi));
}

#define BW_TRACE(slot_, b)                                                                     \
  do {                                                                                         \
    if (a.trace && blockIdx.x < 2 && (b) - blk_beg < 64)                                       \
      a.trace[(blockIdx.x * 64 + ((b) - blk_beg)) * 8 + (slot_)] = globaltimer_ns();           \
  } while (0)

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_bf16_kernel(const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_x,
                      const BwArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;

  uint8_t* stage_base = smem;                                  // kStages operand stages
  uint8_t* ring = smem + kStages * a.stage;                    // nslots fp32 staging slots
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + a.nslots * a.piece);
  uint64_t* p_full = bars;                       // [kMaxSlots] TMA -> converters (per piece)
  uint64_t* p_empty = bars + kMaxSlots;          // [kMaxSlots] converters -> TMA
  uint64_t* full = bars + 2 * kMaxSlots;         // [kStages] converters -> MMA
  uint64_t* empty = bars + 2 * kMaxSlots + 2;    // [kStages] MMA -> converters
  uint64_t* acc_full = bars + 2 * kMaxSlots + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxSlots + 5);
  double* bsum = reinterpret_cast<double*>(bars + 2 * kMaxSlots + 6);   // [8 warps][128]

  auto g_slab = [&](int s, int j) { return stage_base + s * a.stage + j * a.g_slab; };
  auto x_slab = [&](int s, int j) { return stage_base + s * a.stage + a.x_off + j * a.x_slab; };
  auto slot = [&](int r) { return ring + r * a.piece; };

  const int NG = 3 * a.mo * a.mi;
  int gid = 0;
  while (gid + 1 < NG && grp_start(gid + 1, gridDim.x, a) <= (int)blockIdx.x) ++gid;
  const int c_lo = grp_start(gid, gridDim.x, a), c_hi = grp_start(gid + 1, gridDim.x, a);
  const int gi = gid % 3, cib = (gid / 3) % a.mi, cob = gid / (3 * a.mi);
  const int jg = blockIdx.x - c_lo, ng = c_hi - c_lo;
  const int blk_beg = (int)((int64_t)jg * a.num_blocks / ng);
  const int blk_end = (int)((int64_t)(jg + 1) * a.num_blocks / ng);
  const int t0 = gi * kTg;
  const int Wp = a.Wp;
  const int xrows = (a.rg + 2) * Wp;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nslots; ++i) {
      mbar_init(&p_full[i], 1);
      mbar_init(&p_empty[i], kConvThreads);
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], kConvThreads);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tmap_g);
    prefetch_tmap(&tmap_x);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const int n16 = (int)((size_t)kStages * a.stage / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  // pieces per block: 4 g pieces (co 128 = 4 x 32) then 4 x pieces (ci 128 = 4 x 32)
  if (warp == 0) {
    // ===================== TMA producer (fp32 pieces into the staging ring) =====================
    int r = 0;
    uint32_t rph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      const int n = b / a.blocks_per_img;
      const int y0 = (b - n * a.blocks_per_img) * a.rg;
      for (int pc = 0; pc < 2 * kPieces; ++pc) {
        mbar_wait(&p_empty[r], rph ^ 1);
        if (elect_one()) {
          if (pc == 0) BW_TRACE(0, b);
          if (pc < kPieces) {
            mbar_arrive_expect_tx(&p_full[r], (uint32_t)a.P * kPiece * 4u);
            tma_load_4d(&tmap_g, &p_full[r], slot(r), 128 * cob + kPiece * pc, -1, y0, n);
          } else {
            mbar_arrive_expect_tx(&p_full[r], (uint32_t)xrows * kPiece * 4u);
            tma_load_4d(&tmap_x, &p_full[r], slot(r), 128 * cib + kPiece * (pc - kPieces), -1, y0 - 1, n);
          }
        }
        __syncwarp();
        if (++r == a.nslots) r = 0, rph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t id = idesc(1, 128, 128, 1, 1);
    const int ksteps = a.Pp / 16;
    uint64_t boff[kTg];
#pragma unroll
    for (int ti = 0; ti < kTg; ++ti) {
      const int t = t0 + ti;
      boff[ti] = (uint64_t)(int64_t)(((t / 3) * Wp + (t % 3) - 1) * 8);   // shift rows x 128 B / 16
    }
    int s = 0;
    uint32_t ph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (lane == 0) BW_TRACE(3, b);
      uint64_t da = desc_general(smem_u32(g_slab(s, 0)), a.g_slab, 1024, 2, 0);
      uint64_t db = desc_general(smem_u32(x_slab(s, 0)), a.x_slab, 1024, 2, 0);
      if (elect_one()) {
        for (int k = 0; k < ksteps; ++k) {
          const uint32_t accum = (b > blk_beg || k > 0) ? 1u : 0u;
#pragma unroll
          for (int ti = 0; ti < kTg; ++ti)
            mma_f16(tmem_base + (uint32_t)(ti * 128), da, db + boff[ti], id, accum);
          da += 128;   // 16 positions = 16 rows x 128 B, in 16-byte units
          db += 128;
        }
        mma_commit(&empty[s]);
        BW_TRACE(4, b);
      }
      __syncwarp();
      if (++s == kStages) s = 0, ph ^= 1;
    }
    if (elect_one()) mma_commit(acc_full);
    __syncwarp();
  } else {
    // ===================== converters (warps 2..9): fp32 pieces -> swizzled bf16 =====================
    // A piece is `rows` rows of 64 fp32 channels (256 B, unswizzled) = one bf16 slab row of
    // 8 16-byte chunks.  Thread t converts float4 f = t + 256 m (contiguous 16-byte loads,
    // no bank conflicts): row f / 16, channels 4 (f % 16) .. +3 -> 8 bytes of bf16 at chunk
    // (f % 16) / 2 (swizzled: chunk ^ (absolute row & 7)), half (f % 2).  f % 16 == t % 16
    // for every m, so a thread sums the same 4 g channels of each g piece for the bias.
    // 4 float4 in flight per thread (loads first).
    const int tid = threadIdx.x - 64;
    const int c4 = tid & 15, q = c4 >> 1, half = c4 & 1;
    const bool do_bias = gi == 0 && cib == 0;
    float bs[kPieces][4], bk[kPieces][4];
#pragma unroll
    for (int pc = 0; pc < kPieces; ++pc)
#pragma unroll
      for (int e = 0; e < 4; ++e) bs[pc][e] = bk[pc][e] = 0.f;
    auto convert = [&](int r, uint8_t* dst, int rows, float* bf) {
      const float4* src = reinterpret_cast<const float4*>(slot(r));
      const uint32_t dbase = smem_u32(dst);
      const int n4 = rows * 16;
      for (int f0 = tid; f0 < n4; f0 += 4 * kConvThreads) {
        float4 u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int f = f0 + k * kConvThreads;
          u[k] = f < n4 ? src[f] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int f = f0 + k * kConvThreads;
          if (f < n4) {
            const int row = f >> 4;
            const uint32_t raddr = dbase + (uint32_t)row * 128u;
            const int phys = q ^ (int)((raddr >> 7) & 7u);
            *reinterpret_cast<uint2*>(dst + (size_t)row * 128 + phys * 16 + half * 8) =
                make_uint2(pack_bf16(u[k].x, u[k].y), pack_bf16(u[k].z, u[k].w));
          }
          if (bf) {
            bf[0] += u[k].x; bf[1] += u[k].y; bf[2] += u[k].z; bf[3] += u[k].w;
          }
        }
      }
    };
    int r = 0, s = 0;
    uint32_t rph = 0, ph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      mbar_wait(&empty[s], ph ^ 1);
      if (tid == 0) BW_TRACE(1, b);
      long long wt = 0;
#pragma unroll
      for (int pc = 0; pc < kPieces; ++pc) {                     // g pieces: co 64 pc .. 64 pc + 63
        long long t0w = a.trace ? clock64() : 0;
        mbar_wait(&p_full[r], rph);
        if (a.trace) wt += clock64() - t0w;
        if (tid == 0 && pc == 0) BW_TRACE(5, b);
        float bf[4] = {0, 0, 0, 0};
        convert(r, g_slab(s, pc), a.P, do_bias ? bf : nullptr);
        if (do_bias) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {                          // Kahan fold of the block sum
            const float y = bf[e] - bk[pc][e];
            const float t = bs[pc][e] + y;
            bk[pc][e] = (t - bs[pc][e]) - y;
            bs[pc][e] = t;
          }
        }
        mbar_arrive(&p_empty[r]);                                // slot read: TMA may refill it
        if (++r == a.nslots) r = 0, rph ^= 1;
      }
      for (int pc = 0; pc < kPieces; ++pc) {                     // x pieces: ci 64 pc .. 64 pc + 63
        long long t0w = a.trace ? clock64() : 0;
        mbar_wait(&p_full[r], rph);
        if (a.trace) wt += clock64() - t0w;
        convert(r, x_slab(s, pc), xrows, nullptr);
        mbar_arrive(&p_empty[r]);
        if (++r == a.nslots) r = 0, rph ^= 1;
      }
      fence_proxy_async_smem();                                  // bf16 stage -> tensor core (async proxy)
      if (tid == 0) BW_TRACE(2, b);
      if (tid == 0 && a.trace && blockIdx.x < 2 && b - blk_beg < 64)
        a.trace[(blockIdx.x * 64 + (b - blk_beg)) * 8 + 6] = (unsigned long long)wt;
      mbar_arrive(&full[s]);
      if (++s == kStages) s = 0, ph ^= 1;
    }
    if (do_bias) {
      // lanes sharing c4 = lane & 15 combine in fixed order (xor 16), lanes 0..15 publish
      // the warp's 128 channel sums, warps are summed in order by 128 threads
      const int cw = tid / 32;
#pragma unroll
      for (int pc = 0; pc < kPieces; ++pc) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          double d = (double)bs[pc][e] - (double)bk[pc][e];
          d += __shfl_xor_sync(0xffffffffu, d, 16);
          if (lane < 16) bsum[cw * 128 + pc * 64 + 4 * c4 + e] = d;
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid < 128) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += bsum[w * 128 + tid];
        a.part_bias[(size_t)blockIdx.x * 128 + tid] = t;
      }
    }
  }

  // epilogue (warps 6..9 after the converters are done): D[co][ci] per tap -> partial
  if (warp >= 6) {
    const int q = warp & 3;
    const int co = q * 32 + lane;
    float* dst = a.part + (size_t)blockIdx.x * kTg * 128 * 128;
    const bool any = blk_end > blk_beg;
    if (any) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
    const int ntaps = min(kTg, 9 - t0);
    for (int ti = 0; ti < ntaps; ++ti) {
      for (int c = 0; c < 128; c += 16) {
        uint32_t rr[16];
        tmem_ld16(trow + (uint32_t)(ti * 128 + c), rr);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          dst[(size_t)(ti * 128 + c + e) * 128 + co] = any ? __uint_as_float(rr[e]) : 0.f;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// gW[tap][ci][co] = scale * sum over the work group's CTAs of part[cta][ti * 128 + ci'][co']
__global__ void wgrad_bf16_reduce_kernel(const float* __restrict__ part, const double* __restrict__ part_bias,
                                         const BwArgs a, int grid, double scale, float* __restrict__ gw,
                                         float* __restrict__ gb) {
  const int Ci = a.Ci, Co = a.Co;
  const int total = 9 * Ci * Co;
  const int64_t pstride = (int64_t)kTg * 128 * 128;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total + Co; idx += gridDim.x * blockDim.x) {
    if (idx < total) {
      const int co = idx % Co;
      const int ci = (idx / Co) % Ci;
      const int tap = idx / (Co * Ci);
      const int gi = tap / kTg, cob = co / 128, cib = ci / 128;
      const int gid = (cob * a.mi + cib) * 3 + gi;
      const int c_lo = grp_start(gid, grid, a), c_hi = grp_start(gid + 1, grid, a);
      const int64_t off = ((int64_t)(tap - gi * kTg) * 128 + (ci - cib * 128)) * 128 + (co - cob * 128);
      double s = 0.0;
      for (int b = c_lo; b < c_hi; ++b) s += (double)part[b * pstride + off];
      gw[idx] = (float)(scale * s);
    } else if (gb) {
      const int co = idx - total, cob = co / 128;
      const int gid = cob * a.mi * 3;
      const int c_lo = grp_start(gid, grid, a), c_hi = grp_start(gid + 1, grid, a);
      double s = 0.0;
      for (int b = c_lo; b < c_hi; ++b) s += part_bias[(int64_t)b * 128 + (co - cob * 128)];
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

// NHWC fp32 as (C, W, H, N); box = 32 channels x (W+2) columns (from x = -1) x rows, no swizzle
CUtensorMap make_map(const float* t, int n, int h, int w, int c, int rows) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)c * 4, (cuuint64_t)w * c * 4, (cuuint64_t)h * w * c * 4};
  const cuuint32_t box[4] = {(cuuint32_t)kPiece, (cuuint32_t)(w + 2), (cuuint32_t)rows, 1};   // 256 B rows
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(t), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 wgrad) failed (" + std::to_string((int)r) + ")");
  return m;
}

std::mutex g_mu;
std::map<std::tuple<const void*, int, int, int, int, int>, CUtensorMap> g_maps;

CUtensorMap cached(const float* t, int n, int h, int w, int c, int rows) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple((const void*)t, n, h, w, c, rows);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();   // callers hold copies, never references
    it = g_maps.emplace(key, make_map(t, n, h, w, c, rows)).first;
  }
  return it->second;
}

uint32_t round1k(uint64_t v) { return (uint32_t)((v + 1023) / 1024 * 1024); }

struct BwPlan {
  bool ok = false;
  int rg, P, Pp, grid, nslots;
  uint32_t g_slab, x_slab, x_off, stage, piece;
  size_t smem;
};

BwPlan plan(const ConvShape& s) {
  BwPlan p;
  if (s.co % 128 != 0 || s.ci % 128 != 0 || s.w + 2 > 256) return p;
  if (3 * (s.co / 128) * (s.ci / 128) > kNumSMs) return p;
  const int Wp = s.w + 2;
  for (int rg = std::min(s.h, 6); rg >= 1; --rg) {
    BwPlan q = p;
    q.rg = rg;
    q.P = rg * Wp;
    q.Pp = (q.P + 15) / 16 * 16;
    q.g_slab = round1k((uint64_t)q.Pp * 128);
    q.x_slab = (uint32_t)(rg + 2) * Wp * 128u;
    q.x_off = 2 * q.g_slab + kLead;
    q.stage = round1k((uint64_t)q.x_off + 2ull * q.x_slab + kTrail);
    q.piece = round1k((uint64_t)std::max(q.P, (rg + 2) * Wp) * kPiece * 4);
    const size_t fixed = kStages * (size_t)q.stage + (2 * kMaxSlots + 8) * 8 + 8 * 128 * 8 + 256;
    if (fixed + 2 * (size_t)q.piece > (size_t)kMaxSmem) continue;
    q.nslots = (int)std::min<size_t>(kMaxSlots, ((size_t)kMaxSmem - fixed) / q.piece);
    if (q.nslots < 3 && rg > 2) continue;   // prefer a smaller block with a deeper TMA ring
    q.smem = fixed + (size_t)q.nslots * q.piece;
    if ((size_t)kTg * 128 * 128 * 4 > 0 && q.Pp - q.P > 15) continue;
    q.grid = kNumSMs;
    q.ok = true;
    return q;
  }
  return p;
}

int64_t part_bytes(const BwPlan& p) { return ((int64_t)p.grid * kTg * 128 * 128 * 4 + 255) / 256 * 256; }

}  // namespace

unsigned long long* g_bw_trace = nullptr;
void conv3x3_wgrad_bf16_set_trace(unsigned long long* p) { g_bw_trace = p; }

bool conv3x3_wgrad_bf16_supported(const ConvShape& s) { return plan(s).ok; }

int64_t conv3x3_wgrad_bf16_ws_bytes(const ConvShape& s) {
  const BwPlan p = plan(s);
  if (!p.ok) return 0;
  return part_bytes(p) + (int64_t)p.grid * 128 * 8 + 256;
}

void conv3x3_wgrad_bf16(const ConvShape& s, const float* in, const float* g, float scale, float* gw, float* gb,
                        void* ws, cudaStream_t st) {
  const BwPlan p = plan(s);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_wgrad_bf16: unsupported shape");
  BwArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = s.w + 2;
  a.rg = p.rg;
  a.P = p.P;
  a.Pp = p.Pp;
  a.mo = s.co / 128;
  a.mi = s.ci / 128;
  a.blocks_per_img = (s.h + p.rg - 1) / p.rg;
  a.num_blocks = s.n * a.blocks_per_img;
  a.g_slab = p.g_slab;
  a.x_slab = p.x_slab;
  a.x_off = p.x_off;
  a.stage = p.stage;
  a.piece = p.piece;
  a.nslots = p.nslots;
  a.trace = g_bw_trace;
  a.part = static_cast<float*>(ws);
  a.part_bias = reinterpret_cast<double*>(static_cast<char*>(ws) + part_bytes(p));
  const CUtensorMap mg = cached(g, s.n, s.h, s.w, s.co, p.rg);
  const CUtensorMap mx = cached(in, s.n, s.h, s.w, s.ci, p.rg + 2);
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(wgrad_bf16_kernel), kMaxSmem);
  wgrad_bf16_kernel<<<p.grid, kThreads, p.smem, st>>>(mg, mx, a);
  RP_LAUNCHED();
  const int total = 9 * s.ci * s.co + s.co;
  wgrad_bf16_reduce_kernel<<<ceil_div(total, 256), 256, 0, st>>>(a.part, a.part_bias, a, p.grid, (double)scale, gw,
                                                                 gb);
  RP_LAUNCHED();
}

}  // namespace rp::k
