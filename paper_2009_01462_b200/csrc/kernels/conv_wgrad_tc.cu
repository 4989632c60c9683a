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
// 3xTF32 by stacking both operands (the tensor core truncates fp32 to tf32, so the raw
// tile is the hi part and only lo = v - trunc(v) is written):
//   A = [g_hi ; g_lo]   (M = 2 Co = 128: four 32-channel slabs at a uniform stride)
//   B = [x_hi ; x_lo]   (N = 2 Ci: 2 Ci / 32 slabs at a uniform stride)
// so ONE M=128 x N=2Ci x K=8 MMA per (k-step, tap) yields all four products in the
// four quadrants of D; the epilogue adds the quadrants.  The tap loop is innermost, so
// consecutive MMAs share A (the tensor core then runs at full rate, umma_bench).
// TMEM holds 512 fp32 columns = 512 / (2 Ci) taps, so the 9 taps are split into tap
// groups (Ci = 64: 3 groups of 3 taps) and the persistent CTAs (1/SM) into matching CTA
// groups; each CTA accumulates a contiguous range of pixel blocks in TMEM and writes one
// fp32 partial [tap ci][co]; a fixed-order fp64 reduce combines them (deterministic).
// RP_MATH_TF32 skips the lo writes (the lo slabs stay zero).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
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
constexpr int kMaxStages = 4;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kLead = 128;          // zero row in front of the x slabs (tap shift -1)
constexpr int kTrail = 1024;        // zero rows behind them (K padding reads)
constexpr int kMaxTaps = 5;         // taps per group (Ci = 32: 5 + 4)
constexpr int kConvThreads = 256;   // warps 2..9 split the lo parts / bias sums

struct WgArgs {
  int N, H, W, Ci, Co, Wp, rg, P, Pp, three, nstages;
  int CiB;                       // input channels per ci block (Ci == 32: 32, else 64)
  int mo, mi;                    // 64-channel co blocks, CiB-channel ci blocks
  int n2;                        // B columns per tap (2 CiB)
  int tg, ngroups;               // taps per tap group (the last may hold fewer), tap groups
  int blocks_per_img, num_blocks;
  uint32_t g_slab;               // bytes per 32-channel g slab (Pp rows of 128 B; rows >= P stay 0)
  uint32_t x_slab;               // bytes per x slab ((rg+2)*Wp rows of 128 B, packed)
  uint32_t x_off;                // byte offset of x slab 0 in a stage
  uint32_t stage;                // bytes per stage
  float* part;                   // [grid][tg * Ci][Co]
  double* part_bias;             // [grid][Co]
  unsigned long long* trace;     // diagnostics (tools/trace_wgrad.py), null = off
};

// per-block timestamps of CTAs 0/1, first 64 blocks: [0] TMA issue, [1] converters see the
// data, [2] converters done, [3] MMA warp starts the block, [4] block's MMAs issued
#define WG_TRACE(slot, b)                                                                      \
  do {                                                                                         \
    if (a.trace && blockIdx.x < 2 && (b) - blk_beg < 64)                                       \
      a.trace[(blockIdx.x * 64 + ((b) - blk_beg)) * 8 + (slot)] = globaltimer_ns();            \
  } while (0)

// Work groups gid = ((cob * mi + cib) * ngroups + gi) get CTAs in proportion to their
// taps: group gid owns CTAs [grp_start(gid), grp_start(gid + 1)) of a `grid`-CTA launch.
__device__ __forceinline__ int grp_start(int gid, int grid, const WgArgs& a) {
  const int pair = gid / a.ngroups, gi = gid - pair * a.ngroups;
  const int taps = pair * 9 + min(9, gi * a.tg);
  return (int)((int64_t)grid * taps / (9 * a.mo * a.mi));
}

__device__ __forceinline__ float trunc_tf32(float v) { return __uint_as_float(__float_as_uint(v) & 0xffffe000u); }

__device__ __forceinline__ float4 lo_part(float4 v) {
  return make_float4(v.x - trunc_tf32(v.x), v.y - trunc_tf32(v.y), v.z - trunc_tf32(v.z), v.w - trunc_tf32(v.w));
}

// Shared-memory stage: [g_hi 0..1 | g_lo 0..1] (Pp rows each, 1 KB aligned) then a
// 128-byte zero row, the x slabs [x_hi 0..nx-1 | x_lo 0..nx-1] packed back to back (a tap
// shift reads at most one row before / seven rows after a slab; those positions meet
// g == 0, so the neighbour slab's finite data is harmless) and a 1 KB zero tail.  TMA
// and UMMA apply the 128B swizzle on absolute address bits, so the x slabs need only
// 128-byte alignment.
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_x,
                    const WgArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);   // warp-uniform role index
  const int lane = threadIdx.x & 31;
  const int nx = a.CiB / 32;                      // x_hi slabs (as many x_lo slabs follow)
  const int S = a.nstages;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * a.stage);
  uint64_t* full = bars;                       // [S]
  uint64_t* conv = bars + kMaxStages;
  uint64_t* empty = bars + 2 * kMaxStages;
  uint64_t* acc_full = bars + 3 * kMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStages + 1);
  double* bsum = reinterpret_cast<double*>(bars + 3 * kMaxStages + 2);   // [8 warps][64]

  auto g_slab = [&](int s, int j) { return smem + s * a.stage + j * a.g_slab; };
  auto x_slab = [&](int s, int j) { return smem + s * a.stage + a.x_off + j * a.x_slab; };

  // CTA -> (tap group, contiguous block range)
  const int NG = a.mo * a.mi * a.ngroups;
  int gid = 0;
  while (gid + 1 < NG && grp_start(gid + 1, gridDim.x, a) <= (int)blockIdx.x) ++gid;
  const int c_lo = grp_start(gid, gridDim.x, a), c_hi = grp_start(gid + 1, gridDim.x, a);
  const int gi = gid % a.ngroups;
  const int cib = (gid / a.ngroups) % a.mi, cob = gid / (a.ngroups * a.mi);
  const int jg = blockIdx.x - c_lo;
  const int ng = c_hi - c_lo;
  const int blk_beg = (int)((int64_t)jg * a.num_blocks / ng);
  const int blk_end = (int)((int64_t)(jg + 1) * a.num_blocks / ng);
  const int t0 = gi * a.tg;
  const int ntaps = min(a.tg, 9 - t0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], kConvThreads);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
    prefetch_tmap(&tmap_g);
    prefetch_tmap(&tmap_x);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  // Zero the stages once: pads, g rows P..Pp-1 and (TF32) the lo slabs are read by the
  // MMA but never written.
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const int n16 = (int)((size_t)S * a.stage / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int Wp = a.Wp;
  const uint32_t xrows = (uint32_t)(a.rg + 2) * Wp;

  if (warp == 0) {
    // ===================== TMA producer =====================
    int s = 0;
    uint32_t ph = 0;
    const uint32_t bytes = 2u * a.P * 128u + (uint32_t)nx * xrows * 128u;
    for (int b = blk_beg; b < blk_end; ++b) {
      const int n = b / a.blocks_per_img;
      const int y0 = (b - n * a.blocks_per_img) * a.rg;
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        WG_TRACE(0, b);
        mbar_arrive_expect_tx(&full[s], bytes);
        for (int j = 0; j < 2; ++j) tma_load_4d(&tmap_g, &full[s], g_slab(s, j), 64 * cob + 32 * j, -1, y0, n);
        for (int j = 0; j < nx; ++j)
          tma_load_4d(&tmap_x, &full[s], x_slab(s, j), a.CiB * cib + 32 * j, -1, y0 - 1, n);
      }
      __syncwarp();
      if (++s == S) s = 0, ph ^= 1;
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // All offsets precomputed: the issue loop is descriptor adds + UTCHMMA only.
    const uint32_t id = idesc(2, 128, a.n2, 1, 1);
    const int ksteps = a.Pp / 8;
    uint64_t boff[kMaxTaps];
    uint32_t dcol[kMaxTaps];
#pragma unroll
    for (int ti = 0; ti < kMaxTaps; ++ti) {
      const int t = min(t0 + ti, 8);
      boff[ti] = (uint64_t)(int64_t)(((t / 3) * Wp + (t % 3) - 1) * 8);   // shift rows x 128 B / 16
      dcol[ti] = tmem_base + (uint32_t)(ti * a.n2);
    }
    int s = 0;
    uint32_t ph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      mbar_wait(&conv[s], ph);
      tc_fence_after();
      if (lane == 0) WG_TRACE(3, b);
      uint64_t da = desc_general(smem_u32(g_slab(s, 0)), a.g_slab, 512, 1, 0);
      uint64_t db = desc_general(smem_u32(x_slab(s, 0)), a.x_slab, 512, 1, 0);
      if (elect_one()) {
        {
          for (int k = 0; k < ksteps; ++k) {
            const uint32_t accum = (b > blk_beg || k > 0) ? 1u : 0u;
            // A (this k-step's g) is read into the collector once and reused by every tap
            if (ntaps == 1) {
              mma_tf32(dcol[0], da, db + boff[0], id, accum);
            } else {
              mma_tf32_c<1>(dcol[0], da, db + boff[0], id, accum);
#pragma unroll
              for (int ti = 1; ti < kMaxTaps; ++ti) {
                if (ti + 1 < ntaps)
                  mma_tf32_c<2>(dcol[ti], da, db + boff[ti], id, accum);
                else if (ti + 1 == ntaps)
                  mma_tf32_c<3>(dcol[ti], da, db + boff[ti], id, accum);
              }
            }
            da += 64;   // next 8 positions: 8 rows x 128 B, in 16-byte units
            db += 64;
          }
        }
        mma_commit(&empty[s]);
        WG_TRACE(4, b);
      }
      __syncwarp();
      if (++s == S) s = 0, ph ^= 1;
    }
    if (elect_one()) mma_commit(acc_full);
    __syncwarp();
  } else {
    // ===================== converters (warps 2..9): lo parts + bias sums =====================
    const int tid = threadIdx.x - 64;
    // float4 i = tid + 256 m of the g slabs sits in row p = i / 8 (mod Pp) with
    // p & 3 == (tid / 8) & 3 (Pp % 8 == 0), so a thread always meets the same 4 channels of
    // a slab (32-byte granules XOR (p & 3)); slab 0 / 1 decide which accumulator.
    const int cb = ((((tid & 7) >> 1) ^ ((tid >> 3) & 3)) << 3) + ((tid & 1) << 2);
    // bias: per-block fp32 sums folded into Kahan-compensated fp32 running sums (fp64
    // arithmetic runs at a few ops/clk/SM on this part - too slow for the block loop)
    float bs[8] = {0, 0, 0, 0, 0, 0, 0, 0}, bc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool do_bias = gi == 0 && cib == 0;
    const bool do_lo = a.three != 0;
    const int ng4 = a.Pp * 8;            // float4 per g slab
    const int nx4 = nx * (int)xrows * 8; // float4 over all x_hi slabs
    int s = 0;
    uint32_t ph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      mbar_wait(&full[s], ph);
      if (tid == 0) WG_TRACE(1, b);
      if (do_bias || do_lo) {
        const float4* hi = reinterpret_cast<const float4*>(g_slab(s, 0));
        float4* lo = reinterpret_cast<float4*>(g_slab(s, 2));
        float bf[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i0 = tid; i0 < 2 * ng4; i0 += 4 * kConvThreads) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kConvThreads;
            v[u] = i < 2 * ng4 ? hi[i] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kConvThreads;
            if (i < 2 * ng4) {
              if (do_lo) lo[i] = lo_part(v[u]);
              const bool s1 = i >= ng4;
              bf[0] += s1 ? 0.f : v[u].x; bf[1] += s1 ? 0.f : v[u].y;
              bf[2] += s1 ? 0.f : v[u].z; bf[3] += s1 ? 0.f : v[u].w;
              bf[4] += s1 ? v[u].x : 0.f; bf[5] += s1 ? v[u].y : 0.f;
              bf[6] += s1 ? v[u].z : 0.f; bf[7] += s1 ? v[u].w : 0.f;
            }
          }
        }
        if (do_bias) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float y = bf[e] - bc[e];
            const float t = bs[e] + y;
            bc[e] = (t - bs[e]) - y;
            bs[e] = t;
          }
        }
      }
      if (do_lo) {
        const float4* hi = reinterpret_cast<const float4*>(x_slab(s, 0));
        float4* lo = reinterpret_cast<float4*>(x_slab(s, nx));
        for (int i0 = tid; i0 < nx4; i0 += 4 * kConvThreads) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kConvThreads;
            if (i < nx4) v[u] = hi[i];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kConvThreads;
            if (i < nx4) lo[i] = lo_part(v[u]);
          }
        }
      }
      fence_proxy_async_smem();
      if (tid == 0) WG_TRACE(2, b);
      mbar_arrive(&conv[s]);
      if (++s == S) s = 0, ph ^= 1;
    }
    const int cw = tid / 32;   // converter warp 0..7
    if (do_bias) {
      // lanes l, l^10, l^20, l^30 hold the same channels: fixed-order butterfly, then lanes
      // 0..7 (rows p & 3 == 0) publish the warp's 64 sums.
      double bd[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        bd[e] = (double)bs[e] - (double)bc[e];
        bd[e] += __shfl_xor_sync(0xffffffffu, bd[e], 10);
        bd[e] += __shfl_xor_sync(0xffffffffu, bd[e], 20);
      }
      if (lane < 8) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bsum[cw * 64 + cb + e] = bd[e];
          bsum[cw * 64 + 32 + cb + e] = bd[4 + e];
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid < 64) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += bsum[w * 64 + tid];
        a.part_bias[(size_t)blockIdx.x * 64 + tid] = t;
      }
    }
    if (warp >= 6) {
      // ===================== epilogue: D quadrants -> fp32 partial [tap ci][co] =====================
      // TMEM lane r: r < 64 -> g_hi row co = r, r >= 64 -> g_lo row co = r - 64; columns
      // [ti n2, ti n2 + Ci) x_hi, [ti n2 + Ci, (ti+1) n2) x_lo.  Warps on lanes 64..127 park
      // their (hi + lo column) sums in the drained stage memory; the other two add theirs
      // and store coalesced rows of 64 output channels.
      const int q = warp & 3;
      const int co = (q & 1) * 32 + lane;
      float* xbuf = reinterpret_cast<float*>(smem);     // [tg * Ci][64], reuses stage memory
      float* dst = a.part + (size_t)blockIdx.x * a.tg * a.CiB * 64;
      const bool any = blk_end > blk_beg;
      if (any) {
        mbar_wait(acc_full, 0);
        tc_fence_after();
      }
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
      for (int pass = 0; pass < 2; ++pass) {
        const bool mine = (pass == 0) == (q >= 2);
        if (mine) {
          for (int ti = 0; ti < ntaps; ++ti) {
            for (int c = 0; c < a.CiB; c += 16) {
              uint32_t rh[16], rl[16];
              tmem_ld16(trow + (uint32_t)(ti * a.n2 + c), rh);
              tmem_ld16(trow + (uint32_t)(ti * a.n2 + a.CiB + c), rl);
              tmem_wait_ld();
              const int col0 = ti * a.CiB + c;
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const float v = any ? __uint_as_float(rh[e]) + __uint_as_float(rl[e]) : 0.f;
                if (q >= 2)
                  xbuf[(col0 + e) * 64 + co] = v;
                else
                  dst[(size_t)(col0 + e) * 64 + co] = v + xbuf[(col0 + e) * 64 + co];
              }
            }
          }
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
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

// gW[tap][ci][co] (HWIO) = scale * sum over the work group's CTAs of part[cta][ti ci'][co']
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, const double* __restrict__ part_bias,
                                    const WgArgs a, int grid, double scale, float* __restrict__ gw,
                                    float* __restrict__ gb) {
  const int Ci = a.Ci, Co = a.Co;
  const int total = 9 * Ci * Co;
  const int64_t pstride = (int64_t)a.tg * a.CiB * 64;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total + Co; idx += gridDim.x * blockDim.x) {
    if (idx < total) {
      const int co = idx % Co;
      const int ci = (idx / Co) % Ci;
      const int tap = idx / (Co * Ci);
      const int gi = tap / a.tg, cob = co / 64, cib = ci / a.CiB;
      const int gid = (cob * a.mi + cib) * a.ngroups + gi;
      const int c_lo = grp_start(gid, grid, a), c_hi = grp_start(gid + 1, grid, a);
      const int64_t off = ((int64_t)(tap - gi * a.tg) * a.CiB + (ci - cib * a.CiB)) * 64 + (co - cob * 64);
      double s = 0.0;
      for (int b = c_lo; b < c_hi; ++b) s += (double)part[b * pstride + off];
      gw[idx] = (float)(scale * s);
    } else if (gb) {
      const int co = idx - total, cob = co / 64;
      const int gid = cob * a.mi * a.ngroups;
      const int c_lo = grp_start(gid, grid, a), c_hi = grp_start(gid + 1, grid, a);
      double s = 0.0;
      for (int b = c_lo; b < c_hi; ++b) s += part_bias[(int64_t)b * 64 + (co - cob * 64)];
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

struct WgPlan {
  bool ok = false;
  int rg, P, Pp, tg, ngroups, grid, nstages, CiB;
  uint32_t g_slab, x_slab, x_off, stage;
  size_t smem;
};

WgPlan plan(const ConvShape& s, bool three) {
  (void)three;
  WgPlan p;
  if (s.co % 64 != 0 || (s.ci != 32 && s.ci % 64 != 0) || s.w + 2 > 256) return p;
  const int Wp = s.w + 2;
  p.CiB = s.ci == 32 ? 32 : 64;
  const int n2 = 2 * p.CiB;
  const int tg_max = 512 / n2;
  p.ngroups = (9 + tg_max - 1) / tg_max;
  p.tg = (9 + p.ngroups - 1) / p.ngroups;
  if ((s.co / 64) * (s.ci / p.CiB) * p.ngroups > kNumSMs) return p;   // every work group needs a CTA
  // (rows per block, stages) in order of preference; RP_WGRAD_CFG="rg,stages" overrides
  int cand[6][2] = {{2, 2}, {1, 3}, {1, 2}, {0, 0}, {0, 0}, {0, 0}};
  if (const char* e = getenv("RP_WGRAD_CFG")) {
    int r = 0, st = 0;
    if (sscanf(e, "%d,%d", &r, &st) == 2) cand[0][0] = r, cand[0][1] = st;
  }
  for (auto& c : cand) {
    const int rg = std::min(c[0], s.h), st = c[1];
    if (rg < 1 || st < 2 || st > kMaxStages) continue;
    WgPlan q = p;
    q.rg = rg;
    q.nstages = st;
    q.P = rg * Wp;
    q.Pp = (q.P + 7) / 8 * 8;
    q.g_slab = (uint32_t)q.Pp * 128u;
    q.x_slab = (uint32_t)(rg + 2) * Wp * 128u;
    q.x_off = 4 * q.g_slab + kLead;
    q.stage = round1k((uint64_t)q.x_off + (uint64_t)(n2 / 32) * q.x_slab + kTrail);
    (void)s;
    q.smem = st * (size_t)q.stage + (3 * kMaxStages + 2) * 8 + 8 * 64 * 8;
    if (q.smem > (size_t)kMaxSmem) continue;
    if ((size_t)q.tg * q.CiB * 64 * 4 > st * (size_t)q.stage) continue;   // epilogue exchange
    q.grid = kNumSMs;
    q.ok = true;
    return q;
  }
  return p;
}

unsigned long long* g_trace = nullptr;

int64_t part_bytes(const WgPlan& p, const ConvShape& s) {
  (void)s;
  return ((int64_t)p.grid * p.tg * p.CiB * 64 * 4 + 255) / 256 * 256;
}

}  // namespace

void conv3x3_wgrad_tc_set_trace(unsigned long long* p) { g_trace = p; }

bool conv3x3_wgrad_tc_supported(const ConvShape& s, bool three) { return plan(s, three).ok; }

int64_t conv3x3_wgrad_tc_ws_bytes(const ConvShape& s, bool three) {
  const WgPlan p = plan(s, three);
  if (!p.ok) return 0;
  return part_bytes(p, s) + (int64_t)p.grid * 64 * 8 + 256;
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
  a.three = three ? 1 : 0;
  a.CiB = p.CiB;
  a.mo = s.co / 64;
  a.mi = s.ci / p.CiB;
  a.n2 = 2 * p.CiB;
  a.tg = p.tg;
  a.ngroups = p.ngroups;
  a.blocks_per_img = (s.h + p.rg - 1) / p.rg;
  a.num_blocks = s.n * a.blocks_per_img;
  a.nstages = p.nstages;
  a.g_slab = p.g_slab;
  a.x_slab = p.x_slab;
  a.x_off = p.x_off;
  a.stage = p.stage;
  a.trace = g_trace;
  a.part = static_cast<float*>(ws);
  a.part_bias = reinterpret_cast<double*>(static_cast<char*>(ws) + part_bytes(p, s));
  const CUtensorMap mg = cached(g, s.n, s.h, s.w, s.co, p.rg);
  const CUtensorMap mx = cached(in, s.n, s.h, s.w, s.ci, p.rg + 2);
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(wgrad_tc_kernel), kMaxSmem);
  wgrad_tc_kernel<<<p.grid, kThreads, p.smem, st>>>(mg, mx, a);
  RP_LAUNCHED();
  const int total = 9 * s.ci * s.co + s.co;
  wgrad_reduce_kernel<<<ceil_div(total, 256), 256, 0, st>>>(a.part, a.part_bias, a, p.grid, (double)scale, gw, gb);
  RP_LAUNCHED();
}

}  // namespace rp::k
