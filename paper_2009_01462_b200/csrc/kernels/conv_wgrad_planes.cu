// tcgen05 weight gradient from fp16 *plane pairs* (fp32-accurate path, RP_MATH_FP32):
//
//   gW[tap][ci][co] = scale * sum_p x[p + off(tap)][ci] * g[p][co],  gb[co] = scale * sum_p g[p][co]
//
// with x = x0 + x1 and g s = g0 + g1, x0 = fp16(x), x1 = fp16(x - x0) (22 significant bits,
// planes.cuh; the producing epilogues write the planes next to the fp32 tensor, the cotangent
// side with its power-of-two scale s, divided out in the reduce).  Operands go from HBM to the
// MMA by TMA alone -- no fp32 staging, no converter pass -- which is what bounded the fp32
// wgrad kernels (conv_wgrad_tc.cu, conv_wgrad_bf16.cu: three shared-memory passes per block):
//   A = [g0 ; g1]  (M = 128 for a 64-channel co block, MN-major fp16, 128B swizzle)
//   B = [x0 ; x1]  (N = 128 for a 64-channel ci block)
// one M128 x N128 x K16 MMA per (16 positions, tap) yields g0x0 + g1x0 + g0x1 + g1x1 in the
// four quadrants of D (everything above 2^-17 |g x|); the epilogue adds the quadrants.
// Positions are the padded interior frame (rows x (W+2)), taps are shifted B descriptors,
// 3 taps per tap group (TMEM 3 x 128 columns), (co block, ci block, tap group) work groups,
// per-CTA partials and a fixed-order fp64 reduce, as in conv_wgrad_tc.cu.  The bias sums
// g0 + g1 from the staged planes (bias warps, Kahan-compensated fp32).
//
// Single-plane mode (RP_MATH_BF16, config C5): x and g are one bf16 plane each (the bf16
// conv epilogues write them); the two 64-channel atoms of A and B are then channels
// [128 cob, +64) and [128 cob + 64, +64) of the same plane, so the identical MMA stream
// yields a 128 co x 128 ci tile per tap, the epilogue stores all four quadrants and the
// bias warps sum 128 channels.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../common.cuh"
#include "kernels.cuh"
#include "planes.cuh"
#include "umma.cuh"

namespace rp::k {

namespace {

using namespace rp::umma;

constexpr int kThreads = 320;
constexpr int kMaxStages = 4;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kLead = 128;          // zero row before the x slabs (tap shift -1)
constexpr int kTrail = 2048;        // zero rows after them (K padding reads up to 15 rows)
constexpr int kTg = 3;              // taps per group

struct PwArgs {
  int N, H, W, Ci, Co, Wp, rg, P, Pp, nstages;
  int mo, mi;                    // co / ci blocks (64 channels, single: 128)
  int single;                    // 1: one bf16 plane per operand, 128-channel blocks
  int nobias;                    // diagnostics (RP_WGRAD_NOBIAS): skip the bias sums
  int dbg;                       // diagnostics (RP_WGRAD_DBG): 1 no MMA, 2 no x loads, 4 no g loads
  int blocks_per_img, num_blocks;
  uint32_t g_slab;               // bytes per bf16 g plane slab (Pp rows x 128 B, 1 KB aligned)
  uint32_t x_slab;               // bytes per bf16 x plane slab (rg * Wp rows of one filter row, packed)
  uint32_t x_off;
  uint32_t stage;
  float* part;                   // [grid][kTg * cblk (ci)][cblk (co)]
  double* part_bias;             // [grid][cblk]
  int njobs;                     // 1, or 2: two weight gradients of the same shape in one launch
  float* gw[2];                  // reduce: per-job outputs and scales
  float* gb[2];
  double scale[2];
  const float* gsc[2];           // the A (g-side) planes' power-of-two scale (device; null: kActPlaneScale)
  int mc;                        // 1: clusters of 3 CTAs (the tap groups of one work group) share the
                                 //    operand loads by TMA multicast (wgrad_planes_kernel<true>);
                                 // 2: the same CTA-triple mapping without clusters (each loads its own)
};

__device__ __forceinline__ int grp_start(int gid, int grid, const PwArgs& a) {
  return (int)((int64_t)grid * gid / (a.njobs * 3 * a.mo * a.mi));
}

// clustered form: work group w (job, co block, ci block) owns clusters [cgrp_start(w), cgrp_start(w + 1))
// of the ncl = grid / 3 clusters; CTA 3 cl + r of a cluster is tap group r
__host__ __device__ __forceinline__ int cgrp_start(int w, int ncl, const PwArgs& a) {
  return (int)((int64_t)ncl * w / (a.njobs * a.mo * a.mi));
}

// MC (clustered multicast): the three tap groups of a work group run as one
// cluster on the same blocks.  The g planes are identical for them and their x rows overlap
// (filter rows dy = 0..2 shift them by one row), so per stage rank 0 loads the g0 slab, rank 1
// the g1 slab and rank 2 both x slabs over the union of the three groups' rows (rg + 2), each
// multicast into all three CTAs: every operand byte leaves L2 once per cluster instead of once
// per tap group.  A stage is free once all three CTAs' MMAs (multicast commits) and rank 0's
// bias warps (remote arrives) are done with it.
template <bool MC>
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_planes_kernel(const __grid_constant__ CUtensorMap tg0a, const __grid_constant__ CUtensorMap tg1a,
                        const __grid_constant__ CUtensorMap tx0a, const __grid_constant__ CUtensorMap tx1a,
                        const __grid_constant__ CUtensorMap tg0b, const __grid_constant__ CUtensorMap tg1b,
                        const __grid_constant__ CUtensorMap tx0b, const __grid_constant__ CUtensorMap tx1b,
                        const PwArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const int S = a.nstages;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * a.stage);
  uint64_t* full = bars;                        // [S] TMA -> MMA / bias warps
  uint64_t* empty = bars + kMaxStages;          // [S] MMA -> TMA
  uint64_t* bias_free = bars + 2 * kMaxStages;  // [S] bias warps -> TMA
  uint64_t* acc_full = bars + 3 * kMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStages + 1);
  double* bsum = reinterpret_cast<double*>(bars + 3 * kMaxStages + 2);   // [4 warps][128]

  auto g_slab = [&](int s, int j) { return smem + s * a.stage + j * a.g_slab; };
  auto x_slab = [&](int s, int j) { return smem + s * a.stage + a.x_off + j * a.x_slab; };

  int job, gi, cib, cob, jg, ng;
  if constexpr (MC) {
    const int NW = a.njobs * a.mo * a.mi;
    const int ncl = gridDim.x / 3, cl = blockIdx.x / 3;
    int w = 0;
    while (w + 1 < NW && cgrp_start(w + 1, ncl, a) <= cl) ++w;
    const int c_lo = cgrp_start(w, ncl, a), c_hi = cgrp_start(w + 1, ncl, a);
    job = w / (a.mo * a.mi);
    const int gj = w - job * a.mo * a.mi;
    cib = gj % a.mi;
    cob = gj / a.mi;
    gi = (int)cluster_ctarank();
    jg = cl - c_lo;
    ng = c_hi - c_lo;
  } else if (a.mc == 2) {
    // triples: CTA 3 t + r is tap group r of triple t's position range (the MC mapping without
    // clusters): the three CTAs reading the same g and x rows are adjacent in launch order
    const int NW = a.njobs * a.mo * a.mi;
    const int ncl = gridDim.x / 3, cl = blockIdx.x / 3;
    int w = 0;
    while (w + 1 < NW && cgrp_start(w + 1, ncl, a) <= cl) ++w;
    const int c_lo = cgrp_start(w, ncl, a), c_hi = cgrp_start(w + 1, ncl, a);
    job = w / (a.mo * a.mi);
    const int gj = w - job * a.mo * a.mi;
    cib = gj % a.mi;
    cob = gj / a.mi;
    gi = (int)(blockIdx.x % 3);
    jg = cl - c_lo;
    ng = c_hi - c_lo;
  } else {
    const int NG1 = 3 * a.mo * a.mi;                // work groups per job
    const int NG = a.njobs * NG1;
    int gid = 0;
    while (gid + 1 < NG && grp_start(gid + 1, gridDim.x, a) <= (int)blockIdx.x) ++gid;
    const int c_lo = grp_start(gid, gridDim.x, a), c_hi = grp_start(gid + 1, gridDim.x, a);
    job = gid / NG1;
    const int gj = gid - job * NG1;
    gi = gj % 3;
    cib = (gj / 3) % a.mi;
    cob = gj / (3 * a.mi);
    jg = blockIdx.x - c_lo;
    ng = c_hi - c_lo;
  }
  const int blk_beg = (int)((int64_t)jg * a.num_blocks / ng);
  const int blk_end = (int)((int64_t)(jg + 1) * a.num_blocks / ng);
  const int t0 = gi * kTg;
  const int Wp = a.Wp;
  const int xrows = a.rg * Wp;   // x rows of this tap group's filter row only (y0 - 1 + gi ..)
  const bool cl_bias = cib == 0 && !a.nobias;      // this work group sums the bias
  // unclustered: tap group 0 sums it; clustered: the three CTAs hold the same g slab and each sums
  // a third of its rows (a slot is gated by every CTA's bias warps, so they share the work)
  const bool do_bias = (MC || gi == 0) && cl_bias;
  const int bias_p0 = MC ? gi * a.P / 3 : 0, bias_p1 = MC ? (gi + 1) * a.P / 3 : a.P;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MC ? 3 + (cl_bias ? 3 : 0) : 1);
      mbar_init(&bias_free[i], 128);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
    if (job == 0) {
      prefetch_tmap(&tg0a);
      prefetch_tmap(&tg1a);
      prefetch_tmap(&tx0a);
      prefetch_tmap(&tx1a);
    } else {
      prefetch_tmap(&tg0b);
      prefetch_tmap(&tg1b);
      prefetch_tmap(&tx0b);
      prefetch_tmap(&tx1b);
    }
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  {
    // zero only what the MMAs read but TMA never writes: the g slabs' K-padding rows [P, Pp),
    // the lead row before the x slabs (tap shift -1) and the trail after them
    const int pad16 = (a.Pp - a.P) * 8;              // 16-byte words per g slab
    const int lead16 = kLead / 16, trail16 = kTrail / 16;
    const int per_stage = 2 * pad16 + lead16 + trail16;
    for (int i = threadIdx.x; i < S * per_stage; i += blockDim.x) {
      const int st = i / per_stage, r = i - st * per_stage;
      uint8_t* base = smem + (size_t)st * a.stage;
      uint8_t* dst;
      if (r < 2 * pad16) {
        const int j = r / pad16;
        dst = base + (size_t)j * a.g_slab + (size_t)a.P * 128 + (size_t)(r - j * pad16) * 16;
      } else if (r < 2 * pad16 + lead16) {
        dst = base + a.x_off - kLead + (size_t)(r - 2 * pad16) * 16;
      } else {
        dst = base + a.x_off + 2 * (size_t)a.x_slab + (size_t)(r - 2 * pad16 - lead16) * 16;
      }
      *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  if constexpr (MC)
    cluster_sync();   // every CTA's barriers exist before any peer multicasts into its shared memory
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // PDL: let the next grid's prologue overlap this grid's tail; the operands (and the partial
  // buffer the previous reduce read) belong to the previous grids until pdl_wait()
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    // ===================== TMA producer: 4 plane loads per block =====================
    int s = 0;
    uint32_t ph = 0;
    const uint32_t bytes = ((a.dbg & 4) ? 0u : 2u * a.P * 128u) + ((a.dbg & 2) ? 0u : 2u * xrows * 128u);
    auto issue_loads = [&](const CUtensorMap* mg0, const CUtensorMap* mg1, const CUtensorMap* mx0,
                           const CUtensorMap* mx1, int s, int y0, int n) {
        if (a.dbg & 6) {   // diagnostics: a subset of the loads
          if (!(a.dbg & 4)) {
            tma_load_4d(mg0, &full[s], g_slab(s, 0), 64 * cob, -1, y0, n);
            tma_load_4d(mg1, &full[s], g_slab(s, 1), 64 * cob, -1, y0, n);
          }
          if (!(a.dbg & 2)) {
            tma_load_4d(mx0, &full[s], x_slab(s, 0), 64 * cib, -1, y0 - 1 + gi, n);
            tma_load_4d(mx1, &full[s], x_slab(s, 1), 64 * cib, -1, y0 - 1 + gi, n);
          }
        } else if (a.single) {   // the two 64-channel atoms of one plane
          tma_load_4d(mg0, &full[s], g_slab(s, 0), 128 * cob, -1, y0, n);
          tma_load_4d(mg0, &full[s], g_slab(s, 1), 128 * cob + 64, -1, y0, n);
          tma_load_4d(mx0, &full[s], x_slab(s, 0), 128 * cib, -1, y0 - 1 + gi, n);
          tma_load_4d(mx0, &full[s], x_slab(s, 1), 128 * cib + 64, -1, y0 - 1 + gi, n);
        } else {
          tma_load_4d(mg0, &full[s], g_slab(s, 0), 64 * cob, -1, y0, n);
          tma_load_4d(mg1, &full[s], g_slab(s, 1), 64 * cob, -1, y0, n);
          tma_load_4d(mx0, &full[s], x_slab(s, 0), 64 * cib, -1, y0 - 1 + gi, n);
          tma_load_4d(mx1, &full[s], x_slab(s, 1), 64 * cib, -1, y0 - 1 + gi, n);
        }
    };
    if constexpr (MC) {
      // my share of every stage, multicast to the cluster (rank 0: g atom 0, 1: g atom 1, 2: x)
      const uint32_t bytes_mc = 2u * a.P * 128u + 2u * (uint32_t)(a.rg + 2) * Wp * 128u;
      const CUtensorMap* mg0 = job == 0 ? &tg0a : &tg0b;
      const CUtensorMap* mg1 = job == 0 ? (a.single ? &tg0a : &tg1a) : (a.single ? &tg0b : &tg1b);
      const CUtensorMap* mx0 = job == 0 ? &tx0a : &tx0b;
      const CUtensorMap* mx1 = job == 0 ? (a.single ? &tx0a : &tx1a) : (a.single ? &tx0b : &tx1b);
      const int cg0 = a.single ? 128 * cob : 64 * cob, cg1 = a.single ? 128 * cob + 64 : 64 * cob;
      const int cx0 = a.single ? 128 * cib : 64 * cib, cx1 = a.single ? 128 * cib + 64 : 64 * cib;
      for (int b = blk_beg; b < blk_end; ++b) {
        const int n = b / a.blocks_per_img;
        const int y0 = (b - n * a.blocks_per_img) * a.rg;
        mbar_wait(&empty[s], ph ^ 1);   // every CTA (and rank 0's bias warps) released the slot
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[s], bytes_mc);
          if (gi == 0) {
            tma_load_4d_mc(mg0, &full[s], g_slab(s, 0), cg0, -1, y0, n, 0x7);
          } else if (gi == 1) {
            tma_load_4d_mc(mg1, &full[s], g_slab(s, 1), cg1, -1, y0, n, 0x7);
          } else {
            tma_load_4d_mc(mx0, &full[s], x_slab(s, 0), cx0, -1, y0 - 1, n, 0x7);
            tma_load_4d_mc(mx1, &full[s], x_slab(s, 1), cx1, -1, y0 - 1, n, 0x7);
          }
        }
        __syncwarp();
        if (++s == S) s = 0, ph ^= 1;
      }
    } else
    for (int b = blk_beg; b < blk_end; ++b) {
      const int n = b / a.blocks_per_img;
      const int y0 = (b - n * a.blocks_per_img) * a.rg;
      mbar_wait(&empty[s], ph ^ 1);
      if (do_bias) mbar_wait(&bias_free[s], ph ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], bytes);
        // the job's tensor maps are passed as direct grid-constant addresses in each branch
        // (no select between the two sets)
        if (job == 0)
          issue_loads(&tg0a, &tg1a, &tx0a, &tx1a, s, y0, n);
        else
          issue_loads(&tg0b, &tg1b, &tx0b, &tx1b, s, y0, n);
      }
      __syncwarp();
      if (++s == S) s = 0, ph ^= 1;
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t id = idesc(a.single ? 1 : 0, 128, 128, 1, 1);   // single: bf16; pair: fp16
    const int ksteps = a.Pp / 16;
    uint64_t boff[kTg];
#pragma unroll
    for (int ti = 0; ti < kTg; ++ti) {
      const int t = t0 + ti;
      boff[ti] = (uint64_t)(int64_t)(((t % 3) - 1) * 8);   // dx shift (x slab starts at row y0 - 1 + dy); 128 B / 16
    }
    int s = 0;
    uint32_t ph = 0;
    for (int b = blk_beg; b < blk_end; ++b) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      uint64_t da = desc_general(smem_u32(g_slab(s, 0)), a.g_slab, 1024, 2, 0);
      // MC: this tap group's filter row dy = gi starts gi rows into the union slab
      uint64_t db = desc_general(smem_u32(x_slab(s, 0)) + (MC ? (uint32_t)(gi * Wp * 128) : 0u), a.x_slab, 1024, 2, 0);
      if (elect_one()) {
        for (int k = 0; k < ksteps && !(a.dbg & 1); ++k) {
          const uint32_t accum = (b > blk_beg || k > 0) ? 1u : 0u;
          // the 3 taps share A (the g rows of these 16 positions): read it once through the
          // A collector instead of once per MMA (shared-memory operand bandwidth)
          mma_f16_c<1>(tmem_base, da, db + boff[0], id, accum);
          mma_f16_c<2>(tmem_base + 128u, da, db + boff[1], id, accum);
          mma_f16_c<3>(tmem_base + 256u, da, db + boff[2], id, accum);
          da += 128;   // 16 positions = 16 rows x 128 B, in 16-byte units
          db += 128;
        }
        if constexpr (MC)
          mma_commit_mc(&empty[s], 0x7);   // the slot is free in every CTA once all three are done
        else
          mma_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == S) s = 0, ph ^= 1;
    }
    if (elect_one()) mma_commit(acc_full);
    __syncwarp();
  } else if (warp < 6) {
    // ===================== bias warps: sum g0 + g1 over the block's positions =====================
    // thread t: logical 16-byte chunk cq = t % 8 (channels 8 cq .. 8 cq + 7) of rows
    // p = t / 8 + 16 k; the chunk sits at (cq ^ (absolute row & 7)) in the swizzled row.
    if (do_bias) {
      const int tid = threadIdx.x - 64;
      const int cq = tid & 7, r0 = tid >> 3;
      // pair mode: bs[0..7] = channels 8 cq + e of g0 + g1; single: bs[8 j + e] = channel
      // 64 j + 8 cq + e (atom j)
      float bs[16] = {}, bk[16] = {};
      const bool single = a.single != 0;
      int s = 0;
      uint32_t ph = 0;
      for (int b = blk_beg; b < blk_end; ++b) {
        mbar_wait(&full[s], ph);
        float bf[16] = {};
        const uint8_t* p0 = g_slab(s, 0);
        const uint8_t* p1 = g_slab(s, 1);
        const uint32_t base0 = smem_u32(p0), base1 = smem_u32(p1);
        for (int p = bias_p0 + r0; p < bias_p1; p += 16) {
          const int ph0 = (int)(((base0 >> 7) + p) & 7), ph1 = (int)(((base1 >> 7) + p) & 7);
          const uint4 u = *reinterpret_cast<const uint4*>(p0 + (size_t)p * 128 + ((cq ^ ph0) << 4));
          const uint4 v = *reinterpret_cast<const uint4*>(p1 + (size_t)p * 128 + ((cq ^ ph1) << 4));
          if (single) {
            const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&u);
            const __nv_bfloat162* vh = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              bf[2 * e] += __low2float(uh[e]);
              bf[2 * e + 1] += __high2float(uh[e]);
              bf[8 + 2 * e] += __low2float(vh[e]);
              bf[8 + 2 * e + 1] += __high2float(vh[e]);
            }
          } else {
            const __half2* uh = reinterpret_cast<const __half2*>(&u);
            const __half2* vh = reinterpret_cast<const __half2*>(&v);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              bf[2 * e] += __low2float(uh[e]) + __low2float(vh[e]);
              bf[2 * e + 1] += __high2float(uh[e]) + __high2float(vh[e]);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float y = bf[e] - bk[e];
          const float t = bs[e] + y;
          bk[e] = (t - bs[e]) - y;
          bs[e] = t;
        }
        if constexpr (MC) {
          // each CTA's bias warps release the slot in all three CTAs (they all write into this one)
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (tid == 0)
            for (uint32_t r = 0; r < 3; ++r) mbar_arrive_cluster(&empty[s], r);
        } else {
          mbar_arrive(&bias_free[s]);
        }
        if (++s == S) s = 0, ph ^= 1;
      }
      // threads t, t + 8, ... (same cq) combine in fixed order: lanes xor 8, 16, then warps
      const int cw = tid / 32;
      const int nch = single ? 128 : 64;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        if (e >= 8 && !single) break;
        double d = (double)bs[e] - (double)bk[e];
        d += __shfl_xor_sync(0xffffffffu, d, 8);
        d += __shfl_xor_sync(0xffffffffu, d, 16);
        if (lane < 8) bsum[cw * 128 + (e >> 3) * 64 + 8 * cq + (e & 7)] = d;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid < nch) {
        double t = 0.0;
        for (int w = 0; w < 4; ++w) t += bsum[w * 128 + tid];
        a.part_bias[(size_t)blockIdx.x * nch + tid] = t;
      }
    }
  } else {
    // ===================== epilogue: D quadrants -> fp32 partial [tap ci][co] =====================
    // TMEM lane r: r < 64 -> g0 row co = r, r >= 64 -> g1 row co = r - 64; columns
    // [ti 128, ti 128 + 64) x0, [ti 128 + 64, (ti + 1) 128) x1.  Warps on lanes 64..127
    // park their (x0 + x1 column) sums in the drained stage memory; the other two add
    // theirs and store coalesced rows of 64 output channels.
    const int q = warp & 3;
    const int co = (q & 1) * 32 + lane;
    float* xbuf = reinterpret_cast<float*>(smem);     // [kTg * 64][64], reuses stage memory
    float* dst = a.part + (size_t)blockIdx.x * kTg * 64 * 64;
    const bool any = blk_end > blk_beg;
    if (any) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
    }
    // stage memory is drained once the last MMAs completed and the bias warps let go
    if (do_bias) asm volatile("bar.sync 3, 256;" ::: "memory");
    const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
    if (a.single) {
      // lane r = co r, column c = ci c of each tap: every quadrant is its own output
      float* dst1 = a.part + (size_t)blockIdx.x * kTg * 128 * 128;
      const int co1 = q * 32 + lane;
      for (int ti = 0; ti < kTg; ++ti) {
        for (int c = 0; c < 128; c += 16) {
          uint32_t r[16];
          tmem_ld16(trow + (uint32_t)(ti * 128 + c), r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            dst1[(size_t)(ti * 128 + c + e) * 128 + co1] = any ? __uint_as_float(r[e]) : 0.f;
        }
      }
    } else
    for (int pass = 0; pass < 2; ++pass) {
      const bool mine = (pass == 0) == (q >= 2);
      if (mine) {
        for (int ti = 0; ti < kTg; ++ti) {
          for (int c = 0; c < 64; c += 16) {
            uint32_t rh[16], rl[16];
            tmem_ld16(trow + (uint32_t)(ti * 128 + c), rh);
            tmem_ld16(trow + (uint32_t)(ti * 128 + 64 + c), rl);
            tmem_wait_ld();
            const int col0 = ti * 64 + c;
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
  if (do_bias && warp >= 2 && warp < 6) asm volatile("bar.sync 3, 256;" ::: "memory");

  tc_fence_before();
  if constexpr (MC)
    cluster_sync();   // no peer arrives on (or multicasts into) this CTA's shared memory after it exits
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

__global__ void wgrad_planes_reduce_kernel(const float* __restrict__ part, const double* __restrict__ part_bias,
                                           const PwArgs a, int grid) {
  pdl_launch_dependents();   // the next grid's prologue may overlap; it waits before touching memory
  pdl_wait();                // the partials of the weight-gradient grid
  const int Ci = a.Ci, Co = a.Co;
  const int total = 9 * Ci * Co;
  const int cbk = a.single ? 128 : 64;
  const int64_t pstride = (int64_t)kTg * cbk * cbk;
  const int per_job = total + Co;
  for (int gidx = blockIdx.x * blockDim.x + threadIdx.x; gidx < a.njobs * per_job;
       gidx += gridDim.x * blockDim.x) {
    const int job = gidx / per_job;
    const int idx = gidx - job * per_job;
    const int gbase = job * 3 * a.mo * a.mi;
    float* gw = a.gw[job];
    float* gb = a.gb[job];
    // pairs: the g side carries *gsc (null: the activation scale), the x side the activation
    // scale; the bias sums are of the g side alone
    const double gs = a.single ? 1.0 : (a.gsc[job] ? (double)*a.gsc[job] : (double)kActPlaneScale);
    const double scale = a.scale[job] / (a.single ? 1.0 : gs * (double)kActPlaneScale);
    const double bscale = a.scale[job] / gs;
    if (idx < total) {
      const int co = idx % Co;
      const int ci = (idx / Co) % Ci;
      const int tap = idx / (Co * Ci);
      const int gi = tap / kTg, cob = co / cbk, cib = ci / cbk;
      // the CTAs of this (job, co block, ci block, tap group): first + stride * [0, count)
      int first, stride, count;
      if (a.mc) {   // clusters or triples: CTA 3 t + gi
        const int w = job * a.mo * a.mi + cob * a.mi + cib, ncl = grid / 3;
        const int c_lo = cgrp_start(w, ncl, a), c_hi = cgrp_start(w + 1, ncl, a);
        first = 3 * c_lo + gi, stride = 3, count = c_hi - c_lo;
      } else {
        const int gid = gbase + (cob * a.mi + cib) * 3 + gi;
        const int c_lo = grp_start(gid, grid, a), c_hi = grp_start(gid + 1, grid, a);
        first = c_lo, stride = 1, count = c_hi - c_lo;
      }
      const int64_t off = ((int64_t)(tap - gi * kTg) * cbk + (ci - cib * cbk)) * cbk + (co - cob * cbk);
      // 8 loads in flight, 4 accumulators combined in a fixed order (deterministic)
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
      int i0 = 0;
      for (; i0 + 8 <= count; i0 += 8) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldg(part + (int64_t)(first + (i0 + i) * stride) * pstride + off);
#pragma unroll
        for (int i = 0; i < 8; ++i) s4[i & 3] += (double)v[i];
      }
      for (; i0 < count; ++i0) s4[0] += (double)__ldg(part + (int64_t)(first + i0 * stride) * pstride + off);
      gw[idx] = (float)(scale * ((s4[0] + s4[1]) + (s4[2] + s4[3])));
    } else if (gb) {
      const int co = idx - total, cob = co / cbk;
      int first, stride, count;   // the ci-block-0 CTAs of this co block that sum the bias
      if (a.mc == 1) {   // all three CTAs of each cluster (a third of the rows each), in CTA order
        const int w = job * a.mo * a.mi + cob * a.mi, ncl = grid / 3;
        const int c_lo = cgrp_start(w, ncl, a), c_hi = cgrp_start(w + 1, ncl, a);
        first = 3 * c_lo, stride = 1, count = 3 * (c_hi - c_lo);
      } else if (a.mc == 2) {   // triples: tap group 0 of each triple sums its rows
        const int w = job * a.mo * a.mi + cob * a.mi, ncl = grid / 3;
        const int c_lo = cgrp_start(w, ncl, a), c_hi = cgrp_start(w + 1, ncl, a);
        first = 3 * c_lo, stride = 3, count = c_hi - c_lo;
      } else {
        const int gid = gbase + cob * a.mi * 3;
        const int c_lo = grp_start(gid, grid, a), c_hi = grp_start(gid + 1, grid, a);
        first = c_lo, stride = 1, count = c_hi - c_lo;
      }
      double s = 0.0;
      for (int i = 0; i < count; ++i) s += part_bias[(int64_t)(first + i * stride) * cbk + (co - cob * cbk)];
      gb[co] = (float)(bscale * s);
    }
  }
}

// fp32 -> planes (planes.cuh) for tensors not written by a conv epilogue: p1 non-null: the
// fp16 pair of v s (s = *scale, or the activation scale); p1 null: the bf16 single plane
__global__ void split_planes_kernel(const float4* __restrict__ in, int64_t n4, uint2* __restrict__ p0,
                                    uint2* __restrict__ p1, const float* __restrict__ scale) {
  const float sc = scale ? *scale : kActPlaneScale;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    const float vv[4] = {v.x, v.y, v.z, v.w};
    if (p1)
      pack_pair4(vv, sc, p0[i], p1[i]);
    else
      p0[i] = pack_single4(vv);
  }
}

// per-CTA max |v| (exact, order-independent: deterministic)
__global__ void absmax_partial_kernel(const float4* __restrict__ in, int64_t n4, float* __restrict__ part) {
  __shared__ float sh[8];
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, sh[w]);
    part[blockIdx.x] = fmaxf(m, sh[0]);
  }
}

// the scale of a cotangent plane pair from the max partials, computed by every CTA (CTA 0 stores it)
__global__ void split_planes_scaled_kernel(const float4* __restrict__ in, int64_t n4, uint2* __restrict__ p0,
                                           uint2* __restrict__ p1, const float* __restrict__ part, int nparts,
                                           float* __restrict__ scale_out) {
  __shared__ float sh_s;
  if (threadIdx.x < 32) {
    float m = 0.f;
    for (int i = threadIdx.x; i < nparts; i += 32) m = fmaxf(m, part[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) {
      sh_s = cotangent_plane_scale(m);
      if (blockIdx.x == 0) *scale_out = sh_s;
    }
  }
  __syncthreads();
  const float sc = sh_s;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    const float vv[4] = {v.x, v.y, v.z, v.w};
    pack_pair4(vv, sc, p0[i], p1[i]);
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

// bf16 NHWC plane as (C, W, H, N); box = 64 channels (128 B) x (W+2) columns from x = -1 x
// rows, 128-byte swizzle (the MMA's MN-major layout)
CUtensorMap make_map(const void* t, int n, int h, int w, int c, int rows) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  const cuuint32_t box[4] = {64, (cuuint32_t)(w + 2), (cuuint32_t)rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(t), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled (planes) failed (" + std::to_string((int)r) + ")");
  return m;
}

std::mutex g_mu;
std::map<std::tuple<const void*, int, int, int, int, int>, CUtensorMap> g_maps;

CUtensorMap cached(const void* t, int n, int h, int w, int c, int rows) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(t, n, h, w, c, rows);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();   // callers hold copies, never references
    it = g_maps.emplace(key, make_map(t, n, h, w, c, rows)).first;
  }
  return it->second;
}

uint32_t round1k(uint64_t v) { return (uint32_t)((v + 1023) / 1024 * 1024); }

struct PwPlan {
  bool ok = false;
  int rg, P, Pp, grid, nstages;
  uint32_t g_slab, x_slab, x_off, stage;
  size_t smem;
};

// mc: the clustered multicast kernel (x slabs over the union of the three tap groups' rows,
// grid a multiple of 3)
PwPlan plan(const ConvShape& s, bool single = false, bool mc = false) {
  PwPlan p;
  const int cbk = single ? 128 : 64;
  if (s.co % cbk != 0 || s.ci % cbk != 0 || s.w + 2 > 256) return p;
  if (3 * (s.co / cbk) * (s.ci / cbk) > kNumSMs) return p;
  const int Wp = s.w + 2;
  // (rows per block, stages) in order of preference
  const int cand[][2] = {{4, 3}, {3, 3}, {2, 3}, {4, 2}, {2, 2}, {1, 2}};
  static const int forced = [] {   // diagnostics: RP_WGRAD_PCFG = rows * 10 + stages
    const char* e = std::getenv("RP_WGRAD_PCFG");
    return e ? std::atoi(e) : 0;
  }();
  for (const auto& c : cand) {
    if (forced && forced != c[0] * 10 + c[1]) continue;
    const int rg = std::min(c[0], s.h), st = c[1];
    PwPlan q;
    q.rg = rg;
    q.nstages = st;
    q.P = rg * Wp;
    q.Pp = (q.P + 15) / 16 * 16;
    q.g_slab = round1k((uint64_t)q.Pp * 128);
    q.x_slab = (uint32_t)(mc ? rg + 2 : rg) * Wp * 128u;   // one filter row's x rows per tap group (mc: all three)
    q.x_off = 2 * q.g_slab + kLead;
    q.stage = round1k((uint64_t)q.x_off + 2ull * q.x_slab + kTrail);
    // the pair epilogue parks kTg 64x64 fp32 partial sums in the drained stage memory: tiny
    // images (H W <= 4: the dense H = W = 1 case) widen the stage stride to hold them
    const uint64_t park = (uint64_t)kTg * 64 * 64 * 4;
    if ((uint64_t)st * q.stage < park) q.stage = round1k((park + st - 1) / st);
    q.smem = st * (size_t)q.stage + (3 * kMaxStages + 2) * 8 + 4 * 128 * 8 + 256;
    if (q.smem > (size_t)kMaxSmem) continue;
    if ((size_t)kTg * 64 * 64 * 4 > st * (size_t)q.stage) continue;   // the pair epilogue's park buffer
    q.grid = mc ? 3 * (kNumSMs / 3) : kNumSMs;
    q.ok = true;
    return q;
  }
  return p;
}

int64_t part_bytes(const PwPlan& p, bool single = false) {
  const int64_t cbk = single ? 128 : 64;
  return ((int64_t)p.grid * kTg * cbk * cbk * 4 + 255) / 256 * 256;
}

}  // namespace

bool conv3x3_wgrad_planes_supported(const ConvShape& s) { return plan(s).ok; }

int64_t conv3x3_wgrad_planes_ws_bytes(const ConvShape& s) {
  const PwPlan p = plan(s);
  if (!p.ok) return 0;
  return part_bytes(p) + (int64_t)p.grid * 64 * 8 + 256;
}

void split_planes(const float* in, int64_t n, void* p0, void* p1, cudaStream_t st, float* scale_out) {
  if (n <= 0) return;
  if (n % 4) fail(RP_ERR_SHAPE, "split_planes: element count must be a multiple of 4");
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 16 * kNumSMs);
  if (scale_out) {
    if (!p1) fail(RP_ERR_INTERNAL, "split_planes: a scale needs the fp16 pair");
    // [0]: the scale, [kPlaneScalePartOffset ..]: per-CTA max |v|
    float* part = scale_out + kPlaneScalePartOffset;
    const int pgrid = (int)std::min<int64_t>((n4 + 255) / 256, kPlaneScaleMaxParts);
    absmax_partial_kernel<<<pgrid, 256, 0, st>>>(reinterpret_cast<const float4*>(in), n4, part);
    RP_LAUNCHED();
    split_planes_scaled_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(in), n4, static_cast<uint2*>(p0),
                                                     static_cast<uint2*>(p1), part, pgrid, scale_out);
    RP_LAUNCHED();
    return;
  }
  split_planes_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(in), n4, static_cast<uint2*>(p0),
                                           static_cast<uint2*>(p1), nullptr);
  RP_LAUNCHED();
}

void split_planes_from_parts(const float* in, int64_t n, void* p0, void* p1, const float* part, int nparts,
                             float* scale_out, cudaStream_t st) {
  if (n <= 0) return;
  if (n % 4) fail(RP_ERR_SHAPE, "split_planes: element count must be a multiple of 4");
  if (nparts > 2 * kPlaneScaleMaxParts) fail(RP_ERR_INTERNAL, "split_planes: too many max partials");
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 16 * kNumSMs);
  split_planes_scaled_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(in), n4, static_cast<uint2*>(p0),
                                                   static_cast<uint2*>(p1), part, nparts, scale_out);
  RP_LAUNCHED();
}

namespace {
struct WgJob {
  const void *x0, *x1, *g0, *g1;
  float scale;
  float* gw;
  float* gb;
  const float* gsc;   // the g planes' scale (device; null: 1)
};

void launch_wgrad_planes(const ConvShape& s, const WgJob* jobs, int njobs, void* ws, cudaStream_t st, bool single) {
  PwPlan p = plan(s, single);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_wgrad_planes: unsupported shape");
  // RP_WGRAD_MC=1: the clustered multicast kernel.  Measured (C2/C3 shape, one launch): DRAM reads
  // 1.00x algorithmic (135 MB; unclustered 1.36x) and half the L2 traffic, but 1.9x the time --
  // the three CTAs advance in lockstep and every stage's release waits on all of them and on the
  // bias warps, a round trip the 3-stage ring does not cover.  Off by default.
  static const bool mc_on = [] {
    const char* e = std::getenv("RP_WGRAD_MC");
    return e && e[0] == '1';
  }();
  static const int wdbg0 = [] {
    const char* e = std::getenv("RP_WGRAD_DBG");
    return e ? std::atoi(e) : 0;
  }();
  bool mc = false;
  {
    const int cbk0 = single ? 128 : 64;
    PwPlan q = plan(s, single, true);
    if (mc_on && !wdbg0 && q.ok) {
      // one wave of clusters: as many 3-CTA clusters as the GPCs hold at once (not every GPC's SM
      // count is a multiple of 3)
      ensure_max_dynamic_smem(reinterpret_cast<const void*>(wgrad_planes_kernel<true>), kMaxSmem);
      static int max_clusters = -1;
      static size_t max_clusters_smem = 0;
      if (max_clusters < 0 || max_clusters_smem != q.smem) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(q.grid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = q.smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 3;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, wgrad_planes_kernel<true>, &cfg) != cudaSuccess) {
          cudaGetLastError();
          n = 0;
        }
        max_clusters = n;
        max_clusters_smem = q.smem;
      }
      q.grid = 3 * std::min(max_clusters, kNumSMs / 3);
      if (std::getenv("RP_WGRAD_VERBOSE"))
        fprintf(stderr, "wgrad_planes mc: max active clusters %d, grid %d, rg %d, stages %d, smem %zu\n", max_clusters,
                q.grid, q.rg, q.nstages, q.smem);
      if (q.grid > 0 && njobs * (s.co / cbk0) * (s.ci / cbk0) <= q.grid / 3) {
        p = q;
        mc = true;
      }
    }
  }
  const int cbk = single ? 128 : 64;
  PwArgs a{};
  a.single = single ? 1 : 0;
  static const int nobias = std::getenv("RP_WGRAD_NOBIAS") ? 1 : 0;
  a.nobias = nobias;
  static const int wdbg = [] {
    const char* e = std::getenv("RP_WGRAD_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = wdbg;
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = s.w + 2;
  a.rg = p.rg;
  a.P = p.P;
  a.Pp = p.Pp;
  a.nstages = p.nstages;
  a.mo = s.co / cbk;
  a.mi = s.ci / cbk;
  a.blocks_per_img = (s.h + p.rg - 1) / p.rg;
  a.num_blocks = s.n * a.blocks_per_img;
  a.g_slab = p.g_slab;
  a.x_slab = p.x_slab;
  a.x_off = p.x_off;
  a.stage = p.stage;
  a.part = static_cast<float*>(ws);
  a.part_bias = reinterpret_cast<double*>(static_cast<char*>(ws) + part_bytes(p, single));
  a.njobs = njobs;
  // CTAs: every SM (RP_WGRAD_CTAS overrides).  Not shared out among concurrent stages like the
  // convs: the per-CTA partials -- and so the last bits of the gradient -- depend on the grid, and
  // results must not depend on how stages are scheduled (a half grid measured +1.1 % on C3)
  static const int max_ctas = [] {
    const char* e = std::getenv("RP_WGRAD_CTAS");
    const int n = e ? std::atoi(e) : 0;
    return n >= 1 && n <= kNumSMs ? n : kNumSMs;
  }();
  if (!mc) p.grid = std::max(std::min(p.grid, max_ctas), 3 * njobs * a.mo * a.mi);
  if (3 * njobs * a.mo * a.mi > p.grid) fail(RP_ERR_INTERNAL, "conv3x3_wgrad_planes: too many work groups");
  // CTA triples by default (DRAM reads 1.00x algorithmic, C3 +2.7 %); RP_WGRAD_MAP=contiguous
  // restores contiguous CTA ranges per tap group
  static const bool triples = [] {
    const char* e = std::getenv("RP_WGRAD_MAP");
    return !(e && std::string(e) == "contiguous");
  }();
  a.mc = mc ? 1 : 0;
  if (!mc && triples && njobs * a.mo * a.mi <= kNumSMs / 3) {
    a.mc = 2;
    p.grid = 3 * std::max(njobs * a.mo * a.mi, std::min(kNumSMs, max_ctas) / 3);
  }
  const int xrows = mc ? p.rg + 2 : p.rg;
  CUtensorMap m[2][4];   // copies taken under the cache lock
  for (int j = 0; j < njobs; ++j) {
    const WgJob& jb = jobs[j];
    m[j][0] = cached(jb.g0, s.n, s.h, s.w, s.co, p.rg);
    m[j][1] = cached(single ? jb.g0 : jb.g1, s.n, s.h, s.w, s.co, p.rg);
    m[j][2] = cached(jb.x0, s.n, s.h, s.w, s.ci, xrows);
    m[j][3] = cached(single ? jb.x0 : jb.x1, s.n, s.h, s.w, s.ci, xrows);
    a.gw[j] = jb.gw;
    a.gb[j] = jb.gb;
    a.scale[j] = (double)jb.scale;
    a.gsc[j] = jb.gsc;
  }
  if (njobs == 1)
    for (int i = 0; i < 4; ++i) m[1][i] = m[0][i];
  if (mc) {
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(wgrad_planes_kernel<true>), kMaxSmem);
    launch_pdl_cluster(wgrad_planes_kernel<true>, p.grid, kThreads, p.smem, st, 3, m[0][0], m[0][1], m[0][2],
                       m[0][3], m[1][0], m[1][1], m[1][2], m[1][3], a);
  } else {
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(wgrad_planes_kernel<false>), kMaxSmem);
    launch_pdl(wgrad_planes_kernel<false>, p.grid, kThreads, p.smem, st, m[0][0], m[0][1], m[0][2], m[0][3],
               m[1][0], m[1][1], m[1][2], m[1][3], a);
  }
  const int total = njobs * (9 * s.ci * s.co + s.co);
  launch_pdl(wgrad_planes_reduce_kernel, ceil_div(total, 256), 256, 0, st, (const float*)a.part,
             (const double*)a.part_bias, a, p.grid);
}
}  // namespace

void conv3x3_wgrad_planes(const ConvShape& s, const void* x0, const void* x1, const void* g0, const void* g1,
                          float scale, float* gw, float* gb, void* ws, cudaStream_t st, const float* gscale) {
  const WgJob j{x0, x1, g0, g1, scale, gw, gb, gscale};
  launch_wgrad_planes(s, &j, 1, ws, st, false);
}

void conv3x3_wgrad_planes_pair(const ConvShape& s, const void* const xa[2], const void* const ga[2], float scale_a,
                               float* gwa, float* gba, const void* const xb[2], const void* const gb2[2],
                               float scale_b, float* gwb, float* gbb, void* ws, cudaStream_t st, const float* gsc_a,
                               const float* gsc_b) {
  const WgJob j[2] = {{xa[0], xa[1], ga[0], ga[1], scale_a, gwa, gba, gsc_a},
                      {xb[0], xb[1], gb2[0], gb2[1], scale_b, gwb, gbb, gsc_b}};
  launch_wgrad_planes(s, j, 2, ws, st, false);
}

bool conv3x3_wgrad_bf16p_supported(const ConvShape& s) { return plan(s, true).ok; }

int64_t conv3x3_wgrad_bf16p_ws_bytes(const ConvShape& s) {
  const PwPlan p = plan(s, true);
  if (!p.ok) return 0;
  return part_bytes(p, true) + (int64_t)p.grid * 128 * 8 + 256;
}

void conv3x3_wgrad_bf16p(const ConvShape& s, const void* x, const void* g, float scale, float* gw, float* gb,
                         void* ws, cudaStream_t st) {
  const WgJob j{x, nullptr, g, nullptr, scale, gw, gb, nullptr};
  launch_wgrad_planes(s, &j, 1, ws, st, true);
}

bool conv3x3_wgrad_bf16p_pair_supported(const ConvShape& s) {
  const PwPlan p = plan(s, true);
  return p.ok && 2 * 3 * (s.co / 128) * (s.ci / 128) <= p.grid;
}

void conv3x3_wgrad_bf16p_pair(const ConvShape& s, const void* xa, const void* ga, float scale_a, float* gwa,
                              float* gba, const void* xb, const void* gb2, float scale_b, float* gwb, float* gbb,
                              void* ws, cudaStream_t st) {
  const WgJob j[2] = {{xa, nullptr, ga, nullptr, scale_a, gwa, gba, nullptr},
                      {xb, nullptr, gb2, nullptr, scale_b, gwb, gbb, nullptr}};
  launch_wgrad_planes(s, j, 2, ws, st, true);
}

}  // namespace rp::k
