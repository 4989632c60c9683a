// tcgen05 3x3 convolution on fp16 plane pairs with the output POSITIONS as the MMA's M
// (fp32-accurate path, RP_MATH_FP32):
//
//   out[p][co] = epi( sum_{tap, ci} x[p + off(tap)][ci] * w[tap][ci][co] )
//
// (block_forward's matmul(x, W1) / matmul(a, W2) and block_vjp's matmul(upstream, W2^T) /
// matmul(dpre, W1^T), network.cpp:85-104, generalised to 3x3 taps.)
//
// conv_tc.cu puts the output channels on M ([W0; W1] stacked, M = 128 for 64 channels), so the
// x1 plane pays for a W1 x1 product nobody needs: 4 tensor products per fp32 MAC.  Here
//   A = the shifted x-plane halo view, M = 128 frame positions (K-major: [pos][16 ch] in 32-byte
//       rows with the 32B swizzle, one TMA box per plane; a shift by one position is +32 B of
//       start address -- or the [kg][pos][8] interleave conv_tc's B reads, RP_CONV_HALO_SW=0),
//   B = the filter, N = 2 Co rows [W0; W1] for the x0 plane, N = Co rows (W0) for the x1 plane:
// x0 W0 + x0 W1 + x1 W0 is 3 products per MAC (the dropped |W1 x1| <= 2^-24 |W x|, fp32's own
// rounding).  Measured MMA time per tap and 256 positions (tools/umma_bench_pm.py, Co = 64):
// 224.7 cycles against conv_tc's 256.4.  D's row = position, so the epilogue needs no transpose:
// a thread owns one position, adds the W0 and W1 columns, and stores that position's channels.
//
//  * frame, units, halo: as conv_tc.cu (H rows x (W + 1) columns per image; units of two
//    128-position tiles, a shorter tail unit per image; one halo slab per 16-channel chunk
//    serves all 9 taps); the whole prepared filter stays resident in shared memory (Co <= 64).
//  * warp roles (384 threads, persistent, 1 CTA/SM): w0 halo TMA, w1 MMA issuer, w2 filter
//    load, w4-11 two epilogue groups (one tile of each unit each: TMEM -> registers -> W0 + W1,
//    fused bias / tanh / skip / step size -> NHWC stores of the output and its planes through a
//    per-warp swizzled exchange row; the aux operand comes in the same way -- or as 32-byte
//    sector loads / stores of the thread's own position, no exchange: all of them for Co < 64,
//    the plane stores for Co = 64).
//  * CTA pairs (Co = 64 default, see the kernel) and half-GPU grids while several stages run
//    concurrently (conv_pm_set_share) -- DESIGN.md §4.1a.
//  * Co in {16, 32, 64}: config C1's 16-channel network runs on the tensor cores too.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "../common.cuh"
#include "kernels.cuh"
#include "planes.cuh"
#include "umma.cuh"

namespace rp::k {

namespace {

using namespace rp::umma;

constexpr int kThreads = 384;
constexpr int kTile = 128;          // positions per tile (the MMA's M)
constexpr int kS = 2;               // tiles per unit
constexpr int kChunk = 16;          // input channels per halo chunk (one K = 16 step)
constexpr int kMaxSlots = 8;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kPieceBytes = 32 * 1024;   // filter load: bulk copies of <= 32 KB
constexpr int kXchgBytes = 4096;         // per epilogue warp: 32 positions x 32 channels fp32
#ifndef RP_CONV_PAIR_DEFAULT
#define RP_CONV_PAIR_DEFAULT 1              // Co = 64: CTA pairs (measured +1.6 % on C3 over single CTAs) unless RP_CONV_PAIR=0
#endif

struct PmArgs {
  int N, H, W, Ci, Co, Wp, rows_h, T, nchunks, slots;
  int halo_pos;            // positions per halo plane (rows_h x Wp)
  uint32_t plane_bytes;    // one fp16 plane of a chunk's halo: halo_pos x 32 B ([pos][16] or [2 kg][pos][8])
  uint32_t halo_stride;    // bytes per halo slot (pads + two planes)
  uint32_t w_bytes;        // the whole prepared filter
  float h;
  const uint16_t* w;       // prepared filter [chunk][tap][kg 2][2 Co rows][8] fp16 (W * 2^8 pair)
  const float* bias;
  const float* aux;
  float* out;              // null: the planes alone
  uint16_t* p0;            // optional fp16 plane pair of out * (*out_scale)
  uint16_t* p1;
  const float* in_scale;   // the input planes' scale (device scalar; null = kActPlaneScale)
  const float* out_scale;  // the output planes' scale (device scalar; null = kActPlaneScale)
  int sw32;                // halo slab: 32-byte swizzled position rows (1) or the [kg][pos][8] interleave (0)
  int direct;              // epilogue: per-thread 32-byte global accesses of the thread's own position
                           // instead of coalesced ones through the exchange rows, bit mask: 1 aux
                           // loads, 2 fp32 output stores, 4 plane stores
  int dbg;                 // diagnostics (RP_CONV_DBG): 1 no epilogue, 2 no halo TMA, 8 no MMA, 16 no fp32
                           // output stores, 32 no plane stores
};

// Work split: units of kS tiles of one image; T = ceil(frame / 128) tiles per image leaves a
// tail unit when kS does not divide T.  Full units round-robin from CTA 0 up, tail units from
// CTA G - 1 down (every CTA ends within one tile of the mean).
struct Units {
  int f, tl, nf, ntail, fu, T, G;
  // N images (PAIR: image pairs) over G workers (CTAs, PAIR: CTA pairs), this one idx
  __device__ Units(int N, int T_, int idx, int G_) : T(T_), G(G_) {
    fu = T / kS;
    nf = N * fu;
    ntail = (T % kS) ? N : 0;
    f = idx;
    tl = G - 1 - idx;
  }
  __device__ bool next(int& n, int& tile0, int& ntiles) {
    if (f < nf) {
      n = f / fu;
      tile0 = (f - n * fu) * kS;
      ntiles = kS;
      f += G;
      return true;
    }
    if (tl < ntail) {
      n = tl;
      tile0 = fu * kS;
      ntiles = T - tile0;
      tl += G;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ uint4 cat2(uint2 a, uint2 b) { return make_uint4(a.x, a.y, b.x, b.y); }

// 32-byte (one sector) global accesses: a thread moves whole sectors of its own position's row
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, uint4 a, uint4 b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

// PAIR: a cluster of two CTAs (one TPC) runs M = 256 MMAs (cta_group::2): CTA r holds image
// 2 i + r of image pair i at the same frame positions, so both halo slabs sit at the same
// shared-memory offsets and one descriptor serves both A halves; each CTA holds half of B (x0:
// W0 | W1 rows; x1: W0 channels [0, 32) | [32, 64)) -- per CTA 11 KB of operand reads per
// tile and tap instead of 14 KB (the single-CTA form is shared-memory-bandwidth bound).  The
// leader (rank 0) issues every MMA; the peer's TMA completes on the leader's "full" barriers,
// the leader's commits multicast to both CTAs, both epilogues release the leader's accumulators.
template <int EPI, int CO, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    conv3x3_pm_kernel(const __grid_constant__ CUtensorMap tmap, const PmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  static_assert(!PAIR || CO == 64, "CTA-pair form: Co = 64");
  constexpr int kCols = 2 * CO;                                        // accumulator columns per tile
  constexpr int kTmemCols = 2 * kS * kCols < 32 ? 32 : 2 * kS * kCols;  // double-buffered units
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int widx = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;     // worker: CTA or CTA pair
  const int G = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int nitems = PAIR ? (a.N + 1) / 2 : a.N;
  // this CTA's image of work item i
  auto image = [&](int i) { return PAIR ? 2 * i + (int)rank : i; };

  // ---- shared memory: [slots halo slots][filter][barriers]
  // slot: [pad][plane 0][pad][plane 1][pad]; SW32: 256-byte aligned planes (the swizzle atom)
  const uint32_t al = a.sw32 ? 256u : 128u;
  const uint32_t plane_pitch = ((a.plane_bytes + al - 1) & ~(al - 1)) + al;
  auto plane = [&](int s, int p) { return smem + s * a.halo_stride + al + p * plane_pitch; };
  uint8_t* wres = smem + a.slots * a.halo_stride;
  uint8_t* xchg = wres + a.w_bytes;                                    // [8 epilogue warps][kXchgBytes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xchg + 8 * kXchgBytes);
  uint64_t* halo_full = bars;                    // [kMaxSlots]
  uint64_t* halo_empty = bars + kMaxSlots;       // [kMaxSlots]
  uint64_t* w_full = bars + 2 * kMaxSlots;       // [1]
  uint64_t* acc_full = bars + 2 * kMaxSlots + 1; // [2]
  uint64_t* acc_empty = bars + 2 * kMaxSlots + 3;  // [2]
  uint64_t* w_peer = bars + 2 * kMaxSlots + 5;     // PAIR (leader): the peer's filter landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxSlots + 6);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxSlots; ++i) {
      mbar_init(&halo_full[i], 1);
      mbar_init(&halo_empty[i], 1);
    }
    mbar_init(w_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], PAIR ? 16 : 8);   // one arrival per epilogue warp (PAIR: of both CTAs)
    }
    mbar_init(w_peer, 1);
    fence_barrier_init();
    prefetch_tmap(&tmap);
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair<kTmemCols>(tmem_slot);
    else tmem_alloc<kTmemCols>(tmem_slot);
  }
  // zero the 128-byte pads in front of / behind the planes (read only for discarded positions)
  for (int i = threadIdx.x; i < a.slots * 3 * 32; i += blockDim.x) {
    const int s = i / 96, part = (i / 32) % 3, w = i % 32;
    uint8_t* base = part == 0 ? plane(s, 0) - 128 : plane(s, part - 1) + a.plane_bytes;
    reinterpret_cast<uint32_t*>(base)[w] = 0u;
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();   // barrier inits visible to the peer before any remote arrival
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int Wp = a.Wp;
  pdl_launch_dependents();

  if (warp == 2) {
    // ===================== resident filter =====================
    // issued before pdl_wait(): the prepared filter comes from a kernel that completed before
    // the previous grid did (conv_tc.cu, same argument)
    if (elect_one()) {
      mbar_arrive_expect_tx(w_full, a.w_bytes);
      if constexpr (PAIR) {
        // this CTA's halves of B out of the standard prepared filter ([chunk][tap][kg][128 rows][8]):
        // per (chunk, tap) [x0 half: kg x 64 rows][x1 half: kg x 32 rows] = 3 KB
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.w);
        for (int ct = 0; ct < a.nchunks * 9; ++ct) {
          const uint8_t* sct = src + ct * 4096;
          uint8_t* dct = wres + ct * 3072;
          bulk_load(dct, sct + rank * 1024, 1024, w_full);                   // kg 0, rows [64 r, +64)
          bulk_load(dct + 1024, sct + 2048 + rank * 1024, 1024, w_full);     // kg 1
          bulk_load(dct + 2048, sct + rank * 512, 512, w_full);              // kg 0, W0 rows [32 r, +32)
          bulk_load(dct + 2560, sct + 2048 + rank * 512, 512, w_full);       // kg 1
        }
      } else {
        for (uint32_t o = 0; o < a.w_bytes; o += kPieceBytes)
          bulk_load(wres + o, reinterpret_cast<const uint8_t*>(a.w) + o, min((uint32_t)kPieceBytes, a.w_bytes - o),
                    w_full);
      }
    }
    __syncwarp();
    if (PAIR && !leader) {   // tell the leader (which issues the pair's MMAs) that this half landed
      mbar_wait(w_full, 0);
      if (elect_one()) mbar_arrive_cluster(w_peer, 0);
      __syncwarp();
    }
  } else if (warp == 0) {
    // ===================== halo TMA producer =====================
    pdl_wait();
    int hs = 0;
    uint32_t hph = 0;
    Units it(nitems, a.T, widx, G);
    int item, tile0, ntiles;
    while (it.next(item, tile0, ntiles)) {
      const int y0 = tile0 * kTile / Wp;
      const int n = image(item);   // PAIR, odd N: the last peer loads finite filler, stores nothing
      for (int c = 0; c < a.nchunks; ++c) {
        mbar_wait(&halo_empty[hs], hph ^ 1);
        if (elect_one()) {
          if (a.dbg & 2) {
            if (leader) mbar_arrive(&halo_full[hs]);
          } else if constexpr (PAIR) {
            // both CTAs' bytes complete on the leader's barrier
            const uint32_t bar = cluster_addr(&halo_full[hs], 0);
            if (leader) mbar_arrive_expect_tx(&halo_full[hs], 4 * a.plane_bytes);
            if (a.sw32) {
              tma_load_4d_pair(&tmap, bar, plane(hs, 0), kChunk * c, -1, y0 - 1, n);
              tma_load_4d_pair(&tmap, bar, plane(hs, 1), kChunk * c, -1, y0 - 1, n + a.N);
            } else {
              tma_load_5d_pair(&tmap, bar, plane(hs, 0), 0, -1, y0 - 1, 2 * c, n);
              tma_load_5d_pair(&tmap, bar, plane(hs, 1), 0, -1, y0 - 1, 2 * c, n + a.N);
            }
          } else {
            // both planes of the chunk: images [0, N) are plane 0, [N, 2N) plane 1
            mbar_arrive_expect_tx(&halo_full[hs], 2 * a.plane_bytes);
            if (a.sw32) {   // 32-byte box rows (16 channels), 32B-swizzled: half the TMA row count
              tma_load_4d(&tmap, &halo_full[hs], plane(hs, 0), kChunk * c, -1, y0 - 1, n);
              tma_load_4d(&tmap, &halo_full[hs], plane(hs, 1), kChunk * c, -1, y0 - 1, n + a.N);
            } else {
              tma_load_5d(&tmap, &halo_full[hs], plane(hs, 0), 0, -1, y0 - 1, 2 * c, n);
              tma_load_5d(&tmap, &halo_full[hs], plane(hs, 1), 0, -1, y0 - 1, 2 * c, n + a.N);
            }
          }
        }
        __syncwarp();
        if (++hs == a.slots) hs = 0, hph ^= 1;
      }
    }
  } else if (warp == 1 && !leader) {
    mbar_wait(w_full, 0);   // the peer's MMA warp: nothing to issue; no exit with the filter load in flight
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t id_x0 = idesc(0, PAIR ? 256 : 128, kCols);   // x0 x [W0; W1]
    const uint32_t id_x1 = idesc(0, PAIR ? 256 : 128, CO);      // x1 x W0
    const uint32_t lbo_x = (uint32_t)a.halo_pos * 16u;
    // filter slices: single CTA [kg][2 Co rows][8] per (chunk, tap); PAIR [x0: kg x Co rows | x1: kg x Co / 2 rows]
    const uint32_t lbo_w = PAIR ? (uint32_t)CO * 16u : (uint32_t)kCols * 16u;
    const uint32_t lbo_w1 = PAIR ? (uint32_t)CO * 8u : lbo_w;
    const uint32_t w_tap = PAIR ? (uint32_t)CO * 48u : (uint32_t)kCols * 32u;
    const uint32_t w_x1 = PAIR ? (uint32_t)CO * 32u : 0u;   // offset of the x1 half in a slice
    int hs = 0, ab = 0;
    uint32_t hph = 0, aph = 0;
    mbar_wait(w_full, 0);   // unconditionally: no CTA may exit with the filter load in flight
    if (PAIR) mbar_wait_cluster(w_peer, 0);
    tc_fence_after();
    Units it(nitems, a.T, widx, G);
    int item, tile0, ntiles;
    while (it.next(item, tile0, ntiles)) {
      const int f0 = tile0 * kTile;
      const int c0 = f0 - (f0 / Wp) * Wp;
      if (PAIR) mbar_wait_cluster(&acc_empty[ab], aph ^ 1);
      else mbar_wait(&acc_empty[ab], aph ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + (uint32_t)(ab * kS * kCols);
      for (int c = 0; c < a.nchunks; ++c) {
        mbar_wait(&halo_full[hs], hph);
        tc_fence_after();
        // K-major A: interleave ([kg][pos][8], one position = 16 B) or SW32 ([pos][16] in 32-byte
        // swizzled rows, 8-row atoms 256 B apart; one position = 32 B): the start shifts by whole rows
        // (the swizzle follows the absolute address bits, as the TMA wrote it)
        const uint64_t ax0 = a.sw32 ? desc_general(smem_u32(plane(hs, 0)), 16, 256, 6, 0)
                                    : desc_kmajor_interleave(smem_u32(plane(hs, 0)), lbo_x, 128);
        const uint64_t ax1 = a.sw32 ? desc_general(smem_u32(plane(hs, 1)), 16, 256, 6, 0)
                                    : desc_kmajor_interleave(smem_u32(plane(hs, 1)), lbo_x, 128);
        const int pstep = a.sw32 ? 2 : 1;   // 16-byte units per position
        if (elect_one() && !(a.dbg & 8)) {
          for (int dy = 0; dy < 3; ++dy) {
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
              const uint32_t wsl = smem_u32(wres + (uint32_t)(c * 9 + 3 * dy + dx) * w_tap);
              const uint64_t db = desc_kmajor_interleave(wsl, lbo_w, 128);
              const uint64_t db1 = desc_kmajor_interleave(wsl + w_x1, lbo_w1, 128);
              const int64_t row = c0 + dy * Wp + dx - 1;    // halo position of the tile's first row, >= -1
              const uint32_t accum = (c == 0 && dy == 0 && dx == 0) ? 0u : 1u;
#pragma unroll
              for (int s = 0; s < kS; ++s) {
                if (s < ntiles) {
                  const uint64_t ao = (uint64_t)((row + s * kTile) * pstep);   // 16-byte units
                  if constexpr (PAIR) {
                    mma_f16_pair(d0 + s * kCols, ax0 + ao, db, id_x0, accum);
                    mma_f16_pair(d0 + s * kCols, ax1 + ao, db1, id_x1, 1u);
                  } else {
                    mma_f16(d0 + s * kCols, ax0 + ao, db, id_x0, accum);
                    mma_f16(d0 + s * kCols, ax1 + ao, db1, id_x1, 1u);
                  }
                }
              }
            }
          }
        }
        __syncwarp();
        if (elect_one()) {
          if constexpr (PAIR) mma_commit_pair(&halo_empty[hs], 3);
          else mma_commit(&halo_empty[hs]);
        }
        __syncwarp();
        if (++hs == a.slots) hs = 0, hph ^= 1;
      }
      if (elect_one()) {
        if constexpr (PAIR) mma_commit_pair(&acc_full[ab], 3);
        else mma_commit(&acc_full[ab]);
      }
      __syncwarp();
      if (++ab == 2) ab = 0, aph ^= 1;
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    // group g (warps 4 + 4g .. 7 + 4g) drains tile g of every unit; warp w reads TMEM lane
    // quadrant w % 4: thread = position q * 32 + lane of the tile, columns [0, Co) = W0
    // products, [Co, 2 Co) = W1 products of the same output channels.
    pdl_wait();
    const int q = warp & 3;
    const int grp = (warp - 4) >> 2;
    const int pt = q * 32 + lane;
    constexpr bool kBias = EPI == EPI_BIAS || EPI == EPI_BIAS_TANH || EPI == EPI_RESID;
    constexpr bool kAux = EPI == EPI_RESID || EPI == EPI_TANH_BWD || EPI == EPI_ADD;
    const float acc_mul = kWeightPlaneScaleInv / (a.in_scale ? *a.in_scale : kActPlaneScale);
    const float out_mul = a.out_scale ? *a.out_scale : kActPlaneScale;
    const bool planes = a.p0 != nullptr;
    constexpr int kCh = CO < 32 ? CO : 32;      // channels per exchange pass
    constexpr int kNJ = kCh / 4;                // 16-byte pieces per position and pass
    float4* xrow = reinterpret_cast<float4*>(xchg + (warp - 4) * kXchgBytes);
    // the bias in shared memory: a warp-uniform LDS.128 per 4 channels instead of an LDG per
    // channel and position
    float* sbias = reinterpret_cast<float*>(bars + 2 * kMaxSlots + 8);
    if constexpr (kBias) {
      if (threadIdx.x - 128 < (unsigned)CO) sbias[threadIdx.x - 128] = a.bias[threadIdx.x - 128];
      asm volatile("bar.sync 1, 256;" ::: "memory");   // the 8 epilogue warps
    }
    int ab = 0;
    uint32_t aph = 0;
    Units it(nitems, a.T, widx, G);
    int item, tile0, ntiles;
    while (it.next(item, tile0, ntiles)) {
      const int n = image(item);
      const int f = (tile0 + grp) * kTile + pt;
      const int y = f / Wp, X = f - y * Wp;
      const bool valid = grp < ntiles && y < a.H && X >= 1 && n < a.N;
      const int64_t off = valid ? (((int64_t)n * a.H + y) * a.W + (X - 1)) * CO : 0;
      // the tile's aux operand first, coalesced (instruction k: kPW consecutive positions of the
      // warp as whole contiguous rows, 16-byte piece lane % kPR), its latency overlapping the
      // wait for the accumulator; each pass moves its pieces to thread = position through the
      // warp's exchange rows
      constexpr int kPR = CO / 4;       // 16-byte pieces per position row
      constexpr int kPW = 32 / kPR;     // positions per load instruction
      float4 ax[kAux ? kPR : 1];
      if constexpr (kAux) {
        if (a.direct & 1) {
#pragma unroll
          for (int k = 0; k < kPR; k += 2) {
            if (valid) ldg256(a.aux + off + 4 * k, ax[k], ax[k + 1]);
            else ax[k] = ax[k + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else
#pragma unroll
        for (int k = 0; k < kPR; ++k) {
          const int src = k * kPW + lane / kPR, j = lane % kPR;
          const int64_t so = __shfl_sync(0xffffffffu, off, src);
          const bool sv = __shfl_sync(0xffffffffu, (int)valid, src) != 0;
          ax[k] = sv ? __ldg(reinterpret_cast<const float4*>(a.aux + so) + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      mbar_wait(&acc_full[ab], aph);
      tc_fence_after();
      const bool live = grp < ntiles && !(a.dbg & 1);
      const uint32_t tcol = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * kS * kCols + grp * kCols);
#pragma unroll
      for (int hf = 0; hf < CO / kCh; ++hf) {
        // this position's kCh channels [hf kCh, +kCh): W0 + W1 columns, scaled
        float o[kCh];
        if (live) {
#pragma unroll
          for (int cc = 0; cc < kCh / 16; ++cc) {
            uint32_t hi[16], lo[16];
            tmem_ld16(tcol + hf * kCh + cc * 16, hi);
            tmem_ld16(tcol + CO + hf * kCh + cc * 16, lo);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i)
              o[cc * 16 + i] = (__uint_as_float(hi[i]) + __uint_as_float(lo[i])) * acc_mul;
          }
        }
        if (hf == CO / kCh - 1) {   // every accumulator is in registers: the buffer goes back to the MMA
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR) mbar_arrive_cluster_relaxed(&acc_empty[ab], 0);   // the leader's accumulators
            else mbar_arrive_relaxed(&acc_empty[ab]);
          }
        }
        if (!live) continue;
        float4 xa[kAux ? kNJ : 1];
        float bq[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (kAux) {
          if (a.direct & 1) {
#pragma unroll
            for (int j = 0; j < kNJ; ++j) xa[j] = ax[hf * kNJ + j];
          } else {
#pragma unroll
          for (int k = 0; k < kPR; ++k) {
            const int j = lane % kPR;
            if (j / kNJ == hf) {
              const int src = k * kPW + lane / kPR, jj = j - hf * kNJ;
              xrow[src * kNJ + (jj ^ (src & (kNJ - 1)))] = ax[k];
            }
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < kNJ; ++j) xa[j] = xrow[lane * kNJ + (j ^ (lane & (kNJ - 1)))];
          __syncwarp();
          }
        }
        {
#pragma unroll
          for (int i = 0; i < kCh; ++i) {
            const float v = o[i];
            const float xa_i = kAux ? reinterpret_cast<const float*>(&xa[0])[i] : 0.f;
            float bco = 0.f;
            if constexpr (kBias) {
              if ((i & 3) == 0) {
                const float4 b4 = reinterpret_cast<const float4*>(sbias)[(hf * kCh + i) / 4];
                bq[0] = b4.x, bq[1] = b4.y, bq[2] = b4.z, bq[3] = b4.w;
              }
              bco = bq[i & 3];
            }
            float r;
            if constexpr (EPI == EPI_BIAS) r = v + bco;
            else if constexpr (EPI == EPI_BIAS_TANH) r = tanhf(v + bco);
            else if constexpr (EPI == EPI_RESID) r = xa_i + a.h * (v + bco);
            else if constexpr (EPI == EPI_TANH_BWD) r = (a.h * v) * (1.f - xa_i * xa_i);
            else if constexpr (EPI == EPI_ADD) r = xa_i + v;
            else r = a.h * v;
            o[i] = r;
          }
          // stores: per thread (its position's kCh channels as 32-byte sectors), or through the
          // warp's exchange rows (thread = position -> kNJ 16-byte pieces of consecutive positions
          // per instruction: 32 / kNJ positions x kCh * 4 bytes contiguous; 16-byte slots
          // XOR-swizzled by position, conflict-free both ways)
          if (a.direct & 2) {
            if (valid && a.out && !(a.dbg & 16)) {
#pragma unroll
              for (int j = 0; j < kCh / 8; ++j)
                stg256(a.out + off + hf * kCh + 8 * j,
                       make_uint4(__float_as_uint(o[8 * j]), __float_as_uint(o[8 * j + 1]),
                                  __float_as_uint(o[8 * j + 2]), __float_as_uint(o[8 * j + 3])),
                       make_uint4(__float_as_uint(o[8 * j + 4]), __float_as_uint(o[8 * j + 5]),
                                  __float_as_uint(o[8 * j + 6]), __float_as_uint(o[8 * j + 7])));
            }
          } else if (a.out && !(a.dbg & 16)) {
#pragma unroll
            for (int j = 0; j < kNJ; ++j)
              xrow[lane * kNJ + (j ^ (lane & (kNJ - 1)))] =
                  make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kNJ; ++k) {
              const int src = k * (32 / kNJ) + lane / kNJ, j = lane % kNJ;
              const float4 v = xrow[src * kNJ + (j ^ (src & (kNJ - 1)))];
              const int64_t so = __shfl_sync(0xffffffffu, off, src);
              if (__shfl_sync(0xffffffffu, (int)valid, src))
                *reinterpret_cast<float4*>(a.out + so + hf * kCh + 4 * j) = v;
            }
            __syncwarp();
          }
          if (a.direct & 4) {
            if (valid && planes && !(a.dbg & 32)) {
#pragma unroll
              for (int j = 0; j < kCh / 16; ++j) {
                uint2 h0[4], h1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const float v4[4] = {o[16 * j + 4 * u], o[16 * j + 4 * u + 1], o[16 * j + 4 * u + 2],
                                       o[16 * j + 4 * u + 3]};
                  pack_pair4(v4, out_mul, h0[u], h1[u]);
                }
                stg256(a.p0 + off + hf * kCh + 16 * j, cat2(h0[0], h0[1]), cat2(h0[2], h0[3]));
                stg256(a.p1 + off + hf * kCh + 16 * j, cat2(h1[0], h1[1]), cat2(h1[2], h1[3]));
              }
            }
          } else if (planes && !(a.dbg & 32)) {
            // [p0 | p1] of the kCh channels: kNJ / 2 16-byte pieces each
#pragma unroll
            for (int j = 0; j < kNJ / 2; ++j) {
              uint2 h0a, h1a, h0b, h1b;
              const float va[4] = {o[8 * j], o[8 * j + 1], o[8 * j + 2], o[8 * j + 3]};
              const float vb[4] = {o[8 * j + 4], o[8 * j + 5], o[8 * j + 6], o[8 * j + 7]};
              pack_pair4(va, out_mul, h0a, h1a);
              pack_pair4(vb, out_mul, h0b, h1b);
              const uint4 u0 = cat2(h0a, h0b), u1 = cat2(h1a, h1b);
              xrow[lane * kNJ + (j ^ (lane & (kNJ - 1)))] = *reinterpret_cast<const float4*>(&u0);
              xrow[lane * kNJ + ((j + kNJ / 2) ^ (lane & (kNJ - 1)))] = *reinterpret_cast<const float4*>(&u1);
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kNJ; ++k) {
              const int src = k * (32 / kNJ) + lane / kNJ, j = lane % kNJ;
              const float4 v = xrow[src * kNJ + (j ^ (src & (kNJ - 1)))];
              const int64_t so = __shfl_sync(0xffffffffu, off, src);
              uint16_t* dst = j < kNJ / 2 ? a.p0 + so + hf * kCh + 8 * j : a.p1 + so + hf * kCh + 8 * (j - kNJ / 2);
              if (__shfl_sync(0xffffffffu, (int)valid, src)) *reinterpret_cast<float4*>(dst) = v;
            }
            __syncwarp();
          }
        }
      }
      if (++ab == 2) ab = 0, aph ^= 1;
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();   // the peer's TMEM holds MMA results until both are done
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair<kTmemCols>(tmem_base);
    else tmem_dealloc<kTmemCols>(tmem_base);
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

// fp16 planes [2][N][H][W][Ci] viewed as 2N images of 8-channel groups; box {8 ch, W + 1
// columns from x = -1, rows_h rows from y0 - 1, 2 groups, 1 image} = the slot layout
// [2 kg][positions][8], out-of-bounds rows / columns zero-filled
CUtensorMap make_map(const void* planes, const ConvShape& s, int Wp, int rows_h, bool sw32) {
  CUtensorMap m;
  CUresult r;
  if (sw32) {
    // [2N][H][W][Ci] fp16, box {16 ch, W + 1 columns from x = -1, rows_h rows, 1 image}, 32B swizzle
    const cuuint64_t dims[4] = {(cuuint64_t)s.ci, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)(2 * s.n)};
    const cuuint64_t strides[3] = {(cuuint64_t)s.ci * 2, (cuuint64_t)s.w * s.ci * 2, (cuuint64_t)s.h * s.w * s.ci * 2};
    const cuuint32_t box[4] = {16, (cuuint32_t)Wp, (cuuint32_t)rows_h, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(planes), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[5] = {8, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)(s.ci / 8), (cuuint64_t)(2 * s.n)};
    const cuuint64_t strides[4] = {(cuuint64_t)s.ci * 2, (cuuint64_t)s.w * s.ci * 2, 16,
                                   (cuuint64_t)s.h * s.w * s.ci * 2};
    const cuuint32_t box[5] = {8, (cuuint32_t)Wp, (cuuint32_t)rows_h, 2, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void*>(planes), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

std::mutex g_map_mu;
std::map<std::tuple<const void*, int, int, int, int, int, bool>, CUtensorMap> g_maps;

CUtensorMap cached_map(const void* in, const ConvShape& s, int Wp, int rows_h, bool sw32) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto key = std::make_tuple(in, s.n, s.h, s.w, s.ci, rows_h, sw32);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();   // callers hold copies, never references
    it = g_maps.emplace(key, make_map(in, s, Wp, rows_h, sw32)).first;
  }
  return it->second;
}

struct Plan {
  bool ok = false;
  bool sw32 = true;    // halo slab in 32-byte swizzled rows (RP_CONV_HALO_SW=0: the 16-byte interleave)
  bool pair = false;   // CTA-pair form (Co = 64)
  int Wp, rows_h, halo_pos, T, slots;
  uint32_t plane_bytes, halo_stride, w_bytes;
  size_t smem;
};

Plan plan_for(const ConvShape& s, bool allow_pair = true) {
  Plan p;
  if (!(s.co == 16 || s.co == 32 || s.co == 64) || s.ci % kChunk != 0 || s.ci <= 0 || s.w + 1 > 256) return p;
  p.Wp = s.w + 1;
  // a tile's A view reaches rows [c0 - 1, c0 + 2 Wp + 1 + 255] of the halo (c0 < Wp)
  p.rows_h = (3 * p.Wp + kS * kTile + p.Wp - 1) / p.Wp;
  if (p.rows_h > 256) return p;
  p.halo_pos = p.rows_h * p.Wp;
  p.T = (s.h * p.Wp + kTile - 1) / kTile;
  p.plane_bytes = (uint32_t)p.halo_pos * 32u;
  static const bool sw_on = [] {
    const char* e = std::getenv("RP_CONV_HALO_SW");
    return !(e && e[0] == '0');
  }();
  p.sw32 = sw_on;
  const uint32_t al = p.sw32 ? 256u : 128u;
  const uint32_t pitch = ((p.plane_bytes + al - 1) & ~(al - 1)) + al;
  p.halo_stride = al + 2u * pitch;
  static const bool pair_on = [] {
    const char* e = std::getenv("RP_CONV_PAIR");
    return e ? e[0] != '0' : RP_CONV_PAIR_DEFAULT != 0;
  }();
  p.pair = allow_pair && pair_on && s.co == 64;
  // per CTA: the whole filter, or (PAIR) its halves of B -- 3/4 of it
  p.w_bytes = (uint32_t)(s.ci / kChunk) * 9u * (uint32_t)(2 * s.co) * 32u * (p.pair ? 3u : 4u) / 4u;
  const size_t fixed = 8 * kXchgBytes + 1024;   // epilogue exchange, barriers, TMEM slot
  for (int sl = kMaxSlots; sl >= 2 && !p.ok; --sl) {
    const size_t need = (size_t)sl * p.halo_stride + p.w_bytes + fixed;
    if (need <= (size_t)kMaxSmem) p.slots = sl, p.smem = need, p.ok = true;
  }
  return p;
}

// co-resident CTA pairs of the pair kernel at this shared-memory size (normally every TPC: 74;
// 0 where clusters of two do not fit -- the launch then falls back to single CTAs)
template <int EPI>
int max_pairs(size_t smem) {
  static std::mutex mu;
  static std::map<size_t, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(smem);
  if (it == cache.end()) {
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(conv3x3_pm_kernel<EPI, 64, true>), kMaxSmem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kNumSMs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, conv3x3_pm_kernel<EPI, 64, true>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    it = cache.emplace(smem, n).first;
  }
  return it->second;
}

int max_pairs_epi(int epi, size_t smem) {
  switch (epi) {
    case EPI_BIAS: return max_pairs<EPI_BIAS>(smem);
    case EPI_BIAS_TANH: return max_pairs<EPI_BIAS_TANH>(smem);
    case EPI_RESID: return max_pairs<EPI_RESID>(smem);
    case EPI_TANH_BWD: return max_pairs<EPI_TANH_BWD>(smem);
    case EPI_ADD: return max_pairs<EPI_ADD>(smem);
    default: return max_pairs<EPI_SCALE>(smem);
  }
}

thread_local int t_share = 1;   // stages issuing concurrently on this GPU (conv_pm_set_share)

// CTAs per launch: every SM, or a share of them while `t_share` stages run concurrently, so
// several stages' convs run side by side and one's fill and drain overlap the others' steady
// state: SMs / max(2, ways / 2) -- measured on finite data: 4 stages best at 74 CTAs, 8 stages
// at 30-40; RP_CONV_PM_CTAS overrides
int max_ctas() {
  static const int env = [] {
    const char* e = std::getenv("RP_CONV_PM_CTAS");
    const int n = e ? std::atoi(e) : 0;
    return n >= 2 && n <= kNumSMs ? n : 0;
  }();
  if (env) return env;
  return t_share >= 2 ? kNumSMs / std::max(2, t_share / 2) : kNumSMs;
}

template <int EPI, int CO, bool PAIR>
void launch_co(const CUtensorMap& m, const PmArgs& a, size_t smem, int units, cudaStream_t st) {
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(conv3x3_pm_kernel<EPI, CO, PAIR>), kMaxSmem);
  if constexpr (PAIR) {
    const int pairs = max_pairs<EPI>(smem);
    if (pairs < 1) fail(RP_ERR_INTERNAL, "conv3x3_fwd_pm: no CTA pair fits");
    const int grid = 2 * std::min(units, std::min(pairs, max_ctas() / 2));
    launch_pdl_cluster(conv3x3_pm_kernel<EPI, CO, PAIR>, grid, kThreads, smem, st, 2, m, a);
  } else {
    launch_pdl(conv3x3_pm_kernel<EPI, CO, PAIR>, std::min(units, max_ctas()), kThreads, smem, st, m, a);
  }
}

template <int EPI>
void launch_epi(const CUtensorMap& m, const PmArgs& a, size_t smem, int units, bool pair, cudaStream_t st) {
  if (a.Co == 64 && pair)
    launch_co<EPI, 64, true>(m, a, smem, units, st);
  else if (a.Co == 64)
    launch_co<EPI, 64, false>(m, a, smem, units, st);
  else if (a.Co == 32)
    launch_co<EPI, 32, false>(m, a, smem, units, st);
  else
    launch_co<EPI, 16, false>(m, a, smem, units, st);
}

}  // namespace

bool conv3x3_pm_supported(const ConvShape& s) { return plan_for(s).ok; }

void conv_pm_set_share(int ways) { t_share = ways < 1 ? 1 : ways; }
int conv_pm_share() { return t_share; }

void conv3x3_fwd_pm(const ConvShape& s, const float* w_hwio, bool dgrad_weights, const float* bias, const float* aux,
                    float h, int epi, float* out, void* ws, cudaStream_t st, void* out_planes, const void* in_planes,
                    const void* wprep, const float* in_scale, const float* out_scale) {
  if (s.pixels() == 0) return;
  Plan p = plan_for(s);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_fwd_pm: unsupported shape");
  if (p.pair && max_pairs_epi(epi, p.smem) < 1) p = plan_for(s, false);   // no co-resident pairs: single CTAs
  if (!in_planes) fail(RP_ERR_INTERNAL, "conv3x3_fwd_pm: needs plane input");
  if (!wprep) {   // the filter of this conv alone (a stage prepares all of its filters at once)
    prep_filter_planes(w_hwio, dgrad_weights ? s.co : s.ci, dgrad_weights ? s.ci : s.co, dgrad_weights, ws, st);
    wprep = ws;
  }
  PmArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = p.Wp;
  a.rows_h = p.rows_h;
  a.T = p.T;
  a.nchunks = s.ci / kChunk;
  a.slots = p.slots;
  a.halo_pos = p.halo_pos;
  a.plane_bytes = p.plane_bytes;
  a.halo_stride = p.halo_stride;
  a.w_bytes = p.w_bytes;
  a.h = h;
  a.w = static_cast<const uint16_t*>(wprep);
  a.bias = bias;
  a.aux = aux;
  a.out = out;
  a.p0 = static_cast<uint16_t*>(out_planes);
  a.p1 = out_planes ? a.p0 + s.pixels() * s.co : nullptr;
  a.in_scale = in_scale;
  a.out_scale = out_scale;
  static const int dbg = [] {
    const char* e = std::getenv("RP_CONV_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
  // epilogue global accesses: per-thread sectors for Co < 64 (C1: +6 %); for Co = 64 the plane
  // stores alone (C2 / C3 +0.8-1 %; all three per thread: -1-1.5 %; profiles/r02_pm_direct.txt);
  // RP_CONV_PM_DIRECT=<mask 0..7> forces a choice (1 aux loads, 2 fp32 stores, 4 plane stores)
  static const int direct_env = [] {
    const char* e = std::getenv("RP_CONV_PM_DIRECT");
    return e ? (std::atoi(e) & 7) : -1;
  }();
  a.direct = direct_env >= 0 ? direct_env : (s.co < 64 ? 7 : 4);
  // 32-byte accesses need 32-byte aligned rows (C-ABI callers may pass any 16-byte aligned view)
  auto a32 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 31u) == 0; };
  if (!a32(aux)) a.direct &= ~1;
  if (!a32(out)) a.direct &= ~2;
  if (!a32(a.p0) || !a32(a.p1)) a.direct &= ~4;
  a.sw32 = p.sw32 ? 1 : 0;
  const CUtensorMap m = cached_map(in_planes, s, p.Wp, p.rows_h, p.sw32);
  // work items: units of one image, or (PAIR) of an image pair
  const int units = (p.pair ? (s.n + 1) / 2 : s.n) * ((p.T + kS - 1) / kS);
  switch (epi) {
    case EPI_BIAS: launch_epi<EPI_BIAS>(m, a, p.smem, units, p.pair, st); break;
    case EPI_BIAS_TANH: launch_epi<EPI_BIAS_TANH>(m, a, p.smem, units, p.pair, st); break;
    case EPI_RESID: launch_epi<EPI_RESID>(m, a, p.smem, units, p.pair, st); break;
    case EPI_TANH_BWD: launch_epi<EPI_TANH_BWD>(m, a, p.smem, units, p.pair, st); break;
    case EPI_ADD: launch_epi<EPI_ADD>(m, a, p.smem, units, p.pair, st); break;
    default: launch_epi<EPI_SCALE>(m, a, p.smem, units, p.pair, st); break;
  }
  RP_LAUNCHED();
}

}  // namespace rp::k
