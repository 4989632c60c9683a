// tcgen05 implicit-GEMM 3x3 convolution with bf16 operands and fp32 accumulation
// (RP_MATH_BF16, config C5: "BF16 tensor-core conv path with fp32 accumulation").
//
//   out[p][co] = epi( sum_{tap, ci} bf16(in[p + off(tap)][ci]) * bf16(w[tap][ci][co]) )
//
// Same structure as conv_tc.cu (interior-frame halo, taps as shifted UMMA descriptors,
// weights as the shared A operand, persistent warp-specialised CTAs), re-tiled for
// kind::f16: M = 128 output channels per block (no hi / lo stacking), K = 16 channels
// per MMA, 32-channel halo chunks, one N <= 256 MMA per (unit, tap, k-step).
//  * fp32-input mode: TMA brings the fp32 halo, converter warps round it to bf16 (RNE) into
//    the K-major interleaved layout the MMA reads; 2 fp32 + 2 bf16 halo slots, 3 weight
//    stages; one epilogue group, a channel per lane.
//  * bf16-input (tape) mode, BIN: the input is a bf16 tensor loaded by TMA straight into the
//    MMA layout (the values the converters would produce); 4 bf16 halo slots, 5 weight
//    stages; the converter warps form a second epilogue group and the epilogue is transposed
//    through shared memory (a thread owns 4 channels of a position: 16-byte fp32 / 8-byte
//    bf16 accesses).  Optional bf16 outputs: out16 = bf16(out), out16d = bf16(1 - out^2).
// The epilogue applies the fused bias / tanh / skip / (1 - a^2) / step size of the fp32
// kernel on fp32 accumulators.  TMEM: 2 units x 2 tiles x 128 columns.
#include <cuda.h>
#include <cuda_bf16.h>

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
constexpr int kWStages = 3;          // weight ring depth, fp32-input mode
constexpr int kBfMax = 4;            // bf16 halo slots, max (bf16-input mode)
constexpr int kWMax = 6;             // weight ring depth, max
constexpr int kChunk = 32;           // input channels per halo chunk
constexpr int kS = 2;                // 128-position tiles per unit
constexpr int kMaxSmem = 227 * 1024;

struct BfArgs {
  int N, H, W, Ci, Co, Wp, rows_h, T, halo_pos, nchunks;
  uint32_t raw_bytes;   // fp32 halo chunk: [8 groups][positions][4 ch]
  uint32_t raw_stride;  // bytes per fp32 slot
  uint32_t bf_bytes;    // bf16 halo chunk: [4 kg][positions][8 ch]
  uint32_t bf_stride;   // bytes per bf16 slot (with zero pads before / after)
  uint32_t w_tap;       // bytes of one tap's A operand: 4 kg x 128 rows x 16 B
  int nbf, nw;          // bf16 halo slots, weight ring depth
  float h;
  const __nv_bfloat16* w;   // prepped [cb][chunk][tap][kg][128 rows][8]
  const float* bias;
  const float* aux;
  const __nv_bfloat16* aux16;   // EPI_DTANH16: bf16(1 - a^2)
  float* out;                   // may be null (bf16 tape outputs only)
  __nv_bfloat16* out16;         // optional bf16 copy of out (the bf16 wgrad's operand)
  __nv_bfloat16* out16d;        // optional bf16(1 - out^2)
  int sw64;                     // BIN: the halo slab in 64-byte 64B-swizzled rows ([pos][32 ch]), else [kg][pos][8]
  int dbg;                      // diagnostics (RP_BF16_DBG): 1 no aux loads, 2 no stores
};

// Work split as in conv_tc.cu: full kS-tile units round-robin from CTA 0, the per-image
// tail units from CTA G-1 downwards; the 128-channel output block cb is outermost.
struct UnitIter {
  int f, tl, nf, ntail, fu, T, NT, G;
  __device__ UnitIter(int mtiles, int N, int T_) : T(T_) {
    G = gridDim.x;
    fu = T / kS;
    nf = mtiles * N * fu;
    ntail = (T % kS) ? mtiles * N : 0;
    NT = N;
    f = blockIdx.x;
    tl = G - 1 - (int)blockIdx.x;
  }
  __device__ bool next(int& cb, int& n, int& tile0, int& ntiles) {
    if (f < nf) {
      cb = f / (NT * fu);
      const int r = f - cb * NT * fu;
      n = r / fu;
      tile0 = (r - n * fu) * kS;
      ntiles = kS;
      f += G;
      return true;
    }
    if (tl < ntail) {
      cb = tl / NT;
      n = tl - cb * NT;
      tile0 = fu * kS;
      ntiles = T - tile0;
      tl += G;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);   // .x = a (low half), RNE
  return *reinterpret_cast<const uint32_t*>(&v);
}

// BIN: the input is a bf16 tensor; TMA writes the halo chunk straight into the bf16 slot
// (box 8 channels x positions x 4 channel groups = the [kg][pos][8] layout the MMA reads),
// the converter warps idle and the MMA waits on the TMA barrier.
template <int EPI, bool BIN>
__global__ void __launch_bounds__(kThreads, 1)
    conv3x3_bf16_kernel(const __grid_constant__ CUtensorMap tmap, const BfArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;

  const uint32_t w_stage = 3 * a.w_tap;
  uint8_t* raw_base = smem;                                    // 2 fp32 slots
  uint8_t* bf_base = smem + 2 * a.raw_stride;                  // 2 bf16 slots
  const int nbf = a.nbf, nw = a.nw;
  uint8_t* w_base = bf_base + nbf * a.bf_stride;               // nw stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(w_base + nw * w_stage);
  uint64_t* raw_full = bars;                    // [kBfMax] TMA -> converters (BIN: TMA -> MMA)
  uint64_t* raw_empty = bars + kBfMax;          // [kBfMax] converters -> TMA
  uint64_t* bf_full = bars + 2 * kBfMax;        // [kBfMax] converters -> MMA
  uint64_t* bf_empty = bars + 3 * kBfMax;       // [kBfMax] MMA -> converters (BIN: MMA -> TMA)
  uint64_t* w_full = bars + 4 * kBfMax;         // [kWMax]
  uint64_t* w_empty = bars + 4 * kBfMax + kWMax;
  uint64_t* acc_full = bars + 4 * kBfMax + 2 * kWMax;    // [2]
  uint64_t* acc_empty = bars + 4 * kBfMax + 2 * kWMax + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * kBfMax + 2 * kWMax + 4);
  float* xchg = reinterpret_cast<float*>(bars + 64);         // BIN epilogue: [2 groups][8 pos][128 co]
  int* pos_tab = reinterpret_cast<int*>(xchg + 2 * 8 * 128); // BIN epilogue: [2 groups][128]

  auto raw_s = [&](int s) { return raw_base + s * a.raw_stride; };
  // BIN + SW64: 512-byte aligned slabs (the swizzle atom); the front pad holds the shift -1 row
  const bool sw = BIN && a.sw64;
  auto bf_s = [&](int s) { return bf_base + s * a.bf_stride + (sw ? 512 : 128); };
  auto w_s = [&](int s) { return w_base + s * w_stage; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kBfMax; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], 128);
      mbar_init(&bf_full[i], 128);
      mbar_init(&bf_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], BIN ? 256 : 128);   // every epilogue thread, once per unit
    }
    for (int i = 0; i < kWMax; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  // zero the 128-byte pads around the bf16 halo (read only for discarded positions)
  for (int i = threadIdx.x; i < nbf * 2 * 32; i += blockDim.x) {
    const int s = i / 64, part = (i / 32) & 1, w = i % 32;
    uint8_t* base = part == 0 ? bf_s(s) - 128 : bf_s(s) + a.bf_bytes;
    reinterpret_cast<uint32_t*>(base)[w] = 0u;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int Wp = a.Wp;
  // PDL: the next grid's prologue may overlap this grid's tail; everything below reads or
  // overwrites data of the previous grids
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    // ===================== TMA producer =====================
    int rs = 0, ws = 0;
    uint32_t rph = 0, wph = 0;
    const uint32_t wbytes = 3 * a.w_tap;
    UnitIter it(a.Co / 128, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (it.next(cb, n, tile0, ntiles)) {
      const __nv_bfloat16* wcb = a.w + (int64_t)cb * a.nchunks * 9 * (a.w_tap / 2);
      const int y0 = (tile0 * 128) / Wp;
      for (int c = 0; c < a.nchunks; ++c) {
        if constexpr (BIN) {
          mbar_wait(&bf_empty[rs], rph ^ 1);   // the MMA is done with this bf16 slot
          if (elect_one()) {
            mbar_arrive_expect_tx(&raw_full[rs], a.bf_bytes);
            if (sw)   // 64-byte box rows (32 channels): a quarter of the 16-byte rows' TMA row count
              tma_load_4d(&tmap, &raw_full[rs], bf_s(rs), kChunk * c, -1, y0 - 1, n);
            else
              tma_load_5d(&tmap, &raw_full[rs], bf_s(rs), 0, -1, y0 - 1, 4 * c, n);
          }
        } else {
          mbar_wait(&raw_empty[rs], rph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&raw_full[rs], a.raw_bytes);
            tma_load_5d(&tmap, &raw_full[rs], raw_s(rs), 0, -1, y0 - 1, 8 * c, n);
          }
        }
        __syncwarp();
        if (++rs == (BIN ? nbf : 2)) rs = 0, rph ^= 1;
        for (int dy = 0; dy < 3; ++dy) {
          mbar_wait(&w_empty[ws], wph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&w_full[ws], wbytes);
            bulk_load(w_s(ws), wcb + ((int64_t)c * 9 + 3 * dy) * (a.w_tap / 2), wbytes, &w_full[ws]);
          }
          __syncwarp();
          if (++ws == nw) ws = 0, wph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t kg_x = (uint32_t)a.halo_pos * 16u;     // bytes between 8-channel groups (halo)
    const uint32_t kg_w = 128u * 16u;                     // bytes between 8-channel groups (weights)
    const uint64_t xj = (uint64_t)((2 * kg_x) >> 4);      // one K = 16 step of B, 16-byte units
    const uint64_t wj = (uint64_t)((2 * kg_w) >> 4);
    const uint64_t wtap = (uint64_t)(a.w_tap >> 4);
    int bs = 0, ws = 0, ab = 0;
    uint32_t bph = 0, wph = 0, aph = 0;
    UnitIter it(a.Co / 128, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (it.next(cb, n, tile0, ntiles)) {
      const int f0 = tile0 * 128;
      const int c0 = f0 - (f0 / Wp) * Wp;
      // one MMA spans the unit's frame positions (N = 256 for two tiles, the image's last
      // tile only as far as the frame goes): A is read once per (tap, k-step) instead of once
      // per tile (an N = 128 MMA with a fresh A costs ~107 cycles against 64)
      const int nvalid = min(ntiles * 128, a.H * Wp - f0);
      const uint32_t id_unit = idesc(1, 128, (nvalid + 15) / 16 * 16);
      mbar_wait(&acc_empty[ab], aph ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + (uint32_t)(ab * kS * 128);
      for (int c = 0; c < a.nchunks; ++c) {
        mbar_wait(BIN ? &raw_full[bs] : &bf_full[bs], bph);
        tc_fence_after();
        // B: interleave ([kg][pos][8]: a position = 16 B, a K step = 2 kg) or SW64 ([pos][32] in
        // 64-byte rows, 8-row atoms 512 B apart: a position = 64 B, a K step = 32 B into the row)
        const uint64_t dx0 = sw ? desc_general(smem_u32(bf_s(bs)), 16, 512, 4, 0)
                                : desc_kmajor_interleave(smem_u32(bf_s(bs)), kg_x, 128);
        const int64_t pstep = sw ? 4 : 1;
        const uint64_t xjs = sw ? 2 : xj;
        for (int dy = 0; dy < 3; ++dy) {
          mbar_wait(&w_full[ws], wph);
          tc_fence_after();
          const uint64_t dw0 = desc_kmajor_interleave(smem_u32(w_s(ws)), kg_w, 128);
          const uint64_t bb = dx0 + (uint64_t)((int64_t)(c0 + dy * Wp - 1) * pstep);
          const bool first = (c == 0 && dy == 0);
          if (elect_one()) {
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const uint64_t da = dw0 + dx * wtap + j * wj;
                const uint32_t accum = (first && dx == 0 && j == 0) ? 0u : 1u;
                mma_f16(d0, da, bb + (uint64_t)(dx * pstep) + j * xjs, id_unit, accum);
              }
            }
            mma_commit(&w_empty[ws]);
          }
          __syncwarp();
          if (++ws == nw) ws = 0, wph ^= 1;
        }
        if (elect_one()) mma_commit(&bf_empty[bs]);
        __syncwarp();
        if (++bs == nbf) bs = 0, bph ^= 1;
      }
      if (elect_one()) mma_commit(&acc_full[ab]);
      __syncwarp();
      if (++ab == 2) ab = 0, aph ^= 1;
    }
  } else if (!BIN && warp < 6) {
    {
    // ===================== converters: fp32 halo -> bf16 K-major interleave =====================
    // raw [g = 8 groups of 4 ch][pos][4 floats]  ->  bf16 [k = 4 groups of 8 ch][pos][8 bf16]
    const int tid = threadIdx.x - 64;
    int rs = 0, bs = 0;
    uint32_t rph = 0, bph = 0;
    const int hp = a.halo_pos;
    UnitIter it(a.Co / 128, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (it.next(cb, n, tile0, ntiles)) {
      for (int c = 0; c < a.nchunks; ++c) {
        mbar_wait(&raw_full[rs], rph);
        mbar_wait(&bf_empty[bs], bph ^ 1);
        const float4* raw = reinterpret_cast<const float4*>(raw_s(rs));
        uint4* bf = reinterpret_cast<uint4*>(bf_s(bs));
        for (int i = tid; i < 4 * hp; i += 128) {
          const int k = i / hp, p = i - k * hp;
          const float4 u = raw[(2 * k) * hp + p];
          const float4 v = raw[(2 * k + 1) * hp + p];
          bf[i] = make_uint4(pack_bf16(u.x, u.y), pack_bf16(u.z, u.w), pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
        }
        fence_proxy_async_smem();
        mbar_arrive(&bf_full[bs]);
        mbar_arrive(&raw_empty[rs]);
        if (++rs == 2) rs = 0, rph ^= 1;
        if (++bs == nbf) bs = 0, bph ^= 1;
      }
    }
    }
  } else {
    // ===================== epilogue =====================
    if constexpr (BIN) {
    // Two groups of 4 warps (the idle converter warps 2-5 and warps 6-9); group g drains tile g
    // of every unit.  Batches of 8 positions: each warp moves its 32 rows (output channels) x 8
    // columns to shared memory as [position][128 co]; the group reads it back transposed -- a
    // thread owns 4 consecutive channels of a position (two items per batch) -- and finishes
    // the fused epilogue with vector loads and stores: 16-byte fp32, 8-byte bf16 (the per-lane
    // 2-byte bf16 accesses of a channel-per-lane epilogue ran at a fraction of the bandwidth).
    // The next batch's aux operand is loaded before the current one is finished.
    const int q = warp & 3;
    const int grp = warp >= 6 ? 0 : 1;
    const int gtid = (warp & 3) * 32 + lane;              // 0..127 within the group
    constexpr bool kBias = EPI == EPI_BIAS || EPI == EPI_BIAS_TANH || EPI == EPI_RESID;
    constexpr bool kAux = EPI == EPI_RESID || EPI == EPI_TANH_BWD || EPI == EPI_ADD;
    constexpr bool kAux16 = EPI == EPI_DTANH16;
    float* buf = xchg + grp * 8 * 128;
    int* tab = pos_tab + grp * 128;
    const uint32_t grp_bar = 6 + grp;
    const int cg = gtid & 31;                             // channel group: channels 4 cg .. 4 cg + 3
    const int pr0 = gtid >> 5;                            // items: positions pr0 and pr0 + 4 of a batch
    int ab = 0;
    uint32_t aph = 0;
    UnitIter it(a.Co / 128, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (it.next(cb, n, tile0, ntiles)) {
      const int64_t img = (int64_t)n * a.H * a.W;
      const int co4 = cb * 128 + 4 * cg;
      float4 bias = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kBias) bias = *reinterpret_cast<const float4*>(a.bias + co4);
      mbar_wait(&acc_full[ab], aph);
      tc_fence_after();
      if (grp < ntiles) {
        const int fb = (tile0 + grp) * 128;
        {
          const int f = fb + gtid, y = f / Wp, X = f - y * Wp;
          asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");   // previous tile's readers are done
          tab[gtid] = (y < a.H && X >= 1 && X <= a.W) ? (y * a.W + (X - 1)) * a.Co : -1;
          asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");
        }
        const uint32_t tcol = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * kS + grp) * 128);
        const float* auxb = kAux ? a.aux + img * a.Co + co4 : nullptr;
        const __nv_bfloat16* auxb16 = kAux16 ? a.aux16 + img * a.Co + co4 : nullptr;
        float* outb = a.out ? a.out + img * a.Co + co4 : nullptr;
        __nv_bfloat16* outb16 = a.out16 ? a.out16 + img * a.Co + co4 : nullptr;
        __nv_bfloat16* outb16d = a.out16d ? a.out16d + img * a.Co + co4 : nullptr;
        const int nb = min(16, (a.H * Wp - fb + 7) / 8);  // 8-position batches with frame positions
        float4 ax[2];
        auto load = [&](int b, float4 (&x)[2]) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int o = tab[8 * b + pr0 + 4 * j];
            x[j] = make_float4(1.f, 1.f, 1.f, 1.f);
            if constexpr (kAux) {
              if (o >= 0) x[j] = __ldg(reinterpret_cast<const float4*>(auxb + o));
            }
            if constexpr (kAux16) {
              if (o >= 0) {
                const uint2 u = __ldg(reinterpret_cast<const uint2*>(auxb16 + o));
                x[j] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                                   __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
              }
            }
          }
        };
        // aux loads run two batches ahead (a ring of three register pairs)
        float4 ax1[2];
        if (kAux || kAux16) {
          load(0, ax);
          if (nb > 1) load(1, ax1);
        }
        // batch b + 1's accumulators are loaded while batch b is finished (double-buffered
        // registers: the TMEM load latency leaves the critical path)
        uint32_t rn[8];
        if (nb > 0) tmem_ld8(tcol, rn);
        for (int b = 0; b < nb; ++b) {
          uint32_t r[8];
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) r[e] = rn[e];
          if (b + 1 < nb) tmem_ld8(tcol + (uint32_t)(8 * (b + 1)), rn);
          asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");   // buf free
#pragma unroll
          for (int e = 0; e < 8; ++e) buf[e * 128 + q * 32 + lane] = __uint_as_float(r[e]);
          asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");
          float4 axn[2];
          if ((kAux || kAux16) && b + 2 < nb) load(b + 2, axn);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int pr = pr0 + 4 * j;
            const int off = tab[8 * b + pr];
            if (off < 0) continue;
            const float4 v4 = *reinterpret_cast<const float4*>(buf + pr * 128 + 4 * cg);
            const float v[4] = {v4.x, v4.y, v4.z, v4.w};
            const float bb[4] = {bias.x, bias.y, bias.z, bias.w};
            const float xa[4] = {ax[j].x, ax[j].y, ax[j].z, ax[j].w};
            float o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if constexpr (EPI == EPI_BIAS) o[i] = v[i] + bb[i];
              else if constexpr (EPI == EPI_BIAS_TANH) o[i] = tanhf(v[i] + bb[i]);
              else if constexpr (EPI == EPI_RESID) o[i] = xa[i] + a.h * (v[i] + bb[i]);
              else if constexpr (EPI == EPI_TANH_BWD) o[i] = (a.h * v[i]) * (1.f - xa[i] * xa[i]);
              else if constexpr (EPI == EPI_ADD) o[i] = xa[i] + v[i];
              else if constexpr (EPI == EPI_DTANH16) o[i] = (a.h * v[i]) * xa[i];
              else o[i] = a.h * v[i];
            }
            if (a.dbg & 2) continue;
            if (outb) *reinterpret_cast<float4*>(outb + off) = make_float4(o[0], o[1], o[2], o[3]);
            if (outb16)
              *reinterpret_cast<uint2*>(outb16 + off) = make_uint2(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]));
            if (outb16d)
              *reinterpret_cast<uint2*>(outb16d + off) =
                  make_uint2(pack_bf16(1.f - o[0] * o[0], 1.f - o[1] * o[1]), pack_bf16(1.f - o[2] * o[2], 1.f - o[3] * o[3]));
          }
          if (kAux || kAux16) ax[0] = ax1[0], ax[1] = ax1[1], ax1[0] = axn[0], ax1[1] = axn[1];
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
      if (++ab == 2) ab = 0, aph ^= 1;
    }
    } else {
    // TMEM lane r = output channel cb*128 + r; a warp owns lanes 32q..32q+31 and walks the
    // positions 16 columns at a time: one 128-byte store per position (NHWC).  bf16-input
    // mode: the idle converter warps (2-5) form a second group, group g drains tile g of
    // every unit; the aux operand of the next 16 positions is loaded before the current ones
    // are finished, so the loads' latency overlaps the stores.
    const int q = warp & 3;
    const int grp = BIN ? (warp >= 6 ? 0 : 1) : 0;
    constexpr bool kBias = EPI == EPI_BIAS || EPI == EPI_BIAS_TANH || EPI == EPI_RESID;
    constexpr bool kAux = EPI == EPI_RESID || EPI == EPI_TANH_BWD || EPI == EPI_ADD;
    constexpr bool kAux16 = EPI == EPI_DTANH16;
    int ab = 0;
    uint32_t aph = 0;
    UnitIter it(a.Co / 128, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (it.next(cb, n, tile0, ntiles)) {
      const int64_t img = (int64_t)n * a.H * a.W;
      const int co = cb * 128 + q * 32 + lane;
      const float bias = kBias ? __ldg(a.bias + co) : 0.f;
      const float* auxb = kAux ? a.aux + img * a.Co + co : nullptr;
      float* outb = a.out ? a.out + img * a.Co + co : nullptr;
      __nv_bfloat16* outb16 = a.out16 ? a.out16 + img * a.Co + co : nullptr;
      __nv_bfloat16* outb16d = a.out16d ? a.out16d + img * a.Co + co : nullptr;
      const __nv_bfloat16* auxb16 = kAux16 ? a.aux16 + img * a.Co + co : nullptr;
      const __nv_bfloat16* auxb16_pair = kAux16 ? a.aux16 + img * a.Co + (co & ~1) : nullptr;
      const bool odd_ch = co & 1;
      mbar_wait(&acc_full[ab], aph);
      tc_fence_after();
      const int s_lo = BIN ? grp : 0, s_hi = BIN ? min(grp + 1, ntiles) : ntiles;
      for (int s = s_lo; s < s_hi; ++s) {
        const uint32_t tcol = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)((ab * kS + s) * 128);
        const int fb = (tile0 + s) * 128;
        const int nb = min(8, (a.H * Wp - fb + 15) / 16);   // 16-position batches with frame positions
        int off[16];
        float ax[16];
        auto load = [&](int f0, int (&o)[16], float (&x)[16]) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int f = f0 + e, y = f / Wp, X = f - y * Wp;
            o[e] = (y < a.H && X >= 1 && X <= a.W) ? (y * a.W + (X - 1)) * a.Co : -1;
          }
          if constexpr (kAux) {
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = o[e] >= 0 ? auxb[o[e]] : 0.f;
          }
          if constexpr (kAux16) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              // 32-bit read-only loads of the channel pair (lanes 2i, 2i+1 share the word), the
              // lane's half selected: the 16-bit loads ran this epilogue at half speed
              const uint32_t u = (o[e] >= 0 && !(a.dbg & 1))
                                     ? __ldg(reinterpret_cast<const unsigned int*>(auxb16_pair + o[e]))
                                     : 0x3f803f80u;
              x[e] = __uint_as_float(odd_ch ? (u & 0xffff0000u) : (u << 16));
            }
          }
        };
        load(fb, off, ax);
        for (int b = 0; b < nb; ++b) {
          int offn[16];
          float axn[16];
          if (b + 1 < nb) load(fb + 16 * (b + 1), offn, axn);
          uint32_t r[16];
          tmem_ld16(tcol + (uint32_t)(16 * b), r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            if (off[e] < 0) continue;                           // warp-uniform
            const float v = __uint_as_float(r[e]);
            float o;
            if constexpr (EPI == EPI_BIAS) o = v + bias;
            else if constexpr (EPI == EPI_BIAS_TANH) o = tanhf(v + bias);
            else if constexpr (EPI == EPI_RESID) o = ax[e] + a.h * (v + bias);
            else if constexpr (EPI == EPI_TANH_BWD) o = (a.h * v) * (1.f - ax[e] * ax[e]);
            else if constexpr (EPI == EPI_ADD) o = ax[e] + v;
            else if constexpr (EPI == EPI_DTANH16) o = (a.h * v) * ax[e];
            else o = a.h * v;
            if (a.dbg & 2) continue;
            if (outb) outb[off[e]] = o;
            if (outb16) outb16[off[e]] = __float2bfloat16_rn(o);
            if (outb16d) outb16d[off[e]] = __float2bfloat16_rn(1.f - o * o);
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) off[e] = offn[e], ax[e] = axn[e];
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
      if (++ab == 2) ab = 0, aph ^= 1;
    }
    }  // BIN / channel-per-lane epilogue
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// HWIO fp32 -> bf16 A operand [cb][chunk][tap'][kg][128 rows][8]: row r = output channel
// 128 cb + r, element e = input channel 32 chunk + 8 kg + e.  flip = dgrad (tap' = 8 - tap,
// ci' = co, co' = ci).
__global__ void prep_weights_bf16_kernel(const float* __restrict__ w, int ci_src, int co_src, int flip,
                                         __nv_bfloat16* __restrict__ out) {
  const int Ci = flip ? co_src : ci_src;
  const int Co = flip ? ci_src : co_src;
  const int64_t per_cb = 9LL * Ci * 128;
  const int64_t total = per_cb * (Co / 128);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int cb = (int)(idx / per_cb);
    const int64_t li = idx - cb * per_cb;
    const int e = (int)(li & 7);
    const int r = (int)((li >> 3) & 127);
    const int64_t rest = li >> 10;              // (chunk, tap, kg)
    const int kg = (int)(rest % 4);
    const int tap = (int)((rest / 4) % 9);
    const int chunk = (int)(rest / 36);
    const int ci = chunk * kChunk + kg * 8 + e;
    const int co = cb * 128 + r;
    const float v = !flip ? w[((int64_t)tap * ci_src + ci) * co_src + co]
                          : w[((int64_t)(8 - tap) * ci_src + co) * co_src + ci];
    out[idx] = __float2bfloat16_rn(v);
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

// NHWC fp32 as 5-D (4 ch, W, H, C/4 groups, N); box (4, W+2 from x = -1, rows, 8 groups, 1)
CUtensorMap make_halo_map(const float* in, const ConvShape& s, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {4, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)(s.ci / 4), (cuuint64_t)s.n};
  const cuuint64_t strides[4] = {(cuuint64_t)s.ci * 4, (cuuint64_t)s.w * s.ci * 4, 16,
                                 (cuuint64_t)s.h * s.w * s.ci * 4};
  const cuuint32_t box[5] = {4, (cuuint32_t)Wp, (cuuint32_t)rows_h, 8, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 conv) failed (" + std::to_string((int)r) + ")");
  return m;
}

// NHWC bf16 as 5-D (8 ch, W, H, C/8 groups, N); box (8, W+2 from x = -1, rows, 4 groups, 1):
// the bf16 slot layout [kg][pos][8]
CUtensorMap make_halo_map16(const void* in, const ConvShape& s, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {8, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)(s.ci / 8), (cuuint64_t)s.n};
  const cuuint64_t strides[4] = {(cuuint64_t)s.ci * 2, (cuuint64_t)s.w * s.ci * 2, 16,
                                 (cuuint64_t)s.h * s.w * s.ci * 2};
  const cuuint32_t box[5] = {8, (cuuint32_t)Wp, (cuuint32_t)rows_h, 4, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 conv, bf16 in) failed (" + std::to_string((int)r) + ")");
  return m;
}

bool halo_sw64() {
  static const bool on = [] {
    const char* e = std::getenv("RP_BF16_HALO_SW");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct Plan {
  bool ok = false;
  int Wp, rows_h, halo_pos, T;
  uint32_t raw_bytes, raw_stride, bf_bytes, bf_stride, w_tap;
  int nbf = 2, nw = kWStages;
  size_t smem;
};

Plan plan_for(const ConvShape& s, bool bin = false) {
  Plan p;
  if (s.co % 128 != 0 || s.ci % kChunk != 0 || s.w + 1 > 256) return p;
  p.Wp = s.w + 1;   // W + 1 frame columns: x = -1 of row y + 1 is x = W of row y (conv_tc.cu)
  p.rows_h = (3 * p.Wp + 128 * kS + p.Wp - 1) / p.Wp;
  if (p.rows_h > 256) return p;
  p.halo_pos = p.rows_h * p.Wp;
  p.T = (s.h * p.Wp + 127) / 128;
  p.raw_bytes = (uint32_t)p.halo_pos * kChunk * 4u;
  p.raw_stride = bin ? 0u : (p.raw_bytes + 1023) / 1024 * 1024;   // bf16 input: no fp32 staging
  p.bf_bytes = (uint32_t)p.halo_pos * kChunk * 2u;
  p.bf_stride = ((bin && halo_sw64() ? 512 : 128) + p.bf_bytes + 128 + 1023) / 1024 * 1024;
  p.w_tap = 4u * 128u * 16u;
  const size_t fixed = 512 + 1024;
  if (bin) {
    const size_t fixed_bin = 512 + 2 * 8 * 128 * 4 + 2 * 128 * 4 + 1024;   // + exchange and position tables
    // no fp32 staging: the freed space deepens the bf16 halo ring and the weight ring (the
    // halo of a 32-channel chunk feeds 2304 MMA cycles; 2 slots left its TMA latency exposed)
    p.ok = false;
    for (int nb = kBfMax; nb >= 2 && !p.ok; --nb)
      for (int w = kWMax; w >= kWStages && !p.ok; --w) {
        const size_t need = nb * (size_t)p.bf_stride + w * 3 * (size_t)p.w_tap + fixed_bin;
        if (need <= (size_t)kMaxSmem) p.nbf = nb, p.nw = w, p.smem = need, p.ok = true;
      }
    return p;
  }
  p.smem = 2 * (size_t)p.raw_stride + 2 * (size_t)p.bf_stride + kWStages * 3 * (size_t)p.w_tap + fixed;
  p.ok = p.smem <= (size_t)kMaxSmem;
  return p;
}

// NHWC bf16 as 4-D (C, W, H, N); box (32 ch, W+2 from x = -1, rows, 1), 64B swizzle: the SW64
// slab [pos][32 ch]
CUtensorMap make_halo_map16_sw(const void* in, const ConvShape& s, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {(cuuint64_t)s.ci, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)s.n};
  const cuuint64_t strides[3] = {(cuuint64_t)s.ci * 2, (cuuint64_t)s.w * s.ci * 2, (cuuint64_t)s.h * s.w * s.ci * 2};
  const cuuint32_t box[4] = {(cuuint32_t)kChunk, (cuuint32_t)Wp, (cuuint32_t)rows_h, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 conv, SW64) failed (" + std::to_string((int)r) + ")");
  return m;
}

std::mutex g_map_mu;
std::map<std::tuple<const void*, int, int, int, int, int, int>, CUtensorMap> g_maps;

CUtensorMap cached_map(const void* in, const ConvShape& s, int Wp, int rows_h, bool bin = false) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  const int kind = bin ? (halo_sw64() ? 2 : 1) : 0;
  auto key = std::make_tuple(in, s.n, s.h, s.w, s.ci, rows_h, kind);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();   // callers hold copies, never references
    it = g_maps.emplace(key, kind == 2   ? make_halo_map16_sw(in, s, Wp, rows_h)
                             : kind == 1 ? make_halo_map16(in, s, Wp, rows_h)
                                         : make_halo_map(static_cast<const float*>(in), s, Wp, rows_h)).first;
  }
  return it->second;
}

template <int EPI, bool BIN>
void launch(const CUtensorMap& m, const BfArgs& a, size_t smem, int grid, cudaStream_t st) {
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(conv3x3_bf16_kernel<EPI, BIN>), kMaxSmem);
  launch_pdl(conv3x3_bf16_kernel<EPI, BIN>, grid, kThreads, smem, st, m, a);
}

template <bool BIN>
void launch_epi(int epi, const CUtensorMap& m, const BfArgs& a, size_t smem, int grid, cudaStream_t st) {
  switch (epi) {
    case EPI_BIAS: launch<EPI_BIAS, BIN>(m, a, smem, grid, st); break;
    case EPI_BIAS_TANH: launch<EPI_BIAS_TANH, BIN>(m, a, smem, grid, st); break;
    case EPI_RESID: launch<EPI_RESID, BIN>(m, a, smem, grid, st); break;
    case EPI_TANH_BWD: launch<EPI_TANH_BWD, BIN>(m, a, smem, grid, st); break;
    case EPI_ADD: launch<EPI_ADD, BIN>(m, a, smem, grid, st); break;
    case EPI_DTANH16: launch<EPI_DTANH16, BIN>(m, a, smem, grid, st); break;
    default: launch<EPI_SCALE, BIN>(m, a, smem, grid, st); break;
  }
}

}  // namespace

bool conv3x3_bf16_supported(const ConvShape& s) { return plan_for(s).ok; }

int64_t conv3x3_bf16_ws_bytes(const ConvShape& s) { return 9LL * s.ci * s.co * 2 + 256; }

namespace {
void conv_bf16_any(const ConvShape& s, const void* in, bool bin, const float* w_hwio, bool dgrad_weights,
                   const float* bias, const float* aux, const void* aux16, float h, int epi, float* out, void* out16,
                   void* out16d, void* ws, cudaStream_t st) {
  if (s.pixels() == 0) return;
  const Plan p = plan_for(s, bin);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_fwd_bf16: unsupported shape");
  if (epi == EPI_DTANH16 && !aux16) fail(RP_ERR_INTERNAL, "conv3x3_fwd_bf16: EPI_DTANH16 needs aux16");
  __nv_bfloat16* wp = static_cast<__nv_bfloat16*>(ws);
  const int ci_src = dgrad_weights ? s.co : s.ci;
  const int co_src = dgrad_weights ? s.ci : s.co;
  const int64_t total = 9LL * s.ci * s.co;
  prep_weights_bf16_kernel<<<(int)std::min<int64_t>(ceil_div(total, 256), 16 * kNumSMs), 256, 0, st>>>(
      w_hwio, ci_src, co_src, dgrad_weights ? 1 : 0, wp);
  RP_LAUNCHED();
  BfArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = p.Wp;
  a.rows_h = p.rows_h;
  a.T = p.T;
  a.halo_pos = p.halo_pos;
  a.nchunks = s.ci / kChunk;
  a.raw_bytes = p.raw_bytes;
  a.raw_stride = p.raw_stride;
  a.bf_bytes = p.bf_bytes;
  a.bf_stride = p.bf_stride;
  a.sw64 = halo_sw64() ? 1 : 0;
  a.w_tap = p.w_tap;
  a.nbf = p.nbf;
  a.nw = p.nw;
  a.h = h;
  a.w = wp;
  a.bias = bias;
  a.aux = aux;
  a.aux16 = static_cast<const __nv_bfloat16*>(aux16);
  a.out = out;
  a.out16 = static_cast<__nv_bfloat16*>(out16);
  a.out16d = static_cast<__nv_bfloat16*>(out16d);
  static const int dbg = [] {
    const char* e = std::getenv("RP_BF16_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
  const CUtensorMap m = cached_map(in, s, p.Wp, p.rows_h, bin);
  const int units = (s.co / 128) * s.n * ((p.T + kS - 1) / kS);
  const int grid = std::min(units, kNumSMs);
  if (bin)
    launch_epi<true>(epi, m, a, p.smem, grid, st);
  else
    launch_epi<false>(epi, m, a, p.smem, grid, st);
  RP_LAUNCHED();
}
}  // namespace

void conv3x3_fwd_bf16(const ConvShape& s, const float* in, const float* w_hwio, bool dgrad_weights, const float* bias,
                      const float* aux, float h, int epi, float* out, void* ws, cudaStream_t st, void* out_bf16) {
  conv_bf16_any(s, in, false, w_hwio, dgrad_weights, bias, aux, nullptr, h, epi, out, out_bf16, nullptr, ws, st);
}

void conv3x3_fwd_bf16_in16(const ConvShape& s, const void* in16, const float* w_hwio, bool dgrad_weights,
                           const float* bias, const float* aux, const void* aux16, float h, int epi, float* out,
                           void* out16, void* out16d, void* ws, cudaStream_t st) {
  conv_bf16_any(s, in16, true, w_hwio, dgrad_weights, bias, aux, aux16, h, epi, out, out16, out16d, ws, st);
}

}  // namespace rp::k
