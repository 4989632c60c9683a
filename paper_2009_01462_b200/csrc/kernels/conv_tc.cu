// tcgen05 implicit-GEMM 3x3 convolution (fprop and dgrad), NHWC fp32, sm_100a.
//
//   out[p][co] = epi( sum_{tap, ci} in[p + off(tap)][ci] * w[tap][ci][co] )
//
// (block_forward's matmul(x, W1) / matmul(a, W2) and block_vjp's matmul(upstream,
// W2^T) / matmul(dpre, W1^T), network.cpp:85-104, generalised to 3x3 taps.)
//
// Design:
//  * Output positions live in the zero-padded "interior frame" of one image (H rows x
//    (W+1) columns, flattened; the one zero column x = -1 of a row is also the previous
//    row's x = W): tap (dy,dx) is then a constant shift of dy*(W+1)+dx positions, so one
//    halo slab per 16-channel chunk, loaded once by TMA (out-of-bounds rows/columns
//    zero-filled), serves all 9 taps as 9 shifted UMMA descriptors.  The padding column is
//    computed and discarded.
//  * D^T = W^T x: the MMA's A operand is the (tiny) weight tile, M = 128 rows = the 64 output
//    channels stacked twice ([W_hi; W_lo] / [W0; W1]); B is the shifted halo view, N = the
//    unit's positions (<= 256).  Consecutive MMAs share A through the collector.
//  * Operand modes.  PLANES (the fp32 default): the input arrives as an fp16 plane pair
//    x s = x0 + x1 (planes.cuh: 22 significant bits, power-of-two scale s) written by the
//    producing epilogue and loaded by TMA straight into the MMA layout; A = [W0; W1] (fp16
//    pair of W 2^8), two kind::f16 MMAs per 16 channels accumulate all four products, the
//    epilogue divides the scales out; Co = 64 keeps the whole prepared filter resident in
//    shared memory.  X3TF32 / X3BF16 / TF32 read
//    the fp32 halo and let converter warps (w2-5) write the low parts.
//  * operands are K-major "interleaved" (no swizzle): every position is 16 contiguous bytes
//    per 4 (tf32) or 8 (bf16) channels, so a shift by one position is +16 B of descriptor
//    start address.
//  * a unit = two consecutive tiles of <= 128 positions of one image (PLANES: the frame split
//    into equal units), accumulators in TMEM double-buffered across units.
//  * warp roles (480 threads, persistent, 1 CTA/SM): w0 halo TMA, w14 weight TMA, w1 MMA
//    issuer (whole warp walks the loop so descriptors stay warp-uniform; one elected lane
//    issues), w2-5 converters (fp32-operand modes), w6-13 two epilogue groups (one tile of
//    each unit each: TMEM -> registers -> shared transpose -> hi + lo -> fused bias / tanh /
//    skip / step size -> 16-byte NHWC stores of the output and its planes).
//  * Programmatic dependent launch: the next grid's prologue and resident-filter load overlap
//    this grid's tail (pdl_wait before touching the previous grid's data).
#include <cuda.h>
#include <cuda_bf16.h>

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

constexpr int kThreads = 480;       // w0 halo TMA, w1 MMA, w2-5 converters, w6-13 epilogue, w14 weight TMA
constexpr int kWStages = 3;          // one weight stage = one filter row (3 taps) of one chunk
constexpr int kWMax = 8;             // barrier slots for the weight ring (PLANES: up to 8 stages)
constexpr int kChunk = 16;           // input channels per halo chunk
constexpr bool kUseCollector = false;  // A-operand collector reuse, tf32 modes (measured: no gain)
#ifndef RP_CONV_COLLECTOR_BF
#define RP_CONV_COLLECTOR_BF 1
#endif
constexpr bool kUseCollectorBF = RP_CONV_COLLECTOR_BF;   // X3BF16: A reuse across the 6 MMAs of a tap
constexpr int kS = 2;                // 128-position tiles per unit
constexpr int kEpiB = 16;            // epilogue batch (positions per TMEM load / exchange)
constexpr int kEpiJ = kEpiB / 8;     // positions per thread and batch (128 threads x 4 channels)
constexpr int kMaxSmem = 220 * 1024;      // streaming plans
constexpr int kMaxSmemRes = 227 * 1024;   // resident-weight plan (the sm_100 per-CTA maximum)
constexpr int kWResMax = 12;              // resident weight stages (Ci = 64: 4 chunks x 3 filter rows)

// Operand modes: TF32 (x and W truncated to tf32), X3TF32 ([W_hi; W_lo] x {x_hi, x_lo}) and
// X3BF16 (the default fp32-accurate path, capi_ops.cu fp32_split) ([W0; W1] x {x0, x1, x2} with bf16 splits: W to
// 16 significant bits, x to 24; products W0x0 .. W1x2 cover everything above 2^-18 of |W x|,
// in 3 MMAs of K = 16 per 16 channels instead of 4 of K = 8).
// MODE_PLANES: the input arrives as an fp16 plane pair (x s = x0 + x1, written by the
// producing conv's epilogue): TMA loads both planes straight into the MMA layout (no
// converters) and [W0; W1] x {x0, x1} is 2 MMAs per 16 channels (~2^-23 relative).
enum { MODE_TF32 = 0, MODE_X3TF32 = 1, MODE_X3BF16 = 2, MODE_PLANES = 3 };

struct TcArgs {
  int N, H, W, Ci, Co, Wp, rows_h, T, num_tiles, halo_pos, nchunks;
  uint32_t halo_bytes;  // one raw (or lo) halo buffer
  uint32_t halo_stride; // bytes per halo slot (raw + lo + pads)
  uint32_t w_tap;       // bytes of one tap's A operand (128 rows x 16 channels x 4 B; bf16: x 2 B)
  uint32_t plane_bytes; // X3BF16: one bf16 plane of the halo chunk (halo_pos x 32 B)
  uint32_t raw_stride;  // X3BF16: bytes per raw fp32 halo slot ([pos][16 ch], TMA target)
  int raw_slots;        // X3BF16: depth of the raw ring (2 or 3); PLANES: halo slots (2..4)
  int wstages;          // depth of the weight ring (<= kWMax); resident: stages of the whole filter
  int resident;         // PLANES, Co = 64: the co block's whole prepped filter stays in shared memory
  int tile;             // frame positions per tile (<= 128; PLANES: the image's frame split into equal units)
  float h;
  const float* w;       // prepped [chunk][tap][kg][128 rows][4]
  const float* bias;
  const float* aux;
  float* out;
  uint16_t* p0;                // optional fp16 plane pair of out * (*out_scale) (planes.cuh)
  uint16_t* p1;
  const float* in_scale;       // PLANES: the input planes' scale (device scalar; null = kActPlaneScale)
  const float* out_scale;      // the output planes' scale (device scalar; null = kActPlaneScale)
  float wscale_inv;            // 1 / the prepared filter's scale (PLANES: 2^-8)
  unsigned long long* trace;   // diagnostics (tools/trace_conv.py): per-unit timestamps, null = off
  int dbg;                     // diagnostics (RP_CONV_DBG): 1 no epilogue, 2 no halo TMA, 4 no weight TMA, 8 no MMA
};

__device__ __forceinline__ float rna_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// The tensor core reads an fp32 operand as tf32 by dropping the low 13 mantissa bits
// (measured: 1 + 2^-11 + 2^-12 enters as 1.0), so the raw halo already is x_hi and only
// x_lo = x - trunc(x) (exact in fp32) has to be written.
__device__ __forceinline__ float trunc_tf32(float v) { return __uint_as_float(__float_as_uint(v) & 0xffffe000u); }

// Work split.  A unit is kS tiles (128 frame positions each) of one image and one
// 64-channel output block cb; T = ceil(frame / 128) tiles per image leaves one shorter
// "tail" unit per image when kS does not divide T.  Full units go round-robin from CTA
// 0 upwards, tail units round-robin from CTA G-1 downwards, so the CTAs that get one
// full unit less get the extra tail: every CTA ends within one tile of the mean (plain
// round-robin over mixed units left the busiest CTA 9% above it).  cb is the outermost
// index, so CTAs working on the same images at the same time share the halo in L2.
struct UnitIter {
  int f, tl, nf, ntail, fu, T, NT, G;
  __device__ UnitIter(int mtiles, int N, int T_) : T(T_) {
    G = gridDim.x;
    fu = T / kS;                              // full units per image
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

template <int EPI>
__device__ __forceinline__ float epi_value(float acc, float bias, int64_t idx, const TcArgs& a) {
  if constexpr (EPI == EPI_BIAS) return acc + bias;
  if constexpr (EPI == EPI_BIAS_TANH) return tanhf(acc + bias);
  if constexpr (EPI == EPI_RESID) return __ldg(a.aux + idx) + a.h * (acc + bias);
  if constexpr (EPI == EPI_TANH_BWD) {
    const float t = __ldg(a.aux + idx);
    return (a.h * acc) * (1.f - t * t);
  }
  if constexpr (EPI == EPI_ADD) return a.aux[idx] + acc;
  return a.h * acc;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// v = p0 + p1 + p2 in bf16 (RNE at each step); returns the three packed planes
__device__ __forceinline__ void split3_bf16(const float (&v)[8], uint4& p0, uint4& p1, uint4& p2) {
  float r1[8], r2[8];
  uint32_t a[4], b[4], c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    a[i] = *reinterpret_cast<const uint32_t*>(&h);
    r1[2 * i] = v[2 * i] - __low2float(h);
    r1[2 * i + 1] = v[2 * i + 1] - __high2float(h);
    const __nv_bfloat162 m = __floats2bfloat162_rn(r1[2 * i], r1[2 * i + 1]);
    b[i] = *reinterpret_cast<const uint32_t*>(&m);
    r2[2 * i] = r1[2 * i] - __low2float(m);
    r2[2 * i + 1] = r1[2 * i + 1] - __high2float(m);
    c[i] = pack_bf16x2(r2[2 * i], r2[2 * i + 1]);
  }
  p0 = make_uint4(a[0], a[1], a[2], a[3]);
  p1 = make_uint4(b[0], b[1], b[2], b[3]);
  p2 = make_uint4(c[0], c[1], c[2], c[3]);
}

// the same for 4 values: three packed bf16x4 planes
__device__ __forceinline__ void split3_bf16_4(const float (&v)[4], uint2& p0, uint2& p1, uint2& p2) {
  uint32_t a[2], b[2], c[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    a[i] = *reinterpret_cast<const uint32_t*>(&h);
    const float r0 = v[2 * i] - __low2float(h), r1 = v[2 * i + 1] - __high2float(h);
    const __nv_bfloat162 m = __floats2bfloat162_rn(r0, r1);
    b[i] = *reinterpret_cast<const uint32_t*>(&m);
    c[i] = pack_bf16x2(r0 - __low2float(m), r1 - __high2float(m));
  }
  p0 = make_uint2(a[0], a[1]);
  p1 = make_uint2(b[0], b[1]);
  p2 = make_uint2(c[0], c[1]);
}

template <int EPI, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tmap, const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);   // warp-uniform role index
  const int lane = threadIdx.x & 31;

  // ---- shared memory carve-up
  const uint32_t w_stage = 3 * a.w_tap;
  constexpr bool BF = MODE == MODE_X3BF16;
  constexpr bool PL = MODE == MODE_PLANES;
  constexpr bool BFL = BF || PL;                              // bf16 plane layout in the halo slots
  // X3BF16: [2 plane slots][raw_slots raw slots][weights]...; PLANES: [raw_slots plane
  // slots][weights]...; else [2 halo slots][weights]...
  const int hslots = PL ? a.raw_slots : 2;
  uint8_t* halo_base = smem;
  uint8_t* raw_base = smem + 2 * a.halo_stride;               // X3BF16 only
  uint8_t* w_base = smem + hslots * a.halo_stride + (BF ? a.raw_slots * a.raw_stride : 0u);   // kWStages stages
  const int wst = a.wstages;
  float* xchg = reinterpret_cast<float*>(w_base + wst * w_stage);   // [2 groups][hi, lo][kEpiB pos][64 ch]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xchg + 2 * 2 * kEpiB * 64);
  uint64_t* halo_full = bars;        // [4]
  uint64_t* halo_conv = bars + 4;    // [4]
  uint64_t* halo_empty = bars + 8;   // [4]
  uint64_t* w_full = bars + 12;      // [kWMax]
  uint64_t* w_empty = bars + 12 + kWMax;
  uint64_t* acc_full = bars + 12 + 2 * kWMax;   // [2]
  uint64_t* acc_empty = bars + 14 + 2 * kWMax;  // [2]
  uint64_t* raw_full = bars + 16 + 2 * kWMax;   // [3] X3BF16: TMA -> converters
  uint64_t* raw_empty = bars + 19 + 2 * kWMax;  // [3] X3BF16: converters -> TMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22 + 2 * kWMax);
  int* pos_tab = reinterpret_cast<int*>(bars + 64);   // [2 groups][128] epilogue position -> NHWC offset

  constexpr bool THREE = MODE != MODE_TF32;
  auto halo_raw = [&](int s) { return halo_base + s * a.halo_stride + 128; };
  auto halo_lo = [&](int s) { return halo_base + s * a.halo_stride + 256 + a.halo_bytes; };
  // X3BF16: planes p = 0..2 of bf16 [2 kg][positions][8], each between 128-byte zero pads
  // (plane pitch rounded to 128 B: the planes are TMA destinations in the PLANES mode)
  const uint32_t plane_pitch = ((a.plane_bytes + 127u) & ~127u) + 128u;
  auto plane = [&](int s, int p) { return halo_base + s * a.halo_stride + 128 + p * plane_pitch; };
  auto raw_slot = [&](int r) { return raw_base + r * a.raw_stride; };
  auto w_s = [&](int s) { return w_base + s * w_stage; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(&halo_full[i], 1);
      mbar_init(&halo_conv[i], 128);
      mbar_init(&halo_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 256);
    }
    for (int i = 0; i < kWMax; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], 128);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  // zero the 128-byte pads around the halo buffers (read only for discarded positions)
  if constexpr (BFL) {
    constexpr int kParts = PL ? 3 : 4;      // front pad + one behind each plane
    for (int i = threadIdx.x; i < hslots * kParts * 32; i += blockDim.x) {
      const int s = i / (kParts * 32), part = (i / 32) % kParts, w = i % 32;
      uint8_t* base = part == 0 ? halo_base + s * a.halo_stride : plane(s, part - 1) + a.plane_bytes;
      reinterpret_cast<uint32_t*>(base)[w] = 0u;
    }
  } else {
    for (int i = threadIdx.x; i < 2 * 3 * 32; i += blockDim.x) {
      const int s = i / 96, part = (i / 32) % 3, w = i % 32;
      uint8_t* base = halo_base + s * a.halo_stride +
                      (part == 0 ? 0 : part == 1 ? 128 + a.halo_bytes : 256 + 2 * a.halo_bytes);
      reinterpret_cast<uint32_t*>(base)[w] = 0u;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int Wp = a.Wp;
  // PDL: the next conv / wgrad may now be scheduled; its prologue (barriers, TMEM, the resident
  // filter load) then overlaps this grid's tail on the SMs it frees
  pdl_launch_dependents();

  if (warp != 14) pdl_wait();   // every role below reads or overwrites the previous grid's data
  if (warp == 0) {
    // ===================== halo TMA producer =====================
    // X3BF16: into the raw ring, released by the converters (runs up to raw_slots chunks
    // ahead of the converters, independent of the MMA); else into the halo slot the MMA
    // releases.
    int hs = 0;
    uint32_t hph = 0;
    const int nslots = BF ? a.raw_slots : hslots;
    UnitIter it(a.Co / 64, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (it.next(cb, n, tile0, ntiles)) {
      const int f0 = tile0 * a.tile;
      const int y0 = f0 / Wp;
      for (int c = 0; c < a.nchunks; ++c) {
        mbar_wait(BF ? &raw_empty[hs] : &halo_empty[hs], hph ^ 1);
        if (elect_one()) {
          if constexpr (BF) {
            mbar_arrive_expect_tx(&raw_full[hs], a.halo_bytes);
            tma_load_4d(&tmap, &raw_full[hs], raw_slot(hs), kChunk * c, -1, y0 - 1, n);
          } else if constexpr (PL) {
            // both planes of the chunk: images [0, N) are plane 0, [N, 2N) plane 1
            if (a.dbg & 2) { mbar_arrive(&halo_full[hs]); } else {
            mbar_arrive_expect_tx(&halo_full[hs], 2 * a.plane_bytes);
            tma_load_5d(&tmap, &halo_full[hs], plane(hs, 0), 0, -1, y0 - 1, 2 * c, n);
            tma_load_5d(&tmap, &halo_full[hs], plane(hs, 1), 0, -1, y0 - 1, 2 * c, n + a.N);
            }
          } else {
            mbar_arrive_expect_tx(&halo_full[hs], a.halo_bytes);
            tma_load_5d(&tmap, &halo_full[hs], halo_raw(hs), 0, -1, y0 - 1, 4 * c, n);
          }
        }
        __syncwarp();
        if (++hs == nslots) hs = 0, hph ^= 1;
      }
    }
  } else if (warp == 14) {
    // ===================== weight TMA producer =====================
    int ws = 0;
    uint32_t wph = 0;
    const uint32_t wbytes = 3 * a.w_tap;
    if (a.resident) {
      // the whole filter of the single co block, once per launch (stage c * 3 + dy = slot c * 3 + dy):
      // the per-unit weight stream was ~16 B/clk/SM of L2 traffic on top of the halo and the epilogue.
      // Issued before pdl_wait(): the prepared filter comes from a kernel that completed before
      // the previous grid did (a plainly launched prep kernel, or one before a PDL chain member
      // that itself waited).
      if (elect_one()) {
        mbar_arrive_expect_tx(&w_full[0], (uint32_t)wst * wbytes);
        for (int i = 0; i < wst; ++i)
          bulk_load(w_s(i), reinterpret_cast<const uint8_t*>(a.w) + (int64_t)i * wbytes, wbytes, &w_full[0]);
      }
      __syncwarp();
    }
    pdl_wait();
    UnitIter it(a.Co / 64, a.N, a.T);
    int cb, n, tile0, ntiles;
    while (!a.resident && it.next(cb, n, tile0, ntiles)) {
      const uint8_t* wcb = reinterpret_cast<const uint8_t*>(a.w) + (int64_t)cb * a.nchunks * 9 * a.w_tap;
      for (int c = 0; c < a.nchunks; ++c) {
        for (int dy = 0; dy < 3; ++dy) {
          mbar_wait(&w_empty[ws], wph ^ 1);
          if (elect_one()) {
            if (a.dbg & 4) { mbar_arrive(&w_full[ws]); } else {
            mbar_arrive_expect_tx(&w_full[ws], wbytes);
            bulk_load(w_s(ws), wcb + ((int64_t)c * 9 + 3 * dy) * a.w_tap, wbytes, &w_full[ws]);
            }
          }
          __syncwarp();
          if (++ws == wst) ws = 0, wph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t id = BFL ? idesc(1, 128, 128) : idesc(2, 128, 128);
    const uint32_t kg_x = (uint32_t)a.halo_pos * 16u;     // bytes between channel groups (halo)
    const uint32_t kg_w = 128u * 16u;                     // bytes between channel groups (weights)
    const uint64_t xj = (uint64_t)((2 * kg_x) >> 4);      // K-step (8 channels) of B, 16-byte units
    const uint64_t wj = (uint64_t)((2 * kg_w) >> 4);
    const uint64_t wtap = (uint64_t)(a.w_tap >> 4);
    int hs = 0, ws = 0, ab = 0;
    uint32_t hph = 0, wph = 0, aph = 0;
    UnitIter it(a.Co / 64, a.N, a.T);
    int cb, n, tile0, ntiles, ui = 0;
    if (a.resident) {   // unconditionally: a CTA without units must not exit with the load in flight
      mbar_wait(&w_full[0], 0);
      tc_fence_after();
    }
    while (it.next(cb, n, tile0, ntiles)) {                   // warp-uniform
      const int u = ui++;
      const int f0 = tile0 * a.tile;
      const int c0 = f0 - (f0 / Wp) * Wp;
      const int nvalid = min(ntiles * a.tile, a.H * Wp - f0);           // frame positions of the unit
      const uint32_t id_unit = idesc(0, 128, (nvalid + 15) / 16 * 16);  // PLANES (fp16 pairs): N = 16 .. 256
      mbar_wait(&acc_empty[ab], aph ^ 1);
      tc_fence_after();
      if (a.trace && blockIdx.x < 2 && lane == 0 && u < 64) a.trace[(blockIdx.x * 64 + u) * 8 + 0] = globaltimer_ns();
      const long long clk_u0 = a.trace ? clock64() : 0;
      const uint32_t d0 = tmem_base + (uint32_t)(ab * kS * 128);
      long long wait_h = 0, wait_w = 0;
      for (int c = 0; c < a.nchunks; ++c) {
        long long tw = a.trace ? clock64() : 0;
        mbar_wait((THREE && !PL) ? &halo_conv[hs] : &halo_full[hs], hph);
        if (a.trace) wait_h += clock64() - tw;
        tc_fence_after();
        if (a.trace && blockIdx.x < 2 && lane == 0 && u < 64 && c == 0) a.trace[(blockIdx.x * 64 + u) * 8 + 4] = globaltimer_ns();
        const uint64_t dxh0 = desc_kmajor_interleave(smem_u32(BFL ? plane(hs, 0) : halo_raw(hs)), kg_x, 128);
        const uint64_t dxl0 = desc_kmajor_interleave(smem_u32(BFL ? plane(hs, 1) : halo_lo(hs)), kg_x, 128);
        const uint64_t dxq0 = desc_kmajor_interleave(smem_u32(plane(hs, BF ? 2 : 0)), kg_x, 128);
        for (int dy = 0; dy < 3; ++dy) {
          long long tw2 = a.trace ? clock64() : 0;
          if (!a.resident) mbar_wait(&w_full[ws], wph);
          if (a.trace) wait_w += clock64() - tw2;
          tc_fence_after();
          const uint64_t dw0 = desc_kmajor_interleave(smem_u32(w_s(ws)), kg_w, 128);
          const int64_t row = c0 + dy * Wp - 1;              // positions; >= -1
          const uint64_t bh = dxh0 + (uint64_t)row;          // 16-byte units: one position = 1
          const uint64_t bl = dxl0 + (uint64_t)row;
          const uint64_t bq = dxq0 + (uint64_t)row;
          const bool first = (c == 0 && dy == 0);
          if (PL) {
            // 16 channels = one K = 16 step; A = [W0; W1] (fp16), B = planes x0, x1.  One MMA
            // spans the unit's frame positions (N = 256 for two tiles; the image's last tile
            // only as far as the frame goes, e.g. 64 of 128 positions at 32x32)
            if (elect_one()) {
              if (!(a.dbg & 8))
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const uint64_t da = dw0 + dx * wtap;
                const uint32_t accum = (first && dx == 0) ? 0u : 1u;
                mma_f16_c<1>(d0, da, bh + dx, id_unit, accum);
                mma_f16_c<3>(d0, da, bl + dx, id_unit, 1u);
              }
              if (!a.resident) mma_commit(&w_empty[ws]);
            }
          } else if (BF) {
            // 16 channels = one K = 16 step; A = [W0; W1] (bf16), B = planes x0, x1, x2
            if (elect_one()) {
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const uint64_t da = dw0 + dx * wtap;
                const uint32_t accum = (first && dx == 0) ? 0u : 1u;
                if (kUseCollectorBF) {   // the 3 ntiles MMAs of one tap share A through the collector
                  mma_f16_c<1>(d0, da, bh + dx, id, accum);
                  mma_f16_c<2>(d0, da, bl + dx, id, 1u);
                  if (ntiles > 1) {
                    mma_f16_c<2>(d0, da, bq + dx, id, 1u);
                    mma_f16_c<2>(d0 + 128, da, bh + dx + 128, id, accum);
                    mma_f16_c<2>(d0 + 128, da, bl + dx + 128, id, 1u);
                    mma_f16_c<3>(d0 + 128, da, bq + dx + 128, id, 1u);
                  } else {
                    mma_f16_c<3>(d0, da, bq + dx, id, 1u);
                  }
                } else {
#pragma unroll
                  for (int s = 0; s < kS; ++s) {
                    if (s < ntiles) {
                      const uint64_t boff = (uint64_t)(dx + 128 * s);
                      mma_f16(d0 + s * 128, da, bh + boff, id, accum);
                      mma_f16(d0 + s * 128, da, bl + boff, id, 1u);
                      mma_f16(d0 + s * 128, da, bq + boff, id, 1u);
                    }
                  }
                }
              }
              mma_commit(&w_empty[ws]);
            }
          } else if (elect_one()) {
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const uint64_t da = dw0 + dx * wtap + j * wj;   // A: weights, shared by the next MMAs
                const uint32_t accum = (first && dx == 0 && j == 0) ? 0u : 1u;
                // the 2 ntiles MMAs (tiles x {x_hi, x_lo}) may read A through the collector
                if (THREE && kUseCollector) {
                  const uint64_t b0 = (uint64_t)dx + j * xj;
                  mma_tf32_c<1>(d0, da, bh + b0, id, accum);
                  if (ntiles > 1) {
                    mma_tf32_c<2>(d0, da, bl + b0, id, 1u);
                    mma_tf32_c<2>(d0 + 128, da, bh + b0 + 128, id, accum);
                    mma_tf32_c<3>(d0 + 128, da, bl + b0 + 128, id, 1u);
                  } else {
                    mma_tf32_c<3>(d0, da, bl + b0, id, 1u);
                  }
                } else {
#pragma unroll
                  for (int s = 0; s < kS; ++s) {
                    if (s < ntiles) {
                      const uint64_t boff = (uint64_t)(dx + 128 * s) + j * xj;
                      mma_tf32(d0 + s * 128, da, bh + boff, id, accum);
                      if (THREE) mma_tf32(d0 + s * 128, da, bl + boff, id, 1u);
                    }
                  }
                }
              }
            }
            mma_commit(&w_empty[ws]);
          }
          __syncwarp();
          if (++ws == wst) ws = 0, wph ^= 1;
        }
        if (elect_one()) mma_commit(&halo_empty[hs]);
        __syncwarp();
        if (++hs == hslots) hs = 0, hph ^= 1;
      }
      if (elect_one()) mma_commit(&acc_full[ab]);
      __syncwarp();
      if (a.trace && blockIdx.x < 2 && lane == 0 && u < 64) {
        a.trace[(blockIdx.x * 64 + u) * 8 + 1] = globaltimer_ns();
        a.trace[(blockIdx.x * 64 + u) * 8 + 5] = (unsigned long long)wait_h;   // cycles waiting for the halo
        a.trace[(blockIdx.x * 64 + u) * 8 + 6] = (unsigned long long)wait_w;   // cycles waiting for weights
        a.trace[(blockIdx.x * 64 + u) * 8 + 7] = (unsigned long long)(clock64() - clk_u0);   // SM cycles of the unit's issue
      }
      if (++ab == 2) ab = 0, aph ^= 1;
    }
  } else if (warp < 6) {
    // ===================== converters (hi/lo split of the halo) =====================
    const int tid = threadIdx.x - 64;
    if constexpr (BF) {
      // raw [pos][16 ch] fp32 (raw ring) -> planes [2 kg of 8 ch][pos][8 bf16] (plane slot);
      // one float4 (4 channels of one position) per thread and step: conflict-free LDS.128,
      // three STS.64
      const int hp = a.halo_pos;
      int rs = 0, hs = 0;
      uint32_t rph = 0, hph = 0;
      UnitIter it(a.Co / 64, a.N, a.T);
      int cb, n, tile0, ntiles;
      while (it.next(cb, n, tile0, ntiles)) {
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&raw_full[rs], rph);
          mbar_wait(&halo_empty[hs], hph ^ 1);      // the MMA is done with this plane slot
          const float4* raw = reinterpret_cast<const float4*>(raw_slot(rs));
          uint2* p0 = reinterpret_cast<uint2*>(plane(hs, 0));
          uint2* p1 = reinterpret_cast<uint2*>(plane(hs, 1));
          uint2* p2 = reinterpret_cast<uint2*>(plane(hs, 2));
          for (int i = tid; i < 4 * hp; i += 128) {
            const float4 v = raw[i];
            const int pos = i >> 2, q = i & 3;
            const int o = ((q >> 1) * hp + pos) * 2 + (q & 1);
            const float vv[4] = {v.x, v.y, v.z, v.w};
            split3_bf16_4(vv, p0[o], p1[o], p2[o]);
          }
          mbar_arrive(&raw_empty[rs]);
          fence_proxy_async_smem();
          mbar_arrive(&halo_conv[hs]);
          if (++rs == a.raw_slots) rs = 0, rph ^= 1;
          if (++hs == 2) hs = 0, hph ^= 1;
        }
      }
    } else if constexpr (THREE && !PL) {
      int hs = 0;
      uint32_t hph = 0;
      const int n16 = (int)(a.halo_bytes / 16);
      UnitIter it(a.Co / 64, a.N, a.T);
      int cb, n, tile0, ntiles;
      while (it.next(cb, n, tile0, ntiles)) {
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&halo_full[hs], hph);
          float4* raw = reinterpret_cast<float4*>(halo_raw(hs));
          float4* lo = reinterpret_cast<float4*>(halo_lo(hs));
          for (int i = tid; i < n16; i += 128) {
            const float4 v = raw[i];
            float4 l;
            l.x = v.x - trunc_tf32(v.x); l.y = v.y - trunc_tf32(v.y);
            l.z = v.z - trunc_tf32(v.z); l.w = v.w - trunc_tf32(v.w);
            lo[i] = l;
          }
          fence_proxy_async_smem();
          mbar_arrive(&halo_conv[hs]);
          if (++hs == 2) hs = 0, hph ^= 1;
        }
      }
    }
  } else if (warp < 14) {
    // ===================== epilogue =====================
    // Two groups of 4 warps; group g finishes tile s = g of every unit (both tiles of a unit
    // drain in parallel).  D row r: r < 64 -> W_hi (W0) products for co = r, r >= 64 ->
    // W_lo (W1) products for co = r - 64.  Batches of 16 positions: every warp moves its 32
    // rows (TMEM lane quadrant) to shared memory as [hi|lo][position][64 ch]; the group then
    // reads it back transposed -- thread t owns channels 4 (t & 15) .. +3 of positions
    // t >> 4 and (t >> 4) + 8 -- and finishes hi + lo, the fused epilogue and the stores with
    // 16-byte vectors (coalesced NHWC rows).  The exchange buffer (16 KB for both groups) fits
    // beside the resident filter and three halo slots because the slots are packed to 128 B;
    // the tile's aux operand (16 float4 per thread) is loaded before the first batch, so a
    // tile pays one memory latency.  Frame position -> NHWC offset comes from a per-tile table.
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int grp = (warp - 6) >> 2;        // tile of the unit this warp drains
    const int gtid = (int)threadIdx.x - 192 - grp * 128;
    constexpr bool kBias = EPI == EPI_BIAS || EPI == EPI_BIAS_TANH || EPI == EPI_RESID;
    constexpr bool kAux = EPI == EPI_RESID || EPI == EPI_TANH_BWD || EPI == EPI_ADD;
    float* buf = xchg + grp * 2 * kEpiB * 64;                  // [2: hi, lo][kEpiB positions][64 ch]
    float* wrow = buf + (q >> 1) * kEpiB * 64 + (q & 1) * 32 + lane;   // this lane's channel column
    const int c4 = gtid & 15;                             // channels 4 c4 .. 4 c4 + 3 (read-back)
    const int prow = gtid >> 4;                           // position prow of each batch
    int* tab = pos_tab + grp * 128;
    const uint32_t grp_bar = 6 + grp;                     // the group (128 threads)
    // operand scales (planes.cuh): the accumulator carries wscale x in_scale, the output planes
    // out_scale (device scalars written by earlier kernels: read after pdl_wait)
    const float acc_mul = a.wscale_inv / (a.in_scale ? *a.in_scale : (MODE == MODE_PLANES ? kActPlaneScale : 1.f));
    const float out_mul = a.out_scale ? *a.out_scale : kActPlaneScale;
    int ab = 0;
    uint32_t aph = 0;
    UnitIter it(a.Co / 64, a.N, a.T);
    int cb, n, tile0, ntiles, ui = 0;
    while (it.next(cb, n, tile0, ntiles)) {
      const int u = ui++;
      const int64_t img = (int64_t)n * a.H * a.W;
      const int co = cb * 64 + 4 * c4;
      float4 bias = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kBias) bias = make_float4(__ldg(a.bias + co), __ldg(a.bias + co + 1), __ldg(a.bias + co + 2), __ldg(a.bias + co + 3));
      mbar_wait(&acc_full[ab], aph);
      tc_fence_after();
      if (a.trace && blockIdx.x < 2 && threadIdx.x == 192) a.trace[(blockIdx.x * 64 + min(u, 63)) * 8 + 2] = globaltimer_ns();
      if (grp < ntiles && !(a.dbg & 1)) {
        {
          const int f = (tile0 + grp) * a.tile + gtid;
          const int y = f / Wp, X = f - y * Wp;
          asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");   // the last tile's readers are done
          tab[gtid] = (gtid < a.tile && y < a.H && X >= 1 && X <= a.W) ? (y * a.W + (X - 1)) * a.Co : -1;
          asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");   // table visible
        }
        const uint32_t tcol = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * kS * 128 + grp * a.tile);
        const float* auxb = kAux ? a.aux + img * a.Co + co : nullptr;
        float* outb = a.out ? a.out + img * a.Co + co : nullptr;   // null: the planes alone
        const bool planes = a.p0 != nullptr;
        uint16_t* p0b = planes ? a.p0 + img * a.Co + co : nullptr;
        uint16_t* p1b = planes ? a.p1 + img * a.Co + co : nullptr;
        const int fvalid = min(a.tile, a.H * Wp - (tile0 + grp) * a.tile);   // frame positions of this tile
        const int nb = (fvalid + kEpiB - 1) / kEpiB;                          // batches with frame positions
        float4 ax[128 / 8];                                   // [batch][j]: one float4 per position owned
        if constexpr (kAux) {
#pragma unroll
          for (int b = 0; b < 128 / kEpiB; ++b)
#pragma unroll
            for (int j = 0; j < kEpiJ; ++j) {
              const int o = b < nb ? tab[b * kEpiB + prow + 8 * j] : -1;
              ax[b * kEpiJ + j] = o >= 0 ? __ldg(reinterpret_cast<const float4*>(auxb + o)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        // batch b's accumulators are loaded while batch b - 1 is finished (double-buffered
        // registers: the TMEM load latency is off the critical path)
        uint32_t rn[kEpiB];
        if (nb > 0) {
          if constexpr (kEpiB == 16) tmem_ld16(tcol, rn);
          else tmem_ld8(tcol, *reinterpret_cast<uint32_t(*)[8]>(&rn[0]));
        }
#pragma unroll
        for (int b = 0; b < 128 / kEpiB; ++b) {
          if (b < nb) {   // group-uniform
            uint32_t r[kEpiB];
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < kEpiB; ++e) r[e] = rn[e];
            if (b + 1 < nb) {
              if constexpr (kEpiB == 16) tmem_ld16(tcol + (uint32_t)((b + 1) * kEpiB), rn);
              else tmem_ld8(tcol + (uint32_t)((b + 1) * kEpiB), *reinterpret_cast<uint32_t(*)[8]>(&rn[0]));
            }
            asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");   // buf free
#pragma unroll
            for (int e = 0; e < kEpiB; ++e) wrow[e * 64] = __uint_as_float(r[e]);
            asm volatile("bar.sync %0, 128;" ::"r"(grp_bar) : "memory");
#pragma unroll
            for (int j = 0; j < kEpiJ; ++j) {
              const int pr = prow + 8 * j;
              const int off = tab[b * kEpiB + pr];
              if (off < 0) continue;
              const float4 hv = *reinterpret_cast<const float4*>(buf + pr * 64 + 4 * c4);
              const float4 lv = *reinterpret_cast<const float4*>(buf + kEpiB * 64 + pr * 64 + 4 * c4);
              const float v[4] = {(hv.x + lv.x) * acc_mul, (hv.y + lv.y) * acc_mul, (hv.z + lv.z) * acc_mul,
                                  (hv.w + lv.w) * acc_mul};
              const float bb[4] = {bias.x, bias.y, bias.z, bias.w};
              const float4 axj = ax[b * kEpiJ + j];
              const float xa[4] = {axj.x, axj.y, axj.z, axj.w};
              float o[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if constexpr (EPI == EPI_BIAS) o[i] = v[i] + bb[i];
                else if constexpr (EPI == EPI_BIAS_TANH) o[i] = tanhf(v[i] + bb[i]);
                else if constexpr (EPI == EPI_RESID) o[i] = xa[i] + a.h * (v[i] + bb[i]);
                else if constexpr (EPI == EPI_TANH_BWD) o[i] = (a.h * v[i]) * (1.f - xa[i] * xa[i]);
                else if constexpr (EPI == EPI_ADD) o[i] = xa[i] + v[i];
                else o[i] = a.h * v[i];
              }
              if (outb) *reinterpret_cast<float4*>(outb + off) = make_float4(o[0], o[1], o[2], o[3]);
              if (planes) pack_pair4(o, out_mul, *reinterpret_cast<uint2*>(p0b + off), *reinterpret_cast<uint2*>(p1b + off));
            }
          }
        }
      }
      if (a.trace && blockIdx.x < 2 && threadIdx.x == 192) a.trace[(blockIdx.x * 64 + min(u, 63)) * 8 + 3] = globaltimer_ns();
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

// weights HWIO src[tap][ci][co] -> prepped A operand [cb][chunk][tap'][kg][128 rows][4]
// per 64-channel output block cb: row r < 64 holds w_hi[co = 64 cb + r], r >= 64 holds
// w_lo[co = 64 cb + r - 64] (TF32 mode: the same split; x enters truncated).  fprop
// (flip = 0) or dgrad (flip = 1: tap' = 8 - tap, ci' = co, co' = ci).
__global__ void prep_weights_kernel(const float* __restrict__ w, int ci_src, int co_src, int flip,
                                    float* __restrict__ out) {
  const int Ci = flip ? co_src : ci_src;
  const int Co = flip ? ci_src : co_src;   // multiple of 64
  const int64_t per_cb = 9LL * Ci * 128;
  const int64_t total = per_cb * (Co / 64);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int cb = (int)(idx / per_cb);
    const int64_t li = idx - cb * per_cb;
    const int e = (int)(li & 3);
    const int r = (int)((li >> 2) & 127);
    const int64_t rest = li >> 9;               // (chunk, tap, kg)
    const int kg = (int)(rest % 4);
    const int tap = (int)((rest / 4) % 9);
    const int chunk = (int)(rest / 36);
    const int ci = chunk * kChunk + kg * 4 + e;
    const int co = cb * 64 + (r < 64 ? r : r - 64);
    float v;
    if (!flip)
      v = w[((int64_t)tap * ci_src + ci) * co_src + co];
    else
      v = w[((int64_t)(8 - tap) * ci_src + co) * co_src + ci];
    const float h = rna_tf32(v);
    out[idx] = r < 64 ? h : v - h;
  }
}

// X3BF16 weights: [cb][chunk][tap'][kg (2)][128 rows][8 bf16]: row r < 64 holds
// W0 = bf16(w[co = 64 cb + r]), r >= 64 holds W1 = bf16(w - W0) for co = 64 cb + r - 64.
__device__ __forceinline__ __nv_bfloat16 prep_bf16x2_elem(const float* __restrict__ w, int ci_src, int co_src,
                                                          int flip, int64_t idx) {
  const int Ci = flip ? co_src : ci_src;
  const int64_t per_cb = 9LL * Ci * 128;
  {
    const int cb = (int)(idx / per_cb);
    const int64_t li = idx - cb * per_cb;
    const int e = (int)(li & 7);
    const int r = (int)((li >> 3) & 127);
    const int64_t rest = li >> 10;              // (chunk, tap, kg)
    const int kg = (int)(rest % 2);
    const int tap = (int)((rest / 2) % 9);
    const int chunk = (int)(rest / 18);
    const int ci = chunk * kChunk + kg * 8 + e;
    const int co = cb * 64 + (r < 64 ? r : r - 64);
    const float v = !flip ? w[((int64_t)tap * ci_src + ci) * co_src + co]
                          : w[((int64_t)(8 - tap) * ci_src + co) * co_src + ci];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    return r < 64 ? h : __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

__global__ void prep_weights_bf16x2_kernel(const float* __restrict__ w, int ci_src, int co_src, int flip,
                                           __nv_bfloat16* __restrict__ out) {
  const int64_t total = 9LL * ci_src * co_src * 2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    out[idx] = prep_bf16x2_elem(w, ci_src, co_src, flip, idx);
}

// Both filters of every block of a stage in one launch (plane path): filter j of block b
// (parameters at pb + b * block_stride + off[j], HWIO ci_src[j] x co_src[j]) goes to
// out + (2 b + j) * felems in the layout prep_weights_bf16x2_kernel writes.
struct FilterPair {
  int64_t off[2];
  int ci_src[2], co_src[2];
  int flip;
};

// PLANES filters: the same layout, rows r < 64 W0 = fp16(W 2^8), r >= 64 W1 = fp16(W 2^8 - W0)
// (planes.cuh: |W| < 2^7).  Co < 64 (conv_pm.cu only): R = 2 Co rows per (chunk, tap, kg), r < Co
// W0, r >= Co W1 -- for Co = 64 the same bytes, so both kernels read one prepared filter.
__device__ __forceinline__ __half prep_f16x2_elem(const float* __restrict__ w, int ci_src, int co_src, int flip,
                                                  int64_t idx) {
  const int Ci = flip ? co_src : ci_src;
  const int Co = flip ? ci_src : co_src;
  const int R = Co < 64 ? 2 * Co : 128;       // rows per (chunk, tap, kg) and output-channel block
  const int half = R / 2;
  const int64_t per_cb = 9LL * Ci * R;
  const int cb = (int)(idx / per_cb);
  const int64_t li = idx - cb * per_cb;
  const int e = (int)(li & 7);
  const int r = (int)((li >> 3) % R);
  const int64_t rest = (li >> 3) / R;         // (chunk, tap, kg)
  const int kg = (int)(rest % 2);
  const int tap = (int)((rest / 2) % 9);
  const int chunk = (int)(rest / 18);
  const int ci = chunk * kChunk + kg * 8 + e;
  const int co = cb * half + (r < half ? r : r - half);
  const float v = (!flip ? w[((int64_t)tap * ci_src + ci) * co_src + co]
                         : w[((int64_t)(8 - tap) * ci_src + co) * co_src + ci]) * kWeightPlaneScale;
  const __half h = __float2half_rn(v);
  return r < half ? h : __float2half_rn(v - __half2float(h));
}

__global__ void prep_weights_f16x2_kernel(const float* __restrict__ w, int ci_src, int co_src, int flip,
                                          __half* __restrict__ out) {
  const int64_t total = 9LL * ci_src * co_src * 2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    out[idx] = prep_f16x2_elem(w, ci_src, co_src, flip, idx);
}

__global__ void prep_filters_planes_kernel(const float* __restrict__ pb, int64_t block_stride, int nblocks,
                                           const FilterPair fp, int64_t felems, __half* __restrict__ out) {
  const int64_t total = (int64_t)nblocks * 2 * felems;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = idx / felems;
    const int b = (int)(f >> 1), j = (int)(f & 1);
    out[idx] = prep_f16x2_elem(pb + b * block_stride + fp.off[j], fp.ci_src[j], fp.co_src[j], fp.flip, idx - f * felems);
  }
}

// ---------------------------------------------------------------- host side
unsigned long long* g_trace = nullptr;
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

// X3BF16 raw halo: plain NHWC box {16 ch, W + 2, rows, 1} (64-byte rows), zero fill
// outside the image
CUtensorMap make_raw_map(const float* in, const ConvShape& s, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {(cuuint64_t)s.ci, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)s.n};
  const cuuint64_t strides[3] = {(cuuint64_t)s.ci * 4, (cuuint64_t)s.w * s.ci * 4, (cuuint64_t)s.h * s.w * s.ci * 4};
  const cuuint32_t box[4] = {(cuuint32_t)kChunk, (cuuint32_t)Wp, (cuuint32_t)rows_h, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// PLANES input: bf16 planes [2][N][H][W][C] (p1 = p0 + N H W C) viewed as 2N images in
// 8-channel groups, box {8 ch, W + 2, rows, 2 groups, 1}: the slot layout [2 kg][pos][8].
CUtensorMap make_planes_map(const void* planes, const ConvShape& s, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {8, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)(s.ci / 8), (cuuint64_t)(2 * s.n)};
  const cuuint64_t strides[4] = {(cuuint64_t)s.ci * 2, (cuuint64_t)s.w * s.ci * 2, 16,
                                 (cuuint64_t)s.h * s.w * s.ci * 2};
  const cuuint32_t box[5] = {8, (cuuint32_t)Wp, (cuuint32_t)rows_h, 2, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void*>(planes), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
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
  bool ok = false;
  int Wp, rows_h, halo_pos, T, units_per_img;
  uint32_t halo_bytes, w_tap, halo_stride, plane_bytes, raw_stride = 0;
  int raw_slots = 0, wstages = kWStages;
  bool resident = false;
  int tile = 128;
  size_t smem;
};

Plan plan_for(const ConvShape& s, int mode = MODE_X3TF32) {
  Plan p;
  if (s.co % 64 != 0 || s.ci % kChunk != 0 || s.w + 1 > 256) return p;
  // W + 1 frame columns: one zero column (x = -1) per row also serves as the previous row's
  // right pad (x = W), so 1/W of the MMA work is padding instead of 2/W
  p.Wp = s.w + 1;
  static const bool equal_units = [] {
    const char* e = std::getenv("RP_CONV_EQUAL_UNITS");
    return !(e && e[0] == '0');
  }();
  if (mode == MODE_PLANES && equal_units) {
    // equal units: the image's frame in ceil(frame / 256) units of two tiles, the tile rounded
    // up to 16 positions (32x32: 1056 = 5 units of 224 positions instead of 4 x 256 + a 32-position
    // tail unit that paid a whole unit's halo loads and MMA issue)
    const int frame = s.h * p.Wp;
    const int units = (frame + 2 * 128 - 1) / (2 * 128);
    p.tile = std::min(128, ((frame + 2 * units - 1) / (2 * units) + 15) / 16 * 16);
  }
  p.rows_h = (3 * p.Wp + p.tile * kS + p.Wp - 1) / p.Wp;
  if (p.rows_h > 256) return p;
  p.halo_pos = p.rows_h * p.Wp;
  p.T = (s.h * p.Wp + p.tile - 1) / p.tile;
  p.units_per_img = (p.T + kS - 1) / kS;
  p.halo_bytes = (uint32_t)p.halo_pos * 64u;
  p.plane_bytes = (uint32_t)p.halo_pos * 32u;
  const size_t fixed_bytes = 2 * 2 * kEpiB * 64 * 4 + 512 + 1024;   // xchg + barriers + table
  if (mode == MODE_PLANES) {
    p.w_tap = 128u * kChunk * 2u;
    p.halo_stride = (128 + 2 * (p.plane_bytes + 255) + 127) / 128 * 128;   // plane-pair slot (128 B aligned TMA targets)
    // resident filter (one co block, every (chunk, filter row) stage) + 3 halo slots (2 if short)
    const int nst = 3 * (s.ci / kChunk);
    const int res_slots = nst * 3 * (size_t)p.w_tap + fixed_bytes + 3 * (size_t)p.halo_stride <= (size_t)kMaxSmemRes ? 3 : 2;
    const size_t need_res = nst * 3 * (size_t)p.w_tap + fixed_bytes + res_slots * (size_t)p.halo_stride;
    static const bool res_off = [] {
      const char* e = std::getenv("RP_CONV_RESIDENT");
      return e && e[0] == '0';
    }();
    if (!res_off && s.co == 64 && nst <= kWResMax && need_res <= (size_t)kMaxSmemRes) {
      p.resident = true;
      p.wstages = nst;
      p.raw_slots = res_slots;
      p.smem = need_res;
      p.ok = true;
      return p;
    }
    // deepest weight ring first (the weight stream is the one the MMA waits on), then the
    // most halo slots that still fit
    p.ok = false;
    for (int wst = 6; wst >= kWStages && !p.ok; --wst)
      for (int hs = 4; hs >= 2 && !p.ok; --hs) {
        const size_t need = wst * 3 * (size_t)p.w_tap + fixed_bytes + hs * (size_t)p.halo_stride;
        if (need <= (size_t)kMaxSmem) p.wstages = wst, p.raw_slots = hs, p.smem = need, p.ok = true;
      }
    if (!p.ok) return p;
  } else if (mode == MODE_X3BF16) {
    p.w_tap = 128u * kChunk * 2u;
    p.halo_stride = (128 + 3 * (p.plane_bytes + 255) + 1023) / 1024 * 1024;   // plane slot (128 B pitch)
    p.raw_stride = (p.halo_bytes + 1023) / 1024 * 1024;
    const size_t base = 2 * (size_t)p.halo_stride + kWStages * 3 * (size_t)p.w_tap + fixed_bytes;
    p.raw_slots = base + 3 * (size_t)p.raw_stride <= (size_t)kMaxSmem ? 3 : 2;
    p.smem = base + p.raw_slots * (size_t)p.raw_stride;
  } else {
    p.w_tap = 128u * kChunk * 4u;
    p.halo_stride = (128 + p.halo_bytes + 128 + p.halo_bytes + 128 + 1023) / 1024 * 1024;
    p.smem = 2 * (size_t)p.halo_stride + kWStages * 3 * (size_t)p.w_tap + fixed_bytes;
  }
  p.ok = p.smem <= (size_t)kMaxSmem;
  return p;
}

std::mutex g_map_mu;
std::map<std::tuple<const void*, int, int, int, int, int, int>, CUtensorMap> g_maps;

// kind: 0 interleaved fp32 halo, 1 raw fp32 [pos][16], 2 bf16 plane pair
CUtensorMap cached_map(const void* in, const ConvShape& s, int Wp, int rows_h, int kind) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto key = std::make_tuple(in, s.n, s.h, s.w, s.ci, rows_h, kind);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();   // callers hold copies, never references
    const float* f = static_cast<const float*>(in);
    it = g_maps.emplace(key, kind == 2   ? make_planes_map(in, s, Wp, rows_h)
                             : kind == 1 ? make_raw_map(f, s, Wp, rows_h)
                                         : make_halo_map(f, s, Wp, rows_h))
             .first;
  }
  return it->second;
}

template <int EPI, int MODE>
void launch_cfg(const CUtensorMap& m, const TcArgs& a, size_t smem, int grid, cudaStream_t st) {
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(conv3x3_tc_kernel<EPI, MODE>), kMaxSmemRes);
  launch_pdl(conv3x3_tc_kernel<EPI, MODE>, grid, kThreads, smem, st, m, a);
}

template <int EPI>
void launch_epi(const CUtensorMap& m, const TcArgs& a, int mode, size_t smem, int grid, cudaStream_t st) {
  if (mode == MODE_PLANES)
    launch_cfg<EPI, MODE_PLANES>(m, a, smem, grid, st);
  else if (mode == MODE_X3BF16)
    launch_cfg<EPI, MODE_X3BF16>(m, a, smem, grid, st);
  else if (mode == MODE_X3TF32)
    launch_cfg<EPI, MODE_X3TF32>(m, a, smem, grid, st);
  else
    launch_cfg<EPI, MODE_TF32>(m, a, smem, grid, st);
}

}  // namespace

bool conv3x3_tc_supported(const ConvShape& s) { return plan_for(s).ok; }

void conv3x3_tc_set_trace(unsigned long long* p) { g_trace = p; }

int64_t conv3x3_tc_ws_bytes(const ConvShape& s) { return 9LL * s.ci * 2 * s.co * 4 + 256; }

void prep_filters_planes(const float* pb, int64_t block_stride, int nblocks, const int64_t off[2],
                         const int ci_src[2], const int co_src[2], bool dgrad, void* out, cudaStream_t st) {
  if (nblocks <= 0) return;
  FilterPair fp{};
  for (int j = 0; j < 2; ++j) fp.off[j] = off[j], fp.ci_src[j] = ci_src[j], fp.co_src[j] = co_src[j];
  fp.flip = dgrad ? 1 : 0;
  const int64_t felems = 9LL * ci_src[0] * co_src[0] * 2;
  if (9LL * ci_src[1] * co_src[1] * 2 != felems) fail(RP_ERR_INTERNAL, "prep_filters_planes: filter sizes differ");
  const int64_t total = (int64_t)nblocks * 2 * felems;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 16 * kNumSMs);
  prep_filters_planes_kernel<<<grid, 256, 0, st>>>(pb, block_stride, nblocks, fp, felems, static_cast<__half*>(out));
  RP_LAUNCHED();
}

void prep_filter_planes(const float* w_hwio, int ci_src, int co_src, bool dgrad, void* out, cudaStream_t st) {
  const int64_t total = 9LL * ci_src * co_src * 2;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 16 * kNumSMs);
  prep_weights_f16x2_kernel<<<grid, 256, 0, st>>>(w_hwio, ci_src, co_src, dgrad ? 1 : 0, static_cast<__half*>(out));
  RP_LAUNCHED();
}

void conv3x3_fwd_tc(const ConvShape& s, const float* in, const float* w_hwio, bool dgrad_weights, const float* bias,
                    const float* aux, float h, int epi, float* out, int mode, void* ws, cudaStream_t st,
                    void* out_planes, const void* in_planes, const void* wprep, const float* in_scale,
                    const float* out_scale) {
  if (s.pixels() == 0) return;
  if (in_planes) mode = MODE_PLANES;
  const Plan p = plan_for(s, mode);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_fwd_tc: unsupported shape");
  // the weight tensor handed in is HWIO of the *forward* conv; for dgrad it has
  // (ci_src, co_src) = (s.co, s.ci)
  const int ci_src = dgrad_weights ? s.co : s.ci;
  const int co_src = dgrad_weights ? s.ci : s.co;
  const int64_t total = 9LL * s.ci * 2 * s.co;
  const int pgrid = (int)std::min<int64_t>(ceil_div(total, 256), 16 * kNumSMs);
  if (wprep && mode != MODE_PLANES) fail(RP_ERR_INTERNAL, "conv3x3_fwd_tc: prepared filters are plane-mode only");
  if (wprep) {
    // prepared by prep_filters_planes for the whole stage
  } else if (mode == MODE_PLANES) {
    prep_weights_f16x2_kernel<<<pgrid, 256, 0, st>>>(w_hwio, ci_src, co_src, dgrad_weights ? 1 : 0,
                                                     static_cast<__half*>(ws));
    RP_LAUNCHED();
  } else if (mode == MODE_X3BF16) {
    prep_weights_bf16x2_kernel<<<pgrid, 256, 0, st>>>(w_hwio, ci_src, co_src, dgrad_weights ? 1 : 0,
                                                      static_cast<__nv_bfloat16*>(ws));
    RP_LAUNCHED();
  } else {
    prep_weights_kernel<<<pgrid, 256, 0, st>>>(w_hwio, ci_src, co_src, dgrad_weights ? 1 : 0,
                                               static_cast<float*>(ws));
    RP_LAUNCHED();
  }
  const float* wp = static_cast<const float*>(wprep ? wprep : ws);
  TcArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Ci = s.ci;
  a.Co = s.co;
  a.Wp = p.Wp;
  a.rows_h = p.rows_h;
  a.T = p.T;
  a.num_tiles = (s.co / 64) * s.n * p.T;
  a.halo_pos = p.halo_pos;
  a.nchunks = s.ci / kChunk;
  a.halo_bytes = p.halo_bytes;
  a.halo_stride = p.halo_stride;
  a.w_tap = p.w_tap;
  a.plane_bytes = p.plane_bytes;
  a.raw_stride = p.raw_stride;
  a.raw_slots = p.raw_slots;
  a.wstages = p.wstages;
  a.resident = p.resident ? 1 : 0;
  a.tile = p.tile;
  a.h = h;
  a.w = wp;
  a.bias = bias;
  a.aux = aux;
  a.out = out;
  a.p0 = static_cast<uint16_t*>(out_planes);
  a.p1 = out_planes ? a.p0 + s.pixels() * s.co : nullptr;
  if (in_scale && mode != MODE_PLANES) fail(RP_ERR_INTERNAL, "conv3x3_fwd_tc: an input scale needs plane input");
  a.in_scale = in_scale;
  a.out_scale = out_scale;
  a.wscale_inv = mode == MODE_PLANES ? kWeightPlaneScaleInv : 1.f;
  a.trace = g_trace;
  static const int dbg = [] {
    const char* e = std::getenv("RP_CONV_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
  const CUtensorMap m = mode == MODE_PLANES ? cached_map(in_planes, s, p.Wp, p.rows_h, 2)
                                              : cached_map(in, s, p.Wp, p.rows_h, mode == MODE_X3BF16 ? 1 : 0);
  const int grid = std::min(a.num_tiles, kNumSMs);
  switch (epi) {
    case EPI_BIAS: launch_epi<EPI_BIAS>(m, a, mode, p.smem, grid, st); break;
    case EPI_BIAS_TANH: launch_epi<EPI_BIAS_TANH>(m, a, mode, p.smem, grid, st); break;
    case EPI_RESID: launch_epi<EPI_RESID>(m, a, mode, p.smem, grid, st); break;
    case EPI_TANH_BWD: launch_epi<EPI_TANH_BWD>(m, a, mode, p.smem, grid, st); break;
    case EPI_ADD: launch_epi<EPI_ADD>(m, a, mode, p.smem, grid, st); break;
    default: launch_epi<EPI_SCALE>(m, a, mode, p.smem, grid, st); break;
  }
  RP_LAUNCHED();
}

}  // namespace rp::k
