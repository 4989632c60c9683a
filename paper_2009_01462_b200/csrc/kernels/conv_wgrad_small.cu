// tcgen05 weight gradient for the 16-channel plane path (config C1: C = hidden = 16):
//
//   gW[tap][ci][co] = scale * sum_p x[p + off(tap)][ci] * g[p][co],  gb[co] = scale * sum_p g[p][co]
//
// (block_vjp's matmul(a^T, upstream) / matmul(x^T, dpre) and col_sum, network.cpp:98-103,
// generalised to 3x3 taps), from the fp16 plane pairs x 2^7 = x0 + x1, g s = g0 + g1 the plane
// convs (conv_pm.cu) write.  conv_wgrad_planes.cu tiles 64-channel blocks; here a 16-channel
// operand is too narrow for that tiling, so the positions p are the MMA's K and both operands
// are MN-major views of the same TMA slabs the convs read ([8-channel group][position][8]):
//   A = [g0; g1]           M = 64 rows (2 Co; Co = 16 pads with rows nobody reads),
//   B = [x0; x1] shifted   N = 32 rows per tap (a shift by one position is +16 B of start),
// one M64 x N32 x K16 MMA per (16 positions, tap) into that tap's 32 TMEM columns: all four
// products g0x0 + g1x0 + g0x1 + g1x1, added in the epilogue.  The bias sums ride on the centre
// tap's MMA: its B gets an extra 8-row group of ones (N = 40).
//  * work: the frame tiles (H rows x (W + 1) columns, 128 positions, as the convs) of all images
//    in contiguous ranges per CTA; the accumulators stay in TMEM for the CTA's whole range, then
//    go to per-CTA partials; a fixed-order fp64 reduce (deterministic, like conv_wgrad_planes.cu).
//  * warp roles (256 threads, persistent): w0 TMA producer, w1 MMA issuer, w4-7 epilogue.
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

constexpr int kThreads = 256;
constexpr int kTile = 128;           // frame positions per work item (8 K-steps)
constexpr int kMaxSlots = 6;
constexpr int kMaxSmem = 227 * 1024;
constexpr int kTapCols = 32;         // TMEM columns per tap: [x0 kg0, x0 kg1, x1 kg0, x1 kg1] x 8
constexpr int kBiasTap = 4;          // the centre tap carries the ones group (its shift is >= 0)

struct WsArgs {
  int N, H, W, Co, Wp, rows_h, T, ntiles, slots;
  uint32_t S;               // bytes per 8-channel group region of a slot (rows_h x Wp x 16)
  uint32_t slot_bytes;
  int ga;                   // g groups (2 Co / 8); the x groups follow them (Co = 16: A's rows 32-63,
                            // which nobody reads, are the x groups -- finite data)
  float* part;              // [grid][2 g planes][9][16 ci][Co]
  float* part_bias;         // [grid][2][Co]
  // reduce
  float* gw;
  float* gb;
  double scale;
  const float* gscale;      // the g planes' scale (device scalar; null = kActPlaneScale)
  int dbg;                  // diagnostics (RP_WGRAD_SMALL_DBG): 1 no MMA, 2 no TMA
};

// TMEM column block of tap t: the centre tap last (its N = 40 reaches past 32 columns)
__host__ __device__ constexpr int tap_slot(int t) { return t < kBiasTap ? t : (t == kBiasTap ? 8 : t - 1); }

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_small_kernel(const __grid_constant__ CUtensorMap mx0, const __grid_constant__ CUtensorMap mx1,
                       const __grid_constant__ CUtensorMap mg0, const __grid_constant__ CUtensorMap mg1,
                       const WsArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  const int lane = threadIdx.x & 31;
  // slot: [ga groups: g0 kg.., g1 kg..][4 groups: x0 kg0, x0 kg1, x1 kg0, x1 kg1][ones], S bytes each;
  // x's shift -1 reads the last g position before it (finite; its partner g is a pad column, 0)
  auto slot = [&](int s) { return smem + s * a.slot_bytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.slots * a.slot_bytes);
  uint64_t* full = bars;                  // [kMaxSlots]
  uint64_t* empty = bars + kMaxSlots;     // [kMaxSlots]
  uint64_t* done = bars + 2 * kMaxSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxSlots + 1);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
    prefetch_tmap(&mx0);
    prefetch_tmap(&mx1);
    prefetch_tmap(&mg0);
    prefetch_tmap(&mg1);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  // the ones group of every slot = 1.0 (the boxes fill the g and x groups completely)
  for (int s = 0; s < a.slots; ++s) {
    uint4* ones = reinterpret_cast<uint4*>(slot(s) + (a.ga + 4) * a.S);
    for (uint32_t i = threadIdx.x; i < a.S / 16; i += blockDim.x) ones[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int Wp = a.Wp;
  const int t_beg = (int)((int64_t)a.ntiles * blockIdx.x / gridDim.x);
  const int t_end = (int)((int64_t)a.ntiles * (blockIdx.x + 1) / gridDim.x);
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    // ===================== TMA producer =====================
    int s = 0;
    uint32_t ph = 0;
    for (int t = t_beg; t < t_end; ++t) {
      const int n = t / a.T, f0 = (t - n * a.T) * kTile;
      const int y0 = f0 / Wp;
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* b = slot(s);
        const uint32_t gplane = (uint32_t)(a.Co / 8) * a.S, xplane = 2 * a.S;   // one plane's 8-channel groups
        if (a.dbg & 2) {
          mbar_arrive(&full[s]);
        } else {
        mbar_arrive_expect_tx(&full[s], 2 * gplane + 2 * xplane);
        // g at its own positions (rows from y0), x with the one-row / one-column halo
        tma_load_5d(&mg0, &full[s], b, 0, -1, y0, 0, n);
        tma_load_5d(&mg1, &full[s], b + gplane, 0, -1, y0, 0, n);
        tma_load_5d(&mx0, &full[s], b + a.ga * a.S, 0, -1, y0 - 1, 0, n);
        tma_load_5d(&mx1, &full[s], b + a.ga * a.S + xplane, 0, -1, y0 - 1, 0, n);
        }
      }
      __syncwarp();
      if (++s == a.slots) s = 0, ph ^= 1;
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t id = idesc(0, 64, kTapCols, 1, 1);
    const uint32_t id_b = idesc(0, 64, kTapCols + 8, 1, 1);
    int s = 0;
    uint32_t ph = 0;
    bool first = true;
    for (int t = t_beg; t < t_end; ++t) {
      const int n = t / a.T, f0 = (t - n * a.T) * kTile;
      const int c0 = f0 - (f0 / Wp) * Wp;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        // MN-major, no swizzle: 8 positions x 16 B core matrices (LBO 128 B along K), 8-channel
        // groups S apart (SBO)
        const uint64_t da = desc_kmajor_interleave(smem_u32(slot(s)), 128, a.S) + (uint64_t)c0;
        const uint64_t dx = desc_kmajor_interleave(smem_u32(slot(s) + a.ga * a.S), 128, a.S);
        for (int k = 0; k < ((a.dbg & 1) ? 0 : kTile / 16); ++k) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int dy = tap / 3, dxx = tap % 3;
            const uint64_t db = dx + (uint64_t)(c0 + dy * Wp + dxx - 1 + 16 * k);
            mma_f16(tmem_base + (uint32_t)(tap_slot(tap) * kTapCols), da + (uint64_t)(16 * k), db,
                    tap == kBiasTap ? id_b : id, (first && k == 0) ? 0u : 1u);
          }
        }
        mma_commit(&empty[s]);
      }
      __syncwarp();
      first = false;
      if (++s == a.slots) s = 0, ph ^= 1;
    }
    if (elect_one()) {
      if (t_end > t_beg) mma_commit(done);
      else mbar_arrive(done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    // M = 64 accumulator rows live in TMEM lanes 32 (r / 16) + r % 16 (tools/umma_m64_layout.py):
    // warp q (lane quadrant) holds rows 16 q .. 16 q + 15 in its lanes 0..15; row r = g plane
    // r / Co, output channel r % Co.
    const int q = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    const int r = 16 * q + (lane & 15);
    const bool live = lane < 16 && r < 2 * a.Co && t_end > t_beg;
    const int gp = r / a.Co, co = r % a.Co;
    const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16);
    float* part = a.part + ((int64_t)blockIdx.x * 2 + gp) * 9 * 16 * a.Co;
#pragma unroll 1
    for (int tap = 0; tap < 9; ++tap) {
      uint32_t v[16], w[16];
      tmem_ld16(tq + (uint32_t)(tap_slot(tap) * kTapCols), v);        // x0 ci 0..15
      tmem_ld16(tq + (uint32_t)(tap_slot(tap) * kTapCols + 16), w);   // x1 ci 0..15
      tmem_wait_ld();
      if (live)
        for (int ci = 0; ci < 16; ++ci)
          part[(tap * 16 + ci) * a.Co + co] = __uint_as_float(v[ci]) + __uint_as_float(w[ci]);
    }
    uint32_t b[8];
    tmem_ld8(tq + (uint32_t)(tap_slot(kBiasTap) * kTapCols + kTapCols), b);
    tmem_wait_ld();
    if (lane < 16 && r < 2 * a.Co)
      a.part_bias[((int64_t)blockIdx.x * 2 + gp) * a.Co + co] = t_end > t_beg ? __uint_as_float(b[0]) : 0.f;
    if (!live && lane < 16 && r < 2 * a.Co)
      for (int i = 0; i < 9 * 16; ++i) part[i * a.Co + co] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// gw = scale / (kActPlaneScale gs) sum_cta sum_gplane part, gb = scale / gs sum_cta sum_gplane
// bias part, in fp64 and a fixed order (deterministic): a CTA owns 32 consecutive outputs (coalesced
// loads); its 32 warps sum fixed 32nds of the partials, combined in order.
__global__ void __launch_bounds__(1024) wgrad_small_reduce_kernel(const WsArgs a, int grid) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ double red[32][33];
  const int nw = 9 * 16 * a.Co;
  const int lane = threadIdx.x & 31, wg = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const bool bias = i >= nw;
  const float* src = bias ? a.part_bias + (i - nw) : a.part + i;
  const int64_t cstride = bias ? 2LL * a.Co : 2LL * nw;   // per CTA
  const int64_t gstride = bias ? a.Co : nw;               // per g plane
  double acc = 0.0;
  if (i < nw + a.Co) {
    const int c_lo = grid * wg / 32, c_hi = grid * (wg + 1) / 32;
    float v[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c_lo + j;
      v[2 * j] = c < c_hi ? src[c * cstride] : 0.f;
      v[2 * j + 1] = c < c_hi ? src[c * cstride + gstride] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) acc += (double)v[j];
    for (int c = c_lo + 8; c < c_hi; ++c) acc += (double)src[c * cstride] + (double)src[c * cstride + gstride];
  }
  red[wg][lane] = acc;
  __syncthreads();
  if (wg == 0 && i < nw + a.Co && (!bias || a.gb)) {
    double s = 0.0;
    for (int j = 0; j < 32; ++j) s += red[j][lane];
    const double gs = a.gscale ? (double)*a.gscale : (double)kActPlaneScale;
    if (bias) a.gb[i - nw] = (float)(s * a.scale / gs);
    else a.gw[i] = (float)(s * a.scale / ((double)kActPlaneScale * gs));
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

// one fp16 plane [N][H][W][C] in 8-channel groups; box {8 ch, W + 1 columns from x = -1, rows_h
// rows, C / 8 groups, 1 image} -> [group][rows_h][W + 1][8]
CUtensorMap make_map(const void* planes, int n, int h, int w, int c, int Wp, int rows_h) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {8, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)(c / 8), (cuuint64_t)n};
  const cuuint64_t strides[4] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, 16, (cuuint64_t)h * w * c * 2};
  const cuuint32_t box[5] = {8, (cuuint32_t)Wp, (cuuint32_t)rows_h, (cuuint32_t)(c / 8), 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void*>(planes), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

std::mutex g_map_mu;
std::map<std::tuple<const void*, int, int, int, int, int>, CUtensorMap> g_maps;

CUtensorMap cached_map(const void* p, int n, int h, int w, int c, int Wp, int rows_h) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto key = std::make_tuple(p, n, h, w, c, rows_h);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    if (g_maps.size() > 4096) g_maps.clear();   // callers hold copies, never references
    it = g_maps.emplace(key, make_map(p, n, h, w, c, Wp, rows_h)).first;
  }
  return it->second;
}

struct Plan {
  bool ok = false;
  int Wp, rows_h, T, ga, slots, grid;
  uint32_t S, slot_bytes;
  size_t smem;
};

Plan plan(const ConvShape& s) {
  Plan p;
  if (s.ci != 16 || !(s.co == 16 || s.co == 32) || s.w + 1 > 256 || s.n < 1) return p;
  p.Wp = s.w + 1;
  // g reads positions [c0, c0 + 128) from row y0, x [c0 - 1, c0 + 2 Wp + 128] from row y0 - 1
  p.rows_h = (p.Wp - 1 + kTile + 2 * p.Wp + 1 + p.Wp - 1) / p.Wp;
  // the group stride of a box (rows_h Wp 16 B) is also the slot's: a multiple of 128 B keeps every
  // TMA destination 128-byte aligned
  while ((p.rows_h * p.Wp) % 8) ++p.rows_h;
  if (p.rows_h > 256) return p;
  p.T = (s.h * p.Wp + kTile - 1) / kTile;
  p.S = (uint32_t)(p.rows_h * p.Wp * 16);
  p.ga = 2 * s.co / 8;
  p.slot_bytes = (p.ga + 5) * p.S;
  p.slot_bytes = (p.slot_bytes + 127u) & ~127u;
  const size_t fixed = 256;
  for (int sl = kMaxSlots; sl >= 2 && !p.ok; --sl) {
    const size_t need = (size_t)sl * p.slot_bytes + fixed;
    if (need <= (size_t)kMaxSmem) p.slots = sl, p.smem = need, p.ok = true;
  }
  p.grid = std::min(kNumSMs, s.n * p.T);
  return p;
}

int64_t part_floats(const Plan& p, const ConvShape& s) { return (int64_t)p.grid * 2 * (9 * 16 * s.co + s.co); }

}  // namespace

bool conv3x3_wgrad_small_supported(const ConvShape& s) { return plan(s).ok; }

int64_t conv3x3_wgrad_small_ws_bytes(const ConvShape& s) {
  const Plan p = plan(s);
  return p.ok ? part_floats(p, s) * 4 + 256 : 0;
}

void conv3x3_wgrad_small(const ConvShape& s, const void* x0, const void* x1, const void* g0, const void* g1,
                         float scale, float* gw, float* gb, void* ws, cudaStream_t st, const float* gscale) {
  if (s.pixels() == 0) {
    RP_CUDA(cudaMemsetAsync(gw, 0, 9LL * s.ci * s.co * 4, st));
    if (gb) RP_CUDA(cudaMemsetAsync(gb, 0, (size_t)s.co * 4, st));
    return;
  }
  const Plan p = plan(s);
  if (!p.ok) fail(RP_ERR_INTERNAL, "conv3x3_wgrad_small: unsupported shape");
  WsArgs a{};
  a.N = s.n;
  a.H = s.h;
  a.W = s.w;
  a.Co = s.co;
  a.Wp = p.Wp;
  a.rows_h = p.rows_h;
  a.T = p.T;
  a.ntiles = s.n * p.T;
  a.slots = p.slots;
  a.S = p.S;
  a.slot_bytes = p.slot_bytes;
  a.ga = p.ga;
  a.part = static_cast<float*>(ws);
  a.part_bias = a.part + (int64_t)p.grid * 2 * 9 * 16 * s.co;
  a.gw = gw;
  a.gb = gb;
  a.scale = scale;
  a.gscale = gscale;
  static const int dbg = [] {
    const char* e = std::getenv("RP_WGRAD_SMALL_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
  const CUtensorMap mx0 = cached_map(x0, s.n, s.h, s.w, s.ci, p.Wp, p.rows_h);
  const CUtensorMap mx1 = cached_map(x1, s.n, s.h, s.w, s.ci, p.Wp, p.rows_h);
  const CUtensorMap mg0 = cached_map(g0, s.n, s.h, s.w, s.co, p.Wp, p.rows_h);
  const CUtensorMap mg1 = cached_map(g1, s.n, s.h, s.w, s.co, p.Wp, p.rows_h);
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(wgrad_small_kernel), kMaxSmem);
  launch_pdl(wgrad_small_kernel, p.grid, kThreads, p.smem, st, mx0, mx1, mg0, mg1, a);
  RP_LAUNCHED();
  const int total = 9 * 16 * s.co + s.co;
  launch_pdl(wgrad_small_reduce_kernel, ceil_div(total, 32), 1024, 0, st, a, p.grid);
  RP_LAUNCHED();
}

}  // namespace rp::k
