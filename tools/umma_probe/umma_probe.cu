// Diagnostic tool, NOT part of the product library (built separately by
// tools/umma_probe/build.sh into tools/umma_probe/librp_probe.so).
// One tcgen05.mma (M=128, N=16, K=8, tf32) on known operands in a chosen
// shared-memory layout, to pin down UMMA descriptor semantics on the device.  Exposed
// as rp_debug_umma_probe (tests only; never on the training path).
#include "common.cuh"
#include "kernels/umma.cuh"
#include <cuda_fp16.h>

// standalone: the product library's launch counter is not linked in
namespace rp {
__attribute__((weak)) void note_launch() {}
}

namespace rp::k {

namespace {

using namespace rp::umma;

// A[m][k] = a_src[m*8 + k], B[n][k] = b_src[n*8 + k]; D = A B^T (128 x 16).
// mode 0: A, B K-major interleave;  mode 1: A, B MN-major interleave.
__global__ void umma_probe_kernel(const float* a_src, const float* b_src, int mode, uint32_t a_lbo, uint32_t a_sbo,
                                  uint32_t b_lbo, uint32_t b_sbo, float* out) {
  __shared__ __align__(1024) float sa[128 * 8];
  __shared__ __align__(1024) float sb[16 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    int idx;
    if ((mode & 1) == 0)  // K-major: core (8 rows x 4 k); k-core stride a_lbo, row-group stride a_sbo
      idx = (k / 4) * (a_lbo / 4) + (m / 8) * (a_sbo / 4) + (m % 8) * 4 + (k % 4);
    else            // MN-major: core (8 k x 4 m); k-group stride a_lbo, m-group stride a_sbo
      idx = (k / 8) * (a_lbo / 4) + (m / 4) * (a_sbo / 4) + (k % 8) * 4 + (m % 4);
    sa[idx] = a_src[i];
  }
  for (int i = tid; i < 16 * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8;
    int idx;
    if ((mode & 1) == 0)
      idx = (k / 4) * (b_lbo / 4) + (n / 8) * (b_sbo / 4) + (n % 8) * 4 + (k % 4);
    else
      idx = (k / 8) * (b_lbo / 4) + (n / 4) * (b_sbo / 4) + (k % 8) * 4 + (n % 4);
    sb[idx] = b_src[i];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<32>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    // mode bit 1: swap the LBO / SBO descriptor fields (placement unchanged)
    const bool sw = mode & 2;
    const uint64_t da = sw ? desc_kmajor_interleave(smem_u32(sa), a_sbo, a_lbo)
                           : desc_kmajor_interleave(smem_u32(sa), a_lbo, a_sbo);
    const uint64_t db = sw ? desc_kmajor_interleave(smem_u32(sb), b_sbo, b_lbo)
                           : desc_kmajor_interleave(smem_u32(sb), b_lbo, b_sbo);
    mma_tf32(tmem, da, db, idesc(2, 128, 16, mode & 1, mode & 1), 0u);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = tid / 32;
  uint32_t r[16];
  tmem_ld16(tmem + ((uint32_t)(w * 32) << 16), r);
  tmem_wait_ld();
  for (int j = 0; j < 16; ++j) out[(w * 32 + (tid % 32)) * 16 + j] = __uint_as_float(r[j]);
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

// SW128_32B MN-major tf32 probe: A = 128 channels (4 groups of 32) x 8 positions, B = 32
// channels x 8 positions, rows (positions) 128 B apart starting `off` rows into a
// 1024-aligned buffer; 32-byte granules XOR-swizzled with the absolute row index mod 4.
__global__ void umma_probe_sw32_kernel(const float* a_src, const float* b_src, int off, int base_field, int swz_abs,
                                       float* out) {
  __shared__ __align__(1024) float sa[4 * 16 * 32];   // 4 groups x 16 rows x 32 floats
  __shared__ __align__(1024) float sb[16 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * 16 * 32; i += blockDim.x) sa[i] = 0.f;
  for (int i = tid; i < 16 * 32; i += blockDim.x) sb[i] = 0.f;
  __syncthreads();
  auto place = [&](float* base, int group_bytes, int m, int k, float v) {
    const int g = m / 32, c = m % 32;
    const int row = off + k;                       // row index within the group's block
    const int rphase = swz_abs ? (row & 3) : (k & 3);
    const int gran = (c / 8) ^ rphase;
    const int byte = g * group_bytes + row * 128 + gran * 32 + (c % 8) * 4;
    base[byte / 4] = v;
  };
  for (int i = tid; i < 128 * 8; i += blockDim.x) place(sa, 16 * 128, i / 8, i % 8, a_src[i]);
  for (int i = tid; i < 32 * 8; i += blockDim.x) place(sb, 16 * 128, i / 8, i % 8, b_src[i]);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<32>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint64_t da = desc_general(smem_u32(sa) + off * 128, 16 * 128, 512, 1, base_field);
    const uint64_t db = desc_general(smem_u32(sb) + off * 128, 16 * 128, 512, 1, base_field);
    mma_tf32(tmem, da, db, idesc(2, 128, 32, 1, 1), 0u);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = tid / 32;
  for (int h = 0; h < 2; ++h) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + h * 16, r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) out[(w * 32 + (tid % 32)) * 32 + h * 16 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

}  // namespace

void umma_probe(const float* a, const float* b, int mode, uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo,
                uint32_t b_sbo, float* out, cudaStream_t st) {
  umma_probe_kernel<<<1, 128, 0, st>>>(a, b, mode, a_lbo, a_sbo, b_lbo, b_sbo, out);
  RP_LAUNCHED();
}

}  // namespace rp::k

extern "C" int rp_debug_umma_probe_sw32(const float* a, const float* b, int off, int base_field, int swz_abs,
                                        float* out) {
  try {
    rp::k::umma_probe_sw32_kernel<<<1, 128>>>(a, b, off, base_field, swz_abs, out);
    RP_LAUNCHED();
    RP_CUDA(cudaDeviceSynchronize());
    return 0;
  } catch (const rp::Error& e) {
    return e.code;
  }
}

extern "C" int rp_debug_umma_probe(const float* a, const float* b, int mode, uint32_t a_lbo, uint32_t a_sbo,
                                   uint32_t b_lbo, uint32_t b_sbo, float* out) {
  try {
    rp::k::umma_probe(a, b, mode, a_lbo, a_sbo, b_lbo, b_sbo, out, nullptr);
    RP_CUDA(cudaDeviceSynchronize());
    return 0;
  } catch (const rp::Error& e) {
    return e.code;
  }
}

// ---------------------------------------------------------------------------
// MMA throughput microbenchmark: every CTA issues `reps` back-to-back tcgen05.mma of
// one configuration on fixed smem operands; cycles per MMA -> out[blockIdx.x].
// cfg: fmt (0 f16, 1 bf16, 2 tf32), N, layout (0 interleave, 2 SW128), a/b major.
namespace rp::k {
namespace {
__global__ void __launch_bounds__(128, 1) umma_bench_kernel(int fmt, int N, int layout, int a_mn, int b_mn, int reps,
                                                            int nacc, int nops, int chain, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  if (tid == 0) umma::mbar_init(&bar2, 1);
  for (int i = tid; i < 192 * 1024 / 4; i += 128) {
    uint32_t v = 0x3c003c00u;
    if (b_mn == 2) {   // pseudo-random finite fp32 in [1, 2) with random sign / mantissa
      uint32_t h = (uint32_t)i * 2654435761u;
      h ^= h >> 15;
      h *= 2246822519u;
      h ^= h >> 13;
      v = 0x3f800000u | (h & 0x807fffffu);
    }
    reinterpret_cast<uint32_t*>(sm)[i] = v;
  }
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_barrier_init();
  }
  if (tid < 32) umma::tmem_alloc<512>(&slot);
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = slot;
  const int warp_u = __shfl_sync(0xffffffffu, tid / 32, 0);   // warp-uniform for the compiler
  if (warp_u == 0) {   // whole warp runs the issue loop; one elected lane issues
    const uint32_t a0 = umma::smem_u32(sm), b0 = umma::smem_u32(sm + 32 * 1024);
    uint64_t da, db;
    if (layout == 0 || layout == 4) {  // interleave: K-major lbo = rows*16, sbo = 128 (4: M = 64)
      da = umma::desc_general(a0, 128 * 16, 128, 0, 0);
      db = umma::desc_general(b0, N * 16, 128, 0, 0);
    } else if (layout == 1 && a_mn) {   // SW128_32B MN-major: 32-element groups 8 KB apart
      da = umma::desc_general(a0, 8192, 512, 1, 0);
      db = umma::desc_general(b0, 8192, 512, 1, 0);
    } else if (layout == 3) {            // as layout 1 with the wgrad kernel's slab strides
      da = umma::desc_general(a0, 9216, 512, 1, 0);
      db = umma::desc_general(umma::smem_u32(sm + 40 * 1024) + 1024, 18432, 512, 1, 0);
    } else if (layout == 6) {            // SW32 K-major: 8 rows x 32 B atoms, sbo = 256
      da = umma::desc_general(a0, 16, 256, 6, 0);
      db = umma::desc_general(b0, 16, 256, 6, 0);
    } else {            // SW128 K-major: sbo = 1024
      da = umma::desc_general(a0, 16, 1024, layout, 0);
      db = umma::desc_general(b0, 16, 1024, layout, 0);
    }
    const uint32_t id = umma::idesc(fmt, layout == 4 ? 64 : 128, N, a_mn, b_mn);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const long long t0 = clock64();
    if (nops == 86 || nops == 85) {
      // bf16: A reused by 4 MMAs (86: collector fill/use/use/lastuse, 85: plain), B rotating
      for (int r = 0; r < reps; r += 4) {
        if (umma::elect_one()) {
          if (nops == 86) {
            umma::mma_f16_c<1>(tm, da, db, id, r > 0);
            umma::mma_f16_c<2>(tm + N, da, db + 256, id, r > 0);
            umma::mma_f16_c<2>(tm, da, db + 512, id, 1);
            umma::mma_f16_c<3>(tm + N, da, db + 768, id, 1);
          } else {
            umma::mma_f16(tm, da, db, id, r > 0);
            umma::mma_f16(tm + N, da, db + 256, id, r > 0);
            umma::mma_f16(tm, da, db + 512, id, 1);
            umma::mma_f16(tm + N, da, db + 768, id, 1);
          }
        }
        __syncwarp();
      }
    } else if (nops == 98) {
      // A reused by 4 MMAs (collector fill/use/use/lastuse), B rotating over 4 regions
      for (int r = 0; r < reps; r += 4) {
        if (umma::elect_one()) {
          umma::mma_tf32_c<1>(tm, da, db, id, r > 0);
          umma::mma_tf32_c<2>(tm + N, da, db + 256, id, r > 0);
          umma::mma_tf32_c<2>(tm, da, db + 512, id, 1);
          umma::mma_tf32_c<3>(tm + N, da, db + 768, id, 1);
        }
        __syncwarp();
      }
    } else if (nops == 89 || nops == 88 || nops == 87) {
      // conv_tc fprop pattern (88: without the collector): A = weights [kg][128][4] (LBO
      // 2 KB), 3 taps x 2 k-steps per stage; B = halo K-major interleave with LBO =
      // chain*16 (halo positions), x_hi at 64 KB, x_lo at 96 KB, 2 tiles of 128 positions
      const uint32_t w0 = umma::smem_u32(sm), xh = umma::smem_u32(sm + 64 * 1024), xl = umma::smem_u32(sm + 96 * 1024);
      const uint32_t kgx = (uint32_t)chain * 16u;
      const uint64_t dw = umma::desc_kmajor_interleave(w0, 2048, 128);
      const uint64_t bh = umma::desc_kmajor_interleave(xh, kgx, 128);
      const uint64_t bl = umma::desc_kmajor_interleave(xl, kgx, 128);
      const uint32_t idn = umma::idesc(2, 128, 128);
      const uint64_t xj = (uint64_t)((2 * kgx) >> 4);
      int dy = 0;
      for (int r = 0; r < reps; r += 24) {
        const uint64_t row = (uint64_t)(dy * 34 + 5);
        if (umma::elect_one()) {
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint64_t da = dw + dx * 512 + j * 256;
              const uint64_t b0 = row + dx + j * xj;
              if (nops != 88) {
                umma::mma_tf32_c<1>(tm, da, bh + b0, idn, 1u);
                umma::mma_tf32_c<2>(tm, da, bl + b0, idn, 1u);
                umma::mma_tf32_c<2>(tm + 128, da, bh + b0 + 128, idn, 1u);
                umma::mma_tf32_c<3>(tm + 128, da, bl + b0 + 128, idn, 1u);
              } else {
                umma::mma_tf32(tm, da, bh + b0, idn, 1u);
                umma::mma_tf32(tm, da, bl + b0, idn, 1u);
                umma::mma_tf32(tm + 128, da, bh + b0 + 128, idn, 1u);
                umma::mma_tf32(tm + 128, da, bl + b0 + 128, idn, 1u);
              }
            }
          }
          if (nops == 87) umma::mma_commit(&bar2);   // 87: commit after every stage (as conv_tc)
        }
        __syncwarp();
        if (++dy == 3) dy = 0;
      }
    } else if (nops == 80 || nops == 81 || nops == 82) {
      // conv_tc PLANES pattern (bf16): A = weights [kg 2][128][8] (LBO 2 KB) per tap, B = plane
      // pair (x0 at 64 KB, x1 at 96 KB), K-major interleave with LBO = chain * 16 (halo
      // positions), N = 256; per filter row 3 taps x {x0 fill, x1 lastuse}.  80: B shifted by
      // dy * 34 + dx - 1 positions as in the kernel; 81: no shifts (B 128 B aligned); 82: as 80
      // without the collector
      const uint32_t w0 = umma::smem_u32(sm), xh = umma::smem_u32(sm + 64 * 1024), xl = umma::smem_u32(sm + 96 * 1024);
      const uint32_t kgx = (uint32_t)chain * 16u;
      const uint64_t dw = umma::desc_kmajor_interleave(w0, 2048, 128);
      const uint64_t bh = umma::desc_kmajor_interleave(xh, kgx, 128);
      const uint64_t bl = umma::desc_kmajor_interleave(xl, kgx, 128);
      const uint32_t idn = umma::idesc(1, 128, 256);
      int dy = 0;
      for (int r = 0; r < reps; r += 6) {
        const uint64_t row = nops == 81 ? 0 : (uint64_t)(dy * 34 + 1);
        if (umma::elect_one()) {
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const uint64_t da = dw + dx * 256;
            const uint64_t b0 = row + (nops == 81 ? 0 : dx);
            if (nops == 82) {
              umma::mma_f16(tm, da, bh + b0, idn, 1u);
              umma::mma_f16(tm, da, bl + b0, idn, 1u);
            } else {
              umma::mma_f16_c<1>(tm, da, bh + b0, idn, 1u);
              umma::mma_f16_c<3>(tm, da, bl + b0, idn, 1u);
            }
          }
        }
        __syncwarp();
        if (++dy == 3) dy = 0;
      }
    } else if (nops == 70 || nops == 71 || nops == 72) {
      // positions-as-M plane conv pattern (conv_pm): A = the shifted x-plane halo (M = 128
      // positions, K-major interleave, LBO = chain * 16), B = the filter [kg 2][2 Co rows][8]
      // (LBO = 2 Co x 16 B); per tap and 128-position tile: x0 x [W0; W1] (N = 2 Co) and x1 x W0
      // (N = Co).  N = the 2 Co of the call; 71: both with N = 2 Co (4 products); 72: x0 only.
      const uint32_t w0 = umma::smem_u32(sm), xh = umma::smem_u32(sm + 64 * 1024), xl = umma::smem_u32(sm + 96 * 1024);
      const uint32_t kgx = (uint32_t)chain * 16u;
      const uint64_t dw = umma::desc_kmajor_interleave(w0, (uint32_t)N * 16u, 128);
      const uint64_t ah = umma::desc_kmajor_interleave(xh, kgx, 128);
      const uint64_t al = umma::desc_kmajor_interleave(xl, kgx, 128);
      const uint32_t id_full = umma::idesc(0, 128, N);
      const uint32_t id_half = umma::idesc(0, 128, nops == 71 ? N : N / 2);
      const uint64_t wtap = (uint64_t)(N * 32 / 16);   // one tap's filter (2 kg x N rows x 16 B) in 16 B units
      int dy = 0;
      const int per = nops == 72 ? 6 : 12;
      for (int r = 0; r < reps; r += per) {
        const uint64_t row = (uint64_t)(dy * 34 + 1);
        if (umma::elect_one()) {
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const uint64_t db = dw + dx * wtap;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const uint64_t a0 = row + dx + (uint64_t)(t * 128);
              umma::mma_f16(tm + (uint32_t)(t * 256), ah + a0, db, id_full, 1u);
              if (nops != 72) umma::mma_f16(tm + (uint32_t)(t * 256), al + a0, db, id_half, 1u);
            }
          }
        }
        __syncwarp();
        if (++dy == 3) dy = 0;
      }
    } else if (nops >= 60 && nops <= 64) {
      // wgrad_small pattern (conv_wgrad_small.cu): positions are K; A = g groups, B = x groups,
      // both MN-major no-swizzle ([group][position][8], group stride S = chain * 16 B, LBO = 128 B
      // between 8-position core matrices); per K-step (16 positions) 9 taps with B shifted by
      // dy * 34 + dx - 1 positions, each into its own TMEM column block of N.
      // 60: M = 64 (layout 4) / 128 (else); 61: all taps into one column block; 62: K-major
      // descriptors instead (same bytes, wrong math; rate only); 63: tap shifts 0
      const uint32_t S = (uint32_t)chain * 16u;
      const uint32_t ga = umma::smem_u32(sm), gx = umma::smem_u32(sm + 64 * 1024);
      const bool mn = nops != 62;
      const uint64_t dA = mn ? umma::desc_kmajor_interleave(ga, 128, S) : umma::desc_kmajor_interleave(ga, S, 128);
      const uint64_t dB = mn ? umma::desc_kmajor_interleave(gx, 128, S) : umma::desc_kmajor_interleave(gx, S, 128);
      const uint32_t idm = umma::idesc(0, layout == 4 ? 64 : 128, N, mn ? 1 : 0, mn ? 1 : 0);
      int k = 0;
      for (int r = 0; r < reps; r += 9) {
        if (umma::elect_one()) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int sh = nops == 63 ? 0 : (tap / 3) * 34 + (tap % 3) - 1 + 1;
            umma::mma_f16(tm + (uint32_t)((nops == 61 ? 0 : tap) * N), dA + (uint64_t)(16 * k),
                          dB + (uint64_t)(sh + 16 * k), idm, 1u);
          }
        }
        __syncwarp();
        if (++k == 8) k = 0;
      }
    } else if (nops == 93) {
      // 94 without the k-step advance (B offsets fixed per tap)
      for (int r = 0; r < reps; r += nacc) {
        if (umma::elect_one()) {
          for (int t = 0; t < nacc; ++t)
            umma::mma_tf32(tm + (uint32_t)(t * N), da, db + (uint64_t)(t * chain * 8), id, r > 0);
        }
        __syncwarp();
      }
    } else if (nops == 92) {
      // 95 with the whole loop inside one elected lane (as wgrad issues)
      if (umma::elect_one()) {
        int k = 0;
        for (int r = 0; r < reps; r += nacc) {
          const uint64_t kadv = (uint64_t)(k * 64);
          for (int t = 0; t < nacc; ++t)
            umma::mma_tf32(tm + (uint32_t)(t * N), da + kadv, db + kadv + (uint64_t)(t * chain * 8), id, r > 0);
          if (++k == 3) k = 0;
        }
      }
      __syncwarp();
    } else if (nops == 90) {
      // 92 with the A collector: fill on the first tap of a k-step, use, lastuse on the last
      if (umma::elect_one()) {
        int k = 0;
        for (int r = 0; r < reps; r += nacc) {
          const uint64_t kadv = (uint64_t)(k * 64);
          const uint64_t a_k = da + kadv;
          umma::mma_tf32_c<1>(tm, a_k, db + kadv, id, r > 0);
          for (int t = 1; t + 1 < nacc; ++t)
            umma::mma_tf32_c<2>(tm + (uint32_t)(t * N), a_k, db + kadv + (uint64_t)(t * chain * 8), id, r > 0);
          umma::mma_tf32_c<3>(tm + (uint32_t)((nacc - 1) * N), a_k, db + kadv + (uint64_t)((nacc - 1) * chain * 8),
                              id, r > 0);
          if (++k == 3) k = 0;
        }
      }
      __syncwarp();
    } else if (nops == 91) {
      // 95 with the k-step advance applied to A only
      int k = 0;
      for (int r = 0; r < reps; r += nacc) {
        const uint64_t kadv = (uint64_t)(k * 64);
        if (umma::elect_one()) {
          for (int t = 0; t < nacc; ++t)
            umma::mma_tf32(tm + (uint32_t)(t * N), da + kadv, db + (uint64_t)(t * chain * 8), id, r > 0);
        }
        __syncwarp();
        if (++k == 3) k = 0;
      }
    } else if (nops == 95 || nops == 94) {
      // wgrad pattern: per k-step (A advances 8 rows = 64 units; 94: A fixed) nacc taps,
      // B = k-step + tap shift of t * chain rows, accumulator t
      int k = 0;
      for (int r = 0; r < reps; r += nacc) {
        const uint64_t kadv = (uint64_t)(k * 64);
        if (umma::elect_one()) {
          for (int t = 0; t < nacc; ++t)
            umma::mma_tf32(tm + (uint32_t)(t * N), nops == 95 ? da + kadv : da, db + kadv + (uint64_t)(t * chain * 8),
                           id, r > 0);
        }
        __syncwarp();
        if (++k == 3) k = 0;
      }
    } else if (nops == 96) {
      // A same, B rotating over start offsets 0, chain, 2 chain, 3 chain (16-byte units)
      for (int r = 0; r < reps; r += 4) {
        if (umma::elect_one()) {
          umma::mma_tf32(tm, da, db, id, r > 0);
          umma::mma_tf32(tm + N, da, db + (uint64_t)chain, id, r > 0);
          umma::mma_tf32(tm + 2 * N, da, db + (uint64_t)(2 * chain), id, r > 0);
          umma::mma_tf32(tm, da, db + (uint64_t)(3 * chain), id, 1);
        }
        __syncwarp();
      }
    } else if (nops == 97) {
      // same pattern without the collector
      for (int r = 0; r < reps; r += 4) {
        if (umma::elect_one()) {
          umma::mma_tf32(tm, da, db, id, r > 0);
          umma::mma_tf32(tm + N, da, db + 256, id, r > 0);
          umma::mma_tf32(tm, da, db + 512, id, 1);
          umma::mma_tf32(tm + N, da, db + 768, id, 1);
        }
        __syncwarp();
      }
    } else if (nops == 99) {
      // unrolled: 4 accumulators, compile-time offsets
      for (int r = 0; r < reps; r += 4) {
        if (umma::elect_one()) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t dq = tm + (uint32_t)((q % nacc) * N);
            if (fmt == 2)
              umma::mma_tf32(dq, da + q * 256, db, id, r > 0);
            else
              umma::mma_f16(dq, da + q * 256, db, id, r > 0);
          }
        }
        __syncwarp();
      }
    } else {
      int g = 0, gi = 0, op = 0;
      for (int r = 0; r < reps; ++r) {
        const uint32_t d = tm + (uint32_t)(g * N);
        const uint64_t aoff = (uint64_t)(op * 256);
        if (umma::elect_one()) {
          if (fmt == 2)
            umma::mma_tf32(d, da + aoff, db, id, r >= nacc * chain);
          else
            umma::mma_f16(d, da + aoff, db, id, r >= nacc * chain);
        }
        __syncwarp();
        if (++op == nops) op = 0;
        if (++gi == chain) {
          gi = 0;
          if (++g == nacc) g = 0;
        }
      }
    }
    if (umma::elect_one()) umma::mma_commit(&bar);
    __syncwarp();
    umma::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (float)(t1 - t0) / reps;
  }
  umma::tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    umma::tc_fence_after();
    umma::tmem_dealloc<512>(tmem);
  }
}
}  // namespace
}  // namespace rp::k

extern "C" int rp_debug_umma_bench(int fmt, int N, int layout, int a_mn, int b_mn, int reps, int nacc, int nops,
                                   int chain, int grid, float* out) {
  try {
    RP_CUDA(cudaFuncSetAttribute(rp::k::umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024));
    rp::k::umma_bench_kernel<<<grid, 128, 192 * 1024>>>(fmt, N, layout, a_mn, b_mn, reps, nacc, nops, chain, out);
    RP_LAUNCHED();
    RP_CUDA(cudaDeviceSynchronize());
    return 0;
  } catch (const rp::Error& e) {
    return e.code;
  }
}


// Where does row i of an M = 64 kind::f16 MMA's D land in TMEM?  A[i][k] = (k == 0) ? i + 1 : 0
// (64 x 16 fp16, K-major interleave), B[n][k] = (k == 0) ? 1 : 0 (16 x 16): D[i][n] = i + 1.
// Writes TMEM lanes 0..127, columns 0..15 to out[lane * 16 + col] (untouched lanes: -1).
namespace rp::k {
__global__ void umma_m64_layout_kernel(float* out) {
  __shared__ __align__(1024) uint16_t sa[64 * 16];
  __shared__ __align__(1024) uint16_t sb[16 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  // K-major interleave: core matrix = 8 rows x 8 halves (16 B); lbo = distance between the two
  // K-halves (k 0-7, 8-15), sbo = distance between 8-row groups
  for (int i = tid; i < 64 * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    const int idx = (k / 8) * (64 * 8) + (m / 8) * 64 + (m % 8) * 8 + (k % 8);
    sa[idx] = k == 0 ? __half_as_ushort(__float2half((float)(m + 1))) : 0;
  }
  for (int i = tid; i < 16 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    const int idx = (k / 8) * (16 * 8) + (n / 8) * 64 + (n % 8) * 8 + (k % 8);
    sb[idx] = k == 0 ? __half_as_ushort(__float2half(1.f)) : 0;
  }
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_barrier_init();
  }
  if (tid < 32) umma::tmem_alloc<32>(&slot);
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = slot;
  // pre-fill TMEM with -1 so untouched lanes show
  {
    const int w = tid / 32;
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(-1.f);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(tmem + ((uint32_t)(w * 32) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                 "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),
                 "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  if (tid < 32) {
    const uint64_t da = umma::desc_general(umma::smem_u32(sa), 64 * 8 * 2, 64 * 2, 0, 0);
    const uint64_t db = umma::desc_general(umma::smem_u32(sb), 16 * 8 * 2, 64 * 2, 0, 0);
    if (umma::elect_one()) {
      umma::mma_f16(tmem, da, db, umma::idesc(0, 64, 16), 0u);
      umma::mma_commit(&bar);
    }
    __syncwarp();
  }
  umma::mbar_wait(&bar, 0);
  umma::tc_fence_after();
  const int w = tid / 32;
  uint32_t r[16];
  umma::tmem_ld16(tmem + ((uint32_t)(w * 32) << 16), r);
  umma::tmem_wait_ld();
  for (int j = 0; j < 16; ++j) out[(w * 32 + (tid % 32)) * 16 + j] = __uint_as_float(r[j]);
  umma::tc_fence_before();
  __syncthreads();
  if (tid < 32) umma::tmem_dealloc<32>(tmem);
}
}  // namespace rp::k

extern "C" int rp_debug_umma_m64_layout(float* out) {
  try {
    rp::k::umma_m64_layout_kernel<<<1, 128>>>(out);
    RP_LAUNCHED();
    RP_CUDA(cudaDeviceSynchronize());
    return 0;
  } catch (const rp::Error& e) {
    return e.code;
  }
}

// ---------------------------------------------------------------------------
// TMA throughput by box shape: every CTA loads `iters` conv-halo boxes of an fp16 NHWC tensor
// [n][h][w][c] (image blockIdx.x + 148 i, rows from -1, columns from -1, zero fill) into a ring of
// `depth` 32 KB slots; cycles for the whole loop -> out[blockIdx.x].  cg = channels per box row
// (8: 16-byte rows in two 8-channel groups, the plane convs' box {8, W + 1, rows, 2}; 16 / 32 / 64:
// 32 / 64 / 128-byte rows {cg, W + 1, rows}).
namespace rp::k {
namespace {
__global__ void __launch_bounds__(32, 1) tma_bench_kernel(const __grid_constant__ CUtensorMap m, int n_img, int groups5,
                                                          int iters, int depth, uint32_t box_bytes, int five,
                                                          float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) umma::mbar_init(&bars[i], 1);
    umma::fence_barrier_init();
  }
  __syncwarp();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters + depth; ++i) {
      if (i >= depth) umma::mbar_wait(&bars[(i - depth) % depth], ((i - depth) / depth) & 1);
      if (i < iters) {
        const int s = i % depth;
        const int img = (blockIdx.x + 148 * i) % n_img;
        umma::mbar_arrive_expect_tx(&bars[s], box_bytes);
        if (five)
          umma::tma_load_5d(&m, &bars[s], sm + s * 32768, 0, -1, -1, 0, img);
        else
          umma::tma_load_4d(&m, &bars[s], sm + s * 32768, 0, -1, -1, img);
      }
    }
    out[blockIdx.x] = (float)(clock64() - t0);
  }
  (void)groups5;
}
}  // namespace
}  // namespace rp::k

extern "C" int rp_debug_tma_bench(const void* data, int n, int h, int w, int c, int cg, int rows, int iters, int depth,
                                  float* out) {
  try {
    typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    RP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    Enc enc = reinterpret_cast<Enc>(p);
    CUtensorMap m;
    uint32_t box_bytes;
    const int Wp = w + 1;
    int five;
    if (cg == 8) {   // {8, Wp, rows, c / 8, 1}: 16-byte rows, all groups in one box
      const cuuint64_t dims[5] = {8, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)(c / 8), (cuuint64_t)n};
      const cuuint64_t strides[4] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, 16, (cuuint64_t)h * w * c * 2};
      const cuuint32_t box[5] = {8, (cuuint32_t)Wp, (cuuint32_t)rows, 2, 1};   // one 16-channel chunk
      const cuuint32_t es[5] = {1, 1, 1, 1, 1};
      if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void*>(data), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 99;
      box_bytes = (uint32_t)(16 * Wp * rows * 2);
      five = 1;
    } else {         // {cg, Wp, rows, 1}: cg * 2-byte rows (only the first cg channels)
      const cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
      const cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
      const cuuint32_t box[4] = {(cuuint32_t)cg, (cuuint32_t)Wp, (cuuint32_t)rows, 1};
      const cuuint32_t es[4] = {1, 1, 1, 1};
      if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(data), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 98;
      box_bytes = (uint32_t)(2 * cg * Wp * rows);
      five = 0;
    }
    if (box_bytes > 32768) return 97;
    RP_CUDA(cudaFuncSetAttribute(rp::k::tma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
    rp::k::tma_bench_kernel<<<148, 32, depth * 32768>>>(m, n, c / 8, iters, depth, box_bytes, five, out);
    RP_CUDA(cudaGetLastError());
    RP_CUDA(cudaDeviceSynchronize());
    return 0;
  } catch (const rp::Error& e) {
    return e.code;
  }
}
