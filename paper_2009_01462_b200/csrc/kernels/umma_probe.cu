// Diagnostic: one tcgen05.mma (M=128, N=16, K=8, tf32) on known operands in a chosen
// shared-memory layout, to pin down UMMA descriptor semantics on the device.  Exposed
// as rp_debug_umma_probe (tests only; never on the training path).
#include "../common.cuh"
#include "umma.cuh"

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
