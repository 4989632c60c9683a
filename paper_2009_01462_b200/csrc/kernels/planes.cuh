// Plane encodings of fp32 tensors for the tensor cores.
//
//  * plane PAIR (fp32 math): v * s = p0 + p1 with p0 = fp16(v s), p1 = fp16(v s - p0), round to
//    nearest.  Each fp16 carries an 11-bit significand, so the pair holds 22 bits: the residual
//    |v s - p0 - p1| <= 2^-24 |v s| while p1 is a normal fp16 -- fp32's own rounding.  The four
//    products W0x0 + W1x0 + W0x1 + W1x1 of two pairs therefore reproduce an fp32 product to
//    ~2^-23, for the price of two bf16-rate MMAs.  fp16's exponent range is narrow, so every
//    pair carries a power-of-two scale s (exact) that keeps p1 a normal number (the tensor core
//    loses most of a subnormal low plane: measured, an unscaled |x| <= 1 pair ran at ~2^-18
//    relative, a scaled one at ~2^-24): weights s = kWeightPlaneScale (|W| < 2^7), forward
//    activations s = kActPlaneScale (|x| < 2^8; the "NULL scale" of every plane API), the
//    cotangent side (g, dpre, whose magnitude is set by beta / # and the loss) a per-stage s
//    computed on device from max |g| so that the largest element sits at 2^kCotangentPlaneExp
//    (headroom 2^(16 - kCotangentPlaneExp) for growth through the stage's blocks).  Consumers
//    divide the accumulator by the operands' scales.
//  * SINGLE plane (bf16 math, config C5): p0 = bf16(v), unscaled.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

namespace rp::k {

constexpr float kWeightPlaneScale = 256.f;       // weights enter the plane MMAs as W * 2^8
constexpr float kWeightPlaneScaleInv = 1.f / 256.f;
constexpr int kCotangentPlaneExp = 8;            // max |g s| in [2^7, 2^8)
constexpr float kActPlaneScale = 128.f;          // forward activations x, a enter as v 2^7

__device__ __forceinline__ uint32_t half2_bits(__half2 h) { return *reinterpret_cast<const uint32_t*>(&h); }
__device__ __forceinline__ uint32_t bf162_bits(__nv_bfloat162 h) { return *reinterpret_cast<const uint32_t*>(&h); }

// fp16 pair of 4 values times s (packed 4 x fp16 per plane)
__device__ __forceinline__ void pack_pair4(const float (&v)[4], float s, uint2& p0, uint2& p1) {
  const float a = v[0] * s, b = v[1] * s, c = v[2] * s, d = v[3] * s;
  const __half2 h0 = __floats2half2_rn(a, b), h1 = __floats2half2_rn(c, d);
  const __half2 l0 = __floats2half2_rn(a - __low2float(h0), b - __high2float(h0));
  const __half2 l1 = __floats2half2_rn(c - __low2float(h1), d - __high2float(h1));
  p0 = make_uint2(half2_bits(h0), half2_bits(h1));
  p1 = make_uint2(half2_bits(l0), half2_bits(l1));
}

// bf16 single plane of 4 values
__device__ __forceinline__ uint2 pack_single4(const float (&v)[4]) {
  return make_uint2(bf162_bits(__floats2bfloat162_rn(v[0], v[1])), bf162_bits(__floats2bfloat162_rn(v[2], v[3])));
}

__device__ __forceinline__ float half_bits_to_float(uint16_t b) { return __half2float(__ushort_as_half(b)); }
__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) {
  return __bfloat162float(__ushort_as_bfloat16(b));
}

// power-of-two scale that puts max|v| in [2^(E-1), 2^E), E = kCotangentPlaneExp (1 for 0 / non-finite)
__device__ __forceinline__ float cotangent_plane_scale(float vmax) {
  if (!(vmax > 0.f) || !isfinite(vmax)) return 1.f;
  int e = 0;
  frexpf(vmax, &e);                                   // vmax = m 2^e, m in [0.5, 1)
  int k = kCotangentPlaneExp - e;
  k = k < -126 ? -126 : (k > 126 ? 126 : k);
  return ldexpf(1.f, k);
}

}  // namespace rp::k
