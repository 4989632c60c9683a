// C ABI, op layer (include/respar_b200.h "rp_op_*"): stream-ordered kernels on
// caller-owned device buffers.  The C++ host classes (host/trainer.cpp) reach the GPU
// only through these entry points.
#include <cstdlib>
#include <string>
#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>

#include "capi_guard.hpp"
#include "common.cuh"
#include "kernels/kernels.cuh"
#include "profile.hpp"

#ifndef RP_CONV_PM_DEFAULT
#define RP_CONV_PM_DEFAULT 1   // Co = 64: conv_pm.cu (measured +4 % on C3 under the power cap) unless RP_CONV_PM=0
#endif

namespace rp {

namespace {

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int64_t align256(int64_t v) { return (v + 255) / 256 * 256; }

void need(const void* p, const char* what) {
  if (!p) fail(RP_ERR_RANGE, std::string(what) + ": null pointer");
}

struct Carve {
  char* base;
  int64_t cap;
  int64_t off = 0;
  template <class T>
  T* take(int64_t count) {
    const int64_t bytes = align256(count * (int64_t)sizeof(T));
    if (off + bytes > cap) fail(RP_ERR_RANGE, "workspace too small");
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

k::ConvShape shape(const rp_geometry& g, int nrows, int ci, int co) { return {nrows, g.height, g.width, ci, co}; }

double conv_flops(const k::ConvShape& s) { return 2.0 * 9.0 * s.ci * s.co * (double)s.pixels(); }
// algorithmic HBM bytes of one conv launch: read the input, write the output, plus
// the epilogue's aux tensor when it has one (weights are negligible)
double conv_bytes(const k::ConvShape& s, bool aux) {
  return 4.0 * (double)s.pixels() * (s.ci + s.co + (aux ? s.co : 0));
}

// fp32-accurate conv operand split for the fprop / dgrad kernel: 3xBF16 (default: 3 K=16
// MMAs per 16 channels instead of 4 K=8 ones; measured 2-5 % faster, ~4e-6 relative) or
// 3xTF32 (RP_FP32_SPLIT=tf32x3, ~1e-6 relative), read once.
int fp32_split() {
  static const int m = [] {
    const char* e = std::getenv("RP_FP32_SPLIT");
    return (e && std::string(e) == "tf32x3") ? (int)k::TC_MODE_X3TF32 : (int)k::TC_MODE_X3BF16;
  }();
  return m;
}

void check_math(int math) {
  if (math < RP_MATH_FP32 || math > RP_MATH_SIMT) fail(RP_ERR_CONFIG, "unknown math mode");
}

}  // namespace

// bytes reserved at the front of an op workspace for per-call weight relayouts
int64_t weight_ws_bytes(const rp_geometry& g) {
  const int64_t C = g.channels, Ch = g.hidden;
  return align256(std::max({k::conv3x3_tc_ws_bytes({1, 1, 1, (int)C, (int)Ch}),
                            k::conv3x3_tc_ws_bytes({1, 1, 1, (int)Ch, (int)C}), (int64_t)(9 * C * Ch * 4)}));
}

int64_t wgrad_ws_bytes(const k::ConvShape& s) {
  return std::max({k::conv3x3_wgrad_ws_bytes(s), k::conv3x3_wgrad_tc_ws_bytes(s, true),
                   k::conv3x3_wgrad_tc_ws_bytes(s, false), k::conv3x3_wgrad_bf16_ws_bytes(s),
                   k::conv3x3_wgrad_planes_ws_bytes(s), k::conv3x3_wgrad_bf16p_ws_bytes(s),
                   k::conv3x3_wgrad_small_ws_bytes(s)});
}

// The plane-pair block path (fp32 math): every conv of the block on the tcgen05 kernel, whose
// epilogue also writes the fp16 plane pair (v s = p0 + p1, planes.cuh) of its output, so both weight
// gradients run on the TMA-fed plane wgrad (conv_wgrad_planes.cu). RP_WGRAD_PLANES=0 turns
// it off (the fp32-operand 3xTF32 wgrad then runs).
// Plane-input convs: the positions-as-M kernel (conv_pm.cu, 3 products per MAC) or conv_tc.cu's
// channels-as-M kernel (4 products; Co % 64 == 0).  g_plane_conv: -1 auto (conv_pm where it is
// the only kernel or RP_CONV_PM_DEFAULT), 0 conv_tc where supported, 1 conv_pm where supported;
// initialised from RP_CONV_PM, set by rp_op_set_plane_conv_kernel.
std::atomic<int> g_plane_conv{[] {
  const char* e = std::getenv("RP_CONV_PM");
  return e ? (std::atoi(e) != 0 ? 1 : 0) : -1;
}()};

bool plane_conv_pm(const k::ConvShape& s) {
  if (!k::conv3x3_pm_supported(s)) return false;
  if (!k::conv3x3_tc_supported(s)) return true;
  const int f = g_plane_conv.load(std::memory_order_relaxed);
  return f >= 0 ? f != 0 : RP_CONV_PM_DEFAULT != 0;
}

bool plane_wgrad_supported(const k::ConvShape& s) {
  return k::conv3x3_wgrad_planes_supported(s) || k::conv3x3_wgrad_small_supported(s);
}

bool plane_conv_supported(const k::ConvShape& s) { return k::conv3x3_pm_supported(s) || k::conv3x3_tc_supported(s); }

bool planes_path(const rp_geometry& g, int nrows, int math) {
  static const bool enabled = [] {
    const char* e = std::getenv("RP_WGRAD_PLANES");
    return !(e && std::string(e) == "0");
  }();
  if (!enabled || math != RP_MATH_FP32 || nrows <= 0) return false;
  const k::ConvShape s1{nrows, g.height, g.width, g.channels, g.hidden};
  const k::ConvShape s2{nrows, g.height, g.width, g.hidden, g.channels};
  return plane_conv_supported(s1) && plane_conv_supported(s2) && plane_wgrad_supported(s1) &&
         plane_wgrad_supported(s2);
}

// The bf16 tape path (bf16 math): the bf16 conv epilogues also write a bf16 copy of their
// output (the block inputs x, the activations a, dpre and the cotangent g), so both weight
// gradients run on the TMA-fed single-plane wgrad (conv_wgrad_planes.cu, bf16p) instead of
// staging fp32 operands through converter warps.  RP_BF16_TAPE=0 turns it off.
bool bf16_tape_path(const rp_geometry& g, int nrows, int math) {
  static const bool enabled = [] {
    const char* e = std::getenv("RP_BF16_TAPE");
    return !(e && std::string(e) == "0");
  }();
  if (!enabled || math != RP_MATH_BF16 || nrows <= 0) return false;
  const k::ConvShape s1{nrows, g.height, g.width, g.channels, g.hidden};
  const k::ConvShape s2{nrows, g.height, g.width, g.hidden, g.channels};
  return k::conv3x3_bf16_supported(s1) && k::conv3x3_bf16_supported(s2) && k::conv3x3_wgrad_bf16p_supported(s1) &&
         k::conv3x3_wgrad_bf16p_supported(s2);
}

// Weight gradient (+ bias sums): tcgen05 when the math mode and shape allow, SIMT otherwise.
void wgrad(const k::ConvShape& s, const float* in, const float* gout, float scale, float* gw, float* gb, int math,
           void* ws, cudaStream_t st) {
  prof::Scope ps(RP_PROF_CONV_WGRAD, st, conv_flops(s), conv_bytes(s, false));
  const bool three = math != RP_MATH_TF32;
  if (math == RP_MATH_BF16 && k::conv3x3_wgrad_bf16_supported(s)) {
    k::conv3x3_wgrad_bf16(s, in, gout, scale, gw, gb, ws, st);
    return;
  }
  if (math != RP_MATH_SIMT && k::conv3x3_wgrad_tc_supported(s, three)) {
    k::conv3x3_wgrad_tc(s, in, gout, scale, gw, gb, three, ws, st);
    return;
  }
  k::conv3x3_wgrad_simt(s, in, gout, scale, gw, gb, ws, st);
}

int64_t op_workspace_bytes(const rp_geometry& g, int nrows) {
  const int64_t C = g.channels, Ch = g.hidden;
  int64_t wg = wgrad_ws_bytes(shape(g, nrows, (int)Ch, (int)C));
  wg = std::max(wg, wgrad_ws_bytes(shape(g, nrows, (int)C, (int)Ch)));
  wg = std::max(wg, wgrad_ws_bytes(shape(g, nrows, g.in_channels, (int)C)));
  wg = std::max(wg, k::stem_wgrad_ws_bytes(shape(g, nrows, g.in_channels, (int)C)));
  const int64_t head = k::head_ws_bytes(nrows, g.channels, g.classes);
  return std::max(weight_ws_bytes(g) + align256(wg), head) + 256;
}

// One 3x3 conv with a fused epilogue: the tcgen05 kernel (3xTF32 or TF32) when the
// math mode asks for tensor cores and the shape is supported, the SIMT kernel otherwise.
// dgrad: `w` is the forward conv's HWIO weight; the conv runs on the cotangent.
void conv(const k::ConvShape& s, const float* in, const float* w, bool dgrad, const float* bias, const float* aux,
          float h, int epi, float* out, int math, void* wws, int prof_cls, bool aux_read, cudaStream_t st,
          void* out_planes = nullptr, const void* in_planes = nullptr, const void* wprep = nullptr,
          const float* in_scale = nullptr, const float* out_scale = nullptr) {
  prof::Scope ps(prof_cls, st, conv_flops(s),
                 conv_bytes(s, aux_read) + (out_planes ? 4.0 * s.pixels() * s.co : 0.0) - (out ? 0.0 : 4.0 * s.pixels() * s.co));
  if (out_planes || in_planes) {   // only the fp32 tcgen05 kernels read / write plane pairs (planes_path())
    if (math != RP_MATH_FP32) fail(RP_ERR_INTERNAL, "conv: plane i/o needs fp32 math");
    if (in_planes && plane_conv_pm(s)) {
      k::conv3x3_fwd_pm(s, w, dgrad, bias, aux, h, epi, out, wws, st, out_planes, in_planes, wprep, in_scale,
                        out_scale);
      return;
    }
    if (!k::conv3x3_tc_supported(s)) fail(RP_ERR_INTERNAL, "conv: plane i/o needs fp32 tcgen05");
    k::conv3x3_fwd_tc(s, in, w, dgrad, bias, aux, h, epi, out, fp32_split(), wws, st, out_planes, in_planes,
                      in_planes ? wprep : nullptr, in_scale, out_scale);
    return;
  }
  // RP_MATH_BF16: bf16 operands where the bf16 kernel tiles the shape (Co % 128, Ci % 32),
  // the fp32-accurate 3xTF32 kernel elsewhere (never less precise than asked for)
  if (math == RP_MATH_BF16 && k::conv3x3_bf16_supported(s)) {
    k::conv3x3_fwd_bf16(s, in, w, dgrad, bias, aux, h, epi, out, wws, st);
    return;
  }
  if (math != RP_MATH_SIMT && k::conv3x3_tc_supported(s)) {
    k::conv3x3_fwd_tc(s, in, w, dgrad, bias, aux, h, epi, out, math == RP_MATH_TF32 ? k::TC_MODE_TF32 : fp32_split(),
                      wws, st);
    return;
  }
  const float* wk = w;
  if (dgrad) {
    k::conv3x3_dgrad_weights(w, s.co, s.ci, static_cast<float*>(wws), st);
    wk = static_cast<const float*>(wws);
  }
  k::conv3x3_fwd_simt(s, in, wk, bias, aux, h, epi, out, st);
}

void block_fwd(const rp_geometry& g, int nrows, const float* x, const float* pb, float* a, float* x_next, int math,
               void* ws, int64_t ws_bytes, cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const bool tanh_act = g.activation == RP_ACT_TANH;
  if (ws_bytes < weight_ws_bytes(g)) fail(RP_ERR_RANGE, "block_fwd: workspace too small");
  const k::ConvShape s1 = shape(g, nrows, g.channels, g.hidden), s2 = shape(g, nrows, g.hidden, g.channels);
  // conv1 + b1 + act  ->  a      (network.cpp:85-86)
  conv(s1, x, pb + L.w1, false, pb + L.b1, nullptr, 1.f, tanh_act ? k::EPI_BIAS_TANH : k::EPI_BIAS, a, math, ws,
       RP_PROF_CONV_FPROP, false, st);
  // conv2 + b2, *h, + x  ->  x'   (network.cpp:87)
  conv(s2, a, pb + L.w2, false, pb + L.b2, x, (float)g.step_h, k::EPI_RESID, x_next, math, ws, RP_PROF_CONV_FPROP,
       true, st);
}

void block_bwd(const rp_geometry& g, int nrows, const float* x, const float* a, const float* pb, float* gio,
               float* dpre, float* gb, int math, void* ws, int64_t ws_bytes, cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const int C = g.channels, Ch = g.hidden;
  const bool tanh_act = g.activation == RP_ACT_TANH;
  const float h = (float)g.step_h;
  Carve cv{static_cast<char*>(ws), ws_bytes};
  void* wws = cv.take<char>(weight_ws_bytes(g));
  const int64_t wg_bytes = std::max(wgrad_ws_bytes(shape(g, nrows, Ch, C)), wgrad_ws_bytes(shape(g, nrows, C, Ch)));
  void* wgws = cv.take<char>(wg_bytes);
  // dpre = h (g * W2^T) (1 - a^2)                              (network.cpp:100-101)
  conv(shape(g, nrows, C, Ch), gio, pb + L.w2, true, nullptr, a, h, tanh_act ? k::EPI_TANH_BWD : k::EPI_SCALE, dpre,
       math, wws, RP_PROF_CONV_DGRAD, tanh_act, st);
  // gW2 = h a^T g, gb2 = h sum g                               (network.cpp:98-99)
  wgrad(shape(g, nrows, Ch, C), a, gio, h, gb + L.w2, gb + L.b2, math, wgws, st);
  // gW1 = x^T dpre, gb1 = sum dpre                             (network.cpp:102-103)
  wgrad(shape(g, nrows, C, Ch), x, dpre, 1.f, gb + L.w1, gb + L.b1, math, wgws, st);
  // g <- g + dpre * W1^T   (in place)                          (network.cpp:104)
  conv(shape(g, nrows, Ch, C), dpre, pb + L.w1, true, nullptr, gio, 1.f, k::EPI_ADD, gio, math, wws,
       RP_PROF_CONV_DGRAD, true, st);
}

// Plane-pair variants: a_p / x_next_p / x_p / g_p / dpre_p are fp16 [2][elements] pairs
// (planes.cuh); the cotangent-side pairs g_p / dpre_p carry the stage's scale *gscale.
// filters (nullable): the block's two prepared plane-mode filters (prep_planes_filters), else
// each conv prepares its own.
int64_t planes_filter_bytes(const rp_geometry& g) { return 9LL * g.channels * g.hidden * 2 * 2; }

void prep_planes_filters(const rp_geometry& g, const float* pb, int nblocks, bool dgrad, void* out, cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const int C = g.channels, Ch = g.hidden;
  // forward: conv1 (W1: C -> Ch), conv2 (W2: Ch -> C); input gradient in block_bwd order:
  // dgrad2 (W2 flipped), dgrad1 (W1 flipped)
  const int64_t off[2] = {dgrad ? L.w2 : L.w1, dgrad ? L.w1 : L.w2};
  const int ci_src[2] = {dgrad ? Ch : C, dgrad ? C : Ch};
  const int co_src[2] = {dgrad ? C : Ch, dgrad ? Ch : C};
  k::prep_filters_planes(pb, L.block_stride, nblocks, off, ci_src, co_src, dgrad, out, st);
}

void block_fwd_planes(const rp_geometry& g, int nrows, const float* x, const void* x_p, const float* pb, float* a,
                      float* x_next, void* a_p, void* x_next_p, const void* filters, void* ws, int64_t ws_bytes,
                      cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const bool tanh_act = g.activation == RP_ACT_TANH;
  if (ws_bytes < weight_ws_bytes(g)) fail(RP_ERR_RANGE, "block_fwd: workspace too small");
  const k::ConvShape s1 = shape(g, nrows, g.channels, g.hidden), s2 = shape(g, nrows, g.hidden, g.channels);
  const char* f = static_cast<const char*>(filters);
  const int64_t fb = planes_filter_bytes(g);
  conv(s1, x, pb + L.w1, false, pb + L.b1, nullptr, 1.f, tanh_act ? k::EPI_BIAS_TANH : k::EPI_BIAS, a, RP_MATH_FP32,
       ws, RP_PROF_CONV_FPROP, false, st, a_p, x_p, f);
  conv(s2, a, pb + L.w2, false, pb + L.b2, x, (float)g.step_h, k::EPI_RESID, x_next, RP_MATH_FP32, ws,
       RP_PROF_CONV_FPROP, true, st, x_next_p, a_p, f ? f + fb : nullptr);
}

void wgrad_planes(const k::ConvShape& s, const void* xp, const void* gp, float scale, float* gw, float* gb, void* ws,
                  cudaStream_t st, const float* gscale) {
  prof::Scope ps(RP_PROF_CONV_WGRAD, st, conv_flops(s), 4.0 * (double)s.pixels() * (s.ci + s.co));
  const auto* x0 = static_cast<const uint16_t*>(xp);   // fp16 bits
  const auto* g0 = static_cast<const uint16_t*>(gp);
  if (!k::conv3x3_wgrad_planes_supported(s)) {   // the 16-channel form (plane_wgrad_supported)
    k::conv3x3_wgrad_small(s, x0, x0 + s.pixels() * s.ci, g0, g0 + s.pixels() * s.co, scale, gw, gb, ws, st, gscale);
    return;
  }
  k::conv3x3_wgrad_planes(s, x0, x0 + s.pixels() * s.ci, g0, g0 + s.pixels() * s.co, scale, gw, gb, ws, st, gscale);
}

void block_bwd_planes(const rp_geometry& g, int nrows, const void* x_p, const float* a, const void* a_p,
                      const float* pb, float* gio, void* g_p, const float* gscale, float* dpre, void* dpre_p,
                      float* gb, const void* filters, void* ws, int64_t ws_bytes, cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const int C = g.channels, Ch = g.hidden;
  const bool tanh_act = g.activation == RP_ACT_TANH;
  const float h = (float)g.step_h;
  Carve cv{static_cast<char*>(ws), ws_bytes};
  void* wws = cv.take<char>(weight_ws_bytes(g));
  const int64_t wg_bytes = std::max(wgrad_ws_bytes(shape(g, nrows, Ch, C)), wgrad_ws_bytes(shape(g, nrows, C, Ch)));
  void* wgws = cv.take<char>(wg_bytes);
  // dpre = h (g * W2^T) (1 - a^2) as planes only: its consumers (wgrad1, dgrad1) read the
  // planes, so the fp32 dpre is not written                     (network.cpp:100-101)
  const char* f = static_cast<const char*>(filters);
  const int64_t fb = planes_filter_bytes(g);
  (void)dpre;
  // (the dpre planes keep the cotangent scale: in and out scale are both *gscale)
  conv(shape(g, nrows, C, Ch), gio, pb + L.w2, true, nullptr, a, h, tanh_act ? k::EPI_TANH_BWD : k::EPI_SCALE, nullptr,
       RP_MATH_FP32, wws, RP_PROF_CONV_DGRAD, tanh_act, st, dpre_p, g_p, f, gscale, gscale);
  if (C == Ch && k::conv3x3_wgrad_planes_supported(shape(g, nrows, C, Ch)) && !std::getenv("RP_WGRAD_UNPAIRED")) {
    // gW1 = x^T dpre, gb1 = sum dpre and gW2 = h a^T g, gb2 = h sum g in ONE launch (same
    // shape): half the launches' prologues, epilogues and reduces   (network.cpp:98-103)
    const k::ConvShape sw = shape(g, nrows, C, Ch);
    prof::Scope ps(RP_PROF_CONV_WGRAD, st, 2 * conv_flops(sw), 2 * 4.0 * (double)sw.pixels() * (sw.ci + sw.co));
    const auto* x0 = static_cast<const uint16_t*>(x_p);
    const auto* d0 = static_cast<const uint16_t*>(dpre_p);
    const auto* a0 = static_cast<const uint16_t*>(a_p);
    const auto* g0 = static_cast<const uint16_t*>(g_p);
    const int64_t ne = sw.pixels() * C;
    const void* xa[2] = {x0, x0 + ne};
    const void* ga[2] = {d0, d0 + ne};
    const void* xb[2] = {a0, a0 + ne};
    const void* gb2[2] = {g0, g0 + ne};
    k::conv3x3_wgrad_planes_pair(sw, xa, ga, 1.f, gb + L.w1, gb + L.b1, xb, gb2, h, gb + L.w2, gb + L.b2, wgws, st,
                                 gscale, gscale);
  } else {
    // gW1 = x^T dpre, gb1 = sum dpre first, while dgrad2's dpre planes are still in L2
    //                                                               (network.cpp:102-103)
    wgrad_planes(shape(g, nrows, C, Ch), x_p, dpre_p, 1.f, gb + L.w1, gb + L.b1, wgws, st, gscale);
    // gW2 = h a^T g, gb2 = h sum g (before dgrad1 overwrites the g planes) (network.cpp:98-99)
    wgrad_planes(shape(g, nrows, Ch, C), a_p, g_p, h, gb + L.w2, gb + L.b2, wgws, st, gscale);
  }
  // g <- g + dpre * W1^T in place, and the planes of the new g   (network.cpp:104)
  conv(shape(g, nrows, Ch, C), dpre, pb + L.w1, true, nullptr, gio, 1.f, k::EPI_ADD, gio, RP_MATH_FP32, wws,
       RP_PROF_CONV_DGRAD, true, st, g_p, dpre_p, f ? f + fb : nullptr, gscale, gscale);
}

// bf16 tape variants.  Every conv reads its input as a bf16 tensor (TMA straight into the
// MMA layout) -- the same values the fp32-input bf16 kernel's converters would produce (RNE)
// -- and the tape holds bf16 only: x16 (block input), a16 (activation), d16 = bf16(1 - a^2)
// (the tanh derivative), dpre16, g16.  The fp32 residual stream x (EPI_RESID's aux, the stage
// output) and the fp32 cotangent g (EPI_ADD's aux) stay fp32.
void block_fwd_bf16t(const rp_geometry& g, int nrows, const float* x, const void* x16, const float* pb, void* a16,
                     void* d16, float* x_next, void* x_next16, void* ws, int64_t ws_bytes, cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const bool tanh_act = g.activation == RP_ACT_TANH;
  if (ws_bytes < weight_ws_bytes(g)) fail(RP_ERR_RANGE, "block_fwd: workspace too small");
  const k::ConvShape s1 = shape(g, nrows, g.channels, g.hidden), s2 = shape(g, nrows, g.hidden, g.channels);
  {   // a = act(conv1(x) + b1): bf16 a and bf16 (1 - a^2)   (network.cpp:85-86)
    prof::Scope ps(RP_PROF_CONV_FPROP, st, conv_flops(s1), 2.0 * s1.pixels() * (s1.ci + s1.co * (tanh_act ? 2 : 1)));
    k::conv3x3_fwd_bf16_in16(s1, x16, pb + L.w1, false, pb + L.b1, nullptr, nullptr, 1.f,
                             tanh_act ? k::EPI_BIAS_TANH : k::EPI_BIAS, nullptr, a16, tanh_act ? d16 : nullptr, ws,
                             st);
  }
  {   // x' = x + h (conv2(a) + b2), fp32 and bf16                (network.cpp:87)
    prof::Scope ps(RP_PROF_CONV_FPROP, st, conv_flops(s2),
                   2.0 * s2.pixels() * s2.ci + 8.0 * s2.pixels() * s2.co + (x_next16 ? 2.0 * s2.pixels() * s2.co : 0.0));
    k::conv3x3_fwd_bf16_in16(s2, a16, pb + L.w2, false, pb + L.b2, x, nullptr, (float)g.step_h, k::EPI_RESID, x_next,
                             x_next16, nullptr, ws, st);
  }
}

void wgrad_bf16p(const k::ConvShape& s, const void* x16, const void* g16, float scale, float* gw, float* gb, void* ws,
                 cudaStream_t st) {
  prof::Scope ps(RP_PROF_CONV_WGRAD, st, conv_flops(s), 2.0 * (double)s.pixels() * (s.ci + s.co));
  k::conv3x3_wgrad_bf16p(s, x16, g16, scale, gw, gb, ws, st);
}

void block_bwd_bf16t(const rp_geometry& g, int nrows, const void* x16, const void* a16, const void* d16,
                     const float* pb, float* gio, void* g16, void* dpre16, float* gb, void* ws, int64_t ws_bytes,
                     cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const int C = g.channels, Ch = g.hidden;
  const bool tanh_act = g.activation == RP_ACT_TANH;
  const float h = (float)g.step_h;
  Carve cv{static_cast<char*>(ws), ws_bytes};
  void* wws = cv.take<char>(weight_ws_bytes(g));
  const int64_t wg_bytes = std::max(wgrad_ws_bytes(shape(g, nrows, Ch, C)), wgrad_ws_bytes(shape(g, nrows, C, Ch)));
  void* wgws = cv.take<char>(wg_bytes);
  const k::ConvShape sd2 = shape(g, nrows, C, Ch), sd1 = shape(g, nrows, Ch, C);
  {   // dpre = h (g * W2^T) (1 - a^2), bf16                      (network.cpp:100-101)
    prof::Scope ps(RP_PROF_CONV_DGRAD, st, conv_flops(sd2), 2.0 * sd2.pixels() * (sd2.ci + sd2.co * (tanh_act ? 2 : 1)));
    k::conv3x3_fwd_bf16_in16(sd2, g16, pb + L.w2, true, nullptr, nullptr, tanh_act ? d16 : nullptr, h,
                             tanh_act ? k::EPI_DTANH16 : k::EPI_SCALE, nullptr, dpre16, nullptr, wws, st);
  }
  const k::ConvShape sw = shape(g, nrows, C, Ch);
  if (C == Ch && k::conv3x3_wgrad_bf16p_pair_supported(sw) && !std::getenv("RP_WGRAD_UNPAIRED")) {
    // gW1 = x^T dpre, gb1 = sum dpre and gW2 = h a^T g, gb2 = h sum g in one launch
    //                                                                (network.cpp:98-103)
    prof::Scope ps(RP_PROF_CONV_WGRAD, st, 2 * conv_flops(sw), 2 * 2.0 * (double)sw.pixels() * (sw.ci + sw.co));
    k::conv3x3_wgrad_bf16p_pair(sw, x16, dpre16, 1.f, gb + L.w1, gb + L.b1, a16, g16, h, gb + L.w2, gb + L.b2, wgws,
                                st);
  } else {
    // gW1 = x^T dpre, gb1 = sum dpre first, while dpre16 is still in L2   (network.cpp:102-103)
    wgrad_bf16p(shape(g, nrows, C, Ch), x16, dpre16, 1.f, gb + L.w1, gb + L.b1, wgws, st);
    // gW2 = h a^T g, gb2 = h sum g (before dgrad1 rewrites g16)             (network.cpp:98-99)
    wgrad_bf16p(shape(g, nrows, Ch, C), a16, g16, h, gb + L.w2, gb + L.b2, wgws, st);
  }
  {   // g <- g + dpre * W1^T in place, and its bf16 copy           (network.cpp:104)
    prof::Scope ps(RP_PROF_CONV_DGRAD, st, conv_flops(sd1), 2.0 * sd1.pixels() * sd1.ci + 10.0 * sd1.pixels() * sd1.co);
    k::conv3x3_fwd_bf16_in16(sd1, dpre16, pb + L.w1, true, nullptr, gio, nullptr, 1.f, k::EPI_ADD, gio, g16, nullptr,
                             wws, st);
  }
}

void stem_fwd(const rp_geometry& g, int nrows, const float* xr, const float* ps, float* x0, cudaStream_t st,
              void* p0 = nullptr, void* p1 = nullptr) {
  const ParamLayout L = ParamLayout::of(g);
  const k::ConvShape sh = shape(g, nrows, g.in_channels, g.channels);
  prof::Scope scope(RP_PROF_STEM, st, conv_flops(sh), conv_bytes(sh, false));
  if (k::stem_supported(sh)) {
    k::stem_fwd(sh, xr, ps + L.s_w, ps + L.s_b, x0, st, p0, p1);
    return;
  }
  k::conv3x3_fwd_simt(sh, xr, ps + L.s_w, ps + L.s_b, nullptr, 1.f, k::EPI_BIAS, x0, st);
  if (p0) k::split_planes(x0, sh.pixels() * sh.co, p0, p1, st);
}

void stem_bwd(const rp_geometry& g, int nrows, const float* xr, const float* g0, float* gs, void* ws,
              int64_t ws_bytes, cudaStream_t st) {
  const ParamLayout L = ParamLayout::of(g);
  const k::ConvShape sh = shape(g, nrows, g.in_channels, g.channels);
  prof::Scope scope(RP_PROF_STEM, st, conv_flops(sh), conv_bytes(sh, false));
  if (k::stem_supported(sh)) {
    if (k::stem_wgrad_ws_bytes(sh) > ws_bytes) fail(RP_ERR_RANGE, "stem_bwd: workspace too small");
    k::stem_wgrad(sh, xr, g0, 1.f, gs + L.s_w, gs + L.s_b, ws, st);
    return;
  }
  if (k::conv3x3_wgrad_ws_bytes(sh) > ws_bytes) fail(RP_ERR_RANGE, "stem_bwd: workspace too small");
  k::conv3x3_wgrad_simt(sh, xr, g0, 1.f, gs + L.s_w, gs + L.s_b, ws, st);
}

void head_fwd(const rp_geometry& g, int nrows, const float* x_end, const float* pt, float* pooled, float* logits,
              cudaStream_t st) {
  prof::Scope scope(RP_PROF_HEAD, st, 0.0, 4.0 * nrows * g.height * g.width * g.channels);
  k::head_forward(nrows, g.height * g.width, g.channels, g.classes, x_end, pt, pt + (int64_t)g.channels * g.classes,
                  pooled, logits, st);
}

void head_loss_bwd(const rp_geometry& g, int nrows, const float* pooled, const float* logits, const float* pt,
                   const int32_t* labels, double* loss_dev, float* gt, float* g_out, void* ws, int64_t ws_bytes,
                   cudaStream_t st, void* p0 = nullptr, void* p1 = nullptr, float* scale = nullptr) {
  if (k::head_ws_bytes(nrows, g.channels, g.classes) > ws_bytes) fail(RP_ERR_RANGE, "head: workspace too small");
  prof::Scope scope(RP_PROF_HEAD, st, 0.0, 4.0 * nrows * g.height * g.width * g.channels);
  k::head_loss_backward(nrows, g.height * g.width, g.channels, g.classes, pooled, logits, pt, labels, loss_dev, gt,
                        gt + (int64_t)g.channels * g.classes, g_out, ws, st, p0, p1, scale);
}

void init_params(const rp_geometry& g, float* params, uint64_t* state, cudaStream_t st) {
  // make_net (network.cpp:49-68): s, blocks (w1, w2), t; Glorot with conv fans; zero biases.
  const ParamLayout L = ParamLayout::of(g);
  RP_CUDA(cudaMemsetAsync(params, 0, L.total * sizeof(float), st));
  auto glorot = [&](float* dst, int64_t fan_in, int64_t fan_out, int64_t n, double gain) {
    const double a = std::sqrt(6.0 / (double)(fan_in + fan_out));
    k::fill_uniform(dst, n, *state, -a, a, gain, st);
    *state += (uint64_t)n * kGamma;
  };
  const int64_t Ci = g.in_channels, C = g.channels, Ch = g.hidden;
  glorot(params + L.s_w, 9 * Ci, 9 * C, 9 * Ci * C, 2.0);
  const double branch = 2.2 / std::sqrt((double)std::max(g.blocks, 1));
  for (int l = 0; l < g.blocks; ++l) {
    float* pb = params + L.block0 + (int64_t)l * L.block_stride;
    glorot(pb + L.w1, 9 * C, 9 * Ch, 9 * C * Ch, 1.2);
    glorot(pb + L.w2, 9 * Ch, 9 * C, 9 * Ch * C, branch);
  }
  glorot(params + L.t_w, C, g.classes, C * g.classes, 1.0);
}

}  // namespace rp

using namespace rp;

extern "C" {

int64_t rp_op_workspace_bytes(const rp_geometry* g, int32_t nrows, int32_t math) {
  int64_t out = -1;
  guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    check_math(math);
    out = op_workspace_bytes(*g, nrows);
  });
  return out;
}

int64_t rp_op_reduce_workspace_bytes(void) { return k::reduce_workspace_bytes(); }

int rp_op_fill_uniform(float* dst, int64_t n, uint64_t* state, double lo, double hi, double scale, void* stream) {
  return guard([&] {
    need(state, "state");
    if (!(lo < hi)) fail(RP_ERR_RANGE, "rng_uniform: requires lo < hi");
    if (n > 0) need(dst, "dst");
    k::fill_uniform(dst, n, *state, lo, hi, scale, S(stream));
    *state += (uint64_t)n * kGamma;
  });
}

int rp_op_fill_normal(float* dst, int64_t n, uint64_t* state, double mean, double sigma, int32_t accumulate,
                      void* stream) {
  return guard([&] {
    need(state, "state");
    if (sigma < 0.0) fail(RP_ERR_RANGE, "rng_normal: sigma must be >= 0");
    if (n > 0) need(dst, "dst");
    k::fill_normal(dst, n, *state, mean, sigma, accumulate != 0, S(stream));
    *state += (uint64_t)(2 * n) * kGamma;
  });
}

int rp_op_init_params(const rp_geometry* g, float* params, uint64_t* state, void* stream) {
  return guard([&] {
    need(g, "geometry");
    need(params, "params");
    need(state, "state");
    validate_geometry(*g);
    init_params(*g, params, state, S(stream));
  });
}

int rp_op_psi(int32_t kind, const float* lam, const float* x, int64_t n, double* out, void* ws, void* stream) {
  return guard([&] {
    need(out, "out");
    if (kind < 0 || kind > 2) fail(RP_ERR_RANGE, "unknown penalty kind");
    if (n == 0) {
      *out = 0.0;
      return;
    }
    need(ws, "ws");
    double* dev = reinterpret_cast<double*>(static_cast<char*>(ws) + k::reduce_workspace_bytes() - 16);
    k::psi_device(kind, lam, x, n, ws, dev, S(stream));
    RP_CUDA(cudaMemcpyAsync(out, dev, sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
    RP_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int rp_op_psi_grad(int32_t kind, const float* lam, const float* x, int64_t n, double scale, float* out, void* ws,
                   void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 2) fail(RP_ERR_RANGE, "unknown penalty kind");
    k::psi_grad(kind, lam, x, n, scale, out, ws, S(stream));
  });
}

int rp_op_synthetic_grad(int32_t kind, const float* lam_next, const float* x_end, const float* kappa_next, int64_t n,
                         double w, float* g, void* ws, void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 2) fail(RP_ERR_RANGE, "unknown penalty kind");
    prof::Scope scope(RP_PROF_SYNTHETIC, S(stream), 0.0, (double)n * (kappa_next ? 16.0 : 12.0));
    k::synthetic_grad(kind, lam_next, x_end, kappa_next, n, w, g, ws, S(stream));
  });
}

int rp_op_synthetic_grad_planes(int32_t kind, const float* lam_next, const float* x_end, const float* kappa_next,
                                int64_t n, double w, float* g, void* p0, void* p1, float* scale, void* ws,
                                void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 2) fail(RP_ERR_RANGE, "unknown penalty kind");
    need(p0, "p0");
    if (p1) need(scale, "scale");
    // the pair: + a second read of g for the scaled split
    prof::Scope scope(RP_PROF_SYNTHETIC, S(stream), 0.0, (double)n * ((kappa_next ? 16.0 : 12.0) + (p1 ? 8.0 : 2.0)));
    k::synthetic_grad(kind, lam_next, x_end, kappa_next, n, w, g, ws, S(stream), p0, p1, scale);
  });
}

int64_t rp_op_plane_scale_bytes(void) { return k::plane_scale_bytes(); }

int rp_op_correct(int32_t kind, float* lam, const float* x_prev, const float* p, float* kappa, int64_t n, double w,
                  double eta_l, int32_t update_lambda, double kappa_coef, int32_t update_kappa, void* ws,
                  void* stream) {
  return guard([&] {
    if (kind < 0 || kind > 2) fail(RP_ERR_RANGE, "unknown penalty kind");
    const double per = (update_lambda ? 12.0 + (kappa ? 4.0 : 0.0) : 8.0) + (update_kappa ? 8.0 : 0.0);
    prof::Scope scope(RP_PROF_CORRECT, S(stream), 0.0, (double)n * per);
    k::correct(kind, lam, x_prev, p, kappa, n, w, eta_l, update_lambda != 0, kappa_coef, update_kappa != 0, ws,
               S(stream));
  });
}

int rp_op_sgd(float* w, const float* g, float* v, int64_t n, double lr, double momentum, void* stream) {
  return guard([&] {
    prof::Scope scope(RP_PROF_SGD, S(stream), 0.0, (double)n * (v ? 20.0 : 12.0));
    k::sgd(w, g, v, n, lr, momentum, S(stream));
  });
}

int64_t rp_op_conv3x3_workspace_bytes(int32_t ci, int32_t co);

int rp_op_conv3x3(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const float* in, const float* w_hwio,
                  int32_t dgrad, const float* bias, const float* aux, double hstep, int32_t epi, float* out,
                  int32_t math, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    check_math(math);
    if (epi < 0 || epi > 5) fail(RP_ERR_RANGE, "conv3x3: unknown epilogue");
    if (n < 0 || h < 1 || w < 1 || ci < 1 || co < 1) fail(RP_ERR_SHAPE, "conv3x3: bad shape");
    const k::ConvShape s{n, h, w, ci, co};
    if (ws_bytes < rp_op_conv3x3_workspace_bytes(std::min(ci, co), std::max(ci, co)))
      fail(RP_ERR_RANGE, "conv3x3: workspace too small");
    conv(s, in, w_hwio, dgrad != 0, bias, aux, (float)hstep, epi, out, math, ws, RP_PROF_OTHER,
         aux != nullptr, S(stream));
  });
}

int rp_op_conv3x3_wgrad(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const float* in, const float* gout,
                        double scale, float* gw, float* gb, int32_t math, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    check_math(math);
    if (n < 1 || h < 1 || w < 1 || ci < 1 || co < 1) fail(RP_ERR_SHAPE, "conv3x3_wgrad: bad shape");
    const k::ConvShape s{n, h, w, ci, co};
    if (ws_bytes < wgrad_ws_bytes(s)) fail(RP_ERR_RANGE, "conv3x3_wgrad: workspace too small");
    wgrad(s, in, gout, (float)scale, gw, gb, math, ws, S(stream));
  });
}

int rp_op_set_concurrent_stages(int32_t ways) {
  return guard([&] {
    if (ways < 1) fail(RP_ERR_RANGE, "set_concurrent_stages: ways must be >= 1");
    k::conv_pm_set_share(ways);
  });
}

int32_t rp_op_concurrent_stages(void) { return k::conv_pm_share(); }

int rp_op_set_plane_conv_kernel(int32_t which) {
  return guard([&] {
    if (which < -1 || which > 1) fail(RP_ERR_RANGE, "set_plane_conv_kernel: which must be -1, 0 or 1");
    g_plane_conv.store(which);
  });
}

int32_t rp_op_plane_conv_kernel(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co) {
  const k::ConvShape s{n, h, w, ci, co};
  return plane_conv_pm(s) ? 1 : (k::conv3x3_tc_supported(s) ? 0 : -1);
}

int rp_op_conv3x3_planes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const void* in_planes,
                         const float* w_hwio, int32_t dgrad, const float* bias, const float* aux, double hstep,
                         int32_t epi, float* out, void* out_planes, const float* in_scale, const float* out_scale,
                         void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    if (epi < 0 || epi > 5) fail(RP_ERR_RANGE, "conv3x3_planes: unknown epilogue");
    if (n < 0 || h < 1 || w < 1 || ci < 1 || co < 1) fail(RP_ERR_SHAPE, "conv3x3_planes: bad shape");
    const k::ConvShape s{n, h, w, ci, co};
    if (!plane_conv_supported(s)) fail(RP_ERR_SHAPE, "conv3x3_planes: unsupported shape (Co % 64 or Co in {16, 32}, Ci % 16)");
    if (ws_bytes < rp_op_conv3x3_workspace_bytes(std::min(ci, co), std::max(ci, co)))
      fail(RP_ERR_RANGE, "conv3x3_planes: workspace too small");
    if (n > 0) need(in_planes, "in_planes");
    conv(s, nullptr, w_hwio, dgrad != 0, bias, aux, (float)hstep, epi, out, RP_MATH_FP32, ws, RP_PROF_OTHER,
         aux != nullptr, S(stream), out_planes, in_planes, nullptr, in_scale, out_scale);
  });
}

int64_t rp_op_conv3x3_wgrad_workspace_bytes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co) {
  return wgrad_ws_bytes({n, h, w, ci, co});
}

int64_t rp_op_conv3x3_workspace_bytes(int32_t ci, int32_t co) {
  // either orientation (fprop ci -> co, or its dgrad co -> ci)
  return align256(std::max({k::conv3x3_tc_ws_bytes({1, 1, 1, ci, co}), k::conv3x3_tc_ws_bytes({1, 1, 1, co, ci}),
                            (int64_t)9 * ci * co * 4}));
}

int rp_op_block_fwd(const rp_geometry* g, int32_t nrows, const float* x, const float* pb, float* a, float* x_next,
                    int32_t math, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    check_math(math);
    if (nrows <= 0) return;
    block_fwd(*g, nrows, x, pb, a, x_next, math, ws, ws_bytes, S(stream));
  });
}

int rp_op_block_bwd(const rp_geometry* g, int32_t nrows, const float* x, const float* a, const float* pb,
                    float* g_io, float* dpre, float* gb, int32_t math, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    check_math(math);
    if (nrows <= 0) return;
    need(ws, "ws");
    block_bwd(*g, nrows, x, a, pb, g_io, dpre, gb, math, ws, ws_bytes, S(stream));
  });
}

int32_t rp_op_block_planes_supported(const rp_geometry* g, int32_t nrows, int32_t math) {
  if (!g || nrows <= 0) return 0;
  return planes_path(*g, nrows, math) ? 1 : 0;
}

int rp_op_block_fwd_planes(const rp_geometry* g, int32_t nrows, const float* x, const void* x_planes,
                           const float* pb, float* a, float* x_next, void* a_planes, void* x_next_planes,
                           const void* filters, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    if (!planes_path(*g, nrows, RP_MATH_FP32)) fail(RP_ERR_SHAPE, "block_fwd_planes: geometry not on the plane path");
    need(x, "x");
    need(x_planes, "x_planes");
    need(pb, "pb");
    need(a, "a");
    need(x_next, "x_next");
    need(a_planes, "a_planes");
    block_fwd_planes(*g, nrows, x, x_planes, pb, a, x_next, a_planes, x_next_planes, filters, ws, ws_bytes,
                     S(stream));
  });
}

int64_t rp_op_planes_filters_bytes(const rp_geometry* g, int32_t nblocks) {
  if (!g || nblocks <= 0) return 0;
  return (int64_t)nblocks * 2 * planes_filter_bytes(*g);
}

int rp_op_prep_planes_filters(const rp_geometry* g, const float* pb, int32_t nblocks, int32_t dgrad, void* out,
                              void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    if (nblocks <= 0) return;
    need(pb, "pb");
    need(out, "out");
    prep_planes_filters(*g, pb, nblocks, dgrad != 0, out, S(stream));
  });
}

int rp_op_block_bwd_planes(const rp_geometry* g, int32_t nrows, const void* x_planes, const float* a,
                           const void* a_planes, const float* pb, float* g_io, void* g_planes, const float* g_scale,
                           float* dpre, void* dpre_planes, float* gb, const void* filters, void* ws,
                           int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    if (!planes_path(*g, nrows, RP_MATH_FP32)) fail(RP_ERR_SHAPE, "block_bwd_planes: geometry not on the plane path");
    if (ws_bytes < op_workspace_bytes(*g, nrows)) fail(RP_ERR_RANGE, "block_bwd_planes: workspace too small");
    need(x_planes, "x_planes");
    need(a, "a");
    need(a_planes, "a_planes");
    need(pb, "pb");
    need(g_io, "g_io");
    need(g_planes, "g_planes");
    need(dpre, "dpre");
    need(dpre_planes, "dpre_planes");
    need(gb, "gb");
    block_bwd_planes(*g, nrows, x_planes, a, a_planes, pb, g_io, g_planes, g_scale, dpre, dpre_planes, gb, filters,
                     ws, ws_bytes, S(stream));
  });
}

int32_t rp_op_block_bf16_tape_supported(const rp_geometry* g, int32_t nrows, int32_t math) {
  if (!g || nrows <= 0) return 0;
  return bf16_tape_path(*g, nrows, math) ? 1 : 0;
}

int rp_op_block_fwd_bf16t(const rp_geometry* g, int32_t nrows, const float* x, const void* x16, const float* pb,
                          void* a16, void* d16, float* x_next, void* x_next16, void* ws, int64_t ws_bytes,
                          void* stream) {
  return guard([&] {
    need(g, "geometry");
    if (!bf16_tape_path(*g, nrows, RP_MATH_BF16)) fail(RP_ERR_SHAPE, "block_fwd_bf16t: geometry not on the bf16 tape path");
    need(x, "x");
    need(x16, "x16");
    need(pb, "pb");
    need(a16, "a16");
    if (g->activation == RP_ACT_TANH) need(d16, "d16");
    need(x_next, "x_next");
    block_fwd_bf16t(*g, nrows, x, x16, pb, a16, d16, x_next, x_next16, ws, ws_bytes, S(stream));
  });
}

int rp_op_block_bwd_bf16t(const rp_geometry* g, int32_t nrows, const void* x16, const void* a16, const void* d16,
                          const float* pb, float* g_io, void* g16, void* dpre16, float* gb, void* ws,
                          int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    if (!bf16_tape_path(*g, nrows, RP_MATH_BF16)) fail(RP_ERR_SHAPE, "block_bwd_bf16t: geometry not on the bf16 tape path");
    if (ws_bytes < op_workspace_bytes(*g, nrows)) fail(RP_ERR_RANGE, "block_bwd_bf16t: workspace too small");
    need(x16, "x16");
    need(a16, "a16");
    if (g->activation == RP_ACT_TANH) need(d16, "d16");
    need(pb, "pb");
    need(g_io, "g_io");
    need(g16, "g16");
    need(dpre16, "dpre16");
    need(gb, "gb");
    block_bwd_bf16t(*g, nrows, x16, a16, d16, pb, g_io, g16, dpre16, gb, ws, ws_bytes, S(stream));
  });
}

int64_t rp_op_conv3x3_wgrad_bf16p_workspace_bytes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co) {
  return k::conv3x3_wgrad_bf16p_ws_bytes(k::ConvShape{n, h, w, ci, co});
}

int rp_op_conv3x3_wgrad_bf16p(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const void* x16,
                              const void* g16, double scale, float* gw, float* gb, void* ws, int64_t ws_bytes,
                              void* stream) {
  return guard([&] {
    const k::ConvShape s{n, h, w, ci, co};
    if (!k::conv3x3_wgrad_bf16p_supported(s)) fail(RP_ERR_SHAPE, "conv3x3_wgrad_bf16p: unsupported shape");
    if (ws_bytes < k::conv3x3_wgrad_bf16p_ws_bytes(s)) fail(RP_ERR_RANGE, "conv3x3_wgrad_bf16p: workspace too small");
    need(x16, "x16");
    need(g16, "g16");
    need(gw, "gw");
    wgrad_bf16p(s, x16, g16, (float)scale, gw, gb, ws, S(stream));
  });
}

int rp_op_split_planes(const float* in, int64_t n, void* p0, void* p1, float* scale_out, void* stream) {
  return guard([&] {
    if (n > 0) {
      need(in, "in");
      need(p0, "p0");
    }
    if (scale_out && !p1) fail(RP_ERR_RANGE, "split_planes: a scale needs the plane pair (p1)");
    k::split_planes(in, n, p0, p1, S(stream), scale_out);
  });
}

int64_t rp_op_conv3x3_wgrad_planes_workspace_bytes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co) {
  const k::ConvShape s{n, h, w, ci, co};
  return std::max(k::conv3x3_wgrad_planes_ws_bytes(s), k::conv3x3_wgrad_small_ws_bytes(s));
}

int rp_op_conv3x3_wgrad_planes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const void* x0, const void* x1,
                               const void* g0, const void* g1, double scale, const float* g_scale, float* gw,
                               float* gb, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    const k::ConvShape s{n, h, w, ci, co};
    const bool small = !k::conv3x3_wgrad_planes_supported(s) && k::conv3x3_wgrad_small_supported(s);
    if (!small && !k::conv3x3_wgrad_planes_supported(s))
      fail(RP_ERR_SHAPE, "conv3x3_wgrad_planes: unsupported shape (Ci, Co % 64 == 0, or Ci 16 and Co in {16, 32})");
    if (ws_bytes < (small ? k::conv3x3_wgrad_small_ws_bytes(s) : k::conv3x3_wgrad_planes_ws_bytes(s)))
      fail(RP_ERR_RANGE, "conv3x3_wgrad_planes: workspace too small");
    need(x0, "x0");
    need(x1, "x1");
    need(g0, "g0");
    need(g1, "g1");
    need(gw, "gw");
    prof::Scope ps(RP_PROF_CONV_WGRAD, S(stream), conv_flops(s), 2.0 * (double)s.pixels() * (s.ci + s.co));
    if (small)
      k::conv3x3_wgrad_small(s, x0, x1, g0, g1, (float)scale, gw, gb, ws, S(stream), g_scale);
    else
      k::conv3x3_wgrad_planes(s, x0, x1, g0, g1, (float)scale, gw, gb, ws, S(stream), g_scale);
  });
}

int rp_op_stem_fwd(const rp_geometry* g, int32_t nrows, const float* x_raw, const float* ps, float* x0, int32_t math,
                   void*, int64_t, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    check_math(math);
    if (nrows <= 0) return;
    stem_fwd(*g, nrows, x_raw, ps, x0, S(stream));
  });
}

int rp_op_stem_fwd_planes(const rp_geometry* g, int32_t nrows, const float* x_raw, const float* ps, float* x0, void* p0,
                          void* p1, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    need(p0, "p0");
    if (nrows <= 0) return;
    stem_fwd(*g, nrows, x_raw, ps, x0, S(stream), p0, p1);
  });
}

int rp_op_stem_bwd(const rp_geometry* g, int32_t nrows, const float* x_raw, const float* g0, float* gs, void* ws,
                   int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    if (nrows <= 0) return;
    stem_bwd(*g, nrows, x_raw, g0, gs, ws, ws_bytes, S(stream));
  });
}

int rp_op_head_fwd(const rp_geometry* g, int32_t nrows, const float* x_end, const float* pt, float* pooled,
                   float* logits, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    head_fwd(*g, nrows, x_end, pt, pooled, logits, S(stream));
  });
}

int rp_op_head_loss_bwd(const rp_geometry* g, int32_t nrows, const float* pooled, const float* logits,
                        const float* pt, const int32_t* labels, double* loss_dev, float* gt, float* g_out, void* ws,
                        int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    head_loss_bwd(*g, nrows, pooled, logits, pt, labels, loss_dev, gt, g_out, ws, ws_bytes, S(stream));
  });
}

int rp_op_head_loss_bwd_planes(const rp_geometry* g, int32_t nrows, const float* pooled, const float* logits,
                               const float* pt, const int32_t* labels, double* loss_dev, float* gt, float* g_out,
                               void* p0, void* p1, float* scale, void* ws, int64_t ws_bytes, void* stream) {
  return guard([&] {
    need(g, "geometry");
    validate_geometry(*g);
    need(p0, "p0");
    if (p1) need(scale, "scale");
    head_loss_bwd(*g, nrows, pooled, logits, pt, labels, loss_dev, gt, g_out, ws, ws_bytes, S(stream), p0, p1, scale);
  });
}

int rp_op_argmax_hits(const float* logits, const int32_t* labels, int32_t nrows, int32_t classes, int64_t* hits,
                      void* ws, void* stream) {
  return guard([&] {
    need(hits, "hits");
    need(ws, "ws");
    auto* dev = static_cast<unsigned long long*>(ws);
    k::argmax_hits(logits, labels, nrows, classes, dev, S(stream));
    unsigned long long h = 0;
    RP_CUDA(cudaMemcpyAsync(&h, dev, sizeof(h), cudaMemcpyDeviceToHost, S(stream)));
    RP_CUDA(cudaStreamSynchronize(S(stream)));
    *hits = (int64_t)h;
  });
}

int64_t rp_op_eval_workspace_bytes(int32_t nrows) { return k::eval_ws_bytes(std::max(0, nrows)) + 16; }

int rp_op_eval_loss_accuracy(const float* logits, const int32_t* labels, int32_t nrows, int32_t classes,
                             double* loss_out, int64_t* hits_out, int32_t* pred, void* ws, int64_t ws_bytes,
                             void* stream) {
  return guard([&] {
    if (nrows < 0 || classes < 2 || classes > 1024) fail(RP_ERR_SHAPE, "eval: bad shape");
    need(ws, "ws");
    if (ws_bytes < rp_op_eval_workspace_bytes(nrows)) fail(RP_ERR_RANGE, "eval: workspace too small");
    if (nrows > 0) {
      need(logits, "logits");
      need(labels, "labels");
    }
    double* out2 = static_cast<double*>(ws);
    k::eval_loss_hits(logits, labels, nrows, classes, out2, pred, static_cast<char*>(ws) + 16, S(stream));
    double h[2] = {0.0, 0.0};
    RP_CUDA(cudaMemcpyAsync(h, out2, sizeof(h), cudaMemcpyDeviceToHost, S(stream)));
    RP_CUDA(cudaStreamSynchronize(S(stream)));
    if (loss_out) *loss_out = h[0];
    if (hits_out) *hits_out = (int64_t)h[1];
  });
}

}  // extern "C"
