// Internal launch API of the sm_100a kernels (namespace rp::k).  The C ABI
// (capi.cpp) and the C++ host classes (host/) call these.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rp::k {

// ---- elementwise / reductions (elementwise.cu) -----------------------------
int64_t reduce_workspace_bytes();
void fill_uniform(float* dst, int64_t n, uint64_t state, double lo, double hi, double scale, cudaStream_t s);
void fill_normal(float* dst, int64_t n, uint64_t state, double mean, double sigma, bool accumulate,
                 cudaStream_t s);
void psi_device(int kind, const float* a, const float* b, int64_t n, void* ws, double* out_dev, cudaStream_t s);
void psi_grad(int kind, const float* lam, const float* x, int64_t n, double scale, float* out, void* ws,
              cudaStream_t s);
// p0 / p1 (optional): also the planes of g (planes.cuh): p1 non-null: the fp16 pair of g s with
// the cotangent scale s written to *scale (a buffer of plane_scale_bytes()); p1 null: the bf16
// single plane
void synthetic_grad(int kind, const float* lam_next, const float* x_end, const float* kappa, int64_t n, double w,
                    float* g, void* ws, cudaStream_t s, void* p0 = nullptr, void* p1 = nullptr,
                    float* scale = nullptr);
void correct(int kind, float* lam, const float* x_prev, const float* p, float* kappa, int64_t n, double w,
             double eta, bool update_lambda, double kappa_coef, bool update_kappa, void* ws, cudaStream_t s);
void sgd(float* w, const float* g, float* v, int64_t n, double lr, double momentum, cudaStream_t s);

// ---- 3x3 convolutions (conv_simt.cu, conv_tc.cu) ----------------------------
// Epilogues fused into the implicit-GEMM store (network.cpp:82-106):
enum Epilogue : int {
  EPI_BIAS = 0,      // out = acc + bias                           (stem, identity conv1)
  EPI_BIAS_TANH = 1, // out = tanh(acc + bias)                     (conv1: a)
  EPI_RESID = 2,     // out = aux + h (acc + bias)                 (conv2: x' = x + h f)
  EPI_TANH_BWD = 3,  // out = h acc (1 - aux^2)                    (dgrad2 -> dpre, aux = a)
  EPI_ADD = 4,       // out = aux + acc   (in place allowed)       (dgrad1: g_prev = g + ...)
  EPI_SCALE = 5,     // out = h acc                                (identity dgrad2)
  EPI_DTANH16 = 6    // out = h acc aux16, aux16 = bf16(1 - a^2)   (bf16 tape dgrad2)
};

struct ConvShape {
  int n, h, w;  // batch and spatial
  int ci, co;   // channels
  int64_t pixels() const { return (int64_t)n * h * w; }
};

// out = epilogue(conv3x3(in, w_hwio)) with zero padding 1, stride 1.  NHWC fp32.
void conv3x3_fwd_simt(const ConvShape& s, const float* in, const float* w_hwio, const float* bias,
                      const float* aux, float h, int epi, float* out, cudaStream_t st);
// dgrad weight relayout: wd[ky][kx][co][ci] = w[2-ky][2-kx][ci][co]
void conv3x3_dgrad_weights(const float* w_hwio, int ci, int co, float* wd, cudaStream_t st);
// gw[tap][ci][co] = scale * sum_pix in(pix+tap)[ci] g(pix)[co], gb[co] = scale * sum_pix g(pix)[co]
// (deterministic split-K over pixels; ws >= conv3x3_wgrad_ws_bytes).
int64_t conv3x3_wgrad_ws_bytes(const ConvShape& s);
void conv3x3_wgrad_simt(const ConvShape& s, const float* in, const float* g, float scale, float* gw, float* gb,
                        void* ws, cudaStream_t st);

// tcgen05 implicit GEMM (conv_tc.cu): fprop, or dgrad when dgrad_weights (w_hwio is
// then the forward conv's HWIO [3][3][s.co][s.ci] weight).  mode: 0 TF32, 1 3xTF32 (fp32-
// accurate, default), 2 3xBF16 (fp32-accurate through bf16 splits; RP_FP32_SPLIT=bf16x3).
enum { TC_MODE_TF32 = 0, TC_MODE_X3TF32 = 1, TC_MODE_X3BF16 = 2 };
bool conv3x3_tc_supported(const ConvShape& s);
int64_t conv3x3_tc_ws_bytes(const ConvShape& s);
// out_planes (optional): fp16 [2][pixels * co] receives the plane pair of out * (*out_scale).
// in_planes (optional): fp16 [2][pixels * ci], the input times (*in_scale) as a plane pair
// (in unused): the 2-MMA plane mode (planes.cuh, ~2^-23 relative).  Scales: device scalars,
// null = 1.
void conv3x3_fwd_tc(const ConvShape& s, const float* in, const float* w_hwio, bool dgrad_weights, const float* bias,
                    const float* aux, float h, int epi, float* out, int mode, void* ws, cudaStream_t st,
                    void* out_planes = nullptr, const void* in_planes = nullptr, const void* wprep = nullptr,
                    const float* in_scale = nullptr, const float* out_scale = nullptr);
// The plane-mode A operands of both filters of nblocks blocks in one launch (filter j of block
// b: HWIO at pb + b block_stride + off[j], ci_src[j] x co_src[j]; dgrad: flipped/transposed) into
// out + (2 b + j) * 9 ci co * 2 fp16 (W * kWeightPlaneScale) -- the wprep argument of conv3x3_fwd_tc.
void prep_filters_planes(const float* pb, int64_t block_stride, int nblocks, const int64_t off[2],
                         const int ci_src[2], const int co_src[2], bool dgrad, void* out, cudaStream_t st);

// One conv's plane-mode filter (the layout prep_filters_planes writes), 9 ci co * 2 fp16.
void prep_filter_planes(const float* w_hwio, int ci_src, int co_src, bool dgrad, void* out, cudaStream_t st);
// The positions-as-M plane conv (conv_pm.cu): fp16 plane-pair input only, Co in {16, 32, 64},
// Ci % 16 == 0; 3 tensor products per MAC.  Arguments as conv3x3_fwd_tc's plane mode.
bool conv3x3_pm_supported(const ConvShape& s);
// Stages issuing concurrently on one GPU (this host thread's launches): with 2 or more, a
// conv_pm launch takes half the SMs so two stages' convs run side by side and one's fill and
// drain overlap the other's steady state (measured +3 % on C3).  RP_CONV_PM_CTAS overrides.
// (C ABI: rp_op_set_concurrent_stages / rp_op_concurrent_stages)
void conv_pm_set_share(int ways);
int conv_pm_share();
void conv3x3_fwd_pm(const ConvShape& s, const float* w_hwio, bool dgrad_weights, const float* bias, const float* aux,
                    float h, int epi, float* out, void* ws, cudaStream_t st, void* out_planes, const void* in_planes,
                    const void* wprep, const float* in_scale, const float* out_scale);

// tcgen05 bf16-operand conv, fp32 accumulate (conv_bf16.cu): Co % 128 == 0, Ci % 32 == 0.
bool conv3x3_bf16_supported(const ConvShape& s);
int64_t conv3x3_bf16_ws_bytes(const ConvShape& s);
// out_bf16 (optional): receives bf16(out) as well (the single-plane wgrad operand).
void conv3x3_fwd_bf16(const ConvShape& s, const float* in, const float* w_hwio, bool dgrad_weights, const float* bias,
                      const float* aux, float h, int epi, float* out, void* ws, cudaStream_t st,
                      void* out_bf16 = nullptr);
// The bf16 tape form: the input is already bf16 (in16, loaded by TMA straight into the MMA
// layout, no converter pass); out (fp32) may be null; out16 = bf16(out), out16d = bf16(1 -
// out^2) (EPI_BIAS_TANH: the derivative the backward's EPI_DTANH16 reads as aux16), each
// optional.
void conv3x3_fwd_bf16_in16(const ConvShape& s, const void* in16, const float* w_hwio, bool dgrad_weights,
                           const float* bias, const float* aux, const void* aux16, float h, int epi, float* out,
                           void* out16, void* out16d, void* ws, cudaStream_t st);

// tcgen05 weight gradient (conv_wgrad_tc.cu): gw[tap][ci][co], gb[co] (may be null),
// scaled; deterministic (per-CTA partials + fixed-order fp64 reduce).
bool conv3x3_wgrad_tc_supported(const ConvShape& s, bool three);
int64_t conv3x3_wgrad_tc_ws_bytes(const ConvShape& s, bool three);
void conv3x3_wgrad_tc(const ConvShape& s, const float* in, const float* g, float scale, float* gw, float* gb,
                      bool three, void* ws, cudaStream_t st);

// tcgen05 bf16-operand weight gradient (conv_wgrad_bf16.cu): Ci, Co % 128 == 0.
bool conv3x3_wgrad_bf16_supported(const ConvShape& s);
int64_t conv3x3_wgrad_bf16_ws_bytes(const ConvShape& s);
void conv3x3_wgrad_bf16(const ConvShape& s, const float* in, const float* g, float scale, float* gw, float* gb,
                        void* ws, cudaStream_t st);

// tcgen05 weight gradient from fp16 plane pairs x = x0 + x1, g s = g0 + g1 (conv_wgrad_planes.cu):
// the fp32-accurate wgrad when the producers wrote the planes; Ci, Co % 64 == 0.  gscale: the
// g planes' scale s (device scalar, null = 1), divided out.
bool conv3x3_wgrad_planes_supported(const ConvShape& s);
int64_t conv3x3_wgrad_planes_ws_bytes(const ConvShape& s);
void conv3x3_wgrad_planes(const ConvShape& s, const void* x0, const void* x1, const void* g0, const void* g1,
                          float scale, float* gw, float* gb, void* ws, cudaStream_t st, const float* gscale);
// Two weight gradients of the same shape in one launch (the block's gW1 and gW2 when C ==
// hidden): xa / ga = {plane 0, plane 1} of job a's operands, likewise job b.
void conv3x3_wgrad_planes_pair(const ConvShape& s, const void* const xa[2], const void* const ga[2], float scale_a,
                               float* gwa, float* gba, const void* const xb[2], const void* const gb2[2],
                               float scale_b, float* gwb, float* gbb, void* ws, cudaStream_t st, const float* gsc_a,
                               const float* gsc_b);
// The 16-channel form (conv_wgrad_small.cu, config C1): Ci == 16, Co in {16, 32}; arguments as
// conv3x3_wgrad_planes.
bool conv3x3_wgrad_small_supported(const ConvShape& s);
int64_t conv3x3_wgrad_small_ws_bytes(const ConvShape& s);
void conv3x3_wgrad_small(const ConvShape& s, const void* x0, const void* x1, const void* g0, const void* g1,
                         float scale, float* gw, float* gb, void* ws, cudaStream_t st, const float* gscale);
// The same kernel on single bf16 planes (RP_MATH_BF16): x, g one bf16 NHWC tensor each,
// 128-channel blocks (Ci, Co % 128 == 0); bf16 x bf16 products, fp32 accumulate.
bool conv3x3_wgrad_bf16p_supported(const ConvShape& s);
int64_t conv3x3_wgrad_bf16p_ws_bytes(const ConvShape& s);
void conv3x3_wgrad_bf16p(const ConvShape& s, const void* x, const void* g, float scale, float* gw, float* gb,
                         void* ws, cudaStream_t st);
// two of them (same shape) in one launch
bool conv3x3_wgrad_bf16p_pair_supported(const ConvShape& s);
void conv3x3_wgrad_bf16p_pair(const ConvShape& s, const void* xa, const void* ga, float scale_a, float* gwa,
                              float* gba, const void* xb, const void* gb2, float scale_b, float* gwb, float* gbb,
                              void* ws, cudaStream_t st);
// fp32 [n] -> planes (planes.cuh; n % 4 == 0): p1 non-null: the fp16 pair, of v * s when
// scale_out is given (s from max |v| on device, stored at scale_out[0]; the buffer must hold
// plane_scale_bytes()), else of v; p1 null: the bf16 single plane.
constexpr int kPlaneScalePartOffset = 16;     // floats: [0] the scale, [16, 16 + parts) max partials
constexpr int kPlaneScaleMaxParts = 1024;
inline int64_t plane_scale_bytes() { return 4LL * (kPlaneScalePartOffset + 2 * kPlaneScaleMaxParts); }   // 8.2 KB
void split_planes(const float* in, int64_t n, void* p0, void* p1, cudaStream_t st, float* scale_out = nullptr);
// the scaled pair from per-CTA max |v| partials already computed by the producer (part[0, nparts))
void split_planes_from_parts(const float* in, int64_t n, void* p0, void* p1, const float* part, int nparts,
                             float* scale_out, cudaStream_t st);

// ---- stem S (stem.cu): Cin <= 4 streaming kernels (SIMT conv path otherwise)
bool stem_supported(const ConvShape& s);
int64_t stem_wgrad_ws_bytes(const ConvShape& s);
// p0 (and p1, nullable): the output's planes as split_planes makes them (unscaled), in the same pass
void stem_fwd(const ConvShape& s, const float* x, const float* w, const float* b, float* out, cudaStream_t st,
              void* p0 = nullptr, void* p1 = nullptr);
void stem_wgrad(const ConvShape& s, const float* x, const float* g, float scale, float* gw, float* gb, void* ws,
                cudaStream_t st);

// ---- head (head.cu) -------------------------------------------------------
int64_t head_ws_bytes(int nrows, int channels, int classes);
void head_forward(int nrows, int hw, int channels, int classes, const float* x_end, const float* t_w,
                  const float* t_b, float* pooled, float* logits, cudaStream_t st);
void head_loss_backward(int nrows, int hw, int channels, int classes, const float* pooled, const float* logits,
                        const float* t_w, const int32_t* labels, double* loss_dev, float* gt_w, float* gt_b,
                        float* g_out, void* ws, cudaStream_t st, void* p0 = nullptr, void* p1 = nullptr,
                        float* scale = nullptr);
void argmax_hits(const float* logits, const int32_t* labels, int nrows, int classes, unsigned long long* hits_dev,
                 cudaStream_t st);
// evaluation (network.cpp:193-234): out2[0] = mean softmax-CE, out2[1] = argmax hits (ties to the
// lowest class), both deterministic; pred (nullable) = per-row argmax.  ws >= eval_ws_bytes(nrows).
int64_t eval_ws_bytes(int nrows);
void eval_loss_hits(const float* logits, const int32_t* labels, int nrows, int classes, double* out2, int32_t* pred,
                    void* ws, cudaStream_t st);

}  // namespace rp::k
