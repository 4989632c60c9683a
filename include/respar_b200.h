/*
 * respar_b200.h — C ABI of the B200-native layer-parallel ResNet training step.
 *
 * This is the drop-in boundary.  The reference (respar,
 * /root/reference/proj) has no FFI of its own: its boundary is the C++ library API
 * in include/respar/ (*.hpp), consumed by train(), the CLI and the pybind11 module.
 * The B200 build keeps that C++ surface (paper_2009_01462_b200/csrc/host/respar_b200.hpp,
 * namespace respar::b200) and puts this C ABI under it and beside it:
 *
 *   - rp_op_*      stream-ordered kernels on caller-owned device buffers
 *                  (what the C++ host classes call);
 *   - rp_trainer_* an opaque DecoupledTrainer handle, one entry point per reference
 *                  method (what a ctypes / cffi / pybind front end binds).
 *
 * Conventions
 *   - every function returns int status (RP_OK = 0); rp_last_error() returns the
 *     thread-local message of the last failure.  No C++ exception crosses the ABI;
 *     the C++ and Python wrappers rethrow the reference's exception types
 *     (ShapeError / ConfigError / std::logic_error / std::invalid_argument /
 *     StageError) from the status code.
 *   - device pointers are plain pointers; `stream` is a cudaStream_t passed as void*.
 *   - the caller owns every buffer it passes; a trainer handle owns only its own
 *     device state (parameters, lambda/kappa/boundary storage, tapes, workspaces).
 *   - tensors are NHWC fp32 (a reference Tensor(rows = N*H*W, cols = C) is the
 *     same bytes); conv weights are HWIO [3][3][Cin][Cout] (the centre tap is the
 *     reference's in x out matrix, x . W).
 *   - flat parameter layout == the reference make_net draw order
 *     (include/respar/network.hpp:43-45):
 *       s.w [3,3,Cin,C] s.b [C] { w1 [3,3,C,Ch] b1 [Ch] w2 [3,3,Ch,C] b2 [C] } x L
 *       t.w [C,classes] t.b [classes]
 */
#ifndef RESPAR_B200_H
#define RESPAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference's exception types) ---------------- */
enum {
  RP_OK = 0,
  RP_ERR_SHAPE = 1,    /* respar::ShapeError            (tensor.hpp:11-13)   */
  RP_ERR_CONFIG = 2,   /* respar::ConfigError           (config.hpp:13-15)   */
  RP_ERR_STATE = 3,    /* std::logic_error  (protocol)  (decoupled.cpp:89-92, 197-199, 160-163) */
  RP_ERR_RANGE = 4,    /* std::invalid_argument         (decoupled.cpp:66-69, 100-104, 117-122) */
  RP_ERR_STAGE = 5,    /* respar::StageError            (runtime.hpp:15-20)  */
  RP_ERR_CUDA = 6,
  RP_ERR_NCCL = 7,
  RP_ERR_DIVERGED = 8, /* std::runtime_error non-finite (decoupled.cpp:249-264) */
  RP_ERR_INTERNAL = 9
};

/* enums mirror penalty.hpp:15, config.hpp:17, network.hpp:12 */
enum { RP_PSI_SQUARED_L2 = 0, RP_PSI_L1 = 1, RP_PSI_LINF = 2 };
enum { RP_MODE_SERIAL = 0, RP_MODE_PENALTY = 1, RP_MODE_ALM = 2 };
enum { RP_ACT_TANH = 0, RP_ACT_IDENTITY = 1 };
/* conv arithmetic: fp32-accurate (3xTF32 tensor cores), plain TF32, bf16 tensor
 * cores with fp32 accumulate, or the SIMT FFMA path kept as an on-device checker. */
enum { RP_MATH_FP32 = 0, RP_MATH_TF32 = 1, RP_MATH_BF16 = 2, RP_MATH_SIMT = 3 };
/* multiplier rule: the reference's (decoupled.cpp:157-170) or the textbook one
 * kappa += beta (lambda - X) (north_star wording; opt-in only). */
enum { RP_KAPPA_RULE_REFERENCE = 0, RP_KAPPA_RULE_TEXTBOOK = 1 };
/* per-stage state buffers (StageState, decoupled.hpp:29-32) for get/set_state & co. */
enum { RP_STATE_LAMBDA = 0, RP_STATE_KAPPA = 1, RP_STATE_BOUNDARY_OUT = 2, RP_STATE_BOUNDARY_ADJOINT = 3 };

/* ResidualNet geometry (network.hpp:29-41 + conv geometry). */
typedef struct rp_geometry {
  int32_t in_channels; /* reference in_dim   */
  int32_t height;
  int32_t width;
  int32_t channels;    /* reference d        */
  int32_t hidden;      /* reference h        */
  int32_t blocks;      /* reference L        */
  int32_t classes;
  int32_t activation;  /* RP_ACT_*           */
  double step_h;       /* x + h f(x); 1 == reference */
} rp_geometry;

/* StepParams (decoupled.hpp:45-52). */
typedef struct rp_step_params {
  double beta;
  double tau;           /* < 0: single correction pass */
  double lr;
  double lambda_lr;
  double kappa_lr;
  int32_t max_corrections;
  double momentum;      /* 0 == the reference's plain gradient descent */
} rp_step_params;

const char* rp_last_error(void);
int rp_version(void);
/* Number of kernel launches this thread has issued through the library (for the
 * bench's gpu_launches claim). */
uint64_t rp_launch_count(void);
int64_t rp_param_count(const rp_geometry* g);
/* Offsets (in floats) of s.w, block l's w1, t.w in the flat layout. */
int64_t rp_param_offset_block(const rp_geometry* g, int32_t block);
int64_t rp_param_offset_head(const rp_geometry* g);

/* ---- live kernel profiling (bench roofline) ------------------------------- */
/* While enabled, every kernel class launched through the op layer is bracketed by
 * CUDA events on its own stream, with its algorithmic FLOPs and HBM bytes. */
enum { RP_PROF_CONV_FPROP = 0, RP_PROF_CONV_DGRAD = 1, RP_PROF_CONV_WGRAD = 2, RP_PROF_SYNTHETIC = 3,
       RP_PROF_CORRECT = 4, RP_PROF_SGD = 5, RP_PROF_HEAD = 6, RP_PROF_STEM = 7, RP_PROF_OTHER = 8,
       RP_PROF_NUM_CLASSES = 9 };
int rp_profile_enable(int32_t on);
/* Per class: launches, summed device ms, summed algorithmic FLOPs and bytes (arrays of
 * RP_PROF_NUM_CLASSES); synchronises the recorded events and clears the records. */
int rp_profile_collect(int64_t* launches, double* ms, double* flops, double* bytes);
const char* rp_profile_class_name(int32_t cls);

/* ---- stream-ordered ops on caller-owned device buffers --------------------- */
/* Counter-based splitmix64 fill: value i = lo + (hi-lo) * ((mix(state + (i+1)*gamma) >> 11) * 2^-53),
 * bit-identical to n calls of Rng::next_double (tensor.cpp:163-185), rounded to fp32.
 * Returns the advanced state in *state. */
int rp_op_fill_uniform(float* dst, int64_t n, uint64_t* state, double lo, double hi, double scale,
                       void* stream);
/* Box-Muller normal (tensor.cpp:187-197), 2 draws per value; dst += value when accumulate. */
int rp_op_fill_normal(float* dst, int64_t n, uint64_t* state, double mean, double sigma,
                      int32_t accumulate, void* stream);
/* Glorot-uniform conv net init (network.cpp:49-68), draw order s, blocks (w1, w2), t. */
int rp_op_init_params(const rp_geometry* g, float* params, uint64_t* state, void* stream);

/* Small reductions (psi, the LInf argmax) use `ws` (>= rp_op_reduce_workspace_bytes()). */
int64_t rp_op_reduce_workspace_bytes(void);
/* psi (penalty.cpp:38-58) over n elements, deterministic, fp64 accumulation; *out is host
 * (the call synchronises `stream`). */
int rp_op_psi(int32_t kind, const float* lam, const float* x, int64_t n, double* out, void* ws,
              void* stream);
/* psi_grads (penalty.cpp:60-87): d_lambda * scale into out (device); d_x == -d_lambda. */
int rp_op_psi_grad(int32_t kind, const float* lam, const float* x, int64_t n, double scale, float* out,
                   void* ws, void* stream);
/* Synthetic-loss upstream (decoupled.cpp:105-110): g = w d_x psi(lam_next, x_end) + kappa_next,
 * w = beta/# (kappa_next may be NULL == zero). */
int rp_op_synthetic_grad(int32_t kind, const float* lam_next, const float* x_end, const float* kappa_next,
                         int64_t n, double w, float* g, void* ws, void* stream);
/* Plane encodings (the tensor-core operands of the fp32 and bf16 paths):
 *   plane PAIR  (fp32 math): two fp16 [elements] buffers p0, p1 with v s = p0 + p1,
 *                p0 = fp16(v s), p1 = fp16(v s - p0) -- 22 significant bits (|v s - p0 - p1|
 *                <= 2^-24 |v s|) -- and a power-of-two scale s: 2^7 for forward activations
 *                (the meaning of every NULL scale argument; |v| < 2^8), the cotangent side a
 *                device scale (a buffer of rp_op_plane_scale_bytes(), the scale at float [0])
 *                set so max |g s| is in [2^7, 2^8).
 *   SINGLE plane (bf16 math): p0 = bf16(v). */
int64_t rp_op_plane_scale_bytes(void);
/* The same, also writing the planes of g for the tape paths: p1 non-NULL: the fp16 pair of
 * g s with s computed from max |g| and stored in *scale; p1 NULL: the bf16 single plane. */
int rp_op_synthetic_grad_planes(int32_t kind, const float* lam_next, const float* x_end, const float* kappa_next,
                                int64_t n, double w, float* g, void* p0, void* p1, float* scale, void* ws,
                                void* stream);
/* One correct_aux pass and/or correct_multiplier (decoupled.cpp:135-170), fused:
 *   if update_lambda: lam -= eta_l * (w d_lambda psi(lam, x_prev) + p - kappa)
 *   if update_kappa:  kappa -= kappa_coef * (lam - x_prev)   (lam already updated)
 * kappa may be NULL (== 0) when update_kappa == 0. */
int rp_op_correct(int32_t kind, float* lam, const float* x_prev, const float* p, float* kappa, int64_t n,
                  double w, double eta_l, int32_t update_lambda, double kappa_coef, int32_t update_kappa,
                  void* ws, void* stream);
/* W -= lr * g (apply_updates, network.cpp:174-191); with momentum: v = mu v + g; W -= lr v. */
int rp_op_sgd(float* w, const float* g, float* v, int64_t n, double lr, double momentum, void* stream);

/* One 3x3 conv (zero pad 1, stride 1) NHWC [n,h,w,ci] -> [n,h,w,co] with a fused
 * epilogue: 0 acc+bias, 1 tanh(acc+bias), 2 aux+h(acc+bias), 3 h acc (1-aux^2),
 * 4 aux+acc (out may equal aux), 5 h acc.  dgrad != 0: input-gradient conv, w_hwio is
 * the forward conv's [3][3][co][ci] weight.  math RP_MATH_FP32 (3xTF32 tcgen05),
 * RP_MATH_TF32, RP_MATH_SIMT. */
int rp_op_conv3x3(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const float* in, const float* w_hwio,
                  int32_t dgrad, const float* bias, const float* aux, double hstep, int32_t epi, float* out,
                  int32_t math, void* ws, int64_t ws_bytes, void* stream);
int64_t rp_op_conv3x3_workspace_bytes(int32_t ci, int32_t co);
/* The same conv reading its input as an fp16 plane pair (in_planes = [2][n h w ci]:
 * x in_s = p0 + p1) on a tcgen05 plane kernel (Co in {16, 32} or Co % 64 == 0, Ci % 16 == 0;
 * fp32-class accuracy); out_planes (optional, [2][n h w co] fp16) receives the plane pair of
 * out out_s.  in_scale / out_scale: device scalars (NULL = the activation scale 2^7). */
int rp_op_conv3x3_planes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const void* in_planes,
                         const float* w_hwio, int32_t dgrad, const float* bias, const float* aux, double hstep,
                         int32_t epi, float* out, void* out_planes, const float* in_scale, const float* out_scale,
                         void* ws, int64_t ws_bytes, void* stream);
/* Which plane kernel the plane convs use: 1 positions-as-M (conv_pm.cu: Co <= 64, 3 tensor
 * products per MAC), 0 channels-as-M (conv_tc.cu: Co % 64 == 0, 4 products), -1 the default
 * (process-wide; the env var RP_CONV_PM sets the initial value).  A shape only one kernel takes
 * always runs on it.  rp_op_plane_conv_kernel reports the choice for a shape (1, 0; -1 none). */
int rp_op_set_plane_conv_kernel(int32_t which);
/* Stages issuing kernels concurrently on the calling thread's GPU (default 1).  With n >= 2,
 * each positions-as-M plane conv takes 1 / max(2, n / 2) of the SMs, so several stages' convs
 * run side by side and one's fill and drain overlap the others' steady state.  The trainer sets
 * it around a stage's launches (thread-local; RP_CONV_PM_CTAS overrides the grid). */
int rp_op_set_concurrent_stages(int32_t ways);
int32_t rp_op_concurrent_stages(void);
int32_t rp_op_plane_conv_kernel(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co);
/* Weight gradient of that conv: gw[3][3][ci][co] = scale sum_p in[p+tap][ci] gout[p][co],
 * gb[co] = scale sum_p gout[p][co] (gb may be NULL).  Deterministic. */
int rp_op_conv3x3_wgrad(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const float* in, const float* gout,
                        double scale, float* gw, float* gb, int32_t math, void* ws, int64_t ws_bytes, void* stream);
int64_t rp_op_conv3x3_wgrad_workspace_bytes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co);

/* Planes of an fp32 tensor (n % 4 == 0): p1 non-NULL: the fp16 pair of v 2^7 (scale_out NULL) or of
 * v s with s computed from max |v| and stored in *scale_out (a rp_op_plane_scale_bytes()
 * buffer); p1 NULL: p0 alone is the bf16 single plane. */
int rp_op_split_planes(const float* in, int64_t n, void* p0, void* p1, float* scale_out, void* stream);
/* Weight gradient from fp16 plane pairs (x 2^7 = x0 + x1, gout g_s = g0 + g1 with g_scale the
 * device scale, NULL = 2^7), Ci and Co multiples of 64, or Ci 16 and Co in {16, 32}: the
 * fp32-accurate tcgen05 wgrad fed by TMA alone. */
int rp_op_conv3x3_wgrad_planes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const void* x0, const void* x1,
                               const void* g0, const void* g1, double scale, const float* g_scale, float* gw,
                               float* gb, void* ws, int64_t ws_bytes, void* stream);
int64_t rp_op_conv3x3_wgrad_planes_workspace_bytes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co);

/* Residual block on nrows samples (network.cpp:82-106), block params at `pb` in the
 * flat layout (w1 b1 w2 b2).  Forward writes a (tape) and x_next.  Backward takes the
 * cotangent at the block output in g_io and overwrites it with the cotangent at the
 * block input; writes the block's gradients at `gb` (same layout as pb); dpre is
 * caller scratch of the hidden activation size. */
int rp_op_block_fwd(const rp_geometry* g, int32_t nrows, const float* x, const float* pb, float* a,
                    float* x_next, int32_t math, void* ws, int64_t ws_bytes, void* stream);
int rp_op_block_bwd(const rp_geometry* g, int32_t nrows, const float* x, const float* a, const float* pb,
                    float* g_io, float* dpre, float* gb, int32_t math, void* ws, int64_t ws_bytes,
                    void* stream);
/* Plane-pair block path (RP_MATH_FP32 only): every conv reads its input as an fp16 plane
 * pair (each a [2][elements] fp16 buffer: p0 then p1) and writes the plane pair of its
 * output (a, x_next, dpre, the updated cotangent) next to the fp32 tensor; both weight
 * gradients run on rp_op_conv3x3_wgrad_planes.  fp32-class accuracy (22-bit operands,
 * fp32 accumulation).  x_next_planes may be NULL (a stage's last block).  Backward reads
 * g_planes as the planes of g_io g_scale on entry (g_scale: the device scale written by
 * rp_op_synthetic_grad_planes / rp_op_head_loss_bwd_planes / rp_op_split_planes) and
 * leaves the planes of the new g_io (same scale) there. */
int32_t rp_op_block_planes_supported(const rp_geometry* g, int32_t nrows, int32_t math);
int rp_op_block_fwd_planes(const rp_geometry* g, int32_t nrows, const float* x, const void* x_planes,
                           const float* pb, float* a, float* x_next, void* a_planes, void* x_next_planes,
                           const void* filters, void* ws, int64_t ws_bytes, void* stream);
int rp_op_block_bwd_planes(const rp_geometry* g, int32_t nrows, const void* x_planes, const float* a,
                           const void* a_planes, const float* pb, float* g_io, void* g_planes, const float* g_scale,
                           float* dpre, void* dpre_planes, float* gb, const void* filters, void* ws,
                           int64_t ws_bytes, void* stream);
/* The plane path's tcgen05 filter operands for nblocks consecutive blocks (pb = the first
 * block's parameters) in one launch: dgrad = 0 the forward filters (W1, W2), 1 the
 * input-gradient filters (W2, W1 flipped and transposed), one pair per block, each pair
 * rp_op_planes_filters_bytes(g, 1) bytes.  Passing a block's pair as `filters` to the two ops
 * above skips their per-conv preparation (nullable: each conv then prepares its own).  The
 * pair reflects the parameters at preparation time. */
int64_t rp_op_planes_filters_bytes(const rp_geometry* g, int32_t nblocks);
/* The bf16 tape path (RP_MATH_BF16, C and hidden multiples of 128): every conv reads a bf16
 * copy of its input by TMA (the values the fp32-input bf16 conv rounds to), and the tape is
 * bf16 only.  Forward: x (fp32 residual stream) and x16 = bf16(x) in; a16 = bf16(a), d16 =
 * bf16(1 - a^2) (tanh only; NULL for identity), x_next (fp32) and x_next16 (may be NULL: the
 * stage's last block) out.  Backward: g_io (fp32, updated in place) and g16 = bf16(g_io) in,
 * g16 rewritten with the new cotangent, dpre16 scratch, gb the block's gradients. */
int32_t rp_op_block_bf16_tape_supported(const rp_geometry* g, int32_t nrows, int32_t math);
int rp_op_block_fwd_bf16t(const rp_geometry* g, int32_t nrows, const float* x, const void* x16, const float* pb,
                          void* a16, void* d16, float* x_next, void* x_next16, void* ws, int64_t ws_bytes,
                          void* stream);
int rp_op_block_bwd_bf16t(const rp_geometry* g, int32_t nrows, const void* x16, const void* a16, const void* d16,
                          const float* pb, float* g_io, void* g16, void* dpre16, float* gb, void* ws,
                          int64_t ws_bytes, void* stream);
/* Weight gradient from single bf16 copies (bf16 x bf16 products, fp32 accumulate), Ci and Co
 * multiples of 128. */
int rp_op_conv3x3_wgrad_bf16p(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co, const void* x16,
                              const void* g16, double scale, float* gw, float* gb, void* ws, int64_t ws_bytes,
                              void* stream);
int64_t rp_op_conv3x3_wgrad_bf16p_workspace_bytes(int32_t n, int32_t h, int32_t w, int32_t ci, int32_t co);
int rp_op_prep_planes_filters(const rp_geometry* g, const float* pb, int32_t nblocks, int32_t dgrad, void* out,
                              void* stream);
/* Device workspace the block/stem/head ops need for nrows samples (weight relayouts,
 * deterministic split-K partials). */
int64_t rp_op_workspace_bytes(const rp_geometry* g, int32_t nrows, int32_t math);
/* Stem S (affine_forward, network.cpp:108-110 as a 3x3 conv Cin->C). */
int rp_op_stem_fwd(const rp_geometry* g, int32_t nrows, const float* x_raw, const float* ps, float* x0,
                   int32_t math, void* ws, int64_t ws_bytes, void* stream);
/* The stem forward writing, in the same pass, the planes of x0 that rp_op_split_planes makes
 * without a scale argument (p1 non-NULL: the fp16 pair of x0 2^7; NULL: the bf16 single
 * plane): the first block's tape input. */
int rp_op_stem_fwd_planes(const rp_geometry* g, int32_t nrows, const float* x_raw, const float* ps, float* x0,
                          void* p0, void* p1, void* stream);
int rp_op_stem_bwd(const rp_geometry* g, int32_t nrows, const float* x_raw, const float* g0, float* gs,
                   void* ws, int64_t ws_bytes, void* stream);
/* Head T forward (affine_forward, network.cpp:108-110, as GAP + affine): pooled [nrows, C]
 * and logits [nrows, classes] (device, caller-owned). */
int rp_op_head_fwd(const rp_geometry* g, int32_t nrows, const float* x_end, const float* pt, float* pooled,
                   float* logits, void* stream);
/* loss_phi (network.cpp:193-221) + T backward: mean softmax-CE into *loss_dev (device
 * double), T grads at gt (t.w then t.b), cotangent at the trunk output into g_out (NHWC).
 * Labels are device int32 (out-of-range labels give a NaN loss). */
int rp_op_head_loss_bwd(const rp_geometry* g, int32_t nrows, const float* pooled, const float* logits,
                        const float* pt, const int32_t* labels, double* loss_dev, float* gt, float* g_out,
                        void* ws, int64_t ws_bytes, void* stream);
/* rp_op_head_loss_bwd also writing the cotangent's planes (as rp_op_split_planes makes them:
 * p1 non-NULL the scaled fp16 pair with its scale in *scale, NULL the bf16 single plane): the
 * last stage's first backward conv input. */
int rp_op_head_loss_bwd_planes(const rp_geometry* g, int32_t nrows, const float* pooled, const float* logits,
                               const float* pt, const int32_t* labels, double* loss_dev, float* gt, float* g_out,
                               void* p0, void* p1, float* scale, void* ws, int64_t ws_bytes, void* stream);
/* Argmax hits (accuracy, network.cpp:223-234; ties -> lowest class); *hits host. */
/* loss_phi's value and accuracy of device logits [nrows, classes] (network.cpp:193-234), both
 * reduced on device in a fixed order: *loss (host) = mean softmax-CE (fp64), *hits (host) =
 * argmax hits (ties to the lowest class); pred (device, nullable) = per-row argmax. */
int64_t rp_op_eval_workspace_bytes(int32_t nrows);
int rp_op_eval_loss_accuracy(const float* logits, const int32_t* labels, int32_t nrows, int32_t classes,
                             double* loss, int64_t* hits, int32_t* pred, void* ws, int64_t ws_bytes, void* stream);
int rp_op_argmax_hits(const float* logits, const int32_t* labels, int32_t nrows, int32_t classes,
                      int64_t* hits, void* ws, void* stream);

/* ---- DecoupledTrainer handle (decoupled.hpp:56-120) ------------------------ */
typedef struct rp_trainer rp_trainer;

/* DecoupledTrainer(ResidualNet net, int stages, TrainMode, PenaltyKind, int num_samples)
 * (decoupled.hpp:58-59).  params_host: flat fp32 parameters (NULL: Glorot init from
 * *seed_state on device).  devices/ndev: stage k runs on devices[floor(k*ndev/K)]
 * (NULL/0 == the current device). mode RP_MODE_SERIAL builds a K=1 serial trainer. */
int rp_trainer_create(const rp_geometry* g, int32_t stages, int32_t mode, int32_t penalty,
                      int32_t num_samples, const float* params_host, uint64_t* seed_state,
                      int32_t math, const int32_t* devices, int32_t ndev, rp_trainer** out);
int rp_trainer_destroy(rp_trainer* t);

/* ---- stage-sharded trainer (one process per GPU) -----------------
 * Holds stages [stage_lo, stage_hi) of the K-stage net on `device`, plus -- when
 * stage_hi < K -- a ghost of stage stage_hi (lambda, kappa, received p) because the
 * holder of stage k-1 corrects boundary k.  One iteration on rank r
 * (paper_2009_01462_b200/distributed.py):
 *   rp_trainer_step_local            parallel phase + inner-boundary corrections
 *   send p_{stage_lo} to rank r-1 || receive p_{stage_hi} into the ghost's adjoint
 *   rp_trainer_correct_ghost         correct_aux / correct_multiplier of boundary stage_hi
 *   send the ghost's lambda to rank r+1 || receive lambda_{stage_lo} from rank r-1
 * The exchanges are NCCL point-to-point on rp_trainer_stage_stream(k) streams; no
 * collective touches the data path (the parameters are disjoint per stage).
 * Replaces the in-process StagePool (runtime.hpp:33-67) for multi-GPU runs. */
int rp_trainer_create_local(const rp_geometry* g, int32_t stages, int32_t mode, int32_t penalty, int32_t num_samples,
                            const float* params_host, uint64_t* seed_state, int32_t math, int32_t device,
                            int32_t stage_lo, int32_t stage_hi, rp_trainer** out);
int rp_trainer_local_range(rp_trainer* t, int32_t* stage_lo, int32_t* stage_hi);
/* reset_lambda_from_forward over the local stages: x_dev = raw inputs of all samples
 * (stage_lo == 0) or NULL (stage_lo's lambda already holds the upstream boundary). */
int rp_trainer_reset_local(rp_trainer* t, const float* x_dev);
int rp_trainer_step_local(rp_trainer* t, const float* x_dev, const int32_t* labels_dev, int32_t nrows, int32_t row0,
                          const rp_step_params* p);
int rp_trainer_correct_ghost(rp_trainer* t, const rp_step_params* p, int32_t row0, int32_t nrows);
/* device pointer of a state buffer ([num_samples][H W C] fp32) of a local or ghost stage;
 * which: RP_STATE_LAMBDA 0, KAPPA 1, BOUNDARY_OUT 2, BOUNDARY_ADJOINT 3 */
int rp_trainer_state_device(rp_trainer* t, int32_t k, int32_t which, float** ptr);
int rp_trainer_stage_stream(rp_trainer* t, int32_t k, void** stream);
int rp_trainer_loss_device(rp_trainer* t, double** ptr);
/* Evaluation forward of the local stages (decoupled.cpp:332-347 split across ranks): in =
 * raw inputs (stage_lo == 0) or the upstream boundary features [nrows][H W C]; out = the
 * features after stage_hi - 1, or logits [nrows][classes] when the last stage is local. */
int rp_trainer_forward_local(rp_trainer* t, const float* in_dev, int32_t nrows, float* out_dev);
int rp_trainer_set_kappa_rule(rp_trainer* t, int32_t rule);
/* CUDA graphs for step / step_device (on != 0): the iteration is captured once per
 * (inputs, rows, StepParams, multiplier state) and replayed; single-pass corrections
 * (tau < 0 or max_corrections == 1) only, others run eagerly.  Off by default. */
int rp_trainer_set_graphs(rp_trainer* t, int32_t on);
int rp_trainer_get_params(rp_trainer* t, float* host);
int rp_trainer_set_params(rp_trainer* t, const float* host);
/* Gradients of the last stage_backward_update / step (flat layout, host). */
int rp_trainer_get_grads(rp_trainer* t, float* host);
/* reset_lambda_from_forward (decoupled.cpp:44-63); x is host NHWC [num_samples,H,W,Cin]. */
int rp_trainer_reset_lambda_from_forward(rp_trainer* t, const float* x_host);
/* step (decoupled.cpp:172-194).  Host buffers (H2D inside) ... */
int rp_trainer_step(rp_trainer* t, const float* x_host, const int32_t* labels_host, int32_t nrows,
                    int32_t row0, const rp_step_params* p, double* loss_out);
/* ... or device buffers already resident (loss_out NULL: no host sync; the loss stays
 * on device and rp_trainer_last_loss() reads it). */
int rp_trainer_step_device(rp_trainer* t, const float* x_dev, const int32_t* labels_dev, int32_t nrows,
                           int32_t row0, const rp_step_params* p, double* loss_out);
int rp_trainer_last_loss(rp_trainer* t, double* loss_out);
/* The pieces of step (decoupled.hpp:71-89).  Host buffers. */
int rp_trainer_take_snapshot(rp_trainer* t, int32_t k, int32_t row0, int32_t nrows);
int rp_trainer_stage_forward(rp_trainer* t, int32_t k, const float* x_host, int32_t nrows, int32_t row0);
int rp_trainer_stage_backward_update(rp_trainer* t, int32_t k, const int32_t* labels_host, int32_t nrows,
                                     double beta, double lr, int32_t row0);
int rp_trainer_correct_aux(rp_trainer* t, int32_t k, const rp_step_params* p, int32_t row0, int32_t nrows);
int rp_trainer_correct_multiplier(rp_trainer* t, int32_t k, double beta, double kappa_lr, int32_t row0,
                                  int32_t nrows);
int rp_trainer_correction_gradient(rp_trainer* t, int32_t k, double beta, int32_t row0, int32_t nrows,
                                   float* out_host);
/* violation_report (decoupled.cpp:196-205): per_stage[K] host. */
int rp_trainer_violation_report(rp_trainer* t, double* per_stage, double* max_violation,
                                int64_t* normalizer);
/* Per-stage state (decoupled.hpp:29-32): which 0 lambda, 1 kappa, 2 boundary_out, 3 boundary_adjoint. */
int rp_trainer_get_state(rp_trainer* t, int32_t k, int32_t which, float* host);
int rp_trainer_set_state(rp_trainer* t, int32_t k, int32_t which, const float* host);
/* Full serial forward (eval, decoupled.cpp:332-347): logits host [n, classes]. */
int rp_trainer_forward(rp_trainer* t, const float* x_host, int32_t nrows, float* logits_host);
/* Evaluation on device (decoupled.cpp:332-347: the full serial forward, then loss_phi and
 * accuracy, network.cpp:193-234): *loss = mean softmax-CE, *accuracy = argmax hits / nrows
 * (ties to the lowest class).  Labels are validated (std::invalid_argument). */
int rp_trainer_evaluate(rp_trainer* t, const float* x_host, const int32_t* labels_host, int32_t nrows,
                        double* loss, double* accuracy);
int64_t rp_trainer_iteration(rp_trainer* t);
int32_t rp_trainer_stages(rp_trainer* t);
/* Device-side timing of the last step: max over stage streams (ms). */
int rp_trainer_last_step_ms(rp_trainer* t, float* ms);
/* Device-timed region on the trainer's control stream: which = 0 begins (records an
 * event after all previously issued work), which = 1 ends and returns the elapsed ms. */
int rp_trainer_region(rp_trainer* t, int32_t which, float* ms);

/* serial_train_step (network.cpp:236-244) on a K=1 trainer made with RP_MODE_SERIAL. */
int rp_serial_train_step(rp_trainer* t, const float* x_host, const int32_t* labels_host, int32_t nrows,
                         double lr, double* loss_out);

/* ---- stage pipeline over NCCL (StagePool replacement across processes, runtime.hpp:33-67) --
 * One process per B200: each holds the stage-sharded trainers (rp_trainer_create_local) of
 * its stages and a pipeline that runs DecoupledTrainer::step (decoupled.cpp:172-194) with the
 * neighbour exchange -- p_k upstream, the corrected lambda_k downstream -- as NCCL point-to-point
 * transfers on dedicated streams, in `chunks` row chunks, overlapped with the corrections
 * (host/pipeline.hpp).  Two communicators over the same ranks (one per direction); peers are
 * ranks in them (-1: none).  NCCL is opened at run time (dlopen; RP_NCCL_LIBRARY overrides).
 * A rank may list several consecutive trainers (the single-process loopback: peers = own rank). */
typedef struct rp_comm rp_comm;
typedef struct rp_pipeline rp_pipeline;
int rp_comm_unique_id(uint8_t* id128);
int rp_comm_create(const uint8_t* id128, int32_t nranks, int32_t rank, int32_t device, rp_comm** out);
int rp_comm_destroy(rp_comm* c);
int rp_pipeline_create(rp_comm* comm_a, rp_comm* comm_b, rp_trainer* const* trainers, const int32_t* prev_peer,
                       const int32_t* next_peer, int32_t ntrainers, int32_t chunks, rp_pipeline** out);
/* reset_lambda_from_forward (decoupled.cpp:44-63) as a chained forward; x_full: device raw
 * inputs of all num_samples rows (read on the rank holding stage 0). */
int rp_pipeline_reset_lambda_from_forward(rp_pipeline* p, const float* x_full_dev);
/* One iteration on device buffers; loss_out (nullable) only on the rank holding stage K-1. */
int rp_pipeline_step(rp_pipeline* p, const float* x_dev, const int32_t* labels_dev, int32_t nrows, int32_t row0,
                     const rp_step_params* sp, double* loss_out);
int rp_pipeline_loss(rp_pipeline* p, double* loss_out);
/* Capture the step (kernels, events, NCCL calls) in a CUDA graph and replay it. */
int rp_pipeline_set_graphs(rp_pipeline* p, int32_t on);
/* which 0: start a device-timed region; 1: end it, *ms = elapsed (every stream joined). */
int rp_pipeline_region(rp_pipeline* p, int32_t which, float* ms);
int rp_pipeline_sync(rp_pipeline* p);
int rp_pipeline_destroy(rp_pipeline* p);

#ifdef __cplusplus
}
#endif

#endif /* RESPAR_B200_H */
