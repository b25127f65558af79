/*
 * ckb200.h — C ABI of the B200 (sm_100a) engine for the online-BP CNN hot
 * path of arXiv 1102.0183 (reference package `convkit`).
 *
 * Two seams are exported, both plain C (pointers + sizes, no torch types):
 *
 *  1. Operator seam — one entry per compute kernel the reference engine
 *     resolves at call time through `convkit.kernels` (network.py:182,189,
 *     238,243,247,257).  Same argument meaning as the numba kernels, with the
 *     numpy array shapes spelled out as (maps, rows, pitch) and all buffers
 *     DEVICE pointers owned by the caller.
 *
 *  2. Network seam — a device-resident net replacing `NetworkState`
 *     (network.py:81-304) and the per-image loops of `training.train_epoch` /
 *     `training.evaluate` (training.py:126-156): one persistent kernel runs
 *     forward -> loss -> backward -> update for every image of an epoch.
 *
 * Every function returns CK_OK (0) or a negative CK_E_* status; the message
 * of the last failure on the calling thread is ck_last_error().  The Python
 * layer maps the codes onto the reference's exception classes (errors.py).
 * Functions on one ck_net are not re-entrant; different nets are independent.
 */
#ifndef CKB200_H
#define CKB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CK_OK 0
#define CK_E_DIMENSION (-1) /* DimensionError */
#define CK_E_GEOMETRY (-2)  /* GeometryError  */
#define CK_E_CONFIG (-3)    /* ConfigError    */
#define CK_E_STATE (-4)     /* StateError     */
#define CK_E_PRECISION (-5) /* PrecisionError */
#define CK_E_CUDA (-6)      /* CUDA runtime failure */
#define CK_E_NOMEM (-7)     /* device allocation failed */

typedef void* ck_stream_t; /* a cudaStream_t; NULL = legacy default stream */

const char* ck_last_error(void);
int ck_abi_version(void);
int ck_kernel_launches(int64_t* count); /* kernels launched by this library so far */

/* ------------------------------------------------------------------------
 * 1. Operator seam (convkit.kernels, kernels.py:70-180).
 *    Map stacks are (maps, rows, pitch) float32 with map stride rows*pitch;
 *    tables are the reference's int64 CSR arrays (topology.py:102-116).
 * ---------------------------------------------------------------------- */

/* kernels.conv_fwd (kernels.py:70-87): a = bias + sum_k sum_v sum_u w*src in
 * f32, sequential bias->k->v->u order without FMA; y = f32(1.7159*tanh_f64(
 * 0.6666*a)). */
int ck_conv_fwd(const float* src, int n_src, int src_rows, int src_pitch,
                const float* arena, const int64_t* fwd_offsets,
                const int64_t* fwd_srcs, const int64_t* fwd_widx,
                const int64_t* bias_off, int kx, int ky, int sx, int sy,
                float* a_out, float* y_out, int n_dest, int out_rows,
                int out_pitch, int out_w, int out_h, ck_stream_t stream);

/* kernels.pull_bwd (kernels.py:90-121): gather deltas into every source cell
 * (f64 accumulation of f32 products, one rounding). */
int ck_pull_bwd(const float* delta_next, int n_dest, int dest_rows,
                int dest_pitch, int dest_w, int dest_h, const float* arena,
                const int64_t* bwd_offsets, const int64_t* bwd_dests,
                const int64_t* bwd_widx, int kx, int ky, int sx, int sy,
                float* out, int n_src, int out_rows, int out_pitch, int src_w,
                int src_h, ck_stream_t stream);

/* kernels.weight_grad (kernels.py:124-141). */
int ck_weight_grad(const float* delta_next, int n_dest, int dest_rows,
                   int dest_pitch, int dest_w, int dest_h, const float* y_prev,
                   int n_src, int src_rows, int src_pitch,
                   const int64_t* pair_dest, const int64_t* pair_src,
                   const int64_t* pair_off, int n_pairs, int kx, int ky,
                   int sx, int sy, float* g_arena, ck_stream_t stream);

/* kernels.bias_grad (kernels.py:144-151). */
int ck_bias_grad(const float* delta_next, int n_dest, int dest_rows,
                 int dest_pitch, int dest_w, int dest_h,
                 const int64_t* bias_off, float* g_arena, ck_stream_t stream);

/* kernels.maxpool_fwd (kernels.py:154-172): strict '>' so ties keep the first
 * cell in row-major scan; arg_r/arg_c are (maps, out_h, out_w) int64. */
int ck_maxpool_fwd(const float* src, int n_maps, int src_rows, int src_pitch,
                   int px, int py, float* out, int out_rows, int out_pitch,
                   int out_w, int out_h, int64_t* arg_r, int64_t* arg_c,
                   ck_stream_t stream);

/* kernels.maxpool_bwd (kernels.py:175-180): delta_prev[m,arg_r,arg_c] +=
 * delta_next[m,r,c] (caller zeroes delta_prev, network.py:256). */
int ck_maxpool_bwd(const float* delta_next, int n_maps, int next_rows,
                   int next_pitch, int out_w, int out_h, const int64_t* arg_r,
                   const int64_t* arg_c, float* delta_prev, int prev_rows,
                   int prev_pitch, ck_stream_t stream);

/* Fixed contrast layer (filters.py:153-175): out map f*C+c = correlate(
 * channel c, filter f) with replicated border, f64 accumulate, one rounding.
 * coeffs holds n_filters (fh, fw) blocks back to back (all the same size). */
int ck_contrast(const float* src, int n_ch, int rows, int pitch, int w, int h,
                const double* coeffs, int n_filters, int fh, int fw,
                float* out, int out_rows, int out_pitch, ck_stream_t stream);

/* FC-side operators.  The reference computes these inline with numpy
 * (not through convkit.kernels); they are exported so a caller can run every
 * layer of NetworkState.forward/backward/apply_gradients on the device.
 * Same arithmetic as the fused engine, so results equal its bits. */

/* network.py:193-199: a = x @ W + b (W is (n_in, n_out) row-major; f64
 * accumulation, rounded once, then + b in f32), y = 1.7159*tanh(0.6666*a)
 * in the NEP-50 f32 chain of layers.py:23-25.  a_out may be NULL. */
int ck_fc_fwd(const float* x, int n_in, const float* weights, const float* bias, int n_out,
              float* a_out, float* y_out, ck_stream_t stream);

/* network.py:214-218 + 268-273: xgrad = W @ delta from the weights BEFORE
 * the update (f64, rounded once; NULL to skip), grad_w = outer(x, delta),
 * grad_b = delta (each NULL to skip), and for eta > 0 the in-place SGD step
 * W -= f32(eta*grad_w), b -= f32(eta*grad_b).  eta == 0: no update;
 * eta < 0: CK_E_CONFIG (network.py:266-267). */
int ck_fc_bwd_update(const float* x, int n_in, float* weights, float* bias, int n_out,
                     const float* delta, float* xgrad, float* grad_w, float* grad_b,
                     double eta, ck_stream_t stream);

/* layers.py:28-30 applied as network.py:219/226/251-252 do:
 * delta *= activation_deriv(a) over the logical (w, h) cells of a pitched
 * (maps, rows, pitch) stack; an FC vector is (1, 1, n) with w = n, h = 1. */
int ck_act_deriv_mul(const float* a, float* delta, int n_maps, int rows, int pitch, int w,
                     int h, ck_stream_t stream);

/* network.py:268-273: params -= f32(eta * grads) element-wise (conv arenas
 * and FC weights alike).  eta <= 0: CK_E_CONFIG. */
int ck_sgd_update(float* params, const float* grads, int64_t n, double eta,
                  ck_stream_t stream);

/* backprop.py:22-39: delta_j = f32((y_j - t_j) * f'(a_j)) in f64 and
 * *loss = 0.5 * sum (y - t)^2 (numpy pairwise order).  targets are f64
 * (training.targets_for); scratch holds n doubles; loss may be NULL. */
int ck_output_deltas(const float* y, const float* a, const double* targets, int n,
                     float* delta, double* loss, double* scratch, ck_stream_t stream);

/* ------------------------------------------------------------------------
 * 2. Network seam (NetworkState, network.py:81-304; training.py:126-199).
 * ---------------------------------------------------------------------- */

enum {
  CK_LAYER_INPUT = 0,
  CK_LAYER_IMGPROC = 1,
  CK_LAYER_CONV = 2,
  CK_LAYER_POOL = 3,
  CK_LAYER_FC = 4
};

/* One resolved layer (arch.py resolve_geometry + topology.ConnectionTable).
 * All pointers are HOST pointers read during ck_net_create only. */
typedef struct ck_layer_desc {
  int32_t kind;
  int32_t maps, width, height; /* output geometry; FC: maps = neurons, 1x1 */
  int32_t kx, ky, sx, sy;      /* conv kernel and skipping factors */
  int32_t px, py;              /* pool region */
  int32_t n_pairs;             /* conv: connected (dest, src) pairs */
  int32_t arena_size;          /* conv: n_pairs*kx*ky + maps */
  const int64_t* fwd_offsets;  /* conv: maps+1 */
  const int64_t* fwd_srcs;     /* conv: n_pairs, sorted per dest */
  const int64_t* fwd_widx;     /* conv: n_pairs arena offsets */
  const int64_t* bias_offset;  /* conv: maps */
  int32_t n_filters;           /* imgproc: expanded filter count */
  int32_t filter_h, filter_w;  /* imgproc: common size of every filter */
  const double* filter_coeffs; /* imgproc: n_filters*fh*fw row-major */
} ck_layer_desc;

typedef struct ck_net ck_net;

/* Execution team used by the persistent training kernel:
 * CK_TEAM_CLUSTER = one thread-block cluster per net (hardware cluster
 * barrier, up to 16 CTAs); CK_TEAM_GRID = one cooperative grid per net;
 * CK_TEAM_AUTO (default) = a grid team of one CTA per SM, the SMs split
 * evenly between the nets of one launch.  Results do not depend on the team. */
enum { CK_TEAM_AUTO = 0, CK_TEAM_CLUSTER = 1, CK_TEAM_GRID = 2 };

int ck_net_create(const ck_layer_desc* layers, int n_layers, int device,
                  ck_net** out);
int ck_net_destroy(ck_net* net);
int ck_net_set_team(ck_net* net, int kind, int ctas, int threads);
int ck_net_get_team(const ck_net* net, int* kind, int* ctas, int* threads);
int ck_net_num_params(const ck_net* net, int64_t* n);
/* Whole parameter vector in NetworkState.parameters() order (conv arenas,
 * FC weights (n_in, n_out) row-major, FC bias). */
int ck_net_set_params(ck_net* net, const float* host, int64_t n);
int ck_net_get_params(ck_net* net, float* host, int64_t n);

/* Per-sample calls with HOST buffers (synchronous). x is (C, H, W) dense f32,
 * targets n_classes f64.  forward writes the output activations.  These (and
 * set/get_params, read_buffer) first wait for the whole device, so they are
 * ordered after any asynchronous work a caller enqueued on its own streams
 * (ck_net_train_epoch / ck_net_eval / ck_committee_train_epoch). */
int ck_net_forward(ck_net* net, const float* x, float* y_out);
int ck_net_backward(ck_net* net, const double* targets); /* fills grads */
int ck_net_apply_gradients(ck_net* net, double eta);     /* w -= f32(eta)*g */
int ck_net_train_step(ck_net* net, const float* x, const double* targets,
                      double eta, double* loss);

/* Inspection of a layer's buffers after the last call (dense, unpitched):
 * which = CK_BUF_A | CK_BUF_Y | CK_BUF_DELTA (float32), CK_BUF_ARG (int32
 * index of the winner in the whole source layer, m*src_h*src_w + r*src_w + c),
 * CK_BUF_GRAD (float32 arena / FC W then b). */
enum { CK_BUF_A = 0, CK_BUF_Y = 1, CK_BUF_DELTA = 2, CK_BUF_ARG = 3, CK_BUF_GRAD = 4 };
int ck_net_buffer_size(const ck_net* net, int layer, int which, int64_t* count);
int ck_net_read_buffer(ck_net* net, int layer, int which, void* host, int64_t count);

/* Device-resident online epoch (training.train_epoch, training.py:126-146):
 * images (n_total, C, H, W) uint8 on the device, lut[256] = f32(b/127.5-1)
 * (lut NULL: images points at float32 (n_total, C, H, W) inputs instead),
 * labels int32, order int32 (the visit order, length n).  Targets are +-1
 * one-hot in f64.  mean_loss (host) = sum(loss_i)/n in visit order.
 * losses (device, nullable) receives each image's loss. */
int ck_net_train_epoch(ck_net* net, const uint8_t* images, const float* lut,
                       const int32_t* labels, const int32_t* order, int64_t n,
                       double eta, double* losses, double* mean_loss,
                       ck_stream_t stream);

/* Several independent nets (a committee, training.run_experiment) trained
 * concurrently in ONE launch, one team per net, sharing images and order. */
int ck_committee_train_epoch(ck_net* const* nets, int n_nets,
                             const uint8_t* images, const float* lut,
                             const int32_t* labels, const int32_t* order,
                             int64_t n, double eta, double* mean_losses,
                             ck_stream_t stream);

/* Batched evaluation (training.evaluate / NetworkState.predict): predicted
 * class (first maximum) for images[first .. first+n) into pred (device int32);
 * outputs (device, nullable) receives the n_classes activations per image. */
int ck_net_eval(ck_net* net, const uint8_t* images, const float* lut,
                int64_t first, int64_t n, int32_t* pred, float* outputs,
                ck_stream_t stream);

/* Instrumented PROG_TRAIN run over n images (%globaltimer ns, averaged):
 * phase_ns[p] = the slowest CTA's work in phase p (previous barrier exit to
 * its last warp done), phase_ns[n_phases + p] = the barrier after it (slowest
 * work end to barrier exit).  max_phases must be >= 2 * n_phases. */
int ck_net_profile_epoch(ck_net* net, const uint8_t* images, const float* lut,
                         const int32_t* labels, const int32_t* order, int64_t n,
                         double eta, int64_t* phase_ns, int max_phases,
                         int* n_phases);

/* Human-readable phase program (0 train, 1 forward, 2 backward, 3 apply,
 * 4 eval) for diagnostics and DESIGN.md. */
int ck_net_describe_program(const ck_net* net, int prog, char* buf, int cap);

/* Specialised training kernels.  Nets whose geometry equals one compiled
 * into the library (the BASELINE configs, generated from
 * paper_1102_0183_b200/configs.py) train with a kernel in which every size,
 * offset and op choice is a compile-time constant; results are bit-identical
 * to the generic kernel.  ck_net_spec_source prints the C++ spec of a net
 * (host only, used by the build); ck_net_set_specialized(net, 0) forces the
 * generic kernel; ck_net_kernel_info names the kernel a training launch uses
 * ("specialised:<name>" or "generic"). */
int ck_net_spec_source(const ck_layer_desc* layers, int n_layers, const char* name, char* buf,
                       int64_t cap, int64_t* len);
int ck_net_set_specialized(ck_net* net, int enable);
int ck_net_kernel_info(const ck_net* net, char* buf, int cap);

/* Development aid: arm per-phase sub-timers of the training kernel.  Thread
 * 0 of team rank `rank` writes %globaltimer at numbered points into
 * dev_buf[phase * 32 + point] (>= 32 * n_phases int64, device); NULL disarms. */
int ck_debug_subprof(long long* dev_buf, int rank);


/* ------------------------------------------------------------------------
 * 3. On-line deformation (convkit.augment, augment.py:63-170), used by
 *    training.train_epoch when the config's deformation is enabled
 *    (training.py:140-144).  Field meaning as augment.DeformationConfig /
 *    DeformationParams; sigma is the config's (one per call).
 * ---------------------------------------------------------------------- */
typedef struct ck_deform_cfg {
  double translate_max, rotate_max, scale_max, shear_max; /* fraction, deg, fraction, deg */
  double elastic_sigma, elastic_alpha_max;                /* px */
} ck_deform_cfg;

typedef struct ck_deform_params {
  double translate_x, translate_y; /* fraction of width / height */
  double rotate;                   /* degrees, counterclockwise */
  double scale_x, scale_y;
  double shear_h;                  /* degrees */
  double elastic_alpha;            /* px */
  uint32_t seed;                   /* elastic field seed */
  uint32_t pad;
} ck_deform_params;

/* Deform every image i < n of images (n, C, H, W) (uint8 + lut, or float32
 * when lut is NULL) with augment.sample_params(cfg, [seed, epoch, i]) drawn on
 * the device (numpy SeedSequence + PCG64, bit-exact) into out (n, C, H, W)
 * float32 (device).  gauss_w: the 2*radius+1 normalised Gaussian taps of
 * scipy's _gaussian_kernel1d(elastic_sigma, 0, int(3*sigma+0.5)) (device
 * f64).  params_out (device, nullable) receives the drawn parameters. */
int ck_deform_epoch(const uint8_t* images, const float* lut, int channels, int height,
                    int width, int64_t n, const ck_deform_cfg* cfg, const double* gauss_w,
                    int radius, uint64_t seed, uint64_t epoch, ck_deform_params* params_out,
                    float* out, ck_stream_t stream);

/* augment.deform_channels (augment.py:150-170) with explicit per-image
 * parameters (device array of n). */
int ck_deform_apply(const uint8_t* images, const float* lut, int channels, int height,
                    int width, int64_t n, const ck_deform_params* params,
                    const double* gauss_w, int radius, float* out, ck_stream_t stream);

/* ------------------------------------------------------------------------
 * 4. Tensor-core batched evaluation (training.evaluate / predict at
 *    throughput, within a stated tolerance — NOT bit-exact; ck_net_eval is
 *    the bit-exact path).  Every conv / contrast / FC layer is an implicit
 *    GEMM on tcgen05 (fp16 operands, f32 accumulation in TMEM); passes = 3
 *    splits operands into fp16 hi+lo (Ah*Bh + Ah*Bl + Al*Bh, ~f32 accurate),
 *    passes = 1 is plain fp16.  The plan is built from the same layer
 *    descriptions as ck_net_create and owns activation buffers for
 *    max_batch images; ck_tc_set_params converts a parameter vector in
 *    NetworkState.parameters() order (DEVICE pointer, e.g.
 *    ck_net_device_params) into its weight matrices.
 * ---------------------------------------------------------------------- */
typedef struct ck_tc_eval ck_tc_eval;
int ck_tc_create(const ck_layer_desc* layers, int n_layers, int device, int64_t max_batch,
                 int passes, ck_tc_eval** out);
int ck_tc_destroy(ck_tc_eval* plan);
int ck_tc_set_params(ck_tc_eval* plan, const float* params, ck_stream_t stream);
int ck_tc_eval_run(ck_tc_eval* plan, const uint8_t* images, const float* lut, int64_t first,
                   int64_t n, int32_t* pred, float* outputs, ck_stream_t stream);

/* ------------------------------------------------------------------------
 * Tensor-core training variant (opt-in, its own tolerance):
 * online training of input -> (conv, stride 1 -> maxpool)+ -> fc+ nets with
 * every conv forward, weight gradient and delta pull as a tcgen05 implicit
 * GEMM (fp16 hi/lo split, f32 accumulation), the reference's protocol
 * otherwise (network.py:163-282: one update per image, training.py:126-146
 * visit order).  `params` is the net's DEVICE parameter vector
 * (ck_net_device_params): the plan trains it in place, so the exact path and
 * this one share the weights.  Not bit-exact: see tests/test_gpu_tct.py. */
typedef struct ck_tct ck_tct;
int ck_tct_create(const ck_layer_desc* layers, int n_layers, int device, float* params,
                  ck_tct** out);
int ck_tct_destroy(ck_tct* plan);
int ck_tct_train_epoch(ck_tct* plan, const uint8_t* images, const float* lut,
                       const int32_t* labels, const int32_t* order, int64_t n, double eta,
                       double* mean_loss, ck_stream_t stream);
/* Device pointer of a net's parameter vector (valid until ck_net_destroy). */
int ck_net_device_params(const ck_net* net, const float** params);

#ifdef __cplusplus
}
#endif
#endif /* CKB200_H */
