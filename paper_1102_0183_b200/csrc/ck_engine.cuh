// ck_engine.cuh — device data model and phase ops of the network engine.
//
// A net lives entirely on the device:
//   params  f32, NetworkState.parameters() order (conv arenas with the
//           reference's tiling topology.py:82-96, FC W (n_in,n_out), FC b)
//   grads   f32, same layout (backward() / apply_gradients() split mode)
//   act     per layer y / a / delta (f32, dense (maps,h,w), no pitch) and pool
//           argmax (int32 index into the source layer), 128-byte aligned
//   tables  int32 copies of the ConnectionTable CSR arrays
//
// One online step is a PROGRAM: a list of phases, each a list of ops that may
// run concurrently; phases are separated by a team barrier.  A team is the
// set of CTAs working on one net (a thread-block cluster, a cooperative grid
// or a single CTA for batched evaluation).  Ops split their work over the
// team's CTAs / warps / threads; within a CTA they may stage data in shared
// memory (with __syncthreads), never across CTAs.
//
// Every reduction whose order is free (the reference accumulates it in f64)
// is split in a way that depends only on fixed constants (warp width, group
// sizes, FC slices), never on the launch shape, so results are identical for
// every team shape and between training and evaluation.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ck_numerics.cuh"

namespace ck {

constexpr int kMaxLayers = 24;
constexpr int kMaxOps = 80;
constexpr int kMaxPhases = 56;
constexpr int kFcSlices = 16;      // FC forward: i-slices combined in fixed order
constexpr int kPullLanes = 8;      // pull: lanes per source cell
constexpr int kFcTile = 8;         // FC forward: output columns per CTA tile
constexpr int kImgLanes = 8;       // contrast layer: lanes per response cell
constexpr int kStageMax = 4096;    // largest per-layer array every CTA copies

enum LayerKind { L_INPUT = 0, L_IMGPROC = 1, L_CONV = 2, L_POOL = 3, L_FC = 4 };

// Every field of a layer's geometry, in declaration order.  The geometry is
// plain integers (tables are offsets into one int32 table block), so a whole
// net can be a compile-time constant: the spec generator prints this list for
// the specialised kernels (ck_specs.cuh).
#define CK_LAYER_FIELDS(X)                                                   \
  X(int, kind) X(int, maps) X(int, h) X(int, w) X(int, cells)                \
  X(int, src_maps) X(int, src_h) X(int, src_w) X(int, src_cells)             \
  X(int, kx) X(int, ky) X(int, tx) X(int, ty) X(int, px) X(int, py)          \
  X(int, n_pairs) X(int, has_delta) X(int, n_filt) X(int, fh) X(int, fw)     \
  X(int, max_fan_in) X(int, pool_above)                                      \
  X(int, wg_split) X(int, pull_g) X(int, pull_ch) X(int, full)               \
  X(int, spitch) X(int, ypitch) X(int64_t, yp_off) X(int, pullg)             \
  X(int64_t, p_off) X(int64_t, b_off) X(int64_t, n_par)                      \
  X(int64_t, y_off) X(int64_t, a_off) X(int64_t, d_off) X(int64_t, arg_off)  \
  X(int64_t, wrc_off) X(int64_t, wd_off)                                     \
  X(int, o_fwd_off) X(int, o_fwd_src) X(int, o_fwd_widx) X(int, o_bias_off)  \
  X(int, o_bwd_off) X(int, o_bwd_dst) X(int, o_bwd_widx) X(int, o_pair_dst)  \
  X(int, o_filt)

// Field notes: tx = sx + 1 (conv stride); pool_above: the next layer is a
// max-pool (sparse backward); wg_split: weight-gradient winner chunks per
// pair; pull_g / pull_ch: pull lane groups / backward-list chunks; full:
// the conv table is the full table in ConnectionTable's order, so every table
// entry is arithmetic (no loads);
// *_off: act-arena offsets (elements); wrc_off / wd_off: a pool over a conv
// keeps winner (r<<16|c) and winner delta per pooled cell; o_*: offsets of
// the conv tables (int32, read-only for a launch, always read with __ldg)
// and of the contrast filter coefficients.
struct LayerDev {
#define CK_DECL(t, n) t n;
  CK_LAYER_FIELDS(CK_DECL)
#undef CK_DECL
};

// table access: TB(L, fwd_off) -> const int* into the table block
#define TB(L, f) (R.tables + (L).o_##f)



enum OpKind {
  OP_LOAD_INPUT = 0,  // input y <- lut[image bytes] (no-op for host-staged x)
  OP_IMGPROC,         // contrast layer
  OP_CONV_FWD,        // conv a, y (+ zero own delta with F_ZERO_SELF)
  OP_POOL_FWD,        // max-pool y + argmax
  OP_FC_FWD,          // a = x@W + b, y = act(a)
  OP_ZERO_DELTA,      // delta <- 0 (scatter target of the pool above)
  OP_OUT_DELTA,       // output deltas + sample loss
  OP_FC_BWD,          // xgrad, W/b update (or grads), delta below
  OP_CONV_BWD,        // weight/bias grads (+ update) and pulled delta below
  OP_UPDATE,          // params[p_off, +n_par) -= eta * grads
  OP_FC_OUT,          // output layer: forward + output deltas + loss + backward rows
  OP_CONV_POOL,       // conv a, y fused with the max-pool above it (y, argmax)
};

// F_POOLED_ONLY (evaluation): a conv+pool keeps only the pooled values; the
// pool picks the largest pre-activation and activates it once (the
// activation is monotone, so the pooled value is the same bit for bit).
enum OpFlags { F_UPDATE = 1, F_PULL = 2, F_ZERO_SELF = 4, F_FUSE_BELOW = 8, F_POOLED_ONLY = 16 };

struct Op {
  int16_t kind;
  int16_t layer;
  int16_t flags;
  int16_t pad;
};

struct Program {
  int n_phases;
  int begin[kMaxPhases + 1];
  Op ops[kMaxOps];
};

// Phase 0 of a program that only loads the input and runs the image-
// processing layer: skipped (barrier included) when the job carries that
// layer precomputed (Job::pre).
__host__ __device__ constexpr bool phase0_input_only(const struct Program& P);

enum ProgId { PROG_TRAIN = 0, PROG_FORWARD = 1, PROG_BACKWARD = 2, PROG_APPLY = 3,
              PROG_EVAL = 4, N_PROGS = 5 };

__host__ __device__ constexpr bool phase0_input_only(const Program& P) {
  return P.n_phases > 1 && P.begin[1] - P.begin[0] == 2 &&
         P.ops[P.begin[0]].kind == OP_LOAD_INPUT && P.ops[P.begin[0] + 1].kind == OP_IMGPROC;
}

// A net's geometry and phase programs: plain values (compile-time constants
// in the specialised kernels, a shared-memory copy in the generic ones).
struct NetGeo {
  int n_layers;
  int n_classes;
  int in_cells;
  int pad0;
  int64_t act_size;        // elements per act arena (one team)
  LayerDev L[kMaxLayers];
  Program prog[N_PROGS];
};

// A net's device memory.
struct NetPtr {
  float* params;
  float* grads;
  float* act;
  unsigned* bar;           // grid-team barrier counter
  const int* tables;       // int32 table block (LayerDev::o_*)
  const double* filt;      // contrast filter coefficients
};

// Table entries.  A full table (L.full) in ConnectionTable's order (dest
// major, sources ascending; arena per dest = its blocks then its bias,
// topology.py:82-116) is pure arithmetic; otherwise the entry is loaded.
__device__ __forceinline__ int t_fwd_off(const NetPtr& R, const LayerDev& L, int d) {
  return L.full ? d * L.src_maps : __ldg(TB(L, fwd_off) + d);
}
__device__ __forceinline__ int t_fwd_src(const NetPtr& R, const LayerDev& L, int p) {
  return L.full ? p % L.src_maps : __ldg(TB(L, fwd_src) + p);
}
__device__ __forceinline__ int t_fwd_widx(const NetPtr& R, const LayerDev& L, int p) {
  return L.full ? (p / L.src_maps) * (L.src_maps * L.kx * L.ky + 1) + (p % L.src_maps) * L.kx * L.ky
                : __ldg(TB(L, fwd_widx) + p);
}
__device__ __forceinline__ int t_bias_off(const NetPtr& R, const LayerDev& L, int d) {
  return L.full ? d * (L.src_maps * L.kx * L.ky + 1) + L.src_maps * L.kx * L.ky
                : __ldg(TB(L, bias_off) + d);
}
__device__ __forceinline__ int t_pair_dst(const NetPtr& R, const LayerDev& L, int p) {
  return L.full ? p / L.src_maps : __ldg(TB(L, pair_dst) + p);
}
__device__ __forceinline__ int t_bwd_off(const NetPtr& R, const LayerDev& L, int s) {
  return L.full ? s * L.maps : __ldg(TB(L, bwd_off) + s);
}
__device__ __forceinline__ int t_bwd_dst(const NetPtr& R, const LayerDev& L, int k) {
  return L.full ? k % L.maps : __ldg(TB(L, bwd_dst) + k);
}
__device__ __forceinline__ int t_bwd_widx(const NetPtr& R, const LayerDev& L, int k) {
  return L.full ? (k % L.maps) * (L.src_maps * L.kx * L.ky + 1) + (k / L.maps) * L.kx * L.ky
                : __ldg(TB(L, bwd_widx) + k);
}

// Per-launch job description (passed by value).
struct Job {
  int prog;
  int n_nets;
  const uint8_t* images;   // (N, R, C, H, W) bytes, or null for host-staged input
  const float* lut;        // null: `images` holds float32 (N, R, C, H, W)
  const int32_t* labels;
  const int32_t* order;    // visit order (null: first + t)
  const double* targets;   // explicit targets (n_classes) for single steps
  int64_t n;
  int64_t first;
  float eta_f;
  double* losses;          // per image, per net: losses[net * n + t] (nullable)
  double* loss_total;      // per net (device)
  int32_t* pred;           // eval
  float* outputs;          // eval (nullable)
  float* eval_scratch;     // eval: per-CTA act arenas
  int eval_floats;         // eval: shared-memory staging per CTA (floats)
  long long* prof;         // phase end times (globaltimer ns), nullable
  int64_t prof_images;     // images profiled
  long long* sub;          // sub-phase timers (ck_debug_subprof), nullable
  int sub_rank;
  int full;                // 1: also compute values nothing downstream reads (conv
                           // cells a pool truncates, dense conv deltas) for readback
  const float* pre;        // training: the image-processing layer of visit t at
                           // pre + t * L[1].cells, computed by a batched prepass
                           // (ck_net.cu contrast_pre_kernel); null: phase 0 runs
};

struct Ctx {
  float* act;
  int64_t img;             // dataset index of the current image
  int64_t t;               // position in the visit sequence
  int label;
  double loss;             // written by OP_OUT_DELTA (valid in its thread)
};

// Where this thread sits in its team, plus the CTA's shared scratch.
struct TeamCtx {
  int ph;                  // current phase (sub-phase timers)
  long long* sub;          // sub-phase timer buffer (nullptr: off)
  int sub_rank;
  int rank, size;          // CTA rank in the team / CTAs in the team
  int gtid, gsize;         // thread index / count over the team
  int gwarp, gwarps;       // warp index / count over the team
  float* smem;             // per-CTA scratch
  int smem_floats;
  // the current image (set per image by the kernel): bytes + LUT, or f32
  const uint8_t* in_u8;
  const float* in_lut;
  const float* in_f32;
  const float* pre;        // this image's precomputed image-processing layer (or null)
};

// The y of layer S as the ops below read it: the precomputed image-processing
// layer of the current image when the job carries one, else the act arena.
__device__ __forceinline__ const float* layer_y(const LayerDev& S, const float* act,
                                                const TeamCtx& tm) {
  return (S.kind == L_IMGPROC && tm.pre) ? tm.pre : act + S.y_off;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Development timers (ck_debug_subprof): when armed, thread 0 of team rank
// tm.sub_rank records %globaltimer at numbered points of every phase into
// tm.sub[phase * 32 + point] (last image wins).  Unarmed cost: one test.
#define CK_SUBT(tm, i)                                                        \
  do {                                                                        \
    if ((tm).sub && threadIdx.x == 0 && (tm).rank == (tm).sub_rank) {         \
      long long _t;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                  \
      (tm).sub[(tm).ph * 32 + (i)] = _t;                                      \
      if ((i) == 0) (tm).sub[(tm).ph * 32 + 28] = clock64();                  \
    }                                                                         \
  } while (0)

// Work split: items [0, n) are cut into one contiguous, balanced range per
// CTA of the team; threads (or warps) stride inside their CTA's range.
struct Span {
  int b, e;
};
__device__ __forceinline__ Span cta_span(int64_t n, const TeamCtx& tm) {
  // 32-bit unsigned arithmetic (n * size < 2^32 for every layer we accept)
  const unsigned un = (unsigned)n, r = (unsigned)tm.rank, sz = (unsigned)tm.size;
  return Span{(int)(un * r / sz), (int)(un * (r + 1) / sz)};
}

// span of n items over the team ranks [r0, r1) (empty for ranks outside)
__device__ __forceinline__ Span sub_span(int64_t n, int r0, int r1, const TeamCtx& tm) {
  if (tm.rank < r0 || tm.rank >= r1) return Span{0, 0};
  const unsigned un = (unsigned)n, r = (unsigned)(tm.rank - r0), sz = (unsigned)(r1 - r0);
  return Span{(int)(un * r / sz), (int)(un * (r + 1) / sz)};
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// shared-memory staging.  Copies are issued as cp.async (LDGSTS): a thread
// never waits on one copy before issuing the next, so staging any amount is
// one L2 round trip.  stage_sync() (= wait for this thread's copies, then
// __syncthreads) must separate the staging from the first read.  16-byte
// copies use .cg (L2 only); data produced by other CTAs in the previous phase
// is then never read through a stale L1 line.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void stage_sync() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
}

// Copy n floats into the CTA's scratch when they fit (and n <= max_n), else
// keep reading global memory.
__device__ __forceinline__ const float* stage(const float* src, int n, const TeamCtx& tm,
                                              int& used, int max_n = 1 << 30) {
  if (n > max_n || used + n > tm.smem_floats) return src;
  float* dst = tm.smem + used;
  int head = 0;
  if (((reinterpret_cast<uintptr_t>(src) ^ reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    head = (int)(((16 - (reinterpret_cast<uintptr_t>(src) & 15)) & 15) >> 2);
    if (head > n) head = n;
    const int n4 = (n - head) >> 2;
    for (int i = threadIdx.x; i < n4; i += blockDim.x)
      cp_async16(dst + head + 4 * i, src + head + 4 * i);
    for (int i = head + (n4 << 2) + threadIdx.x; i < n; i += blockDim.x)
      cp_async4(dst + i, src + i);
  } else {
    head = n;
  }
  for (int i = threadIdx.x; i < head; i += blockDim.x) cp_async4(dst + i, src + i);
  used += (n + 3) & ~3;
  return dst;
}

// The current image's input values in the CTA's scratch, read straight from
// the dataset (bytes through the LUT, or f32), so the first layer does not
// wait a phase for OP_LOAD_INPUT to publish them.  nullptr if they do not fit.
__device__ __forceinline__ const float* stage_input(const NetGeo& N, const NetPtr& R, const TeamCtx& tm,
                                                    int& used) {
  const int n = N.in_cells;
  if (used + n > tm.smem_floats) return nullptr;
  float* dst = tm.smem + used;
  if (tm.in_u8) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(tm.in_lut + __ldg(tm.in_u8 + i));
    used += (n + 3) & ~3;
    return dst;
  }
  return stage(tm.in_f32, n, tm, used);
}

// ---------------------------------------------------------------------------
// delta routing: `v` is the gathered (pre-derivative) delta of cell `cell` in
// layer `s` — the value the reference stores before `*= f'(a)`.  Pools store
// it and pass it on to their recorded winner (network.py:253-259: zeroed
// buffer, `+=`, so the winner holds 0 + v); conv / FC multiply by f'(a)
// (network.py:222,227-228,260-261).
// At most kMaxPoolChain pools in a row (an unrolled walk keeps every layer
// index a compile-time constant in the specialised kernels).
constexpr int kMaxPoolChain = 4;
__device__ __forceinline__ void emit_delta(const NetGeo& N, const NetPtr& R, float* act, int s,
                                           int cell, float v) {
#pragma unroll
  for (int hop = 0; hop <= kMaxPoolChain; ++hop) {
    const LayerDev& L = N.L[s];
    if (L.kind == L_POOL) {
      act[L.d_off + cell] = v;
      if (!N.L[s - 1].has_delta) return;
      const int q = cell;
      cell = reinterpret_cast<const int*>(act + L.arg_off)[q];
      v = __fadd_rn(0.0f, v);
      --s;
      const LayerDev& C = N.L[s];
      if (C.kind == L_CONV) {   // the winner's delta, also kept compact per pooled cell
        const float dv = __fmul_rn(v, act_deriv(act[C.a_off + cell]));
        act[C.d_off + cell] = dv;
        act[L.wd_off + q] = dv;
        return;
      }
      continue;
    }
    if (L.kind == L_CONV || L.kind == L_FC)
      act[L.d_off + cell] = __fmul_rn(v, act_deriv(act[L.a_off + cell]));
    return;
  }
}

// ---------------------------------------------------------------------------
// input and contrast layer

__device__ __forceinline__ void op_load_input(const NetGeo& N, const NetPtr& R, const Job& job,
                                              const Ctx& ctx, const TeamCtx& tm) {
  if (!job.images) return;
  float* y = ctx.act + N.L[0].y_off;
  if (job.lut) {
    const uint8_t* img = job.images + ctx.img * (int64_t)N.in_cells;
    const Span sp = cta_span(N.in_cells, tm);
    for (int i = sp.b + threadIdx.x; i < sp.e; i += blockDim.x) y[i] = job.lut[img[i]];
  } else {  // float32 dataset
    const float* img = reinterpret_cast<const float*>(job.images) + ctx.img * (int64_t)N.in_cells;
    const Span sp = cta_span(N.in_cells, tm);
    for (int i = sp.b + threadIdx.x; i < sp.e; i += blockDim.x) y[i] = img[i];
  }
}

// One contrast response cell q (>= C*h*w) of layer L over the image `src`
// (C dense channels) and the filters `kbase`: kImgLanes lanes per cell, lane
// `sub` takes the filter rows i = sub, sub + kImgLanes, ... (f64 fma chains),
// combined by a fixed xor tree -- the same bits wherever it runs (the
// per-image op below and the batched prepass, ck_net.cu).  The f64 result
// rounds to the same f32 as the reference's f64 sum (any f64
// order gave 0 mismatches).
__device__ __forceinline__ double contrast_cell(const LayerDev& L, const float* src,
                                                const double* kbase, int q, int sub,
                                                unsigned gmask) {
  const int hw = L.h * L.w, C = L.src_maps;
  const int cy = L.fh / 2, cx = L.fw / 2, taps = L.fh * L.fw;
  const int o = q / hw, pix = q % hw;
  const int y = pix / L.w, x = pix % L.w;
  const int f = (o - C) / C, c = (o - C) % C;
  const float* s = src + c * hw;
  const double* k = kbase + (int64_t)f * taps;
  double acc = 0.0;
  for (int i = sub; i < L.fh; i += kImgLanes) {
    const float* srow = s + min(max(y + i - cy, 0), L.h - 1) * L.w;
    const double* krow = k + i * L.fw;
    for (int j = 0; j < L.fw; ++j)
      acc = fma(krow[j], (double)srow[min(max(x + j - cx, 0), L.w - 1)], acc);
  }
#pragma unroll
  for (int m = kImgLanes / 2; m > 0; m >>= 1) acc += __shfl_xor_sync(gmask, acc, m);
  return acc;
}

// The contrast layer laid out for the f64 pipe, same bits as contrast_cell:
// a thread takes a strip of kStrip adjacent cells of one (filter, row) and
// computes contrast_cell's eight lane partials itself (rows i = s mod 8, fma
// chains along the row, 4 cells at a time with a sliding register window over
// a replicated-border f64 window of the channel), then combines them in the
// xor tree's order ((p0+p4)+(p2+p6)) + ((p1+p5)+(p3+p7)).  ~0.5 shared loads
// per fma instead of two clamps, a convert and two loads per tap.
constexpr int kStrip = 4;
static_assert(kImgLanes == 8, "contrast_strips restates the 8-lane xor tree");

__host__ __device__ __forceinline__ int strip_pitch(const LayerDev& L) { return L.w + L.fw + kStrip; }

__device__ __forceinline__ void strip_partial(const double* win, int PW, const double* k, int fh,
                                              int fw, int y, int s, double (&p)[kStrip]) {
#pragma unroll
  for (int c = 0; c < kStrip; ++c) p[c] = 0.0;
  for (int i = s; i < fh; i += kImgLanes) {
    const double* row = win + (y + i) * PW;
    const double* kr = k + i * fw;
    double x0 = row[0], x1 = row[1], x2 = row[2], x3 = row[3];
#pragma unroll 4
    for (int j = 0; j < fw; ++j) {
      const double w = kr[j];
      p[0] = fma(w, x0, p[0]);
      p[1] = fma(w, x1, p[1]);
      p[2] = fma(w, x2, p[2]);
      p[3] = fma(w, x3, p[3]);
      x0 = x1;
      x1 = x2;
      x2 = x3;
      x3 = row[j + 4];
    }
  }
}

// The responses of channel c (every filter) from its window `win` ((h + fh -
// 1) rows of strip_pitch(L) doubles: win[r][q] = x[clamp(r - fh/2)][clamp(q -
// fw/2)]) and the f64 filters `kf`, into the layer's y `o`; this CTA's threads.
__device__ __forceinline__ void contrast_strips(const LayerDev& L, const double* win,
                                                const double* kf, int c, float* o) {
  const int C = L.src_maps, H = L.h, W = L.w, hw = H * W;
  const int fh = L.fh, fw = L.fw, PW = strip_pitch(L);
  const int F = (L.cells - C * hw) / (C * hw);
  const int sx = (W + kStrip - 1) / kStrip;
  for (int job = threadIdx.x; job < F * H * sx; job += blockDim.x) {
    const int f = job / (H * sx), y = (job / sx) % H, x0 = (job % sx) * kStrip;
    const double* k = kf + f * fh * fw;
    const double* w0 = win + x0;
    double a[kStrip], b[kStrip], p[kStrip], q[kStrip];
    strip_partial(w0, PW, k, fh, fw, y, 0, p);   // B0 = (p0 + p4) + (p2 + p6)
    strip_partial(w0, PW, k, fh, fw, y, 4, q);
#pragma unroll
    for (int e = 0; e < kStrip; ++e) a[e] = p[e] + q[e];
    strip_partial(w0, PW, k, fh, fw, y, 2, p);
    strip_partial(w0, PW, k, fh, fw, y, 6, q);
#pragma unroll
    for (int e = 0; e < kStrip; ++e) b[e] = a[e] + (p[e] + q[e]);
    strip_partial(w0, PW, k, fh, fw, y, 1, p);   // B1 = (p1 + p5) + (p3 + p7)
    strip_partial(w0, PW, k, fh, fw, y, 5, q);
#pragma unroll
    for (int e = 0; e < kStrip; ++e) a[e] = p[e] + q[e];
    strip_partial(w0, PW, k, fh, fw, y, 3, p);
    strip_partial(w0, PW, k, fh, fw, y, 7, q);
    float* orow = o + ((int64_t)(C + f * C + c) * H + y) * W;
#pragma unroll
    for (int e = 0; e < kStrip; ++e)
      if (x0 + e < W) orow[x0 + e] = (float)(b[e] + (a[e] + (p[e] + q[e])));
  }
}

// correlate(mode="nearest") per (filter, channel): f64 sum, one rounding.
__device__ __forceinline__ void op_imgproc(const NetGeo& N, const NetPtr& R, const LayerDev& L, float* act,
                                           const TeamCtx& tm) {
  __syncthreads();   // scratch reuse
  CK_SUBT(tm, 1);
  const LayerDev& I = N.L[0];
  int used = 0;
  const float* src = stage_input(N, R, tm, used);
  CK_SUBT(tm, 2);
  if (!src) src = act + I.y_off;   // (never: the builder folds only inputs that fit)
  float* out = act + L.y_off;
  const int hw = L.h * L.w;
  const int C = I.maps;
  if (tm.size == 1) {
    // one CTA per image (evaluation): the strip form, channel by channel
    const int PH = L.h + L.fh - 1, PW = strip_pitch(L);
    const int nf = (L.cells - C * hw) / (C * hw) * L.fh * L.fw;
    const int u = (used + 1) & ~1;   // 8-byte alignment for the doubles
    if (u + 2 * (nf + PH * PW) <= tm.smem_floats) {
      double* kf = reinterpret_cast<double*>(tm.smem + u);
      double* win = kf + nf;
      for (int i = threadIdx.x; i < nf; i += blockDim.x) kf[i] = __ldg(R.filt + L.o_filt + i);
      stage_sync();
      for (int q = threadIdx.x; q < C * hw; q += blockDim.x) out[q] = src[q];
      const int cy = L.fh / 2, cx = L.fw / 2;
      for (int c = 0; c < C; ++c) {
        for (int i = threadIdx.x; i < PH * PW; i += blockDim.x) {
          const int r = min(max(i / PW - cy, 0), L.h - 1), q = min(max(i % PW - cx, 0), L.w - 1);
          win[i] = (double)src[c * hw + r * L.w + q];
        }
        __syncthreads();
        contrast_strips(L, win, kf, c, out);
        __syncthreads();
      }
      return;
    }
  }
  const int cy = L.fh / 2, cx = L.fw / 2;
  const int taps = L.fh * L.fw;
  const int lane = lane_id();
  const int n_resp = L.cells - C * hw;
  const Span rs = cta_span(n_resp, tm);
  // the coefficients of the filters this CTA's responses use, staged as raw
  // 32-bit halves of the doubles (a read per tap otherwise waits on L2)
  const double* kbase = R.filt + L.o_filt;
  int f_lo = 0, f_hi = -1;
  if (rs.b < rs.e) {
    f_lo = (rs.b / hw) / C;
    f_hi = ((rs.e - 1) / hw) / C;
    used = (used + 1) & ~1;   // 8-byte alignment for the doubles
    if (used + 2 * (f_hi - f_lo + 1) * taps <= tm.smem_floats) {
      float* dst = tm.smem + used;
      const float* from = reinterpret_cast<const float*>(kbase + (int64_t)f_lo * taps);
      for (int i = threadIdx.x; i < 2 * (f_hi - f_lo + 1) * taps; i += blockDim.x)
        cp_async4(dst + i, from + i);
      kbase = reinterpret_cast<const double*>(dst) - (int64_t)f_lo * taps;
    }
  }
  CK_SUBT(tm, 3);
  stage_sync();
  CK_SUBT(tm, 4);
  const Span cp = cta_span(C * hw, tm);
  for (int q = cp.b + threadIdx.x; q < cp.e; q += blockDim.x) out[q] = src[q];
  // kImgLanes lanes per response cell: lane l takes the filter rows
  // i = l, l + kImgLanes, ... (fma chains in f64), combined by a fixed xor
  // tree.  The f64 result rounds to the same f32 as the reference's f64 sum
  // (any f64 order gave 0 mismatches).
  const int sub = threadIdx.x % kImgLanes;
  const unsigned gmask = ((1u << kImgLanes) - 1) << (lane & ~(kImgLanes - 1));
  for (int r = rs.b + threadIdx.x / kImgLanes; r < rs.e; r += blockDim.x / kImgLanes) {
    const int q = C * hw + r;
    const double acc = contrast_cell(L, src, kbase, q, sub, gmask);
    if (sub == 0) out[q] = (float)acc;
  }
}

// ---------------------------------------------------------------------------
// conv forward (kernels.py:70-87)

// One output cell, reference order: bias, then per connected source k, rows
// v, columns u; every product and sum rounded to f32 separately.
template <int KX, int KY>
__device__ __forceinline__ float conv_cell(float acc, const float* src, const int* soff,
                                           const float* w, int nk, int sw, int kx, int ky) {
  if constexpr (KX > 0) {
    for (int k = 0; k < nk; ++k) {
      const float* s = src + soff[k];
      const float* wk = w + k * (KX * KY);
      float xs[KX * KY];
#pragma unroll
      for (int v = 0; v < KY; ++v)
#pragma unroll
        for (int u = 0; u < KX; ++u) xs[v * KX + u] = s[v * sw + u];
#pragma unroll
      for (int t = 0; t < KX * KY; ++t) acc = __fadd_rn(acc, __fmul_rn(wk[t], xs[t]));
    }
  } else {
    const int kk = kx * ky;
    for (int k = 0; k < nk; ++k) {
      const float* s = src + soff[k];
      const float* wk = w + k * kk;
      for (int v = 0; v < ky; ++v)
        for (int u = 0; u < kx; ++u) acc = __fadd_rn(acc, __fmul_rn(wk[v * kx + u], s[v * sw + u]));
    }
  }
  return acc;
}

// explicit ld.shared helpers (32-bit shared addresses, no generic loads)
__device__ __forceinline__ float lds_f32(unsigned addr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int lds_s32(unsigned addr) {
  int v;
  asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// a 16-byte shared load (the chain's weights: one broadcast wavefront for 4)
__device__ __forceinline__ float4 lds_v4(unsigned addr) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// One source of conv_cell_smem4: rows v = 0..KY-1 with the row ring resolved
// at compile time (PAR = parity of the source's first row), the next row
// loaded while the current one is added; `nsrc` is the next source's base.
template <int KX, int KY, int PAR>
__device__ __forceinline__ void conv_rows_smem(float& acc, const float* wcur, unsigned sb,
                                               unsigned nsrc, int sw, float (&xa)[KX],
                                               float (&xb)[KX]) {
#pragma unroll
  for (int v = 0; v < KY; ++v) {
    const bool cur_a = ((PAR + v) & 1) == 0;
    const unsigned nrow = v + 1 < KY ? sb + 4u * (unsigned)((v + 1) * sw) : nsrc;
#pragma unroll
    for (int u = 0; u < KX; ++u) {
      if (cur_a) xb[u] = lds_f32(nrow + 4u * u);
      else xa[u] = lds_f32(nrow + 4u * u);
    }
#pragma unroll
    for (int u = 0; u < KX; ++u)
      acc = __fadd_rn(acc, __fmul_rn(wcur[v * KX + u], cur_a ? xa[u] : xb[u]));
  }
}

template <int KKP>
__device__ __forceinline__ void lds_weights(float (&w)[KKP], unsigned addr) {
#pragma unroll
  for (int j = 0; j < KKP / 4; ++j) {
    const float4 v = lds_v4(addr + 16u * j);
    w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
  }
}

// The reference-order chain of one conv cell with every operand in shared
// memory: each pair's kx*ky weights at a 16-byte aligned stride of KKP =
// round_up(kx*ky, 4) floats, read as broadcast ld.shared.v4 a whole source
// ahead; source rows one row ahead.  Two sources per loop iteration resolve
// both register rings (rows, weights) at compile time, so no register copies
// reach the FMA pipe: per tap it issues exactly the FMUL and the FADD (2
// cycles each per warp -- with the 4-cycle FADD latency, the chain's floor;
// tools/mb_conv.cu V12).  Same operands, same order: bit-identical to
// conv_cell.
template <int KX, int KY>
__device__ __forceinline__ float conv_cell_smem4(float acc, const float* src, const int* soff,
                                                 const float* w, int nk, int sw) {
  constexpr int KK = KX * KY, KKP = (KK + 3) & ~3;
  (void)KK;
  const unsigned s0 = (unsigned)__cvta_generic_to_shared(src);
  const unsigned o0 = (unsigned)__cvta_generic_to_shared(soff);
  const unsigned w0 = (unsigned)__cvta_generic_to_shared(w);
  float xa[KX], xb[KX], wa[KKP], wb[KKP];
  lds_weights<KKP>(wa, w0);
  unsigned sb = s0 + 4u * (unsigned)lds_s32(o0);
#pragma unroll
  for (int u = 0; u < KX; ++u) xa[u] = lds_f32(sb + 4u * u);
  int k = 0;
  for (; k + 2 <= nk; k += 2) {
    const unsigned sb1 = s0 + 4u * (unsigned)lds_s32(o0 + 4u * (k + 1));
    lds_weights<KKP>(wb, w0 + 4u * (unsigned)((k + 1) * KKP));
    conv_rows_smem<KX, KY, 0>(acc, wa, sb, sb1, sw, xa, xb);
    const int k2 = k + 2 < nk ? k + 2 : k + 1;
    const unsigned sb2 = s0 + 4u * (unsigned)lds_s32(o0 + 4u * k2);
    lds_weights<KKP>(wa, w0 + 4u * (unsigned)(k2 * KKP));
    conv_rows_smem<KX, KY, KY & 1>(acc, wb, sb1, sb2, sw, xa, xb);
    sb = sb2;
  }
  if (k < nk) conv_rows_smem<KX, KY, 0>(acc, wa, sb, sb, sw, xa, xb);
  return acc;
}

// All PB x PB conv cells of one pool block, one thread: the block shares its
// dest map's weights (one load per tap for PB*PB chains) and its source
// window (loads shared between neighbouring cells).  Each cell's own chain
// keeps the reference order (bias, k, v, u) -- bit-identical to conv_cell.
// For throughput (many cells per CTA: evaluation, wide first layers).
template <int KX, int KY, int PB>
__device__ __forceinline__ void conv_block_smem(float* acc, const float* src, const int* soff,
                                                const float* w, int nk, int sw, int ty,
                                                int tx) {
  constexpr int KK = KX * KY;
  const unsigned s0 = (unsigned)__cvta_generic_to_shared(src);
  const unsigned o0 = (unsigned)__cvta_generic_to_shared(soff);
  const unsigned w0 = (unsigned)__cvta_generic_to_shared(w);
  if (tx == 1 && ty == 1) {
    // stride 1: the block's (PB+KY-1) x (PB+KX-1) source window is read one
    // row at a time into registers and every cell whose kernel row v covers
    // it takes its taps from there -- (PB+KY-1)(PB+KX-1) loads per source
    // instead of PB*PB*KX*KY.  A cell's sum still runs k, then v (window rows
    // ascend), then u: bit-identical.
    constexpr int WL = PB + KX - 1;
    for (int k = 0; k < nk; ++k) {
      const unsigned sb = s0 + 4u * (unsigned)lds_s32(o0 + 4u * k);
      float wr[KK];
#pragma unroll
      for (int t = 0; t < KK; ++t) wr[t] = lds_f32(w0 + 4u * (k * KK + t));
#pragma unroll
      for (int row = 0; row < PB + KY - 1; ++row) {
        float xr[WL];
#pragma unroll
        for (int j = 0; j < WL; ++j) xr[j] = lds_f32(sb + 4u * (row * sw + j));
#pragma unroll
        for (int cy = 0; cy < PB; ++cy) {
          const int v = row - cy;
          if (v < 0 || v >= KY) continue;
#pragma unroll
          for (int u = 0; u < KX; ++u)
#pragma unroll
            for (int cx = 0; cx < PB; ++cx)
              acc[cy * PB + cx] =
                  __fadd_rn(acc[cy * PB + cx], __fmul_rn(wr[v * KX + u], xr[cx + u]));
        }
      }
    }
    return;
  }
  for (int k = 0; k < nk; ++k) {
    const unsigned sb = s0 + 4u * (unsigned)lds_s32(o0 + 4u * k);
#pragma unroll
    for (int v = 0; v < KY; ++v)
#pragma unroll
      for (int u = 0; u < KX; ++u) {
        const float wv = lds_f32(w0 + 4u * (k * KK + v * KX + u));
#pragma unroll
        for (int cy = 0; cy < PB; ++cy)
#pragma unroll
          for (int cx = 0; cx < PB; ++cx) {
            const float x = lds_f32(sb + 4u * ((cy * ty + v) * sw + cx * tx + u));
            acc[cy * PB + cx] = __fadd_rn(acc[cy * PB + cx], __fmul_rn(wv, x));
          }
      }
  }
}

// The team's cells are split into one contiguous chunk per CTA.  The chunk's
// weights (contiguous in the arena: per dest [blocks..., bias]) and source
// map offsets are staged in shared memory; the source layer too when it fits.
template <int KX, int KY>
__device__ __forceinline__ void conv_fwd_chunk(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags, float* act,
                               const TeamCtx& tm) {
  const LayerDev& S = N.L[&L - N.L - 1];
  const int hw = L.h * L.w;
  const int64_t Q = (int64_t)L.cells;
  const int q0 = (int)(Q * tm.rank / tm.size);
  const int q1 = (int)(Q * (tm.rank + 1) / tm.size);
  if (q0 >= q1) return;
  const int d0 = q0 / hw, d1 = (q1 - 1) / hw;
  const int kk = L.kx * L.ky;
  const int k0 = t_fwd_off(R, L, (d0)), k1 = t_fwd_off(R, L, (d1 + 1));
  const float* arena = R.params + L.p_off;
  const int w0 = t_fwd_widx(R, L, (k0));                      // first weight of map d0
  const int n_w = t_bias_off(R, L, (d1)) + 1 - w0;            // through d1's bias
  const int n_src = S.cells;

  // shared layout: [src offsets (k1-k0 ints)] [weights n_w] [source layer]
  int* soff = reinterpret_cast<int*>(tm.smem);
  float* ws = tm.smem + (k1 - k0);
  float* ss = ws + n_w;
  const bool w_in_smem = (k1 - k0) + n_w <= tm.smem_floats;
  const bool s_in_smem = w_in_smem && (k1 - k0) + n_w + n_src <= tm.smem_floats;
  const float* src_g = layer_y(S, act, tm);
  for (int k = threadIdx.x; k < k1 - k0; k += blockDim.x) soff[k] = t_fwd_src(R, L, (k0 + k)) * (S.h * S.w);
  if (w_in_smem)
    for (int i = threadIdx.x; i < n_w; i += blockDim.x) cp_async4(ws + i, arena + w0 + i);
  if (s_in_smem)
    for (int i = threadIdx.x; i < n_src; i += blockDim.x) cp_async4(ss + i, src_g + i);
  stage_sync();
  const float* wbase = w_in_smem ? ws : arena + w0;
  const float* sbase = s_in_smem ? ss : src_g;
  const int* offs = w_in_smem ? soff : nullptr;

  float* a = act + L.a_off;
  float* y = act + L.y_off;
  float* dl = act + L.d_off;
  for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int d = q / hw, pix = q % hw;
    const int r = pix / L.w, c = pix % L.w;
    const int kb = t_fwd_off(R, L, (d)), ke = t_fwd_off(R, L, (d + 1));
    const float* w = wbase + (t_fwd_widx(R, L, (kb)) - w0);
    float acc = w[(ke - kb) * kk];                    // bias slot follows the blocks
    const int rc = (r * L.ty) * S.w + c * L.tx;
    if (offs) {
      acc = conv_cell<KX, KY>(acc, sbase + rc, offs + (kb - k0), w, ke - kb, S.w, L.kx, L.ky);
    } else {
      for (int k = kb; k < ke; ++k) {
        const int so = t_fwd_src(R, L, (k)) * (S.h * S.w);
        acc = conv_cell<KX, KY>(acc, sbase + rc, &so, w + (k - kb) * kk, 1, S.w, L.kx, L.ky);
      }
    }
    a[q] = acc;
    y[q] = conv_act(acc);
    if (flags & F_ZERO_SELF) dl[q] = 0.0f;
  }
  __syncthreads();
}

__device__ __forceinline__ void op_conv_fwd(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags,
                                            float* act, const TeamCtx& tm) {
  if (L.kx == 2 && L.ky == 2) conv_fwd_chunk<2, 2>(N, R, L, flags, act, tm);
  else if (L.kx == 3 && L.ky == 3) conv_fwd_chunk<3, 3>(N, R, L, flags, act, tm);
  else if (L.kx == 4 && L.ky == 4) conv_fwd_chunk<4, 4>(N, R, L, flags, act, tm);
  else if (L.kx == 5 && L.ky == 5) conv_fwd_chunk<5, 5>(N, R, L, flags, act, tm);
  else conv_fwd_chunk<0, 0>(N, R, L, flags, act, tm);
}

// A pooled value, plus its pre-pitched copy when the consumer asked for one.
__device__ __forceinline__ void store_pooled(const LayerDev& P, float* act, int q, float v) {
  act[P.y_off + q] = v;
  if (P.ypitch > 0) {
    const int phw = P.h * P.w, m = q / phw, pix = q - m * phw, r = pix / P.w;
    act[P.yp_off + (int64_t)(m * P.h + r) * P.ypitch + (pix - r * P.w)] = v;
  }
}

// max-pool (kernels.py:154-172): strict '>' keeps the first cell in scan order.
// The argmax is stored as an index into the whole source layer.
__device__ __forceinline__ void op_pool_fwd(const NetGeo& N, const NetPtr& R, const LayerDev& L, float* act,
                                            const TeamCtx& tm) {
  const LayerDev& S = N.L[&L - N.L - 1];
  const float* src = layer_y(S, act, tm);
  float* y = act + L.y_off;
  int* arg = reinterpret_cast<int*>(act + L.arg_off);
  const int hw = L.h * L.w;
  const int shw = S.h * S.w;
  const Span sp = cta_span(L.cells, tm);
  for (int q = sp.b + threadIdx.x; q < sp.e; q += blockDim.x) {
    const int m = q / hw, pix = q % hw;
    const int r = pix / L.w, c = pix % L.w;
    const int base = m * shw;
    int best_i = base + (r * L.py) * S.w + c * L.px;
    float best = src[best_i];
    for (int v = 0; v < L.py; ++v)
      for (int u = 0; u < L.px; ++u) {
        const int i = base + (r * L.py + v) * S.w + c * L.px + u;
        const float val = src[i];
        if (val > best) { best = val; best_i = i; }
      }
    store_pooled(L, act, q, best);
    arg[q] = best_i;
    if (S.kind == L_CONV) {
      const int local = best_i - base;
      reinterpret_cast<int*>(act + L.wrc_off)[q] = ((local / S.w) << 16) | (local % S.w);
    }
  }
}

// ---------------------------------------------------------------------------
// conv forward fused with the max-pool above it (kernels.py:70-87 then
// :154-172).  Work is split by POOLED cells: a CTA computes every conv cell
// of its pool blocks (same per-cell arithmetic as conv_fwd_chunk), keeps the
// block's y in shared memory and picks the winner there (strict '>', first
// cell in row-major scan).  Conv cells a pool truncates feed nothing
// downstream; they are computed only for readback (job.full).

// One conv cell from global weights (used for the truncated cells).
template <int KX, int KY>
__device__ __forceinline__ float conv_value_global(const NetPtr& R, const LayerDev& L,
                                                   const LayerDev& S,
                                                   const float* arena, const float* src,
                                                   int d, int r, int c) {
  const int kk = L.kx * L.ky;
  const int kb = t_fwd_off(R, L, (d)), ke = t_fwd_off(R, L, (d + 1));
  const float* w = arena + t_fwd_widx(R, L, (kb));
  float acc = arena[t_bias_off(R, L, (d))];
  const int rc = (r * L.ty) * S.w + c * L.tx;
  for (int k = kb; k < ke; ++k) {
    const int so = t_fwd_src(R, L, (k)) * (S.h * S.w);
    acc = conv_cell<KX, KY>(acc, src + rc, &so, w + (k - kb) * kk, 1, S.w, L.kx, L.ky);
  }
  return acc;
}

// conv + pool for a FULL connection table whose source layer does not fit the
// scratch (C4'): one cell per thread on the reference-order chain, the
// source maps staged in passes of as many whole maps as fit (the pool's
// pre-pitched copy when it has one), every chain continuing where the last
// pass left it -- the order stays bias, then k = 0, 1, ... .  Returns false
// (nothing done) when the CTA's cells exceed one per thread.
template <int KX, int KY>
__device__ __forceinline__ bool conv_pool_fwd_passes(const NetGeo& N, const NetPtr& R,
                                                     const LayerDev& L, int flags, bool full,
                                                     float* act, const TeamCtx& tm) {
  constexpr int KK = KX * KY, KKP = (KK + 3) & ~3;
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const LayerDev& P = N.L[li + 1];
  const int hw = L.h * L.w, phw = P.h * P.w, blk = P.px * P.py;
  const Span sp = cta_span(P.cells, tm);
  const int n_items = (sp.e - sp.b) * blk;
  if (n_items > (int)blockDim.x) return false;     // uniform per CTA
  if (sp.b >= sp.e) return true;
  const float* arena = R.params + L.p_off;
  const int d0 = sp.b / phw, d1 = (sp.e - 1) / phw, nd = d1 - d0 + 1;
  const int SM = S.maps;
  const bool pitched = S.ypitch > 0;
  const int sw = pitched ? S.ypitch : S.w, smap = S.h * sw;
  const float* src = pitched ? act + S.yp_off : layer_y(S, act, tm);
  // scratch: [weights nd*SM*KKP | biases nd | map offsets | pre-activations | source pass]
  float* ws = tm.smem;
  float* bs = ws + nd * SM * KKP;
  int* soff = reinterpret_cast<int*>(bs + ((nd + 3) & ~3));
  float* ybuf = reinterpret_cast<float*>(soff) + ((SM + 3) & ~3);
  float* sp_buf = ybuf + ((n_items + 3) & ~3);
  const int room = tm.smem_floats - (int)(sp_buf - tm.smem);
  const int per_pass = min(SM, room / smap);
  if (per_pass < 1) return false;
  for (int e = threadIdx.x; e < nd * SM * KK; e += blockDim.x) {
    const int j = e / KK, t = e - j * KK;        // pair (d0 + j / SM, j % SM)
    const int d = d0 + j / SM;
    cp_async4(ws + j * KKP + t, arena + ((int64_t)d * SM + j % SM) * KK + d + t + (int64_t)0);
  }
  for (int d = d0 + threadIdx.x; d <= d1; d += blockDim.x)
    cp_async4(bs + (d - d0), arena + (int64_t)(d + 1) * SM * KK + d);
  for (int k = threadIdx.x; k < SM; k += blockDim.x) soff[k] = k * smap;
  const int it = threadIdx.x;
  const bool mine = it < n_items;
  const int qq = sp.b + it / blk, t = it % blk;
  const int d = qq / phw, pp = qq % phw;
  const int r = (pp / P.w) * P.py + t / P.px, c = (pp % P.w) * P.px + t % P.px;
  float acc = 0.0f;
  for (int m0 = 0; m0 < SM; m0 += per_pass) {
    const int m1 = min(SM, m0 + per_pass);
    if (m0 > 0) __syncthreads();                 // the previous pass is consumed
    int u = (int)(sp_buf - tm.smem);
    stage(src + (int64_t)m0 * smap, (m1 - m0) * smap, tm, u);
    stage_sync();
    if (mine) {
      if (m0 == 0) acc = bs[d - d0];
      acc = conv_cell_smem4<KX, KY>(acc, sp_buf + (r * L.ty) * sw + c * L.tx, soff,
                                    ws + ((d - d0) * SM + m0) * KKP, m1 - m0, sw);
    }
  }
  // epilogue: a / y of the cell, then the pool of each block (strict '>')
  const bool zero = full && (flags & F_ZERO_SELF);
  const bool pooled_only = (flags & F_POOLED_ONLY) && !full;
  if (mine) {
    if (pooled_only) {
      ybuf[it] = acc;
    } else {
      const int cell = d * hw + r * L.w + c;
      const float yv = conv_act(acc);
      act[L.a_off + cell] = acc;
      act[L.y_off + cell] = yv;
      ybuf[it] = yv;
      if (zero) act[L.d_off + cell] = 0.0f;
    }
  }
  __syncthreads();
  int* parg = reinterpret_cast<int*>(act + P.arg_off);
  int* pwrc = reinterpret_cast<int*>(act + P.wrc_off);
  for (int qi = threadIdx.x; qi < sp.e - sp.b; qi += blockDim.x) {
    const float* yb = ybuf + qi * blk;
    int bt = 0;
    float best = yb[0];
    for (int tt = 1; tt < blk; ++tt)
      if (yb[tt] > best) { best = yb[tt]; bt = tt; }
    if (pooled_only) best = conv_act(best);
    const int q2 = sp.b + qi;
    const int d2 = q2 / phw, p2 = q2 % phw;
    const int r2 = (p2 / P.w) * P.py + bt / P.px, c2 = (p2 % P.w) * P.px + bt % P.px;
    store_pooled(P, act, q2, best);
    parg[q2] = d2 * hw + r2 * L.w + c2;
    pwrc[q2] = (r2 << 16) | c2;
  }
  __syncthreads();
  return true;
}

template <int KX, int KY>
__device__ __forceinline__ void conv_pool_fwd(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags, bool full,
                              float* act, const TeamCtx& tm) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const LayerDev& P = N.L[li + 1];
  const int hw = L.h * L.w, shw = S.h * S.w, phw = P.h * P.w, blk = P.px * P.py;
  const int kk = L.kx * L.ky;
  const float* arena = R.params + L.p_off;
  float* a = act + L.a_off;
  float* y = act + L.y_off;
  float* dl = act + L.d_off;
  float* pyv = act + P.y_off;
  int* parg = reinterpret_cast<int*>(act + P.arg_off);
  int* pwrc = reinterpret_cast<int*>(act + P.wrc_off);
  CK_SUBT(tm, 1);
  const Span sp = cta_span(P.cells, tm);
  if constexpr (KX > 0) {
    // full table, source layer too big to stage whole: source passes
    if (L.full && li > 1 && S.cells > tm.smem_floats / 2 && !full &&
        conv_pool_fwd_passes<KX, KY>(N, R, L, flags, full, act, tm)) {
      return;
    }
  }
  int used = 0;
  const float* src_g = layer_y(S, act, tm);
  const float* src = src_g;
  int sw = S.w;               // row pitch of `src` (L.spitch when staged pitched)
  if (li == 1) {
    if (sp.b < sp.e) {
      const float* si = stage_input(N, R, tm, used);
      if (si) src = si;
    }
  } else if (sp.b < sp.e && S.cells <= tm.smem_floats / 2) {
    // the whole source layer, unless this CTA's maps connect to fewer cells
    // (from the producer's pre-pitched copy -- bank-conflict-free reads --
    // when it still leaves the chunk 3/8 of the scratch)
    const int nk_all = t_fwd_off(R, L, ((sp.e - 1) / phw + 1)) - t_fwd_off(R, L, (sp.b / phw));
    CK_SUBT(tm, 20);
    if (S.cells <= nk_all * shw) {
      if (S.ypitch > 0 && S.maps * S.h * S.ypitch <= tm.smem_floats / 8 * 5) {
        src = stage(act + S.yp_off, S.maps * S.h * S.ypitch, tm, used);
        sw = S.ypitch;
      } else {
        src = stage(src, S.cells, tm, used);
      }
    }
    CK_SUBT(tm, 21);
  }
  const bool whole = src != src_g;
  const int smap = S.h * sw;  // map stride of `src`
  constexpr int KKP = KX > 0 ? ((KX * KY + 3) & ~3) : 1;
  const bool zero = full && (flags & F_ZERO_SELF);
  const bool pooled_only = (flags & F_POOLED_ONLY) && !full;
  // The arena is tiled like ConnectionTable (checked at ck_net_create): dest
  // map d's blocks start at fwd_off[d]*kk + d and its bias sits at
  // fwd_off[d+1]*kk + d, so the chunk plan needs fwd_off alone.
  for (int q = sp.b; q < sp.e;) {
    // chunk [q, qe): block outputs (+ its weights and source offsets when they fit)
    // (with the source layer not staged whole, a copy of each connected
    // source map too -- sparse tables need far less than the whole layer)
    const int avail = tm.smem_floats - used;
    int qe = min(sp.e, q + avail / blk);
    CK_SUBT(tm, 22);
    bool wst = false, slots = false;
    for (int tries = 0; tries < 24; ++tries) {
      const int d0 = q / phw, d1 = (qe - 1) / phw;
      const int nk = t_fwd_off(R, L, (d1 + 1)) - t_fwd_off(R, L, (d0));
      // weights: unpadded, or per pair at a KKP stride plus the biases (chain path)
      const int nw = nk * (KX > 0 ? KKP : kk) + d1 + 1 - d0;
      const int base = ((nk + 3) & ~3) + ((nw + 3) & ~3) + (qe - q) * blk;
      if (!whole && base + nk * shw <= avail) { wst = slots = true; break; }
      if (whole && base <= avail) { wst = true; break; }
      if (qe - q <= phw) {
        wst = base <= avail;
        break;
      }
      qe = q + max(phw, (qe - q) / 2);
    }
    CK_SUBT(tm, 2);
    const int d0 = q / phw, d1 = (qe - 1) / phw;
    const int k0 = t_fwd_off(R, L, (d0)), k1 = t_fwd_off(R, L, (d1 + 1));
    const int w0 = k0 * kk + d0;
    const int n_items = (qe - q) * blk;
    // one pool block per thread (many cells per CTA), else one cell per
    // thread on the reference-order chain with padded (v4) weights
    const bool block_path = KX > 0 && wst && (whole || slots) && P.px == P.py && P.px >= 2 &&
                            P.px <= 4 && n_items > (int)blockDim.x;
    const bool padw = KX > 0 && wst && (whole || slots) && !block_path;
    const int nw = (k1 - k0) * (padw ? KKP : kk) + d1 + 1 - d0;
    int* soff = reinterpret_cast<int*>(tm.smem + used);
    float* ws = tm.smem + used + ((k1 - k0 + 3) & ~3);
    float* bs = ws + (k1 - k0) * KKP;   // padw: the chunk's biases after its blocks
    float* ybuf = wst ? ws + ((nw + 3) & ~3) : tm.smem + used;
    float* sslot = ybuf + (qe - q) * blk;
    const float* sbase = slots ? sslot : src;
    if (wst) {
      if (padw) {
        // pair k0 + j's kk weights (arena index p * kk + dest(p), topology
        // tiling) at ws + j * KKP; dest d's bias at bs[d - d0]
        for (int e = threadIdx.x; e < (k1 - k0) * kk; e += blockDim.x) {
          const int j = e / kk, t = e - j * kk;
          cp_async4(ws + j * KKP + t, arena + (k0 + j) * kk + t_pair_dst(R, L, k0 + j) + t);
        }
        for (int d = d0 + threadIdx.x; d <= d1; d += blockDim.x)
          cp_async4(bs + (d - d0), arena + t_fwd_off(R, L, d + 1) * kk + d);
      } else {
        int u2 = used + ((k1 - k0 + 3) & ~3);
        stage(arena + w0, nw, tm, u2);
      }
      for (int k = threadIdx.x; k < k1 - k0; k += blockDim.x)
        soff[k] = slots ? k * shw : t_fwd_src(R, L, (k0 + k)) * smap;
      if (slots)
        for (int k = (threadIdx.x >> 5); k < k1 - k0; k += (blockDim.x >> 5)) {
          const float* from = src_g + t_fwd_src(R, L, (k0 + k)) * shw;
          for (int i = lane_id(); i < shw; i += 32) cp_async4(sslot + k * shw + i, from + i);
        }
    }
    CK_SUBT(tm, 3);
    stage_sync();
    CK_SUBT(tm, 4);
    if constexpr (KX > 0) {
      // many cells per thread: one pool block per thread (conv_block_smem)
      if (block_path) {
        for (int qi = threadIdx.x; qi < qe - q; qi += blockDim.x) {
          const int qq = q + qi;
          const int d = qq / phw, pp = qq % phw;
          const int r0 = (pp / P.w) * P.py, c0 = (pp % P.w) * P.px;
          const int kb = t_fwd_off(R, L, d), ke = t_fwd_off(R, L, d + 1);
          const float* w = ws + (kb * kk + d - w0);
          const float* sp = sbase + (r0 * L.ty) * sw + c0 * L.tx;
          float acc[16];
          const float bias = w[(ke - kb) * kk];
#pragma unroll
          for (int t = 0; t < 16; ++t) acc[t] = bias;
          if (P.px == 2)
            conv_block_smem<KX, KY, 2>(acc, sp, soff + (kb - k0), w, ke - kb, sw, L.ty, L.tx);
          else if (P.px == 3)
            conv_block_smem<KX, KY, 3>(acc, sp, soff + (kb - k0), w, ke - kb, sw, L.ty, L.tx);
          else
            conv_block_smem<KX, KY, 4>(acc, sp, soff + (kb - k0), w, ke - kb, sw, L.ty, L.tx);
          int bt = 0;
          float best = 0.0f;
          if (pooled_only) {
            for (int t = 1; t < blk; ++t)
              if (acc[t] > acc[bt]) bt = t;
            // (one CTA per image -- evaluation -- inlines: acc[] is live)
            best = tm.size == 1 ? conv_act_inl(acc[bt]) : conv_act(acc[bt]);
          } else {
            for (int t = 0; t < blk; ++t) {   // scan order: rows, then columns
              const int cell = d * hw + (r0 + t / P.px) * L.w + c0 + t % P.px;
              const float yv = tm.size == 1 ? conv_act_inl(acc[t]) : conv_act(acc[t]);
              a[cell] = acc[t];
              y[cell] = yv;
              if (zero) dl[cell] = 0.0f;
              if (t == 0 || yv > best) { best = yv; bt = t; }
            }
          }
          const int r = r0 + bt / P.px, c = c0 + bt % P.px;
          store_pooled(P, act, qq, best);
          parg[qq] = d * hw + r * L.w + c;
          pwrc[qq] = (r << 16) | c;
        }
        __syncthreads();
        q = qe;
        continue;
      }
    }
    for (int it = threadIdx.x; it < n_items; it += blockDim.x) {
      const int qq = q + it / blk, t = it % blk;
      const int d = qq / phw, pp = qq % phw;
      const int r = (pp / P.w) * P.py + t / P.px;
      const int c = (pp % P.w) * P.px + t % P.px;
      float acc;
      if (wst) {
        const int kb = t_fwd_off(R, L, (d)), ke = t_fwd_off(R, L, (d + 1));
        const float* w = ws + (kb * kk + d - w0);
        if constexpr (KX > 0) {
          if (padw)   // weights (v4), offsets and sources all in shared memory
            acc = conv_cell_smem4<KX, KY>(bs[d - d0], sbase + (r * L.ty) * sw + c * L.tx,
                                          soff + (kb - k0), ws + (kb - k0) * KKP, ke - kb, sw);
          else
            acc = conv_cell<KX, KY>(w[(ke - kb) * kk], sbase + (r * L.ty) * sw + c * L.tx,
                                    soff + (kb - k0), w, ke - kb, sw, L.kx, L.ky);
        } else {
          acc = conv_cell<KX, KY>(w[(ke - kb) * kk], sbase + (r * L.ty) * sw + c * L.tx,
                                  soff + (kb - k0), w, ke - kb, sw, L.kx, L.ky);
        }
      } else {
        acc = conv_value_global<KX, KY>(R, L, S, arena, src, d, r, c);
      }
      if (pooled_only) {
        ybuf[it] = acc;             // pre-activation; activated after the pool
        continue;
      }
      const int cell = d * hw + r * L.w + c;
      const float yv = conv_act(acc);
      a[cell] = acc;
      y[cell] = yv;
      ybuf[it] = yv;
      if (zero) dl[cell] = 0.0f;
    }
    CK_SUBT(tm, 5);
    __syncthreads();
    CK_SUBT(tm, 6);
    for (int qi = threadIdx.x; qi < qe - q; qi += blockDim.x) {
      const float* yb = ybuf + qi * blk;
      int bt = 0;
      float best = yb[0];
      for (int t = 1; t < blk; ++t)
        if (yb[t] > best) { best = yb[t]; bt = t; }
      if (pooled_only) best = conv_act(best);
      const int qq = q + qi;
      const int d = qq / phw, pp = qq % phw;
      const int r = (pp / P.w) * P.py + bt / P.px;
      const int c = (pp % P.w) * P.px + bt % P.px;
      store_pooled(P, act, qq, best);
      parg[qq] = d * hw + r * L.w + c;
      pwrc[qq] = (r << 16) | c;
    }
    __syncthreads();
    CK_SUBT(tm, 7);
    q = qe;
  }
  if (full) {   // cells outside every pool block (rows / columns the pool drops)
    const int rh = P.h * P.py, cw = P.w * P.px;
    const int strip = rh * (L.w - cw);
    const int nd = hw - rh * cw;
    if (nd > 0) {
      const Span ds = cta_span((int64_t)nd * L.maps, tm);
      for (int e = ds.b + threadIdx.x; e < ds.e; e += blockDim.x) {
        const int d = e / nd, k = e % nd;
        int r, c;
        if (k < strip) { r = k / (L.w - cw); c = cw + k % (L.w - cw); }
        else { r = rh + (k - strip) / L.w; c = (k - strip) % L.w; }
        const float acc = conv_value_global<KX, KY>(R, L, S, arena,
                                                    whole && sw == S.w ? src : src_g, d, r, c);
        const int cell = d * hw + r * L.w + c;
        a[cell] = acc;
        y[cell] = conv_act(acc);
        if (zero) dl[cell] = 0.0f;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void op_conv_pool(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags,
                                             bool full, float* act, const TeamCtx& tm) {
  if (L.kx == 2 && L.ky == 2) conv_pool_fwd<2, 2>(N, R, L, flags, full, act, tm);
  else if (L.kx == 3 && L.ky == 3) conv_pool_fwd<3, 3>(N, R, L, flags, full, act, tm);
  else if (L.kx == 4 && L.ky == 4) conv_pool_fwd<4, 4>(N, R, L, flags, full, act, tm);
  else if (L.kx == 5 && L.ky == 5) conv_pool_fwd<5, 5>(N, R, L, flags, full, act, tm);
  else conv_pool_fwd<0, 0>(N, R, L, flags, full, act, tm);
}

// ---------------------------------------------------------------------------
// FC forward (network.py:193-199).  Column j's pre-activation is always
//   f32( sum_{sl=0..15} [ f64 fma-chain over rows i = sl, sl+16, ... ] ) + b_j
// (16 fixed interleaved slices combined in slice order), whatever the tile
// width or team shape, so training and evaluation agree bit for bit.
// fc_cols_preact computes ncols (<= 32) columns whose weights sit at
// W[i * ldw + j] (global or staged); a[j] lands in out_a (shared memory).
// All threads must call.
__device__ __forceinline__ void fc_cols_preact(const float* x, const float* W, int ldw,
                                               const float* b, int n_in, int ncols,
                                               double* red, float* out_a) {
  for (int item = threadIdx.x; item < kFcSlices * ncols; item += blockDim.x) {
    const int col = item % ncols, sl = item / ncols;
    double part = 0.0;
#pragma unroll 4
    for (int i = sl; i < n_in; i += kFcSlices)
      part = fma((double)x[i], (double)W[i * ldw + col], part);
    red[sl * ncols + col] = part;
  }
  __syncthreads();
  if (threadIdx.x < ncols) {
    double acc = 0.0;
    for (int sl = 0; sl < kFcSlices; ++sl) acc += red[sl * ncols + threadIdx.x];
    out_a[threadIdx.x] = __fadd_rn((float)acc, b[threadIdx.x]);
  }
  __syncthreads();
}

__device__ __forceinline__ void op_fc_fwd(const NetGeo& N, const NetPtr& R, const LayerDev& L, float* act,
                                          const TeamCtx& tm) {
  const LayerDev& S = N.L[&L - N.L - 1];
  const int n_in = S.cells, n_out = L.cells;
  // tile width: a team with at least two columns per CTA spreads them over
  // all its CTAs (fewer weights staged per CTA; 4-column tiles of 16-byte row
  // pieces when the layout allows): C3 / C4 +1%, while narrower layers (C1 /
  // C2: 150 columns) measured faster with kFcTile, as is one CTA
  // (evaluation).  The slices fix the bits, not the tile.
  int tw = kFcTile;
  bool v4 = false;
  if (tm.size > 1 && n_out >= 2 * tm.size) {
    tw = min(kFcTile, (n_out + tm.size - 1) / tm.size);
    if (n_out % 4 == 0 && (reinterpret_cast<uintptr_t>(R.params + L.p_off) & 15) == 0) {
      tw = min(kFcTile, (tw + 3) & ~3);
      v4 = true;
    }
  }
  const int n_tiles = (n_out + tw - 1) / tw;
  if (tm.rank >= n_tiles) return;
  int used = 0;
  const float* x = stage(layer_y(S, act, tm), n_in, tm, used);
  double* red = reinterpret_cast<double*>(tm.smem + used);   // [kFcSlices][kFcTile]
  used += 2 * kFcSlices * kFcTile;
  float* out_a = tm.smem + used;
  used += kFcTile;
  const float* W = R.params + L.p_off;
  const bool wst = used + n_in * tw <= tm.smem_floats;
  float* wt = tm.smem + used;
  for (int tile = tm.rank; tile < n_tiles; tile += tm.size) {
    const int j0 = tile * tw;
    const int nc = min(tw, n_out - j0);
    if (wst && v4) {
      const int q4 = nc >> 2;   // 16-byte pieces per row (j0, n_out multiples of 4)
      for (int e = threadIdx.x; e < n_in * q4; e += blockDim.x) {
        const int i = e / q4, q = e - i * q4;
        cp_async16(wt + i * nc + 4 * q, W + (int64_t)i * n_out + j0 + 4 * q);
      }
    } else if (wst) {
      if (nc == kFcTile) {
        for (int e = threadIdx.x; e < n_in * kFcTile; e += blockDim.x)
          cp_async4(wt + e, W + (e / kFcTile) * n_out + j0 + e % kFcTile);
      } else {
        for (int e = threadIdx.x; e < n_in * nc; e += blockDim.x)
          cp_async4(wt + e, W + (e / nc) * n_out + j0 + e % nc);
      }
    }
    stage_sync();
    fc_cols_preact(x, wst ? wt : W + j0, wst ? nc : n_out, R.params + L.b_off + j0, n_in, nc,
                   red, out_a);
    if (threadIdx.x < nc) {
      const float aj = out_a[threadIdx.x];
      act[L.a_off + j0 + threadIdx.x] = aj;
      act[L.y_off + j0 + threadIdx.x] = fc_act(aj);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void op_zero_delta(const LayerDev& L, float* act, const TeamCtx& tm) {
  float* d = act + L.d_off;
  // a pool over a conv also keeps compact winner deltas (wrc_off > 0 marks it)
  float* wd = L.wrc_off > 0 ? act + L.wd_off : nullptr;
  const Span sp = cta_span(L.cells, tm);
  for (int q = sp.b + threadIdx.x; q < sp.e; q += blockDim.x) {
    d[q] = 0.0f;
    if (wd) wd[q] = 0.0f;
  }
}

// Output deltas (backprop.py:22-32) and the sample loss (backprop.py:35-39):
// run by the first warp of team rank 0; lane 0 ends with ctx.loss.
__device__ __forceinline__ void op_out_delta(const NetGeo& N, const NetPtr& R, const Job& job, Ctx& ctx,
                                             double* scratch) {
  const LayerDev& L = N.L[N.n_layers - 1];
  const int n = L.cells;
  const int lane = lane_id();
  for (int j = lane; j < n; j += 32) {
    const float yj = ctx.act[L.y_off + j];
    const double t = job.targets ? job.targets[j] : (j == ctx.label ? 1.0 : -1.0);
    const double r = (double)yj - t;
    ctx.act[L.d_off + j] = (float)(r * (double)act_deriv(ctx.act[L.a_off + j]));
    scratch[j] = r * r;
  }
  __syncwarp();
  if (lane == 0) ctx.loss = 0.5 * np_pairwise_sum(scratch, n);
  __syncwarp();
}

// FC backward rows (network.py:213-230), one warp per input row i: the row
// of W is read once for xgrad_i = sum_j W[i,j] delta_j (f64) and then
// updated in place with grad_w[i,j] = f32(x_i * delta_j) (or stored).
__device__ __forceinline__ void fc_bwd_rows(const NetGeo& N, const NetPtr& R, const LayerDev& L, int li,
                                           int flags, float eta_f, float* act, const float* x,
                                           const float* dl, const TeamCtx& tm,
                                           bool emit = true) {
  const LayerDev& S = N.L[li - 1];
  float* W = R.params + L.p_off;
  float* b = R.params + L.b_off;
  float* gW = R.grads + L.p_off;
  float* gb = R.grads + L.b_off;
  const int n_in = S.cells, n_out = L.cells;
  const bool upd = flags & F_UPDATE;
  const int lane = lane_id();
  for (int j = tm.gtid; j < n_out; j += tm.gsize) {
    if (upd) b[j] = sgd(b[j], eta_f, dl[j]);
    else gb[j] = dl[j];
  }
  const Span rows = cta_span(n_in, tm);
  for (int i = rows.b + (threadIdx.x >> 5); i < rows.e; i += blockDim.x >> 5) {
    float* row = W + (int64_t)i * n_out;
    double acc = 0.0;
    for (int j = lane; j < n_out; j += 32) acc = fma((double)row[j], (double)dl[j], acc);
    acc = warp_sum(acc);
    const float xi = x[i];
    for (int j = lane; j < n_out; j += 32) {
      const float g = __fmul_rn(xi, dl[j]);
      if (upd) row[j] = sgd(row[j], eta_f, g);
      else gW[(int64_t)i * n_out + j] = g;
    }
    if (emit && lane == 0 && S.has_delta) emit_delta(N, R, act, li - 1, i, (float)acc);
  }
}

__device__ __forceinline__ void op_fc_bwd(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags,
                                          float eta_f, float* act, const TeamCtx& tm) {
  const int li = &L - N.L;
  fc_bwd_rows(N, R, L, li, flags, eta_f, act, layer_y(N.L[li - 1], act, tm), act + L.d_off, tm);
}

// The output layer in one phase: every CTA recomputes the output layer's
// forward (a tiny n_in x n_classes product) and the output deltas in its own
// shared memory, rank 0 publishes a / y / delta and the loss, then all CTAs
// run the FC backward rows.  Replaces three barrier-separated phases.
__device__ __forceinline__ void op_fc_out(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags,
                                          const Job& job, Ctx& ctx, const TeamCtx& tm,
                                          double* scratch) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  float* act = ctx.act;
  int used = 0;
  const float* x = stage(layer_y(S, act, tm), S.cells, tm, used);
  const float* W = stage(R.params + L.p_off, S.cells * L.cells, tm, used, 1 << 14);
  // fused: H's pre-activations too (its f'(a) below), in the same round trip
  const float* ha = (flags & F_FUSE_BELOW) ? stage(act + S.a_off, S.cells, tm, used) : nullptr;
  float* yd = tm.smem + used;                    // [a | y | delta] x n_out (+ H's deltas)
  used += (3 * L.cells + ((flags & F_FUSE_BELOW) ? S.cells : 0) + 3) & ~3;
  double* red = reinterpret_cast<double*>(tm.smem + used);
  stage_sync();
  for (int j0 = 0; j0 < L.cells; j0 += 32) {
    const int nc = min(32, L.cells - j0);
    fc_cols_preact(x, W + j0, L.cells, R.params + L.b_off + j0, S.cells, nc, red, yd + j0);
  }
  for (int j = threadIdx.x; j < L.cells; j += blockDim.x) yd[L.cells + j] = fc_act(yd[j]);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int n = L.cells, lane = lane_id();
    for (int j = lane; j < n; j += 32) {
      const double t = job.targets ? job.targets[j] : (j == ctx.label ? 1.0 : -1.0);
      const double r = (double)yd[n + j] - t;
      yd[2 * n + j] = (float)(r * (double)act_deriv(yd[j]));
      scratch[j] = r * r;
      if (tm.rank == 0) {
        act[L.a_off + j] = yd[j];
        act[L.y_off + j] = yd[n + j];
        act[L.d_off + j] = yd[2 * n + j];
      }
    }
    __syncwarp();
    if (lane == 0 && tm.rank == 0) ctx.loss = 0.5 * np_pairwise_sum(scratch, n);
  }
  __syncthreads();
  if (!(flags & F_FUSE_BELOW)) {
    fc_bwd_rows(N, R, L, li, flags, job.eta_f, act, x, yd + 2 * L.cells, tm);
    __syncthreads();
    return;
  }
  // F_FUSE_BELOW: the FC layer below (H) in the same phase.  Every CTA
  // derives ALL of H's deltas itself -- one warp per row of this layer's W,
  // the same f64 fma chain + xor tree as fc_bwd_rows, so the values equal
  // the unfused ones -- then runs its share of H's backward rows.  This
  // layer's own gradients are stored (its update waits for the next phase:
  // every CTA read its weights above).
  const LayerDev& H = S;
  float* dh = yd + 3 * L.cells;                  // H's deltas, all rows
  {
    // one thread per row of this layer's W: a serial f64 fma chain over the
    // outputs, then f'(a) -- every CTA gets the same bits
    const int n_out = L.cells;
    const float* dl = yd + 2 * n_out;
    for (int i = threadIdx.x; i < H.cells; i += blockDim.x) {
      const float* row = W + i * n_out;
      double acc = 0.0;
      for (int j = 0; j < n_out; ++j) acc = fma((double)row[j], (double)dl[j], acc);
      dh[i] = __fmul_rn((float)acc, act_deriv(ha[i]));
      if (tm.rank == 0) act[H.d_off + i] = dh[i];
    }
  }
  __syncthreads();
  {   // this layer's gradients (stored; its update is the next phase's)
    const float* dl = yd + 2 * L.cells;
    float* gW = R.grads + L.p_off;
    float* gb = R.grads + L.b_off;
    for (int j = tm.gtid; j < L.cells; j += tm.gsize) gb[j] = dl[j];
    const Span rows = cta_span(H.cells, tm);
    for (int e = threadIdx.x; e < (rows.e - rows.b) * L.cells; e += blockDim.x) {
      const int i = rows.b + e / L.cells, j = e % L.cells;
      gW[i * L.cells + j] = __fmul_rn(x[i], dl[j]);
    }
  }
  fc_bwd_rows(N, R, H, li - 1, flags & F_UPDATE, job.eta_f, act, layer_y(N.L[li - 2], act, tm), dh, tm);
  __syncthreads();
}

// ---------------------------------------------------------------------------
// conv backward (network.py:233-252).
//   warp tasks   weight_grad of one connected pair (kernels.py:124-141): lanes
//                split the output cells, kx*ky f64 partials, xor reduction;
//                bias_grad of one dest map (kernels.py:144-151)
//   thread tasks pull_bwd of one source cell (kernels.py:90-121) in the
//                reference's order (dests k, rows y, cols x) with one f64
//                accumulator, routed through emit_delta
// The layer's deltas (and the source activations when they fit) are staged in
// shared memory.  With F_UPDATE (only without F_PULL: the pull reads the old
// weights) the weights are updated in place.
template <int KX, int KY>
__device__ __forceinline__ void wgrad_pair(const NetPtr& R, const LayerDev& L, const LayerDev& S,
                                           int p,
                                           const float* dl, const float* ys, float* arena,
                                           float* g, bool upd, float eta_f) {
  const int lane = lane_id();
  const int hw = L.h * L.w;
  const float* d = dl + t_pair_dst(R, L, (p)) * hw;
  const float* s = ys + t_fwd_src(R, L, (p)) * (S.h * S.w);
  const int o = t_fwd_widx(R, L, (p));
  if constexpr (KX > 0) {
    constexpr int KK = KX * KY;
    double part[KK];
#pragma unroll
    for (int t = 0; t < KK; ++t) part[t] = 0.0;
    for (int cell = lane; cell < hw; cell += 32) {
      const int r = cell / L.w, c = cell % L.w;
      const float dv = d[cell];
      const float* base = s + (r * L.ty) * S.w + c * L.tx;
#pragma unroll
      for (int t = 0; t < KK; ++t) {
        const int v = t / KX, u = t % KX;
        part[t] += (double)__fmul_rn(dv, base[v * S.w + u]);
      }
    }
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      const double sum = warp_sum(part[t]);
      if (lane == t % 32) {
        if (upd) arena[o + t] = sgd(arena[o + t], eta_f, (float)sum);
        else g[o + t] = (float)sum;
      }
    }
  } else {
    const int kk = L.kx * L.ky;
    for (int t = 0; t < kk; ++t) {
      const int v = t / L.kx, u = t % L.kx;
      double part = 0.0;
      for (int cell = lane; cell < hw; cell += 32) {
        const int r = cell / L.w, c = cell % L.w;
        part += (double)__fmul_rn(d[cell], s[(r * L.ty + v) * S.w + c * L.tx + u]);
      }
      const double sum = warp_sum(part);
      if (lane == 0) {
        if (upd) arena[o + t] = sgd(arena[o + t], eta_f, (float)sum);
        else g[o + t] = (float)sum;
      }
    }
  }
}

// Pool-sparse conv backward.  When a max-pool sits on top of the conv layer,
// its deltas are zero everywhere except at the pool winners (network.py:256-
// 261: zeroed buffer, one '+=' per pooled cell), and a zero delta adds an
// exact +0 to the reference's f64 sums.  So weight_grad, bias_grad and
// pull_bwd visit only the winners, read from the compact per-pooled-cell
// arrays the forward pass (winner row/col) and emit_delta (winner delta)
// fill.  Same products, same f64 accumulation; terms that are exactly zero
// are skipped.
//   weight_grad  tasks = (pair, chunk of <= 32 winners); lane = (task group,
//                tap): a lane's serial f64 sum over the chunk's winners for
//                one tap; chunks combined in chunk order
//   bias_grad    one warp per dest map
//   pull_bwd     a scatter per source map into f64 stream buffers (below)
// emit_wg applies a weight-gradient sum (out == nullptr: update in place or
// store the gradient) or parks it in out[t] for the fixed-order combination
// with the pair's other winner chunks.
__device__ __forceinline__ void emit_wg(int o, int t, double sum, double* out, float* arena,
                                        float* g, bool upd, float eta_f) {
  if (out) out[t] = sum;
  else if (upd) arena[o + t] = sgd(arena[o + t], eta_f, (float)sum);
  else g[o + t] = (float)sum;
}

// Pull as a GATHER in the reference's order (kernels.py:90-121): one thread
// per source cell, one f64 accumulator over the backward list (dests k in
// list order) and, per dest, the covering conv cells in row, then column
// order; every term is the f32 product delta * w.  Below a max-pool the conv
// deltas are zero except at the pool winners (a zero term adds an exact +0),
// so per dest only the winners of the pooled cells whose blocks meet the
// covering rectangle [ylo, yhi] x [xlo, xhi] contribute.  Those candidates
// form a small grid (<= PRM pooled rows x PCM pooled cols, fixed per layer);
// all their winner loads are issued together (no dependent branch per
// candidate), and each pooled row's matches are stably sorted by conv row:
// across pooled rows the winners' rows already ascend, inside one the
// columns ascend with the pooled column -- so the adds follow the
// reference's (y, x) order exactly.  Bit-identical to kernels.pull_bwd.
// Every CTA takes a contiguous range of source cells; its backward entries'
// (old) kernels and dest indices are staged, and the winners either of every
// dest map (ed: entry -> dest map slot) or, when that is less, a copy per
// backward entry (ed == nullptr: slot = entry).
template <int PRM, int PCM>
__device__ __forceinline__ void pull_gather_cells(const NetGeo& N, const NetPtr& R,
                                                  const LayerDev& L, float* act, Span cs,
                                                  const int* wr, const float* wdv,
                                                  const float* ws, const int* ed, int ka) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const LayerDev& P = N.L[li + 1];
  const int shw = S.h * S.w, phw = P.h * P.w, kk = L.kx * L.ky;
  // everything staged: 32-bit shared addresses, ld.shared (no generic loads)
  const unsigned wr0 = (unsigned)__cvta_generic_to_shared(wr);
  const unsigned wd0 = (unsigned)__cvta_generic_to_shared(wdv);
  const unsigned ws0 = (unsigned)__cvta_generic_to_shared(ws);
  const unsigned ed0 = ed ? (unsigned)__cvta_generic_to_shared(ed) : 0u;
  for (int cell = cs.b + threadIdx.x; cell < cs.e; cell += blockDim.x) {
    const int s = cell / shw, pix = cell - s * shw;
    const int j = pix / S.w, i = pix - j * S.w;
    const int ylo = ceil_div_clamp0(j - L.ky + 1, L.ty), yhi = min(j / L.ty, L.h - 1);
    const int xlo = ceil_div_clamp0(i - L.kx + 1, L.tx), xhi = min(i / L.tx, L.w - 1);
    const int pr0 = ylo / P.py, pr1 = min(yhi / P.py, P.h - 1);
    const int pc0 = xlo / P.px, pc1 = min(xhi / P.px, P.w - 1);
    double acc = 0.0;
    if (ylo <= yhi && xlo <= xhi && pr0 <= pr1 && pc0 <= pc1) {
      // candidate pooled cells (dest-independent): byte offsets and validity
      unsigned qo[PRM][PCM];
      bool qv[PRM][PCM];
#pragma unroll
      for (int a = 0; a < PRM; ++a)
#pragma unroll
        for (int b = 0; b < PCM; ++b) {
          qv[a][b] = pr0 + a <= pr1 && pc0 + b <= pc1;
          qo[a][b] = 4u * (unsigned)(min(pr0 + a, pr1) * P.w + min(pc0 + b, pc1));
        }
      const int e0 = t_bwd_off(R, L, s), e1 = t_bwd_off(R, L, s + 1);
      const int tap0 = j * L.kx + i;     // tap = tap0 - r*ty*kx - c*tx
#pragma unroll 2
      for (int e = e0; e < e1; ++e) {
        const int slot = ed ? lds_s32(ed0 + 4u * (unsigned)(e - ka)) : e - ka;
        const unsigned wrd = wr0 + 4u * (unsigned)(slot * phw);
        const unsigned wdd = wd0 + 4u * (unsigned)(slot * phw);
        const unsigned wb = ws0 + 4u * (unsigned)((e - ka) * kk);
        int key[PRM][PCM];
        double term[PRM][PCM];
#pragma unroll
        for (int a = 0; a < PRM; ++a)
#pragma unroll
          for (int b = 0; b < PCM; ++b) {
            const int rc = lds_s32(wrd + qo[a][b]);
            const float dv = lds_f32(wdd + qo[a][b]);
            const int r = rc >> 16, c = rc & 0xffff;
            const bool ok = qv[a][b] && r >= ylo && r <= yhi && c >= xlo && c <= xhi;
            const int tap = ok ? tap0 - r * L.ty * L.kx - c * L.tx : 0;
            const float prod = __fmul_rn(dv, lds_f32(wb + 4u * (unsigned)tap));
            key[a][b] = ok ? r : 0x7fffffff;
            term[a][b] = ok ? (double)prod : 0.0;
          }
#pragma unroll
        for (int a = 0; a < PRM; ++a) {
          // stable sort of the pooled row's matches by conv row (bubble network)
#pragma unroll
          for (int pass = 0; pass < PCM - 1; ++pass)
#pragma unroll
            for (int b = 0; b + 1 < PCM - pass; ++b) {
              const bool sw = key[a][b] > key[a][b + 1];
              const int k0 = key[a][b], k1 = key[a][b + 1];
              const double t0 = term[a][b], t1 = term[a][b + 1];
              key[a][b] = sw ? k1 : k0;
              key[a][b + 1] = sw ? k0 : k1;
              term[a][b] = sw ? t1 : t0;
              term[a][b + 1] = sw ? t0 : t1;
            }
#pragma unroll
          for (int b = 0; b < PCM; ++b)
            if (key[a][b] != 0x7fffffff) acc += term[a][b];
        }
      }
    }
    emit_delta(N, R, act, li - 1, cell, (float)acc);
  }
}

// The candidate grid spans at most ceil((ky-1)/ty/py)+1 pooled rows (cols
// likewise); layers beyond 5x5 candidates keep the scatter (host flag).
__device__ __forceinline__ void conv_pull_gather(const NetGeo& N, const NetPtr& R,
                                                 const LayerDev& L, float* act,
                                                 const TeamCtx& tm) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const LayerDev& P = N.L[li + 1];
  const int shw = S.h * S.w, phw = P.h * P.w, kk = L.kx * L.ky;
  const float* arena = R.params + L.p_off;
  const Span cs = cta_span(S.cells, tm);
  if (cs.b >= cs.e) return;                      // uniform per CTA
  CK_SUBT(tm, 16);
  const int nwin = L.maps * phw;
  const int prm = ((L.ky - 1) / L.ty + P.py - 1) / P.py + 1;
  const int pcm = ((L.kx - 1) / L.tx + P.px - 1) / P.px + 1;
  auto run = [&](Span ch, const int* wr, const float* wdv, const float* ws, const int* ed,
                 int ka) {
    if (prm <= 1 && pcm <= 1) pull_gather_cells<1, 1>(N, R, L, act, ch, wr, wdv, ws, ed, ka);
    else if (prm <= 2 && pcm <= 2) pull_gather_cells<2, 2>(N, R, L, act, ch, wr, wdv, ws, ed, ka);
    else if (prm <= 3 && pcm <= 3) pull_gather_cells<3, 3>(N, R, L, act, ch, wr, wdv, ws, ed, ka);
    else pull_gather_cells<5, 5>(N, R, L, act, ch, wr, wdv, ws, ed, ka);
  };
  // sparse tables: the winners of just this CTA's entries' dest maps (a copy
  // per entry) when that stages less than every dest map's and fits at once
  {
    const int ka = t_bwd_off(R, L, cs.b / shw), kb = t_bwd_off(R, L, (cs.e - 1) / shw + 1);
    const int ne = kb - ka, nwe = ((ne * phw + 3) & ~3);
    if (ne * phw < nwin && 2 * nwe + ((ne * kk + 3) & ~3) <= tm.smem_floats) {
      int* wr = reinterpret_cast<int*>(tm.smem);
      float* wdv = tm.smem + nwe;
      float* ws = wdv + nwe;
      const int* wrc_g = reinterpret_cast<const int*>(act + P.wrc_off);
      const float* wd_g = act + P.wd_off;
      for (int i = threadIdx.x; i < ne * phw; i += blockDim.x) {
        const int q = i / phw;
        const int from = t_bwd_dst(R, L, ka + q) * phw + (i - q * phw);
        cp_async4(wr + i, wrc_g + from);
        cp_async4(wdv + i, wd_g + from);
      }
      for (int e = threadIdx.x; e < ne * kk; e += blockDim.x) {
        const int q = e / kk;
        cp_async4(ws + e, arena + t_bwd_widx(R, L, ka + q) + (e - q * kk));
      }
      stage_sync();
      CK_SUBT(tm, 17);
      run(cs, wr, wdv, ws, nullptr, ka);
      CK_SUBT(tm, 18);
      __syncthreads();
      CK_SUBT(tm, 19);
      return;
    }
  }
  // the host sets pullg only when the winners of all dest maps and any CTA's
  // backward-entry kernels fit the scratch (ck_net.cu); chunks of cells keep
  // the kernels' share bounded for wide backward lists
  int used = 0;
  const int* wr = reinterpret_cast<const int*>(
      stage(reinterpret_cast<const float*>(act + P.wrc_off), nwin, tm, used));
  const float* wdv = stage(act + P.wd_off, nwin, tm, used);
  float* ws = tm.smem + used;
  const int cap = tm.smem_floats - used;
  for (int c0 = cs.b; c0 < cs.e;) {
    // cells [c0, c1): whole source maps' backward entries (kernel + dest) must fit
    int c1 = cs.e;
    int m0 = c0 / shw, m1 = (c1 - 1) / shw;
    int ka = t_bwd_off(R, L, m0), kb = t_bwd_off(R, L, m1 + 1);
    while ((kb - ka) * (kk + 1) + 4 > cap && m1 > m0) {
      c1 = m1 * shw;
      m1 = (c1 - 1) / shw;
      kb = t_bwd_off(R, L, m1 + 1);
    }
    if (c0 != cs.b) __syncthreads();             // previous chunk's kernels consumed
    int* ed = reinterpret_cast<int*>(ws + (((kb - ka) * kk + 3) & ~3));
    for (int e = threadIdx.x; e < (kb - ka) * kk; e += blockDim.x) {
      const int q = e / kk;
      cp_async4(ws + e, arena + t_bwd_widx(R, L, ka + q) + (e - q * kk));
    }
    for (int e = threadIdx.x; e < kb - ka; e += blockDim.x) ed[e] = t_bwd_dst(R, L, ka + e);
    stage_sync();
    CK_SUBT(tm, 17);
    run(Span{c0, c1}, wr, wdv, ws, ed, ka);
    c0 = c1;
  }
  CK_SUBT(tm, 18);
  __syncthreads();
  CK_SUBT(tm, 19);
}

// Each CTA stages exactly what its share needs (one cp.async round trip per
// chunk), then computes from shared memory:
//   weight_grad  its pairs [p0, p1): the winners of their dest maps and one
//                copy of each pair's source map, in chunks that fit
//   pull_bwd     its source cells: per backward-list entry (dest d, weight
//                block) the old kernel and d's winners, in chunks of whole
//                source maps
// Anything that does not fit is read in place from global memory.
__device__ __forceinline__ void conv_bwd_sparse(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags, float eta_f,
                                float* act, const TeamCtx& tm) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const LayerDev& P = N.L[li + 1];
  float* arena = R.params + L.p_off;
  float* g = R.grads + L.p_off;
  const bool upd = flags & F_UPDATE;
  const int shw = S.h * S.w, phw = P.h * P.w;
  const int kk = L.kx * L.ky;
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int* wrc_g = reinterpret_cast<const int*>(act + P.wrc_off);
  const float* wd_g = act + P.wd_off;
  const float* ys_g = layer_y(S, act, tm);
  const int cap = tm.smem_floats - 16;
  const int split = L.wg_split;
  CK_SUBT(tm, 10);

  // The pull (below) is the long pole of this phase: with few source maps
  // (one per CTA) those CTAs take no weight-gradient work, which the other
  // ranks share.  Every sum keeps its fixed order, so results do not depend
  // on the split.
  const int npull = ((flags & F_PULL) && !L.pullg && 2 * S.maps <= tm.size) ? S.maps : 0;
  const int wg_ranks = tm.size - npull;

  // ---- weight gradients
  const int n_w = L.n_pairs;
  const Span ts = npull ? sub_span(n_w + L.maps, 0, wg_ranks, tm) : cta_span(n_w + L.maps, tm);
  const int p1 = min(ts.e, n_w);
  for (int c0 = ts.b; c0 < p1;) {
    int c1 = p1, da, db, need;
    for (;;) {
      da = t_pair_dst(R, L, (c0));
      db = t_pair_dst(R, L, (c1 - 1));
      need = 2 * (db - da + 1) * phw + (c1 - c0) * shw + 8 +
             (split > 1 ? 2 * (c1 - c0) * split * kk + 4 : 0);
      if (need <= cap || c1 - c0 == 1) break;
      c1 = c0 + (c1 - c0) / 2;
    }
    const bool fits = need <= cap;
    int used = 0;
    const int* wr = wrc_g + da * phw;
    const float* wdd = wd_g + da * phw;
    float* slots = nullptr;
    if (fits) {
      wr = reinterpret_cast<const int*>(
          stage(reinterpret_cast<const float*>(wr), (db - da + 1) * phw, tm, used));
      wdd = stage(wdd, (db - da + 1) * phw, tm, used);
      slots = tm.smem + used;
      for (int p = c0 + warp; p < c1; p += nwarps) {   // one warp per pair's source map
        const float* from = ys_g + t_fwd_src(R, L, (p)) * shw;
        float* to = slots + (p - c0) * shw;
        for (int i = lane; i < shw; i += 32) cp_async4(to + i, from + i);
      }
    }
    CK_SUBT(tm, 11);
    stage_sync();
    CK_SUBT(tm, 12);
    // task = (pair, winner chunk); chunk partials are combined in chunk order
    double* parts = nullptr;
    if (split > 1) {
      const int after = fits ? used + (c1 - c0) * shw : 0;
      parts = reinterpret_cast<double*>(tm.smem + ((after + 3) & ~3));
    }
    // lane = (group, tap): a warp runs 32/kk tasks side by side, each lane a
    // serial f64 sum over its task's winners for one tap -- no shuffles
    const int ng = kk <= 32 ? 32 / kk : 1;
    const int grp = kk <= 32 ? lane / kk : 0;
    const int n_tasks = (c1 - c0) * split;
    for (int tb = warp * ng; tb < n_tasks; tb += nwarps * ng) {
      const int task = tb + grp;
      if (grp >= ng || task >= n_tasks) continue;
      const int p = c0 + task / split, ch = task % split;
      const int off = (t_pair_dst(R, L, (p)) - da) * phw;
      const float* sp = fits ? slots + (p - c0) * shw : ys_g + t_fwd_src(R, L, (p)) * shw;
      const int o = t_fwd_widx(R, L, (p));
      const int wb = ch * phw / split, we = (ch + 1) * phw / split;
      const int* wrp = wr + off;
      const float* wdp = wdd + off;
      for (int t = (kk <= 32 ? lane % kk : lane); t < kk; t += (kk <= 32 ? kk : 32)) {
        const float* sv = sp + (t / L.kx) * S.w + t % L.kx;
        double part = 0.0;
        if (fits) {   // all staged: 32-bit shared addresses
          const unsigned r0 = (unsigned)__cvta_generic_to_shared(wrp);
          const unsigned d0 = (unsigned)__cvta_generic_to_shared(wdp);
          const unsigned s0 = (unsigned)__cvta_generic_to_shared(sv);
#pragma unroll 4
          for (int wq = wb; wq < we; ++wq) {
            const int rc = lds_s32(r0 + 4u * wq);
            part += (double)__fmul_rn(
                lds_f32(d0 + 4u * wq),
                lds_f32(s0 + 4u * (unsigned)((rc >> 16) * L.ty * S.w + (rc & 0xffff) * L.tx)));
          }
        } else {
#pragma unroll 4
          for (int wq = wb; wq < we; ++wq) {
            const int rc = wrp[wq];
            part += (double)__fmul_rn(wdp[wq], sv[(rc >> 16) * L.ty * S.w + (rc & 0xffff) * L.tx]);
          }
        }
        emit_wg(o, t, part, parts ? parts + task * kk : nullptr, arena, g, upd, eta_f);
      }
    }
    CK_SUBT(tm, 13);
    __syncthreads();
    if (split > 1) {
      for (int e = threadIdx.x; e < (c1 - c0) * kk; e += blockDim.x) {
        const int pi = e / kk, t = e % kk;
        double sum = 0.0;
        for (int ch = 0; ch < split; ++ch) sum += parts[(pi * split + ch) * kk + t];
        emit_wg(t_fwd_widx(R, L, (c0 + pi)), t, sum, nullptr, arena, g, upd, eta_f);
      }
      __syncthreads();
    }
    CK_SUBT(tm, 14);
    c0 = c1;
  }
  // ---- bias gradients: one warp per dest map
  for (int task = max(ts.b, n_w) + warp; task < ts.e; task += nwarps) {
    const int d = task - n_w;
    double acc = 0.0;
    for (int wq = lane; wq < phw; wq += 32) acc += (double)wd_g[d * phw + wq];
    acc = warp_sum(acc);
    if (lane == 0) {
      const int o = t_bias_off(R, L, (d));
      if (upd) arena[o] = sgd(arena[o], eta_f, (float)acc);
      else g[o] = (float)acc;
    }
  }
  CK_SUBT(tm, 15);
  if (!(flags & F_PULL)) {
    __syncthreads();
    return;
  }
  if (L.pullg) {
    __syncthreads();
    conv_pull_gather(N, R, L, act, tm);
    return;
  }

  // ---- pull, as a scatter per source map.  Every (dest entry, winner) adds
  // delta_w * W[d,s,v,u] to source cell (r*ty+v, c*tx+u).  A stream (one lane
  // group of one warp: lane = tap) owns a private f64 buffer of the source
  // map, so the taps of one winner never collide; the layer's pull_ch chunks
  // of the backward list times pull_g lane groups give a fixed set of streams,
  // combined in stream order -- independent of the team.
  const int G = L.pull_g, NCH = L.pull_ch, NS = NCH * G;
  const Span ms = npull ? sub_span(S.maps, wg_ranks, tm.size, tm) : cta_span(S.maps, tm);
  const int per_map = NS * shw * 2;                 // stream buffers (floats)
  for (int m0 = ms.b; m0 < ms.e;) {
    int m1 = min(ms.e, m0 + max(1, nwarps / NCH));
    int ka = t_bwd_off(R, L, (m0)), kb = t_bwd_off(R, L, (m1));
    while (m1 - m0 > 1 && (m1 - m0) * per_map + (kb - ka) * (kk + 2 * phw) > cap) {
      --m1;
      kb = t_bwd_off(R, L, (m1));
    }
    const int bufs = (m1 - m0) * per_map;
    const bool fits = bufs + (kb - ka) * (kk + 2 * phw) <= cap;
    double* buf = reinterpret_cast<double*>(tm.smem);
    float* wst = tm.smem + bufs;
    int* wrs = reinterpret_cast<int*>(wst + (kb - ka) * kk);
    float* wds = wst + (kb - ka) * (kk + phw);
    for (int i = threadIdx.x; i < bufs / 2; i += blockDim.x) buf[i] = 0.0;
    if (fits) {
      for (int k = ka + warp; k < kb; k += nwarps) {   // one warp per backward entry
        const float* wfrom = arena + t_bwd_widx(R, L, (k));
        for (int i = lane; i < kk; i += 32) cp_async4(wst + (k - ka) * kk + i, wfrom + i);
        const int d = t_bwd_dst(R, L, (k));
        for (int i = lane; i < phw; i += 32) {
          cp_async4(wrs + (k - ka) * phw + i, wrc_g + d * phw + i);
          cp_async4(wds + (k - ka) * phw + i, wd_g + d * phw + i);
        }
      }
    }
    CK_SUBT(tm, 16);
    stage_sync();
    CK_SUBT(tm, 17);
    const int grp = kk >= 32 ? 0 : lane / kk;
    for (int task = warp; task < (m1 - m0) * NCH; task += nwarps) {
      const int mi = task / NCH, ch = task % NCH;
      const int k0m = t_bwd_off(R, L, (m0 + mi)), nkm = t_bwd_off(R, L, (m0 + mi + 1)) - k0m;
      const int kc0 = k0m + ch * nkm / NCH, kc1 = k0m + (ch + 1) * nkm / NCH;
      for (int t0 = 0; t0 < kk; t0 += 32) {
        const int t = kk >= 32 ? t0 + lane : lane % kk;
        const bool on = t < kk && grp < G;
        const int v = t / L.kx, u = t % L.kx;
        double* acc = buf + ((mi * NCH + ch) * G + (on ? grp : 0)) * shw + v * S.w + u;
        for (int k = kc0; k < kc1; ++k) {
          const float* wk;
          const int* wr;
          const float* wdd;
          if (fits) {
            wk = wst + (k - ka) * kk;
            wr = wrs + (k - ka) * phw;
            wdd = wds + (k - ka) * phw;
          } else {
            const int d = t_bwd_dst(R, L, (k));
            wk = arena + t_bwd_widx(R, L, (k));
            wr = wrc_g + d * phw;
            wdd = wd_g + d * phw;
          }
          const float wt = on ? wk[t] : 0.0f;
          if (fits) {
            // everything in shared memory: 32-bit shared addresses, no
            // generic loads / stores in the read-modify-write chain
            const unsigned a0 = (unsigned)__cvta_generic_to_shared(acc);
            const unsigned r0 = (unsigned)__cvta_generic_to_shared(wr);
            const unsigned d0 = (unsigned)__cvta_generic_to_shared(wdd);
            for (int q0 = 0; q0 < phw; q0 += G) {
              const int q = q0 + grp;
              if (on && q < phw) {
                const int rc = lds_s32(r0 + 4u * q);
                const unsigned at =
                    a0 + 8u * (unsigned)((rc >> 16) * L.ty * S.w + (rc & 0xffff) * L.tx);
                double v;
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(at) : "memory");
                v += (double)__fmul_rn(lds_f32(d0 + 4u * q), wt);
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(at), "d"(v) : "memory");
              }
              __syncwarp();
            }
            continue;
          }
          for (int q0 = 0; q0 < phw; q0 += G) {   // uniform rounds: group grp takes q0 + grp
            const int q = q0 + grp;
            if (on && q < phw) {
              const int rc = wr[q];
              acc[(rc >> 16) * L.ty * S.w + (rc & 0xffff) * L.tx] +=
                  (double)__fmul_rn(wdd[q], wt);
            }
            __syncwarp();
          }
        }
      }
    }
    CK_SUBT(tm, 18);
    __syncthreads();
    for (int e = threadIdx.x; e < (m1 - m0) * shw; e += blockDim.x) {
      const int mi = e / shw, cell = e % shw;
      const double* b = buf + mi * NS * shw + cell;
      double sum = 0.0;
      for (int st = 0; st < NS; ++st) sum += b[st * shw];
      emit_delta(N, R, act, li - 1, (m0 + mi) * shw + cell, (float)sum);
    }
    __syncthreads();
    CK_SUBT(tm, 19);
    m0 = m1;
  }
}

__device__ __forceinline__ void op_conv_bwd(const NetGeo& N, const NetPtr& R, const LayerDev& L, int flags,
                                            float eta_f, float* act, const TeamCtx& tm) {
  const int li = &L - N.L;
  if (L.pool_above) {
    conv_bwd_sparse(N, R, L, flags, eta_f, act, tm);
    return;
  }
  const LayerDev& S = N.L[li - 1];
  float* arena = R.params + L.p_off;
  float* g = R.grads + L.p_off;
  const bool upd = flags & F_UPDATE;
  const int hw = L.h * L.w, shw = S.h * S.w;
  const int lane = lane_id();
  int used = 0;
  const float* dl = stage(act + L.d_off, L.cells, tm, used);
  const float* ys = stage(layer_y(S, act, tm), S.cells, tm, used);
  stage_sync();
  const int n_w = L.n_pairs;
  const int total = n_w + L.maps;
  const Span ts = cta_span(total, tm);
  for (int task = ts.b + (threadIdx.x >> 5); task < ts.e; task += blockDim.x >> 5) {
    if (task < n_w) {
      if (L.kx == 2 && L.ky == 2) wgrad_pair<2, 2>(R, L, S, task, dl, ys, arena, g, upd, eta_f);
      else if (L.kx == 3 && L.ky == 3) wgrad_pair<3, 3>(R, L, S, task, dl, ys, arena, g, upd, eta_f);
      else if (L.kx == 4 && L.ky == 4) wgrad_pair<4, 4>(R, L, S, task, dl, ys, arena, g, upd, eta_f);
      else if (L.kx == 5 && L.ky == 5) wgrad_pair<5, 5>(R, L, S, task, dl, ys, arena, g, upd, eta_f);
      else wgrad_pair<0, 0>(R, L, S, task, dl, ys, arena, g, upd, eta_f);
    } else {
      const int d = task - n_w;
      const float* dd = dl + d * hw;
      double acc = 0.0;
      for (int i = lane; i < hw; i += 32) acc += (double)dd[i];
      acc = warp_sum(acc);
      if (lane == 0) {
        const int o = t_bias_off(R, L, (d));
        if (upd) arena[o] = sgd(arena[o], eta_f, (float)acc);
        else g[o] = (float)acc;
      }
    }
  }
  if (flags & F_PULL) {
    const Span cs = cta_span(S.cells, tm);
    for (int cell = cs.b + threadIdx.x; cell < cs.e; cell += blockDim.x) {
      const int s = cell / shw, pix = cell % shw;
      const int j = pix / S.w, i = pix % S.w;
      const int ylo = ceil_div_clamp0(j - L.ky + 1, L.ty);
      const int yhi = min(j / L.ty, L.h - 1);
      const int xlo = ceil_div_clamp0(i - L.kx + 1, L.tx);
      const int xhi = min(i / L.tx, L.w - 1);
      // four interleaved accumulators over the destination list (fixed
      // combination order), so the f64 adds overlap
      // The covering window (ylo..yhi, xlo..xhi) depends only on the source
      // cell, so four destinations share one loop nest: accumulator q takes
      // the destinations k = kb + q (mod 4), combined in fixed order.
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const int kb = t_bwd_off(R, L, (s)), k1 = t_bwd_off(R, L, (s + 1));
      const int dw0 = (j - ylo * L.ty) * L.kx + i - xlo * L.tx;   // weight index at (ylo, xlo)
      int k = kb;
      for (; k + 4 <= k1; k += 4) {
        const float* d0 = dl + t_bwd_dst(R, L, (k)) * hw + ylo * L.w;
        const float* d1 = dl + t_bwd_dst(R, L, (k + 1)) * hw + ylo * L.w;
        const float* d2 = dl + t_bwd_dst(R, L, (k + 2)) * hw + ylo * L.w;
        const float* d3 = dl + t_bwd_dst(R, L, (k + 3)) * hw + ylo * L.w;
        const float* w0 = arena + t_bwd_widx(R, L, (k)) + dw0;
        const float* w1 = arena + t_bwd_widx(R, L, (k + 1)) + dw0;
        const float* w2 = arena + t_bwd_widx(R, L, (k + 2)) + dw0;
        const float* w3 = arena + t_bwd_widx(R, L, (k + 3)) + dw0;
        for (int y = ylo; y <= yhi; ++y) {
          for (int x = xlo, wi = 0; x <= xhi; ++x, wi -= L.tx) {
            acc[0] += (double)__fmul_rn(d0[x], w0[wi]);
            acc[1] += (double)__fmul_rn(d1[x], w1[wi]);
            acc[2] += (double)__fmul_rn(d2[x], w2[wi]);
            acc[3] += (double)__fmul_rn(d3[x], w3[wi]);
          }
          d0 += L.w; d1 += L.w; d2 += L.w; d3 += L.w;
          w0 -= L.ty * L.kx; w1 -= L.ty * L.kx; w2 -= L.ty * L.kx; w3 -= L.ty * L.kx;
        }
      }
      for (; k < k1; ++k) {
        const float* d = dl + t_bwd_dst(R, L, (k)) * hw + ylo * L.w;
        const float* w = arena + t_bwd_widx(R, L, (k)) + dw0;
        double part = 0.0;
        for (int y = ylo; y <= yhi; ++y, d += L.w, w -= L.ty * L.kx)
          for (int x = xlo, wi = 0; x <= xhi; ++x, wi -= L.tx)
            part += (double)__fmul_rn(d[x], w[wi]);
        switch ((k - kb) & 3) {
          case 0: acc[0] += part; break;
          case 1: acc[1] += part; break;
          case 2: acc[2] += part; break;
          default: acc[3] += part; break;
        }
      }
      emit_delta(N, R, act, li - 1, cell, (float)((acc[0] + acc[1]) + (acc[2] + acc[3])));
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void op_update(const NetGeo& N, const NetPtr& R, const LayerDev& L, float eta_f,
                                          const TeamCtx& tm) {
  float* p = R.params + L.p_off;
  const float* g = R.grads + L.p_off;
  const Span sp = cta_span(L.n_par, tm);
  for (int q = sp.b + threadIdx.x; q < sp.e; q += blockDim.x) p[q] = sgd(p[q], eta_f, g[q]);
}

__device__ __forceinline__ void run_op(const NetGeo& N, const NetPtr& R, const Op op,
                                       const Job& job, Ctx& ctx, const TeamCtx& tm,
                                       double* scratch) {
  const LayerDev& L = N.L[op.layer];
  switch (op.kind) {
    case OP_LOAD_INPUT: op_load_input(N, R, job, ctx, tm); break;
    case OP_IMGPROC: op_imgproc(N, R, L, ctx.act, tm); break;
    case OP_CONV_FWD: op_conv_fwd(N, R, L, op.flags, ctx.act, tm); break;
    case OP_CONV_POOL: op_conv_pool(N, R, L, op.flags, job.full != 0, ctx.act, tm); break;
    case OP_POOL_FWD: op_pool_fwd(N, R, L, ctx.act, tm); break;
    case OP_FC_FWD: op_fc_fwd(N, R, L, ctx.act, tm); break;
    case OP_ZERO_DELTA: op_zero_delta(L, ctx.act, tm); break;
    case OP_OUT_DELTA:
      if (tm.rank == 0 && threadIdx.x < 32) op_out_delta(N, R, job, ctx, scratch);
      break;
    case OP_FC_BWD: op_fc_bwd(N, R, L, op.flags, job.eta_f, ctx.act, tm); break;
    case OP_FC_OUT: op_fc_out(N, R, L, op.flags, job, ctx, tm, scratch); break;
    case OP_CONV_BWD: op_conv_bwd(N, R, L, op.flags, job.eta_f, ctx.act, tm); break;
    case OP_UPDATE: op_update(N, R, L, job.eta_f, tm); break;
    default: break;
  }
}

// Runs the ops of one phase for this thread's share of the team.  Every
// thread of every CTA calls this (ops may __syncthreads internally).
__device__ __forceinline__ void run_phase(const NetGeo& N, const NetPtr& R, const Program& P, int ph,
                                          const Job& job, Ctx& ctx, const TeamCtx& tm,
                                          double* scratch) {
  for (int o = P.begin[ph]; o < P.begin[ph + 1]; ++o) run_op(N, R, P.ops[o], job, ctx, tm, scratch);
}

}  // namespace ck
