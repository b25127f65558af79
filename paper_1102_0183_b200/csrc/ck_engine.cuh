// ck_engine.cuh — device data model and phase ops of the network engine.
//
// A net lives entirely on the device:
//   params  f32, NetworkState.parameters() order (conv arenas with the
//           reference's tiling topology.py:82-96, FC W (n_in,n_out), FC b)
//   grads   f32, same layout (backward() / apply_gradients() split mode)
//   act     per layer y / a / delta (f32, dense (maps,h,w), no pitch) and pool
//           argmax (int32 flat source index), 128-byte aligned
//   tables  int32 copies of the ConnectionTable CSR arrays
//
// One online step is a PROGRAM: a list of phases, each a list of ops that may
// run concurrently; phases are separated by a team barrier.  A team is the
// set of CTAs working on one net (a thread-block cluster, a cooperative grid
// or a single CTA for batched evaluation).  All ops distribute their work
// over the team's threads (gtid, gsize) and never need a barrier inside.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ck_numerics.cuh"

namespace ck {

constexpr int kMaxLayers = 24;
constexpr int kMaxOps = 80;
constexpr int kMaxPhases = 56;

enum LayerKind { L_INPUT = 0, L_IMGPROC = 1, L_CONV = 2, L_POOL = 3, L_FC = 4 };

struct LayerDev {
  int kind;
  int maps, h, w, cells;           // output geometry
  int src_maps, src_h, src_w, src_cells;
  int kx, ky, tx, ty;              // conv (tx = sx + 1)
  int px, py;                      // pool
  int n_pairs;
  int has_delta;
  int n_filt, fh, fw;              // imgproc
  int64_t p_off, b_off, n_par;     // params: conv arena / FC W, FC bias, count
  int64_t y_off, a_off, d_off, arg_off;  // act arena offsets (elements)
  const int* fwd_off;              // conv tables (device, int32)
  const int* fwd_src;
  const int* fwd_widx;
  const int* bias_off;
  const int* bwd_off;
  const int* bwd_dst;
  const int* bwd_widx;
  const int* pair_dst;
  const double* filt;              // imgproc coefficients (n_filt, fh, fw)
};

enum OpKind {
  OP_LOAD_INPUT = 0,  // input y <- lut[image bytes] (no-op for host-staged x)
  OP_IMGPROC,         // contrast layer
  OP_CONV_FWD,        // conv a, y (+ zero own delta when aux & 1)
  OP_POOL_FWD,        // max-pool y + argmax
  OP_FC_FWD,          // a = x@W + b, y = act(a)
  OP_ZERO_DELTA,      // delta <- 0 (scatter target of the pool above)
  OP_OUT_DELTA,       // output deltas + sample loss
  OP_FC_BWD,          // xgrad, W/b update (or grads), delta below
  OP_CONV_BWD,        // weight/bias grads (+ update) and pulled delta below
  OP_UPDATE,          // params[p_off, +n_par) -= eta * grads
};

enum OpFlags { F_UPDATE = 1, F_PULL = 2, F_ZERO_SELF = 4 };

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

enum ProgId { PROG_TRAIN = 0, PROG_FORWARD = 1, PROG_BACKWARD = 2, PROG_APPLY = 3,
              PROG_EVAL = 4, N_PROGS = 5 };

struct NetDev {
  int n_layers;
  int n_classes;
  int in_cells;
  int pad0;
  float* params;
  float* grads;
  float* act;
  int64_t act_size;        // elements per act arena (one team)
  unsigned* bar;           // grid-team barrier words (count, generation)
  LayerDev L[kMaxLayers];
  Program prog[N_PROGS];
};

// Per-launch job description (passed by value).
struct Job {
  int prog;
  int n_nets;
  const uint8_t* images;   // (N, C, H, W) bytes, or null for host-staged input
  const float* lut;        // null: `images` holds float32 (N, C, H, W)
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
};

struct Ctx {
  float* act;
  int64_t img;             // dataset index of the current image
  int64_t t;               // position in the visit sequence
  int label;
  double loss;             // written by OP_OUT_DELTA (valid in its thread)
};

// ---------------------------------------------------------------------------
// delta routing: `v` is the gathered (pre-derivative) delta of cell `cell` in
// layer `s` — the value the reference stores before `*= f'(a)`.  Pools store
// it and pass it on to their recorded winner (network.py:253-259: zeroed
// buffer, `+=`, so the winner holds 0 + v); conv / FC multiply by f'(a)
// (network.py:222,227-228,260-261).
__device__ __forceinline__ void emit_delta(const NetDev& N, float* act, int s,
                                           int cell, float v) {
  for (;;) {
    const LayerDev& L = N.L[s];
    if (L.kind == L_POOL) {
      act[L.d_off + cell] = v;
      if (!N.L[s - 1].has_delta) return;
      cell = reinterpret_cast<const int*>(act + L.arg_off)[cell];
      v = __fadd_rn(0.0f, v);
      --s;
      continue;
    }
    if (L.kind == L_CONV || L.kind == L_FC)
      act[L.d_off + cell] = __fmul_rn(v, act_deriv(act[L.a_off + cell]));
    return;
  }
}

// ---------------------------------------------------------------------------
// ops

__device__ __forceinline__ void op_load_input(const NetDev& N, const Job& job,
                                              const Ctx& ctx, int gtid, int gsize) {
  if (!job.images) return;
  float* y = ctx.act + N.L[0].y_off;
  if (job.lut) {
    const uint8_t* img = job.images + ctx.img * (int64_t)N.in_cells;
    for (int i = gtid; i < N.in_cells; i += gsize) y[i] = job.lut[img[i]];
  } else {  // float32 dataset
    const float* img = reinterpret_cast<const float*>(job.images) + ctx.img * (int64_t)N.in_cells;
    for (int i = gtid; i < N.in_cells; i += gsize) y[i] = img[i];
  }
}

__device__ __forceinline__ void op_imgproc(const NetDev& N, const LayerDev& L,
                                           float* act, int gtid, int gsize) {
  const LayerDev& I = N.L[0];
  const float* src = act + I.y_off;
  float* out = act + L.y_off;
  const int hw = L.h * L.w;
  const int C = I.maps;
  const int cy = L.fh / 2, cx = L.fw / 2;
  for (int q = gtid; q < L.cells; q += gsize) {
    const int o = q / hw, pix = q % hw;
    if (o < C) { out[q] = src[q]; continue; }
    const int y = pix / L.w, x = pix % L.w;
    const int f = (o - C) / C, c = (o - C) % C;
    const float* s = src + c * hw;
    const double* k = L.filt + (int64_t)f * L.fh * L.fw;
    double acc = 0.0;
    for (int i = 0; i < L.fh; ++i) {
      const float* row = s + min(max(y + i - cy, 0), L.h - 1) * L.w;
      for (int j = 0; j < L.fw; ++j)
        acc = __dadd_rn(acc, __dmul_rn(k[i * L.fw + j], (double)row[min(max(x + j - cx, 0), L.w - 1)]));
    }
    out[q] = (float)acc;
  }
}

__device__ __forceinline__ void op_conv_fwd(const NetDev& N, const LayerDev& L, int flags,
                                            float* act, int gtid, int gsize) {
  const LayerDev& S = N.L[&L - N.L - 1];
  const float* src = act + S.y_off;
  const float* arena = N.params + L.p_off;
  float* a = act + L.a_off;
  float* y = act + L.y_off;
  float* dl = act + L.d_off;
  const int hw = L.h * L.w;
  const int shw = S.h * S.w;
  const int kx = L.kx, ky = L.ky;
  for (int q = gtid; q < L.cells; q += gsize) {
    const int d = q / hw, pix = q % hw;
    const int r = pix / L.w, c = pix % L.w;
    float acc = arena[L.bias_off[d]];
    const int k1 = L.fwd_off[d + 1];
    for (int k = L.fwd_off[d]; k < k1; ++k) {
      const float* s = src + L.fwd_src[k] * shw + (r * L.ty) * S.w + c * L.tx;
      const float* w = arena + L.fwd_widx[k];
      for (int v = 0; v < ky; ++v)
        for (int u = 0; u < kx; ++u)
          acc = __fadd_rn(acc, __fmul_rn(w[v * kx + u], s[v * S.w + u]));
    }
    a[q] = acc;
    y[q] = conv_act(acc);
    if (flags & F_ZERO_SELF) dl[q] = 0.0f;
  }
}

__device__ __forceinline__ void op_pool_fwd(const NetDev& N, const LayerDev& L,
                                            float* act, int gtid, int gsize) {
  const LayerDev& S = N.L[&L - N.L - 1];
  const float* src = act + S.y_off;
  float* y = act + L.y_off;
  int* arg = reinterpret_cast<int*>(act + L.arg_off);
  const int hw = L.h * L.w;
  const int shw = S.h * S.w;
  for (int q = gtid; q < L.cells; q += gsize) {
    const int m = q / hw, pix = q % hw;
    const int r = pix / L.w, c = pix % L.w;
    const float* s = src + m * shw;
    int best_i = (r * L.py) * S.w + c * L.px;
    float best = s[best_i];
    for (int v = 0; v < L.py; ++v)
      for (int u = 0; u < L.px; ++u) {
        const int i = (r * L.py + v) * S.w + c * L.px + u;
        const float val = s[i];
        if (val > best) { best = val; best_i = i; }
      }
    y[q] = best;
    arg[q] = best_i;
  }
}

__device__ __forceinline__ void op_fc_fwd(const NetDev& N, const LayerDev& L,
                                          float* act, int gtid, int gsize) {
  const LayerDev& S = N.L[&L - N.L - 1];
  const float* x = act + S.y_off;
  const float* W = N.params + L.p_off;
  const float* b = N.params + L.b_off;
  const int n_in = S.cells, n_out = L.cells;
  for (int j = gtid; j < n_out; j += gsize) {
    double acc = 0.0;
    for (int i = 0; i < n_in; ++i)
      acc = fma((double)x[i], (double)W[(int64_t)i * n_out + j], acc);
    const float aj = __fadd_rn((float)acc, b[j]);
    act[L.a_off + j] = aj;
    act[L.y_off + j] = fc_act(aj);
  }
}

__device__ __forceinline__ void op_zero_delta(const LayerDev& L, float* act, int gtid,
                                              int gsize) {
  float* d = act + L.d_off;
  for (int q = gtid; q < L.cells; q += gsize) d[q] = 0.0f;
}

// Output deltas (backprop.py:22-32) and the sample loss (backprop.py:35-39):
// run by the first warp of team rank 0; lane 0 ends with ctx.loss.
__device__ __forceinline__ void op_out_delta(const NetDev& N, const Job& job, Ctx& ctx,
                                             double* scratch) {
  const LayerDev& L = N.L[N.n_layers - 1];
  const int n = L.cells;
  const int lane = threadIdx.x & 31;
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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// FC backward, one warp per input row i (network.py:213-230): the row of W
// is read once for xgrad_i = sum_j W[i,j] delta_j and then updated in place
// with grad_w[i,j] = f32(x_i * delta_j) (or stored as a gradient).
__device__ __forceinline__ void op_fc_bwd(const NetDev& N, const LayerDev& L, int flags,
                                          float eta_f, float* act, int gtid, int gsize) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const float* x = act + S.y_off;
  const float* dl = act + L.d_off;
  float* W = N.params + L.p_off;
  float* b = N.params + L.b_off;
  float* gW = N.grads + L.p_off;
  float* gb = N.grads + L.b_off;
  const int n_in = S.cells, n_out = L.cells;
  const bool upd = flags & F_UPDATE;
  const int lane = gtid & 31;
  for (int j = gtid; j < n_out; j += gsize) {
    if (upd) b[j] = sgd(b[j], eta_f, dl[j]);
    else gb[j] = dl[j];
  }
  for (int i = gtid >> 5; i < n_in; i += gsize >> 5) {
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
    if (lane == 0 && S.has_delta) emit_delta(N, act, li - 1, i, (float)acc);
  }
}

// Conv backward (network.py:233-252): weight_grad (kernels.py:124-141),
// bias_grad (kernels.py:144-151) and, when the layer below keeps deltas,
// pull_bwd (kernels.py:90-121) routed through emit_delta.  With F_UPDATE the
// weights are updated in place (legal only without F_PULL: pull reads them).
__device__ __forceinline__ void op_conv_bwd(const NetDev& N, const LayerDev& L, int flags,
                                            float eta_f, float* act, int gtid, int gsize) {
  const int li = &L - N.L;
  const LayerDev& S = N.L[li - 1];
  const float* dl = act + L.d_off;
  const float* ys = act + S.y_off;
  float* arena = N.params + L.p_off;
  float* g = N.grads + L.p_off;
  const bool upd = flags & F_UPDATE;
  const int kk = L.kx * L.ky;
  const int hw = L.h * L.w, shw = S.h * S.w;
  const int n_w = L.n_pairs * kk;
  const int n_b = L.maps;
  const int n_p = (flags & F_PULL) ? S.cells : 0;
  const int total = n_w + n_b + n_p;
  for (int q = gtid; q < total; q += gsize) {
    if (q < n_w) {
      const int p = q / kk, vu = q % kk;
      const int v = vu / L.kx, u = vu % L.kx;
      const float* d = dl + L.pair_dst[p] * hw;
      const float* s = ys + L.fwd_src[p] * shw + v * S.w + u;
      double acc = 0.0;
      for (int r = 0; r < L.h; ++r) {
        const float* srow = s + r * L.ty * S.w;
        const float* drow = d + r * L.w;
        for (int c = 0; c < L.w; ++c)
          acc = __dadd_rn(acc, (double)__fmul_rn(drow[c], srow[c * L.tx]));
      }
      const int o = L.fwd_widx[p] + vu;
      if (upd) arena[o] = sgd(arena[o], eta_f, (float)acc);
      else g[o] = (float)acc;
    } else if (q < n_w + n_b) {
      const int d = q - n_w;
      const float* dd = dl + d * hw;
      double acc = 0.0;
      for (int i = 0; i < hw; ++i) acc = __dadd_rn(acc, (double)dd[i]);
      const int o = L.bias_off[d];
      if (upd) arena[o] = sgd(arena[o], eta_f, (float)acc);
      else g[o] = (float)acc;
    } else {
      const int cell = q - n_w - n_b;
      const int s = cell / shw, pix = cell % shw;
      const int j = pix / S.w, i = pix % S.w;
      const int ylo = ceil_div_clamp0(j - L.ky + 1, L.ty);
      const int yhi = min(j / L.ty, L.h - 1);
      const int xlo = ceil_div_clamp0(i - L.kx + 1, L.tx);
      const int xhi = min(i / L.tx, L.w - 1);
      double acc = 0.0;
      const int k1 = L.bwd_off[s + 1];
      for (int k = L.bwd_off[s]; k < k1; ++k) {
        const float* d = dl + L.bwd_dst[k] * hw;
        const float* w = arena + L.bwd_widx[k];
        for (int y = ylo; y <= yhi; ++y) {
          const float* wrow = w + (j - y * L.ty) * L.kx + i;
          const float* drow = d + y * L.w;
          for (int x = xlo; x <= xhi; ++x)
            acc = __dadd_rn(acc, (double)__fmul_rn(drow[x], wrow[-x * L.tx]));
        }
      }
      emit_delta(N, act, li - 1, cell, (float)acc);
    }
  }
}

__device__ __forceinline__ void op_update(const NetDev& N, const LayerDev& L, float eta_f,
                                          int gtid, int gsize) {
  float* p = N.params + L.p_off;
  const float* g = N.grads + L.p_off;
  for (int64_t q = gtid; q < L.n_par; q += gsize) p[q] = sgd(p[q], eta_f, g[q]);
}

// Runs the ops of one phase for this thread's share of the team.
__device__ __forceinline__ void run_phase(const NetDev& N, const Program& P, int ph,
                                          const Job& job, Ctx& ctx, int team_rank,
                                          int gtid, int gsize, double* scratch) {
  for (int o = P.begin[ph]; o < P.begin[ph + 1]; ++o) {
    const Op op = P.ops[o];
    const LayerDev& L = N.L[op.layer];
    switch (op.kind) {
      case OP_LOAD_INPUT: op_load_input(N, job, ctx, gtid, gsize); break;
      case OP_IMGPROC: op_imgproc(N, L, ctx.act, gtid, gsize); break;
      case OP_CONV_FWD: op_conv_fwd(N, L, op.flags, ctx.act, gtid, gsize); break;
      case OP_POOL_FWD: op_pool_fwd(N, L, ctx.act, gtid, gsize); break;
      case OP_FC_FWD: op_fc_fwd(N, L, ctx.act, gtid, gsize); break;
      case OP_ZERO_DELTA: op_zero_delta(L, ctx.act, gtid, gsize); break;
      case OP_OUT_DELTA:
        if (team_rank == 0 && threadIdx.x < 32) op_out_delta(N, job, ctx, scratch);
        break;
      case OP_FC_BWD: op_fc_bwd(N, L, op.flags, job.eta_f, ctx.act, gtid, gsize); break;
      case OP_CONV_BWD: op_conv_bwd(N, L, op.flags, job.eta_f, ctx.act, gtid, gsize); break;
      case OP_UPDATE: op_update(N, L, job.eta_f, gtid, gsize); break;
      default: break;
    }
  }
}

}  // namespace ck
