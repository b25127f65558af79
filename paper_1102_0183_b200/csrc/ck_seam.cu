// ck_seam.cu — the operator seam: one CUDA kernel per reference kernel of
// convkit.kernels (kernels.py:70-180) plus the contrast layer, each with the
// reference's argument meaning over caller-owned, pitched device buffers.
//
// Every output cell has exactly one writer (the reference's race-freedom
// rule, kernels.py:1-11), so results do not depend on the launch shape.
// These kernels serve single-layer calls through the Python seam
// (paper_1102_0183_b200.kernels); the training hot path is the fused
// persistent kernel in ck_net.cu, which reuses the same arithmetic.
#include <stdio.h>

#include <mutex>

#include "ck_host.h"
#include "ck_numerics.cuh"

namespace ck {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" +
                 cudaGetErrorString(e) + ")";
  return e == cudaErrorMemoryAllocation ? CK_E_NOMEM : CK_E_CUDA;
}

void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// -------------------------------------------------------------------------
// conv_fwd (kernels.py:70-87): one thread per output cell, reference order.
__global__ void seam_conv_fwd(const float* __restrict__ src, int64_t src_map,
                              int src_pitch, const float* __restrict__ arena,
                              const int64_t* __restrict__ fwd_off,
                              const int64_t* __restrict__ fwd_src,
                              const int64_t* __restrict__ fwd_widx,
                              const int64_t* __restrict__ bias_off, int kx,
                              int ky, int tx, int ty, float* a_out, float* y_out,
                              int n_dest, int64_t out_map, int out_pitch,
                              int out_w, int out_h) {
  const int64_t cells = (int64_t)n_dest * out_h * out_w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % out_w);
    const int r = (int)((i / out_w) % out_h);
    const int d = (int)(i / ((int64_t)out_w * out_h));
    float acc = arena[bias_off[d]];
    for (int64_t k = fwd_off[d]; k < fwd_off[d + 1]; ++k) {
      const float* s = src + fwd_src[k] * src_map;
      const float* w = arena + fwd_widx[k];
      for (int v = 0; v < ky; ++v) {
        const float* row = s + (int64_t)(r * ty + v) * src_pitch + c * tx;
        for (int u = 0; u < kx; ++u) acc = __fadd_rn(acc, __fmul_rn(w[v * kx + u], row[u]));
      }
    }
    const int64_t o = d * out_map + (int64_t)r * out_pitch + c;
    a_out[o] = acc;
    y_out[o] = conv_act(acc);
  }
}

// pull_bwd (kernels.py:90-121): gather per source cell.
__global__ void seam_pull_bwd(const float* __restrict__ dn, int64_t dn_map,
                              int dn_pitch, int dest_w, int dest_h,
                              const float* __restrict__ arena,
                              const int64_t* __restrict__ bwd_off,
                              const int64_t* __restrict__ bwd_dst,
                              const int64_t* __restrict__ bwd_widx, int kx,
                              int ky, int tx, int ty, float* out, int n_src,
                              int64_t out_map, int out_pitch, int src_w,
                              int src_h) {
  const int64_t cells = (int64_t)n_src * src_h * src_w;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cells;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % src_w);
    const int j = (int)((q / src_w) % src_h);
    const int s = (int)(q / ((int64_t)src_w * src_h));
    const int ylo = ceil_div_clamp0(j - ky + 1, ty);
    const int yhi = min(j / ty, dest_h - 1);
    const int xlo = ceil_div_clamp0(i - kx + 1, tx);
    const int xhi = min(i / tx, dest_w - 1);
    double acc = 0.0;
    for (int64_t k = bwd_off[s]; k < bwd_off[s + 1]; ++k) {
      const float* d = dn + bwd_dst[k] * dn_map;
      const int64_t off = bwd_widx[k];
      for (int y = ylo; y <= yhi; ++y) {
        const float* wrow = arena + off + (int64_t)(j - y * ty) * kx;
        for (int x = xlo; x <= xhi; ++x)
          acc = __dadd_rn(acc, (double)__fmul_rn(d[(int64_t)y * dn_pitch + x], wrow[i - x * tx]));
      }
    }
    out[s * out_map + (int64_t)j * out_pitch + i] = (float)acc;
  }
}

// weight_grad (kernels.py:124-141): one thread per (pair, v, u).
__global__ void seam_weight_grad(const float* __restrict__ dn, int64_t dn_map,
                                 int dn_pitch, int dest_w, int dest_h,
                                 const float* __restrict__ yp, int64_t yp_map,
                                 int yp_pitch, const int64_t* __restrict__ pdst,
                                 const int64_t* __restrict__ psrc,
                                 const int64_t* __restrict__ poff, int n_pairs,
                                 int kx, int ky, int tx, int ty, float* g) {
  const int kk = kx * ky;
  const int64_t items = (int64_t)n_pairs * kk;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < items;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(q / kk);
    const int vu = (int)(q % kk);
    const int v = vu / kx, u = vu % kx;
    const float* d = dn + pdst[p] * dn_map;
    const float* s = yp + psrc[p] * yp_map;
    double acc = 0.0;
    for (int r = 0; r < dest_h; ++r) {
      const float* drow = d + (int64_t)r * dn_pitch;
      const float* srow = s + (int64_t)(r * ty + v) * yp_pitch + u;
      for (int c = 0; c < dest_w; ++c)
        acc = __dadd_rn(acc, (double)__fmul_rn(drow[c], srow[c * tx]));
    }
    g[poff[p] + vu] = (float)acc;
  }
}

// bias_grad (kernels.py:144-151): one warp per destination map; lanes take
// whole rows so the f64 partial sums combine in a fixed order.
__global__ void seam_bias_grad(const float* __restrict__ dn, int64_t dn_map,
                               int dn_pitch, int dest_w, int dest_h, int n_dest,
                               const int64_t* __restrict__ bias_off, float* g) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_dest) return;
  const float* d = dn + warp * dn_map;
  double acc = 0.0;
  if (lane == 0) {
    for (int r = 0; r < dest_h; ++r)
      for (int c = 0; c < dest_w; ++c)
        acc = __dadd_rn(acc, (double)d[(int64_t)r * dn_pitch + c]);
    g[bias_off[warp]] = (float)acc;
  }
}

// maxpool_fwd (kernels.py:154-172).
__global__ void seam_maxpool_fwd(const float* __restrict__ src, int64_t src_map,
                                 int src_pitch, int px, int py, float* out,
                                 int64_t out_map, int out_pitch, int out_w,
                                 int out_h, int n_maps, int64_t* arg_r,
                                 int64_t* arg_c) {
  const int64_t cells = (int64_t)n_maps * out_h * out_w;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cells;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q % out_w);
    const int r = (int)((q / out_w) % out_h);
    const int m = (int)(q / ((int64_t)out_w * out_h));
    const float* s = src + m * src_map;
    int br = r * py, bc = c * px;
    float best = s[(int64_t)br * src_pitch + bc];
    for (int v = 0; v < py; ++v)
      for (int u = 0; u < px; ++u) {
        const float val = s[(int64_t)(r * py + v) * src_pitch + c * px + u];
        if (val > best) { best = val; br = r * py + v; bc = c * px + u; }
      }
    out[m * out_map + (int64_t)r * out_pitch + c] = best;
    arg_r[q] = br;
    arg_c[q] = bc;
  }
}

// maxpool_bwd (kernels.py:175-180): += into the recorded winner.
__global__ void seam_maxpool_bwd(const float* __restrict__ dn, int64_t dn_map,
                                 int dn_pitch, int out_w, int out_h, int n_maps,
                                 const int64_t* __restrict__ arg_r,
                                 const int64_t* __restrict__ arg_c, float* dp,
                                 int64_t dp_map, int dp_pitch) {
  const int64_t cells = (int64_t)n_maps * out_h * out_w;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cells;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q % out_w);
    const int r = (int)((q / out_w) % out_h);
    const int m = (int)(q / ((int64_t)out_w * out_h));
    float* cell = dp + m * dp_map + arg_r[q] * dp_pitch + arg_c[q];
    *cell = __fadd_rn(*cell, dn[m * dn_map + (int64_t)r * dn_pitch + c]);
  }
}

// contrast layer (filters.py:168-172): correlate, mode="nearest".
__global__ void seam_contrast(const float* __restrict__ src, int n_ch,
                              int64_t src_map, int pitch, int w, int h,
                              const double* __restrict__ coeffs, int n_filters,
                              int fh, int fw, float* out, int64_t out_map,
                              int out_pitch) {
  const int64_t cells = (int64_t)n_filters * n_ch * h * w;
  const int cy = fh / 2, cx = fw / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cells;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(q % w);
    const int y = (int)((q / w) % h);
    const int fc = (int)(q / ((int64_t)w * h));  // filter-major, then channel
    const int f = fc / n_ch, c = fc % n_ch;
    const float* s = src + c * src_map;
    const double* k = coeffs + (int64_t)f * fh * fw;
    double acc = 0.0;
    for (int i = 0; i < fh; ++i) {
      const int yy = min(max(y + i - cy, 0), h - 1);
      for (int j = 0; j < fw; ++j) {
        const int xx = min(max(x + j - cx, 0), w - 1);
        acc = __dadd_rn(acc, __dmul_rn(k[i * fw + j], (double)s[(int64_t)yy * pitch + xx]));
      }
    }
    out[fc * out_map + (int64_t)y * out_pitch + x] = (float)acc;
  }
}


// ---------------------------------------------------------------------------
// FC-side seam (the reference does these inline in numpy, network.py:193-199,
// 209-230, 264-273; backprop.py:22-39).  Same arithmetic as the fused engine
// (ck_engine.cuh fc_cols_preact / fc_bwd_rows / op_out_delta), so a layer run
// through the seam gives the engine's bits.
constexpr int kSeamFcSlices = 16;

// a_j = f32(sum over 16 interleaved row slices of f64 fma chains) + b_j;
// y_j = fc_act(a_j).  A CTA takes 32 columns x the 16 slices (thread = slice
// sl, column j: the chain over rows i = sl, sl + 16, ...; consecutive threads
// read consecutive columns of a row of W), the slices combined in order.
__global__ void __launch_bounds__(32 * kSeamFcSlices)
seam_fc_fwd(const float* __restrict__ x, int n_in, const float* __restrict__ W,
            const float* __restrict__ b, int n_out, float* a, float* y) {
  __shared__ double red[kSeamFcSlices][32];
  const int col = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + col;
  double part = 0.0;
  if (j < n_out)
    for (int i = sl; i < n_in; i += kSeamFcSlices)
      part = fma((double)__ldg(x + i), (double)__ldg(W + (int64_t)i * n_out + j), part);
  red[sl][col] = part;
  __syncthreads();
  if (sl == 0 && j < n_out) {
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < kSeamFcSlices; ++s) acc += red[s][col];
    const float aj = __fadd_rn((float)acc, b[j]);
    if (a) a[j] = aj;
    y[j] = fc_act(aj);
  }
}

__device__ __forceinline__ double seam_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per input row i: xgrad_i = f32(sum_j W[i,j] delta_j) (f64, lane
// stride + xor tree) from the OLD weights, then grad_w[i,j] = f32(x_i delta_j)
// stored and/or applied (w -= f32(eta * g)).  Row 0's warp also does the bias.
__global__ void seam_fc_bwd(const float* __restrict__ x, int n_in, float* W, float* b,
                            int n_out, const float* __restrict__ delta, float* xgrad,
                            float* grad_w, float* grad_b, float eta_f, int update) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n_in) return;
  float* row = W + (int64_t)i * n_out;
  double acc = 0.0;
  for (int j = lane; j < n_out; j += 32) acc = fma((double)row[j], (double)delta[j], acc);
  acc = seam_warp_sum(acc);
  if (xgrad && lane == 0) xgrad[i] = (float)acc;
  __syncwarp();
  const float xi = x[i];
  for (int j = lane; j < n_out; j += 32) {
    const float g = __fmul_rn(xi, delta[j]);
    if (grad_w) grad_w[(int64_t)i * n_out + j] = g;
    if (update) row[j] = sgd(row[j], eta_f, g);
  }
  if (i == 0) {
    for (int j = lane; j < n_out; j += 32) {
      if (grad_b) grad_b[j] = delta[j];
      if (update) b[j] = sgd(b[j], eta_f, delta[j]);
    }
  }
}

// delta[m, r, c] = f32(delta * activation_deriv(a)) over the logical cells
// of a pitched stack (network.py:219, 226, 251-252).
__global__ void seam_act_deriv_mul(const float* __restrict__ a, float* delta, int n_maps,
                                   int64_t map_stride, int pitch, int w, int h) {
  const int64_t cells = (int64_t)n_maps * h * w;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cells;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q % w);
    const int r = (int)((q / w) % h);
    const int m = (int)(q / ((int64_t)w * h));
    const int64_t o = m * map_stride + (int64_t)r * pitch + c;
    delta[o] = __fmul_rn(delta[o], act_deriv(a[o]));
  }
}

// params -= f32(eta * grads) (network.py:268-273, NEP-50 weak eta).
__global__ void seam_sgd_update(float* params, const float* __restrict__ grads, int64_t n,
                                float eta_f) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    params[q] = sgd(params[q], eta_f, grads[q]);
}

// output_deltas (backprop.py:22-32) in f64, rounded once; sample_loss
// (backprop.py:35-39) = 0.5 * numpy pairwise sum of (y - t)^2.  One warp.
__global__ void seam_output_deltas(const float* __restrict__ y, const float* __restrict__ a,
                                   const double* __restrict__ targets, int n, float* delta,
                                   double* loss, double* scratch) {
  const int lane = threadIdx.x;
  for (int j = lane; j < n; j += 32) {
    const double r = (double)y[j] - targets[j];
    delta[j] = (float)(r * (double)act_deriv(a[j]));
    scratch[j] = r * r;
  }
  __syncwarp();
  if (lane == 0 && loss) *loss = 0.5 * np_pairwise_sum(scratch, n);
}

static int finish_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, what);
  return CK_OK;
}

}  // namespace ck

using namespace ck;

extern "C" {

const char* ck_last_error(void) { return g_last_error.c_str(); }
int ck_abi_version(void) { return 1; }
int ck_kernel_launches(int64_t* count) {
  if (!count) return set_error(CK_E_CONFIG, "null count");
  *count = g_launches.load();
  return CK_OK;
}

int ck_conv_fwd(const float* src, int n_src, int src_rows, int src_pitch,
                const float* arena, const int64_t* fwd_offsets,
                const int64_t* fwd_srcs, const int64_t* fwd_widx,
                const int64_t* bias_off, int kx, int ky, int sx, int sy,
                float* a_out, float* y_out, int n_dest, int out_rows,
                int out_pitch, int out_w, int out_h, ck_stream_t stream) {
  CK_CHECK(n_src >= 1 && n_dest >= 1, CK_E_DIMENSION, "map counts must be >= 1");
  CK_CHECK(kx >= 1 && ky >= 1 && sx >= 0 && sy >= 0, CK_E_GEOMETRY, "bad kernel/skip");
  CK_CHECK(out_w >= 1 && out_h >= 1 && out_w <= out_pitch && out_h <= out_rows,
           CK_E_DIMENSION, "output geometry exceeds its buffer");
  CK_CHECK((out_h - 1) * (sy + 1) + ky <= src_rows, CK_E_DIMENSION, "source too small");
  const int64_t cells = (int64_t)n_dest * out_h * out_w;
  seam_conv_fwd<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      src, (int64_t)src_rows * src_pitch, src_pitch, arena, fwd_offsets, fwd_srcs,
      fwd_widx, bias_off, kx, ky, sx + 1, sy + 1, a_out, y_out, n_dest,
      (int64_t)out_rows * out_pitch, out_pitch, out_w, out_h);
  return finish_launch("ck_conv_fwd");
}

int ck_pull_bwd(const float* delta_next, int n_dest, int dest_rows,
                int dest_pitch, int dest_w, int dest_h, const float* arena,
                const int64_t* bwd_offsets, const int64_t* bwd_dests,
                const int64_t* bwd_widx, int kx, int ky, int sx, int sy,
                float* out, int n_src, int out_rows, int out_pitch, int src_w,
                int src_h, ck_stream_t stream) {
  CK_CHECK(n_src >= 1 && n_dest >= 1, CK_E_DIMENSION, "map counts must be >= 1");
  CK_CHECK(kx >= 1 && ky >= 1 && sx >= 0 && sy >= 0, CK_E_GEOMETRY, "bad kernel/skip");
  CK_CHECK(src_w <= out_pitch && src_h <= out_rows && dest_w <= dest_pitch &&
               dest_h <= dest_rows, CK_E_DIMENSION, "geometry exceeds its buffer");
  const int64_t cells = (int64_t)n_src * src_h * src_w;
  seam_pull_bwd<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      delta_next, (int64_t)dest_rows * dest_pitch, dest_pitch, dest_w, dest_h, arena,
      bwd_offsets, bwd_dests, bwd_widx, kx, ky, sx + 1, sy + 1, out, n_src,
      (int64_t)out_rows * out_pitch, out_pitch, src_w, src_h);
  return finish_launch("ck_pull_bwd");
}

int ck_weight_grad(const float* delta_next, int n_dest, int dest_rows,
                   int dest_pitch, int dest_w, int dest_h, const float* y_prev,
                   int n_src, int src_rows, int src_pitch,
                   const int64_t* pair_dest, const int64_t* pair_src,
                   const int64_t* pair_off, int n_pairs, int kx, int ky,
                   int sx, int sy, float* g_arena, ck_stream_t stream) {
  CK_CHECK(n_dest >= 1 && n_src >= 1, CK_E_DIMENSION, "map counts must be >= 1");
  CK_CHECK(kx >= 1 && ky >= 1 && sx >= 0 && sy >= 0, CK_E_GEOMETRY, "bad kernel/skip");
  if (n_pairs == 0) return CK_OK;
  const int64_t items = (int64_t)n_pairs * kx * ky;
  seam_weight_grad<<<blocks_for(items, 128), 128, 0, (cudaStream_t)stream>>>(
      delta_next, (int64_t)dest_rows * dest_pitch, dest_pitch, dest_w, dest_h, y_prev,
      (int64_t)src_rows * src_pitch, src_pitch, pair_dest, pair_src, pair_off,
      n_pairs, kx, ky, sx + 1, sy + 1, g_arena);
  return finish_launch("ck_weight_grad");
}

int ck_bias_grad(const float* delta_next, int n_dest, int dest_rows,
                 int dest_pitch, int dest_w, int dest_h,
                 const int64_t* bias_off, float* g_arena, ck_stream_t stream) {
  CK_CHECK(n_dest >= 1, CK_E_DIMENSION, "map count must be >= 1");
  const int64_t threads = (int64_t)n_dest * 32;
  seam_bias_grad<<<blocks_for(threads, 128), 128, 0, (cudaStream_t)stream>>>(
      delta_next, (int64_t)dest_rows * dest_pitch, dest_pitch, dest_w, dest_h, n_dest,
      bias_off, g_arena);
  return finish_launch("ck_bias_grad");
}

int ck_maxpool_fwd(const float* src, int n_maps, int src_rows, int src_pitch,
                   int px, int py, float* out, int out_rows, int out_pitch,
                   int out_w, int out_h, int64_t* arg_r, int64_t* arg_c,
                   ck_stream_t stream) {
  CK_CHECK(n_maps >= 1, CK_E_DIMENSION, "map count must be >= 1");
  CK_CHECK(px >= 1 && py >= 1, CK_E_GEOMETRY, "pool region must be >= 1");
  CK_CHECK(out_h * py <= src_rows && out_w * px <= src_pitch && out_w <= out_pitch &&
               out_h <= out_rows, CK_E_DIMENSION, "pool geometry exceeds its buffers");
  const int64_t cells = (int64_t)n_maps * out_h * out_w;
  seam_maxpool_fwd<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      src, (int64_t)src_rows * src_pitch, src_pitch, px, py, out,
      (int64_t)out_rows * out_pitch, out_pitch, out_w, out_h, n_maps, arg_r, arg_c);
  return finish_launch("ck_maxpool_fwd");
}

int ck_maxpool_bwd(const float* delta_next, int n_maps, int next_rows,
                   int next_pitch, int out_w, int out_h, const int64_t* arg_r,
                   const int64_t* arg_c, float* delta_prev, int prev_rows,
                   int prev_pitch, ck_stream_t stream) {
  CK_CHECK(n_maps >= 1, CK_E_DIMENSION, "map count must be >= 1");
  const int64_t cells = (int64_t)n_maps * out_h * out_w;
  seam_maxpool_bwd<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      delta_next, (int64_t)next_rows * next_pitch, next_pitch, out_w, out_h, n_maps,
      arg_r, arg_c, delta_prev, (int64_t)prev_rows * prev_pitch, prev_pitch);
  return finish_launch("ck_maxpool_bwd");
}

int ck_contrast(const float* src, int n_ch, int rows, int pitch, int w, int h,
                const double* coeffs, int n_filters, int fh, int fw, float* out,
                int out_rows, int out_pitch, ck_stream_t stream) {
  CK_CHECK(n_ch >= 1 && n_filters >= 1, CK_E_DIMENSION, "need channels and filters");
  CK_CHECK(fh >= 1 && fw >= 1 && fh <= h && fw <= w, CK_E_GEOMETRY,
           "filter larger than image");
  const int64_t cells = (int64_t)n_filters * n_ch * h * w;
  seam_contrast<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      src, n_ch, (int64_t)rows * pitch, pitch, w, h, coeffs, n_filters, fh, fw, out,
      (int64_t)out_rows * out_pitch, out_pitch);
  return finish_launch("ck_contrast");
}

int ck_fc_fwd(const float* x, int n_in, const float* weights, const float* bias, int n_out,
              float* a_out, float* y_out, ck_stream_t stream) {
  CK_CHECK(n_in >= 1 && n_out >= 1, CK_E_DIMENSION, "FC sizes must be >= 1");
  CK_CHECK(x && weights && bias && y_out, CK_E_CONFIG, "null FC buffer");
  seam_fc_fwd<<<(n_out + 31) / 32, 32 * kSeamFcSlices, 0, (cudaStream_t)stream>>>(
      x, n_in, weights, bias, n_out, a_out, y_out);
  return finish_launch("ck_fc_fwd");
}

int ck_fc_bwd_update(const float* x, int n_in, float* weights, float* bias, int n_out,
                     const float* delta, float* xgrad, float* grad_w, float* grad_b,
                     double eta, ck_stream_t stream) {
  CK_CHECK(n_in >= 1 && n_out >= 1, CK_E_DIMENSION, "FC sizes must be >= 1");
  CK_CHECK(x && weights && bias && delta, CK_E_CONFIG, "null FC buffer");
  CK_CHECK(eta >= 0.0, CK_E_CONFIG, "learning rate must be >= 0 (0 = no update)");
  const int warps = 8;
  seam_fc_bwd<<<blocks_for(n_in, warps), warps * 32, 0, (cudaStream_t)stream>>>(
      x, n_in, weights, bias, n_out, delta, xgrad, grad_w, grad_b, (float)eta, eta > 0.0);
  return finish_launch("ck_fc_bwd_update");
}

int ck_act_deriv_mul(const float* a, float* delta, int n_maps, int rows, int pitch, int w,
                     int h, ck_stream_t stream) {
  CK_CHECK(n_maps >= 1 && w >= 1 && h >= 1 && w <= pitch && h <= rows, CK_E_DIMENSION,
           "bad stack geometry");
  const int64_t cells = (int64_t)n_maps * h * w;
  seam_act_deriv_mul<<<blocks_for(cells, 256), 256, 0, (cudaStream_t)stream>>>(
      a, delta, n_maps, (int64_t)rows * pitch, pitch, w, h);
  return finish_launch("ck_act_deriv_mul");
}

int ck_sgd_update(float* params, const float* grads, int64_t n, double eta,
                  ck_stream_t stream) {
  CK_CHECK(eta > 0.0, CK_E_CONFIG, "learning rate must be > 0");
  if (n <= 0) return CK_OK;
  seam_sgd_update<<<blocks_for(n, 256) < 4096 ? blocks_for(n, 256) : 4096, 256, 0,
                    (cudaStream_t)stream>>>(params, grads, n, (float)eta);
  return finish_launch("ck_sgd_update");
}

int ck_output_deltas(const float* y, const float* a, const double* targets, int n,
                     float* delta, double* loss, double* scratch, ck_stream_t stream) {
  CK_CHECK(n >= 1, CK_E_DIMENSION, "need at least one output");
  CK_CHECK(y && a && targets && delta && scratch, CK_E_CONFIG, "null buffer");
  seam_output_deltas<<<1, 32, 0, (cudaStream_t)stream>>>(y, a, targets, n, delta, loss,
                                                        scratch);
  return finish_launch("ck_output_deltas");
}

}  // extern "C"
