/*
 * ck_oracle.c — CPU restatement of the reference's compute kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or the timed CPU reference.  The product path
 * (paper_1102_0183_b200) never links or calls it.
 *
 * Each function restates one numba kernel of convkit kernels.py with the
 * reference's exact arithmetic (probed):
 *   conv_fwd     kernels.py:70-87   f32 sequential bias->k->v->u, mul and add
 *                                   rounded separately (build with
 *                                   -ffp-contract=off), y = f32(1.7159 *
 *                                   tanh_f64(0.6666 * (double)a))
 *   pull_bwd     kernels.py:90-121  f64 accumulator of f32-rounded products
 *   weight_grad  kernels.py:124-141 f64 accumulator of f32-rounded products
 *   bias_grad    kernels.py:144-151 f64 accumulator
 *   maxpool_fwd  kernels.py:154-172 strict '>' (first cell in scan wins)
 *   maxpool_bwd  kernels.py:175-180 f32 '+=' into the winner
 *   contrast     filters.py:168-172 (scipy ndimage.correlate, mode nearest:
 *                                   f64 sum, one rounding)
 * Like numba's prange, the outer loop is split over OpenMP threads with one
 * writer per output cell, so results do not depend on the thread count.
 * Pitched buffers: map stride and row pitch are explicit (elements).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>

#define ACT_SCALE 1.7159
#define ACT_GAIN 0.6666

static int floordiv(int a, int b) { /* Python // for b > 0 */
  int q = a / b;
  if ((a % b != 0) && (a < 0)) q -= 1;
  return q;
}

void oracle_conv_fwd(const float* src, int64_t src_map, int64_t src_pitch,
                     const float* arena, const int64_t* fwd_off,
                     const int64_t* fwd_src, const int64_t* fwd_widx,
                     const int64_t* bias_off, int kx, int ky, int sx, int sy,
                     float* a_out, float* y_out, int n_dest, int64_t out_map,
                     int64_t out_pitch, int out_w, int out_h) {
  const int tx = sx + 1, ty = sy + 1;
#pragma omp parallel for schedule(static)
  for (int d = 0; d < n_dest; ++d) {
    for (int r = 0; r < out_h; ++r) {
      for (int c = 0; c < out_w; ++c) {
        float acc = arena[bias_off[d]];
        for (int64_t k = fwd_off[d]; k < fwd_off[d + 1]; ++k) {
          const float* s = src + fwd_src[k] * src_map;
          const int64_t off = fwd_widx[k];
          for (int v = 0; v < ky; ++v) {
            const int64_t row = (int64_t)(r * ty + v) * src_pitch;
            for (int u = 0; u < kx; ++u) {
              const float prod = arena[off + v * kx + u] * s[row + c * tx + u];
              acc = acc + prod;
            }
          }
        }
        const int64_t o = d * out_map + r * out_pitch + c;
        a_out[o] = acc;
        y_out[o] = (float)(ACT_SCALE * tanh(ACT_GAIN * (double)acc));
      }
    }
  }
}

void oracle_pull_bwd(const float* dn, int64_t dn_map, int64_t dn_pitch, int dest_w,
                     int dest_h, const float* arena, const int64_t* bwd_off,
                     const int64_t* bwd_dst, const int64_t* bwd_widx, int kx,
                     int ky, int sx, int sy, float* out, int n_src,
                     int64_t out_map, int64_t out_pitch, int src_w, int src_h) {
  const int tx = sx + 1, ty = sy + 1;
#pragma omp parallel for schedule(static)
  for (int s = 0; s < n_src; ++s) {
    for (int j = 0; j < src_h; ++j) {
      int ylo = -floordiv(-(j - ky + 1), ty);
      if (ylo < 0) ylo = 0;
      int yhi = j / ty;
      if (yhi > dest_h - 1) yhi = dest_h - 1;
      for (int i = 0; i < src_w; ++i) {
        int xlo = -floordiv(-(i - kx + 1), tx);
        if (xlo < 0) xlo = 0;
        int xhi = i / tx;
        if (xhi > dest_w - 1) xhi = dest_w - 1;
        double acc = 0.0;
        for (int64_t k = bwd_off[s]; k < bwd_off[s + 1]; ++k) {
          const float* d = dn + bwd_dst[k] * dn_map;
          const int64_t off = bwd_widx[k];
          for (int y = ylo; y <= yhi; ++y) {
            const int64_t wrow = off + (int64_t)(j - y * ty) * kx;
            for (int x = xlo; x <= xhi; ++x) {
              const float prod = d[y * dn_pitch + x] * arena[wrow + (i - x * tx)];
              acc += (double)prod;
            }
          }
        }
        out[s * out_map + j * out_pitch + i] = (float)acc;
      }
    }
  }
}

void oracle_weight_grad(const float* dn, int64_t dn_map, int64_t dn_pitch,
                        int dest_w, int dest_h, const float* yp, int64_t yp_map,
                        int64_t yp_pitch, const int64_t* pdst,
                        const int64_t* psrc, const int64_t* poff, int n_pairs,
                        int kx, int ky, int sx, int sy, float* g) {
  const int tx = sx + 1, ty = sy + 1;
#pragma omp parallel for schedule(static)
  for (int p = 0; p < n_pairs; ++p) {
    const float* d = dn + pdst[p] * dn_map;
    const float* s = yp + psrc[p] * yp_map;
    for (int v = 0; v < ky; ++v)
      for (int u = 0; u < kx; ++u) {
        double acc = 0.0;
        for (int r = 0; r < dest_h; ++r) {
          const int64_t row = (int64_t)(r * ty + v) * yp_pitch;
          for (int c = 0; c < dest_w; ++c) {
            const float prod = d[r * dn_pitch + c] * s[row + c * tx + u];
            acc += (double)prod;
          }
        }
        g[poff[p] + v * kx + u] = (float)acc;
      }
  }
}

void oracle_bias_grad(const float* dn, int64_t dn_map, int64_t dn_pitch, int dest_w,
                      int dest_h, int n_dest, const int64_t* bias_off, float* g) {
#pragma omp parallel for schedule(static)
  for (int d = 0; d < n_dest; ++d) {
    double acc = 0.0;
    for (int r = 0; r < dest_h; ++r)
      for (int c = 0; c < dest_w; ++c) acc += (double)dn[d * dn_map + r * dn_pitch + c];
    g[bias_off[d]] = (float)acc;
  }
}

void oracle_maxpool_fwd(const float* src, int64_t src_map, int64_t src_pitch, int px,
                        int py, float* out, int64_t out_map, int64_t out_pitch,
                        int out_w, int out_h, int n_maps, int64_t* arg_r,
                        int64_t* arg_c) {
#pragma omp parallel for schedule(static)
  for (int m = 0; m < n_maps; ++m)
    for (int r = 0; r < out_h; ++r)
      for (int c = 0; c < out_w; ++c) {
        int br = r * py, bc = c * px;
        float best = src[m * src_map + br * src_pitch + bc];
        for (int v = 0; v < py; ++v)
          for (int u = 0; u < px; ++u) {
            const float val = src[m * src_map + (int64_t)(r * py + v) * src_pitch + c * px + u];
            if (val > best) {
              best = val;
              br = r * py + v;
              bc = c * px + u;
            }
          }
        out[m * out_map + r * out_pitch + c] = best;
        const int64_t q = ((int64_t)m * out_h + r) * out_w + c;
        arg_r[q] = br;
        arg_c[q] = bc;
      }
}

void oracle_maxpool_bwd(const float* dn, int64_t dn_map, int64_t dn_pitch, int out_w,
                        int out_h, int n_maps, const int64_t* arg_r,
                        const int64_t* arg_c, float* dp, int64_t dp_map,
                        int64_t dp_pitch) {
#pragma omp parallel for schedule(static)
  for (int m = 0; m < n_maps; ++m)
    for (int r = 0; r < out_h; ++r)
      for (int c = 0; c < out_w; ++c) {
        const int64_t q = ((int64_t)m * out_h + r) * out_w + c;
        float* cell = dp + m * dp_map + arg_r[q] * dp_pitch + arg_c[q];
        *cell = *cell + dn[m * dn_map + r * dn_pitch + c];
      }
}

/* correlate(channel, coeffs, mode="nearest") for every (filter, channel),
 * output map f*n_ch + c; f64 accumulation, one rounding to f32. */
void oracle_contrast(const float* src, int n_ch, int64_t src_map, int64_t pitch, int w,
                     int h, const double* coeffs, int n_filters, int fh, int fw,
                     float* out, int64_t out_map, int64_t out_pitch) {
  const int cy = fh / 2, cx = fw / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int f = 0; f < n_filters; ++f)
    for (int c = 0; c < n_ch; ++c) {
      const float* s = src + c * src_map;
      const double* k = coeffs + (int64_t)f * fh * fw;
      float* o = out + ((int64_t)f * n_ch + c) * out_map;
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          double acc = 0.0;
          for (int i = 0; i < fh; ++i) {
            int yy = y + i - cy;
            yy = yy < 0 ? 0 : (yy > h - 1 ? h - 1 : yy);
            for (int j = 0; j < fw; ++j) {
              int xx = x + j - cx;
              xx = xx < 0 ? 0 : (xx > w - 1 ? w - 1 : xx);
              acc += k[i * fw + j] * (double)s[yy * pitch + xx];
            }
          }
          o[y * out_pitch + x] = (float)acc;
        }
    }
}

/* worker threads of every oracle kernel (kernels.set_workers analogue) */
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int oracle_get_threads(void) { return omp_get_max_threads(); }
