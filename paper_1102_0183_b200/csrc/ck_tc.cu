// ck_tc.cu — batched test-set evaluation on the 5th-generation tensor cores.
//
// The bit-exact evaluation path (ck_net_eval) keeps the reference's
// sequential f32 conv chains and therefore runs on the SIMT pipes.  This file
// is the throughput path the north star allows "within a stated tolerance":
// every convolution, the contrast layer and every fully connected layer is an
// implicit GEMM on tcgen05 (kind::f16, FP32 accumulation in TMEM):
//
//   D[m, n] = sum_k A[m, k] * B[n, k]
//     m = (image, out row, out col)              (M tile: 128 rows)
//     n = destination map / neuron               (N <= 512, one TMEM column each)
//     k = (source map, kernel row v, kernel col u)   (K chunks of 64)
//   A[m, k] = X[image, s, r*ty + v - cy, c*tx + u - cx]   (gathered, clamped
//             for the contrast layer's replicated border)
//   B[n, k] = the layer's weight (zero where the connection table has no pair)
//
// Precision modes: passes = 1 rounds A and B to fp16 (11-bit significand);
// passes = 3 splits both into fp16 hi + lo parts and accumulates
// Ah*Bh + Ah*Bl + Al*Bh (K' = 3K), which is within a few f32 ulps of an f32
// GEMM.  Neither is bit-exact with the reference's sequential f32 chain, so
// labels are compared by agreement rate (tests/test_gpu_tc.py).
//
// Per CTA (256 threads, persistent over (row tile, column tile) pairs; two or
// more CTAs per SM so one CTA's epilogue overlaps another's gather / MMAs):
//   * all threads gather the A chunk (128 x 64 fp16) straight into shared
//     memory in the UMMA no-swizzle K-major core-matrix layout (8 rows x 16 B
//     per core matrix; K-adjacent cores 128 B apart, 8-row groups 1 KB apart);
//   * thread 0 streams the matching B chunk (pre-laid-out in HBM in the same
//     layout) with one cp.async.bulk (TMA bulk copy) onto an mbarrier;
//   * thread 0 issues tcgen05.mma (M=128, N<=256 per instruction, K=16) for
//     the chunk and tcgen05.commit's it onto the stage's mbarrier, so the
//     gather of chunk c+1 overlaps the MMAs of chunk c (when two stages fit);
//     K chunks are 16, 32 or 64 wide to match small-K first layers;
//   * epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32*(w%4)..+31),
//     the max-pool of the layer above fused in (M is ordered by pool
//     blocks) on the raw accumulators, then bias + scaled tanh once per
//     pooled value (both monotone); store (image, map, row, col) f32.
// Unfused pools, the contrast layer and the argmax are small SIMT kernels.
#include <cuda_fp16.h>
#include <math.h>

#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "ck_host.h"
#include "ck_tc_common.cuh"

namespace ck {
namespace tc {

struct GemmLayer {
  int S, H, W;                 // source maps / rows / cols
  int kx, ky, tx, ty, cx, cy;  // kernel, stride (skip + 1), centre offset (contrast)
  int N, OH, OW;               // destinations, output rows / cols
  int K, K_pad, N_pad, passes, parts;    // parts: 2 (hi + lo) when passes == 3
  int bk;                      // K per chunk: 16, 32 or 64 (small K wastes no MMA / gather work)
  int act;                     // 1: 1.7159 tanh(0.6666 a); 0: identity
  int dst_maps, dst_off;       // output tensor map count and this layer's first map
  int px, py, PH, PW;          // fused max-pool (1x1: none); output is (PH, PW)
  int P, bpt;                  // rows per pool block (px*py), blocks per 128-row tile
  int Nt, n_tiles;             // columns per CTA tile (<= 256), column tiles
  const float* X;              // (B, S, H, W)
  float* Y;                    // (B, dst_maps, OH, OW)
  const __half* Bw;            // (K_pad / BK, parts, N_pad * BK) core-matrix layout
  const float* bias;           // N (nullable)
  const int* kdec;             // K_pad tap codes (see gemm_kernel), -1 for padding
};

// 1.7159 tanh(0.6666 a) through exp: |error| ~1e-7, a few instructions
// instead of tanhf's slow path (this path is within tolerance, not exact).
__device__ __forceinline__ float act_fast(float a) {
  const float e = __expf(2.f * kActGain * fminf(fmaxf(a, -40.f), 40.f));
  return kActScale * (1.f - __fdividef(2.f, e + 1.f));
}

// Shared memory: [A stages (hi[, lo]) | B stages (hi[, lo]) | kdec | barriers].
// One gather per K chunk feeds every pass: with SPLIT the chunk is stored as
// fp16 hi and lo parts and the MMAs Ah*Bh + Ah*Bl + Al*Bh run back to back.
// kdec[k]: CLAMP (contrast) s<<16 | v<<8 | u; otherwise the element offset
// s*H*W + v*W + u of the tap relative to the row's window origin; -1 = pad.
template <bool CLAMP, bool SPLIT, int BKT>
__global__ void __launch_bounds__(THREADS, BKT == 64 ? 3 : 4) gemm_kernel(GemmLayer G, int64_t M, int tmem_cols,
                                                          int stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NP = SPLIT ? 2 : 1;                 // operand parts
  constexpr int KC = BKT / 8;                       // core matrices along K per chunk
  constexpr int RG = KC * 128;                      // bytes per 8-row group
  const int a_bytes = BM * BKT * 2;                 // one part of one stage
  const int b_bytes = G.Nt * BKT * 2;               // one part of one stage (a column tile)
  uint8_t* As = smem;                               // [stage][part] a_bytes
  uint8_t* Bs = smem + stages * NP * a_bytes;       // [stage][part] b_bytes (hi then lo)
  int* kdec = reinterpret_cast<int*>(Bs + stages * NP * b_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(kdec + ((G.K_pad + 1) & ~1));
  float* epi = reinterpret_cast<float*>(bars + 4);   // [2][BM][17] epilogue staging
  uint64_t* load_bar = bars;        // [stages]: B chunk landed
  uint64_t* mma_bar = bars + 2;     // [stages]: MMAs reading stage s done
  __shared__ uint32_t tmem_slot;
  __shared__ int64_t obase_s[BM];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = tid; k < G.K_pad; k += THREADS) kdec[k] = G.kdec[k];
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  const int HW = G.H * G.W;
  const int chunks = G.K_pad / BKT;
  int64_t g = 0;                          // global chunk counter (stage phases)

  // M counts pool blocks: tile t holds blocks [t*bpt, (t+1)*bpt), P rows
  // each (row-major inside the block, the pool's scan order); the last
  // 128 - bpt*P rows of a tile are idle.
  const int pcells = G.PH * G.PW;
  const int64_t m_tiles = (M + G.bpt - 1) / G.bpt;
  for (int64_t lt = blockIdx.x; lt < m_tiles * G.n_tiles; lt += gridDim.x) {
    const int64_t tile = lt / G.n_tiles;           // row tile
    const int n0 = (int)(lt - tile * G.n_tiles) * G.Nt;   // first column of the column tile
    const int nw = min(G.Nt, G.N_pad - n0);
    const int row = tid & (BM - 1);
    const int64_t blk = tile * G.bpt + row / G.P;
    const bool valid = row < G.bpt * G.P && blk < M;
    const float* xrow = G.X;
    int r0 = 0, c0 = 0;
    if (valid) {
      const int64_t img = blk / pcells;
      const int pc = (int)(blk - img * pcells);
      const int w = row % G.P;
      const int r = (pc / G.PW) * G.py + w / G.px;
      const int c = (pc % G.PW) * G.px + w % G.px;
      r0 = r * G.ty - G.cy;
      c0 = c * G.tx - G.cx;
      xrow = G.X + img * (int64_t)G.S * HW + (CLAMP ? 0 : r0 * G.W + c0);
    }
    for (int ch = 0; ch < chunks; ++ch, ++g) {
      const int st = stages == 2 ? (int)(g & 1) : 0;
      const int64_t use = stages == 2 ? (g >> 1) : g;   // uses of this stage so far
      if (use >= 1) mbar_wait(&mma_bar[st], (unsigned)((use - 1) & 1));
      uint8_t* a_st = As + st * NP * a_bytes;
      uint8_t* b_st = Bs + st * NP * b_bytes;
      if (tid == 0) {
        const __half* bsrc = G.Bw + (int64_t)ch * NP * G.N_pad * BKT + (int64_t)n0 * BKT;
        expect_tx(&load_bar[st], NP * nw * BKT * 2);
        bulk_copy(b_st, bsrc, nw * BKT * 2, &load_bar[st]);
        if (SPLIT) bulk_copy(b_st + b_bytes, bsrc + (int64_t)G.N_pad * BKT, nw * BKT * 2, &load_bar[st]);
      }
      const int kc0 = ch * BKT;
      // all loads of this thread first (latency overlap), then convert
      float x[KC / 2][8];
#pragma unroll
      for (int it = 0; it < KC / 2; ++it) {
        const int kg = (tid >> 7) + 2 * it;          // core matrix along K
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int dec = kdec[kc0 + kg * 8 + e];
          x[it][e] = 0.f;
          if (valid && dec >= 0) {
            if (CLAMP) {
              const int s = dec >> 16, v = (dec >> 8) & 0xFF, u = dec & 0xFF;
              const int rr = min(max(r0 + v, 0), G.H - 1);
              const int cc = min(max(c0 + u, 0), G.W - 1);
              x[it][e] = __ldg(xrow + (int64_t)s * HW + rr * G.W + cc);
            } else {
              x[it][e] = __ldg(xrow + dec);
            }
          }
        }
      }
#pragma unroll
      for (int it = 0; it < KC / 2; ++it) {
        const int kg = (tid >> 7) + 2 * it;
        const int off = (row >> 3) * RG + kg * 128 + (row & 7) * 16;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const __half h0 = __float2half_rn(x[it][e]), h1 = __float2half_rn(x[it][e + 1]);
          hi[e >> 1] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
          if (SPLIT) {
            const __half l0 = __float2half_rn(x[it][e] - __half2float(h0));
            const __half l1 = __float2half_rn(x[it][e + 1] - __half2float(h1));
            lo[e >> 1] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
          }
        }
        *reinterpret_cast<uint4*>(a_st + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        if (SPLIT) *reinterpret_cast<uint4*>(a_st + a_bytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        mbar_wait(&load_bar[st], (unsigned)(use & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ah = smem_u32(a_st), bh = smem_u32(b_st);
#pragma unroll
        for (int ks = 0; ks < BKT / 16; ++ks) {
          const uint32_t id = instr_desc(nw);
          const uint32_t boff = ks * 256;
          const uint64_t a_hi = umma_desc(ah + ks * 256, 128, RG);
          const uint64_t b_hi = umma_desc(bh + boff, 128, RG);
          mma_f16(tmem, a_hi, b_hi, id, (ch > 0 || ks > 0) ? 1 : 0);
          if (SPLIT) {
            mma_f16(tmem, a_hi, umma_desc(bh + b_bytes + boff, 128, RG), id, 1);
            mma_f16(tmem, umma_desc(ah + a_bytes + ks * 256, 128, RG), b_hi, id, 1);
          }
        }
        mma_commit(&mma_bar[st]);
      }
    }
    // epilogue: wait for the tile's last MMAs
    {
      const int64_t gl = g - 1;
      const int st = stages == 2 ? (int)(gl & 1) : 0;
      const int64_t use = stages == 2 ? (gl >> 1) : gl;
      mbar_wait(&mma_bar[st], (unsigned)(use & 1));
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid < G.bpt) {                // output base of each pool block of the tile
      const int64_t gb = tile * G.bpt + tid;
      const int64_t img = gb / pcells;
      obase_s[tid] = gb < M ? (img * G.dst_maps + G.dst_off) * (int64_t)pcells + (gb - img * pcells)
                            : -1;
    }
    __syncthreads();
    {
      // two warp groups take alternate 16-column chunks; warp w reads TMEM
      // lanes 32*(w%4)..+31 (its rows).  Activated values go through a
      // per-group staging tile so the pool max runs across rows.
      const int quarter = warp & 3, grp = warp >> 2, gtid = tid & 127;
      float* stage = epi + grp * (BM * 17);
      for (int c16 = grp; c16 * 16 < nw; c16 += 2) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + c16 * 16, v);
        const int erow = quarter * 32 + lane;
        // raw accumulators: bias and activation are monotone, so they are
        // applied once per pooled value below (max(f(a_i + b)) = f(max a_i + b))
#pragma unroll
        for (int i = 0; i < 16; ++i) stage[erow * 17 + i] = v[i];
        group_sync(grp);
        // thread -> (block b, columns i0, i0 + istep, ...): no divisions
        const int istep = BM / G.bpt;
        if (gtid < istep * G.bpt) {
          const int b = gtid % G.bpt;
          const int64_t ob = obase_s[b];
          if (ob >= 0) {
            for (int i = gtid / G.bpt; i < 16; i += istep) {
              const int n = n0 + c16 * 16 + i;
              if (n >= G.N) break;
              const float* col = stage + b * G.P * 17 + i;
              float best = col[0];
              for (int w = 1; w < G.P; ++w) {
                const float xv = col[w * 17];
                if (xv > best) best = xv;
              }
              float a = best + (G.bias ? __ldg(G.bias + n) : 0.f);
              if (G.act) a = act_fast(a);
              G.Y[ob + (int64_t)n * pcells] = a;
            }
          }
        }
        group_sync(grp);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// B[n, k] = src[wmap[n * K_pad + k]] (or 0) in the chunked core-matrix
// layout: per K chunk the hi block, then (parts = 2) the lo block.
__global__ void fill_weights(const float* __restrict__ src, const int* __restrict__ wmap, int N_pad,
                             int K_pad, int parts, int bk, __half* __restrict__ out) {
  const int64_t total = (int64_t)parts * N_pad * K_pad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % K_pad);
    const int n = (int)((i / K_pad) % N_pad);
    const int p = (int)(i / ((int64_t)K_pad * N_pad));
    const int idx = wmap[(int64_t)n * K_pad + k];
    const float w = idx >= 0 ? src[idx] : 0.f;
    const __half hi = __float2half_rn(w);
    const __half h = p == 1 ? __float2half_rn(w - __half2float(hi)) : hi;
    const int ch = k / bk;
    const int kk = k % bk;
    const int64_t off = ((int64_t)ch * parts + p) * N_pad * bk +
                        ((n >> 3) * (bk * 16) + (kk >> 3) * 128 + (n & 7) * 16 + (kk & 7) * 2) / 2;
    out[off] = h;
  }
}

__global__ void load_input(const uint8_t* __restrict__ images, const float* __restrict__ lut,
                           int64_t first, int64_t n_vals, int64_t per_img, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_vals;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = first * per_img + i;
    out[i] = lut ? __ldg(lut + images[src]) : reinterpret_cast<const float*>(images)[src];
  }
}

// max-pool, strict '>' (first maximum in row-major scan), trailing cells dropped
__global__ void pool_kernel(const float* __restrict__ X, int maps_total, int H, int W, int px, int py,
                            int OH, int OW, float* __restrict__ Y) {
  const int64_t total = (int64_t)maps_total * OH * OW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % OW);
    const int r = (int)((i / OW) % OH);
    const int64_t m = i / ((int64_t)OW * OH);
    const float* src = X + m * H * W + (int64_t)(r * py) * W + c * px;
    float best = src[0];
    for (int v = 0; v < py; ++v)
      for (int u = 0; u < px; ++u) {
        const float x = src[v * W + u];
        if (x > best) best = x;
      }
    Y[i] = best;
  }
}

// contrast layer originals: maps [0, C) of the output = the input channels
__global__ void copy_maps(const float* __restrict__ X, int64_t per_img_in, int64_t per_img_out,
                          int64_t n_img, float* __restrict__ Y) {
  const int64_t total = n_img * per_img_in;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / per_img_in;
    Y[b * per_img_out + (i - b * per_img_in)] = X[i];
  }
}

__global__ void argmax_kernel(const float* __restrict__ Y, int64_t n, int n_cls, int32_t* pred,
                              float* outputs) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
       b += (int64_t)gridDim.x * blockDim.x) {
    const float* y = Y + b * n_cls;
    int best = 0;
    for (int j = 1; j < n_cls; ++j)
      if (y[j] > y[best]) best = j;
    pred[b] = best;
    if (outputs)
      for (int j = 0; j < n_cls; ++j) outputs[b * n_cls + j] = y[j];
  }
}

// ---------------------------------------------------------------------------
// host plan

// Contrast responses on the SIMT pipes (a GEMM with N = filters x channels
// would leave the tensor core mostly idle and gather-bound): one CTA per
// (image, channel), replicated-border window staged in shared memory, each
// thread a strip of 4 cells with a sliding register window; f32 FMA.
__global__ void __launch_bounds__(256) contrast_kernel(const float* __restrict__ X, int C, int H, int W,
                                                       const float* __restrict__ coef, int F, int fh,
                                                       int fw, float* __restrict__ Y, int out_maps) {
  extern __shared__ float sm[];
  const int cy = fh / 2, cx = fw / 2;
  const int PW = W + fw - 1 + 4, PHh = H + fh - 1;
  float* win = sm;                       // PHh x PW
  float* cf = sm + PHh * PW;             // F x fh x fw
  const int64_t img = blockIdx.x / C;
  const int c = blockIdx.x % C;
  const float* src = X + (img * C + c) * (int64_t)H * W;
  for (int i = threadIdx.x; i < PHh * PW; i += blockDim.x) {
    const int r = min(max(i / PW - cy, 0), H - 1), q = min(max(i % PW - cx, 0), W - 1);
    win[i] = src[r * W + q];
  }
  for (int i = threadIdx.x; i < F * fh * fw; i += blockDim.x) cf[i] = coef[i];
  __syncthreads();
  const int strips = (W + 3) / 4;
  // filters in pairs: each window load feeds 2 filters x 4 cells
  const int fpairs = (F + 1) / 2;
  for (int job = threadIdx.x; job < fpairs * H * strips; job += blockDim.x) {
    const int f0 = 2 * (job / (H * strips));
    const bool two = f0 + 1 < F;
    const int r = (job / strips) % H;
    const int c0 = (job % strips) * 4;
    float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int v = 0; v < fh; ++v) {
      const float* w = win + (r + v) * PW + c0;
      const float* k0 = cf + (f0 * fh + v) * fw;
      const float* k1 = two ? k0 + fh * fw : k0;
      float x0 = w[0], x1 = w[1], x2 = w[2], x3 = w[3];
      for (int u = 0; u < fw; ++u) {
        const float a = k0[u], b = k1[u];
        acc0[0] = fmaf(a, x0, acc0[0]);
        acc0[1] = fmaf(a, x1, acc0[1]);
        acc0[2] = fmaf(a, x2, acc0[2]);
        acc0[3] = fmaf(a, x3, acc0[3]);
        acc1[0] = fmaf(b, x0, acc1[0]);
        acc1[1] = fmaf(b, x1, acc1[1]);
        acc1[2] = fmaf(b, x2, acc1[2]);
        acc1[3] = fmaf(b, x3, acc1[3]);
        x0 = x1; x1 = x2; x2 = x3; x3 = w[u + 4];
      }
    }
    float* out0 = Y + ((img * out_maps + C + f0 * C + c) * (int64_t)H + r) * W;
    float* out1 = out0 + (int64_t)C * H * W;
    for (int q = 0; q < 4 && c0 + q < W; ++q) {
      out0[c0 + q] = acc0[q];
      if (two) out1[c0 + q] = acc1[q];
    }
  }
}

// The contrast responses when every filter is low-rank (hat<N> is a
// difference of two separable Gaussians: rank 2): filter f = sum_r u_fr v_fr^T,
// so a response is R horizontal passes (fw taps) then R vertical passes (fh
// taps) -- 2R(fh+fw) instead of fh*fw multiply-adds per cell (hat21: 84 vs
// 441).  One CTA per (image, channel): the replicated-border window and the
// horizontal results of every (filter, rank term) in shared memory.  f32;
// the factors come from an f64 eigendecomposition on the host (within this
// path's tolerance; the exact engine keeps the reference's f64 correlation).
__global__ void __launch_bounds__(256) contrast_sep_kernel(
    const float* __restrict__ X, int C, int H, int W, const float* __restrict__ uv, int F, int R,
    int fh, int fw, float* __restrict__ Y, int out_maps) {
  extern __shared__ float sm[];
  const int cy = fh / 2, cx = fw / 2;
  const int PW = W + fw - 1, PHh = H + fh - 1;
  float* win = sm;                             // PHh x PW
  float* hor = win + PHh * PW;                 // [F*R][PHh][W]
  float* fac = hor + (size_t)F * R * PHh * W;  // per (f, r): u (fh) then v (fw)
  const int64_t img = blockIdx.x / C;
  const int c = blockIdx.x % C;
  const float* src = X + (img * C + c) * (int64_t)H * W;
  for (int i = threadIdx.x; i < PHh * PW; i += blockDim.x) {
    const int r = min(max(i / PW - cy, 0), H - 1), q = min(max(i % PW - cx, 0), W - 1);
    win[i] = src[r * W + q];
  }
  for (int i = threadIdx.x; i < F * R * (fh + fw); i += blockDim.x) fac[i] = uv[i];
  __syncthreads();
  for (int i = threadIdx.x; i < F * R * PHh * W; i += blockDim.x) {
    const int fr = i / (PHh * W), y = (i / W) % PHh, x = i % W;
    const float* v = fac + fr * (fh + fw) + fh;
    const float* w = win + y * PW + x;
    float acc = 0.f;
    for (int j = 0; j < fw; ++j) acc = fmaf(v[j], w[j], acc);
    hor[i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < F * H * W; i += blockDim.x) {
    const int f = i / (H * W), y = (i / W) % H, x = i % W;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
      const float* u = fac + (f * R + r) * (fh + fw);
      const float* h = hor + ((size_t)(f * R + r) * PHh + y) * W + x;
      for (int t = 0; t < fh; ++t) acc = fmaf(u[t], h[t * W], acc);
    }
    Y[((img * out_maps + C + f * C + c) * (int64_t)H + y) * W + x] = acc;
  }
}

enum StepKind { ST_GEMM = 0, ST_POOL = 1, ST_COPY = 2, ST_CONTRAST = 3 };

struct Step {
  int kind;
  int layer;
  GemmLayer g;                  // ST_GEMM (X, Y patched per chunk)
  int64_t M_per_img;            // GEMM rows per image
  int tmem_cols;
  int clamp, stages, ctas_per_sm;
  size_t smem;
  int src_buf, dst_buf;         // activation buffer indices
  // pool / copy
  int maps, H, W, px, py, OH, OW;
  int64_t per_in, per_out;
  // parameter source
  int64_t param_off;            // offset of the layer's parameters (-1: fixed)
  int* d_wmap = nullptr;
  int* d_kdec = nullptr;
  int* d_bmap = nullptr;
  __half* d_B = nullptr;
  float* d_bias = nullptr;
  float* d_fixed = nullptr;     // contrast coefficients (f32)
  int F = 0, fh = 0, fw = 0, out_maps = 0;   // contrast
  int rank = 0;                 // > 0: separable factors in d_fixed (contrast_sep_kernel)
};

}  // namespace tc
}  // namespace ck

struct ck_tc_eval {
  int device = 0;
  int passes = 3;
  int64_t max_batch = 0;
  int n_classes = 0;
  int64_t in_per_img = 0;
  std::vector<ck::tc::Step> steps;
  std::vector<float*> bufs;            // activation buffers (max_batch * cells each)
  std::vector<int64_t> buf_cells;
  int final_buf = 0;
  int sms = 148;
};

namespace ck {
namespace tc {

static int64_t round_up(int64_t v, int64_t q) { return (v + q - 1) / q * q; }

// Low-rank factors of an fh x fw filter K (row-major, f64): the eigenpairs of
// K^T K by cyclic Jacobi sweeps give K = sum_r (K v_r) v_r^T over the
// eigenvectors v_r with non-negligible eigenvalues.  Returns the rank, or 0
// when the filter is not low-rank enough to pay (or the reconstruction is not
// within 1e-12 of K's largest entry); factors: per r, u_r (fh) then v_r (fw).
static int low_rank(const double* K, int fh, int fw, std::vector<double>& fac) {
  const int n = fw;
  std::vector<double> A((size_t)n * n, 0.0), V((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    V[i * n + i] = 1.0;
    for (int j = 0; j < n; ++j)
      for (int t = 0; t < fh; ++t) A[i * n + j] += K[t * fw + i] * K[t * fw + j];
  }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A[p * n + q] * A[p * n + q];
    if (off < 1e-60) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (fabs(A[p * n + q]) < 1e-300) continue;
        const double th = 0.5 * atan2(2 * A[p * n + q], A[q * n + q] - A[p * n + p]);
        const double c = cos(th), s = sin(th);
        for (int k = 0; k < n; ++k) {          // A <- J^T A J, V <- V J
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  double kmax = 0.0, lmax = 0.0;
  for (int i = 0; i < fh * fw; ++i) kmax = std::max(kmax, fabs(K[i]));
  for (int i = 0; i < n; ++i) lmax = std::max(lmax, A[i * n + i]);
  fac.clear();
  int rank = 0;
  std::vector<double> rec((size_t)fh * fw, 0.0);
  for (int r = 0; r < n; ++r) {
    if (A[r * n + r] <= 1e-12 * lmax) continue;   // sigma_r <= 1e-6 sigma_max: noise of K^T K
    std::vector<double> u(fh, 0.0);
    for (int t = 0; t < fh; ++t)
      for (int j = 0; j < fw; ++j) u[t] += K[t * fw + j] * V[j * n + r];
    for (int t = 0; t < fh; ++t) fac.push_back(u[t]);
    for (int j = 0; j < fw; ++j) fac.push_back(V[j * n + r]);
    for (int t = 0; t < fh; ++t)
      for (int j = 0; j < fw; ++j) rec[t * fw + j] += u[t] * V[j * n + r];
    ++rank;
  }
  double err = 0.0;
  for (int i = 0; i < fh * fw; ++i) err = std::max(err, fabs(rec[i] - K[i]));
  if (rank == 0 || err > 1e-12 * kmax || 2 * rank * (fh + fw) * 2 > fh * fw) return 0;
  return rank;
}

static int make_gemm(ck_tc_eval* P, Step& st, int S, int H, int W, int kx, int ky, int tx, int ty,
                     int cx, int cy, int N, int OH, int OW, int act, int dst_maps, int dst_off,
                     int px, int py, const std::vector<int>& kdec_host_in,
                     const std::vector<int>& wmap, const std::vector<int>& bmap) {
  GemmLayer& g = st.g;
  g.S = S; g.H = H; g.W = W; g.kx = kx; g.ky = ky; g.tx = tx; g.ty = ty; g.cx = cx; g.cy = cy;
  g.N = N; g.OH = OH; g.OW = OW; g.act = act; g.dst_maps = dst_maps; g.dst_off = dst_off;
  g.px = px; g.py = py; g.PH = OH / py; g.PW = OW / px; g.P = px * py;
  CK_CHECK(g.P <= BM, CK_E_DIMENSION, "tensor-core eval: pool region above 128 cells");
  g.bpt = BM / g.P;
  g.K = S * kx * ky;
  g.bk = g.K <= 16 ? 16 : g.K <= 32 ? 32 : BK;
  g.K_pad = (int)round_up(g.K, g.bk);
  g.N_pad = (int)round_up(N, 16);
  CK_CHECK(g.N_pad <= 512, CK_E_DIMENSION, "tensor-core eval: more than 512 outputs per layer");
  CK_CHECK(kx < 256 && ky < 256 && S < 32768, CK_E_DIMENSION, "tensor-core eval: kernel too large");
  g.passes = P->passes;
  g.parts = g.passes == 3 ? 2 : 1;
  // column tiles of <= 256 (one MMA per K step; TMEM <= 256 columns, so
  // two CTAs fit an SM's 512 columns)
  g.n_tiles = (g.N_pad + 255) / 256;
  g.Nt = (int)round_up((g.N_pad + g.n_tiles - 1) / g.n_tiles, 16);
  int cols = 32;
  while (cols < g.Nt) cols <<= 1;
  st.tmem_cols = cols;
  st.M_per_img = (int64_t)g.PH * g.PW;   // pool blocks per image
  st.clamp = cx > 0 || cy > 0;
  auto smem_for = [&](int stages) {
    return (size_t)stages * g.parts * ((size_t)BM * g.bk * 2 + (size_t)g.Nt * g.bk * 2) +
           (size_t)((g.K_pad + 1) & ~1) * 4 + 4 * 8 + 2 * BM * 17 * 4;
  };
  // CTAs per SM: shared memory (228 KB per SM, 1 KB reserved per CTA) and
  // TMEM (512 columns per SM) bound it.  Several resident CTAs overlap one
  // CTA's epilogue with another's gather and MMAs, so a single-stage ring
  // that fits two CTAs beats a double-buffered one that fits only one.
  auto occ = [&](size_t sm) {
    const int by_smem = sm <= 220 * 1024 ? (int)((228 * 1024) / (sm + 1024)) : 0;
    return std::min(by_smem, 512 / cols);
  };
  st.stages = occ(smem_for(2)) >= std::max(1, occ(smem_for(1))) ? 2 : 1;
  st.smem = smem_for(st.stages);
  // registers: gemm_kernel's launch bounds give 3 / 4 CTAs of 256 threads
  // per SM for K chunks of 64 / 32-or-16
  const int by_regs = g.bk == 64 ? 3 : 4;
  st.ctas_per_sm = std::max(1, std::min(occ(st.smem), by_regs));
  CK_CHECK(st.smem <= 220 * 1024, CK_E_DIMENSION, "tensor-core eval: tile exceeds shared memory");
  // The block scheduler only sees registers and shared memory: with the
  // launch bounds' register caps more CTAs than TMEM holds (512 / cols) could
  // co-reside and spin in tcgen05.alloc.  Pad the dynamic shared memory so
  // that shared memory alone caps residency at the TMEM limit.
  {
    const int tmem_limit = 512 / cols;
    const size_t need = (size_t)(228 * 1024) / (tmem_limit + 1) - 1024 + 128;
    if (tmem_limit < by_regs && st.smem < need) st.smem = need;
  }
  std::vector<int> kdec(g.K_pad, -1);
  for (int k = 0; k < g.K; ++k) {
    const int dec = kdec_host_in[k];
    kdec[k] = st.clamp ? dec : (dec >> 16) * H * W + ((dec >> 8) & 0xFF) * W + (dec & 0xFF);
  }
  std::vector<int> wm((size_t)g.N_pad * g.K_pad, -1);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < g.K; ++k) wm[(size_t)n * g.K_pad + k] = wmap[(size_t)n * g.K + k];
  CK_CUDA_TRY(cudaMalloc(&st.d_kdec, sizeof(int) * g.K_pad));
  CK_CUDA_TRY(cudaMemcpy(st.d_kdec, kdec.data(), sizeof(int) * g.K_pad, cudaMemcpyHostToDevice));
  CK_CUDA_TRY(cudaMalloc(&st.d_wmap, sizeof(int) * wm.size()));
  CK_CUDA_TRY(cudaMemcpy(st.d_wmap, wm.data(), sizeof(int) * wm.size(), cudaMemcpyHostToDevice));
  CK_CUDA_TRY(cudaMalloc(&st.d_B, sizeof(__half) * (size_t)g.parts * g.N_pad * g.K_pad));
  if (!bmap.empty()) {
    CK_CUDA_TRY(cudaMalloc(&st.d_bmap, sizeof(int) * N));
    CK_CUDA_TRY(cudaMemcpy(st.d_bmap, bmap.data(), sizeof(int) * N, cudaMemcpyHostToDevice));
    CK_CUDA_TRY(cudaMalloc(&st.d_bias, sizeof(float) * N));
  }
  g.kdec = st.d_kdec;
  g.Bw = st.d_B;
  g.bias = st.d_bias;
  st.kind = ST_GEMM;
  return CK_OK;
}

typedef void (*GemmFn)(GemmLayer, int64_t, int, int);
template <int BKT>
static GemmFn gemm_fn_bk(bool clamp, bool split) {
  if (clamp) return split ? gemm_kernel<true, true, BKT> : gemm_kernel<true, false, BKT>;
  return split ? gemm_kernel<false, true, BKT> : gemm_kernel<false, false, BKT>;
}
static GemmFn gemm_fn(bool clamp, bool split, int bk) {
  return bk == 16 ? gemm_fn_bk<16>(clamp, split)
                  : bk == 32 ? gemm_fn_bk<32>(clamp, split) : gemm_fn_bk<64>(clamp, split);
}

__global__ void gather_bias(const float* __restrict__ params, const int* __restrict__ bmap, int n,
                            float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = params[bmap[i]];
}

}  // namespace tc
}  // namespace ck

using ck::tc::Step;

extern "C" {

int ck_tc_create(const ck_layer_desc* layers, int n_layers, int device, int64_t max_batch,
                 int passes, ck_tc_eval** out) {
  CK_CHECK(layers && out && n_layers >= 2, CK_E_CONFIG, "bad arguments");
  CK_CHECK(passes == 1 || passes == 3, CK_E_CONFIG, "passes must be 1 or 3");
  CK_CHECK(max_batch >= 1, CK_E_CONFIG, "max_batch must be >= 1");
  CK_CHECK(layers[0].kind == CK_LAYER_INPUT, CK_E_CONFIG, "first layer must be the input");
  CK_CUDA_TRY(cudaSetDevice(device));
  ck_tc_eval* P = new ck_tc_eval();
  P->device = device;
  P->passes = passes;
  P->max_batch = max_batch;
  CK_CUDA_TRY(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device));
  auto fail = [&](int rc) {
    ck_tc_destroy(P);
    return rc;
  };
  // activation buffers per layer, allocated only for layers that are read
  // or written (a conv fused with its pool writes the pool's buffer)
  P->bufs.assign(n_layers, nullptr);
  for (int i = 0; i < n_layers; ++i)
    P->buf_cells.push_back((int64_t)layers[i].maps * layers[i].width * layers[i].height);
  auto need = [&](int i) {
    if (P->bufs[i]) return CK_OK;
    if (cudaMalloc(&P->bufs[i], sizeof(float) * P->buf_cells[i] * max_batch) != cudaSuccess)
      return ck::set_error(CK_E_NOMEM, "tensor-core eval: activation buffers");
    return CK_OK;
  };
  P->in_per_img = P->buf_cells[0];
  if (int rc = need(0)) return fail(rc);
  int64_t poff = 0;   // parameter offset (NetworkState.parameters() order)
  for (int i = 1; i < n_layers; ++i) {
    const ck_layer_desc& L = layers[i];
    const ck_layer_desc& Pv = layers[i - 1];
    Step st;
    st.layer = i;
    st.src_buf = i - 1;
    st.dst_buf = i;
    st.param_off = -1;
    const int S = Pv.maps, H = Pv.height, W = Pv.width;
    // a conv followed by a max-pool: the pool runs in the GEMM epilogue
    const bool fuse = L.kind == CK_LAYER_CONV && i + 1 < n_layers &&
                      layers[i + 1].kind == CK_LAYER_POOL &&
                      layers[i + 1].px * layers[i + 1].py <= ck::tc::BM;
    if (fuse) st.dst_buf = i + 1;
    if (int rc = need(st.dst_buf)) return fail(rc);
    if (L.kind == CK_LAYER_POOL) {
      st.kind = ck::tc::ST_POOL;
      st.maps = S; st.H = H; st.W = W; st.px = L.px; st.py = L.py; st.OH = L.height; st.OW = L.width;
      P->steps.push_back(st);
      continue;
    }
    if (L.kind == CK_LAYER_IMGPROC) {
      // originals, then the filter responses (SIMT, f32)
      Step cp = st;
      cp.kind = ck::tc::ST_COPY;
      cp.per_in = (int64_t)S * H * W;
      cp.per_out = (int64_t)L.maps * L.height * L.width;
      P->steps.push_back(cp);
      st.kind = ck::tc::ST_CONTRAST;
      st.F = L.n_filters; st.fh = L.filter_h; st.fw = L.filter_w; st.out_maps = L.maps;
      st.maps = S; st.H = H; st.W = W;
      std::vector<float> coef((size_t)st.F * st.fh * st.fw);
      for (size_t j = 0; j < coef.size(); ++j) coef[j] = (float)L.filter_coeffs[j];
      st.smem = sizeof(float) * ((size_t)(H + st.fh - 1) * (W + st.fw - 1 + 4) + coef.size());
      // low-rank filters (every one of the same rank R): separable passes
      {
        std::vector<double> all, f1;
        int R = -1;
        for (int f = 0; f < st.F && R != 0; ++f) {
          const int r = ck::tc::low_rank(L.filter_coeffs + (size_t)f * st.fh * st.fw, st.fh,
                                         st.fw, f1);
          R = (R < 0 || R == r) ? r : 0;
          all.insert(all.end(), f1.begin(), f1.end());
        }
        const size_t sm_sep = sizeof(float) * ((size_t)(H + st.fh - 1) * (W + st.fw - 1) +
                                               (size_t)st.F * std::max(R, 0) * (H + st.fh - 1) * W +
                                               all.size());
        if (R > 0 && sm_sep <= 200 * 1024 && !getenv("CKB200_TC_NOSEP")) {
          st.rank = R;
          st.smem = sm_sep;
          coef.assign(all.begin(), all.end());
        }
      }
      CK_CHECK(st.smem <= 200 * 1024, CK_E_DIMENSION, "tensor-core eval: contrast window too large");
      if (cudaMalloc(&st.d_fixed, sizeof(float) * coef.size()) != cudaSuccess ||
          cudaMemcpy(st.d_fixed, coef.data(), sizeof(float) * coef.size(),
                     cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(ck::set_error(CK_E_NOMEM, "tensor-core eval: filter coefficients"));
      P->steps.push_back(st);
      continue;
    }
    if (L.kind == CK_LAYER_CONV) {
      const int kx = L.kx, ky = L.ky, N = L.maps, K = S * kx * ky;
      std::vector<int> kdec(K), wmap((size_t)N * K, -1), bmap(N);
      for (int s = 0; s < S; ++s)
        for (int v = 0; v < ky; ++v)
          for (int u = 0; u < kx; ++u) kdec[(s * ky + v) * kx + u] = s << 16 | v << 8 | u;
      for (int d = 0; d < N; ++d) {
        for (int64_t p = L.fwd_offsets[d]; p < L.fwd_offsets[d + 1]; ++p) {
          const int s = (int)L.fwd_srcs[p];
          for (int v = 0; v < ky; ++v)
            for (int u = 0; u < kx; ++u)
              wmap[(size_t)d * K + (s * ky + v) * kx + u] =
                  (int)(poff + L.fwd_widx[p] + v * kx + u);
        }
        bmap[d] = (int)(poff + L.bias_offset[d]);
      }
      const int px = fuse ? layers[i + 1].px : 1, py = fuse ? layers[i + 1].py : 1;
      int rc = ck::tc::make_gemm(P, st, S, H, W, kx, ky, L.sx + 1, L.sy + 1, 0, 0, N, L.height,
                                 L.width, 1, N, 0, px, py, kdec, wmap, bmap);
      if (rc) return fail(rc);
      st.param_off = poff;
      poff += L.arena_size;
      P->steps.push_back(st);
      if (fuse) ++i;   // the pool layer is done
      continue;
    }
    if (L.kind == CK_LAYER_FC) {
      const int n_in = S * H * W, N = L.maps;
      std::vector<int> kdec(n_in), wmap((size_t)N * n_in), bmap(N);
      for (int s = 0; s < S; ++s)
        for (int v = 0; v < H; ++v)
          for (int u = 0; u < W; ++u) kdec[(s * H + v) * W + u] = s << 16 | v << 8 | u;
      for (int o = 0; o < N; ++o) {
        for (int k = 0; k < n_in; ++k) wmap[(size_t)o * n_in + k] = (int)(poff + (int64_t)k * N + o);
        bmap[o] = (int)(poff + (int64_t)n_in * N + o);
      }
      int rc = ck::tc::make_gemm(P, st, S, H, W, W, H, 1, 1, 0, 0, N, 1, 1, 1, N, 0, 1, 1, kdec,
                                 wmap, bmap);
      if (rc) return fail(rc);
      st.param_off = poff;
      poff += (int64_t)n_in * N + N;
      P->steps.push_back(st);
      continue;
    }
    return fail(ck::set_error(CK_E_CONFIG, "tensor-core eval: unsupported layer kind"));
  }
  CK_CHECK(layers[n_layers - 1].kind == CK_LAYER_FC, CK_E_CONFIG, "last layer must be the output");
  for (auto& st : P->steps) {
    if (st.kind == ck::tc::ST_GEMM)
      if (cudaSuccess != cudaFuncSetAttribute(ck::tc::gemm_fn(st.clamp, st.g.parts == 2, st.g.bk),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024)) return fail(ck::set_error(CK_E_CUDA, "tensor-core eval: kernel attributes"));
    if (st.kind == ck::tc::ST_CONTRAST)
      if (cudaSuccess != cudaFuncSetAttribute(ck::tc::contrast_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ||
          cudaSuccess != cudaFuncSetAttribute(ck::tc::contrast_sep_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) return fail(ck::set_error(CK_E_CUDA, "tensor-core eval: kernel attributes"));
  }

  P->n_classes = layers[n_layers - 1].maps;
  P->final_buf = n_layers - 1;
  CK_CUDA_TRY(cudaDeviceSynchronize());
  *out = P;
  return CK_OK;
}

int ck_tc_destroy(ck_tc_eval* P) {
  if (!P) return CK_OK;
  cudaSetDevice(P->device);
  for (float* b : P->bufs) cudaFree(b);
  for (auto& st : P->steps) {
    cudaFree(st.d_wmap);
    cudaFree(st.d_kdec);
    cudaFree(st.d_bmap);
    cudaFree(st.d_B);
    cudaFree(st.d_bias);
    cudaFree(st.d_fixed);
  }
  delete P;
  return CK_OK;
}

int ck_tc_set_params(ck_tc_eval* P, const float* params, ck_stream_t stream) {
  CK_CHECK(P && params, CK_E_CONFIG, "null argument");
  CK_CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  for (auto& st : P->steps) {
    if (st.kind != ck::tc::ST_GEMM || st.param_off < 0) continue;
    ck::tc::fill_weights<<<P->sms * 4, 256, 0, s>>>(params, st.d_wmap, st.g.N_pad, st.g.K_pad,
                                                     st.g.parts, st.g.bk, st.d_B);
    ck::tc::gather_bias<<<(st.g.N + 255) / 256, 256, 0, s>>>(params, st.d_bmap, st.g.N,
                                                             st.d_bias);
    ck::count_launch(2);
  }
  CK_CUDA_TRY(cudaGetLastError());
  return CK_OK;
}

int ck_tc_eval_run(ck_tc_eval* P, const uint8_t* images, const float* lut, int64_t first, int64_t n,
                   int32_t* pred, float* outputs, ck_stream_t stream) {
  CK_CHECK(P && images && pred, CK_E_CONFIG, "null argument");
  CK_CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t b0 = 0; b0 < n; b0 += P->max_batch) {
    const int64_t nb = std::min(P->max_batch, n - b0);
    ck::tc::load_input<<<P->sms * 4, 256, 0, s>>>(images, lut, first + b0, nb * P->in_per_img,
                                                  P->in_per_img, P->bufs[0]);
    ck::count_launch();
    for (auto& st : P->steps) {
      const float* X = P->bufs[st.src_buf];
      float* Y = P->bufs[st.dst_buf];
      if (st.kind == ck::tc::ST_POOL) {
        const int64_t total = nb * st.maps * (int64_t)st.OH * st.OW;
        ck::tc::pool_kernel<<<ck::blocks_for(total, 256), 256, 0, s>>>(
            X, (int)(nb * st.maps), st.H, st.W, st.px, st.py, st.OH, st.OW, Y);
      } else if (st.kind == ck::tc::ST_CONTRAST && st.rank > 0) {
        ck::tc::contrast_sep_kernel<<<(int)(nb * st.maps), 256, st.smem, s>>>(
            X, st.maps, st.H, st.W, st.d_fixed, st.F, st.rank, st.fh, st.fw, Y, st.out_maps);
      } else if (st.kind == ck::tc::ST_CONTRAST) {
        ck::tc::contrast_kernel<<<(int)(nb * st.maps), 256, st.smem, s>>>(
            X, st.maps, st.H, st.W, st.d_fixed, st.F, st.fh, st.fw, Y, st.out_maps);
      } else if (st.kind == ck::tc::ST_COPY) {
        ck::tc::copy_maps<<<P->sms * 4, 256, 0, s>>>(X, st.per_in, st.per_out, nb, Y);
      } else {
        ck::tc::GemmLayer g = st.g;
        g.X = X;
        g.Y = Y;
        const int64_t M = nb * st.M_per_img;
        const int64_t tiles = (M + g.bpt - 1) / g.bpt * g.n_tiles;
        const int grid = (int)std::min<int64_t>(tiles, (int64_t)P->sms * st.ctas_per_sm);
        ck::tc::gemm_fn(st.clamp, st.g.parts == 2, st.g.bk)<<<grid, ck::tc::THREADS, st.smem, s>>>(
            g, M, st.tmem_cols, st.stages);
      }
      ck::count_launch();
    }
    ck::tc::argmax_kernel<<<ck::blocks_for(nb, 256), 256, 0, s>>>(
        P->bufs[P->final_buf], nb, P->n_classes, pred + b0,
        outputs ? outputs + b0 * P->n_classes : nullptr);
    ck::count_launch();
  }
  CK_CUDA_TRY(cudaGetLastError());
  return CK_OK;
}

}  // extern "C"
