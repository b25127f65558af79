// ck_tct.cu — tensor-core training variant for wide nets.
//
// Opt-in, outside the bit-exact contract, with its own stated tolerance
// (tests/test_gpu_tct.py): online training -- one update per image, the
// reference's protocol (network.py:163-282) -- where every convolution's
// forward, weight gradient and delta pull is an implicit GEMM on the 5th-gen
// tensor cores (tcgen05.mma kind::f16, fp16 hi/lo split of both operands,
// Ah*Bh + Ah*Bl + Al*Bh, f32 accumulation in TMEM):
//
//   forward   D[m=(r,c), n=d]        = sum_{k=(s,v,u)} X_s[r+v, c+u]  W[d,s,v,u]
//   wgrad     D[m=(s,v,u), n=d]      = sum_{k=(r,c)}   X_s[r+v, c+u]  delta_d[r,c]
//   pull      D[m=(i,j), n=s]        = sum_{k=(d,v,u)} delta_d[i-v, j-u] W[d,s,v,u]
//
// All three are one kernel (tgemm): A[m, k] = X[rowbase[m] + kdec[k]] gathered
// by all threads into the UMMA core-matrix layout (the pull reads a delta map
// with a zero border of kx-1 / ky-1, so every tap is in range), B pre-laid-out
// per image by tfill from an index map into the parameters (forward, pull) or
// the delta maps (wgrad), split-K over CTAs when M x N has few tiles, partial
// sums added in split order by their consumers.  The glue stays on the SIMT pipes: activation +
// max-pool with argmax (the reference's activation and strict '>' scan), the
// FC layers and output deltas (the C-ABI seam kernels of ck_seam.cu), routing
// the pooled deltas to the conv winners, the SGD updates.
//
// Supported: input -> (conv k, stride 1 -> maxpool)+ -> fc+ -> output, any
// connection tables (unconnected pairs are zero in B and not updated).
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "ck_host.h"
#include "ck_numerics.cuh"
#include "ck_tc_common.cuh"

extern "C" {
int ck_fc_fwd(const float* x, int n_in, const float* weights, const float* bias, int n_out,
              float* a_out, float* y_out, ck_stream_t stream);
int ck_fc_bwd_update(const float* x, int n_in, float* weights, float* bias, int n_out,
                     const float* delta, float* xgrad, float* grad_w, float* grad_b,
                     double eta, ck_stream_t stream);
int ck_act_deriv_mul(const float* a, float* delta, int n_maps, int rows, int pitch, int w,
                     int h, ck_stream_t stream);
int ck_output_deltas(const float* y, const float* a, const double* targets, int n,
                     float* delta, double* loss, double* scratch, ck_stream_t stream);
}

namespace ck {
namespace tct {

using namespace ck::tc;

constexpr int kPad = INT_MIN;      // kdec entry of a padded K column

struct TG {
  int M, N, K_pad, N_pad, Nt, n_tiles, splits, cps;  // cps: K chunks per split
  const float* X;
  const int* rowbase;              // M entries
  const int* kdec;                 // K_pad entries (kPad: padding)
  const __half* Bw;                // [chunk][part][N_pad * BKT] core-matrix layout
  float* D;                        // [split][M][N]
};

// One (row tile, column tile, K split) per CTA; single-stage: gather the A
// chunk while the B chunk's bulk copy is in flight, three MMAs per 16-wide K
// step (hi*hi, hi*lo, lo*hi), then the next chunk once the MMAs are done.
template <int BKT>
__global__ void __launch_bounds__(THREADS, 1) tgemm_kernel(TG G, int tmem_cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int KC = BKT / 8;
  constexpr int RG = KC * 128;
  const int a_bytes = BM * BKT * 2;
  const int b_bytes = G.Nt * BKT * 2;
  uint8_t* As = smem;                          // hi, lo
  uint8_t* Bs = smem + 2 * a_bytes;            // hi, lo
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + 2 * b_bytes);
  uint64_t* load_bar = bars;
  uint64_t* mma_bar = bars + 1;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x % G.splits;
  const int rest = blockIdx.x / G.splits;
  const int nt = rest % G.n_tiles, mt = rest / G.n_tiles;
  if (tid == 0) {
    mbar_init(load_bar, 1);
    mbar_init(mma_bar, 1);
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
  const int row = tid & (BM - 1);
  const int m = mt * BM + row;
  const bool valid = m < G.M;
  const int rb = valid ? __ldg(G.rowbase + m) : 0;
  const int n0 = nt * G.Nt;
  const int nw = min(G.Nt, G.N_pad - n0);
  const int c0 = split * G.cps;
  const int c1 = min(G.K_pad / BKT, c0 + G.cps);
  for (int ch = c0; ch < c1; ++ch) {
    const int lc = ch - c0;
    if (lc > 0) mbar_wait(mma_bar, (unsigned)((lc - 1) & 1));   // stage free
    if (tid == 0) {
      const __half* bsrc = G.Bw + (int64_t)ch * 2 * G.N_pad * BKT + (int64_t)n0 * BKT;
      expect_tx(load_bar, 2 * nw * BKT * 2);
      bulk_copy(Bs, bsrc, nw * BKT * 2, load_bar);
      bulk_copy(Bs + b_bytes, bsrc + (int64_t)G.N_pad * BKT, nw * BKT * 2, load_bar);
    }
    float x[KC / 2][8];
#pragma unroll
    for (int it = 0; it < KC / 2; ++it) {
      const int kg = (tid >> 7) + 2 * it;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int dec = __ldg(G.kdec + ch * BKT + kg * 8 + e);
        x[it][e] = (valid && dec != kPad) ? __ldg(G.X + rb + dec) : 0.f;
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
        const __half l0 = __float2half_rn(x[it][e] - __half2float(h0));
        const __half l1 = __float2half_rn(x[it][e + 1] - __half2float(h1));
        lo[e >> 1] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
      }
      *reinterpret_cast<uint4*>(As + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(As + a_bytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      mbar_wait(load_bar, (unsigned)(lc & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = smem_u32(As), bh = smem_u32(Bs);
      const uint32_t id = instr_desc(nw);
#pragma unroll
      for (int ks = 0; ks < BKT / 16; ++ks) {
        const uint64_t a_hi = umma_desc(ah + ks * 256, 128, RG);
        const uint64_t b_hi = umma_desc(bh + ks * 256, 128, RG);
        mma_f16(tmem, a_hi, b_hi, id, (lc > 0 || ks > 0) ? 1 : 0);
        mma_f16(tmem, a_hi, umma_desc(bh + b_bytes + ks * 256, 128, RG), id, 1);
        mma_f16(tmem, umma_desc(ah + a_bytes + ks * 256, 128, RG), b_hi, id, 1);
      }
      mma_commit(mma_bar);
    }
  }
  if (c1 > c0) mbar_wait(mma_bar, (unsigned)((c1 - c0 - 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    // warp w reads TMEM lanes 32*(w%4)..+31 (its rows); the two warp groups
    // take alternate 16-column chunks
    const int quarter = warp & 3, grp = warp >> 2;
    const int erow = quarter * 32 + lane;
    const int me = mt * BM + erow;
    float* drow = G.D + ((int64_t)split * G.M + me) * G.N;
    for (int c16 = grp; c16 * 16 < nw; c16 += 2) {
      float v[16];
      if (c1 > c0) {
        tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + c16 * 16, v);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      if (me < G.M) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c16 * 16 + i;
          if (n < G.N) drow[n] = v[i];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// B[n, k] = src[map[n * K_pad + k]] (0 where map < 0), fp16 hi / lo parts in
// the chunked core-matrix layout tgemm's bulk copies expect.
__global__ void tfill_kernel(const float* __restrict__ src, const int* __restrict__ map, int N_pad,
                             int K_pad, int bk, __half* __restrict__ out) {
  const int64_t total = (int64_t)N_pad * K_pad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % K_pad);
    const int n = (int)(i / K_pad);
    const int idx = map[i];
    const float w = idx >= 0 ? src[idx] : 0.f;
    const __half hi = __float2half_rn(w);
    const __half lo = __float2half_rn(w - __half2float(hi));
    const int ch = k / bk, kk = k % bk;
    const int64_t base = (int64_t)ch * 2 * N_pad * bk;
    const int64_t in = ((n >> 3) * (bk * 16) + (kk >> 3) * 128 + (n & 7) * 16 + (kk & 7) * 2) / 2;
    out[base + in] = hi;
    out[base + (int64_t)N_pad * bk + in] = lo;
  }
}

// the visit's input image (bytes through the LUT, or f32) and its targets
__global__ void load_visit(const uint8_t* images, const float* lut, const int32_t* order,
                           const int32_t* labels, const int* t_ptr, int cells, int n_classes,
                           float* x, double* targets) {
  const int t = *t_ptr;
  const int64_t img = order ? order[t] : t;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += gridDim.x * blockDim.x)
    x[i] = lut ? lut[images[img * cells + i]]
               : reinterpret_cast<const float*>(images)[img * cells + i];
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < n_classes; j += blockDim.x)
      targets[j] = j == labels[img] ? 1.0 : -1.0;
}

// end of a visit: its loss into the per-visit array, then the next visit
__global__ void next_visit(int* t_ptr, const double* loss_slot, double* losses) {
  losses[*t_ptr] = *loss_slot;
  *t_ptr += 1;
}

// a = D + bias (per dest column), y = 1.7159 tanh(0.6666 a) in f32 (the
// exact engine uses the reference's f64 tanh; this path is within its
// tolerance), then the max-pool over y: strict '>', first cell in row-major
// scan; the pooled y, the winner's cell and -- for the backward -- a at every
// conv cell.
__device__ __forceinline__ float split_sum(const float* __restrict__ part, int splits, int64_t mn,
                                           int64_t i) {
  float v = part[i];
  for (int p = 1; p < splits; ++p) v += part[(int64_t)p * mn + i];
  return v;
}

__global__ void act_pool_kernel(const float* __restrict__ D, int splits,
                                const float* __restrict__ params,
                                const int* __restrict__ bias_idx, int maps, int OH, int OW,
                                int px, int py, int PH, int PW, float* a_out, float* pool_y,
                                int* pool_arg) {
  const int64_t mn = (int64_t)OH * OW * maps;
  const int total = maps * PH * PW;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    const int d = q / (PH * PW), pp = q % (PH * PW);
    const int r0 = (pp / PW) * py, c0 = (pp % PW) * px;
    const float b = params[bias_idx[d]];
    float best = 0.f;
    int bi = 0;
    for (int v = 0; v < py; ++v)
      for (int u = 0; u < px; ++u) {
        const int cell = (r0 + v) * OW + c0 + u;
        const float a = __fadd_rn(split_sum(D, splits, mn, (int64_t)cell * maps + d), b);
        a_out[d * OH * OW + cell] = a;
        const float y = fc_act(a);   // f32 tanh: this path is within tolerance, not exact
        if ((v == 0 && u == 0) || y > best) {
          best = y;
          bi = cell;
        }
      }
    pool_y[q] = best;
    pool_arg[q] = bi;
  }
}

// pooled deltas -> the conv winners: delta_conv = f32(v * f'(a)) in the dense
// delta maps and in the zero-bordered copy the pull gathers from.  `xg` is
// the pooled delta of cell q; from a pull GEMM it sits at D[pix * ld + map].
// position of B[n, k] (the hi half; the lo half follows N_pad * bk later)
// in tgemm's chunked core-matrix layout
__host__ __device__ __forceinline__ int64_t bpos(int n, int k, int N_pad, int bk) {
  const int ch = k / bk, kk = k % bk;
  return (int64_t)ch * 2 * N_pad * bk +
         ((n >> 3) * (bk * 16) + (kk >> 3) * 128 + (n & 7) * 16 + (kk & 7) * 2) / 2;
}

__device__ __forceinline__ void put_split(__half* B, int64_t pos, int64_t lo_off, float w) {
  const __half hi = __float2half_rn(w);
  B[pos] = hi;
  B[pos + lo_off] = __float2half_rn(w - __half2float(hi));
}

// pooled deltas -> the conv winners; also the winner's entry of the weight-
// gradient GEMM's B (its n = dest map, k = conv cell) -- the rest is zero
__global__ void route_kernel(const float* __restrict__ xg, int ld, int splits, int64_t mn,
                             int maps, int PH, int PW, const int* __restrict__ pool_arg,
                             const float* __restrict__ a_conv, int OH, int OW, int bx, int by,
                             float* dense, float* padded, __half* Bwg, int wg_npad, int wg_bk) {
  const int total = maps * PH * PW;
  const int PWd = OW + 2 * bx, PHd = OH + 2 * by;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    const int d = q / (PH * PW), pix = q % (PH * PW);
    const float v = ld > 0 ? split_sum(xg, splits, mn, (int64_t)pix * ld + d) : xg[q];
    const int cell = pool_arg[q];
    const float dv = __fmul_rn(__fadd_rn(0.0f, v), act_deriv(a_conv[d * OH * OW + cell]));
    dense[d * OH * OW + cell] = dv;
    const int r = cell / OW, c = cell % OW;
    padded[(int64_t)d * PHd * PWd + (r + by) * PWd + c + bx] = dv;
    put_split(Bwg, bpos(d, cell, wg_npad, wg_bk), (int64_t)wg_npad * wg_bk, dv);
  }
}

// SGD on the conv arena: every connected pair's taps from the wgrad GEMM
// (row (s, v, u), column d), the biases from the dense delta maps (f64 sums)
__global__ void conv_update_kernel(const float* __restrict__ Dw, int splits, int64_t mn, int maps,
                                   int kk, const int* __restrict__ pair_dst,
                                   const int* __restrict__ pair_src,
                                   const int* __restrict__ pair_widx, int n_pairs,
                                   const int* __restrict__ bias_idx, const float* __restrict__ dense,
                                   int ohw, float eta_f, float* params,
                                   __half* Bf, int f_npad, int f_bk, __half* Bp, int p_npad,
                                   int p_bk) {
  const int total = n_pairs * kk;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int p = i / kk, t = i % kk;
    const int d = pair_dst[p], sm = pair_src[p];
    const float g = split_sum(Dw, splits, mn, ((int64_t)sm * kk + t) * maps + d);
    float* w = params + pair_widx[p] + t;
    const float nw = sgd(*w, eta_f, g);
    *w = nw;
    // the forward / pull GEMMs' B copies of this weight
    put_split(Bf, bpos(d, sm * kk + t, f_npad, f_bk), (int64_t)f_npad * f_bk, nw);
    if (Bp) put_split(Bp, bpos(sm, d * kk + t, p_npad, p_bk), (int64_t)p_npad * p_bk, nw);
  }
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int d = warp; d < maps; d += nwarps) {
    double acc = 0.0;
    for (int c = lane; c < ohw; c += 32) acc += (double)dense[d * ohw + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) params[bias_idx[d]] = sgd(params[bias_idx[d]], eta_f, (float)acc);
  }
}

}  // namespace tct
}  // namespace ck

using namespace ck;
using namespace ck::tct;

// ---------------------------------------------------------------------------
// host plan

namespace {

struct TGemmPlan {
  TG g{};
  int bk = 64, tmem_cols = 32;
  size_t smem = 0;
  int grid = 0;
  int* d_rowbase = nullptr;
  int* d_kdec = nullptr;
  int* d_map = nullptr;           // tfill index map (N_pad x K_pad)
  __half* d_B = nullptr;
  float* d_part = nullptr;        // [splits][M][N]
  float* d_out = nullptr;         // reduced (== d_part when splits == 1)
  const float* fill_src = nullptr;
};

struct ConvPlan {
  int li;                         // layer index of the conv (pool at li + 1)
  int S, SH, SW, Dm, OH, OW, kx, ky, px, py, PH, PW, n_pairs, kk;
  bool pull;                      // the source layer keeps deltas
  TGemmPlan fwd, wg, pl;
  const float* x_src = nullptr;   // the source layer's y (input image or pool y)
  float* a_conv = nullptr;
  float* pool_y = nullptr;
  int* pool_arg = nullptr;
  float* dense = nullptr;
  float* padded = nullptr;
  int* d_bias_idx = nullptr;
  int* d_pair_dst = nullptr;
  int* d_pair_src = nullptr;
  int* d_pair_widx = nullptr;
};

struct FcPlan {
  int n_in, n_out;
  int64_t w_off, b_off;
  float *a, *y, *delta, *xgrad;
};

}  // namespace

struct ck_tct {
  int device = 0;
  int sms = 148;
  int n_classes = 0;
  int in_cells = 0;
  float* params = nullptr;        // the net's device parameters (shared with ck_net)
  std::vector<ConvPlan> convs;
  std::vector<FcPlan> fcs;
  float* x_in = nullptr;
  double* targets = nullptr;
  double* scratch = nullptr;
  double* losses = nullptr;
  int64_t losses_cap = 0;
  int* t_ptr = nullptr;
  double* loss_slot = nullptr;
  std::vector<void*> allocs;
  // one visit's launches, captured once per (dataset, order, eta) and replayed
  // per image: every kernel finds its image through t_ptr
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  const void* key[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  double key_eta = 0.0;
};

namespace {

int tmalloc(ck_tct* P, void** p, size_t bytes) {
  if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess)
    return set_error(CK_E_NOMEM, "tensor-core training: device allocation");
  cudaMemset(*p, 0, std::max<size_t>(bytes, 16));
  P->allocs.push_back(*p);
  return CK_OK;
}

template <class T>
int upload(ck_tct* P, T** dst, const std::vector<T>& v) {
  if (int rc = tmalloc(P, (void**)dst, sizeof(T) * v.size())) return rc;
  if (cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return set_error(CK_E_CUDA, "tensor-core training: upload");
  return CK_OK;
}

int round_up_i(int v, int q) { return (v + q - 1) / q * q; }

// One GEMM D[M x N] = A[M x K] B[N x K]^T with the gather tables and the B map.
int make_tgemm(ck_tct* P, TGemmPlan& G, int M, int N, int K, const std::vector<int>& rowbase,
               const std::vector<int>& kdec_in, const std::vector<int>& map_in,
               const float* fill_src) {
  G.bk = K <= 16 ? 16 : K <= 32 ? 32 : 64;
  const int K_pad = round_up_i(K, G.bk);
  const int N_pad = round_up_i(N, 16);
  CK_CHECK(N_pad <= 512 * 4, CK_E_DIMENSION, "tensor-core training: layer too wide");
  const int n_tiles = (N_pad + 255) / 256;
  const int Nt = round_up_i((N_pad + n_tiles - 1) / n_tiles, 16);
  int cols = 32;
  while (cols < Nt) cols <<= 1;
  G.tmem_cols = cols;
  const int m_tiles = (M + BM - 1) / BM;
  const int chunks = K_pad / G.bk;
  // split K so that about one CTA per SM has work
  int splits = std::max(1, std::min(chunks, P->sms / std::max(1, m_tiles * n_tiles)));
  const int cps = (chunks + splits - 1) / splits;
  splits = (chunks + cps - 1) / cps;
  G.g.M = M;
  G.g.N = N;
  G.g.K_pad = K_pad;
  G.g.N_pad = N_pad;
  G.g.Nt = Nt;
  G.g.n_tiles = n_tiles;
  G.g.splits = splits;
  G.g.cps = cps;
  G.grid = m_tiles * n_tiles * splits;
  G.smem = (size_t)2 * BM * G.bk * 2 + (size_t)2 * Nt * G.bk * 2 + 64;
  CK_CHECK(G.smem <= 220 * 1024, CK_E_DIMENSION, "tensor-core training: tile too large");
  std::vector<int> kdec(K_pad, kPad);
  std::copy(kdec_in.begin(), kdec_in.end(), kdec.begin());
  std::vector<int> map((size_t)N_pad * K_pad, -1);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) map[(size_t)n * K_pad + k] = map_in[(size_t)n * K + k];
  if (int rc = upload(P, &G.d_rowbase, rowbase)) return rc;
  if (int rc = upload(P, &G.d_kdec, kdec)) return rc;
  if (int rc = upload(P, &G.d_map, map)) return rc;
  if (int rc = tmalloc(P, (void**)&G.d_B, sizeof(__half) * 2 * (size_t)N_pad * K_pad)) return rc;
  if (int rc = tmalloc(P, (void**)&G.d_part, sizeof(float) * (size_t)splits * M * N)) return rc;
  G.d_out = G.d_part;
  G.g.rowbase = G.d_rowbase;
  G.g.kdec = G.d_kdec;
  G.g.Bw = G.d_B;
  G.g.D = G.d_part;
  G.fill_src = fill_src;
  return CK_OK;
}

typedef void (*TgemmFn)(TG, int);
TgemmFn tgemm_fn(int bk) {
  return bk == 16 ? tgemm_kernel<16> : bk == 32 ? tgemm_kernel<32> : tgemm_kernel<64>;
}

// B from its source through the index map (weights: once per epoch call,
// after which the updates keep it current)
void fill_B(ck_tct* P, TGemmPlan& G, cudaStream_t s) {
  tfill_kernel<<<P->sms * 2, 256, 0, s>>>(G.fill_src, G.d_map, G.g.N_pad, G.g.K_pad, G.bk, G.d_B);
  count_launch();
}

// the GEMM alone: partial sums per K split (the consumers add them in order)
int run_tgemm(ck_tct* P, TGemmPlan& G, const float* X, cudaStream_t s) {
  (void)P;
  G.g.X = X;
  tgemm_fn(G.bk)<<<G.grid, THREADS, G.smem, s>>>(G.g, G.tmem_cols);
  count_launch();
  return CK_OK;
}

}  // namespace

extern "C" {

int ck_tct_create(const ck_layer_desc* layers, int n_layers, int device, float* params,
                  ck_tct** out) {
  CK_CHECK(layers && out && params && n_layers >= 3, CK_E_CONFIG, "bad arguments");
  CK_CHECK(layers[0].kind == CK_LAYER_INPUT, CK_E_CONFIG, "first layer must be the input");
  CK_CUDA_TRY(cudaSetDevice(device));
  ck_tct* P = new ck_tct();
  P->device = device;
  P->params = params;
  CK_CUDA_TRY(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device));
  auto fail = [&](int rc) {
    ck_tct_destroy(P);
    return rc;
  };
  P->in_cells = layers[0].maps * layers[0].width * layers[0].height;
  if (int rc = tmalloc(P, (void**)&P->x_in, sizeof(float) * P->in_cells)) return fail(rc);
  const float* prev_y = P->x_in;
  int64_t poff = 0;
  int i = 1;
  for (; i < n_layers && layers[i].kind == CK_LAYER_CONV; i += 2) {
    const ck_layer_desc& L = layers[i];
    const ck_layer_desc& S = layers[i - 1];
    if (i + 1 >= n_layers || layers[i + 1].kind != CK_LAYER_POOL)
      return fail(set_error(CK_E_CONFIG, "tensor-core training: every conv needs a max-pool above"));
    if (L.sx != 0 || L.sy != 0)
      return fail(set_error(CK_E_CONFIG, "tensor-core training: strided convs are not supported"));
    const ck_layer_desc& Pl = layers[i + 1];
    ConvPlan C;
    C.li = i;
    C.S = S.maps; C.SH = S.height; C.SW = S.width;
    C.Dm = L.maps; C.OH = L.height; C.OW = L.width; C.kx = L.kx; C.ky = L.ky;
    C.px = Pl.px; C.py = Pl.py; C.PH = Pl.height; C.PW = Pl.width;
    C.n_pairs = L.n_pairs;
    C.kk = L.kx * L.ky;
    C.pull = i > 1;
    C.x_src = prev_y;
    const int kk = C.kk, SHW = C.SH * C.SW, OHW = C.OH * C.OW;
    // weight arena index of (d, s, v, u), -1 where not connected
    std::vector<int> widx((size_t)C.Dm * C.S, -1), pd(C.n_pairs), ps(C.n_pairs), pw(C.n_pairs),
        bidx(C.Dm);
    for (int d = 0; d < C.Dm; ++d) {
      for (int64_t p = L.fwd_offsets[d]; p < L.fwd_offsets[d + 1]; ++p) {
        widx[(size_t)d * C.S + L.fwd_srcs[p]] = (int)(poff + L.fwd_widx[p]);
        pd[p] = d;
        ps[p] = (int)L.fwd_srcs[p];
        pw[p] = (int)(poff + L.fwd_widx[p]);
      }
      bidx[d] = (int)(poff + L.bias_offset[d]);
    }
    // forward: rows (r, c), K = (s, v, u), columns d
    {
      std::vector<int> rb(OHW), kd(C.S * kk), map((size_t)C.Dm * C.S * kk);
      for (int r = 0; r < C.OH; ++r)
        for (int c = 0; c < C.OW; ++c) rb[r * C.OW + c] = r * C.SW + c;
      for (int s = 0; s < C.S; ++s)
        for (int t = 0; t < kk; ++t) kd[s * kk + t] = s * SHW + (t / C.kx) * C.SW + t % C.kx;
      for (int d = 0; d < C.Dm; ++d)
        for (int s = 0; s < C.S; ++s)
          for (int t = 0; t < kk; ++t) {
            const int w = widx[(size_t)d * C.S + s];
            map[((size_t)d * C.S + s) * kk + t] = w < 0 ? -1 : w + t;
          }
      if (int rc = make_tgemm(P, C.fwd, OHW, C.Dm, C.S * kk, rb, kd, map, params)) return fail(rc);
    }
    if (int rc = tmalloc(P, (void**)&C.a_conv, sizeof(float) * C.Dm * OHW)) return fail(rc);
    if (int rc = tmalloc(P, (void**)&C.pool_y, sizeof(float) * C.Dm * C.PH * C.PW)) return fail(rc);
    if (int rc = tmalloc(P, (void**)&C.pool_arg, sizeof(int) * C.Dm * C.PH * C.PW)) return fail(rc);
    if (int rc = tmalloc(P, (void**)&C.dense, sizeof(float) * C.Dm * OHW)) return fail(rc);
    const int PHd = C.OH + 2 * (C.ky - 1), PWd = C.OW + 2 * (C.kx - 1);
    if (int rc = tmalloc(P, (void**)&C.padded, sizeof(float) * (size_t)C.Dm * PHd * PWd)) return fail(rc);
    // weight gradient: rows (s, v, u), K = (r, c), columns d (B = the dense deltas)
    {
      std::vector<int> rb(C.S * kk), kd(OHW), map((size_t)C.Dm * OHW);
      for (int s = 0; s < C.S; ++s)
        for (int t = 0; t < kk; ++t) rb[s * kk + t] = s * SHW + (t / C.kx) * C.SW + t % C.kx;
      for (int r = 0; r < C.OH; ++r)
        for (int c = 0; c < C.OW; ++c) kd[r * C.OW + c] = r * C.SW + c;
      for (int d = 0; d < C.Dm; ++d)
        for (int q = 0; q < OHW; ++q) map[(size_t)d * OHW + q] = d * OHW + q;
      if (int rc = make_tgemm(P, C.wg, C.S * kk, C.Dm, OHW, rb, kd, map, C.dense)) return fail(rc);
    }
    // pull: rows (i, j) of the source maps, K = (d, v, u), columns s (A from
    // the zero-bordered delta maps)
    if (C.pull) {
      std::vector<int> rb(SHW), kd(C.Dm * kk), map((size_t)C.S * C.Dm * kk);
      for (int r = 0; r < C.SH; ++r)
        for (int c = 0; c < C.SW; ++c) rb[r * C.SW + c] = (r + C.ky - 1) * PWd + c + C.kx - 1;
      for (int d = 0; d < C.Dm; ++d)
        for (int t = 0; t < kk; ++t) kd[d * kk + t] = d * PHd * PWd - (t / C.kx) * PWd - t % C.kx;
      for (int s = 0; s < C.S; ++s)
        for (int d = 0; d < C.Dm; ++d)
          for (int t = 0; t < kk; ++t) {
            const int w = widx[(size_t)d * C.S + s];
            map[((size_t)s * C.Dm + d) * kk + t] = w < 0 ? -1 : w + t;
          }
      if (int rc = make_tgemm(P, C.pl, SHW, C.S, C.Dm * kk, rb, kd, map, params)) return fail(rc);
    }
    if (int rc = upload(P, &C.d_bias_idx, bidx)) return fail(rc);
    if (int rc = upload(P, &C.d_pair_dst, pd)) return fail(rc);
    if (int rc = upload(P, &C.d_pair_src, ps)) return fail(rc);
    if (int rc = upload(P, &C.d_pair_widx, pw)) return fail(rc);
    poff += L.arena_size;
    prev_y = C.pool_y;
    P->convs.push_back(C);
  }
  CK_CHECK(!P->convs.empty(), CK_E_CONFIG, "tensor-core training: no conv layer");
  int n_prev = layers[i - 1].maps * layers[i - 1].width * layers[i - 1].height;
  for (; i < n_layers; ++i) {
    const ck_layer_desc& L = layers[i];
    if (L.kind != CK_LAYER_FC)
      return fail(set_error(CK_E_CONFIG, "tensor-core training: expected FC layers after the convs"));
    FcPlan F;
    F.n_in = n_prev;
    F.n_out = L.maps;
    F.w_off = poff;
    F.b_off = poff + (int64_t)F.n_in * F.n_out;
    poff += (int64_t)F.n_in * F.n_out + F.n_out;
    if (int rc = tmalloc(P, (void**)&F.a, sizeof(float) * F.n_out)) return fail(rc);
    if (int rc = tmalloc(P, (void**)&F.y, sizeof(float) * F.n_out)) return fail(rc);
    if (int rc = tmalloc(P, (void**)&F.delta, sizeof(float) * F.n_out)) return fail(rc);
    if (int rc = tmalloc(P, (void**)&F.xgrad, sizeof(float) * F.n_in)) return fail(rc);
    P->fcs.push_back(F);
    n_prev = F.n_out;
  }
  P->n_classes = n_prev;
  if (int rc = tmalloc(P, (void**)&P->targets, sizeof(double) * P->n_classes)) return fail(rc);
  if (int rc = tmalloc(P, (void**)&P->scratch, sizeof(double) * P->n_classes)) return fail(rc);
  if (int rc = tmalloc(P, (void**)&P->t_ptr, sizeof(int))) return fail(rc);
  if (int rc = tmalloc(P, (void**)&P->loss_slot, sizeof(double))) return fail(rc);
  if (cudaStreamCreateWithFlags(&P->cap, cudaStreamNonBlocking) != cudaSuccess)
    return fail(set_error(CK_E_CUDA, "tensor-core training: capture stream"));
  for (int bk : {16, 32, 64})
    if (cudaFuncSetAttribute(tgemm_fn(bk), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             220 * 1024) != cudaSuccess)
      return fail(set_error(CK_E_CUDA, "tensor-core training: kernel attributes"));
  *out = P;
  return CK_OK;
}

int ck_tct_destroy(ck_tct* P) {
  if (!P) return CK_OK;
  cudaSetDevice(P->device);
  if (P->exec) cudaGraphExecDestroy(P->exec);
  if (P->cap) cudaStreamDestroy(P->cap);
  for (void* p : P->allocs) cudaFree(p);
  delete P;
  return CK_OK;
}

static int enqueue_visit(ck_tct* P, const uint8_t* images, const float* lut,
                         const int32_t* labels, const int32_t* order, double eta,
                         cudaStream_t s) {
  const float eta_f = (float)eta;
  ck_stream_t stream = (ck_stream_t)s;
  load_visit<<<8, 256, 0, s>>>(images, lut, order, labels, P->t_ptr, P->in_cells, P->n_classes,
                               P->x_in, P->targets);
  count_launch();
  // forward through the convs
  for (auto& C : P->convs) {
    if (int rc = run_tgemm(P, C.fwd, C.x_src, s)) return rc;
    const int pc = C.Dm * C.PH * C.PW;
    act_pool_kernel<<<blocks_for(pc, 256), 256, 0, s>>>(
        C.fwd.d_part, C.fwd.g.splits, P->params, C.d_bias_idx, C.Dm, C.OH, C.OW, C.px, C.py,
        C.PH, C.PW, C.a_conv, C.pool_y, C.pool_arg);
    count_launch();
  }
  // FC layers, output deltas and loss
  const float* x = P->convs.back().pool_y;
  for (auto& F : P->fcs) {
    if (int rc = ck_fc_fwd(x, F.n_in, P->params + F.w_off, P->params + F.b_off, F.n_out, F.a,
                           F.y, stream)) return rc;
    x = F.y;
  }
  FcPlan& O = P->fcs.back();
  if (int rc = ck_output_deltas(O.y, O.a, P->targets, O.n_out, O.delta, P->loss_slot,
                                P->scratch, stream)) return rc;
  // FC backward (each layer's xgrad from its weights before its update)
  for (int f = (int)P->fcs.size() - 1; f >= 0; --f) {
    FcPlan& F = P->fcs[f];
    const float* fx = f > 0 ? P->fcs[f - 1].y : P->convs.back().pool_y;
    if (int rc = ck_fc_bwd_update(fx, F.n_in, P->params + F.w_off, P->params + F.b_off,
                                  F.n_out, F.delta, F.xgrad, nullptr, nullptr, eta, stream))
      return rc;
    if (f > 0) {
      FcPlan& B = P->fcs[f - 1];
      CK_CUDA_TRY(cudaMemcpyAsync(B.delta, F.xgrad, sizeof(float) * B.n_out,
                                  cudaMemcpyDeviceToDevice, s));
      if (int rc = ck_act_deriv_mul(B.a, B.delta, 1, 1, B.n_out, B.n_out, 1, stream)) return rc;
    }
  }
  // conv backward, top down: route -> weight gradient -> pull (old weights) -> update
  const float* xg = P->fcs.front().xgrad;
  int ld = 0, xsplits = 1;
  int64_t xmn = 0;
  for (int c = (int)P->convs.size() - 1; c >= 0; --c) {
    ConvPlan& C = P->convs[c];
    const int OHW = C.OH * C.OW;
    const int PHd = C.OH + 2 * (C.ky - 1), PWd = C.OW + 2 * (C.kx - 1);
    CK_CUDA_TRY(cudaMemsetAsync(C.dense, 0, sizeof(float) * C.Dm * OHW, s));
    CK_CUDA_TRY(cudaMemsetAsync(C.padded, 0, sizeof(float) * (size_t)C.Dm * PHd * PWd, s));
    CK_CUDA_TRY(cudaMemsetAsync(C.wg.d_B, 0,
                                sizeof(__half) * 2 * (size_t)C.wg.g.N_pad * C.wg.g.K_pad, s));
    const int pc = C.Dm * C.PH * C.PW;
    route_kernel<<<blocks_for(pc, 256), 256, 0, s>>>(
        xg, ld, xsplits, xmn, C.Dm, C.PH, C.PW, C.pool_arg, C.a_conv, C.OH, C.OW, C.kx - 1,
        C.ky - 1, C.dense, C.padded, C.wg.d_B, C.wg.g.N_pad, C.wg.bk);
    count_launch();
    if (int rc = run_tgemm(P, C.wg, C.x_src, s)) return rc;
    if (C.pull) {
      if (int rc = run_tgemm(P, C.pl, C.padded, s)) return rc;   // old weights
      xg = C.pl.d_part;
      ld = C.S;
      xsplits = C.pl.g.splits;
      xmn = (int64_t)C.pl.g.M * C.pl.g.N;
    }
    const int work = std::max(C.n_pairs * C.kk, C.Dm * 32);
    conv_update_kernel<<<blocks_for(work, 256), 256, 0, s>>>(
        C.wg.d_part, C.wg.g.splits, (int64_t)C.wg.g.M * C.wg.g.N, C.Dm, C.kk, C.d_pair_dst,
        C.d_pair_src, C.d_pair_widx, C.n_pairs, C.d_bias_idx, C.dense, OHW, eta_f, P->params,
        C.fwd.d_B, C.fwd.g.N_pad, C.fwd.bk, C.pull ? C.pl.d_B : nullptr,
        C.pull ? C.pl.g.N_pad : 0, C.pull ? C.pl.bk : 0);
    count_launch();
  }
  next_visit<<<1, 1, 0, s>>>(P->t_ptr, P->loss_slot, P->losses);
  count_launch();
  return CK_OK;
}

int ck_tct_train_epoch(ck_tct* P, const uint8_t* images, const float* lut, const int32_t* labels,
                       const int32_t* order, int64_t n, double eta, double* mean_loss,
                       ck_stream_t stream) {
  CK_CHECK(P && images && labels && n >= 1, CK_E_CONFIG, "bad arguments");
  CK_CHECK(eta > 0, CK_E_CONFIG, "learning rate must be > 0");
  CK_CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (n > P->losses_cap) {
    CK_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(P->losses);
    P->losses = nullptr;
    CK_CUDA_TRY(cudaMalloc((void**)&P->losses, sizeof(double) * n));
    P->losses_cap = n;
    if (P->exec) cudaGraphExecDestroy(P->exec);   // captured the old losses pointer
    P->exec = nullptr;
  }
  // (re)capture one visit when its inputs changed; CKB200_TCT_NOGRAPH=1: A/B
  const bool graph = !getenv("CKB200_TCT_NOGRAPH");
  const void* key[5] = {images, lut, labels, order, P->losses};
  if (graph && (!P->exec || memcmp(key, P->key, sizeof(key)) != 0 || eta != P->key_eta)) {
    if (P->exec) cudaGraphExecDestroy(P->exec);
    P->exec = nullptr;
    cudaGraph_t g = nullptr;
    CK_CUDA_TRY(cudaStreamBeginCapture(P->cap, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_visit(P, images, lut, labels, order, eta, P->cap);
    cudaError_t e = cudaStreamEndCapture(P->cap, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_status(e, "tensor-core training: capture");
    e = cudaGraphInstantiate(&P->exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_status(e, "tensor-core training: instantiate");
    memcpy(P->key, key, sizeof(key));
    P->key_eta = eta;
  }
  // the forward / pull GEMMs' B from the current weights (they may have been
  // changed by the exact engine or the host since the last call); the
  // per-image updates keep them current within the epoch
  for (auto& C : P->convs) {
    fill_B(P, C.fwd, s);
    if (C.pull) fill_B(P, C.pl, s);
  }
  CK_CUDA_TRY(cudaMemsetAsync(P->t_ptr, 0, sizeof(int), s));
  for (int64_t t = 0; t < n; ++t) {
    if (graph) {
      CK_CUDA_TRY(cudaGraphLaunch(P->exec, s));
    } else if (int rc = enqueue_visit(P, images, lut, labels, order, eta, s)) {
      return rc;
    }
  }
  CK_CUDA_TRY(cudaGetLastError());
  if (mean_loss) {
    std::vector<double> h(n);
    CK_CUDA_TRY(cudaMemcpyAsync(h.data(), P->losses, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    CK_CUDA_TRY(cudaStreamSynchronize(s));
    double tot = 0;
    for (double v : h) tot += v;
    *mean_loss = tot / (double)n;
  }
  return CK_OK;
}

}  // extern "C"
