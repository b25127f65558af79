// mb_conv.cu — latency of one bit-exact conv cell (C2 conv2: 40 sources x
// 5x5 taps, sequential f32 chain) for staging variants.  Development aid.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_conv tools/mb_conv.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NK = 40, KX = 5, KY = 5, KK = 25, SW = 13, SHW = 169;

// V0: engine's conv_cell (soff indirection, w and x from smem, scalar loads)
__device__ __forceinline__ float cell_v0(float acc, const float* src, const int* soff,
                                         const float* w) {
  for (int k = 0; k < NK; ++k) {
    const float* s = src + soff[k];
    const float* wk = w + k * KK;
    float xs[KK];
#pragma unroll
    for (int v = 0; v < KY; ++v)
#pragma unroll
      for (int u = 0; u < KX; ++u) xs[v * KX + u] = s[v * SW + u];
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, __fmul_rn(wk[t], xs[t]));
  }
  return acc;
}

// V1: products of the NEXT source computed while the current chain runs
// (explicit software pipeline: loads + FMULs of k+1 before the FADDs of k)
__device__ __forceinline__ float cell_v1(float acc, const float* src, const int* soff,
                                         const float* w) {
  float pr[KK];
  {
    const float* s = src + soff[0];
#pragma unroll
    for (int t = 0; t < KK; ++t) pr[t] = __fmul_rn(w[t], s[(t / KX) * SW + t % KX]);
  }
  for (int k = 0; k < NK; ++k) {
    float nx[KK];
    if (k + 1 < NK) {
      const float* s = src + soff[k + 1];
      const float* wk = w + (k + 1) * KK;
#pragma unroll
      for (int t = 0; t < KK; ++t) nx[t] = __fmul_rn(wk[t], s[(t / KX) * SW + t % KX]);
    }
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, pr[t]);
#pragma unroll
    for (int t = 0; t < KK; ++t) pr[t] = nx[t];
  }
  return acc;
}

// V2: like V1 but weights as float4 from a 28-float padded block
__device__ __forceinline__ float cell_v2(float acc, const float* src, const int* soff,
                                         const float* w28) {
  float pr[KK];
  auto prods = [&](int k, float* out) {
    const float* s = src + soff[k];
    const float4* w4 = reinterpret_cast<const float4*>(w28 + k * 28);
    float wv[28];
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const float4 q = w4[i];
      wv[4 * i] = q.x; wv[4 * i + 1] = q.y; wv[4 * i + 2] = q.z; wv[4 * i + 3] = q.w;
    }
#pragma unroll
    for (int t = 0; t < KK; ++t) out[t] = __fmul_rn(wv[t], s[(t / KX) * SW + t % KX]);
  };
  prods(0, pr);
  for (int k = 0; k < NK; ++k) {
    float nx[KK];
    if (k + 1 < NK) prods(k + 1, nx);
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, pr[t]);
#pragma unroll
    for (int t = 0; t < KK; ++t) pr[t] = nx[t];
  }
  return acc;
}


// V3: raw operands of source k+1 loaded into registers at the top of
// iteration k (double buffer), products + chain of k from registers
__device__ __forceinline__ float cell_v3(float acc, const float* src, const int* soff,
                                         const float* w) {
  float xc[KK], wc[KK];
  {
    const float* s = src + soff[0];
#pragma unroll
    for (int t = 0; t < KK; ++t) { xc[t] = s[(t / KX) * SW + t % KX]; wc[t] = w[t]; }
  }
#pragma unroll 2
  for (int k = 0; k < NK; ++k) {
    float xn[KK], wn[KK];
    const int kn = k + 1 < NK ? k + 1 : k;
    const float* s = src + soff[kn];
    const float* wk = w + kn * KK;
#pragma unroll
    for (int t = 0; t < KK; ++t) { xn[t] = s[(t / KX) * SW + t % KX]; wn[t] = wk[t]; }
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, __fmul_rn(wc[t], xc[t]));
#pragma unroll
    for (int t = 0; t < KK; ++t) { xc[t] = xn[t]; wc[t] = wn[t]; }
  }
  return acc;
}


// packed f32x2 (sm_100): two independent RN roundings per instruction
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
// RN(a*b) as fma(a, b, -0) and RN(a+b) as fma(a, 1, b): each exactly one
// rounding, and two FMAs are never contracted into one.
// the constants -0 and 1 come from the caller at run time (opaque to ptxas,
// which otherwise folds them and contracts the pair into one FFMA2)
__device__ unsigned long long g_neg0 = 0x8000000080000000ull, g_one = 0x3f8000003f800000ull;
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b,
                                                   unsigned long long neg0) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(neg0));
  return r;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b,
                                                   unsigned long long one) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(one), "l"(b));
  return r;
}
__device__ __forceinline__ float lo(unsigned long long v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi(unsigned long long v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
// V4: two horizontally adjacent cells per thread, packed chains
__device__ __forceinline__ void cell_v4(float acc, const float* src, const int* soff,
                                        const float* w, float* o0, float* o1) {
  unsigned long long a2 = pk(acc, acc);
  const unsigned long long neg0 = g_neg0, one = g_one;
  for (int k = 0; k < NK; ++k) {
    const float* s = src + soff[k];
    const float* wk = w + k * KK;
    float xs[KY][KX + 1];
#pragma unroll
    for (int v = 0; v < KY; ++v)
#pragma unroll
      for (int u = 0; u < KX + 1; ++u) xs[v][u] = s[v * SW + u];
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      const int v = t / KX, u = t % KX;
      const float wv = wk[t];
      a2 = add2(mul2(pk(wv, wv), pk(xs[v][u], xs[v][u + 1]), neg0), a2, one);
    }
  }
  *o0 = lo(a2);
  *o1 = hi(a2);
}


// V5: four horizontally adjacent cells per thread, two packed chains
__device__ __forceinline__ void cell_v5(float acc, const float* src, const int* soff,
                                        const float* w, float* o) {
  unsigned long long a01 = pk(acc, acc), a23 = pk(acc, acc);
  const unsigned long long neg0 = g_neg0, one = g_one;
  for (int k = 0; k < NK; ++k) {
    const float* s = src + soff[k];
    const float* wk = w + k * KK;
#pragma unroll
    for (int v = 0; v < KY; ++v) {
      float xs[KX + 3];
#pragma unroll
      for (int u = 0; u < KX + 3; ++u) xs[u] = s[v * SW + u];
#pragma unroll
      for (int u = 0; u < KX; ++u) {
        const float wv = wk[v * KX + u];
        const unsigned long long w2 = pk(wv, wv);
        a01 = add2(mul2(w2, pk(xs[u], xs[u + 1]), neg0), a01, one);
        a23 = add2(mul2(w2, pk(xs[u + 2], xs[u + 3]), neg0), a23, one);
      }
    }
  }
  o[0] = lo(a01); o[1] = hi(a01); o[2] = lo(a23); o[3] = hi(a23);
}
// V6: two cells per thread, scalar ops (ILP 2)
__device__ __forceinline__ void cell_v6(float acc, const float* src, const int* soff,
                                        const float* w, float* o) {
  float a0 = acc, a1 = acc;
  for (int k = 0; k < NK; ++k) {
    const float* s = src + soff[k];
    const float* wk = w + k * KK;
#pragma unroll
    for (int v = 0; v < KY; ++v) {
      float xs[KX + 1];
#pragma unroll
      for (int u = 0; u < KX + 1; ++u) xs[u] = s[v * SW + u];
#pragma unroll
      for (int u = 0; u < KX; ++u) {
        const float wv = wk[v * KX + u];
        a0 = __fadd_rn(a0, __fmul_rn(wv, xs[u]));
        a1 = __fadd_rn(a1, __fmul_rn(wv, xs[u + 1]));
      }
    }
  }
  o[0] = a0; o[1] = a1;
}

// V7: the engine's conv_cell_smem4 (rows of x one row ahead, v4 weights a
// source ahead, 28-float padded weight blocks)
__device__ __forceinline__ float cell_v7(float acc, const float* src, const int* soff,
                                         const float* w28) {
  constexpr int KKP = 28;
  float wc[KKP], xr[KX];
  const float* sb = src + soff[0];
  for (int j = 0; j < 7; ++j) {
    const float4 v = reinterpret_cast<const float4*>(w28)[j];
    wc[4 * j] = v.x; wc[4 * j + 1] = v.y; wc[4 * j + 2] = v.z; wc[4 * j + 3] = v.w;
  }
#pragma unroll
  for (int u = 0; u < KX; ++u) xr[u] = sb[u];
  for (int k = 0; k < NK; ++k) {
    const int kn = k + 1 < NK ? k + 1 : k;
    const float* sbn = src + soff[kn];
    float wn[KKP];
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      const float4 v = reinterpret_cast<const float4*>(w28 + kn * KKP)[j];
      wn[4 * j] = v.x; wn[4 * j + 1] = v.y; wn[4 * j + 2] = v.z; wn[4 * j + 3] = v.w;
    }
#pragma unroll
    for (int v = 0; v < KY; ++v) {
      const float* nrow = v + 1 < KY ? sb + (v + 1) * SW : sbn;
      float xn[KX];
#pragma unroll
      for (int u = 0; u < KX; ++u) xn[u] = nrow[u];
#pragma unroll
      for (int u = 0; u < KX; ++u) acc = __fadd_rn(acc, __fmul_rn(wc[v * KX + u], xr[u]));
#pragma unroll
      for (int u = 0; u < KX; ++u) xr[u] = xn[u];
    }
#pragma unroll
    for (int t = 0; t < KKP; ++t) wc[t] = wn[t];
    sb = sbn;
  }
  return acc;
}

// V8: pure dependent chain from registers (latency floor reference)
__device__ __forceinline__ float cell_v8(float acc, const float* src, const int* soff,
                                         const float* w) {
  float wr[KK], xr[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) { wr[t] = w[t]; xr[t] = src[(t / KX) * SW + t % KX]; }
  for (int k = 0; k < NK; ++k) {
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, __fmul_rn(wr[t], xr[t]));
  }
  return acc;
}

// V9: V8 plus one independent shared load per step (issue cost of the LDS)
__device__ __forceinline__ float cell_v9(float acc, const float* src, const int* soff,
                                         const float* w) {
  float wr[KK], xr[KK];
  int junk = 0;
#pragma unroll
  for (int t = 0; t < KK; ++t) { wr[t] = w[t]; xr[t] = src[(t / KX) * SW + t % KX]; }
  for (int k = 0; k < NK; ++k) {
    const float* s = src + soff[k];
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      junk ^= __float_as_int(s[(t / KX) * SW + t % KX]);
      acc = __fadd_rn(acc, __fmul_rn(wr[t], xr[t]));
    }
  }
  return acc + (junk == 12345 ? 1.0f : 0.0f);
}

// V10: x of the next source loaded a whole source ahead (double buffer),
// weights held in registers (timing stand-in: same weights every source)
__device__ __forceinline__ float cell_v10(float acc, const float* src, const int* soff,
                                          const float* w) {
  float wr[KK], xc[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) { wr[t] = w[t]; xc[t] = src[(t / KX) * SW + t % KX]; }
  for (int k = 0; k < NK; ++k) {
    const int kn = k + 1 < NK ? k + 1 : k;
    const float* s = src + soff[kn];
    float xn[KK];
#pragma unroll
    for (int t = 0; t < KK; ++t) xn[t] = s[(t / KX) * SW + t % KX];
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, __fmul_rn(wr[t], xc[t]));
#pragma unroll
    for (int t = 0; t < KK; ++t) xc[t] = xn[t];
  }
  return acc;
}

// V11: FADD-only chain from registers (no FMUL): the add latency alone
__device__ __forceinline__ float cell_v11(float acc, const float* src, const int* soff,
                                          const float* w) {
  float pr[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) pr[t] = w[t] * src[(t / KX) * SW + t % KX];
  for (int k = 0; k < NK; ++k) {
#pragma unroll
    for (int t = 0; t < KK; ++t) acc = __fadd_rn(acc, pr[t]);
  }
  return acc;
}

// V12: no register copies -- the row ring and the weight ring are resolved
// at compile time (two sources per loop iteration), so the FMA pipe sees
// exactly FMUL + FADD per tap (rt 2 cycles each: the 4-cycle floor)
template <int P>
__device__ __forceinline__ void v12_rows(float& acc, const float* wcur, const float* sb,
                                         const float* nsrc, float (&xa)[KX], float (&xb)[KX]) {
#pragma unroll
  for (int v = 0; v < KY; ++v) {
    const bool cur_a = ((P + v) & 1) == 0;
    const float* nrow = v + 1 < KY ? sb + (v + 1) * SW : nsrc;
#pragma unroll
    for (int u = 0; u < KX; ++u) {
      if (cur_a) xb[u] = nrow[u]; else xa[u] = nrow[u];
    }
#pragma unroll
    for (int u = 0; u < KX; ++u)
      acc = __fadd_rn(acc, __fmul_rn(wcur[v * KX + u], cur_a ? xa[u] : xb[u]));
  }
}
__device__ __forceinline__ void v12_w(float (&wd)[28], const float* w28, int k) {
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    const float4 v = reinterpret_cast<const float4*>(w28 + k * 28)[j];
    wd[4 * j] = v.x; wd[4 * j + 1] = v.y; wd[4 * j + 2] = v.z; wd[4 * j + 3] = v.w;
  }
}
__device__ __forceinline__ float cell_v12(float acc, const float* src, const int* soff,
                                          const float* w28) {
  float xa[KX], xb[KX], wa[28], wb[28];
  v12_w(wa, w28, 0);
  const float* sb = src + soff[0];
#pragma unroll
  for (int u = 0; u < KX; ++u) xa[u] = sb[u];
  int k = 0;
  for (; k + 2 <= NK; k += 2) {
    const float* sb1 = src + soff[k + 1];
    v12_w(wb, w28, k + 1);
    v12_rows<0>(acc, wa, sb, sb1, xa, xb);
    const int k2 = k + 2 < NK ? k + 2 : k + 1;
    const float* sb2 = src + soff[k2];
    v12_w(wa, w28, k2);
    v12_rows<KY & 1>(acc, wb, sb1, sb2, xa, xb);
    sb = sb2;
  }
  if (k < NK) v12_rows<0>(acc, wa, sb, sb, xa, xb);
  return acc;
}

// V13: rows prefetched TWO rows ahead (3-buffer ring), weights a source
// ahead (2-buffer ring); both rings resolved at compile time by unrolling 6
// sources per iteration (6*KY rows: divisible by 3 and 2); the tail (< 6
// sources) reuses the same body under a run-time bound.
struct Ring3 { float r[3][KX]; };
template <int G>   // G: sources in this block (compile-time), rows 0..G*KY-1
__device__ __forceinline__ void v13_block(float& acc, const float* src, const int* soff,
                                          const float* w28, int k0, int nk, Ring3& x,
                                          float (&wa)[28], float (&wb)[28]) {
  // on entry: weights of source k0 in wa, rows 0 and 1 of source k0 in x.r[0], x.r[1]
  const float* sbs[G + 1];
#pragma unroll
  for (int j = 0; j <= G; ++j) {
    const int kk = k0 + j < nk ? k0 + j : nk - 1;
    sbs[j] = src + soff[kk];
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    // next source's weights into the other buffer
    {
      const int kn = k0 + j + 1 < nk ? k0 + j + 1 : nk - 1;
      float* wd = (j & 1) ? wa : wb;
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const float4 v = reinterpret_cast<const float4*>(w28 + kn * 28)[q];
        wd[4 * q] = v.x; wd[4 * q + 1] = v.y; wd[4 * q + 2] = v.z; wd[4 * q + 3] = v.w;
      }
    }
    const float* wcur = (j & 1) ? wb : wa;
#pragma unroll
    for (int v = 0; v < KY; ++v) {
      const int row = j * KY + v;
      // prefetch row + 2 (this source's row v+2, or the next source's)
      const float* nrow = v + 2 < KY ? sbs[j] + (v + 2) * SW : sbs[j + 1] + (v + 2 - KY) * SW;
#pragma unroll
      for (int u = 0; u < KX; ++u) x.r[(row + 2) % 3][u] = nrow[u];
#pragma unroll
      for (int u = 0; u < KX; ++u)
        acc = __fadd_rn(acc, __fmul_rn(wcur[v * KX + u], x.r[row % 3][u]));
    }
  }
}
__device__ __forceinline__ float cell_v13(float acc, const float* src, const int* soff,
                                          const float* w28) {
  Ring3 x;
  float wa[28], wb[28];
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const float4 v = reinterpret_cast<const float4*>(w28)[q];
    wa[4 * q] = v.x; wa[4 * q + 1] = v.y; wa[4 * q + 2] = v.z; wa[4 * q + 3] = v.w;
  }
  const float* sb = src + soff[0];
#pragma unroll
  for (int u = 0; u < KX; ++u) { x.r[0][u] = sb[u]; x.r[1][u] = sb[SW + u]; }
  int k = 0;
  for (; k + 6 <= NK; k += 6) v13_block<6>(acc, src, soff, w28, k, NK, x, wa, wb);
  // tail: the ring offsets restart at 0 because 6*KY rows is a multiple of 3
  for (; k < NK; ++k) {
    // one source at a time: row buffers rotate by KY per source -> use block<1>
    // only when KY % 3 == 0; otherwise re-seed the ring (rare: < 6 sources)
    const float* s0 = src + soff[k];
#pragma unroll
    for (int u = 0; u < KX; ++u) { x.r[0][u] = s0[u]; x.r[1][u] = s0[SW + u]; }
    float* wsrc = (k & 1) ? wb : wa;
    (void)wsrc;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const float4 v = reinterpret_cast<const float4*>(w28 + k * 28)[q];
      wa[4 * q] = v.x; wa[4 * q + 1] = v.y; wa[4 * q + 2] = v.z; wa[4 * q + 3] = v.w;
    }
    v13_block<1>(acc, src, soff, w28, k, NK, x, wa, wb);
  }
  return acc;
}

template <int V>
__global__ void bench(const float* gsrc, const float* gw, float* out, long long* cyc, int items) {
  __shared__ float src[NK * SHW];
  __shared__ __align__(16) float w[NK * 28 + 4];
  __shared__ int soff[NK];
  for (int i = threadIdx.x; i < NK * SHW; i += blockDim.x) src[i] = gsrc[i];
  for (int i = threadIdx.x; i < NK * 28; i += blockDim.x)
    w[i] = (V == 2 || V == 7 || V >= 12) ? ((i % 28) < KK ? gw[(i / 28) * KK + i % 28] : 0.f) : (i < NK * KK ? gw[i] : 0.f);
  for (int i = threadIdx.x; i < NK; i += blockDim.x) soff[i] = i * SHW;
  __syncthreads();
  const int it = threadIdx.x;
  if (it >= items) return;
  const int r = (it / 9) % 9, c = it % 9;
  const float* base = src + r * SW + c;
  long long t0 = clock64();
  float a;
  if (V == 0) a = cell_v0(0.1f, base, soff, w);
  else if (V == 1) a = cell_v1(0.1f, base, soff, w);
  else if (V == 2) a = cell_v2(0.1f, base, soff, w);
  else if (V == 3) a = cell_v3(0.1f, base, soff, w);
  else if (V == 7) a = cell_v7(0.1f, base, soff, w);
  else if (V == 8) a = cell_v8(0.1f, base, soff, w);
  else if (V == 9) a = cell_v9(0.1f, base, soff, w);
  else if (V == 10) a = cell_v10(0.1f, base, soff, w);
  else if (V == 11) a = cell_v11(0.1f, base, soff, w);
  else if (V == 12) a = cell_v12(0.1f, base, soff, w);
  else if (V == 13) a = cell_v13(0.1f, base, soff, w);
  else if (V >= 5) {
    const int n = V == 5 ? 4 : 2;
    const int rr = (it / 2) % 9, cc = n * (it % 2);
    float o[4];
    if (V == 5) cell_v5(0.1f, src + rr * SW + cc, soff, w, o);
    else cell_v6(0.1f, src + rr * SW + cc, soff, w, o);
    long long t1 = clock64();
    bool bad = false;
    for (int i = 0; i < n; ++i)
      bad |= __float_as_int(cell_v0(0.1f, src + rr * SW + cc + i, soff, w)) != __float_as_int(o[i]);
    out[blockIdx.x * blockDim.x + it] = bad ? -999.f : o[0];
    cyc[blockIdx.x * blockDim.x + it] = t1 - t0;
    return;
  } else {
    // items are cell PAIRS: cells (r, 2j) and (r, 2j+1) of a 9x10 grid
    const int rr = (it / 4) % 9, cc = 2 * (it % 4);
    float a0, a1;
    cell_v4(0.1f, src + rr * SW + cc, soff, w, &a0, &a1);
    a = a0;
    long long t1 = clock64();
    const float ref0 = cell_v0(0.1f, src + rr * SW + cc, soff, w);
    const float ref1 = cell_v0(0.1f, src + rr * SW + cc + 1, soff, w);
    out[blockIdx.x * blockDim.x + it] =
        (__float_as_int(ref0) != __float_as_int(a0) || __float_as_int(ref1) != __float_as_int(a1))
            ? -999.f : a;
    cyc[blockIdx.x * blockDim.x + it] = t1 - t0;
    return;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + it] = a;
  cyc[blockIdx.x * blockDim.x + it] = t1 - t0;
}

int main() {
  float *gs, *gw, *out;
  long long* cyc;
  cudaMalloc(&gs, NK * SHW * 4);
  cudaMalloc(&gw, NK * KK * 4);
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 4096 * 8);
  float hs[NK * SHW], hw[NK * KK];
  unsigned st = 12345;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (st >> 8) / 16777216.0f; };
  for (int i = 0; i < NK * SHW; ++i) hs[i] = rnd() * 2.f - 1.f;
  for (int i = 0; i < NK * KK; ++i) hw[i] = rnd() * 0.1f - 0.05f;
  cudaMemcpy(gs, hs, sizeof(hs), cudaMemcpyHostToDevice);
  cudaMemcpy(gw, hw, sizeof(hw), cudaMemcpyHostToDevice);
  for (int items : {32, 96}) {
    for (int v = 7; v < 14; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) bench<0><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 1) bench<1><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 2) bench<2><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 3) bench<3><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 4) bench<4><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 5) bench<5><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 6) bench<6><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 7) bench<7><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 8) bench<8><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 9) bench<9><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 10) bench<10><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 11) bench<11><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 12) bench<12><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 13) bench<13><<<1, 128>>>(gs, gw, out, cyc, items);
      }
      cudaDeviceSynchronize();
      long long hc[128];
      float ho[128];
      cudaMemcpy(hc, cyc, 128 * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(ho, out, 128 * 4, cudaMemcpyDeviceToHost);
      long long mx = 0;
      int bad = 0;
      for (int i = 0; i < items; ++i) { mx = hc[i] > mx ? hc[i] : mx; bad += ho[i] == -999.f; }
      if (bad) printf("  MISMATCH in %d items\n", bad);
      printf("items %3d variant %d: max %lld cycles per cell (%.1f per MAC) out0 %.6f\n", items, v,
             mx, mx / 1000.0, ho[0]);
    }
  }
  return 0;
}
