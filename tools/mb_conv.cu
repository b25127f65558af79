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

template <int V>
__global__ void bench(const float* gsrc, const float* gw, float* out, long long* cyc, int items) {
  __shared__ float src[NK * SHW];
  __shared__ __align__(16) float w[NK * 28 + 4];
  __shared__ int soff[NK];
  for (int i = threadIdx.x; i < NK * SHW; i += blockDim.x) src[i] = gsrc[i];
  for (int i = threadIdx.x; i < NK * 28; i += blockDim.x)
    w[i] = V == 2 ? ((i % 28) < KK ? gw[(i / 28) * KK + i % 28] : 0.f) : (i < NK * KK ? gw[i] : 0.f);
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
  for (int items : {32, 64, 128}) {
    for (int v = 0; v < 7; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) bench<0><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 1) bench<1><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 2) bench<2><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 3) bench<3><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 4) bench<4><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 5) bench<5><<<1, 128>>>(gs, gw, out, cyc, items);
        if (v == 6) bench<6><<<1, 128>>>(gs, gw, out, cyc, items);
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
