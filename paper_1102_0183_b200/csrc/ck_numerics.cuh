// ck_numerics.cuh — the reference's float semantics, restated for sm_100a.
//
// The reference's f32 path is not uniformly f32; every
// helper here names the reference expression it reproduces:
//   conv activation   kernels.py:87   f32(1.7159 * tanh_f64(0.6666 * (double)a))
//   FC activation     layers.py:23-25 numpy f32 chain with weak scalars:
//                                     f32(1.7159) * tanh32(f32(0.6666) * a)
//   derivative        layers.py:28-30 f32(1.14381894) * (1 - t*t), t = tanh32(..)
//   output delta      backprop.py:22-32 in f64, rounded once into f32
//   SGD update        network.py:264-273 w = f32(w - f32(f32(eta) * g))
// Explicit __fmul_rn/__fadd_rn keep nvcc from contracting to FMA (the
// reference's LLVM IR has no `contract` flag).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ck {

constexpr double kActScale = 1.7159;
constexpr double kActGain = 0.6666;

// (one out-of-line copy: the f64 tanh is ~100 instructions, and the
// training kernel's per-image code footprint is instruction-cache bound;
// conv_act_inl for the per-pool-block loops, where a call costs register
// saves)
__device__ __forceinline__ float conv_act_inl(float a) {
  return (float)(kActScale * tanh(kActGain * (double)a));
}
static __device__ __noinline__ float conv_act(float a) { return conv_act_inl(a); }

// numpy's float32 tanh is a SIMD approximation (~1 ulp from correctly
// rounded in a third of the cases); the device uses CUDA's tanhf (<= 2 ulp).
// Stated tolerance: a few ulp on FC activations and on every delta (the conv
// activation, which must be bit-exact, keeps the reference's f64 tanh).
static __device__ __noinline__ float tanh32(float z) { return tanhf(z); }

__device__ __forceinline__ float fc_act(float a) {
  return __fmul_rn((float)kActScale, tanh32(__fmul_rn((float)kActGain, a)));
}

__device__ __forceinline__ float act_deriv(float a) {
  const float t = tanh32(__fmul_rn((float)kActGain, a));
  return __fmul_rn((float)(kActScale * kActGain), __fsub_rn(1.0f, __fmul_rn(t, t)));
}

__device__ __forceinline__ float sgd(float w, float eta_f, float g) {
  return __fsub_rn(w, __fmul_rn(eta_f, g));
}

// ceil(n / t) clamped at 0 for t > 0 (kernels.py:100,107 negative floor division)
__device__ __forceinline__ int ceil_div_clamp0(int n, int t) {
  return n > 0 ? (n + t - 1) / t : 0;
}

// numpy pairwise summation of a contiguous f64 vector (the `.sum()` in
// backprop.sample_loss): sequential below 8 elements, 8 partial sums up to
// 128, recursive halving above (n2 = n/2 rounded down to a multiple of 8).
__device__ __forceinline__ double np_pairwise_block(const double* v, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, v[i]);
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = v[j];
  int i = 8;
  const int full = n - (n % 8);
  for (; i < full; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, v[i]);
  return res;
}

// The halving recursion unrolled with an explicit stack (no device recursion):
// leaves (<= 128 elements) are summed left to right and combined bottom-up
// exactly as numpy's recursion combines them.
__device__ inline double np_pairwise_sum(const double* v, int n) {
  if (n <= 128) return np_pairwise_block(v, n);
  // post-order walk: stack of (offset, length, partial sum state)
  int off[16], len[16], state[16];
  double left[16];
  int sp = 0;
  off[0] = 0; len[0] = n; state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int o = off[sp], m = len[sp];
    if (m <= 128) {
      ret = np_pairwise_block(v + o, m);
      --sp;
      continue;
    }
    int n2 = m / 2;
    n2 -= n2 % 8;
    if (state[sp] == 0) {            // descend left
      state[sp] = 1;
      ++sp; off[sp] = o; len[sp] = n2; state[sp] = 0;
    } else if (state[sp] == 1) {     // left done: descend right
      left[sp] = ret;
      state[sp] = 2;
      ++sp; off[sp] = o + n2; len[sp] = m - n2; state[sp] = 0;
    } else {                         // both done
      ret = __dadd_rn(left[sp], ret);
      --sp;
    }
  }
  return ret;
}

}  // namespace ck
