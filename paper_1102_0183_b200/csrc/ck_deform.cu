// ck_deform.cu — on-line training-image deformation on the device
// (convkit.augment, augment.py:63-170; training.py:140-144).
//
// The reference draws every training sample's deformation on the host from
// numpy's default_rng([seed, epoch, i]) (SeedSequence + PCG64), composes an
// affine warp with a Gaussian-smoothed random displacement field
// (scipy.ndimage.gaussian_filter, truncate 3) and resamples each channel once
// with bilinear map_coordinates(mode="grid-constant", cval = median of the
// channel's border).  Here one CTA deforms one image of the epoch:
//
//   thread 0   SeedSequence([seed, epoch, i]) -> PCG64, the 7 uniforms and
//              the bounded elastic seed (bit-exact integer arithmetic), the
//              affine inverse (closed form in f64; numpy's LAPACK inverse
//              differs in the last ulp, absorbed by the final f32 rounding)
//   all        the 2*H*W field uniforms from PCG64(elastic seed), each thread
//              jumping its LCG ahead to its own chunk (O(log n) 128-bit steps)
//   all        separable Gaussian, axis 0 then axis 1, in scipy's symmetric
//              order (out = x0*w0; out += (x[-j] + x[+j]) * w[-j], j = r..1),
//              separately rounded f64 ops (no FMA contraction)
//   all        per channel: border median (f32, numpy's mean of the two middle
//              values), then bilinear resampling in scipy's corner order
//
// Output: float32 (n, C, H, W), image i deformed with [seed, epoch, i]; the
// persistent training kernel then reads it with lut = NULL.  All in shared
// memory: 24*H*W bytes of f64 field + scratch (48x48: 55 KB).
#include <math.h>

#include "ck_host.h"

namespace ck {
namespace {

typedef unsigned __int128 u128;

constexpr uint32_t kInitA = 0x43B0D7E5u, kMultA = 0x931E8875u;
constexpr uint32_t kInitB = 0x8B51F9DDu, kMultB = 0x58F38DEDu;
constexpr uint32_t kMixL = 0xCA01F9DDu, kMixR = 0x4973F715u;
#define kPcgMult ((((u128)2549297995355413924ull) << 64) | (u128)4865540595714422341ull)

struct Pcg {
  u128 state, inc;
  bool has32;
  uint32_t buf32;
};

// numpy bit_generator.pyx SeedSequence: entropy words -> 4-word pool -> 8
// 32-bit output words -> 4 uint64 (little-endian pairs).
__device__ void seed_sequence(const uint32_t* ent, int n_ent, uint64_t out[4]) {
  uint32_t hc = kInitA;
  auto hashmix = [&hc](uint32_t v) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < n_ent; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = kInitB;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= kMultB;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// _coerce_to_uint32_array of one non-negative integer (0 -> one zero word).
__device__ int push_words(uint64_t v, uint32_t* ent, int n) {
  if (v == 0) {
    ent[n++] = 0;
    return n;
  }
  while (v) {
    ent[n++] = (uint32_t)v;
    v >>= 32;
  }
  return n;
}

__device__ Pcg pcg_seed(const uint32_t* ent, int n_ent) {
  uint64_t s[4];
  seed_sequence(ent, n_ent, s);
  Pcg g;
  const u128 initstate = ((u128)s[0] << 64) | s[1];
  const u128 initseq = ((u128)s[2] << 64) | s[3];
  g.inc = (initseq << 1) | 1;
  g.state = g.inc;                       // 0 * mult + inc
  g.state += initstate;
  g.state = g.state * kPcgMult + g.inc;
  g.has32 = false;
  g.buf32 = 0;
  return g;
}

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint64_t pcg_next64(Pcg& g) {
  g.state = g.state * kPcgMult + g.inc;
  return pcg_out(g.state);
}

__device__ uint32_t pcg_next32(Pcg& g) {
  if (g.has32) {
    g.has32 = false;
    return g.buf32;
  }
  const uint64_t v = pcg_next64(g);
  g.has32 = true;
  g.buf32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// state after `delta` further LCG steps (pcg_advance_lcg_128)
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kPcgMult, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double u53(uint64_t v) {
  return __dmul_rn((double)(v >> 11), 1.0 / 9007199254740992.0);
}

// Generator.uniform(lo, hi) = lo + (hi - lo) * next_double
__device__ __forceinline__ double uniform(double lo, double hi, uint64_t v) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u53(v)));
}

// integers(0, 2**31 - 1): buffered_bounded_lemire_uint32 with rng = 2**31 - 2
__device__ uint32_t bounded_seed(Pcg& g) {
  const uint32_t rng = 0x7FFFFFFEu, excl = rng + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thresh = (0xFFFFFFFFu - rng) % excl;
    while (left < thresh) {
      m = (uint64_t)pcg_next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

struct Affine {
  double i00, i01, i10, i11, cx, cy, dx, dy;
};

__device__ Affine affine_inverse(const ck_deform_params& p, int W, int H) {
  const double deg = 3.141592653589793 / 180.0;   // math.radians
  const double rot = __dmul_rn(p.rotate, deg), sh = __dmul_rn(p.shear_h, deg);
  const double c = cos(rot), s = sin(rot), t = tan(sh);
  // m = R @ Shear @ Scale (augment.py:92-97)
  const double m00 = __dmul_rn(c, p.scale_x);
  const double m01 = __dmul_rn(__dsub_rn(__dmul_rn(c, t), s), p.scale_y);
  const double m10 = __dmul_rn(s, p.scale_x);
  const double m11 = __dmul_rn(__dadd_rn(__dmul_rn(s, t), c), p.scale_y);
  const double det = __dsub_rn(__dmul_rn(m00, m11), __dmul_rn(m01, m10));
  Affine a;
  a.i00 = __ddiv_rn(m11, det);
  a.i01 = __ddiv_rn(-m01, det);
  a.i10 = __ddiv_rn(-m10, det);
  a.i11 = __ddiv_rn(m00, det);
  a.cx = (W - 1) / 2.0;
  a.cy = (H - 1) / 2.0;
  a.dx = __dmul_rn(p.translate_x, (double)W);
  a.dy = __dmul_rn(p.translate_y, (double)H);
  return a;
}

__device__ bool is_identity(const ck_deform_params& p) {
  return p.translate_x == 0.0 && p.translate_y == 0.0 && p.rotate == 0.0 &&
         p.scale_x == 1.0 && p.scale_y == 1.0 && p.shear_h == 0.0 && p.elastic_alpha == 0.0;
}

struct DeformArgs {
  const uint8_t* images;   // (n, C, H, W) uint8 (with lut) or float32 (lut null)
  const float* lut;
  int C, H, W;
  int64_t n;
  ck_deform_cfg cfg;
  const double* gauss_w;   // 2*radius+1 taps (device), scipy's normalised kernel
  int radius;
  uint64_t seed, epoch;
  const ck_deform_params* params_in;  // explicit per-image params, or null: draw
  ck_deform_params* params_out;       // nullable
  float* out;
};

__device__ __forceinline__ float load_px(const DeformArgs& A, int64_t idx) {
  return A.lut ? A.lut[A.images[idx]] : reinterpret_cast<const float*>(A.images)[idx];
}

__global__ void __launch_bounds__(256) deform_kernel(DeformArgs A) {
  extern __shared__ double smem[];
  const int HW = A.H * A.W;
  double* f0 = smem;            // row displacement
  double* f1 = smem + HW;       // col displacement
  double* tmp = smem + 2 * HW;  // gaussian scratch
  float* border = reinterpret_cast<float*>(smem + 3 * HW);
  const int nb = 2 * A.W + 2 * (A.H - 2);
  __shared__ ck_deform_params P;
  __shared__ Affine AF;
  __shared__ float bg_s;
  __shared__ float mid_s[2];
  __shared__ Pcg field_rng;

  for (int64_t img = blockIdx.x; img < A.n; img += gridDim.x) {
    if (threadIdx.x == 0) {
      ck_deform_params p;
      if (A.params_in) {
        p = A.params_in[img];
      } else {
        uint32_t ent[8];
        int ne = push_words(A.seed, ent, 0);
        ne = push_words(A.epoch, ent, ne);
        ne = push_words((uint64_t)img, ent, ne);
        Pcg g = pcg_seed(ent, ne);
        double u[6];
        for (int k = 0; k < 6; ++k) u[k] = uniform(-1.0, 1.0, pcg_next64(g));
        const double alpha = uniform(0.0, 1.0, pcg_next64(g));
        const uint32_t es = bounded_seed(g);
        p.translate_x = __dmul_rn(u[0], A.cfg.translate_max);
        p.translate_y = __dmul_rn(u[1], A.cfg.translate_max);
        p.rotate = __dmul_rn(u[2], A.cfg.rotate_max);
        p.scale_x = __dadd_rn(1.0, __dmul_rn(u[3], A.cfg.scale_max));
        p.scale_y = __dadd_rn(1.0, __dmul_rn(u[4], A.cfg.scale_max));
        p.shear_h = __dmul_rn(u[5], A.cfg.shear_max);
        p.elastic_alpha = __dmul_rn(alpha, A.cfg.elastic_alpha_max);
        p.seed = es;
        p.pad = 0;
      }
      if (A.params_out) A.params_out[img] = p;
      P = p;
      AF = affine_inverse(p, A.W, A.H);
      if (p.elastic_alpha > 0.0) {
        uint32_t ent[2];
        const int ne = push_words(p.seed, ent, 0);
        field_rng = pcg_seed(ent, ne);
      }
    }
    __syncthreads();
    const int64_t base = img * (int64_t)A.C * HW;
    if (is_identity(P)) {
      for (int i = threadIdx.x; i < A.C * HW; i += blockDim.x) A.out[base + i] = load_px(A, base + i);
      __syncthreads();
      continue;
    }
    const bool elastic = P.elastic_alpha > 0.0;
    if (elastic) {
      // 2*H*W uniforms in C order; thread t draws a contiguous chunk.
      const int total = 2 * HW;
      const int chunk = (total + blockDim.x - 1) / blockDim.x;
      const int b = threadIdx.x * chunk;
      const int e = min(total, b + chunk);
      if (b < e) {
        Pcg g = field_rng;
        g.state = pcg_advance(g.state, g.inc, (uint64_t)b);
        for (int k = b; k < e; ++k) smem[k] = uniform(-1.0, 1.0, pcg_next64(g));
      }
      __syncthreads();
      // gaussian_filter: correlate1d along axis 0 (rows), then axis 1 (cols)
      const double* w = A.gauss_w + A.radius;  // centred
      const int R = A.radius;
      for (int comp = 0; comp < 2; ++comp) {
        double* f = comp ? f1 : f0;
        for (int i = threadIdx.x; i < HW; i += blockDim.x) {
          const int r = i / A.W, c = i % A.W;
          double acc = __dmul_rn(f[i], w[0]);
          for (int j = R; j >= 1; --j) {
            const double lo = r - j >= 0 ? f[(r - j) * A.W + c] : 0.0;
            const double hi = r + j < A.H ? f[(r + j) * A.W + c] : 0.0;
            acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(lo, hi), w[-j]));
          }
          tmp[i] = acc;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < HW; i += blockDim.x) {
          const int r = i / A.W, c = i % A.W;
          const double* row = tmp + r * A.W;
          double acc = __dmul_rn(row[c], w[0]);
          for (int j = R; j >= 1; --j) {
            const double lo = c - j >= 0 ? row[c - j] : 0.0;
            const double hi = c + j < A.W ? row[c + j] : 0.0;
            acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(lo, hi), w[-j]));
          }
          f[i] = __dmul_rn(P.elastic_alpha, acc);
        }
        __syncthreads();
      }
    }
    // source coordinates (augment.py:101-105, :161-164), kept in f0/f1
    for (int i = threadIdx.x; i < HW; i += blockDim.x) {
      const double rx = __dsub_rn(__dsub_rn((double)(i % A.W), AF.cx), AF.dx);
      const double ry = __dsub_rn(__dsub_rn((double)(i / A.W), AF.cy), AF.dy);
      double rr = __dadd_rn(__dadd_rn(__dmul_rn(AF.i10, rx), __dmul_rn(AF.i11, ry)), AF.cy);
      double cc = __dadd_rn(__dadd_rn(__dmul_rn(AF.i00, rx), __dmul_rn(AF.i01, ry)), AF.cx);
      if (elastic) {
        rr = __dadd_rn(rr, f0[i]);
        cc = __dadd_rn(cc, f1[i]);
      }
      f0[i] = rr;
      f1[i] = cc;
    }
    for (int ch = 0; ch < A.C; ++ch) {
      const int64_t cb = base + (int64_t)ch * HW;
      // border_intensity (augment.py:143-147): median of the 1-px frame
      for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        int r, c;
        if (k < A.W) { r = 0; c = k; }
        else if (k < 2 * A.W) { r = A.H - 1; c = k - A.W; }
        else if (k < 2 * A.W + A.H - 2) { r = 1 + k - 2 * A.W; c = 0; }
        else { r = 1 + k - 2 * A.W - (A.H - 2); c = A.W - 1; }
        border[k] = load_px(A, cb + r * A.W + c);
      }
      __syncthreads();
      // rank of each element in a stable sort; pick ranks (nb-1)/2 and nb/2
      for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        const float v = border[k];
        int rank = 0;
        for (int j = 0; j < nb; ++j) {
          const float o = border[j];
          rank += (o < v) || (o == v && j < k);
        }
        if (rank == (nb - 1) / 2) mid_s[0] = v;
        if (rank == nb / 2) mid_s[1] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0)
        bg_s = (nb & 1) ? mid_s[1] : __fdiv_rn(__fadd_rn(mid_s[0], mid_s[1]), 2.0f);
      __syncthreads();
      const double bg = (double)bg_s;
      for (int i = threadIdx.x; i < HW; i += blockDim.x) {
        const double r = f0[i], c = f1[i];
        const double rf = floor(r), cf = floor(c);
        const double wr0 = __dsub_rn(1.0, __dsub_rn(r, rf));
        const double wc0 = __dsub_rn(1.0, __dsub_rn(c, cf));
        const double wr[2] = {wr0, __dsub_rn(1.0, wr0)};
        const double wc[2] = {wc0, __dsub_rn(1.0, wc0)};
        const int64_t r0 = (int64_t)rf, c0 = (int64_t)cf;
        double t = 0.0;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int64_t rr = r0 + a, cc = c0 + b;
            const double v = (rr >= 0 && rr < A.H && cc >= 0 && cc < A.W)
                                 ? (double)load_px(A, cb + rr * A.W + cc)
                                 : bg;
            t = __dadd_rn(t, __dmul_rn(__dmul_rn(v, wr[a]), wc[b]));
          }
        A.out[cb + i] = __double2float_rn(t);
      }
      __syncthreads();
    }
  }
}

int launch(DeformArgs A, ck_stream_t stream) {
  CK_CHECK(A.n >= 0, CK_E_DIMENSION, "negative image count");
  CK_CHECK(A.C > 0 && A.H >= 2 && A.W >= 2, CK_E_DIMENSION, "deformation needs C>0, H,W>=2");
  CK_CHECK(A.images && A.out, CK_E_CONFIG, "null image buffer");
  if (A.n == 0) return CK_OK;
  const size_t HW = (size_t)A.H * A.W;
  const size_t smem = 3 * HW * sizeof(double) + (2 * A.W + 2 * A.H) * sizeof(float);
  CK_CHECK(smem <= 200 * 1024, CK_E_DIMENSION, "image too large for on-device deformation");
  CK_CHECK(A.radius >= 0 && (A.radius == 0 || A.gauss_w), CK_E_CONFIG, "missing gaussian weights");
  CK_CUDA_TRY(cudaFuncSetAttribute(deform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  int dev = 0, sms = 148;
  CK_CUDA_TRY(cudaGetDevice(&dev));
  CK_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t grid = std::min<int64_t>(A.n, (int64_t)sms * 8);
  deform_kernel<<<(int)grid, 256, smem, (cudaStream_t)stream>>>(A);
  count_launch();
  CK_CUDA_TRY(cudaGetLastError());
  return CK_OK;
}

}  // namespace
}  // namespace ck

extern "C" {

int ck_deform_epoch(const uint8_t* images, const float* lut, int channels, int height,
                    int width, int64_t n, const ck_deform_cfg* cfg, const double* gauss_w,
                    int radius, uint64_t seed, uint64_t epoch, ck_deform_params* params_out,
                    float* out, ck_stream_t stream) {
  CK_CHECK(cfg, CK_E_CONFIG, "null deformation config");
  ck::DeformArgs A{images, lut, channels, height, width, n, *cfg, gauss_w, radius,
                   seed, epoch, nullptr, params_out, out};
  return ck::launch(A, stream);
}

int ck_deform_apply(const uint8_t* images, const float* lut, int channels, int height,
                    int width, int64_t n, const ck_deform_params* params,
                    const double* gauss_w, int radius, float* out, ck_stream_t stream) {
  CK_CHECK(params, CK_E_CONFIG, "null params");
  ck_deform_cfg cfg{};
  ck::DeformArgs A{images, lut, channels, height, width, n, cfg, gauss_w, radius,
                   0, 0, params, nullptr, out};
  return ck::launch(A, stream);
}

}  // extern "C"
