// microbench.cu — B200 instruction throughput / latency and barrier costs
// that decide the engine's design (development aid; results summarised in
// DESIGN.md).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x)                                                              \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

constexpr int ITERS = 4096;

// 8 independent chains per thread -> throughput
template <int OP>
__global__ void tput(float* out, float seed) {
  float f[8];
  double d[8];
  for (int i = 0; i < 8; ++i) { f[i] = seed + i + threadIdx.x; d[i] = f[i]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) f[i] = __fadd_rn(f[i], 1.0001f);
      if (OP == 1) f[i] = __fmul_rn(f[i], 0.9999f);
      if (OP == 2) f[i] = __fmaf_rn(f[i], 0.9999f, 0.5f);
      if (OP == 3) d[i] = __dadd_rn(d[i], 1.0001);
      if (OP == 4) d[i] = __fma_rn(d[i], 0.9999, 0.5);
      if (OP == 5) d[i] = __dadd_rn(d[i], (double)f[i]), f[i] = __fadd_rn(f[i], 1.0f);
      if (OP == 6) f[i] = (float)(d[i] = __dadd_rn(d[i], 1e-3));
      if (OP == 7) f[i] = tanhf(f[i]);
      if (OP == 8) d[i] = tanh(d[i]);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + (float)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 1 chain -> latency
template <int OP>
__global__ void lat(float* out, float seed) {
  float f = seed + threadIdx.x;
  double d = f;
  for (int it = 0; it < ITERS; ++it) {
    if (OP == 0) f = __fadd_rn(f, 1.0001f);
    if (OP == 3) d = __dadd_rn(d, 1.0001);
    if (OP == 5) d = __dadd_rn(d, (double)__int_as_float(__float_as_int(f) ^ it));
  }
  out[threadIdx.x] = f + (float)d;
}

__global__ void cluster_bar(long long* out, int reps) {
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void grid_bar(long long* out, unsigned* bar, int reps) {
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      __threadfence();
      if (atomicAdd(bar, 1u) == gridDim.x - 1) {
        atomicExch(bar, 0u);
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(g + 1) : "memory");
      } else {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
        } while (v == g);
      }
      __threadfence();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <int OP>
int run_tput(const char* name, float* d_out, int blocks, int threads) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tput<OP><<<blocks, threads>>>(d_out, 1.0f);
  CHECK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  tput<OP><<<blocks, threads>>>(d_out, 1.0f);
  cudaEventRecord(b);
  CHECK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * ITERS * 8;
  printf("tput %-22s %8.1f Gop/s  (%.1f lane-ops/clk/SM at 1.965 GHz)\n", name, ops / ms / 1e6,
         ops / (ms * 1e-3) / 148 / 1.965e9);
  return 0;
}

template <int OP>
int run_lat(const char* name, float* d_out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  lat<OP><<<1, 32>>>(d_out, 1.0f);
  CHECK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  lat<OP><<<1, 32>>>(d_out, 1.0f);
  cudaEventRecord(b);
  CHECK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("lat  %-22s %8.2f ns/op\n", name, ms * 1e6 / ITERS);
  return 0;
}

int main() {
  float* d_out;
  CHECK(cudaMalloc(&d_out, 148 * 8 * 1024 * sizeof(float)));
  const int B = 148 * 4, T = 256;
  run_tput<0>("fadd", d_out, B, T);
  run_tput<1>("fmul", d_out, B, T);
  run_tput<2>("ffma", d_out, B, T);
  run_tput<3>("dadd", d_out, B, T);
  run_tput<4>("dfma", d_out, B, T);
  run_tput<5>("dadd+cvt f32->f64", d_out, B, T);
  run_tput<6>("dadd+cvt f64->f32", d_out, B, T);
  run_tput<7>("tanhf", d_out, B, T);
  run_tput<8>("tanh (double)", d_out, B, T);
  run_lat<0>("fadd chain", d_out);
  run_lat<3>("dadd chain", d_out);
  run_lat<5>("dadd(cvt) chain", d_out);

  long long* d_t;
  unsigned* d_bar;
  CHECK(cudaMalloc(&d_t, sizeof(long long)));
  CHECK(cudaMalloc(&d_bar, 2 * sizeof(unsigned)));
  CHECK(cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {2, 4, 8, 16}) {
    for (int thr : {256, 512}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(thr);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const int reps = 10000;
      CHECK(cudaLaunchKernelEx(&cfg, cluster_bar, d_t, reps));
      CHECK(cudaDeviceSynchronize());
      long long cyc;
      CHECK(cudaMemcpy(&cyc, d_t, sizeof(cyc), cudaMemcpyDeviceToHost));
      printf("cluster barrier  size %2d x %3d thr: %6.0f cycles\n", cs, thr, (double)cyc / reps);
    }
  }
  for (int g : {16, 74, 148}) {
    CHECK(cudaMemset(d_bar, 0, 8));
    void* args[] = {&d_t, &d_bar, (void*)nullptr};
    int reps = 2000;
    args[2] = &reps;
    CHECK(cudaLaunchCooperativeKernel((void*)grid_bar, g, 512, args, 0, 0));
    CHECK(cudaDeviceSynchronize());
    long long cyc;
    CHECK(cudaMemcpy(&cyc, d_t, sizeof(cyc), cudaMemcpyDeviceToHost));
    printf("grid barrier     %3d CTAs x 512 thr: %6.0f cycles\n", g, (double)cyc / reps);
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
