// mb_barrier.cu — grid barrier variants on B200 (148 CTAs x 512 threads, one
// per SM, cooperative launch), optionally with every CTA storing W bytes to
// global memory before each barrier (the release then has stores to drain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_barrier tools/mb_barrier.cu
//   V0  red.release.gpu add; spin ld.acquire.gpu           (the engine's GridTeam)
//   V1  red.release.gpu add; spin ld.relaxed.gpu; fence.acq_rel.gpu
//   V2  fence.acq_rel.gpu; red.relaxed.gpu; spin ld.relaxed.gpu; fence.acq_rel.gpu
//   V3  red.release.gpu add; spin ld.acquire.gpu with 4 warps' lane 0 polling
//   V4  atom.add.acq_rel returning the old count; the last arriver skips the spin
//   V5  hierarchical: cluster barrier, V4 among the clusters' rank-0 CTAs,
//       cluster barrier (cluster launch; also prints max co-resident clusters)
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x)                                                                     \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int V>
__global__ void __launch_bounds__(512, 1) bar_kernel(unsigned* bar, float* sink, int words, int reps,
                                                     long long* out) {
  unsigned target = 0;
  const unsigned n = gridDim.x;
  long long t0 = 0;
  for (int i = -10; i < reps; ++i) {
    if (i == 0) t0 = clock64();
    for (int w = threadIdx.x; w < words; w += blockDim.x)
      sink[(size_t)blockIdx.x * words + w] = (float)(i + w);
    __syncthreads();
    if (V == 5) {
      unsigned cr, cn;
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
      asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cn));
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      target += n / cn;
      if (cr == 0 && threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old + 1 != target)
          while ((int)(ld_acq(bar) - target) < 0) {
          }
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      continue;
    }
    target += n;
    if (V == 3) {
      if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      if ((threadIdx.x & 127) == 0)
        while ((int)(ld_acq(bar) - target) < 0) {
        }
    } else if (threadIdx.x == 0) {
      if (V == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while ((int)(ld_acq(bar) - target) < 0) {
        }
      } else if (V == 1) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while ((int)(ld_rlx(bar) - target) < 0) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (V == 2) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while ((int)(ld_rlx(bar) - target) < 0) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (V == 4 || V == 5) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old + 1 != target)
          while ((int)(ld_acq(bar) - target) < 0) {
          }
      }
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int V>
int run(unsigned* bar, float* sink, long long* out, int words, int ctas = 148, int cs = 1) {
  const int reps = 4000;
  CHECK(cudaMemset(bar, 0, 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  CHECK(cudaFuncSetAttribute(bar_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CHECK(cudaFuncSetAttribute(bar_kernel<V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cs;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = cs > 1 ? 2 : 1;
  if (cs > 1) {
    int mc = 0;
    CHECK(cudaOccupancyMaxActiveClusters(&mc, (void*)bar_kernel<V>, &cfg));
    printf("cluster size %d: max active clusters %d (%d CTAs)\n", cs, mc, mc * cs);
    if (mc * cs < ctas) return 0;
  }
  cudaEventRecord(a);
  CHECK(cudaLaunchKernelEx(&cfg, bar_kernel<V>, bar, sink, words, reps, out));
  cudaEventRecord(b);
  CHECK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long cyc[148];
  CHECK(cudaMemcpy(cyc, out, sizeof(cyc), cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < ctas; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  printf("V%d  ctas %3d cluster %2d stores %6d B/CTA: %7.0f cycles/barrier  %6.3f us/barrier (event, incl. stores)\n", V,
         ctas, cs, words * 4, (double)mx / reps, ms * 1e3 / (reps + 10));
  return 0;
}

int main() {
  unsigned* bar;
  float* sink;
  long long* out;
  CHECK(cudaMalloc(&bar, 256));
  CHECK(cudaMalloc(&sink, 148 * 8192 * sizeof(float)));
  CHECK(cudaMalloc(&out, 148 * sizeof(long long)));
  for (int words : {0, 512, 4096}) {
    if (run<0>(bar, sink, out, words)) return 1;
    if (run<1>(bar, sink, out, words)) return 1;
    if (run<2>(bar, sink, out, words)) return 1;
    if (run<3>(bar, sink, out, words)) return 1;
    if (run<4>(bar, sink, out, words)) return 1;
  }
  for (int c : {16, 32, 74}) run<4>(bar, sink, out, 512, c);
  for (int cs : {2, 4, 8}) {
    for (int c : {144, 148})
      if (c % cs == 0) run<5>(bar, sink, out, 512, c, cs);
  }
  return 0;
}
