// mb_barloc.cu — does the grid barrier's latency (148 CTAs, one per SM) depend
// on which L2 slice holds the counter?  Same barrier at 64 counter addresses
// (128-byte lines apart, and 2 MB apart).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void __launch_bounds__(512, 1) gbar(unsigned* bar, int reps, long long* out) {
  unsigned target = 0;
  long long t0 = 0;
  for (int i = -10; i < reps; ++i) {
    if (i == 0) t0 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) {
      target += gridDim.x;
      unsigned old;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
      if (old + 1 != target)
        while ((int)(ld_acq(bar) - target) < 0) {
        }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  unsigned char* base;
  long long* out;
  cudaMalloc(&base, 256 << 20);
  cudaMalloc(&out, 148 * 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 2000;
  for (int k = 0; k < 80; ++k) {
    size_t off = k < 64 ? (size_t)k * 128 : (size_t)(k - 63) * (2 << 20);
    unsigned* bar = (unsigned*)(base + off);
    cudaMemset(bar, 0, 4);
    void* args[] = {&bar, (void*)&reps, &out};
    cudaLaunchCooperativeKernel((void*)gbar, nsm, 512, args, 0, 0);
    cudaDeviceSynchronize();
    long long h[148], mx = 0;
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("offset %10zu: %lld cycles/barrier\n", off, mx / reps);
  }
  return 0;
}
