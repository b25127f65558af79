// mb_timer.cu — cost of reading %globaltimer (and storing it) as the
// sub-phase markers do, in SM cycles (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, long long* sink) {
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    sink[i] = t;
  }
  long long t1 = clock64();
  long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long c0 = clock64();
  while (clock64() - c0 < 200000) {
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 100;
    out[1] = g1 - g0;
  }
}
int main() {
  long long *o, *s;
  cudaMalloc(&o, 16);
  cudaMalloc(&s, 800);
  k<<<1, 32>>>(o, s);
  k<<<1, 32>>>(o, s);
  long long h[2];
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("globaltimer read+store: %lld cycles each; 200000 cycles = %lld ns of globaltimer\n", h[0], h[1]);
  return 0;
}
