// mb_team.cu — barrier latency of 8 teams of 18 CTAs (one CTA per SM, 148
// launched, 144 used) when teams are formed by blockIdx (the engine's
// GridTeam) vs by %smid ranges (SM-local teams).  Prints cycles per barrier
// (max over teams) and each team's smid list for the smid grouping.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void __launch_bounds__(512, 1) team_bar(unsigned* bars, int by_smid, int reps,
                                                   long long* out, int* smids) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int T = 18;
  int team = by_smid ? (int)smid / T : (int)blockIdx.x / T;
  if (team >= 8) return;
  if (threadIdx.x == 0) smids[blockIdx.x] = smid;
  unsigned* bar = bars + team * 32;
  unsigned target = 0;
  long long t0 = 0;
  for (int i = -10; i < reps; ++i) {
    if (i == 0) t0 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) {
      target += T;
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
  unsigned* bars;
  long long* out;
  int* smids;
  cudaMalloc(&bars, 8 * 32 * 4);
  cudaMalloc(&out, 148 * 8);
  cudaMalloc(&smids, 148 * 4);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bars, 0, 8 * 32 * 4);
      cudaMemset(out, 0, 148 * 8);
      int reps = 4000;
      void* args[] = {&bars, &mode, &reps, &out, &smids};
      cudaError_t e = cudaLaunchCooperativeKernel((void*)team_bar, nsm, 512, args, 0, 0);
      if (e != cudaSuccess) { printf("launch %s\n", cudaGetErrorString(e)); return 1; }
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0, mn = 1LL << 62;
      for (int i = 0; i < nsm; ++i)
        if (h[i]) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
      printf("%s teams: max %lld min %lld cycles per barrier\n", mode ? "smid   " : "blockIdx",
             mx / reps, mn / reps);
    }
  }
  int sm[148];
  cudaMemcpy(sm, smids, sizeof(sm), cudaMemcpyDeviceToHost);
  printf("blockIdx -> smid:");
  for (int i = 0; i < nsm; ++i) printf(" %d", sm[i]);
  printf("\n");
  return 0;
}
