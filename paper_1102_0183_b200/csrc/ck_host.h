// ck_host.h — host-side plumbing shared by the C-ABI translation units:
// thread-local last-error text, status helpers and the launch counter that
// backs ck_kernel_launches().
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/ckb200.h"

namespace ck {

int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* where);
void count_launch(int64_t n = 1);

#define CK_CUDA_TRY(expr)                                          \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return ::ck::cuda_status(_e, #expr);    \
  } while (0)

#define CK_CHECK(cond, code, msg)                                  \
  do {                                                             \
    if (!(cond)) return ::ck::set_error((code), (msg));            \
  } while (0)

inline int blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > (1 << 30)) b = 1 << 30;
  return (int)b;
}

}  // namespace ck
