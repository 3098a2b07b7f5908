// fk_error.h — error reporting shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/fk.h"

// Sets the thread's fk_last_error() message and returns code.
int fk_fail(int code, const char* fmt, ...);

#define FK_CUDA(call)                                                                             \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fk_fail(e_ == cudaErrorMemoryAllocation ? FK_ENOMEM : FK_ECUDA, "%s: %s (%s:%d)", \
                     #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

#define FK_TRY(call)              \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != FK_OK) return rc_; \
  } while (0)

struct FkDeviceGuard {
  int prev = -1;
  explicit FkDeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~FkDeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};
