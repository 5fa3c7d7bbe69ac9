// Shared host-side helpers for the C-ABI translation units.
#pragma once
#include <string>

#include "gradcomp_b200.h"

#define GC_ABI_VERSION 1

void gc_set_error(const std::string &msg);

#define GC_REQUIRE(cond, msg)          \
  do {                                 \
    if (!(cond)) {                     \
      gc_set_error(std::string(msg));  \
      return GC_ERR_INVALID;           \
    }                                  \
  } while (0)

#ifdef __CUDACC__
#include <cuda_runtime.h>
// Check the launch that was just enqueued (never synchronises).
#define GC_LAUNCH_CHECK(what)                                                     \
  do {                                                                            \
    cudaError_t e_ = cudaGetLastError();                                          \
    if (e_ != cudaSuccess) {                                                      \
      gc_set_error(std::string(what) + ": " + cudaGetErrorString(e_));            \
      return GC_ERR_CUDA;                                                         \
    }                                                                             \
  } while (0)
#endif
