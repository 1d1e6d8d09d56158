// Internal helpers shared by the C++ engine and the CUDA launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "spectrain.h"

namespace st {

// Thread-local "last error" (st_last_error). Returns the status for chaining.
st_status set_error(st_status s, const char* fmt, ...);
void clear_error();

// Kernel classes for profiling (st_get_profile order).
enum KernelClass { KC_UPDATE = 0, KC_GEMM_FWD = 1, KC_GEMM_DX = 2, KC_GEMM_DW = 3, KC_LOSS = 4, KC_COMM = 5,
                   KC_COUNT = 6 };

}  // namespace st

#define ST_CUDA_TRY(expr)                                                                              \
  do {                                                                                                 \
    cudaError_t e_ = (expr);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      return ::st::set_error(ST_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
  } while (0)

#define ST_TRY(expr)             \
  do {                           \
    st_status s_ = (expr);       \
    if (s_ != ST_OK) return s_;  \
  } while (0)
