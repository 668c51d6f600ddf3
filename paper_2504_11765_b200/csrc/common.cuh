// Shared host-side plumbing for librdkv: error reporting and device facts.
#pragma once
#include <cuda_runtime.h>
#include "../../include/rdkv.h"

namespace rdkv {

// Records a thread-local message (rdkv_last_error) and returns `code`.
int set_error(int code, const char* fmt, ...);

// Number of SMs of the current device (cached per device).
int num_sms();

}  // namespace rdkv

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess)                                                                      \
      return ::rdkv::set_error(RDKV_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,        \
                               cudaGetErrorString(_e));                                         \
  } while (0)

#define RDKV_TRY(expr)        \
  do {                        \
    int _rc = (expr);         \
    if (_rc != 0) return _rc; \
  } while (0)
