// Shared helpers for the purine_b200 kernel library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "purine_b200.h"

namespace bf {

// thread-local last error (bf_last_error)
void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(bf_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// running count of kernels this library launched (bf_launch_count)
void count_launches(int n);

// after `n` launches: map a CUDA error to a return code + message
inline int check_launch(const char* what, int n = 1) {
  count_launches(n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

#define BF_REQUIRE(cond, ...)      \
  do {                             \
    if (!(cond)) {                 \
      ::bf::set_error(__VA_ARGS__); \
      return 2;                    \
    }                              \
  } while (0)

#define BF_CUDA(call, what)                                               \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess) {                                              \
      ::bf::set_error("%s: %s", what, cudaGetErrorString(_e));            \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int sm_count_current();
int gemm_sm_budget();  // SM count minus bf_set_sm_reserve()

// grid for a grid-stride elementwise kernel: multiple of the SM count
inline int elementwise_grid(int64_t work_items, int threads) {
  int sms = sm_count_current();
  int64_t want = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread CTAs per SM
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace bf
