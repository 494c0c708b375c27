// Shared helpers for libncgp_b200: status/error plumbing, launch counting,
// warp reductions and the fixed-order fp64 reduction used everywhere a
// deterministic sum over a long axis is needed.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>

#include "../../include/ncgp_b200.h"

namespace ncgp {

void set_error(const char* fmt, ...);
std::atomic<int64_t>& launch_counter();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define NCGP_CHECK_ARG(cond, code, ...)        \
  do {                                         \
    if (!(cond)) {                             \
      ::ncgp::set_error(__VA_ARGS__);          \
      return (code);                           \
    }                                          \
  } while (0)

#define NCGP_LAUNCHED()                                                      \
  do {                                                                       \
    ::ncgp::launch_counter().fetch_add(1, std::memory_order_relaxed);        \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) {                                                 \
      ::ncgp::set_error("%s:%d: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return NCGP_CUDA_ERROR;                                                \
    }                                                                        \
  } while (0)

#define NCGP_CUDA(call)                                                      \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::ncgp::set_error("%s:%d: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return NCGP_CUDA_ERROR;                                                \
    }                                                                        \
  } while (0)

int sm_count();

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide fixed-order sum (block size multiple of 32, <= 1024).
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem32) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem32[wid] = v;
  __syncthreads();
  T r = 0;
  if (wid == 0) {
    r = (lane < (int)(blockDim.x >> 5)) ? smem32[lane] : T(0);
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace ncgp
