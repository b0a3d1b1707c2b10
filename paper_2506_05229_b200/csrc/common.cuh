// Shared helpers for the ARMT B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <atomic>
#include <string>

#include "../../include/armt_b200.h"

namespace armt {

// ---- error plumbing (host) ---------------------------------------------------
void set_error(const char* fmt, ...);
std::atomic<long long>& launch_counter();

#define ARMT_REQUIRE(cond, code, ...)         \
  do {                                        \
    if (!(cond)) {                            \
      ::armt::set_error(__VA_ARGS__);         \
      return (code);                          \
    }                                         \
  } while (0)

#define ARMT_CHECK_LAUNCH(what)                                                   \
  do {                                                                            \
    cudaError_t e_ = cudaGetLastError();                                          \
    if (e_ != cudaSuccess) {                                                      \
      ::armt::set_error("%s: %s", what, cudaGetErrorString(e_));                  \
      return ARMT_ERR_CUDA;                                                       \
    }                                                                             \
    ::armt::launch_counter().fetch_add(1, std::memory_order_relaxed);             \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

// A forked side stream per calling stream (created on first use, reused by every later
// call and graph capture from that stream): fork() makes the side stream wait for the
// caller's work so far, join() makes the caller wait for the side stream's. nullptr when
// more than 32 calling streams are in use; callers then run their side work in order on
// their own stream.
struct ForkedStream {
  cudaStream_t caller, side;
  cudaEvent_t fork_ev, join_ev;
  int fork();
  int join();
};
ForkedStream* forked_stream(cudaStream_t caller);
bool pdl_enabled();   // programmatic dependent launch for the tensor-core kernels (ARMT_PDL=0: off)

// ---- device helpers -------------------------------------------------------------
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float load_as_f32(const void* p, int dtype, long long i) {
  return dtype == ARMT_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
                            : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void store_from_f32(void* p, int dtype, long long i, float v) {
  if (dtype == ARMT_BF16)
    reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(p)[i] = v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Stable logistic with the reference's branch structure (armt/layers.py:149-156).
__device__ __forceinline__ float sigmoid_ref(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  float e = expf(x);
  return e / (1.f + e);
}
__device__ __forceinline__ float silu_ref(float x) { return x * sigmoid_ref(x); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace armt
