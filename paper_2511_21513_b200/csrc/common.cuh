// common.cuh -- status/error plumbing shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "intattn_b200.h"

#ifndef IA_PROFILE
#define IA_PROFILE 0
#endif

namespace ia {

// Development A/B switch: read from the environment ONLY in the profiling build
// (make profile, -DIA_PROFILE=1); the release library always returns `dflt`, so no
// environment variable can change what the production kernels compute or how.
int dev_knob(const char* name, int dflt);

// Records a detail message for ia_last_error() and returns `status`.
int fail(int status, const char* fmt, ...);
// Checks cudaGetLastError() after a launch.
int check_launch(const char* what);
int num_sms();

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int32_t warp_max_i32(int32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace ia
