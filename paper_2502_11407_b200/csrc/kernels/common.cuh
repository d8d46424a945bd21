// Shared device helpers for the gensor-b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

namespace gb::dev {

void check_cuda(cudaError_t e, const char* what);  // throws gb::Error(Cuda)

// Developer A/B switches (GENSOR_* environment variables) exist only in builds compiled with
// -DGENSOR_DEV_OVERRIDES (make DEV=1); the product library never reads the environment.
inline const char* dev_env(const char* name) {
#ifdef GENSOR_DEV_OVERRIDES
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}
void count_launch(uint64_t n = 1);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size (cached): setting it
// on every launch put host-side attribute work between dependent launches
void set_smem_attr(const void* kern, size_t bytes, const char* what);
template <typename F>
inline void set_smem_attr(F* kern, size_t bytes, const char* what) {
  set_smem_attr(reinterpret_cast<const void*>(kern), bytes, what);
}

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

}  // namespace gb::dev
