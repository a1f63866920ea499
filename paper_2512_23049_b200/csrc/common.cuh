// Shared helpers for the choreo B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/choreo_b200.h"

namespace choreo {

void set_last_error(const char* where, cudaError_t err);

// Record and translate the launch status of the kernel just issued.
inline int launch_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error(where, e);
    return CHOREO_ELAUNCH;
  }
  return CHOREO_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Generic element read of a dtype-coded buffer (f32 or bf16).
__device__ __forceinline__ float load_any(const void* p, int dtype, int64_t i) {
  return dtype == CHOREO_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
                              : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void store_any(void* p, int dtype, int64_t i, float v) {
  if (dtype == CHOREO_BF16)
    reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(p)[i] = v;
}

inline bool dtype_ok(int dt) { return dt == CHOREO_F32 || dt == CHOREO_BF16; }

// Pool element offset of (layer, kv head, page, slot, dim 0).
__host__ __device__ __forceinline__ int64_t pool_off(int layer, int h, int page, int slot,
                                                     int n_kv, int n_pages, int page_size,
                                                     int head_dim) {
  return ((((int64_t)layer * n_kv + h) * n_pages + page) * page_size + slot) * head_dim;
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

}  // namespace choreo
