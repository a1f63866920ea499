// Shared helpers for the choreo B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

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

// Programmatic dependent launch: a kernel that precedes a weight-streaming GEMM lets the
// GEMM (launched with the programmatic-serialization attribute) start its prologue and
// weight prefetch while this kernel still runs; the GEMM waits (griddepcontrol.wait)
// before it reads anything this kernel writes.  A no-op when no dependent is PDL-launched.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Every library kernel is launched with the programmatic-serialization attribute
// (env CHOREO_PDL=0 disables it) and starts with pdl_trigger(); pdl_wait() so the launch
// and CTA rasterisation of kernel N+1 overlap kernel N's execution while its memory work
// still starts after kernel N completed.
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CHOREO_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
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

// stream-K split of `iters` iterations over `grid` CTAs (K7): first iteration of CTA c, and
// the CTA owning iteration i (every CTA owns >= 1 iteration: grid <= iters)
// (32-bit unsigned arithmetic: c * iters and (i + 1) * grid stay below 2^32 for every
// shape here -- grid <= 148, iters <= 2^24 -- and a 64-bit division is a ~100-instruction
// software routine that these kernels inline in many places)
__host__ __device__ __forceinline__ int ln_begin(int c, int iters, int grid) {
  return (int)(((unsigned)c * (unsigned)iters) / (unsigned)grid);
}
__host__ __device__ __forceinline__ int ln_owner(int i, int iters, int grid) {
  return (int)((((unsigned)i + 1u) * (unsigned)grid - 1u) / (unsigned)iters);
}

// element (r, n..n+W-1) of a deferred K7 output (ChoreoK7Pieces): y for tiles one CTA owns,
// else the per-CTA partials of the tile (hi + lo halves already summed per piece) added in
// CTA order from 0 -- the reducer's order, so the values are bit-identical
template <int W, int B = 4>
__device__ __forceinline__ void k7_get(const ChoreoK7Pieces& v, int r, int n, float* out) {
  const int t = n >> 7, nl = n & 127;
  const int lo = t * v.kb, hi = lo + v.kb;
  const int c_lo = ln_owner(lo, v.iters, v.grid), c_hi = ln_owner(hi - 1, v.iters, v.grid);
  if (c_lo == c_hi) {
#pragma unroll
    for (int e = 0; e < W; ++e) out[e] = v.y[(size_t)r * v.n + n + e];
    return;
  }
  const int rows = v.split ? v.nx / 2 : v.nx;  // rows of one piece
  float a[W];
#pragma unroll
  for (int e = 0; e < W; ++e) a[e] = 0.f;
  // pieces are fetched B at a time (all loads in flight together), then added in CTA
  // order: a tile spans ~3-7 CTAs, one dependent round trip per piece would dominate
  for (int c0 = c_lo; c0 <= c_hi; c0 += B) {
    float pa[B][W];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const int cc = c0 + j;
      if (cc <= c_hi) {
        const int sl = ln_begin(cc, v.iters, v.grid) >= lo ? 0 : 1;
        const float* pc = v.ws + ((size_t)(cc * 2 + sl) * rows) * 128 + nl;
#pragma unroll
        for (int e = 0; e < W; ++e) pa[j][e] = pc[r * 128 + e];
      }
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      if (c0 + j <= c_hi) {
#pragma unroll
        for (int e = 0; e < W; ++e) a[e] += pa[j][e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < W; ++e) out[e] = a[e];
}

}  // namespace choreo
