// Row-wise pieces of the forward step around the attention/GEMM hot ops:
// embedding gather, fused residual add + RMSNorm, SiLU-gate, greedy select (K6).
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace choreo {

static thread_local char g_err[256] = "";

void set_last_error(const char* where, cudaError_t err) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(err));
}

// sel (optional): row r embeds sel_src[sel[r]] instead of ids[r] when sel[r] >= 0 -- the
// token a device selection (K6 / K6b) of the previous step wrote, so a pipelined decode
// step needs no host round trip for its input ids.
__global__ void embed_kernel(const void* __restrict__ embed, int dt, int d,
                             const int32_t* __restrict__ ids, const int32_t* __restrict__ sel,
                             const int32_t* __restrict__ sel_src, float* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int si = sel ? sel[r] : -1;
  const int64_t src = (int64_t)(si >= 0 ? sel_src[si] : ids[r]) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) x[(int64_t)r * d + i] = load_any(embed, dt, src + i);
}

// One CTA per output row.  x is the f32 residual stream.
// Split activations: when out_split, row r of the output is written as a bf16
// pair hi = bf16(y), lo = bf16(y - hi) at rows r and n_out + r, so a bf16 GEMM over
// the stacked 2n rows followed by a sum of the halves sees y with ~16 mantissa bits
// (memory-bound decode GEMMs read the weights once either way).  delta_split sums
// such a stacked f32 GEMM output (rows r and n_rows + r) into the residual.
__device__ __forceinline__ void store_split(void* out, int dt, int64_t i_hi, int64_t i_lo,
                                            float y, int split) {
  if (split) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(y);
    reinterpret_cast<__nv_bfloat16*>(out)[i_hi] = hi;
    reinterpret_cast<__nv_bfloat16*>(out)[i_lo] = __float2bfloat16_rn(y - __bfloat162float(hi));
  } else {
    store_any(out, dt, i_hi, y);
  }
}

__global__ void residual_rmsnorm_kernel(float* __restrict__ x, const void* __restrict__ delta,
                                        int delta_dt, int delta_split, int n_rows,
                                        const void* __restrict__ w, int w_dt, int d,
                                        float eps, void* __restrict__ out, int out_dt,
                                        int out_split, const int32_t* __restrict__ row_map) {
  pdl_trigger();
  pdl_wait();
  const int r_out = blockIdx.x;
  const int r = row_map ? row_map[r_out] : r_out;
  float* xr = x + (int64_t)r * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = xr[i];
    if (delta) {
      v += load_any(delta, delta_dt, (int64_t)r * d + i);
      if (delta_split) v += load_any(delta, delta_dt, (int64_t)(n_rows + r) * d + i);
      xr[i] = v;
    }
    ss += v * v;
  }
  if (!out) return;
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    store_split(out, out_dt, (int64_t)r_out * d + i, (int64_t)(gridDim.x + r_out) * d + i,
                xr[i] * inv * load_any(w, w_dt, i), out_split);
}

// Vectorised variant (d % 4 == 0, f32 delta): every load of a row is issued before
// the first use (CH float4 chunks per thread kept in registers across both passes),
// so a row costs ~2 memory latencies instead of one per element.
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4_any(const void* p, int dt, int64_t i) {
  if (dt == CHOREO_BF16) {
    const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p) + i);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  return ld4(reinterpret_cast<const float*>(p) + i);
}
__device__ __forceinline__ void st4_split(void* out, int dt, int64_t i_hi, int64_t i_lo, float4 y,
                                          int split) {
  if (dt == CHOREO_BF16) {
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(y.x, y.y), h1 = __floats2bfloat162_rn(y.z, y.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&h0);
    u.y = *reinterpret_cast<const uint32_t*>(&h1);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + i_hi) = u;
    if (split) {
      const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
      const __nv_bfloat162 l0 = __floats2bfloat162_rn(y.x - f0.x, y.y - f0.y);
      const __nv_bfloat162 l1 = __floats2bfloat162_rn(y.z - f1.x, y.w - f1.y);
      u.x = *reinterpret_cast<const uint32_t*>(&l0);
      u.y = *reinterpret_cast<const uint32_t*>(&l1);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + i_lo) = u;
    }
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + i_hi) = y;
  }
}

template <int CH>
__global__ void __launch_bounds__(1024) residual_rmsnorm_vec(float* __restrict__ x, const float* __restrict__ delta,
                                     int delta_split, int n_rows, const void* __restrict__ w,
                                     int w_dt, int d, float eps, void* __restrict__ out, int out_dt,
                                     int out_split, const int32_t* __restrict__ row_map,
                                     ChoreoK7Pieces pv) {
  pdl_trigger();
  // the norm weight is static: fetched before the dependency wait, off the critical path
  const int nvec = d >> 2;
  float4 wv[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = threadIdx.x + c * blockDim.x;
    wv[c] = out && i < nvec ? ld4_any(w, w_dt, 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl_wait();
  const int r_out = blockIdx.x;
  const int r = row_map ? row_map[r_out] : r_out;
  float* xr = x + (int64_t)r * d;
  float4 v[CH];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = threadIdx.x + c * blockDim.x;
    v[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < nvec) {
      v[c] = ld4(xr + 4 * i);
      if (delta) {
        float4 a;
        if (pv.ws)
          choreo::k7_get<4, 4>(pv, r, 4 * i, &a.x);  // deferred K7 output
        else
          a = ld4(delta + (int64_t)r * d + 4 * i);
        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (delta_split) b = ld4(delta + (int64_t)(n_rows + r) * d + 4 * i);
        v[c].x += a.x + b.x;
        v[c].y += a.y + b.y;
        v[c].z += a.z + b.z;
        v[c].w += a.w + b.w;
        *reinterpret_cast<float4*>(xr + 4 * i) = v[c];
      }
    }
    ss += v[c].x * v[c].x + v[c].y * v[c].y + v[c].z * v[c].z + v[c].w * v[c].w;
  }
  if (!out) return;
  __shared__ float red[33];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[32] / (float)d + eps);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = threadIdx.x + c * blockDim.x;
    if (i < nvec) {
      const float4 y = make_float4(v[c].x * inv * wv[c].x, v[c].y * inv * wv[c].y,
                                   v[c].z * inv * wv[c].z, v[c].w * inv * wv[c].w);
      st4_split(out, out_dt, (int64_t)r_out * d + 4 * i, (int64_t)(gridDim.x + r_out) * d + 4 * i,
                y, out_split);
    }
  }
}

// The same (x += deferred K7 output; h = hi/lo(rmsnorm(x) * w)) with each row split over a
// cluster of kNc CTAs of 128 threads (one float4 per thread): the CTAs are small enough to
// become resident next to the running K7 CTAs (programmatic dependent launch), and the
// row's sum of squares is combined through distributed shared memory in the same order as
// residual_rmsnorm_vec (bit-identical outputs).
constexpr int kNc = 8;
__global__ void __launch_bounds__(128) residual_rmsnorm_cluster(float* __restrict__ x,
                                                               const void* __restrict__ w,
                                                               int w_dt, int d, float eps,
                                                               __nv_bfloat16* __restrict__ out,
                                                               int out_split, int n_rows,
                                                               ChoreoK7Pieces pv) {
  pdl_trigger();
  // CTA `part` of the row's cluster takes the 128-column blocks part, part + 8, part + 16,
  // part + 24 (one per warp): the first two levels of the 32-block butterfly below are then
  // CTA-local and only 8 values cross the cluster
  const int r = blockIdx.x / kNc, part = blockIdx.x % kNc;
  const int blk = part + kNc * (threadIdx.x >> 5);
  const int i = blk * 128 + 4 * (threadIdx.x & 31);  // this thread's 4 columns
  const bool on = blk < d / 128;
  const float4 wv = on ? ld4_any(w, w_dt, i) : make_float4(0.f, 0.f, 0.f, 0.f);
  pdl_wait();
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) {
    float* xr = x + (int64_t)r * d + i;
    v = ld4(xr);
    float4 a;
    choreo::k7_get<4, 8>(pv, r, i, &a.x);  // all of a tile's pieces in one round trip
    v.x += a.x;
    v.y += a.y;
    v.z += a.z;
    v.w += a.w;
    *reinterpret_cast<float4*>(xr) = v;
  }
  // the row's sum of squares in the 1024-thread kernel's exact order (bitwise the same
  // result): per-warp butterfly sums of 128-column blocks, then the butterfly over the 32
  // block sums (xor 16, 8, 4, 2, 1; absent blocks are +0, which adds exactly) -- its xor-16
  // and xor-8 levels inside this CTA, its xor-4, 2, 1 levels over the cluster's 8 partials
  __shared__ float red[4];
  __shared__ float part_s, tot_s;
  float ss = 0.f;
  ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;  // as residual_rmsnorm_vec
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) part_s = (red[0] + red[2]) + (red[1] + red[3]);
  // cluster barrier: every CTA's partial is written before any is read
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    float t = 0.f;
    if (lane < kNc) {
      const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&part_s));
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(lane));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(t) : "r"(remote) : "memory");
    }
    t += __shfl_xor_sync(0xffffffffu, t, 4);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    if (lane == 0) tot_s = t;
  }
  __syncthreads();
  const float tot = tot_s;
  // keep this CTA's shared memory alive until every CTA of the cluster has read it
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (!on) return;
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  const float4 y = make_float4(v.x * inv * wv.x, v.y * inv * wv.y, v.z * inv * wv.z, v.w * inv * wv.w);
  st4_split(out, CHOREO_BF16, (int64_t)r * d + i, (int64_t)(n_rows + r) * d + i, y, out_split);
}

__global__ void silu_mul_kernel(const void* __restrict__ gu, int dt, int in_split, int n_rows,
                                int f, void* __restrict__ out, int out_dt, int out_split) {
  pdl_trigger();
  pdl_wait();
  const int64_t n = (int64_t)n_rows * f, lo_in = (int64_t)n_rows * 2 * f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / f, c = i % f;
    float g = load_any(gu, dt, r * 2 * f + c);
    float u = load_any(gu, dt, r * 2 * f + f + c);
    if (in_split) {
      g += load_any(gu, dt, lo_in + r * 2 * f + c);
      u += load_any(gu, dt, lo_in + r * 2 * f + f + c);
    }
    store_split(out, out_dt, i, n + i, g / (1.0f + expf(-g)) * u, out_split);
  }
}

// f32 gate|up (stacked hi/lo halves when in_split) -> bf16 act (hi/lo when out_split), four
// columns per thread with 16-byte loads (the wide header step's prefill-sized GEMMs go
// through cuBLAS, so this runs over [2R][2F] f32 there).
__global__ void silu_mul_vec4_kernel(const float* __restrict__ gu, int in_split, int n_rows,
                                     int f, __nv_bfloat16* __restrict__ out, int out_split) {
  pdl_trigger();
  pdl_wait();
  const int f4 = f >> 2;
  const int n4 = n_rows * f4;
  const int64_t lo_in = (int64_t)n_rows * 2 * f, lo_out = (int64_t)n_rows * f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const int r = i / f4, c = (i - r * f4) * 4;
    const float* gp = gu + (int64_t)r * 2 * f + c;
    float4 g = *reinterpret_cast<const float4*>(gp);
    float4 u = *reinterpret_cast<const float4*>(gp + f);
    if (in_split) {
      const float4 gl = *reinterpret_cast<const float4*>(gp + lo_in);
      const float4 ul = *reinterpret_cast<const float4*>(gp + lo_in + f);
      g.x += gl.x; g.y += gl.y; g.z += gl.z; g.w += gl.w;
      u.x += ul.x; u.y += ul.y; u.z += ul.z; u.w += ul.w;
    }
    const float y[4] = {g.x / (1.0f + expf(-g.x)) * u.x, g.y / (1.0f + expf(-g.y)) * u.y,
                        g.z / (1.0f + expf(-g.z)) * u.z, g.w / (1.0f + expf(-g.w)) * u.w};
    __nv_bfloat16 h[4], l[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      h[k] = __float2bfloat16_rn(y[k]);
      l[k] = __float2bfloat16_rn(y[k] - __bfloat162float(h[k]));
    }
    const int64_t o = (int64_t)r * f + c;
    *reinterpret_cast<uint2*>(out + o) = *reinterpret_cast<const uint2*>(h);
    if (out_split) *reinterpret_cast<uint2*>(out + lo_out + o) = *reinterpret_cast<const uint2*>(l);
  }
}

// K6: one warp per row; generatable ids are 0..255 and 257 (EOS).  Ties keep the
// lowest id, as np.argmax does (engine.py:371).
__global__ void select_greedy_kernel(const float* __restrict__ logits, int n_rows, int64_t ld,
                                     int split, int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const float* lr = logits + row * ld;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = lane; i < 258; i += 32) {
    if (i == 256) continue;
    const float v = split ? lr[i] + lr[(int64_t)n_rows * ld + i] : lr[i];
    if (v > best || (v == best && i < idx)) { best = v; idx = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) { best = ob; idx = oi; }
  }
  if (lane == 0) out[row] = idx == 0x7fffffff ? 0 : idx;
}

}  // namespace choreo

using namespace choreo;

extern "C" {

int choreo_abi_version(void) { return 100; }

const char* choreo_last_error(void) { return g_err; }

int choreo_embed(const void* embed, int embed_dtype, int d, const int32_t* ids, int n_rows,
                 float* x, void* stream) {
  if (!embed || !ids || !x || d <= 0 || n_rows < 0 || !dtype_ok(embed_dtype)) return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  launch_k(embed_kernel, n_rows, 256, 0, as_stream(stream), embed, embed_dtype, d, ids,
           (const int32_t*)nullptr, (const int32_t*)nullptr, x);
  return launch_status("choreo_embed");
}

int choreo_embed_select(const void* embed, int embed_dtype, int d, const int32_t* ids,
                        const int32_t* sel, const int32_t* sel_src, int n_rows, float* x,
                        void* stream) {
  if (!embed || !ids || !sel || !sel_src || !x || d <= 0 || n_rows < 0 || !dtype_ok(embed_dtype))
    return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  launch_k(embed_kernel, n_rows, 256, 0, as_stream(stream), embed, embed_dtype, d, ids, sel,
           sel_src, x);
  return launch_status("choreo_embed_select");
}

int choreo_residual_rmsnorm(float* x, const void* delta, int delta_dtype, int delta_split,
                            const void* w, int w_dtype, int n_rows, int d, float eps, void* out,
                            int out_dtype, int out_split, const int32_t* row_map, int n_out,
                            void* stream) {
  if (!x || d <= 0 || n_rows < 0) return CHOREO_EINVAL;
  if (out && (!w || !dtype_ok(w_dtype) || !dtype_ok(out_dtype))) return CHOREO_EINVAL;
  if (delta && !dtype_ok(delta_dtype)) return CHOREO_EINVAL;
  if (row_map && (delta || !out)) return CHOREO_EINVAL;
  if (out_split && out_dtype != CHOREO_BF16) return CHOREO_EINVAL;
  const int rows = row_map ? n_out : n_rows;
  if (rows == 0) return CHOREO_OK;
  if (d % 4 == 0 && (!delta || delta_dtype == CHOREO_F32) && d <= 4 * 4 * 1024) {
    const int nvec = d / 4;
    int threads = nvec < 1024 ? ((nvec + 31) / 32) * 32 : 1024;
    if (nvec > 2048) threads = 1024;
    const int ch = (nvec + threads - 1) / threads;
    auto s = as_stream(stream);
#define RMS_VEC(CH)                                                                            \
  launch_k(residual_rmsnorm_vec<CH>, rows, threads, 0, s, x, (const float*)delta, delta_split, n_rows, \
                                                    w, w_dtype, d, eps, out, out_dtype,          \
                                                    out_split, row_map, ChoreoK7Pieces{})
    if (ch == 1) RMS_VEC(1);
    else if (ch == 2) RMS_VEC(2);
    else RMS_VEC(4);
#undef RMS_VEC
    return launch_status("choreo_residual_rmsnorm");
  }
  const int threads = d >= 2048 ? 512 : (d >= 256 ? 256 : 64);
  launch_k(residual_rmsnorm_kernel, rows, threads, 0, as_stream(stream), 
      x, delta, delta_dtype, delta_split, n_rows, w, w_dtype, d, eps, out, out_dtype, out_split,
      row_map);
  return launch_status("choreo_residual_rmsnorm");
}

static bool norm_cluster() {  // measurement switch: CHOREO_NORM_CLUSTER=0 -> 1024-thread CTAs
  static int v = -1;
  if (v < 0) v = getenv("CHOREO_NORM_CLUSTER") ? atoi(getenv("CHOREO_NORM_CLUSTER")) : 1;
  return v != 0;
}

int choreo_residual_rmsnorm_pieces(float* x, const ChoreoK7Pieces* delta, const void* w,
                                   int w_dtype, int n_rows, int d, float eps, void* out,
                                   int out_dtype, int out_split, void* stream) {
  if (!x || !delta || !delta->y || !delta->ws || !out || !w || d <= 0 || n_rows < 0 ||
      delta->n != d || !dtype_ok(w_dtype) || !dtype_ok(out_dtype))
    return CHOREO_EINVAL;
  if (out_split && out_dtype != CHOREO_BF16) return CHOREO_EINVAL;
  if (d % 4 || d > 4 * 4 * 1024) return CHOREO_EUNSUPPORTED;
  if (n_rows == 0) return CHOREO_OK;
  // (128-column blocks must not straddle CTAs: d a multiple of 128 kNc, at most 4 per CTA)
  if (out_dtype == CHOREO_BF16 && d % (128 * kNc) == 0 && d / kNc <= 4 * 128 && norm_cluster()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_rows * kNc);
    cfg.blockDim = dim3(128);
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kNc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, residual_rmsnorm_cluster, x, w, w_dtype, d, eps,
                       reinterpret_cast<__nv_bfloat16*>(out), out_split, n_rows, *delta);
    return launch_status("choreo_residual_rmsnorm_pieces");
  }
  const int nvec = d / 4;
  int threads = nvec < 1024 ? ((nvec + 31) / 32) * 32 : 1024;
  const int ch = (nvec + threads - 1) / threads;
  auto s = as_stream(stream);
#define RMS_VEC(CH)                                                                           \
  launch_k(residual_rmsnorm_vec<CH>, n_rows, threads, 0, s, x, delta->y, 0, n_rows, w, w_dtype, d, \
           eps, out, out_dtype, out_split, (const int32_t*)nullptr, *delta)
  if (ch == 1) RMS_VEC(1);
  else if (ch == 2) RMS_VEC(2);
  else RMS_VEC(4);
#undef RMS_VEC
  return launch_status("choreo_residual_rmsnorm_pieces");
}

int choreo_silu_mul(const void* gu, int gu_dtype, int in_split, int n_rows, int f, void* out,
                    int out_dtype, int out_split, void* stream) {
  if (!gu || !out || f <= 0 || n_rows < 0 || !dtype_ok(gu_dtype) || !dtype_ok(out_dtype))
    return CHOREO_EINVAL;
  if (out_split && out_dtype != CHOREO_BF16) return CHOREO_EINVAL;
  const int64_t n = (int64_t)n_rows * f;
  if (n == 0) return CHOREO_OK;
  if (gu_dtype == CHOREO_F32 && out_dtype == CHOREO_BF16 && f % 4 == 0 &&
      (int64_t)n_rows * 2 * f * (in_split ? 2 : 1) < (1ll << 31)) {
    int64_t blocks = (n / 4 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_k(silu_mul_vec4_kernel, (int)blocks, 256, 0, as_stream(stream),
             reinterpret_cast<const float*>(gu), in_split, n_rows, f,
             reinterpret_cast<__nv_bfloat16*>(out), out_split);
    return launch_status("choreo_silu_mul");
  }
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  launch_k(silu_mul_kernel, (int)blocks, 256, 0, as_stream(stream), gu, gu_dtype, in_split, n_rows, f,
                                                               out, out_dtype, out_split);
  return launch_status("choreo_silu_mul");
}

int choreo_select_greedy(const float* logits, int n_rows, int ld, int vocab, int split,
                         int32_t* out_tok, void* stream) {
  if (!logits || !out_tok || n_rows < 0 || vocab < 258 || ld < vocab) return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  const int warps = 4;
  launch_k(select_greedy_kernel, (n_rows + warps - 1) / warps, 32 * warps, 0, as_stream(stream), 
      logits, n_rows, ld, split, out_tok);
  return launch_status("choreo_select_greedy");
}

}  // extern "C"
