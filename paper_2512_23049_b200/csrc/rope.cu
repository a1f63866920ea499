// K1 rope_append and K2 rerotate: the two position kernels of the global cache.
//
// Rotation is the reference's interleaved-pair RoPE (tensor.py:87-143): pair i of a
// head vector is (x[2i], x[2i+1]) and rotates by delta * base^(-2i/hd).  The cos/sin
// values come from the f64-derived table cos/sin[(delta + W) * (hd/2) + i] stored as
// f32 (tensor.py:103-107), so index math is exact and values match the reference's
// table cast to f32.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace choreo {

// ---- K1 ------------------------------------------------------------------------
// One thread per rotation pair of (row, head); q heads first, then k heads, then v
// (v pairs are copied unrotated).  Writes q (f32) and the pool slot of each row.
template <typename TI, typename TP>
__global__ void rope_append_kernel(const TI* __restrict__ qkv, int ld, int n_rows, int split,
                                   const int32_t* __restrict__ pos,
                                   const int32_t* __restrict__ dst_page,
                                   const int32_t* __restrict__ dst_slot, float* __restrict__ q_out,
                                   TP* __restrict__ kp, TP* __restrict__ vp, int layer, int n_kv,
                                   int n_pages, int page_size, int n_heads, int hd,
                                   const float* __restrict__ cos_t,
                                   const float* __restrict__ sin_t, int max_delta,
                                   ChoreoK7Pieces pv, __nv_bfloat16* __restrict__ q_k5,
                                   float q_scale) {
  pdl_trigger();
  pdl_wait();
  const int half = hd >> 1;
  const int per_row = (n_heads + 2 * n_kv) * half;
  const int64_t total = (int64_t)n_rows * per_row;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(u / per_row);
    int rem = (int)(u % per_row);
    const int head = rem / half;  // 0..n_heads+2*n_kv-1 in qkv column order
    const int i = rem % half;
    const TI* src = qkv + (int64_t)r * ld + head * hd + 2 * i;
    float e, o;
    if (pv.ws) {  // deferred K7 qkv (f32; pairs never straddle a 128-column tile)
      float eo[2];
      k7_get<2>(pv, r, head * hd + 2 * i, eo);
      e = eo[0];
      o = eo[1];
    } else {
      e = to_f32(src[0]);
      o = to_f32(src[1]);
    }
    if (split) {  // stacked hi/lo GEMM halves (rows r and n_rows + r)
      e += to_f32(src[(int64_t)n_rows * ld]);
      o += to_f32(src[(int64_t)n_rows * ld + 1]);
    }
    if (head >= n_heads + n_kv) {  // v: copy
      const int h = head - n_heads - n_kv;
      TP* dst = vp + pool_off(layer, h, dst_page[r], dst_slot[r], n_kv, n_pages, page_size, hd) + 2 * i;
      dst[0] = from_f32<TP>(e);
      dst[1] = from_f32<TP>(o);
      continue;
    }
    const int64_t t = (int64_t)(pos[r] + max_delta) * half + i;
    const float c = cos_t[t], s = sin_t[t];
    const float re = e * c - o * s;
    const float ro = e * s + o * c;
    if (head < n_heads) {
      float* dst = q_out + ((int64_t)r * n_heads + head) * hd + 2 * i;
      dst[0] = re;
      dst[1] = ro;
      if (q_k5) {  // K5 v2's Q record: log2-domain scale, hi/lo bf16 halves [hi hd][lo hd]
        const float a0 = re * q_scale, a1 = ro * q_scale;
        const __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
        const float2 hf = __bfloat1622float2(h);
        __nv_bfloat16* k5 = q_k5 + ((int64_t)r * n_heads + head) * 2 * hd + 2 * i;
        *reinterpret_cast<__nv_bfloat162*>(k5) = h;
        *reinterpret_cast<__nv_bfloat162*>(k5 + hd) = __floats2bfloat162_rn(a0 - hf.x, a1 - hf.y);
      }
    } else {
      const int h = head - n_heads;
      TP* dst = kp + pool_off(layer, h, dst_page[r], dst_slot[r], n_kv, n_pages, page_size, hd) + 2 * i;
      dst[0] = from_f32<TP>(re);
      dst[1] = from_f32<TP>(ro);
    }
  }
}

// ---- K2 ------------------------------------------------------------------------
// One 16-byte vector (8 bf16 / 4 f32 = 4 / 2 pairs) per thread-iteration, 128-bit
// loads and stores, grid-stride over (layer, kv head, listed page, slot, vector).
// Pages with delta == 0 are skipped (reference: zero delta is a bitwise no-op,
// cache.py:152-153); slots past page_len are not touched.
template <typename T>
struct Vec16;
template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
};
template <>
struct Vec16<float> {
  static constexpr int N = 4;
};

// One CTA per (layer, kv head, listed page): the page's valid rows are one contiguous
// [len][hd] chunk, so the CTA reads it with 16-byte vectors, VPT vectors per thread all
// in flight before any is used, rotates in registers and writes back in place.  The cos/
// sin row of the page's delta is staged in shared memory once per CTA.
template <typename T, int VPT>
__global__ void __launch_bounds__(256) rerotate_kernel(
    T* __restrict__ kp, int n_kv, int n_pages, int page_size, int hd,
    const int32_t* __restrict__ pages, const int32_t* __restrict__ page_len,
    const int32_t* __restrict__ delta, int n_list, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, int max_delta) {
  pdl_trigger();
  pdl_wait();
  constexpr int N = Vec16<T>::N;  // elements per 16-byte vector
  extern __shared__ float cs[];   // [hd/2] cos then [hd/2] sin
  const int i = blockIdx.x % n_list;
  const int lh = blockIdx.x / n_list;
  const int dl = delta[i];
  if (dl == 0) return;
  const int len = page_len[i], half = hd >> 1;
  const int64_t trow = (int64_t)(dl + max_delta) * half;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    cs[j] = cos_t[trow + j];
    cs[half + j] = sin_t[trow + j];
  }
  __syncthreads();
  const int layer = lh / n_kv, h = lh % n_kv;
  T* base = kp + pool_off(layer, h, pages[i], 0, n_kv, n_pages, page_size, hd);
  const int vpr = hd / N, nvec = len * vpr;
  for (int v0 = threadIdx.x; v0 < nvec; v0 += blockDim.x * VPT) {
    uint4 raw[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int v = v0 + u * blockDim.x;
      if (v < nvec) raw[u] = *reinterpret_cast<const uint4*>(base + (int64_t)v * N);
    }
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int v = v0 + u * blockDim.x;
      if (v >= nvec) continue;
      T* x = reinterpret_cast<T*>(&raw[u]);
      const int p0 = (v % vpr) * (N / 2);
#pragma unroll
      for (int j = 0; j < N / 2; ++j) {
        const float c = cs[p0 + j], sn = cs[half + p0 + j];
        const float e = to_f32(x[2 * j]), o = to_f32(x[2 * j + 1]);
        x[2 * j] = from_f32<T>(e * c - o * sn);
        x[2 * j + 1] = from_f32<T>(e * sn + o * c);
      }
      *reinterpret_cast<uint4*>(base + (int64_t)v * N) = raw[u];
    }
  }
}

// bf16 pools, head_dim 64 / 128 (the 8B geometry): the page tile comes in by TMA (the
// pool's 2D view [layers*kv*pages*64][hd], SW128 boxes of 64 keys x 64 dims -- the map K4 /
// K5 v2 use), one bulk copy per (layer, kv head, listed page) CTA with no per-thread
// address math on the read side; the valid rows are rotated out of shared memory and
// written back with 16-byte stores (slots past page_len are never written).
template <int HD>
__global__ void __launch_bounds__(128) rerotate_tma_kernel(
    __nv_bfloat16* __restrict__ kp, const __grid_constant__ CUtensorMap tm, int n_kv,
    int n_pages, const int32_t* __restrict__ pages, const int32_t* __restrict__ page_len,
    const int32_t* __restrict__ delta, int n_list, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, int max_delta) {
  using namespace sm100;
  constexpr int kR = HD / 64, kHalf = 64 * 128;
  __shared__ __align__(1024) uint8_t tile[kR * kHalf];
  __shared__ float cs[HD];  // [hd/2] cos then [hd/2] sin
  __shared__ uint64_t bar;
  pdl_trigger();
  const int i = blockIdx.x % n_list;
  const int lh = blockIdx.x / n_list;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  const int dl = delta[i];
  if (dl == 0) return;
  const int len = page_len[i], half = HD >> 1;
  const int layer = lh / n_kv, h = lh % n_kv;
  const int64_t row0 = (((int64_t)layer * n_kv + h) * n_pages + pages[i]) * 64;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, kR * kHalf);
#pragma unroll
    for (int r = 0; r < kR; ++r) tma_load_2d(tile + r * kHalf, &tm, &bar, r * 64, (int)row0);
  }
  const int64_t trow = (int64_t)(dl + max_delta) * half;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    cs[j] = cos_t[trow + j];
    cs[half + j] = sin_t[trow + j];
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  __nv_bfloat16* base = kp + row0 * HD;
  constexpr int vpr = HD / 8;  // 16-byte vectors per key row
  const int nvec = len * vpr;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const int key = v / vpr, cch = v % vpr;
    uint4 raw = *reinterpret_cast<const uint4*>(tile + (cch >> 3) * kHalf + key * 128 +
                                                (((cch & 7) ^ (key & 7)) << 4));
    __nv_bfloat16* x = reinterpret_cast<__nv_bfloat16*>(&raw);
    const int p0 = cch * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float c = cs[p0 + j], sn = cs[half + p0 + j];
      const float e = __bfloat162float(x[2 * j]), o = __bfloat162float(x[2 * j + 1]);
      x[2 * j] = __float2bfloat16_rn(e * c - o * sn);
      x[2 * j + 1] = __float2bfloat16_rn(e * sn + o * c);
    }
    *reinterpret_cast<uint4*>(base + (int64_t)v * 8) = raw;
  }
}

static int grid_for(int64_t total, int threads) {
  int64_t b = (total + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace choreo

using namespace choreo;

extern "C" {

int choreo_rope_append(const void* qkv, int qkv_dtype, int ld_qkv, int n_rows, int qkv_split,
                       const int32_t* pos, const int32_t* dst_page, const int32_t* dst_slot,
                       float* q_out, void* k_pool, void* v_pool, int pool_dtype, int layer,
                       int n_kv, int n_pages, int page_size, int n_heads, int head_dim,
                       const float* cos_t, const float* sin_t, int max_delta, void* stream) {
  if (!qkv || !pos || !dst_page || !dst_slot || !q_out || !k_pool || !v_pool || !cos_t || !sin_t)
    return CHOREO_EINVAL;
  if (!dtype_ok(qkv_dtype) || !dtype_ok(pool_dtype) || head_dim < 2 || (head_dim & 1) ||
      n_kv <= 0 || n_heads % n_kv || ld_qkv < (n_heads + 2 * n_kv) * head_dim)
    return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  const int64_t total = (int64_t)n_rows * (n_heads + 2 * n_kv) * (head_dim / 2);
  const int blocks = grid_for(total, 256);
  auto s = as_stream(stream);
#define K1(TI, TP)                                                                               \
  launch_k(rope_append_kernel<TI, TP>, blocks, 256, 0, s,                                              \
      (const TI*)qkv, ld_qkv, n_rows, qkv_split, pos, dst_page, dst_slot, q_out, (TP*)k_pool, (TP*)v_pool, \
      layer, n_kv, n_pages, page_size, n_heads, head_dim, cos_t, sin_t, max_delta, ChoreoK7Pieces{}, \
      (__nv_bfloat16*)nullptr, 0.f)
  if (qkv_dtype == CHOREO_F32 && pool_dtype == CHOREO_F32) K1(float, float);
  else if (qkv_dtype == CHOREO_F32 && pool_dtype == CHOREO_BF16) K1(float, __nv_bfloat16);
  else if (qkv_dtype == CHOREO_BF16 && pool_dtype == CHOREO_BF16) K1(__nv_bfloat16, __nv_bfloat16);
  else K1(__nv_bfloat16, float);
#undef K1
  return launch_status("choreo_rope_append");
}

int choreo_rope_append_pieces_ex(const ChoreoK7Pieces* qkv, int n_rows, const int32_t* pos,
                                 const int32_t* dst_page, const int32_t* dst_slot, float* q_out,
                                 void* k_pool, void* v_pool, int pool_dtype, int layer, int n_kv,
                                 int n_pages, int page_size, int n_heads, int head_dim,
                                 const float* cos_t, const float* sin_t, int max_delta,
                                 void* q_k5, float q_scale, void* stream);

int choreo_rope_append_pieces(const ChoreoK7Pieces* qkv, int n_rows, const int32_t* pos,
                              const int32_t* dst_page, const int32_t* dst_slot, float* q_out,
                              void* k_pool, void* v_pool, int pool_dtype, int layer, int n_kv,
                              int n_pages, int page_size, int n_heads, int head_dim,
                              const float* cos_t, const float* sin_t, int max_delta,
                              void* stream) {
  return choreo_rope_append_pieces_ex(qkv, n_rows, pos, dst_page, dst_slot, q_out, k_pool, v_pool,
                                      pool_dtype, layer, n_kv, n_pages, page_size, n_heads,
                                      head_dim, cos_t, sin_t, max_delta, nullptr, 0.f, stream);
}

int choreo_rope_append_pieces_ex(const ChoreoK7Pieces* qkv, int n_rows, const int32_t* pos,
                                 const int32_t* dst_page, const int32_t* dst_slot, float* q_out,
                                 void* k_pool, void* v_pool, int pool_dtype, int layer, int n_kv,
                                 int n_pages, int page_size, int n_heads, int head_dim,
                                 const float* cos_t, const float* sin_t, int max_delta,
                                 void* q_k5, float q_scale, void* stream) {
  if (!qkv || !qkv->y || !qkv->ws || !pos || !dst_page || !dst_slot || !q_out || !k_pool ||
      !v_pool || !cos_t || !sin_t)
    return CHOREO_EINVAL;
  if (!dtype_ok(pool_dtype) || head_dim < 2 || (head_dim & 1) || n_kv <= 0 || n_heads % n_kv ||
      qkv->n < (n_heads + 2 * n_kv) * head_dim)
    return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  const int64_t total = (int64_t)n_rows * (n_heads + 2 * n_kv) * (head_dim / 2);
  const int blocks = grid_for(total, 256);
  auto s = as_stream(stream);
  if (pool_dtype == CHOREO_BF16)
    launch_k(rope_append_kernel<float, __nv_bfloat16>, blocks, 256, 0, s, qkv->y, qkv->n, n_rows, 0,
             pos, dst_page, dst_slot, q_out, (__nv_bfloat16*)k_pool, (__nv_bfloat16*)v_pool, layer,
             n_kv, n_pages, page_size, n_heads, head_dim, cos_t, sin_t, max_delta, *qkv,
             reinterpret_cast<__nv_bfloat16*>(q_k5), q_scale);
  else
    launch_k(rope_append_kernel<float, float>, blocks, 256, 0, s, qkv->y, qkv->n, n_rows, 0, pos,
             dst_page, dst_slot, q_out, (float*)k_pool, (float*)v_pool, layer, n_kv, n_pages,
             page_size, n_heads, head_dim, cos_t, sin_t, max_delta, *qkv, (__nv_bfloat16*)nullptr,
             0.f);
  return launch_status("choreo_rope_append_pieces");
}

int choreo_rerotate(void* k_pool, int pool_dtype, int n_layers, int n_kv, int n_pages,
                    int page_size, int head_dim, const int32_t* pages, const int32_t* page_len,
                    const int32_t* delta, int n_list, const float* cos_t, const float* sin_t,
                    int max_delta, void* stream) {
  if (!k_pool || !pages || !page_len || !delta || !cos_t || !sin_t || !dtype_ok(pool_dtype))
    return CHOREO_EINVAL;
  const int vec = pool_dtype == CHOREO_BF16 ? 8 : 4;
  if (head_dim % vec) return CHOREO_EINVAL;
  if (n_list == 0) return CHOREO_OK;
  const int64_t blocks = (int64_t)n_layers * n_kv * n_list;
  if (blocks > 0x7fffffff) return CHOREO_EUNSUPPORTED;
  auto s = as_stream(stream);
  const size_t smem = sizeof(float) * head_dim;
  const uint64_t pool_rows = (uint64_t)n_layers * n_kv * n_pages * page_size;
  if (pool_dtype == CHOREO_BF16 && page_size == 64 && (head_dim == 64 || head_dim == 128) &&
      pool_rows <= 0x7fffffffull) {
    CUtensorMap tm;
    if (!tmap_bf16_2d(&tm, k_pool, pool_rows, (uint64_t)head_dim, 64, 64,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
      return CHOREO_ELAUNCH;
    if (head_dim == 128)
      launch_k(rerotate_tma_kernel<128>, (int)blocks, 128, 0, s, (__nv_bfloat16*)k_pool, tm, n_kv,
               n_pages, pages, page_len, delta, n_list, cos_t, sin_t, max_delta);
    else
      launch_k(rerotate_tma_kernel<64>, (int)blocks, 128, 0, s, (__nv_bfloat16*)k_pool, tm, n_kv,
               n_pages, pages, page_len, delta, n_list, cos_t, sin_t, max_delta);
    return launch_status("choreo_rerotate");
  }
  if (pool_dtype == CHOREO_BF16)
    launch_k(rerotate_kernel<__nv_bfloat16, 4>, (int)blocks, 256, smem, s, 
        (__nv_bfloat16*)k_pool, n_kv, n_pages, page_size, head_dim, pages, page_len, delta, n_list,
        cos_t, sin_t, max_delta);
  else
    launch_k(rerotate_kernel<float, 4>, (int)blocks, 256, smem, s, (float*)k_pool, n_kv, n_pages, page_size,
                                                            head_dim, pages, page_len, delta, n_list,
                                                            cos_t, sin_t, max_delta);
  return launch_status("choreo_rerotate");
}

}  // extern "C"
