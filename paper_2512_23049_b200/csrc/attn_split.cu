// K5 split-KV choreographed attention over assembled work items (SIMT f32 math).
//
// A work item is (row block, run of visible pages) from K3; a CTA takes one
// (item, kv head) pair and all G = n_heads / n_kv query heads of that KV head (GQA),
// so each K/V page is read once per item for G*rows query vectors.  Scores, the
// masked online softmax and P.V run in f32 (reference model.py:177-184,
// tensor.py:65-75); K/V are read from the paged pool in their storage dtype.
// Masking: slot s of a page is visible to row r iff s < page_len and, for pages of
// the row's own message, own_base + s <= row_t[r] (masking.py:36-40 restated on
// pages).  Each (row, head) of an item emits a normalised partial + LSE; the
// combine kernel merges a row's partials (flash-decoding split-KV).
#include <math.h>

#include "common.cuh"

namespace choreo {

constexpr int kThreads = 128;
constexpr int kMaxM = 64;  // rows_per_block * G must not exceed this
constexpr int kKT = 32;    // keys per smem tile

struct SplitParams {
  const float* q;
  const void* k_pool;
  const void* v_pool;
  int layer, n_kv, n_pages, page_size, n_heads;
  const int32_t* row_t;
  const int32_t* vis_page;
  const int32_t* vis_len;
  const int32_t* vis_own;
  const int32_t* items;
  const int32_t* counts;
  float* part_o;
  float* part_lse;
  float scale;
};

template <typename T, int HD>
__global__ void __launch_bounds__(kThreads) attn_split_simt(SplitParams p) {
  constexpr int RPT = kMaxM * HD / kThreads;  // accumulator rows per thread
  constexpr int GROUPS = kThreads / HD;       // row groups in the PV mapping
  extern __shared__ float smem[];
  float* Qs = smem;                        // [kMaxM][HD]
  float* Ks = Qs + kMaxM * HD;             // [kKT][HD + 1]
  float* Vs = Ks + kKT * (HD + 1);         // [kKT][HD]
  float* Ss = Vs + kKT * HD;               // [kMaxM][kKT + 1]
  float* rmax = Ss + kMaxM * (kKT + 1);    // [kMaxM]
  float* rsum = rmax + kMaxM;              // [kMaxM]
  float* alpha = rsum + kMaxM;             // [kMaxM]
  int* rt = reinterpret_cast<int*>(alpha + kMaxM);  // [kMaxM] row_t per local row

  const int tid = threadIdx.x;
  const int G = p.n_heads / p.n_kv;
  const int n_work = p.counts[1] * p.n_kv;
  const T* kp = reinterpret_cast<const T*>(p.k_pool);
  const T* vp = reinterpret_cast<const T*>(p.v_pool);

  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int32_t* it = p.items + 6 * (w / p.n_kv);
    const int kvh = w % p.n_kv;
    const int r0 = it[0], nr = it[1], vb = it[2], nv = it[3], pbase = it[4];
    const int M = nr * G;

    for (int i = tid; i < M * HD; i += kThreads) {
      const int m = i / HD, d = i % HD;
      const int hq = kvh * G + (m % G);
      Qs[i] = p.q[((int64_t)(r0 + m / G) * p.n_heads + hq) * HD + d] * p.scale;
    }
    for (int m = tid; m < M; m += kThreads) {
      rmax[m] = -INFINITY;
      rsum[m] = 0.f;
    }
    for (int r = tid; r < nr; r += kThreads) rt[r] = p.row_t[r0 + r];
    float acc[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) acc[j] = 0.f;
    __syncthreads();

    for (int pi = vb; pi < vb + nv; ++pi) {
      const int page = p.vis_page[pi], len = p.vis_len[pi], own = p.vis_own[pi];
      const int64_t base = pool_off(p.layer, kvh, page, 0, p.n_kv, p.n_pages, p.page_size, HD);
      for (int k0 = 0; k0 < len; k0 += kKT) {
        const int nk = min(kKT, len - k0);
        for (int i = tid; i < nk * HD; i += kThreads) {
          const int k = i / HD, d = i % HD;
          Ks[k * (HD + 1) + d] = to_f32(kp[base + (int64_t)k0 * HD + i]);
          Vs[i] = to_f32(vp[base + (int64_t)k0 * HD + i]);
        }
        __syncthreads();
        for (int i = tid; i < M * kKT; i += kThreads) {
          const int m = i / kKT, k = i % kKT;
          float s = -INFINITY;
          if (k < nk && (own < 0 || own + k0 + k <= rt[m / G])) {
            const float* qr = Qs + m * HD;
            const float* kr = Ks + k * (HD + 1);
            float a = 0.f;
#pragma unroll
            for (int d = 0; d < HD; ++d) a = fmaf(qr[d], kr[d], a);
            s = a;
          }
          Ss[m * (kKT + 1) + k] = s;
        }
        __syncthreads();
        for (int m = tid; m < M; m += kThreads) {
          float* sr = Ss + m * (kKT + 1);
          float tmax = -INFINITY;
          for (int k = 0; k < nk; ++k) tmax = fmaxf(tmax, sr[k]);
          const float old = rmax[m];
          const float nm = fmaxf(old, tmax);
          float sum = 0.f, al = 1.f;
          if (nm == -INFINITY) {
            for (int k = 0; k < nk; ++k) sr[k] = 0.f;
          } else {
            al = old == -INFINITY ? 0.f : expf(old - nm);
            for (int k = 0; k < nk; ++k) {
              const float e = sr[k] == -INFINITY ? 0.f : expf(sr[k] - nm);
              sr[k] = e;
              sum += e;
            }
            rmax[m] = nm;
          }
          rsum[m] = rsum[m] * al + sum;
          alpha[m] = al;
        }
        __syncthreads();
        {
          const int d = tid % HD;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            const int m = tid / HD + j * GROUPS;
            if (m < M) {
              const float* sr = Ss + m * (kKT + 1);
              float a = acc[j] * alpha[m];
              for (int k = 0; k < nk; ++k) a = fmaf(sr[k], Vs[k * HD + d], a);
              acc[j] = a;
            }
          }
        }
        __syncthreads();
      }
    }

    const int d = tid % HD;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int m = tid / HD + j * GROUPS;
      if (m < M) {
        const int hq = kvh * G + (m % G);
        const int64_t pidx = (int64_t)(pbase + m / G) * p.n_heads + hq;
        const float l = rsum[m];
        p.part_o[pidx * HD + d] = l > 0.f ? acc[j] / l : 0.f;
        if (d == 0) p.part_lse[pidx] = l > 0.f ? rmax[m] + logf(l) : -INFINITY;
      }
    }
    __syncthreads();
  }
}

template <typename TO>
__global__ void attn_combine_kernel(const float* __restrict__ part_o,
                                    const float* __restrict__ part_lse,
                                    const int32_t* __restrict__ row_part, int n_heads, int hd,
                                    int split, TO* __restrict__ out) {
  const int r = blockIdx.x;
  const int pb = row_part[3 * r], stride = row_part[3 * r + 1], n = row_part[3 * r + 2];
  for (int i = threadIdx.x; i < n_heads * hd; i += blockDim.x) {
    const int h = i / hd, d = i % hd;
    float mx = -INFINITY;
    for (int c = 0; c < n; ++c) mx = fmaxf(mx, part_lse[(int64_t)(pb + c * stride) * n_heads + h]);
    float num = 0.f, den = 0.f;
    if (mx != -INFINITY) {
      for (int c = 0; c < n; ++c) {
        const int64_t pi = (int64_t)(pb + c * stride) * n_heads + h;
        const float l = part_lse[pi];
        if (l == -INFINITY) continue;
        const float wgt = expf(l - mx);
        num += wgt * part_o[pi * hd + d];
        den += wgt;
      }
    }
    const float y = den > 0.f ? num / den : 0.f;
    const int64_t oi = ((int64_t)r * n_heads + h) * hd + d;
    const TO hi = from_f32<TO>(y);
    out[oi] = hi;
    if (split) out[(int64_t)gridDim.x * n_heads * hd + oi] = from_f32<TO>(y - to_f32(hi));
  }
}

template <typename T, int HD>
static int launch_split(const SplitParams& p, int grid, cudaStream_t s) {
  const size_t smem = sizeof(float) * (kMaxM * HD + kKT * (HD + 1) + kKT * HD +
                                       kMaxM * (kKT + 1) + 4 * kMaxM);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_split_simt<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr_set = true;
  }
  attn_split_simt<T, HD><<<grid, kThreads, smem, s>>>(p);
  return launch_status("choreo_attn_split");
}

template <typename T>
static int dispatch_hd(int hd, const SplitParams& p, int grid, cudaStream_t s) {
  switch (hd) {
    case 8: return launch_split<T, 8>(p, grid, s);
    case 16: return launch_split<T, 16>(p, grid, s);
    case 32: return launch_split<T, 32>(p, grid, s);
    case 64: return launch_split<T, 64>(p, grid, s);
    case 128: return launch_split<T, 128>(p, grid, s);
    default: return CHOREO_EUNSUPPORTED;
  }
}

}  // namespace choreo

using namespace choreo;

extern "C" {

int choreo_attn_split(const float* q, const void* k_pool, const void* v_pool, int pool_dtype,
                      int layer, int n_kv, int n_pages, int page_size, int n_heads, int head_dim,
                      const int32_t* row_t, const int32_t* vis_page, const int32_t* vis_len,
                      const int32_t* vis_own, const int32_t* items, const int32_t* counts,
                      int max_items, float* part_o, float* part_lse, int grid_ctas,
                      void* stream) {
  if (!q || !k_pool || !v_pool || !row_t || !vis_page || !vis_len || !vis_own || !items ||
      !counts || !part_o || !part_lse || !dtype_ok(pool_dtype) || n_kv <= 0 ||
      n_heads % n_kv)
    return CHOREO_EINVAL;
  if (max_items <= 0) return CHOREO_OK;
  SplitParams p{q, k_pool, v_pool, layer, n_kv, n_pages, page_size, n_heads, row_t, vis_page,
                vis_len, vis_own, items, counts, part_o, part_lse,
                1.0f / sqrtf((float)head_dim)};
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  if (grid > 148 * 8) grid = 148 * 8;
  auto s = as_stream(stream);
  return pool_dtype == CHOREO_BF16 ? dispatch_hd<__nv_bfloat16>(head_dim, p, grid, s)
                                   : dispatch_hd<float>(head_dim, p, grid, s);
}

int choreo_attn_combine(const float* part_o, const float* part_lse, const int32_t* row_part,
                        int n_rows, int n_heads, int head_dim, void* out, int out_dtype,
                        int out_split, void* stream) {
  if (!part_o || !part_lse || !row_part || !out || !dtype_ok(out_dtype)) return CHOREO_EINVAL;
  if (out_split && out_dtype != CHOREO_BF16) return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  auto s = as_stream(stream);
  if (out_dtype == CHOREO_BF16)
    attn_combine_kernel<__nv_bfloat16><<<n_rows, 256, 0, s>>>(part_o, part_lse, row_part, n_heads,
                                                              head_dim, out_split, (__nv_bfloat16*)out);
  else
    attn_combine_kernel<float><<<n_rows, 256, 0, s>>>(part_o, part_lse, row_part, n_heads,
                                                      head_dim, 0, (float*)out);
  return launch_status("choreo_attn_combine");
}

}  // extern "C"
