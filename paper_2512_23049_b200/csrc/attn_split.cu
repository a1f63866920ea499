// K5 split-KV choreographed attention over K3 work items.
//
// A work item is (block of <= rows_per_block rows, run of visible pages); a CTA
// takes one (item, kv head) and serves all G = n_heads / n_kv query heads of that
// KV head (GQA), so each K/V page is read once per item for G * rows query
// vectors.  Page-centric K3 items gather every row that sees a parent message, so
// in a parallel decode a shared parent page is read once for all agents.
// Masking: slot s of a page is visible to row r iff s < page_len and, for pages of
// the row's own message, own_base + s <= row_t[r] (masking.py:36-40 on pages).
// Each (row, head) of an item emits a normalised partial + LSE (natural log); the
// combine kernel merges a row's partials (reference model.py:177-184,
// tensor.py:65-75: scores, masked softmax, P.V).
//
// This is the generic path: f32 pools (the fp32 parity variant) and the shapes the
// tensor-core kernels do not take (head_dim not in {64, 128}, page size != 64, a
// bf16 decode with more than 32 query heads per KV head, per-call decode steps); SIMT
// with f32 math over bf16 or f32 pages.  bf16 decode-sized steps run K5 v2
// (attn_decode_v2.cu), prefill-sized ones K4 (attn_prefill_sm100.cu).
#include <math.h>

#include "common.cuh"

namespace choreo {

struct SplitParams {
  const float* q;
  const void* k_pool;
  const void* v_pool;
  int layer, n_kv, n_pages, page_size, n_heads;
  const int32_t* row_t;
  const int32_t* vis_page;
  const int32_t* vis_len;
  const int32_t* vis_own;
  const int32_t* blk_rows;
  const int32_t* items;
  const int32_t* counts;
  float* part_o;
  float* part_lse;
  float scale;
};

// ============================================================ SIMT path
constexpr int kThreads = 128;
constexpr int kMaxM = 64;  // rows_per_block * G must not exceed this
constexpr int kKT = 32;    // keys per smem tile

template <typename T, int HD>
__global__ void __launch_bounds__(kThreads) attn_split_simt(SplitParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int RPT = kMaxM * HD / kThreads;
  constexpr int GROUPS = kThreads / HD;
  extern __shared__ float smem[];
  float* Qs = smem;
  float* Ks = Qs + kMaxM * HD;
  float* Vs = Ks + kKT * (HD + 1);
  float* Ss = Vs + kKT * HD;
  float* rmax = Ss + kMaxM * (kKT + 1);
  float* rsum = rmax + kMaxM;
  float* alpha = rsum + kMaxM;
  int* rt = reinterpret_cast<int*>(alpha + kMaxM);
  int* rid = rt + kMaxM;

  const int tid = threadIdx.x;
  const int G = p.n_heads / p.n_kv;
  const int n_work = p.counts[1] * p.n_kv;
  const T* kp = reinterpret_cast<const T*>(p.k_pool);
  const T* vp = reinterpret_cast<const T*>(p.v_pool);

  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int32_t* it = p.items + 6 * (w / p.n_kv);
    const int kvh = w % p.n_kv;
    const int rb = it[0], nr = it[1], vb = it[2], nv = it[3], pbase = it[4];
    const int M = nr * G;
    for (int r = tid; r < nr; r += kThreads) {
      rid[r] = p.blk_rows[rb + r];
      rt[r] = p.row_t[rid[r]];
    }
    __syncthreads();
    for (int i = tid; i < M * HD; i += kThreads) {
      const int m = i / HD, d = i % HD;
      const int hq = kvh * G + (m % G);
      Qs[i] = p.q[((int64_t)rid[m / G] * p.n_heads + hq) * HD + d] * p.scale;
    }
    for (int m = tid; m < M; m += kThreads) {
      rmax[m] = -INFINITY;
      rsum[m] = 0.f;
    }
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

// ============================================================ combine
// One CTA (4 warps) per (row, head): lanes own 4 head dims each (float4), warps take
// every 4th partial slot of the row's CSR list with the loads of 4 slots in flight and keep
// an online (max, denominator, numerator) -- one pass over the partials, no separate max
// pass -- then the warps' states are merged in smem (LSE rule).
template <typename TO>
__global__ void __launch_bounds__(128) attn_combine_kernel(
    const float* __restrict__ part_o, const float* __restrict__ part_lse,
    const int32_t* __restrict__ row_part_off, const int32_t* __restrict__ row_part, int n_rows,
    int n_heads, int hd, int split, TO* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x / n_heads, h = blockIdx.x % n_heads;
  const int b = row_part_off[r], e = row_part_off[r + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float s_mx[4];
  __shared__ float4 s_num[4][32];
  __shared__ float s_den[4];
  const bool active = 4 * lane < hd;
  float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
  float den = 0.f, mx = -INFINITY;
  auto rescale = [&](float m_new) {
    if (m_new > mx) {
      const float f = mx == -INFINITY ? 0.f : __expf(mx - m_new);
      num.x *= f;
      num.y *= f;
      num.z *= f;
      num.w *= f;
      den *= f;
      mx = m_new;
    }
  };
  auto add = [&](float l, const float4& o) {
    if (l == -INFINITY) return;
    const float wgt = __expf(l - mx);
    den += wgt;
    num.x += wgt * o.x;
    num.y += wgt * o.y;
    num.z += wgt * o.z;
    num.w += wgt * o.w;
  };
  int i = b + warp;
  for (; i + 12 < e; i += 16) {  // 4 slots per warp iteration, loads batched
    int pi[4];
    float l[4];
    float4 o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pi[k] = row_part[i + 4 * k];
      l[k] = part_lse[(int64_t)pi[k] * n_heads + h];
      o[k] = active ? *reinterpret_cast<const float4*>(part_o + ((int64_t)pi[k] * n_heads + h) * hd + 4 * lane)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    rescale(fmaxf(fmaxf(l[0], l[1]), fmaxf(l[2], l[3])));
#pragma unroll
    for (int k = 0; k < 4; ++k) add(l[k], o[k]);
  }
  // the rest (< 16 slots per warp): the same per-slot rescale / add sequence as one slot at a
  // time, with the loads of up to 4 slots issued together (bitwise the same result)
  for (; i < e; i += 16) {
    int pi[4];
    float l[4];
    float4 o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) pi[k] = i + 4 * k < e ? row_part[i + 4 * k] : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      l[k] = -INFINITY;
      o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i + 4 * k < e) {
        l[k] = part_lse[(int64_t)pi[k] * n_heads + h];
        if (active)
          o[k] = *reinterpret_cast<const float4*>(part_o + ((int64_t)pi[k] * n_heads + h) * hd + 4 * lane);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i + 4 * k < e) {
        rescale(l[k]);
        add(l[k], o[k]);
      }
    }
  }
  s_num[warp][lane] = num;
  if (lane == 0) {
    s_den[warp] = den;
    s_mx[warp] = mx;
  }
  __syncthreads();
  if (warp == 0 && active) {
    const float M = fmaxf(fmaxf(s_mx[0], s_mx[1]), fmaxf(s_mx[2], s_mx[3]));
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    float dsum = 0.f;
    for (int k = 0; k < 4; ++k) {
      const float f = s_mx[k] == -INFINITY ? 0.f : __expf(s_mx[k] - M);
      t.x += f * s_num[k][lane].x;
      t.y += f * s_num[k][lane].y;
      t.z += f * s_num[k][lane].z;
      t.w += f * s_num[k][lane].w;
      dsum += f * s_den[k];
    }
    const float inv = dsum > 0.f ? 1.f / dsum : 0.f;
    const float y[4] = {t.x * inv, t.y * inv, t.z * inv, t.w * inv};
    const int64_t oi = ((int64_t)r * n_heads + h) * hd + 4 * lane;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const TO hi = from_f32<TO>(y[k]);
      out[oi + k] = hi;
      if (split) out[(int64_t)n_rows * n_heads * hd + oi + k] = from_f32<TO>(y[k] - to_f32(hi));
    }
  }
}

template <typename T, int HD>
static int launch_simt(const SplitParams& p, int grid, cudaStream_t s) {
  const size_t smem = sizeof(float) * (kMaxM * HD + kKT * (HD + 1) + kKT * HD +
                                       kMaxM * (kKT + 1) + 5 * kMaxM);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_split_simt<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr_set = true;
  }
  launch_k(attn_split_simt<T, HD>, grid, kThreads, smem, s, p);
  return launch_status("choreo_attn_split");
}

template <typename T>
static int dispatch_simt(int hd, const SplitParams& p, int grid, cudaStream_t s) {
  switch (hd) {
    case 8: return launch_simt<T, 8>(p, grid, s);
    case 16: return launch_simt<T, 16>(p, grid, s);
    case 32: return launch_simt<T, 32>(p, grid, s);
    case 64: return launch_simt<T, 64>(p, grid, s);
    case 128: return launch_simt<T, 128>(p, grid, s);
    default: return CHOREO_EUNSUPPORTED;
  }
}

}  // namespace choreo

using namespace choreo;

extern "C" {

int choreo_attn_split(const float* q, const void* k_pool, const void* v_pool, int pool_dtype,
                      int layer, int n_kv, int n_pages, int page_size, int n_heads, int head_dim,
                      const int32_t* row_t, const int32_t* vis_page, const int32_t* vis_len,
                      const int32_t* vis_own, const int32_t* blk_rows, const int32_t* items,
                      const int32_t* counts, int max_items, float* part_o, float* part_lse,
                      int grid_ctas, void* stream) {
  if (!q || !k_pool || !v_pool || !row_t || !vis_page || !vis_len || !vis_own || !blk_rows ||
      !items || !counts || !part_o || !part_lse || !dtype_ok(pool_dtype) || n_kv <= 0 ||
      n_heads % n_kv)
    return CHOREO_EINVAL;
  if (max_items <= 0) return CHOREO_OK;
  SplitParams p{q, k_pool, v_pool, layer, n_kv, n_pages, page_size, n_heads, row_t, vis_page,
                vis_len, vis_own, blk_rows, items, counts, part_o, part_lse,
                1.0f / sqrtf((float)head_dim)};
  auto s = as_stream(stream);
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  if (grid > 148 * 8) grid = 148 * 8;
  return pool_dtype == CHOREO_BF16 ? dispatch_simt<__nv_bfloat16>(head_dim, p, grid, s)
                                   : dispatch_simt<float>(head_dim, p, grid, s);
}

int choreo_attn_combine(const float* part_o, const float* part_lse, const int32_t* row_part_off,
                        const int32_t* row_part, int n_rows, int n_heads, int head_dim, void* out,
                        int out_dtype, int out_split, void* stream) {
  if (!part_o || !part_lse || !row_part_off || !row_part || !out || !dtype_ok(out_dtype))
    return CHOREO_EINVAL;
  if (out_split && out_dtype != CHOREO_BF16) return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  auto s = as_stream(stream);
  if (head_dim % 4 || head_dim > 128) return CHOREO_EUNSUPPORTED;
  const int threads = 128;
  if (out_dtype == CHOREO_BF16)
    launch_k(attn_combine_kernel<__nv_bfloat16>, n_rows * n_heads, threads, 0, s, 
        part_o, part_lse, row_part_off, row_part, n_rows, n_heads, head_dim, out_split,
        (__nv_bfloat16*)out);
  else
    launch_k(attn_combine_kernel<float>, n_rows * n_heads, threads, 0, s, 
        part_o, part_lse, row_part_off, row_part, n_rows, n_heads, head_dim, 0, (float*)out);
  return launch_status("choreo_attn_combine");
}

}  // extern "C"
