// K4 choreographed prefill attention on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Same work items as K5 (K3 page-centric groups; rows_per_block = 128 / G so one item is a
// 128-row M tile of (row, query head) vectors of one KV head) — each item computes
//   S = Q K^T  (tcgen05.mma, M=128, N=64 keys/page, K=head_dim; A and B from SW128 smem)
//   masked online softmax in registers (one TMEM lane = one query vector)
//   O += P V   (tcgen05.mma, M=128, N=head_dim, K=64; P staged bf16 in SW128 smem,
//               V as an MN-major operand straight from the TMA-loaded page)
// and writes a normalised partial + LSE per (row, head) for the combine kernel.
// The message-subset mask is applied at page granularity by construction (an item only
// lists visible pages: whole-tile skip); inside a page only the causal cut of the own
// message and the page's valid length are masked (reference masking.py:36-40,
// model.py:166-168).
//
// Roles (6 warps): warp 0 = TMA producer (K/V pages, 4-stage ring, mbarriers),
// warp 1 = MMA issuer (one thread), warps 2-5 = softmax/correction (TMEM lane quadrant =
// warp % 4), which also stage Q (f32 -> bf16, pre-scaled by log2(e)/sqrt(hd)).
#include <cudaTypedefs.h>
#include <math.h>

#include "common.cuh"
#include "sm100.cuh"

namespace choreo {

struct PrefillParams {
  const float* q;
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
  float scale_log2;
  int* dbg;  // optional progress counters (mapped host memory) for pipeline debugging
};

#define PF_DBG(i, v)                                     \
  do {                                                   \
    if (p.dbg && blockIdx.x == 0) {                      \
      *reinterpret_cast<volatile int*>(p.dbg + (i)) = (v); \
      __threadfence_system();                            \
    }                                                    \
  } while (0)

constexpr int kPfThreads = 192;
constexpr int kPfStages = 4;
constexpr int kPfKeys = 64;        // keys per page / per S tile
constexpr float kRescaleTh = 8.f;  // lazy O rescale threshold (log2 units)

template <int HD>
struct PfSmem {
  static constexpr int kRegions = HD / 64;                  // 64-column SW128 regions
  static constexpr int kQBytes = 128 * 128 * kRegions;      // [128 rows][HD] bf16
  static constexpr int kKVBytes = kPfKeys * 128 * kRegions; // one K (or V) page
  static constexpr int kStageBytes = 2 * kKVBytes;
  static constexpr int kPBytes = 128 * 128;                 // [128 rows][64 keys] bf16
  static constexpr int kTotal = kQBytes + kPfStages * kStageBytes + 2 * kPBytes + 1024;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// S tiles double-buffered in TMEM (cols [0,64) and [64,128)), O at [128, 128+HD);
// P double-buffered in smem.  Per page g (global index over this CTA's items):
//   MMA : S_{g+1} -> TMEM[(g+1)&1] is issued before PV_g, so the tensor core computes the
//         next scores while the softmax warps work on S_g;
//   SMX : ld S_g, release the S buffer, exp2, wait PV_{g-1}, write P_g, lazily rescale O.
template <int HD>
__global__ void __launch_bounds__(kPfThreads, 1)
    attn_prefill_sm100(PrefillParams p, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV) {
  using namespace sm100;
  using S = PfSmem<HD>;
  constexpr int R = S::kRegions;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;
  uint8_t* sKV = sQ + S::kQBytes;
  uint8_t* sP = sKV + kPfStages * S::kStageBytes;
  __shared__ uint64_t full_bar[kPfStages], empty_bar[kPfStages];
  __shared__ uint64_t s_full[2], s_free[2], p_full, o_done, q_full, o_free;
  __shared__ uint32_t tmem_base;
  __shared__ int s_rid[128], s_rt[128];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = p.n_heads / p.n_kv;
  const int n_work = p.counts[1] * p.n_kv;
  if (tid == 0) {
    for (int i = 0; i < kPfStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 128);
    }
    mbar_init(&p_full, 128);
    mbar_init(&o_done, 1);
    mbar_init(&q_full, 128);
    mbar_init(&o_free, 128);
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 1) tmem_alloc(&tmem_base, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS = tmem_base, tO = tmem_base + 128;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t gp = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int32_t* it = p.items + 6 * (w / p.n_kv);
        const int kvh = w % p.n_kv, vb = it[2], nv = it[3];
        for (int pi = vb; pi < vb + nv; ++pi, ++gp) {
          const int st = gp % kPfStages;
          mbar_wait(&empty_bar[st], ((gp / kPfStages) & 1) ^ 1);
          const int row0 = ((p.layer * p.n_kv + kvh) * p.n_pages + p.vis_page[pi]) * kPfKeys;
          uint8_t* dst = sKV + st * S::kStageBytes;
          mbar_arrive_expect_tx(&full_bar[st], S::kStageBytes);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            tma_load_2d(dst + r * kPfKeys * 128, &tmK, &full_bar[st], r * 64, row0);
            tma_load_2d(dst + S::kKVBytes + r * kPfKeys * 128, &tmV, &full_bar[st], r * 64, row0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, kPfKeys, false);
      constexpr uint32_t idO = umma_idesc_bf16(128, HD, true);
      const uint32_t qaddr = smem_addr(sQ);
      auto issue_s = [&](uint32_t g) {
        const int st = g % kPfStages, b = g & 1;
        mbar_wait(&full_bar[st], (g / kPfStages) & 1);
        mbar_wait(&s_free[b], ((g >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kaddr = smem_addr(sKV + st * S::kStageBytes);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k & 3) * 32;
          umma_bf16(tS + 64 * b, umma_desc_sw128(qaddr + (k >> 2) * 128 * 128 + off, 16, 1024),
                    umma_desc_sw128(kaddr + (k >> 2) * kPfKeys * 128 + off, 16, 1024), idS, k > 0);
        }
        umma_commit(&s_full[b]);
      };
      uint32_t gp = 0, ic = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++ic) {
        const int nv = p.items[6 * (w / p.n_kv) + 3];
        mbar_wait(&q_full, ic & 1);
        if (ic > 0) mbar_wait(&o_free, (ic - 1) & 1);
        tc_fence_after();
        issue_s(gp);
        for (int j = 0; j < nv; ++j, ++gp) {
          if (j + 1 < nv) issue_s(gp + 1);
          mbar_wait(&p_full, gp & 1);  // P_j written, O rescaled
          tc_fence_after();
          const int st = gp % kPfStages;
          const uint32_t vaddr = smem_addr(sKV + st * S::kStageBytes) + S::kKVBytes;
          const uint32_t paddr = smem_addr(sP + (gp & 1) * S::kPBytes);
#pragma unroll
          for (int k = 0; k < kPfKeys / 16; ++k)
            umma_bf16(tO, umma_desc_sw128(paddr + k * 32, 16, 1024),
                      umma_desc_sw128(vaddr + k * 2048, kPfKeys * 128, 1024), idO,
                      (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty_bar[st]);
          umma_commit(&o_done);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int quad = warp & 3;       // TMEM lane quadrant
    const int m = quad * 32 + lane;  // query vector (TMEM lane) of this thread
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int st_tid = tid - 64;     // 0..127
    uint32_t gp = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      const int32_t* it = p.items + 6 * (w / p.n_kv);
      const int kvh = w % p.n_kv, rb = it[0], nr = it[1], vb = it[2], nv = it[3], pbase = it[4];
      const int M = nr * G;
      if (st_tid < nr) {
        const int rid = p.blk_rows[rb + st_tid];
        s_rid[st_tid] = rid;
        s_rt[st_tid] = p.row_t[rid];
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      const bool valid = m < M;
      const int my_row = valid ? m / G : 0;
      const int my_t = valid ? s_rt[my_row] : -1;
      {  // stage Q (bf16, SW128 K-major, pre-scaled to the log2 domain)
        const float* qr = p.q + ((int64_t)s_rid[my_row] * p.n_heads + kvh * G + (valid ? m % G : 0)) * HD;
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) {
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
          if (valid) {
            a = *reinterpret_cast<const float4*>(qr + 8 * c);
            b = *reinterpret_cast<const float4*>(qr + 8 * c + 4);
          }
          const float sc = p.scale_log2;
          __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x * sc, a.y * sc);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(a.z * sc, a.w * sc);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x * sc, b.y * sc);
          __nv_bfloat162 h3 = __floats2bfloat162_rn(b.z * sc, b.w * sc);
          uint4 u;
          u.x = *reinterpret_cast<uint32_t*>(&h0);
          u.y = *reinterpret_cast<uint32_t*>(&h1);
          u.z = *reinterpret_cast<uint32_t*>(&h2);
          u.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(sQ + (c >> 3) * 128 * 128 + sw128_offset(m, (c & 7) * 8)) = u;
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&q_full);
      float mrow = -INFINITY, lrow = 0.f;  // mrow = max used for the exponentials (lazy)
      for (int j = 0; j < nv; ++j, ++gp) {
        const int pi = vb + j;
        const int len = p.vis_len[pi], own = p.vis_own[pi];
        const int b = gp & 1;
        mbar_wait(&s_full[b], (gp >> 1) & 1);
        tc_fence_after();
        float s[kPfKeys];
#pragma unroll
        for (int c = 0; c < kPfKeys / 16; ++c) tmem_ld16(tS + 64 * b + lane_off + c * 16, s + c * 16);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&s_free[b]);
        // keys visible to this row: k < lim (own pages: causal cut at my_t)
        int lim = valid ? len : 0;
        if (own >= 0) lim = min(lim, my_t - own + 1);
        float tmax = -INFINITY;
#pragma unroll
        for (int k = 0; k < kPfKeys; ++k) tmax = fmaxf(tmax, k < lim ? s[k] : -INFINITY);
        float alpha = 1.f;
        if (tmax > mrow + kRescaleTh || (mrow == -INFINITY && tmax != -INFINITY)) {
          alpha = mrow == -INFINITY ? 0.f : ex2(mrow - tmax);
          mrow = tmax;
        }
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < kPfKeys; ++k) {
          s[k] = k < lim ? ex2(s[k] - mrow) : 0.f;
          sum += s[k];
        }
        lrow = lrow * alpha + sum;
        if (j > 0) mbar_wait(&o_done, (gp - 1) & 1);  // PV_{g-1} done: O stable, P buffer free
        uint8_t* pb = sP + b * S::kPBytes;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          __nv_bfloat162 h0 = __floats2bfloat162_rn(s[8 * c], s[8 * c + 1]);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(s[8 * c + 2], s[8 * c + 3]);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(s[8 * c + 4], s[8 * c + 5]);
          __nv_bfloat162 h3 = __floats2bfloat162_rn(s[8 * c + 6], s[8 * c + 7]);
          uint4 u;
          u.x = *reinterpret_cast<uint32_t*>(&h0);
          u.y = *reinterpret_cast<uint32_t*>(&h1);
          u.z = *reinterpret_cast<uint32_t*>(&h2);
          u.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(pb + sw128_offset(m, 8 * c)) = u;
        }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HD / 16; ++c) {
            float o[16];
            tmem_ld16(tO + lane_off + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= alpha;
            tmem_st16(tO + lane_off + c * 16, o);
          }
          tmem_wait_st();
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full);
      }
      // ---- epilogue: O / l -> partial, LSE (natural log) ----
      mbar_wait(&o_done, (gp - 1) & 1);
      tc_fence_after();
      {
        // tcgen05.ld is warp-collective: every lane loads, only valid lanes store
        const int64_t pidx = (int64_t)(pbase + (valid ? m / G : 0)) * p.n_heads + kvh * G + m % G;
        const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
        float* dst = p.part_o + pidx * HD;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + lane_off + c * 16, o);
          tmem_wait_ld();
          if (valid) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              *reinterpret_cast<float4*>(dst + c * 16 + i) =
                  make_float4(o[i] * inv, o[i + 1] * inv, o[i + 2] * inv, o[i + 3] * inv);
          }
        }
        if (valid) p.part_lse[pidx] = lrow > 0.f ? (mrow + log2f(lrow)) * 0.6931471805599453f : -INFINITY;
      }
      tc_fence_before();
      mbar_arrive(&o_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, 256);
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 2D view of a pool: rows = layers*kv_heads*pages*page_size, cols = head_dim; box 64x64 SW128.
static bool encode_pool_map(CUtensorMap* map, const void* pool, uint64_t rows, int hd) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)hd, rows};
  const cuuint64_t strides[1] = {(cuuint64_t)hd * 2};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
static int launch_prefill(const PrefillParams& p, const void* k_pool, const void* v_pool,
                          uint64_t rows, int grid, cudaStream_t s) {
  CUtensorMap mk, mv;
  if (!encode_pool_map(&mk, k_pool, rows, HD) || !encode_pool_map(&mv, v_pool, rows, HD))
    return CHOREO_ELAUNCH;
  const int smem = PfSmem<HD>::kTotal;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_sm100<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  attn_prefill_sm100<HD><<<grid, kPfThreads, smem, s>>>(p, mk, mv);
  return launch_status("choreo_prefill_attn");
}

}  // namespace choreo

using namespace choreo;

extern "C" int choreo_prefill_attn_dbg(const float* q, const void* k_pool, const void* v_pool,
                                       int pool_dtype, int n_layers, int layer, int n_kv,
                                       int n_pages, int page_size, int n_heads, int head_dim,
                                       const int32_t* row_t, const int32_t* vis_page,
                                       const int32_t* vis_len, const int32_t* vis_own,
                                       const int32_t* blk_rows, const int32_t* items,
                                       const int32_t* counts, int max_items, float* part_o,
                                       float* part_lse, int grid_ctas, int* dbg, void* stream);

extern "C" int choreo_prefill_attn(const float* q, const void* k_pool, const void* v_pool,
                                   int pool_dtype, int n_layers, int layer, int n_kv, int n_pages,
                                   int page_size, int n_heads, int head_dim, const int32_t* row_t,
                                   const int32_t* vis_page, const int32_t* vis_len,
                                   const int32_t* vis_own, const int32_t* blk_rows,
                                   const int32_t* items, const int32_t* counts, int max_items,
                                   float* part_o, float* part_lse, int grid_ctas, void* stream) {
  return choreo_prefill_attn_dbg(q, k_pool, v_pool, pool_dtype, n_layers, layer, n_kv, n_pages,
                                 page_size, n_heads, head_dim, row_t, vis_page, vis_len, vis_own,
                                 blk_rows, items, counts, max_items, part_o, part_lse, grid_ctas,
                                 nullptr, stream);
}

extern "C" int choreo_prefill_attn_dbg(const float* q, const void* k_pool, const void* v_pool,
                                   int pool_dtype, int n_layers, int layer, int n_kv, int n_pages,
                                   int page_size, int n_heads, int head_dim, const int32_t* row_t,
                                   const int32_t* vis_page, const int32_t* vis_len,
                                   const int32_t* vis_own, const int32_t* blk_rows,
                                   const int32_t* items, const int32_t* counts, int max_items,
                                   float* part_o, float* part_lse, int grid_ctas, int* dbg,
                                   void* stream) {
  if (!q || !k_pool || !v_pool || !row_t || !vis_page || !vis_len || !vis_own || !blk_rows ||
      !items || !counts || !part_o || !part_lse || n_kv <= 0 || n_heads % n_kv)
    return CHOREO_EINVAL;
  if (pool_dtype != CHOREO_BF16 || page_size != kPfKeys || (head_dim != 64 && head_dim != 128) ||
      (n_heads / n_kv) > 128)
    return CHOREO_EUNSUPPORTED;
  if (max_items <= 0) return CHOREO_OK;
  PrefillParams p{q, layer, n_kv, n_pages, page_size, n_heads, row_t, vis_page, vis_len, vis_own,
                  blk_rows, items, counts, part_o, part_lse,
                  1.4426950408889634f / sqrtf((float)head_dim), dbg};
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  if (grid > 148) grid = 148;
  const uint64_t rows = (uint64_t)n_layers * n_kv * n_pages * page_size;
  if (rows > 0x7fffffffull) return CHOREO_EUNSUPPORTED;
  auto s = as_stream(stream);
  return head_dim == 128 ? launch_prefill<128>(p, k_pool, v_pool, rows, grid, s)
                         : launch_prefill<64>(p, k_pool, v_pool, rows, grid, s);
}
