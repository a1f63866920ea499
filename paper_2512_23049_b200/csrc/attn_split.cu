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
// bf16 pools: tensor-core path (mma.sync m16n8k16, f32 accumulate), pages staged by a
// 3-stage cp.async pipeline.  Q and P enter the MMAs as hi/lo bf16 pairs, so the
// only bf16 rounding is the K/V storage itself.  f32 pools (parity variant): SIMT.
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
  int q_split, p_split;  // carry Q / P as hi+lo bf16 pairs in the MMAs (1) or plain bf16 (0)
};

// ============================================================ SIMT path (f32 pools)
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

// ============================================================ tensor-core path (bf16)
constexpr int kMmaThreads = 128;  // 4 warps
constexpr int kStages = 2;        // page double buffer (3 CTAs/SM at hd 128)
constexpr int kPage = 64;         // keys per page (= page_size for this path)

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
// hi = bf16(x), lo = bf16(x - hi), packed pairs
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                              uint32_t& r3, const void* ptr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(ptr)));
}

// Per-item state shared by the warps of a CTA.  Page descriptors of the item are
// pg[j], pl[j], po[j] for j < nv (global vis arrays offset by vb, or a fat record in smem).
struct ItemCtx {
  int kvh, vb, nv, pbase, M, G;
  int n_heads, n_kv, n_pages, page_size, layer;
  const int* s_rid;
  const int* s_rt;
  const int* pg;
  const int* pl;
  const int* po;
};

// One work item on one KV head.  MT = m16 query tiles (G*rows <= 16*MT); the KW = 4/MT
// warp groups split each page's 64 keys (warp w: m-tile w % MT, key slice w / MT) and
// walk their slice in 16-key chunks with an online softmax.  Hi and lo halves of Q and
// P run on separate accumulator chains so consecutive MMAs are independent.
template <int HD, int MT>
__device__ __forceinline__ void mma_item(const SplitParams& p, const ItemCtx& c,
                                         __nv_bfloat16* Ks, __nv_bfloat16* Vs, float* red) {
  constexpr int LD = HD + 8;
  constexpr int NT = HD / 8;
  constexpr int KS = HD / 16;
  constexpr int KW = 4 / MT;
  constexpr int SLICE = kPage / KW;  // keys per warp per page
  constexpr int CHUNKS = SLICE / 16;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int mt = warp % MT, kg = warp / MT;
  const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(p.k_pool);
  const __nv_bfloat16* vp = reinterpret_cast<const __nv_bfloat16*>(p.v_pool);

  auto load_page = [&](int stage, int pi) {
    if (pi < c.vb + c.nv) {
      const int page = c.pg[pi - c.vb], len = c.pl[pi - c.vb];
      const int64_t base = pool_off(c.layer, c.kvh, page, 0, c.n_kv, c.n_pages, c.page_size, HD);
      constexpr int CH = HD / 8;
#pragma unroll 4
      for (int q = tid; q < kPage * CH; q += kMmaThreads) {
        const int row = q / CH, col = (q % CH) * 8;
        const int nb = row < len ? 16 : 0;
        const int64_t src = base + (int64_t)(row < len ? row : 0) * HD + col;
        cp_async16(Ks + (stage * kPage + row) * LD + col, kp + src, nb);
        cp_async16(Vs + (stage * kPage + row) * LD + col, vp + src, nb);
      }
    }
    cp_async_commit();
  };
  load_page(0, c.vb);

  // Q fragments (hi/lo), rows m = mt*16 + {g, g+8}, pre-scaled to the log2 domain
  const float sl2 = p.scale * 1.4426950408889634f;
  uint32_t qh[KS][4], ql[KS][4];
  const int rowA = mt * 16 + g, rowB = rowA + 8;
  const bool vA = rowA < c.M, vB = rowB < c.M;
  const float* qA = p.q + ((int64_t)c.s_rid[vA ? rowA / c.G : 0] * c.n_heads + c.kvh * c.G + rowA % c.G) * HD;
  const float* qB = p.q + ((int64_t)c.s_rid[vB ? rowB / c.G : 0] * c.n_heads + c.kvh * c.G + rowB % c.G) * HD;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int c0 = ks * 16 + 2 * t;
    const float2 z = make_float2(0.f, 0.f);
    const float2 a0 = vA ? *reinterpret_cast<const float2*>(qA + c0) : z;
    const float2 a1 = vB ? *reinterpret_cast<const float2*>(qB + c0) : z;
    const float2 a2 = vA ? *reinterpret_cast<const float2*>(qA + c0 + 8) : z;
    const float2 a3 = vB ? *reinterpret_cast<const float2*>(qB + c0 + 8) : z;
    split2(a0.x * sl2, a0.y * sl2, qh[ks][0], ql[ks][0]);
    split2(a1.x * sl2, a1.y * sl2, qh[ks][1], ql[ks][1]);
    split2(a2.x * sl2, a2.y * sl2, qh[ks][2], ql[ks][2]);
    split2(a3.x * sl2, a3.y * sl2, qh[ks][3], ql[ks][3]);
  }
  const int rtA = vA ? c.s_rt[rowA / c.G] : -1, rtB = vB ? c.s_rt[rowB / c.G] : -1;

  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;

  for (int pi = c.vb; pi < c.vb + c.nv; ++pi) {
    const int stage = (pi - c.vb) & 1;
    load_page(stage ^ 1, pi + 1);  // prefetch next page into the other buffer
    cp_async_wait<1>();
    __syncthreads();
    const int len = c.pl[pi - c.vb], own = c.po[pi - c.vb];
    const __nv_bfloat16* Kt = Ks + stage * kPage * LD;
    const __nv_bfloat16* Vt = Vs + stage * kPage * LD;
#pragma unroll
    for (int ch = 0; ch < CHUNKS; ++ch) {
      const int k0 = kg * SLICE + ch * 16;
      if (k0 >= len) break;
      float sh[2][4], sl[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) sh[j][e] = sl[j][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const __nv_bfloat16* kr = Kt + (k0 + j * 8 + g) * LD + ks * 16 + 2 * t;
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + 8);
          mma16816(sh[j], qh[ks], b0, b1);
          if (p.q_split) mma16816(sl[j], ql[ks], b0, b1);
        }
      }
      float s[2][4];
      float tA = -INFINITY, tB = -INFINITY;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = k0 + j * 8 + 2 * t + e;
          const bool okA = vA && key < len && (own < 0 || own + key <= rtA);
          const bool okB = vB && key < len && (own < 0 || own + key <= rtB);
          s[j][e] = okA ? sh[j][e] + sl[j][e] : -INFINITY;
          s[j][2 + e] = okB ? sh[j][2 + e] + sl[j][2 + e] : -INFINITY;
          tA = fmaxf(tA, s[j][e]);
          tB = fmaxf(tB, s[j][2 + e]);
        }
      tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, 1));
      tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, 2));
      tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, 1));
      tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, 2));
      // lazy rescale: keep the running max unless it grows by more than 8 (log2 units),
      // so the O accumulators are rescaled only rarely (warp-uniform decision)
      float aA = 1.f, aB = 1.f;
      if (tA > mA + 8.f || (mA == -INFINITY && tA != -INFINITY)) {
        aA = mA == -INFINITY ? 0.f : exp2f(mA - tA);
        mA = tA;
      }
      if (tB > mB + 8.f || (mB == -INFINITY && tB != -INFINITY)) {
        aB = mB == -INFINITY ? 0.f : exp2f(mB - tB);
        mB = tB;
      }
      float sumA = 0.f, sumB = 0.f;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          s[j][e] = s[j][e] == -INFINITY ? 0.f : exp2f(s[j][e] - mA);
          s[j][2 + e] = s[j][2 + e] == -INFINITY ? 0.f : exp2f(s[j][2 + e] - mB);
          sumA += s[j][e];
          sumB += s[j][2 + e];
        }
      lA = lA * aA + sumA;
      lB = lB * aB + sumB;
      if (__any_sync(0xffffffffu, aA != 1.f || aB != 1.f)) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          o[n][0] *= aA;
          o[n][1] *= aA;
          o[n][2] *= aB;
          o[n][3] *= aB;
        }
      }
      uint32_t ph[4], pl[4];
      split2(s[0][0], s[0][1], ph[0], pl[0]);
      split2(s[0][2], s[0][3], ph[1], pl[1]);
      split2(s[1][0], s[1][1], ph[2], pl[2]);
      split2(s[1][2], s[1][3], ph[3], pl[3]);
      const int mi = lane >> 3;
      const __nv_bfloat16* vrow = Vt + (k0 + (mi & 1) * 8 + (lane & 7)) * LD + (mi >> 1) * 8;
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_trans(b0, b1, b2, b3, vrow + n * 8);
        mma16816(o[n], ph, b0, b1);
        mma16816(o[n + 1], ph, b2, b3);
        if (p.p_split) {
          mma16816(o[n], pl, b0, b1);
          mma16816(o[n + 1], pl, b2, b3);
        }
      }
    }
    __syncthreads();  // everyone done with this stage before it is refilled
  }
  cp_async_wait<0>();
  lA += __shfl_xor_sync(0xffffffffu, lA, 1);
  lA += __shfl_xor_sync(0xffffffffu, lA, 2);
  lB += __shfl_xor_sync(0xffffffffu, lB, 1);
  lB += __shfl_xor_sync(0xffffffffu, lB, 2);
  // ---- merge the KW key-slice warps of each m-tile through smem (reuses the pages) ----
  float* my = red + warp * (16 * HD + 32);
  if (KW > 1) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      *reinterpret_cast<float2*>(my + g * HD + n * 8 + 2 * t) = make_float2(o[n][0], o[n][1]);
      *reinterpret_cast<float2*>(my + (g + 8) * HD + n * 8 + 2 * t) = make_float2(o[n][2], o[n][3]);
    }
    if (t == 0) {
      my[16 * HD + g] = mA;
      my[16 * HD + g + 8] = mB;
      my[16 * HD + 16 + g] = lA;
      my[16 * HD + 16 + g + 8] = lB;
    }
  }
  __syncthreads();
  if (kg == 0) {
    float fmA = mA, fmB = mB;
#pragma unroll
    for (int k = 1; k < KW; ++k) {
      const float* ot = red + (warp + k * MT) * (16 * HD + 32);
      fmA = fmaxf(fmA, ot[16 * HD + g]);
      fmB = fmaxf(fmB, ot[16 * HD + g + 8]);
    }
    const float wA0 = fmA == -INFINITY ? 0.f : exp2f(mA - fmA);
    const float wB0 = fmB == -INFINITY ? 0.f : exp2f(mB - fmB);
    float LA = lA * wA0, LB = lB * wB0;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      o[n][0] *= wA0;
      o[n][1] *= wA0;
      o[n][2] *= wB0;
      o[n][3] *= wB0;
    }
#pragma unroll
    for (int k = 1; k < KW; ++k) {
      const float* ot = red + (warp + k * MT) * (16 * HD + 32);
      const float wA = fmA == -INFINITY ? 0.f : exp2f(ot[16 * HD + g] - fmA);
      const float wB = fmB == -INFINITY ? 0.f : exp2f(ot[16 * HD + g + 8] - fmB);
      LA += ot[16 * HD + 16 + g] * wA;
      LB += ot[16 * HD + 16 + g + 8] * wB;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const float2 xa = *reinterpret_cast<const float2*>(ot + g * HD + n * 8 + 2 * t);
        const float2 xb = *reinterpret_cast<const float2*>(ot + (g + 8) * HD + n * 8 + 2 * t);
        o[n][0] += wA * xa.x;
        o[n][1] += wA * xa.y;
        o[n][2] += wB * xb.x;
        o[n][3] += wB * xb.y;
      }
    }
    const float ln2 = 0.6931471805599453f;
    if (vA) {
      const int64_t pidx = (int64_t)(c.pbase + rowA / c.G) * c.n_heads + c.kvh * c.G + rowA % c.G;
      const float inv = LA > 0.f ? 1.f / LA : 0.f;
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<float2*>(p.part_o + pidx * HD + n * 8 + 2 * t) =
            make_float2(o[n][0] * inv, o[n][1] * inv);
      if (t == 0) p.part_lse[pidx] = LA > 0.f ? (fmA + log2f(LA)) * ln2 : -INFINITY;
    }
    if (vB) {
      const int64_t pidx = (int64_t)(c.pbase + rowB / c.G) * c.n_heads + c.kvh * c.G + rowB % c.G;
      const float inv = LB > 0.f ? 1.f / LB : 0.f;
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<float2*>(p.part_o + pidx * HD + n * 8 + 2 * t) =
            make_float2(o[n][2] * inv, o[n][3] * inv);
      if (t == 0) p.part_lse[pidx] = LB > 0.f ? (fmB + log2f(LB)) * ln2 : -INFINITY;
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(kMmaThreads, 3) attn_split_mma(SplitParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int LD = HD + 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [kStages][64][LD]
  __nv_bfloat16* Vs = Ks + kStages * kPage * LD;                     // [kStages][64][LD]
  float* red = reinterpret_cast<float*>(smem_raw);  // merge scratch, reuses the page stages
  __shared__ int s_rid[64], s_rt[64];
  const int tid = threadIdx.x;
  const int G = p.n_heads / p.n_kv;
  const int n_work = p.counts[1] * p.n_kv;
  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int32_t* it = p.items + 6 * (w / p.n_kv);
    const int rb = it[0], nr = it[1];
    __syncthreads();  // previous item fully done with smem
    for (int r = tid; r < nr; r += kMmaThreads) {
      const int rid = p.blk_rows[rb + r];
      s_rid[r] = rid;
      s_rt[r] = p.row_t[rid];
    }
    __syncthreads();
    ItemCtx c{w % p.n_kv, it[2], it[3], it[4], nr * G, G, p.n_heads, p.n_kv, p.n_pages,
              p.page_size, p.layer, s_rid, s_rt, p.vis_page + it[2], p.vis_len + it[2],
              p.vis_own + it[2]};
    if (c.M <= 16) mma_item<HD, 1>(p, c, Ks, Vs, red);
    else if (c.M <= 32) mma_item<HD, 2>(p, c, Ks, Vs, red);
    else mma_item<HD, 4>(p, c, Ks, Vs, red);
  }
}

// ============================================================ fused decode (fat items)
// Same math as attn_split_mma, for decode-sized steps: each CTA loads one self-contained
// 256-byte item record (K3 "fat" item) instead of chasing rows / row_t / page descriptors,
// and the LSE combine is fused: after writing its partials a CTA bumps an arrival counter
// per (row, kv head); the CTA that completes a row's count merges that row's partials for
// the G query heads of the KV head and writes the final bf16 (hi/lo) output row.
constexpr int kFatInts = 64;

struct DecodeParams {
  SplitParams sp;
  const int32_t* fat;
  const int32_t* row_part_off;
  const int32_t* row_part;
  int32_t* counters;  // [n_rows * n_kv], zero between launches (finalisers reset them)
  __nv_bfloat16* out;
  int out_split, n_rows;
};

template <int HD>
__device__ void finalize_row(const DecodeParams& d, int rid, int kvh, int G) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = d.row_part_off[rid], e = d.row_part_off[rid + 1];
  const int H = d.sp.n_heads;
  const bool active = 4 * lane < HD;
  for (int j = warp; j < G; j += 4) {
    const int h = kvh * G + j;
    float mx = -INFINITY;
    for (int i = b + lane; i < e; i += 32) mx = fmaxf(mx, d.sp.part_lse[(int64_t)d.row_part[i] * H + h]);
    mx = warp_max(mx);
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
    float den = 0.f;
    if (mx != -INFINITY) {
      for (int i = b; i < e; ++i) {
        const int pi = d.row_part[i];
        const float l = d.sp.part_lse[(int64_t)pi * H + h];
        if (l == -INFINITY) continue;
        const float wgt = __expf(l - mx);
        den += wgt;
        if (active) {
          const float4 o = *reinterpret_cast<const float4*>(d.sp.part_o + ((int64_t)pi * H + h) * HD + 4 * lane);
          num.x += wgt * o.x;
          num.y += wgt * o.y;
          num.z += wgt * o.z;
          num.w += wgt * o.w;
        }
      }
    }
    if (active) {
      const float inv = den > 0.f ? 1.f / den : 0.f;
      const float y[4] = {num.x * inv, num.y * inv, num.z * inv, num.w * inv};
      const int64_t oi = ((int64_t)rid * H + h) * HD + 4 * lane;
      uint32_t hv[2], lv[2];
      for (int k = 0; k < 2; ++k) split2(y[2 * k], y[2 * k + 1], hv[k], lv[k]);
      *reinterpret_cast<uint2*>(d.out + oi) = make_uint2(hv[0], hv[1]);
      if (d.out_split)
        *reinterpret_cast<uint2*>(d.out + (int64_t)d.n_rows * H * HD + oi) = make_uint2(lv[0], lv[1]);
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(kMmaThreads, 3) decode_attn_fused(DecodeParams d) {
  pdl_trigger();
  pdl_wait();
  constexpr int LD = HD + 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* Vs = Ks + kStages * kPage * LD;
  float* red = reinterpret_cast<float*>(smem_raw);
  __shared__ int s_fat[kFatInts];
  __shared__ int s_last[16];
  const SplitParams& p = d.sp;
  const int tid = threadIdx.x;
  const int G = p.n_heads / p.n_kv;
  const int n_work = p.counts[1] * p.n_kv;
  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int kvh = w % p.n_kv;
    __syncthreads();  // previous item fully done with smem
    if (tid < kFatInts) s_fat[tid] = d.fat[(int64_t)(w / p.n_kv) * kFatInts + tid];
    __syncthreads();
    const int nr = s_fat[0];
    ItemCtx c{kvh, 0, s_fat[1], s_fat[2], nr * G, G, p.n_heads, p.n_kv, p.n_pages, p.page_size,
              p.layer, s_fat + 4, s_fat + 20, s_fat + 36, s_fat + 44, s_fat + 52};
    if (c.M <= 16) mma_item<HD, 1>(p, c, Ks, Vs, red);
    else if (c.M <= 32) mma_item<HD, 2>(p, c, Ks, Vs, red);
    else mma_item<HD, 4>(p, c, Ks, Vs, red);
    // ---- fused combine: arrival counters per (row, kv head) ----
    if (!d.counters) continue;  // caller runs choreo_attn_combine instead
    __threadfence();
    __syncthreads();
    if (tid < nr) {
      const int rid = s_fat[4 + tid];
      const int total = d.row_part_off[rid + 1] - d.row_part_off[rid];
      const int old = atomicAdd(&d.counters[rid * p.n_kv + kvh], 1);
      s_last[tid] = (old == total - 1);
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
      if (!s_last[r]) continue;
      __threadfence();
      const int rid = s_fat[4 + r];
      finalize_row<HD>(d, rid, kvh, G);
      if (tid == 0) d.counters[rid * p.n_kv + kvh] = 0;
    }
  }
}

template <int HD>
static int launch_decode(const DecodeParams& d, int grid, cudaStream_t s) {
  constexpr int LD = HD + 8;
  const size_t pages = sizeof(__nv_bfloat16) * 2 * kStages * kPage * LD;
  const size_t merge = sizeof(float) * 4 * (16 * HD + 32);
  const size_t smem = pages > merge ? pages : merge;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(decode_attn_fused<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  launch_k(decode_attn_fused<HD>, grid, kMmaThreads, smem, s, d);
  return launch_status("choreo_decode_attn");
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
  for (; i < e; i += 4) {
    const int pi = row_part[i];
    const float l = part_lse[(int64_t)pi * n_heads + h];
    const float4 o = active ? *reinterpret_cast<const float4*>(part_o + ((int64_t)pi * n_heads + h) * hd + 4 * lane)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    rescale(l);
    add(l, o);
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

template <int HD>
static int launch_mma(const SplitParams& p, int grid, cudaStream_t s) {
  constexpr int LD = HD + 8;
  const size_t pages = sizeof(__nv_bfloat16) * 2 * kStages * kPage * LD;  // 2 x 2 x 17 KiB
  const size_t merge = sizeof(float) * 4 * (16 * HD + 32);
  const size_t smem = pages > merge ? pages : merge;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_split_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  launch_k(attn_split_mma<HD>, grid, kMmaThreads, smem, s, p);
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
                      int grid_ctas, int flags, void* stream) {
  if (!q || !k_pool || !v_pool || !row_t || !vis_page || !vis_len || !vis_own || !blk_rows ||
      !items || !counts || !part_o || !part_lse || !dtype_ok(pool_dtype) || n_kv <= 0 ||
      n_heads % n_kv)
    return CHOREO_EINVAL;
  if (max_items <= 0) return CHOREO_OK;
  SplitParams p{q, k_pool, v_pool, layer, n_kv, n_pages, page_size, n_heads, row_t, vis_page,
                vis_len, vis_own, blk_rows, items, counts, part_o, part_lse,
                1.0f / sqrtf((float)head_dim), (flags & 1) ? 1 : 0, (flags & 2) ? 1 : 0};
  auto s = as_stream(stream);
  const bool mma = pool_dtype == CHOREO_BF16 && page_size == kPage &&
                   (head_dim == 64 || head_dim == 128);
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  const int cap = mma ? 148 * 3 : 148 * 8;
  if (grid > cap) grid = cap;
  if (mma) return head_dim == 128 ? launch_mma<128>(p, grid, s) : launch_mma<64>(p, grid, s);
  return pool_dtype == CHOREO_BF16 ? dispatch_simt<__nv_bfloat16>(head_dim, p, grid, s)
                                   : dispatch_simt<float>(head_dim, p, grid, s);
}

int choreo_decode_attn(const float* q, const void* k_pool, const void* v_pool, int layer, int n_kv,
                       int n_pages, int page_size, int n_heads, int head_dim,
                       const int32_t* fat_items, const int32_t* counts, int max_items,
                       const int32_t* row_part_off, const int32_t* row_part, float* part_o,
                       float* part_lse, int32_t* row_counters, void* out, int out_split,
                       int n_rows, int flags, int grid_ctas, void* stream) {
  if (!q || !k_pool || !v_pool || !fat_items || !counts || !row_part_off || !row_part ||
      !part_o || !part_lse || (row_counters && !out) || n_kv <= 0 || n_heads % n_kv)
    return CHOREO_EINVAL;
  if (page_size != kPage || (head_dim != 64 && head_dim != 128) || (n_heads / n_kv) * 16 > 64 * 16)
    return CHOREO_EUNSUPPORTED;
  if (max_items <= 0) return CHOREO_OK;
  DecodeParams d{{q, k_pool, v_pool, layer, n_kv, n_pages, page_size, n_heads, nullptr, nullptr,
                  nullptr, nullptr, nullptr, nullptr, counts, part_o, part_lse,
                  1.0f / sqrtf((float)head_dim), (flags & 1) ? 1 : 0, (flags & 2) ? 1 : 0},
                 fat_items, row_part_off, row_part, row_counters,
                 reinterpret_cast<__nv_bfloat16*>(out), out_split, n_rows};
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  if (grid > 148 * 3) grid = 148 * 3;
  auto s = as_stream(stream);
  return head_dim == 128 ? launch_decode<128>(d, grid, s) : launch_decode<64>(d, grid, s);
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
