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
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

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
  // When out != nullptr every row has exactly one item: the epilogue writes the final
  // normalised row out[row][head*hd + d] (bf16; hi/lo pair at rows r / n_rows + r when
  // out_split) and no partials / combine are needed.
  __nv_bfloat16* out;
  int out_split, n_rows;
};


constexpr int kPfThreads = 352;     // 11 warps: TMA, MMA tile 0, 2 x 4 softmax, MMA tile 1
constexpr int kPfMma1Warp = 10;
constexpr int kPfStages = 4;
constexpr int kPfKeys = 64;         // keys per page / per S tile
constexpr int kTileM = 128;         // query vectors per tile (TMEM lanes)
constexpr float kRescaleTh = 8.f;   // lazy O rescale threshold (log2 units)

template <int HD>
struct PfSmem {
  static constexpr int kRegions = HD / 64;                  // 64-column SW128 regions
  static constexpr int kQBytes = kTileM * 128 * kRegions;   // one tile's [128][HD] bf16
  static constexpr int kKVBytes = kPfKeys * 128 * kRegions; // one K (or V) page
  static constexpr int kStageBytes = 2 * kKVBytes;
  static constexpr int kTotal = 2 * kQBytes + kPfStages * kStageBytes + 1024;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// sm_100a packed / 3-input forms (FADD2, FMNMX3) halve the softmax instruction count.
__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long x = *reinterpret_cast<unsigned long long*>(&a), y = *reinterpret_cast<unsigned long long*>(&b), z;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(x), "l"(y));
  return *reinterpret_cast<float2*>(&z);
}

// Two query tiles per CTA (M = 2 x 128 query vectors of one KV head) share every K/V
// page, and their MMAs ping-pong on the tensor core: while softmax warpgroup t works on
// S_t, the tensor core runs the other tile's S / PV.  TMEM (512 columns) per tile t:
// S double buffer at [256t, 256t+128), O at [256t+128, 256t+128+HD).  Per page g:
//   MMA : one issuing thread per tile (warps 1 and 10), so a tile's S(g+1) goes out as
//         soon as its PV(g-1) has, independent of the other tile's softmax progress;
//   SMX_t: ld S_t(g), release it, exp2, wait PV_t(g-1),
//          write P_t(g), lazily rescale O_t.
template <int HD>
__global__ void __launch_bounds__(kPfThreads, 1)
    attn_prefill_sm100(PrefillParams p, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV) {
  pdl_trigger();
  pdl_wait();
  using namespace sm100;
  using S = PfSmem<HD>;
  constexpr int R = S::kRegions;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;                                  // [2][kQBytes]
  uint8_t* sKV = sQ + 2 * S::kQBytes;                  // [stages][K | V]
  __shared__ uint64_t full_bar[kPfStages], empty_bar[kPfStages];
  __shared__ uint64_t s_full[2][2], p_full[2][2], o_done[2], q_full[2], o_free[2];
  __shared__ uint32_t tmem_base;
  __shared__ int s_rid[2][kTileM], s_rt[2][kTileM];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = p.n_heads / p.n_kv;
  const int rows_per_tile = kTileM / G;
  const int n_work = p.counts[1] * p.n_kv;
  if (tid == 0) {
    for (int i = 0; i < kPfStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 2);  // one release per tile issuer
    }
    for (int t = 0; t < 2; ++t) {
      for (int i = 0; i < 2; ++i) mbar_init(&s_full[t][i], 1);
      for (int i = 0; i < 2; ++i) mbar_init(&p_full[t][i], 128);
      mbar_init(&o_done[t], 1);
      mbar_init(&q_full[t], 128);
      mbar_init(&o_free[t], 128);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 1) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

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
  } else if (warp == 1 || warp == kPfMma1Warp) {
    // ------------------------------------------------------------ MMA issuers (per tile)
    if (lane == 0) {
      const int t = warp == 1 ? 0 : 1;
      constexpr uint32_t idS = umma_idesc_bf16(kTileM, kPfKeys, false);
      constexpr uint32_t idO = umma_idesc_bf16(kTileM, HD, true);
      // g = global page index (K/V ring), gt = this tile's page index (its barriers).
      // S(gt) goes to TMEM buffer gt&1; the softmax overwrites it with P(gt) (bf16 pairs),
      // which PV(gt) reads as its A operand.  The tensor pipe executes in issue order, so
      // S(gt+2) (same buffer) is issued only after PV(gt) — no extra handshake needed.
      auto issue_s = [&](uint32_t g, uint32_t gt) {
        const int st = g % kPfStages, b = gt & 1;
        mbar_wait(&full_bar[st], (g / kPfStages) & 1);
        tc_fence_after();
        const uint32_t qaddr = smem_addr(sQ + t * S::kQBytes);
        const uint32_t kaddr = smem_addr(sKV + st * S::kStageBytes);
        const uint32_t dS = tmem_base + 256 * t + 64 * b;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k & 3) * 32;
          umma_bf16(dS, umma_desc_sw128(qaddr + (k >> 2) * kTileM * 128 + off, 16, 1024),
                    umma_desc_sw128(kaddr + (k >> 2) * kPfKeys * 128 + off, 16, 1024), idS, k > 0);
        }
        umma_commit(&s_full[t][b]);
      };
      auto issue_pv = [&](uint32_t g, uint32_t gt, bool first) {
        // P(gt) lives in S buffer gt & 1; one barrier per buffer: a softmax group may finish
        // page gt + 1 before this wait runs (S(gt+1) is issued ahead of PV(gt)), so a single
        // barrier could be two phases ahead and its parity wait would never return
        mbar_wait(&p_full[t][gt & 1], (gt >> 1) & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_addr(sKV + (g % kPfStages) * S::kStageBytes) + S::kKVBytes;
        const uint32_t aP = tmem_base + 256 * t + 64 * (gt & 1);
        const uint32_t dO = tmem_base + 256 * t + 128;
#pragma unroll
        for (int k = 0; k < kPfKeys / 16; ++k)
          umma_bf16_tmem_a(dO, aP + k * 8, umma_desc_sw128(vaddr + k * 2048, kPfKeys * 128, 1024),
                           idO, (!first || k > 0) ? 1u : 0u);
        umma_commit(&o_done[t]);
      };
      uint32_t gp = 0, gt = 0, ic = 0;  // ring page, this tile's page, this tile's item
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int32_t* it = p.items + 6 * (w / p.n_kv);
        const int nv = it[3];
        if (t == 1 && it[1] <= rows_per_tile) {
          // tile 1 has no rows in this item: release each page once it has landed (waiting
          // for full keeps this issuer from running a ring round ahead of tile 0)
          for (int j = 0; j < nv; ++j, ++gp) {
            const int st = gp % kPfStages;
            mbar_wait(&full_bar[st], (gp / kPfStages) & 1);
            mbar_arrive(&empty_bar[st]);
          }
          continue;
        }
        mbar_wait(&q_full[t], ic & 1);
        if (ic > 0) mbar_wait(&o_free[t], (ic - 1) & 1);
        tc_fence_after();
        issue_s(gp, gt);
        for (int j = 0; j < nv; ++j, ++gp, ++gt) {
          if (j + 1 < nv) issue_s(gp + 1, gt + 1);
          issue_pv(gp, gt, j == 0);
          umma_commit(&empty_bar[gp % kPfStages]);
        }
        ++ic;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warpgroups
    const int t = (warp - 2) >> 2;      // tile of this warpgroup
    const int quad = warp & 3;          // TMEM lane quadrant
    const int m = quad * 32 + lane;     // query vector (TMEM lane) within the tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem_base + 256 * t, tO = tmem_base + 256 * t + 128;
    const int wg_tid = tid - 64 - 128 * t;  // 0..127
    uint8_t* myQ = sQ + t * S::kQBytes;
    uint32_t gp = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      const int32_t* it = p.items + 6 * (w / p.n_kv);
      const int kvh = w % p.n_kv, rb = it[0], nr = it[1], vb = it[2], nv = it[3], pbase = it[4];
      const int r0 = t * rows_per_tile;                       // first block row of this tile
      const int nr_t = max(0, min(rows_per_tile, nr - r0));   // rows of this tile
      if (nr_t == 0) continue;  // tile unused by this item (the MMA warp skips it too)
      const int M = nr_t * G;
      // the previous item's epilogue (other warps of this group) may still read s_rid / s_rt
      asm volatile("bar.sync %0, 128;\n" ::"r"(1 + t) : "memory");
      if (wg_tid < nr_t) {
        const int rid = p.blk_rows[rb + r0 + wg_tid];
        s_rid[t][wg_tid] = rid;
        s_rt[t][wg_tid] = p.row_t[rid];
      }
      asm volatile("bar.sync %0, 128;\n" ::"r"(1 + t) : "memory");
      const bool valid = m < M;
      const int my_row = valid ? m / G : 0;
      const int my_t = valid ? s_rt[t][my_row] : -1;
      {  // stage Q (bf16, SW128 K-major, pre-scaled to the log2 domain)
        const int rid = nr_t > 0 ? s_rid[t][my_row] : 0;
        const float* qr = p.q + ((int64_t)rid * p.n_heads + kvh * G + (valid ? m % G : 0)) * HD;
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
          *reinterpret_cast<uint4*>(myQ + (c >> 3) * kTileM * 128 + sw128_offset(m, (c & 7) * 8)) = u;
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&q_full[t]);
      float mrow = -INFINITY, lrow = 0.f;  // mrow = max used for the exponentials (lazy)
      for (int j = 0; j < nv; ++j, ++gp) {
        const int pi = vb + j;
        const int len = p.vis_len[pi], own = p.vis_own[pi];
        const int b = gp & 1;
        mbar_wait(&s_full[t][b], (gp >> 1) & 1);
        tc_fence_after();
        float s[kPfKeys];
#pragma unroll
        for (int c = 0; c < kPfKeys / 16; ++c) tmem_ld16(tS + 64 * b + lane_off + c * 16, s + c * 16);
        tmem_wait_ld();
        int lim = valid ? len : 0;  // keys k < lim are visible (own pages: causal cut)
        if (own >= 0) lim = min(lim, my_t - own + 1);
        // warp-uniform fast path: a full page visible to every row of the warp (most parent
        // pages) needs no per-key mask
        const bool full = __all_sync(0xffffffffu, lim >= kPfKeys);
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = -INFINITY;
        if (full) {
#pragma unroll
          for (int k = 0; k < kPfKeys; k += 2) mx[(k >> 1) & 7] = max3(mx[(k >> 1) & 7], s[k], s[k + 1]);
        } else {
#pragma unroll
          for (int k = 0; k < kPfKeys; ++k) mx[k & 7] = fmaxf(mx[k & 7], k < lim ? s[k] : -INFINITY);
        }
        const float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        float alpha = 1.f;
        if (tmax > mrow + kRescaleTh || (mrow == -INFINITY && tmax != -INFINITY)) {
          alpha = mrow == -INFINITY ? 0.f : ex2(mrow - tmax);
          mrow = tmax;
        }
        float sm[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) sm[i] = 0.f;
        if (full) {
          const float2 nm = make_float2(-mrow, -mrow);
          float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                           make_float2(0.f, 0.f)};
#pragma unroll
          for (int k = 0; k < kPfKeys; k += 2) {
            float2 x = add2(make_float2(s[k], s[k + 1]), nm);
            x.x = ex2(x.x);
            x.y = ex2(x.y);
            s[k] = x.x;
            s[k + 1] = x.y;
            acc[(k >> 1) & 3] = add2(acc[(k >> 1) & 3], x);
          }
          const float2 t2 = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
          sm[0] = t2.x + t2.y;
        } else {
#pragma unroll
          for (int k = 0; k < kPfKeys; ++k) {
            const float x = s[k] - mrow;
            const float e = ex2(x);
            s[k] = k < lim ? e : 0.f;
            sm[k & 7] += s[k];
          }
        }
        lrow = lrow * alpha + ((sm[0] + sm[1]) + (sm[2] + sm[3])) + ((sm[4] + sm[5]) + (sm[6] + sm[7]));
        // P(g) -> TMEM over the consumed S buffer (bf16 pairs, 32 columns of this lane)
        {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            __nv_bfloat162 h = __floats2bfloat162_rn(s[2 * c], s[2 * c + 1]);
            pk[c] = *reinterpret_cast<uint32_t*>(&h);
          }
          tmem_st16u(tS + 64 * b + lane_off, pk);
          tmem_st16u(tS + 64 * b + lane_off + 16, pk + 16);
        }
        // rescale the running O only when this warp's reference max moved (rare).  At the
        // item's last page PV_t(g-1) is always awaited: here o_done is at phase g-1 or g
        // (S(g) completing implies PV(g-2) did), so the parity wait is exact, and the
        // epilogue then has only PV_t(g) to wait for.  (Waiting for PV(g-1) in the epilogue
        // instead can deadlock: once PV(g-1) and PV(g) are both done, the barrier's current
        // phase has PV(g-1)'s parity and the wait blocks for a phase that never comes.)
        const bool resc = __any_sync(0xffffffffu, alpha != 1.f);
        if (j > 0 && (resc || j == nv - 1)) {
          mbar_wait(&o_done[t], (gp - 1) & 1);  // PV_t(g-1) done before touching O
          tc_fence_after();
          if (resc) {
#pragma unroll
            for (int c = 0; c < HD / 16; ++c) {
              float o[16];
              tmem_ld16(tO + lane_off + c * 16, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= alpha;
              tmem_st16(tO + lane_off + c * 16, o);
            }
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[t][b]);
      }
      // ---- epilogue: O / l -> partial, LSE (natural log) ----
      // only PV_t(last) can still be pending (PV_t(last-1) was awaited at the last page)
      mbar_wait(&o_done[t], (gp - 1) & 1);
      tc_fence_after();
      {
        // tcgen05.ld is warp-collective: every lane loads, only valid lanes store
        const int head = kvh * G + m % G;
        const int64_t pidx = (int64_t)(pbase + r0 + (valid ? m / G : 0)) * p.n_heads + head;
        const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
        float* dst = p.part_o + pidx * HD;
        __nv_bfloat16* od = p.out ? p.out + ((int64_t)(valid ? s_rid[t][my_row] : 0) * p.n_heads + head) * HD
                                  : nullptr;
        const int64_t lo_off = (int64_t)p.n_rows * p.n_heads * HD;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + lane_off + c * 16, o);
          tmem_wait_ld();
          if (valid) {
            if (od) {
#pragma unroll
              for (int i = 0; i < 16; i += 8) {
                uint4 hi, lo;
                uint32_t* hp = reinterpret_cast<uint32_t*>(&hi);
                uint32_t* lp = reinterpret_cast<uint32_t*>(&lo);
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2) {
                  const float a = o[i + 2 * q2] * inv, b = o[i + 2 * q2 + 1] * inv;
                  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
                  const float2 hf = __bfloat1622float2(h);
                  __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
                  hp[q2] = *reinterpret_cast<uint32_t*>(&h);
                  lp[q2] = *reinterpret_cast<uint32_t*>(&l);
                }
                *reinterpret_cast<uint4*>(od + c * 16 + i) = hi;
                if (p.out_split) *reinterpret_cast<uint4*>(od + lo_off + c * 16 + i) = lo;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(dst + c * 16 + i) =
                    make_float4(o[i] * inv, o[i + 1] * inv, o[i + 2] * inv, o[i + 3] * inv);
            }
          }
        }
        if (valid && !od) p.part_lse[pidx] = lrow > 0.f ? (mrow + log2f(lrow)) * 0.6931471805599453f : -INFINITY;
      }
      tc_fence_before();
      mbar_arrive(&o_free[t]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

// ---------------------------------------------------------------- host side
// 2D view of a pool: rows = layers*kv_heads*pages*page_size, cols = head_dim; box 64x64 SW128.
static bool encode_pool_map(CUtensorMap* map, const void* pool, uint64_t rows, int hd) {
  return tmap_bf16_2d(map, pool, rows, (uint64_t)hd, 64, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
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
    cudaFuncSetAttribute(attn_prefill_sm100<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    attr = true;
  }
  launch_k(attn_prefill_sm100<HD>, grid, kPfThreads, smem, s, p, mk, mv);
  return launch_status("choreo_prefill_attn");
}

}  // namespace choreo

using namespace choreo;

extern "C" int choreo_prefill_attn(const float* q, const void* k_pool, const void* v_pool,
                                   int pool_dtype, int n_layers, int layer, int n_kv, int n_pages,
                                   int page_size, int n_heads, int head_dim, const int32_t* row_t,
                                   const int32_t* vis_page, const int32_t* vis_len,
                                   const int32_t* vis_own, const int32_t* blk_rows,
                                   const int32_t* items, const int32_t* counts, int max_items,
                                   float* part_o, float* part_lse, int grid_ctas, void* out,
                                   int out_split, int n_rows, void* stream) {
  if (!q || !k_pool || !v_pool || !row_t || !vis_page || !vis_len || !vis_own || !blk_rows ||
      !items || !counts || !part_o || !part_lse || n_kv <= 0 || n_heads % n_kv)
    return CHOREO_EINVAL;
  if (pool_dtype != CHOREO_BF16 || page_size != kPfKeys || (head_dim != 64 && head_dim != 128) ||
      (n_heads / n_kv) > 128 || 128 % (n_heads / n_kv))
    return CHOREO_EUNSUPPORTED;
  if (max_items <= 0) return CHOREO_OK;
  PrefillParams p{q, layer, n_kv, n_pages, page_size, n_heads, row_t, vis_page, vis_len, vis_own,
                  blk_rows, items, counts, part_o, part_lse,
                  1.4426950408889634f / sqrtf((float)head_dim),
                  reinterpret_cast<__nv_bfloat16*>(out), out_split, n_rows};
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  if (grid > 148) grid = 148;
  const uint64_t rows = (uint64_t)n_layers * n_kv * n_pages * page_size;
  if (rows > 0x7fffffffull) return CHOREO_EUNSUPPORTED;
  auto s = as_stream(stream);
  if (head_dim == 128) return launch_prefill<128>(p, k_pool, v_pool, rows, grid, s);
  return launch_prefill<64>(p, k_pool, v_pool, rows, grid, s);
}
