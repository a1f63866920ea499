// K5 (v2) choreographed decode attention: TMA page ring + FA2-style mma.sync consumers.
//
// Work unit = (K3 item, kv head): a block of <= 32 / G rows that all see a run of pages
// (page-centric K3 items gather every agent that lists a parent message, so a shared
// parent page is read from HBM once per step for all agents).  Per CTA (persistent, one
// per SM):
//   warp 8      TMA producer: streams each unit's K and V pages (2D tensor maps over the
//               pool, SW128 boxes of 64 keys x 64 dims) into a 4-slot ring, mbarriers;
//   warp 9      unit loader: stages the next unit's rows, page lengths and Q (bf16) in smem;
//   warps 10-11 merge warps (one per m-tile): combine the four key-slice states of a unit
//               and write its partials while the compute warps already stream the next unit;
//   warps 0-7   consumers, warp = (key slice q4 in 0..3, m-tile mt in 0..1): every page's
//               64 keys are split four ways (16 keys per warp), the <= 32 (row, query head)
//               vectors in two m16 tiles; S = Q K^T and O += P V on mma.sync m16n8k16
//               (Q as a hi/lo bf16 pair, P bf16, f32 accumulate) with K / V fragments from
//               ldmatrix on the swizzled
//               tiles, online softmax in registers (lazy O rescale), no per-page CTA barrier;
//   unit end    the four key-slice states of an m-tile are merged through shared memory
//               (asynchronously: slices 1-3 hand over and move on) and one normalised
//               partial + LSE per (row, head) is written for the combine.
// Masking: slot s of a page is visible to row r iff s < page_len and, for the row's own
// pages, own_base + s <= row_t[r] (reference masking.py:36-40, model.py:166-168, 177-184).
#include <cudaTypedefs.h>
#include <math.h>

#include <cuda_fp16.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace choreo {

constexpr int kDvSlots = 4;        // K/V page ring
constexpr int kDvConsumers = 8;    // warps 0-7
constexpr int kDvProducer = 8;     // warp 8: TMA
constexpr int kDvLoader = 9;       // warp 9: unit metadata + Q staging
constexpr int kDvMerge = 10;       // warps 10, 11: merge the key-slice states of m-tile 0 / 1
constexpr int kDvThreads = 32 * 12;
constexpr int kDvUnits = 3;        // unit records the loader may run ahead by
constexpr int kDvMaxPages = 32;    // pages per unit staged in the unit record (host: ppi <= 32)

struct DvParams {
  const float* q;
  int layer, n_kv, n_pages, n_heads;
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
  const int32_t* fat;  // optional K3 item records (rows <= 16): faster unit staging
  int trace_slot;      // diagnostics builds (-DCHOREO_TRACE) only
  // optional: Q already in the unit record's format (log2-domain scale, hi/lo bf16,
  // [row][head][2][HD], written by RoPE) -- staged by 1-D bulk copies instead of loads
  const __nv_bfloat16* q_k5;
  // optional: K3's item order (page count descending).  A step with more units than CTAs
  // deals them longest-first, snaking across the grid; else unit w = blockIdx.x + k * grid
  const int32_t* order;
  // != 0: the step's K3 stamps counts[4] with this tag once its outputs are complete; the
  // loader and producer then do their first lookups before the dependency wait
  int k3_tag;
};

// k-th unit of this CTA (-1: none left).  Round k covers units [k G, k G + G) (G = grid);
// with `snake` odd rounds run backwards, so the CTA that took round k's longest unit takes
// round k+1's shortest.
__device__ __forceinline__ int dv_unit(int k, int n_work, bool snake) {
  const int g = gridDim.x;
  const int s = k * g + ((snake && (k & 1)) ? g - 1 - (int)blockIdx.x : (int)blockIdx.x);
  return s < n_work ? s : -1;
}
// item of each of the 32 units k0 + lane (one round trip for 32 units; -1 past the end)
__device__ __forceinline__ int dv_items32(const DvParams& p, int k0, int lane, int n_work,
                                          bool snake) {
  const int s = dv_unit(k0 + lane, n_work, snake);
  if (s < 0) return -1;
  return snake ? p.order[s / p.n_kv] : s / p.n_kv;
}

#ifdef CHOREO_TRACE
__device__ long long* g_dv_trace = nullptr;
__device__ __forceinline__ void dv_trace(int slot, int i) {
  if (g_dv_trace) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dv_trace[((size_t)(slot & 63) * 148 + blockIdx.x) * 16 + i] = t;
  }
}
static int g_dv_launches = 0;
#define DTR(i) dv_trace(p.trace_slot, i)
#else
#define DTR(i) \
  do {         \
  } while (0)
#endif

template <int HD>
struct DvCfg {
  static constexpr int kR = HD / 64;                      // 64-dim SW128 halves per page
  static constexpr int kHalf = 64 * 128;                  // bytes of one [64][64] bf16 tile
  static constexpr int kSlot = 2 * kR * kHalf;            // K + V of one page
  // merge scratch: per (key slice, m-tile) 16 rows of the slice's NORMALISED O in f16
  // (|O / l| <= max |v|: f16 range is safe, 11-bit mantissa) + (m, l) in f32, then a
  // 4-int header (M, pbase, kvh)
  static constexpr int kMergeRow = HD + 8;                // f16 elements per row (16-B rows)
  static constexpr int kMergeO = 4 * 2 * 16 * kMergeRow * 2;
  static constexpr int kMergeML = 4 * 2 * 16 * 8;
  static constexpr int kMerge = kMergeO + kMergeML + 16;
  static constexpr int kQLd = HD + 8;                     // padded bf16 Q row (conflict-free)
  // unit record: ints [0] M [1] vb [2] nv [3] pbase [4] kvh, [8..40) row_t per vector,
  // [40..72) page len, [72..104) own base; then Q as a hi/lo bf16 pair (hi = bf16(q),
  // lo = bf16(q - hi), pre-scaled): [2][32][kQLd]
  static constexpr int kUnitInts = 128;
  static constexpr int kUnit = kUnitInts * 4 + 2 * 32 * kQLd * 2;
  static constexpr int kTotal = kDvSlots * kSlot + kMerge + kDvUnits * kUnit + 1024;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float dv_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// shared address of (key, 16-byte dim chunk c) in a page's K or V area (SW128 halves)
__device__ __forceinline__ uint32_t dv_addr(uint32_t base, int key, int c) {
  return base + (c >> 3) * (64 * 128) + key * 128 + ((((c & 7) ^ (key & 7))) << 4);
}

template <int HD>
__device__ __forceinline__ void dv_merge_unit(const DvParams& p, const float* merge, int mt,
                                              int lane, int G);

template <int HD>
__global__ void __launch_bounds__(kDvThreads, 1)
    decode_attn_v2(DvParams p, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV) {
  using namespace sm100;
  using C = DvCfg<HD>;
  constexpr int KS = HD / 16;  // k-steps of QK^T
  constexpr int NT = HD / 8;   // n-tiles of O
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* merge = reinterpret_cast<float*>(base + kDvSlots * C::kSlot);
  uint8_t* units = base + kDvSlots * C::kSlot + C::kMerge;  // [kDvUnits][kUnit]
  __shared__ uint64_t full_bar[kDvSlots], empty_bar[kDvSlots];
  __shared__ uint64_t unit_full[kDvUnits], unit_empty[kDvUnits], merge_full, merge_empty;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = p.n_heads / p.n_kv;
  if (tid == 0) {
    for (int i = 0; i < kDvSlots; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], kDvConsumers);
    }
    for (int i = 0; i < kDvUnits; ++i) {
      mbar_init(&unit_full[i], 32);
      mbar_init(&unit_empty[i], kDvConsumers * 32);  // every consumer lane (own reads)
    }
    // merge scratch hand-offs are arrived on by every lane that wrote / read it (each
    // lane's own accesses are then ordered by its own arrive -- no reliance on __syncwarp)
    mbar_init(&merge_full, kDvConsumers * 32);
    mbar_init(&merge_empty, 2 * 32);
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  __syncthreads();
  if (tid == 0) DTR(0);
  // step data (K3's counts and items) only after the programmatic-dependency wait (with
  // every kernel triggering its dependents at its start, a chain of launches can be
  // resident long before this step's K3 finished) -- unless K3 has stamped this step's tag:
  // its outputs are then complete, and the loader / producer look up their first unit while
  // the predecessor (RoPE) still runs, waiting only before they touch its outputs (Q, the
  // appended K/V)
  bool early = false;
  int n_items = 0;
  if (p.k3_tag != 0 && (warp == kDvLoader || warp == kDvProducer)) {
    uint64_t v = 0;  // {tag, n_items}, K3's 64-bit release store
    if (lane == 0)
      asm volatile("ld.acquire.gpu.global.b64 %0, [%1];\n" : "=l"(v) : "l"(p.counts + 4) : "memory");
    early = __shfl_sync(0xffffffffu, (int)(uint32_t)v, 0) == p.k3_tag;
    n_items = __shfl_sync(0xffffffffu, (int)(v >> 32), 0);
  }
  if (!early) {
    pdl_wait();
    n_items = p.counts[1];
  }
  if (tid == 0) DTR(1);
  const int n_work = n_items * p.n_kv;
  const bool snake = p.order != nullptr && n_work > (int)gridDim.x;

  if (warp == kDvLoader) {
    // ------------------------------------------------------------------ unit loader
    // stages each unit's metadata and its Q vectors (bf16, pre-scaled to the log2 domain)
    // one unit ahead of the consumers, so a unit boundary costs no dependent global loads
    int ord = 0;
    for (int u = 0;; ++u) {
      const int w = dv_unit(u, n_work, snake);
      if (w < 0) break;
      if ((u & 31) == 0) ord = dv_items32(p, u, lane, n_work, snake);
      const int item = __shfl_sync(0xffffffffu, ord, u & 31);
      const int sl = u % kDvUnits;
      mbar_wait(&unit_empty[sl], ((u / kDvUnits) & 1) ^ 1);
      if (lane == 0 && u == 0) DTR(14);
      int* ui = reinterpret_cast<int*>(units + sl * C::kUnit);
      __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(units + sl * C::kUnit + C::kUnitInts * 4);
      const int kvh = w % p.n_kv;
      const int32_t* it = p.items + 6 * item;
      const int iv = lane < 5 ? it[lane] : 0;
      int rid, rt;
      if (p.fat) {
        // K3's self-contained item record supplies the rows and their row_t in the same
        // round trip as the item ([4..20) rid, [20..36) row_t)
        const int32_t* fr = p.fat + (int64_t)item * 64;
        const int f0 = fr[lane], f1 = fr[32 + lane];
        const int rr = min(lane / G, 15);
        rid = __shfl_sync(0xffffffffu, f0, 4 + rr);
        const int t0 = __shfl_sync(0xffffffffu, f0, min(20 + rr, 31));
        const int t1 = __shfl_sync(0xffffffffu, f1, max(rr - 12, 0));
        rt = rr < 12 ? t0 : t1;
      }
      const int rb = __shfl_sync(0xffffffffu, iv, 0), nr = __shfl_sync(0xffffffffu, iv, 1);
      if (lane == 0 && u == 0) DTR(12);
      const int vb = __shfl_sync(0xffffffffu, iv, 2), nv = __shfl_sync(0xffffffffu, iv, 3);
      const int pbase = __shfl_sync(0xffffffffu, iv, 4);
      if (!p.fat) {
        rid = lane < nr * G ? p.blk_rows[rb + lane / G] : 0;
        rt = lane < nr * G ? p.row_t[rid] : -1;
      }
      const int M = nr * G;
      if (lane == 0) {
        ui[0] = M;
        ui[1] = vb;
        ui[2] = nv;
        ui[3] = pbase;
        ui[4] = kvh;
      }
      // page lengths / own bases: loads issued here, stored after the Q copies are in flight
      const int vl = lane < nv ? p.vis_len[vb + lane] : 0;
      const int vo = lane < nv ? p.vis_own[vb + lane] : -1;
      if (early && u == 0) pdl_wait();  // Q is the predecessor's output
      if (p.q_k5) {
        // lane m < M: two 256-byte bulk copies (hi, lo) of its vector; lanes >= M zero theirs.
        // The byte count is posted without an arrival: every lane arrives after its stores.
        if (lane == 0) mbar_expect_tx(&unit_full[sl], (uint32_t)M * 2 * HD * 2);
        __syncwarp();
        if (lane < M) {
          const __nv_bfloat16* src = p.q_k5 + ((int64_t)rid * p.n_heads + kvh * G + lane % G) * 2 * HD;
          bulk_g2s(qs + lane * C::kQLd, src, HD * 2, &unit_full[sl]);
          bulk_g2s(qs + (32 + lane) * C::kQLd, src + HD, HD * 2, &unit_full[sl]);
        } else {
#pragma unroll
          for (int d = 0; d < HD; d += 8) {
            *reinterpret_cast<uint4*>(qs + lane * C::kQLd + d) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(qs + (32 + lane) * C::kQLd + d) = make_uint4(0, 0, 0, 0);
          }
        }
        ui[8 + lane] = lane < M ? rt : -1;
        ui[40 + lane] = vl;
        ui[72 + lane] = vo;
        mbar_arrive(&unit_full[sl]);
        if (lane == 0 && u == 0) DTR(3);
        continue;
      }
      ui[8 + lane] = lane < M ? rt : -1;
      ui[40 + lane] = vl;
      ui[72 + lane] = vo;
      // Q: lane = 4 dims of every vector; all loads in flight at once (one round trip),
      // then scaled to the log2 domain and stored as bf16 (rows past M are zero)
      const float sc = p.scale_log2;
      float4 v[32];
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const int r = __shfl_sync(0xffffffffu, rid, m);
        v[m] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < M && 4 * lane < HD)
          v[m] = *reinterpret_cast<const float4*>(p.q + ((int64_t)r * p.n_heads + kvh * G + m % G) * HD + 4 * lane);
      }
#ifdef CHOREO_TRACE
      if (u == 0) {  // consume the loads before the stamp
        float sacc = 0.f;
        for (int m = 0; m < 32; ++m) sacc += v[m].x;
        if (lane == 0) {
          if (sacc == 1234.5f) ui[0] = 0;
          DTR(13);
        }
      }
#endif
      if (4 * lane < HD) {
#pragma unroll
        for (int m = 0; m < 32; ++m) {
          const float a0 = v[m].x * sc, a1 = v[m].y * sc, a2 = v[m].z * sc, a3 = v[m].w * sc;
          const __nv_bfloat162 h01 = __floats2bfloat162_rn(a0, a1), h23 = __floats2bfloat162_rn(a2, a3);
          const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
          *reinterpret_cast<uint2*>(qs + m * C::kQLd + 4 * lane) =
              make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
          *reinterpret_cast<uint2*>(qs + (32 + m) * C::kQLd + 4 * lane) =
              make_uint2(pack_bf16(a0 - f01.x, a1 - f01.y), pack_bf16(a2 - f23.x, a3 - f23.y));
        }
      }
      mbar_arrive(&unit_full[sl]);
      if (lane == 0 && u == 0) DTR(3);
    }
    return;
  }
  if (warp >= kDvMerge) {
    // ------------------------------------------------------------------ merge warps
    const int mt = warp - kDvMerge;
    for (int u = 0; dv_unit(u, n_work, snake) >= 0; ++u) {
      mbar_wait(&merge_full, u & 1);
      dv_merge_unit<HD>(p, merge, mt, lane, G);
      mbar_arrive(&merge_empty);
      if (mt == 0 && lane == 0 && u == 0) DTR(8);
    }
    if (mt == 0 && lane == 0) DTR(9);
    return;
  }
  if (warp == kDvProducer) {
    // ------------------------------------------------------------------ TMA producer
    // the whole warp fetches a unit's record and up to 32 page ids in one round trip each
    // (a per-page dependent load would cap the ring at one page per L2 round trip); lane 0
    // issues the TMA copies
    uint32_t gp = 0;
    const uint64_t pol = l2_policy_evict_first();  // K/V pages: read once per step and layer
    int ord = 0;
    for (int u = 0;; ++u) {
      const int w = dv_unit(u, n_work, snake);
      if (w < 0) break;
      if ((u & 31) == 0) ord = dv_items32(p, u, lane, n_work, snake);
      const int32_t* it = p.items + 6 * __shfl_sync(0xffffffffu, ord, u & 31);
      const int iv = lane < 4 ? it[lane] : 0;
      const int vb = __shfl_sync(0xffffffffu, iv, 2), nv = __shfl_sync(0xffffffffu, iv, 3);
      const int kvh = w % p.n_kv;
      if (early && u == 0) pdl_wait();  // the pages hold the predecessor's K/V appends
      for (int j0 = 0; j0 < nv; j0 += 32) {
        const int pid = j0 + lane < nv ? p.vis_page[vb + j0 + lane] : 0;
        const int nj = min(32, nv - j0);
        for (int jj = 0; jj < nj; ++jj, ++gp) {
          const int page = __shfl_sync(0xffffffffu, pid, jj);
          if (lane == 0) {
            const int st = gp % kDvSlots;
            mbar_wait(&empty_bar[st], ((gp / kDvSlots) & 1) ^ 1);
            if (gp == 0) DTR(2);
            const int row0 = ((p.layer * p.n_kv + kvh) * p.n_pages + page) * 64;
            uint8_t* dst = base + st * C::kSlot;
            mbar_arrive_expect_tx(&full_bar[st], C::kSlot);
#pragma unroll
            for (int r = 0; r < C::kR; ++r) {
              tma_load_2d_hint(dst + r * C::kHalf, &tmK, &full_bar[st], r * 64, row0, pol);
              tma_load_2d_hint(dst + (C::kR + r) * C::kHalf, &tmV, &full_bar[st], r * 64, row0,
                               pol);
            }
          }
          __syncwarp();
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int q4 = warp >> 1, mt = warp & 1;  // key slice, m-tile
  const int g = lane >> 2, t = lane & 3;
  const int k0 = 16 * q4;                   // first key of this warp's slice
  uint32_t gp = 0;
  for (int u = 0; dv_unit(u, n_work, snake) >= 0; ++u) {
    const int sl = u % kDvUnits;
    mbar_wait(&unit_full[sl], (u / kDvUnits) & 1);
    if (warp == 0 && lane == 0 && u == 0) DTR(4);
    const int* ui = reinterpret_cast<const int*>(units + sl * C::kUnit);
    const __nv_bfloat16* qs = reinterpret_cast<const __nv_bfloat16*>(units + sl * C::kUnit + C::kUnitInts * 4);
    const int M = ui[0], nv = ui[2], pbase = ui[3], kvh = ui[4];
    const bool active = mt * 16 < M;  // warp-uniform: this m-tile has query vectors
    const int mA = mt * 16 + g, mB = mA + 8;
    const bool vA = mA < M, vB = mB < M;
    const int rtA = ui[8 + mA], rtB = ui[8 + mB];
    // Q as bf16 A fragments (pre-scaled to the log2 domain; rows past M are zero); the
    // lo halves stay in shared memory (qlo) and are read per page
    const __nv_bfloat16* qlo = qs + 32 * C::kQLd;
    // ldmatrix row address of this lane for the m16 x k16 A fragments of Q lo
    // (matrices: rows 0-7 / 8-15 x k 0-7 / 8-15; 272-byte rows are conflict-free)
    const uint32_t qlo_lane = smem_addr(qlo + (mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * C::kQLd +
                                        (lane >> 4) * 8);
    uint32_t qa[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int c = 16 * ks + 2 * t;
      qa[ks][0] = *reinterpret_cast<const uint32_t*>(qs + mA * C::kQLd + c);
      qa[ks][1] = *reinterpret_cast<const uint32_t*>(qs + mB * C::kQLd + c);
      qa[ks][2] = *reinterpret_cast<const uint32_t*>(qs + mA * C::kQLd + c + 8);
      qa[ks][3] = *reinterpret_cast<const uint32_t*>(qs + mB * C::kQLd + c + 8);
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float mxA = -INFINITY, mxB = -INFINITY, lA = 0.f, lB = 0.f;

    for (int j = 0; j < nv; ++j, ++gp) {
      const int st = gp % kDvSlots;
      mbar_wait(&full_bar[st], (gp / kDvSlots) & 1);
      if (warp == 0 && lane == 0 && u == 0 && j == 0) DTR(5);
      if (active) {
        const uint32_t kb = smem_addr(base + st * C::kSlot);
        const uint32_t vbase = kb + C::kR * C::kHalf;
        // ---- S = Q K^T over this warp's 16 keys (two n8 tiles, two chains each) ----
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        float s0b[4] = {0.f, 0.f, 0.f, 0.f}, s1b[4] = {0.f, 0.f, 0.f, 0.f};
        const int lk = k0 + ((lane >> 4) & 1) * 8 + (lane & 7);
        // hi and lo halves of Q on separate accumulator chains (the lo fragments come from
        // shared memory each page, so Q costs no extra registers)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t r0, r1, r2, r3, ql[4];
          ldsm_x4(dv_addr(kb, lk, 2 * ks + ((lane >> 3) & 1)), r0, r1, r2, r3);
          ldsm_x4(qlo_lane + 32 * ks, ql[0], ql[1], ql[2], ql[3]);  // A fragment of Q lo
          mma_bf16(s0, qa[ks], r0, r1);
          mma_bf16(s1, qa[ks], r2, r3);
          mma_bf16(s0b, ql, r0, r1);
          mma_bf16(s1b, ql, r2, r3);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          s0[e] += s0b[e];
          s1[e] += s1b[e];
        }
        // ---- mask (page length, causal cut of own pages) ----
        const int len = ui[40 + j], own = ui[72 + j];
        int limA = len, limB = len;
        if (own >= 0) {
          limA = min(limA, rtA - own + 1);
          limB = min(limB, rtB - own + 1);
        }
        if (!__all_sync(0xffffffffu, limA >= k0 + 16 && limB >= k0 + 16)) {
          const int ka = k0 + 2 * t;
          s0[0] = ka < limA ? s0[0] : -INFINITY;
          s0[1] = ka + 1 < limA ? s0[1] : -INFINITY;
          s0[2] = ka < limB ? s0[2] : -INFINITY;
          s0[3] = ka + 1 < limB ? s0[3] : -INFINITY;
          s1[0] = ka + 8 < limA ? s1[0] : -INFINITY;
          s1[1] = ka + 9 < limA ? s1[1] : -INFINITY;
          s1[2] = ka + 8 < limB ? s1[2] : -INFINITY;
          s1[3] = ka + 9 < limB ? s1[3] : -INFINITY;
        }
        // ---- online softmax (log2 domain, lazy rescale) ----
        float tA = fmaxf(fmaxf(s0[0], s0[1]), fmaxf(s1[0], s1[1]));
        float tB = fmaxf(fmaxf(s0[2], s0[3]), fmaxf(s1[2], s1[3]));
        tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, 1));
        tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, 2));
        tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, 1));
        tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, 2));
        float aA = 1.f, aB = 1.f;
        if (tA > mxA + 8.f || (mxA == -INFINITY && tA != -INFINITY)) {
          aA = mxA == -INFINITY ? 0.f : dv_ex2(mxA - tA);
          mxA = tA;
        }
        if (tB > mxB + 8.f || (mxB == -INFINITY && tB != -INFINITY)) {
          aB = mxB == -INFINITY ? 0.f : dv_ex2(mxB - tB);
          mxB = tB;
        }
        if (__any_sync(0xffffffffu, aA != 1.f || aB != 1.f)) {
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            o[n][0] *= aA;
            o[n][1] *= aA;
            o[n][2] *= aB;
            o[n][3] *= aB;
          }
          lA *= aA;
          lB *= aB;
        }
        const float nA = mxA == -INFINITY ? 0.f : mxA, nB = mxB == -INFINITY ? 0.f : mxB;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          s0[e] = dv_ex2(s0[e] - nA);
          s1[e] = dv_ex2(s1[e] - nA);
          s0[2 + e] = dv_ex2(s0[2 + e] - nB);
          s1[2 + e] = dv_ex2(s1[2 + e] - nB);
        }
        lA += (s0[0] + s0[1]) + (s1[0] + s1[1]);
        lB += (s0[2] + s0[3]) + (s1[2] + s1[3]);
        uint32_t pa[4] = {pack_bf16(s0[0], s0[1]), pack_bf16(s0[2], s0[3]),
                          pack_bf16(s1[0], s1[1]), pack_bf16(s1[2], s1[3])};
        // ---- O += P V over the same 16 keys ----
        const int lv = k0 + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          uint32_t r0, r1, r2, r3;
          ldsm_x4_t(dv_addr(vbase, lv, 2 * dp + (lane >> 4)), r0, r1, r2, r3);
          mma_bf16(o[2 * dp], pa, r0, r1);
          mma_bf16(o[2 * dp + 1], pa, r2, r3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[st]);
    }

    mbar_arrive(&unit_empty[sl]);
    if (warp == 0 && lane == 0 && u == 0) DTR(6);
    // ---- hand the key-slice state to the merge warps ----
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    lB += __shfl_xor_sync(0xffffffffu, lB, 1);
    lB += __shfl_xor_sync(0xffffffffu, lB, 2);
    if (u > 0) mbar_wait(&merge_empty, (u - 1) & 1);  // the merge warps read unit u-1
    if (active) {
      __half* so = reinterpret_cast<__half*>(merge) + (q4 * 2 + mt) * 16 * C::kMergeRow;
      float2* ml = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(merge) + C::kMergeO) +
                   (q4 * 2 + mt) * 16;
      const float iA = lA > 0.f ? 1.f / lA : 0.f, iB = lB > 0.f ? 1.f / lB : 0.f;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        *reinterpret_cast<__half2*>(so + g * C::kMergeRow + 8 * n + 2 * t) =
            __floats2half2_rn(o[n][0] * iA, o[n][1] * iA);
        *reinterpret_cast<__half2*>(so + (g + 8) * C::kMergeRow + 8 * n + 2 * t) =
            __floats2half2_rn(o[n][2] * iB, o[n][3] * iB);
      }
      if (t == 0) {
        ml[g] = make_float2(mxA, lA);
        ml[g + 8] = make_float2(mxB, lB);
      }
    }
    if (warp == 0 && lane == 0) {
      int* hdr = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(merge) + C::kMergeO + C::kMergeML);
      hdr[0] = M;
      hdr[1] = pbase;
      hdr[2] = kvh;
    }
    mbar_arrive(&merge_full);
    if (warp == 0 && lane == 0 && u == 0) DTR(7);
  }
  if (warp == 0 && lane == 0) DTR(11);
}

// Merge warp of m-tile mt: lane = (row, 64-dim half); combines the four key slices' (O, m,
// l) of each of the tile's 16 rows (LSE rule) and writes the normalised partial + LSE.
template <int HD>
__device__ __forceinline__ void dv_merge_unit(const DvParams& p, const float* merge, int mt,
                                              int lane, int G) {
  using C = DvCfg<HD>;
  constexpr int W = HD / 2;  // dims per lane
  const uint8_t* mb = reinterpret_cast<const uint8_t*>(merge);
  const int* hdr = reinterpret_cast<const int*>(mb + C::kMergeO + C::kMergeML);
  const int M = hdr[0], pbase = hdr[1], kvh = hdr[2];
  const int row = lane >> 1, half = lane & 1;
  const int m = mt * 16 + row;
  if (m >= M) return;
  const float2* ml = reinterpret_cast<const float2*>(mb + C::kMergeO);
  float mk[4], lk[4], mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 v = ml[(k * 2 + mt) * 16 + row];
    mk[k] = v.x;
    lk[k] = v.y;
    mx = fmaxf(mx, mk[k]);
  }
  float wk[4], L = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    wk[k] = (mk[k] == -INFINITY || lk[k] <= 0.f) ? 0.f : lk[k] * dv_ex2(mk[k] - mx);
    L += wk[k];
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) wk[k] *= inv;
  const int64_t pidx = (int64_t)(pbase + m / G) * p.n_heads + kvh * G + m % G;
  float* dst = p.part_o + pidx * HD + half * W;
  const __half* so = reinterpret_cast<const __half*>(merge) + row * C::kMergeRow + half * W;
#pragma unroll 2
  for (int d = 0; d < W; d += 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 x = *reinterpret_cast<const uint4*>(so + (k * 2 + mt) * 16 * C::kMergeRow + d);
      const __half2* h = reinterpret_cast<const __half2*>(&x);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h[e]);
        acc[2 * e] += wk[k] * f.x;
        acc[2 * e + 1] += wk[k] * f.y;
      }
    }
    *reinterpret_cast<float4*>(dst + d) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(dst + d + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  if (half == 0) p.part_lse[pidx] = L > 0.f ? (mx + log2f(L)) * 0.6931471805599453f : -INFINITY;
}

// ---------------------------------------------------------------- host side
static bool dv_pool_map(CUtensorMap* map, const void* pool, uint64_t rows, int hd) {
  return tmap_bf16_2d(map, pool, rows, (uint64_t)hd, 64, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

template <int HD>
static int launch_dv(const DvParams& p, const void* k_pool, const void* v_pool, uint64_t rows,
                     int grid, cudaStream_t s) {
  CUtensorMap mk, mv;
  if (!dv_pool_map(&mk, k_pool, rows, HD) || !dv_pool_map(&mv, v_pool, rows, HD))
    return CHOREO_ELAUNCH;
  constexpr int smem = DvCfg<HD>::kTotal;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(decode_attn_v2<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = true;
  }
  launch_k(decode_attn_v2<HD>, grid, kDvThreads, smem, s, p, mk, mv);
  return launch_status("choreo_decode_attn_v2");
}

}  // namespace choreo

using namespace choreo;

#ifdef CHOREO_TRACE
extern "C" int choreo_dv_set_trace(long long* buf) {
  g_dv_launches = 0;
  return cudaMemcpyToSymbol(g_dv_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -2;
}
#endif

extern "C" int choreo_decode_attn_v2_ex(const float* q, const void* k_pool, const void* v_pool,
                                        int n_layers, int layer, int n_kv, int n_pages,
                                        int page_size, int n_heads, int head_dim,
                                        const int32_t* row_t, const int32_t* vis_page,
                                        const int32_t* vis_len, const int32_t* vis_own,
                                        const int32_t* blk_rows, const int32_t* items,
                                        const int32_t* counts, int max_items, float* part_o,
                                        float* part_lse, const int32_t* fat_items, int grid_ctas,
                                        const void* q_k5, const int32_t* item_order,
                                        int k3_tag, void* stream);

extern "C" int choreo_decode_attn_v2(const float* q, const void* k_pool, const void* v_pool,
                                     int n_layers, int layer, int n_kv, int n_pages, int page_size,
                                     int n_heads, int head_dim, const int32_t* row_t,
                                     const int32_t* vis_page, const int32_t* vis_len,
                                     const int32_t* vis_own, const int32_t* blk_rows,
                                     const int32_t* items, const int32_t* counts, int max_items,
                                     float* part_o, float* part_lse, const int32_t* fat_items,
                                     int grid_ctas, void* stream) {
  return choreo_decode_attn_v2_ex(q, k_pool, v_pool, n_layers, layer, n_kv, n_pages, page_size,
                                  n_heads, head_dim, row_t, vis_page, vis_len, vis_own, blk_rows,
                                  items, counts, max_items, part_o, part_lse, fat_items,
                                  grid_ctas, nullptr, nullptr, 0, stream);
}

extern "C" int choreo_decode_attn_v2_ex(const float* q, const void* k_pool, const void* v_pool,
                                        int n_layers, int layer, int n_kv, int n_pages,
                                        int page_size, int n_heads, int head_dim,
                                        const int32_t* row_t, const int32_t* vis_page,
                                        const int32_t* vis_len, const int32_t* vis_own,
                                        const int32_t* blk_rows, const int32_t* items,
                                        const int32_t* counts, int max_items, float* part_o,
                                        float* part_lse, const int32_t* fat_items, int grid_ctas,
                                        const void* q_k5, const int32_t* item_order,
                                        int k3_tag, void* stream) {
  if (!q || !k_pool || !v_pool || !row_t || !vis_page || !vis_len || !vis_own || !blk_rows ||
      !items || !counts || !part_o || !part_lse || n_kv <= 0 || n_heads % n_kv)
    return CHOREO_EINVAL;
  if (page_size != 64 || (head_dim != 64 && head_dim != 128) || n_heads / n_kv > 32)
    return CHOREO_EUNSUPPORTED;  // items must also hold <= 32 / G rows and <= 32 pages
  if (max_items <= 0) return CHOREO_OK;
  const uint64_t rows = (uint64_t)n_layers * n_kv * n_pages * page_size;
  if (rows > 0x7fffffffull) return CHOREO_EUNSUPPORTED;
  const int G = n_heads / n_kv;
  DvParams p{q, layer, n_kv, n_pages, n_heads, row_t, vis_page, vis_len, vis_own, blk_rows, items,
             counts, part_o, part_lse, 1.4426950408889634f / sqrtf((float)head_dim),
             32 / G <= 16 ? fat_items : nullptr, 0, reinterpret_cast<const __nv_bfloat16*>(q_k5),
             item_order, k3_tag};
#ifdef CHOREO_TRACE
  p.trace_slot = g_dv_launches++;
#endif
  int grid = grid_ctas > 0 ? grid_ctas : max_items * n_kv;
  if (grid > 148) grid = 148;
  auto s = as_stream(stream);
  return head_dim == 128 ? launch_dv<128>(p, k_pool, v_pool, rows, grid, s)
                         : launch_dv<64>(p, k_pool, v_pool, rows, grid, s);
}
