// K8 layer chain: the four weight-streaming projections between two attentions of a
// decode-sized step -- o_proj(l), gate|up(l), down(l), qkv(l+1) -- in ONE persistent
// launch, with the elementwise work of reference model.py:169-189 folded into the GEMM
// epilogues and the phase boundaries turned into completion counters polled on the device.
//
// Why: a decode step streams 16 GB of weights through ~290 small launches; each K7 launch
// pays a fill / drain (first TMA bytes, stream-K fix-up, last tile) of several
// microseconds and every residual/RMSNorm/RoPE kernel between them is a dependent link of
// the chain.  Here one CTA per SM streams the weights of all four GEMMs back to back: the
// weight TMA warp never waits on activations, so the next GEMM's weights are already in
// the ring when the previous GEMM's outputs land.
//
// Roles (224 threads): warp 0 weight TMA, warp 1 tcgen05 MMA issuer, warp 2 activation TMA,
// warps 3-6 epilogue (one TMEM lane quadrant each).  Every phase is a stream-K split of
// its (tile, k-block) space over the CTAs (K7's scheme: swap-AB, 128 weight rows x NX
// activation rows per UMMA, hi/lo activation halves summed in the epilogue; a tile cut
// between CTAs is reduced by its last piece in CTA order, deterministically).
//
// Folded epilogues (reference model.py:169-189, per layer):
//   o_proj : x += attn @ Wo^T ; h_a = hi/lo(x * ffn_norm) ; ssq_a[tile][row] = sum x^2
//   gate|up: act = silu(r * g) * (r * u),  r = rsqrt(mean x^2 + eps) from ssq_a
//   down   : x += act @ Wd^T ; h_b = hi/lo(x * attn_norm(l+1)) ; ssq_b
//   qkv    : (r * (h_b @ Wqkv^T)) -> RoPE(q, k) at the row's position, q (f32) out, k / v
//            appended to the row's pool slot (reference cache.py:98-135)
// RMSNorm is applied as a per-row scale of the NEXT GEMM's output: norm(x) * w @ W^T =
// r * ((x * w) @ W^T), exact in real arithmetic; the GEMM input x * w is carried as a
// hi/lo bf16 pair like every K7 activation.
//
// Dataflow: when a tile's final values are stored, the epilogue adds 1 to done[phase]
// (release).  Before loading a phase's inputs the activation TMA warp acquires
// done[producer] == its tile count (generic -> async proxy fence in between); epilogues
// that need the norm scale or the residual do the same.  Each wait is ONE thread polling
// ONE word with a back-off: per-tile flags polled warp-wide from every SM turned the flag
// lines into an L2 hot spot that slowed the weight stream itself.  The last CTA to exit
// zeroes the counters for the next launch (which reads them only after its
// griddepcontrol.wait).  All waits point to earlier phases, every CTA runs its phases in
// order and the grid is <= one CTA per SM with all CTAs co-resident, so the chain cannot
// deadlock.
#include <cudaTypedefs.h>
#include <math.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace choreo {

constexpr int kChThreads = 224;
constexpr int kChTile = 128;
constexpr int kChKB = 64;
constexpr int kChMaxTiles = 1024;  // per phase (stream-K counters rows)
constexpr int kChSsq = 128;        // row stride of the ssq arrays ([tiles][128])
enum { kPhO = 0, kPhGU = 1, kPhD = 2, kPhQKV = 3, kChPhases = 4 };

struct ChPhase {
  int on;
  int N;        // output columns (gate|up: act columns F)
  int K;        // reduction length
  int n_tiles, KB, iters;
  int x_dep;    // phase whose tiles produce this phase's X (-1: an earlier launch)
  int x_dep_w;  // output columns per tile of that phase
  int x_rows;   // rows of the X buffer (2R when split)
  int ssq_dep;  // phase whose completion guards ssq_in (-1: earlier launch; -2: no scale)
  int ssq_tiles;
  const float* ssq_in;
  float* ssq_out;       // RESID phases: [n_tiles][kChSsq]
  const void* gamma;    // RESID phases: next norm weight (bf16) or null
  void* out;            // RESID: h (bf16 hi/lo [2R][d]); GU: act (bf16 hi/lo [2R][F])
  int x_prev_dep;       // RESID: phase that last wrote x in this launch (-1: none)
};

struct ChParams {
  ChPhase ph[kChPhases];
  float* x;
  int d, R, split, rpad;
  float eps;
  float* q;
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  int layer, n_kv, n_heads, hd, n_pages, page_size;
  const int32_t* pos;
  const int32_t* page;
  const int32_t* slot;
  const float* cos_t;
  const float* sin_t;
  int max_delta;
  float* ws;
  int* counters;
  int* done;  // [kChPhases] tiles completed per phase, [kChPhases] CTAs exited
  int grid, stages;
  int trace_slot;  // diagnostics builds: which launch's trace rows this launch writes
};

struct ChMaps {
  CUtensorMap w[kChPhases];
  CUtensorMap x[kChPhases];
};

template <int NX, int KSUB>
struct ChCfg {
  static constexpr int kWBytes = kChTile * 128;
  static constexpr int kXBytes = NX * 128;
  static constexpr int kStageBytes = KSUB * (kWBytes + kXBytes);
  // ring depth: 196 KB (measured: a sixth stage at NX 16 -- 222 KB -- made the chain and K7
  // slower, not faster)
  static constexpr int kBudget = 196 * 1024;
  static constexpr int kStages = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
  static constexpr int kTmemCols = 2 * NX < 32 ? 32 : 2 * NX;
  static constexpr int smem() { return kStages * kStageBytes + 1024; }
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// One thread: wait until *cnt >= target (acquire), polling with a back-off.
__device__ __forceinline__ void wait_count(const int* cnt, int target) {
  while (ld_acquire(cnt) < target) __nanosleep(32);
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Diagnostics build only (-DCHOREO_TRACE, tools/chain_trace.sh): per-CTA globaltimer stamps.
#ifdef CHOREO_TRACE
__device__ long long* g_chain_trace = nullptr;
__device__ __forceinline__ void chain_trace(int slot, int i) {
  if (g_chain_trace) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_chain_trace[((size_t)(slot & 63) * 148 + blockIdx.x) * 48 + i] = t;
  }
}
static int g_trace_launches = 0;
#define TR(i) chain_trace(p.trace_slot, i)
#else
#define TR(i) \
  do {        \
  } while (0)
#endif

template <int NX, int KSUB>
__global__ void __launch_bounds__(kChThreads, 1)
    chain_sm100(const ChParams p, const __grid_constant__ ChMaps maps) {
  using namespace sm100;
  using C = ChCfg<NX, KSUB>;
  // activation rows per epilogue chunk: 8 at NX 16 (<= 8 rows split, 16 plain), else 16
  constexpr int RC = NX == 16 ? 8 : 16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t full_w[C::kStages], full_x[C::kStages], empty_bar[C::kStages];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ int s_last;
  __shared__ float s_xch[16 * 64];  // gate|up: up values of 16 rows x 64 columns
  __shared__ float s_red[4][16];    // per-quadrant partial sums of squares
  __shared__ float s_r[128];        // per-row RMSNorm scale of the current phase
  __shared__ int s_pos[128];         // qkv: position per row
  __shared__ long long s_koff[128];  // qkv: pool offset of (layer, kv head 0, page, slot, 0)

  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x;
  const int NS = p.stages;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full_w[i], 1);
      mbar_init(&full_x[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
    for (int ph = 0; ph < kChPhases; ++ph)
      if (p.ph[ph].on) {
        tma_prefetch_desc(&maps.w[ph]);
        tma_prefetch_desc(&maps.x[ph]);
      }
  }
  if (warp == 1) tmem_alloc(&tmem_base, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) TR(0);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------- weight TMA producer
      // weights are read exactly once per step: evict-first, so the stream does not push the
      // activations, partial tiles and this kernel's own code out of L2
      const uint64_t pol = l2_policy_evict_first();
      int pb[kChPhases], pe[kChPhases];
#pragma unroll
      for (int ph = 0; ph < kChPhases; ++ph) {
        pb[ph] = p.ph[ph].on ? ln_begin(c, p.ph[ph].iters, p.grid) : 0;
        pe[ph] = p.ph[ph].on ? ln_begin(c + 1, p.ph[ph].iters, p.grid) : 0;
      }
      int j = 0;
#pragma unroll
      for (int ph = 0; ph < kChPhases; ++ph) {
        const ChPhase& P = p.ph[ph];
        if (!P.on) continue;
        const int b = pb[ph], e = pe[ph];
        for (int i = b; i < e; ++i, ++j) {
          const int st = j % NS;
          if (j >= NS) mbar_wait(&empty_bar[st], ((j / NS) & 1) ^ 1);
          if (i == b) TR(1 + ph * 6);
          mbar_arrive_expect_tx(&full_w[st], KSUB * C::kWBytes);
          uint8_t* dst = base + st * C::kStageBytes;
          const int t = i / P.KB, kb = (i % P.KB) * KSUB;
#pragma unroll
          for (int u = 0; u < KSUB; ++u) {
            if (ph == kPhGU) {  // 64 gate rows over the matching 64 up rows
              tma_load_2d_hint(dst + u * C::kWBytes, &maps.w[ph], &full_w[st], (kb + u) * kChKB,
                               t * 64, pol);
              tma_load_2d_hint(dst + u * C::kWBytes + 64 * 128, &maps.w[ph], &full_w[st],
                               (kb + u) * kChKB, P.N + t * 64, pol);
            } else {
              tma_load_2d_hint(dst + u * C::kWBytes, &maps.w[ph], &full_w[st], (kb + u) * kChKB,
                               t * kChTile, pol);
            }
          }
        }
      }
    }
  } else if (warp == 2) {  // ------------------------------- activation TMA producer (warp)
    pdl_wait();  // X of the first phase was written by the previous launch
    int j = 0;
#pragma unroll
    for (int ph = 0; ph < kChPhases; ++ph) {
      const ChPhase& P = p.ph[ph];
      if (!P.on) continue;
      const int b = ln_begin(c, P.iters, p.grid), e = ln_begin(c + 1, P.iters, p.grid);
      if (P.x_dep >= 0 && b < e && lane == 0) {
        // every input column is produced by the x_dep phase; its tiles complete together
        wait_count(p.done + P.x_dep, p.ph[P.x_dep].n_tiles);
        fence_proxy_async_global();
      }
      if (lane == 0) TR(2 + ph * 6);
      if (lane == 0) {
        for (int i = b; i < e; ++i, ++j) {
          const int st = j % NS;
          if (j >= NS) mbar_wait(&empty_bar[st], ((j / NS) & 1) ^ 1);
          const int kb = (i % P.KB) * KSUB;
          mbar_arrive_expect_tx(&full_x[st], KSUB * C::kXBytes);
          uint8_t* xd = base + st * C::kStageBytes + KSUB * C::kWBytes;
#pragma unroll
          for (int u = 0; u < KSUB; ++u) {
            if (p.split) {  // hi rows -> B rows [0, NX/2), lo rows -> [NX/2, NX)
              tma_load_2d(xd + u * C::kXBytes, &maps.x[ph], &full_x[st], (kb + u) * kChKB, 0);
              tma_load_2d(xd + u * C::kXBytes + C::kXBytes / 2, &maps.x[ph], &full_x[st],
                          (kb + u) * kChKB, p.R);
            } else {
              tma_load_2d(xd + u * C::kXBytes, &maps.x[ph], &full_x[st], (kb + u) * kChKB, 0);
            }
          }
        }
      }
      j = __shfl_sync(0xffffffffu, j, 0);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(kChTile, NX, false);
      int j = 0, seg = 0;
#pragma unroll
      for (int ph = 0; ph < kChPhases; ++ph) {
        const ChPhase& P = p.ph[ph];
        if (!P.on) continue;
        const int b = ln_begin(c, P.iters, p.grid), e = ln_begin(c + 1, P.iters, p.grid);
        for (int i = b; i < e; ++i, ++j) {
          const int st = j % NS, kb = i % P.KB;
          const bool first = (i == b) || kb == 0;
          const bool last = (i == e - 1) || kb == P.KB - 1;
          const int buf = seg & 1;
          if (first && seg >= 2) mbar_wait(&acc_empty[buf], ((seg >> 1) - 1) & 1);
          mbar_wait(&full_w[st], (j / NS) & 1);
          mbar_wait(&full_x[st], (j / NS) & 1);
          tc_fence_after();
          if (i == b) TR(3 + ph * 6);
          if (i == e - 1) TR(4 + ph * 6);
          const uint32_t waddr = smem_addr(base + st * C::kStageBytes);
          const uint32_t xaddr = waddr + KSUB * C::kWBytes;
          const uint32_t d = tmem_base + buf * NX;
#pragma unroll
          for (int u = 0; u < KSUB; ++u)
#pragma unroll
            for (int k = 0; k < kChKB / 16; ++k)
              umma_bf16(d, umma_desc_sw128(waddr + u * C::kWBytes + k * 32, 16, 1024),
                        umma_desc_sw128(xaddr + u * C::kXBytes + k * 32, 16, 1024), idesc,
                        (first && u == 0 && k == 0) ? 0u : 1u);
          umma_commit(&empty_bar[st]);
          if (last) {
            umma_commit(&acc_full[buf]);
            ++seg;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    pdl_wait();
    const int quad = warp & 3;
    const int nl = quad * 32 + lane;  // weight row within the tile = TMEM lane
    const int et = tid - 96;          // 0..127
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int R = p.R, rpad = p.rpad, d = p.d;
    int seg = 0;
    // not unrolled: the epilogue runs once per tile and its code is cold in the
    // instruction cache at every phase (the weight stream evicts it from L2), so one copy
    // of it is fetched instead of four
#pragma unroll 1
    for (int ph = 0; ph < kChPhases; ++ph) {
      const ChPhase& P = p.ph[ph];
      if (!P.on) continue;
      const int b = ln_begin(c, P.iters, p.grid), e = ln_begin(c + 1, P.iters, p.grid);
      if (P.x_prev_dep >= 0 && b < e) {  // x was last written by that phase of this launch
        if (et == 0) wait_count(p.done + P.x_prev_dep, p.ph[P.x_prev_dep].n_tiles);
        epi_bar();
      }
      if (P.ssq_dep != -2 && b < e) {
        // per-row RMSNorm scale from the producing phase's partial sums of squares, computed
        // once at the phase start (the producing phase is complete before this phase's
        // inputs load, so the wait overlaps the first MMAs)
        if (et == 0 && P.ssq_dep >= 0) wait_count(p.done + P.ssq_dep, P.ssq_tiles);
        epi_bar();
        if (et < R) {
          float acc = 0.f;
          int s0 = 0;
          for (; s0 + 8 <= P.ssq_tiles; s0 += 8) {  // 8 loads in flight, summed in order
            float v8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v8[k] = __ldcg(P.ssq_in + (size_t)(s0 + k) * kChSsq + et);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += v8[k];
          }
          for (; s0 < P.ssq_tiles; ++s0) acc += __ldcg(P.ssq_in + (size_t)s0 * kChSsq + et);
          s_r[et] = 1.0f / sqrtf(acc / (float)d + p.eps);
          if (ph == kPhQKV) {
            s_pos[et] = __ldg(p.pos + et);
            s_koff[et] = pool_off(p.layer, 0, __ldg(p.page + et), __ldg(p.slot + et), p.n_kv,
                                  p.n_pages, p.page_size, p.hd);
          }
        }
        epi_bar();
      }
      for (int t = b / P.KB; t * P.KB < e; ++t, ++seg) {
        const int buf = seg & 1;
        const int lo = t * P.KB, hi = lo + P.KB;
        const int c_lo = ln_owner(lo, P.iters, p.grid), c_hi = ln_owner(hi - 1, P.iters, p.grid);
        const bool cut = c_lo != c_hi;
        mbar_wait(&acc_full[buf], (seg >> 1) & 1);
        tc_fence_after();
        const bool last_seg = (t + 1) * P.KB >= e;
        if (et == 0 && last_seg) TR(26 + ph * 4);
        const int n = t * kChTile + nl;
        // single-chunk tiles (decode steps): the final pass's own loads (x rows, rotation
        // table entries) go out now, so their latency hides behind the cut-tile protocol
        const bool pre = rpad <= RC;
        float xpre[RC], cpre[RC], spre[RC];
        if (pre && (ph == kPhO || ph == kPhD)) {
#pragma unroll
          for (int i = 0; i < RC; ++i)
            xpre[i] = (i < R && n < P.N) ? __ldcg(p.x + (size_t)i * d + n) : 0.f;
        }
        if (pre && ph == kPhQKV) {
          const int kk = n % p.hd;
          const bool rot = n / p.hd < p.n_heads + p.n_kv && n < P.N;
#pragma unroll
          for (int i = 0; i < RC; ++i) {
            cpre[i] = spre[i] = 0.f;
            if (rot && i < R) {
              const int64_t ti = (int64_t)(s_pos[i] + p.max_delta) * (p.hd >> 1) + (kk >> 1);
              cpre[i] = __ldg(p.cos_t + ti);
              spre[i] = __ldg(p.sin_t + ti);
            }
          }
        }
        const uint32_t tb = tmem_base + lane_off + buf * NX;
        // rows r0 .. r0+RC-1 of the tile's accumulator (hi + lo halves summed) -> v
        auto tmem_rows = [&](int r0, float* v) {
          float a[16], bb[16];
          if (NX == 16 && p.split) {
            tmem_ld16(tb, a);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < RC; ++i) v[i] = a[i] + a[8 + i];
          } else if (NX == 16) {
            tmem_ld8(tb + r0, a);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < RC; ++i) v[i] = a[i];
          } else if (p.split) {
            tmem_ld16(tb + r0, a);
            tmem_ld16(tb + NX / 2 + r0, bb);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < RC; ++i) v[i] = a[i] + bb[i];
          } else {
            tmem_ld16(tb + r0, a);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < RC; ++i) v[i] = a[i];
          }
        };
        float* const ws_ph = p.ws + (size_t)ph * p.grid * 2 * rpad * kChTile;
        if (cut) {
          // piece of a tile cut between CTAs: park it; the last piece reduces in CTA order
          const int slot = (b >= lo) ? 0 : 1;
          float* w = ws_ph + ((size_t)(c * 2 + slot) * rpad) * kChTile + nl;
          for (int r0 = 0; r0 < rpad; r0 += RC) {
            float v[RC];
            tmem_rows(r0, v);
#pragma unroll
            for (int i = 0; i < RC; ++i)
              if (r0 + i < rpad) w[(r0 + i) * kChTile] = v[i];
          }
          tc_fence_before();
          mbar_arrive(&acc_empty[buf]);
          epi_bar();
          if (et == 0) {
            asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
            int* cnt = p.counters + ph * kChMaxTiles + t;
            const int old = atomicAdd(cnt, 1);
            s_last = old == c_hi - c_lo;
            if (s_last) {
              asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
              *cnt = 0;
            }
          }
          epi_bar();
          if (et == 0 && last_seg) TR(27 + ph * 4);
          if (!s_last) continue;
        }
        // ---------------------------------------------------- final values of tile t
        for (int r0 = 0; r0 < rpad; r0 += RC) {
          float v[RC];
          if (cut) {
#pragma unroll
            for (int i = 0; i < RC; ++i) v[i] = 0.f;
            constexpr int RB = RC;
            for (int c0 = c_lo; c0 <= c_hi; c0 += 4) {
              // the pieces of 4 CTAs loaded together, then added in CTA order
              float pv[4][RB];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const int cc = c0 + jj;
                if (cc <= c_hi) {
                  const int sl = (ln_begin(cc, P.iters, p.grid) >= lo) ? 0 : 1;
                  const float* rp = ws_ph + ((size_t)(cc * 2 + sl) * rpad + r0) * kChTile + nl;
#pragma unroll
                  for (int i = 0; i < RB; ++i) pv[jj][i] = r0 + i < rpad ? __ldcg(rp + i * kChTile) : 0.f;
                }
              }
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
                if (c0 + jj <= c_hi) {
#pragma unroll
                  for (int i = 0; i < RB; ++i) v[i] += pv[jj][i];
                }
            }
          } else {
            tmem_rows(r0, v);
          }
#ifdef CHOREO_TRACE
          if (et == 0 && last_seg && r0 == 0 && (ph == kPhD || ph == kPhQKV)) {
            float sacc = 0.f;
            for (int i = 0; i < RC; ++i) sacc += v[i];  // consume the loads before the stamp
            if (sacc == 12345.678f) s_last = 7;
            TR(ph == kPhD ? 42 : 45);
          }
#endif
          if (ph == kPhO || ph == kPhD) {
            // x += y ; h = hi/lo(x * gamma) ; partial sums of squares per row.  Every load of
            // the chunk is issued before any store (stores could alias the loads for the
            // compiler, which would otherwise serialise one L2 round trip per row)
            float sq[RC], xv[RC];
            const float g = (P.gamma && n < P.N)
                                ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(P.gamma)[n])
                                : 0.f;
            __nv_bfloat16* hout = reinterpret_cast<__nv_bfloat16*>(P.out);
            float* const xcol = p.x + n;
#pragma unroll
            for (int i = 0; i < RC; ++i)
              xv[i] = pre ? xpre[i] : (r0 + i < R && n < P.N) ? __ldcg(xcol + (size_t)(r0 + i) * d) : 0.f;
#pragma unroll
            for (int i = 0; i < RC; ++i) {
              sq[i] = 0.f;
              const int row = r0 + i;
              if (row < R && n < P.N) {
                const float xn = xv[i] + v[i];
                __stcg(xcol + (size_t)row * d, xn);
                sq[i] = xn * xn;
                if (P.gamma) {
                  const float u = xn * g;
                  const __nv_bfloat16 h = __float2bfloat16_rn(u);
                  hout[(size_t)row * d + n] = h;
                  if (p.split) hout[(size_t)(R + row) * d + n] = __float2bfloat16_rn(u - __bfloat162float(h));
                }
              }
            }
            if (et == 0 && last_seg && r0 == 0 && ph == kPhD) TR(43);
            if (P.gamma) {
#pragma unroll
              for (int i = 0; i < RC; ++i) {
                const float s = warp_sum(sq[i]);
                if (lane == 0) s_red[quad][i] = s;
              }
              epi_bar();
              if (et < RC && r0 + et < R)
                P.ssq_out[(size_t)t * kChSsq + r0 + et] =
                    (s_red[0][et] + s_red[1][et]) + (s_red[2][et] + s_red[3][et]);
              epi_bar();
            }
          } else if (ph == kPhGU) {
            // lanes 0-63 hold gate, 64-127 up of the same 64 ffn columns
            if (nl >= 64) {
#pragma unroll
              for (int i = 0; i < RC; ++i)
                s_xch[i * 64 + (nl - 64)] = (r0 + i < R) ? s_r[r0 + i] * v[i] : 0.f;
            }
            epi_bar();
            if (nl < 64) {
              __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(P.out);
              const int jcol = t * 64 + nl;
#pragma unroll
              for (int i = 0; i < RC; ++i) {
                const int row = r0 + i;
                if (row < R) {
                  const float gv = s_r[row] * v[i];
                  const float a = gv / (1.0f + expf(-gv)) * s_xch[i * 64 + nl];
                  const __nv_bfloat16 h = __float2bfloat16_rn(a);
                  act[(size_t)row * P.N + jcol] = h;
                  if (p.split)
                    act[(size_t)(R + row) * P.N + jcol] = __float2bfloat16_rn(a - __bfloat162float(h));
                }
              }
            }
            epi_bar();  // s_xch free for the next chunk
          } else {
            // qkv: scale, RoPE (interleaved pairs, partner in the neighbouring lane), append.
            // Row metadata comes from shared memory (staged at the phase start); the rotation
            // table entries of all rows are loaded before any store.
            const int H = p.n_heads, Hk = p.n_kv, hd = p.hd, half = hd >> 1;
            const int head = n / hd, kk = n - head * hd, odd = kk & 1, pair = kk >> 1;
            const bool rot = head < H + Hk && n < P.N;
            float cs[RC], sn[RC], val[RC], other[RC];
#pragma unroll
            for (int i = 0; i < RC; ++i) {
              const int row = r0 + i;
              cs[i] = sn[i] = 0.f;
              if (pre) {
                cs[i] = cpre[i];
                sn[i] = spre[i];
              } else if (rot && row < R) {
                const int64_t ti = (int64_t)(s_pos[row] + p.max_delta) * half + pair;
                cs[i] = __ldg(p.cos_t + ti);
                sn[i] = __ldg(p.sin_t + ti);
              }
            }
#pragma unroll
            for (int i = 0; i < RC; ++i) {
              val[i] = r0 + i < R ? s_r[r0 + i] * v[i] : 0.f;
              other[i] = __shfl_xor_sync(0xffffffffu, val[i], 1);
            }
            // destination of this lane's column: q (f32) or the K / V pool slot of the row
            const int64_t hs = (int64_t)p.n_pages * p.page_size * hd;  // pool stride per kv head
            const int kind = head < H ? 0 : head < H + Hk ? 1 : 2;
            const int64_t coff = kind == 0 ? (int64_t)head * hd + kk
                                 : (int64_t)(kind == 1 ? head - H : head - H - Hk) * hs + kk;
            __nv_bfloat16* const pool = kind == 1 ? p.k_pool : p.v_pool;
#pragma unroll
            for (int i = 0; i < RC; ++i) {
              const int row = r0 + i;
              if (row < R && n < P.N) {
                const float ev = odd ? other[i] : val[i], ov = odd ? val[i] : other[i];
                const float res = odd ? (ev * sn[i] + ov * cs[i]) : (ev * cs[i] - ov * sn[i]);
                if (kind == 0)
                  p.q[(int64_t)row * H * hd + coff] = res;
                else
                  pool[s_koff[row] + coff] = __float2bfloat16_rn(kind == 1 ? res : val[i]);
              }
            }
          }
        }
        if (!cut) {
          tc_fence_before();
          mbar_arrive(&acc_empty[buf]);
        }
        if (et == 0 && last_seg) TR(28 + ph * 4);
        // publish the tile (its consumers in later phases acquire the flag)
        if (ph != kPhQKV && (ph != kPhD || P.gamma)) {
          fence_proxy_async_global();
          epi_bar();
          if (et == 0) {
            asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
            red_release_add(p.done + ph, 1);
          }
        }
        if (et == 0) TR(5 + ph * 6);
        if (et == 0 && last_seg) TR(29 + ph * 4);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) TR(25);
  if (warp == 1) tmem_dealloc(tmem_base, C::kTmemCols);
  if (tid == 0) {  // the last CTA out zeroes the completion counters for the next launch
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    if (atomicAdd(p.done + kChPhases, 1) == p.grid - 1) {
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
      for (int i = 0; i <= kChPhases; ++i) p.done[i] = 0;
    }
  }
}

// Prologue of a chained step: x (+= delta) ; h = hi/lo(x * gamma) ; ssq[chunk][row] over
// 128-column chunks (the format the chain's RESID epilogues write).  One CTA per row,
// one warp per chunk.
__global__ void __launch_bounds__(128) chain_prologue_kernel(float* __restrict__ x,
                                                             const float* __restrict__ delta,
                                                             int d, const __nv_bfloat16* gamma,
                                                             __nv_bfloat16* __restrict__ h,
                                                             int split, int n_rows,
                                                             float* __restrict__ ssq) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_chunks = (d + 127) / 128;
  for (int ch = warp; ch < n_chunks; ch += 4) {
    float s = 0.f;
    for (int k = 0; k < 4; ++k) {
      const int n = ch * 128 + k * 32 + lane;
      if (n < d) {
        float v = x[(size_t)r * d + n];
        if (delta) {
          v += delta[(size_t)r * d + n];
          x[(size_t)r * d + n] = v;
        }
        s += v * v;
        const float u = v * __bfloat162float(gamma[n]);
        const __nv_bfloat16 hh = __float2bfloat16_rn(u);
        h[(size_t)r * d + n] = hh;
        if (split) h[(size_t)(n_rows + r) * d + n] = __float2bfloat16_rn(u - __bfloat162float(hh));
      }
    }
    s = warp_sum(s);
    if (lane == 0) ssq[(size_t)ch * kChSsq + r] = s;
  }
}

// ---------------------------------------------------------------- host side
template <int NX, int KSUB>
static int launch_chain(ChParams& p, const ChMaps& maps, cudaStream_t s) {
  using C = ChCfg<NX, KSUB>;
  p.stages = C::kStages;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(chain_sm100<NX, KSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::smem());
    attr_set = true;
  }
  launch_k(chain_sm100<NX, KSUB>, p.grid, kChThreads, C::smem(), s, p, maps);
  return launch_status("choreo_layer_chain");
}

}  // namespace choreo

using namespace choreo;

extern "C" int choreo_layer_chain(const ChoreoLayerChain* L, void* stream) {
  if (!L || !L->x || !L->ws || !L->counters || !L->done || L->n_rows <= 0 || L->d <= 0 ||
      !(L->phases & 15))
    return CHOREO_EINVAL;
  const int R = L->n_rows, sp = L->split ? 1 : 0, d = L->d;
  const int xr = sp ? 2 * R : R;
  if (xr > 256 || (!sp && R > 128)) return CHOREO_EUNSUPPORTED;
  const int NX = xr <= 16 ? 16 : xr <= 32 ? 32 : xr <= 64 ? 64 : xr <= 128 ? 128 : 256;
  const int rpad = sp ? NX / 2 : NX;
  const int H = L->n_heads, Hk = L->n_kv, hd = L->head_dim, F = L->ffn_dim;
  const int n_qkv = (H + 2 * Hk) * hd;
  if (d % 64 || (H * hd) % 64 || F % 64 || (L->phases & 8 && (hd & 1)))
    return CHOREO_EUNSUPPORTED;
  ChParams p{};
  ChMaps maps{};
  const int ksub = NX >= 128 ? 1 : 2;
  const int kstep = 64 * ksub;
  auto set_phase = [&](int ph, const void* w, int w_rows, const void* xbuf, int N, int K,
                       int n_tiles, int box_w_rows) -> bool {
    ChPhase& P = p.ph[ph];
    P.on = 1;
    P.N = N;
    P.K = K;
    P.n_tiles = n_tiles;
    P.KB = (K + kstep - 1) / kstep;
    P.iters = n_tiles * P.KB;
    P.x_rows = xr;
    P.ssq_dep = -2;
    P.x_dep = -1;
    P.x_prev_dep = -1;
    if (n_tiles > kChMaxTiles) return false;
    return tmap_bf16_2d(&maps.w[ph], w, (uint64_t)w_rows, (uint64_t)K, 64, (uint32_t)box_w_rows,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B) &&
           tmap_bf16_2d(&maps.x[ph], xbuf, (uint64_t)xr, (uint64_t)K, 64,
                        (uint32_t)(sp ? NX / 2 : NX), CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  };
  const int tiles_d = (d + kChTile - 1) / kChTile;
  int prev_resid = -1;  // phase of this launch that last wrote x
  int prev_h = -1;      // phase of this launch whose outputs feed the next GEMM input
  if (L->phases & 1) {  // o_proj + residual + ffn norm
    if (!L->wo || !L->attn || !L->ffn_norm || !L->h_a || !L->ssq_a) return CHOREO_EINVAL;
    if (!set_phase(kPhO, L->wo, d, L->attn, d, H * hd, tiles_d, kChTile)) return CHOREO_ELAUNCH;
    ChPhase& P = p.ph[kPhO];
    P.gamma = L->ffn_norm;
    P.out = L->h_a;
    P.ssq_out = L->ssq_a;
    prev_resid = prev_h = kPhO;
  }
  if (L->phases & 2) {  // gate|up + SwiGLU
    if (!L->w_gu || !L->h_a || !L->act || !L->ssq_a) return CHOREO_EINVAL;
    if (!set_phase(kPhGU, L->w_gu, 2 * F, L->h_a, F, d, F / 64, 64)) return CHOREO_ELAUNCH;
    ChPhase& P = p.ph[kPhGU];
    P.x_dep = prev_h;
    P.x_dep_w = kChTile;
    P.ssq_dep = prev_h;  // -1 when the ffn norm's sums come from an earlier launch
    P.ssq_tiles = tiles_d;
    P.ssq_in = L->ssq_a;
    P.out = L->act;
    prev_h = kPhGU;
  }
  if (L->phases & 4) {  // down + residual (+ next attention norm)
    if (!L->w_down || !L->act) return CHOREO_EINVAL;
    if (!set_phase(kPhD, L->w_down, d, L->act, d, F, tiles_d, kChTile)) return CHOREO_ELAUNCH;
    ChPhase& P = p.ph[kPhD];
    P.x_dep = prev_h;
    P.x_dep_w = 64;
    P.x_prev_dep = prev_resid;
    if (L->attn_norm_next) {
      if (!L->h_b || !L->ssq_b) return CHOREO_EINVAL;
      P.gamma = L->attn_norm_next;
      P.out = L->h_b;
      P.ssq_out = L->ssq_b;
    }
    prev_resid = kPhD;
    prev_h = L->attn_norm_next ? kPhD : -3;
  }
  if (L->phases & 8) {  // qkv + RoPE + K/V append
    if (!L->w_qkv || !L->h_b || !L->ssq_b || !L->q || !L->k_pool || !L->v_pool || !L->pos ||
        !L->page || !L->slot || !L->cos_t || !L->sin_t || prev_h == -3)
      return CHOREO_EINVAL;
    if (!set_phase(kPhQKV, L->w_qkv, n_qkv, L->h_b, n_qkv, d, (n_qkv + kChTile - 1) / kChTile,
                   kChTile))
      return CHOREO_ELAUNCH;
    ChPhase& P = p.ph[kPhQKV];
    P.x_dep = prev_h == kPhD ? kPhD : -1;
    P.x_dep_w = kChTile;
    P.ssq_dep = P.x_dep;
    P.ssq_tiles = tiles_d;
    P.ssq_in = L->ssq_b;
  }
  int grid = 148;
  for (int ph = 0; ph < kChPhases; ++ph)
    if (p.ph[ph].on && p.ph[ph].iters < grid) grid = p.ph[ph].iters;
  p.x = L->x;
  p.d = d;
  p.R = R;
  p.split = sp;
  p.rpad = rpad;
  p.eps = L->eps;
  p.q = L->q;
  p.k_pool = reinterpret_cast<__nv_bfloat16*>(L->k_pool);
  p.v_pool = reinterpret_cast<__nv_bfloat16*>(L->v_pool);
  p.layer = L->layer_qkv;
  p.n_kv = Hk;
  p.n_heads = H;
  p.hd = hd;
  p.n_pages = L->n_pages;
  p.page_size = L->page_size;
  p.pos = L->pos;
  p.page = L->page;
  p.slot = L->slot;
  p.cos_t = L->cos_t;
  p.sin_t = L->sin_t;
  p.max_delta = L->max_delta;
  p.ws = L->ws;
  p.counters = L->counters;
  p.done = L->done;
#ifdef CHOREO_TRACE
  p.trace_slot = g_trace_launches++;
#endif
  p.grid = grid;
  auto s = as_stream(stream);
  switch (NX) {
    case 16: return launch_chain<16, 2>(p, maps, s);
    case 32: return launch_chain<32, 2>(p, maps, s);
    case 64: return launch_chain<64, 2>(p, maps, s);
    case 128: return launch_chain<128, 1>(p, maps, s);
    default: return launch_chain<256, 1>(p, maps, s);
  }
}

#ifdef CHOREO_TRACE
extern "C" int choreo_chain_set_trace(long long* buf) {
  g_trace_launches = 0;
  return cudaMemcpyToSymbol(g_chain_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -2;
}
#endif

extern "C" int choreo_chain_prologue(float* x, const float* delta, int n_rows, int d,
                                     const void* gamma, void* h, int split, float* ssq,
                                     void* stream) {
  if (!x || !gamma || !h || !ssq || n_rows <= 0 || n_rows > kChSsq || d <= 0) return CHOREO_EINVAL;
  launch_k(chain_prologue_kernel, n_rows, 128, 0, as_stream(stream), x, delta, d,
           reinterpret_cast<const __nv_bfloat16*>(gamma), reinterpret_cast<__nv_bfloat16*>(h),
           split, n_rows, ssq);
  return launch_status("choreo_chain_prologue");
}
