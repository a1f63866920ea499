// K7 weight-streaming linear layer for decode-sized steps (tcgen05 + TMEM + TMA, stream-K).
//
// A decode step multiplies a handful of activation rows (8 agents, as hi/lo bf16 pairs:
// 16 rows) by every weight matrix of the model: y[r][n] = sum_k x[r][k] * w[n][k].  The
// work is pure weight streaming (16 GB per step at the Llama-3.1-8B shape), so the kernel
// is built to keep HBM busy, not the tensor core:
//   * swap-AB: a 128-row weight tile is the UMMA A operand (M = 128), the activation rows
//     are the B operand (N = NX = 16/32/64/128), accumulators live in TMEM (NX columns);
//   * stream-K: the (tile, k-block) iteration space is cut into one equal contiguous range
//     per CTA (one CTA per SM), so every SM streams the same number of weight bytes
//     whatever the tile count (qkv: 48 tiles, o_proj/down: 32, gate|up: 224, head: 1002);
//   * TMA producer warp with a 4-stage ring (2 k-blocks = 32 KB of weights + the activation
//     chunk per stage, ~144 KB in flight per SM; weights loaded evict-first), single-thread
//     MMA issue, 4 epilogue warps;
//   * a tile cut between CTAs is reduced deterministically: each piece is written to a
//     per-CTA slot, the last piece to arrive sums all pieces in CTA order -- or, in the
//     deferred mode (choreo_linear_skinny_pieces), the pieces stay in their slots and the
//     consuming kernel sums them in the same order (k7_get, bit-identical);
//   * with split activations (x rows r and R + r are the hi/lo halves of one row) the
//     halves are loaded to B rows r and NX/2 + r and the epilogue adds them: y has R rows.
// Replaces the dense projections of reference model.py:172-174, 185-189, 193 at decode
// sizes (the reference runs them as NumPy matmuls x @ W).
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace choreo {

constexpr int kLnThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kLnTile = 128;     // weight rows per tile (UMMA M)
constexpr int kLnKB = 64;        // k elements per block (one 128-byte SW128 row)

struct LinearParams {
  float* y;       // [out_rows][N] (or, with silu_f > 0, act: bf16 [out_rows (x2 split)][silu_f])
  float* ws;      // [grid][2][NX][128] partial tiles (NX <= 128)
  int* counters;  // [n_tiles], zero between launches (reducers reset them)
  int N, KB, iters, grid, out_rows, split;
  int silu_f;  // > 0: gate|up projection with SiLU(gate)*up fused (tile t = gate rows
               // [64t, 64t+64) over up rows [F + 64t, ...)); N counts act columns (= F)
  int defer;   // 1: cut tiles stay as pieces in ws for the consumer (ChoreoK7Pieces)
  int stages;  // ring depth (<= LnCfg::kStages): sets the shared memory a CTA holds
};

template <int NX, int KSUB>
struct LnCfg {
  static constexpr int kWBytes = kLnTile * 128;  // one k-block of the weight tile
  static constexpr int kXBytes = NX * 128;       // one k-block of the activations
  static constexpr int kStageBytes = KSUB * (kWBytes + kXBytes);
  // at most 4 stages: measured on the 8B decode step (tools/k7_ab.sh), a 4-stage ring (148 KB
  // at NX 16) beats 5 stages by ~1 % and 2 stages lose 8 %
  static constexpr int kStages = (200 * 1024) / kStageBytes > 4 ? 4 : (200 * 1024) / kStageBytes;
  static constexpr int smem(int stages) { return stages * kStageBytes + 1024; }
  static constexpr int kTmemCols = 2 * NX < 32 ? 32 : 2 * NX;
};


template <int NX, int KSUB>
__global__ void __launch_bounds__(kLnThreads, 1)
    linear_skinny_sm100(LinearParams p, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmX) {
  using namespace sm100;
  using C = LnCfg<NX, KSUB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[C::kStages], empty_bar[C::kStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ int s_last;
  __shared__ float s_xch[16 * 64];  // SiLU epilogue: up values of 16 rows x 64 columns

  pdl_trigger();  // the successor may launch now; it waits for this grid to complete
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x;
  const int b = ln_begin(c, p.iters, p.grid), e = ln_begin(c + 1, p.iters, p.grid);
  if (tid == 0) {
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 1) tmem_alloc(&tmem_base, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- TMA producer
      // weights are read once per step: evict-first keeps the step's activations, pieces
      // and code resident in L2 under the 16 GB stream
      const uint64_t pol = l2_policy_evict_first();
      auto load_w = [&](int i, int st) {
        uint8_t* dst = base + st * C::kStageBytes;
        const int t = i / p.KB, kb = (i % p.KB) * KSUB;
        // the KSUB weight boxes go out back to back: 128 rows x KSUB*128 contiguous bytes
#pragma unroll
        for (int u = 0; u < KSUB; ++u)
          if (p.silu_f) {  // 64 gate rows over the matching 64 up rows
            tma_load_2d_hint(dst + u * C::kWBytes, &tmW, &full_bar[st], (kb + u) * kLnKB, t * 64,
                             pol);
            tma_load_2d_hint(dst + u * C::kWBytes + 64 * 128, &tmW, &full_bar[st],
                             (kb + u) * kLnKB, p.silu_f + t * 64, pol);
          } else {
            tma_load_2d_hint(dst + u * C::kWBytes, &tmW, &full_bar[st], (kb + u) * kLnKB,
                             t * kLnTile, pol);
          }
      };
      auto load_x = [&](int i, int st) {
        uint8_t* xd = base + st * C::kStageBytes + KSUB * C::kWBytes;
        const int kb = (i % p.KB) * KSUB;
#pragma unroll
        for (int u = 0; u < KSUB; ++u) {
          if (p.split) {  // hi rows -> smem rows [0, NX/2), lo rows -> [NX/2, NX)
            tma_load_2d(xd + u * C::kXBytes, &tmX, &full_bar[st], (kb + u) * kLnKB, 0);
            tma_load_2d(xd + u * C::kXBytes + C::kXBytes / 2, &tmX, &full_bar[st], (kb + u) * kLnKB,
                        p.out_rows);
          } else {
            tma_load_2d(xd + u * C::kXBytes, &tmX, &full_bar[st], (kb + u) * kLnKB, 0);
          }
        }
      };
      // weights do not depend on the previous kernel: fill the ring with them before the
      // programmatic-dependency wait, then add the activations (written by the predecessor)
      const int NS = p.stages;
      const int pre = min(e - b, NS);
      for (int j = 0; j < pre; ++j) {
        mbar_arrive_expect_tx(&full_bar[j], C::kStageBytes);
        load_w(b + j, j);
      }
      pdl_wait();
      for (int j = 0; j < pre; ++j) load_x(b + j, j);
      for (int i = b + pre; i < e; ++i) {
        const int j = i - b, st = j % NS;
        mbar_wait(&empty_bar[st], ((j / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&full_bar[st], C::kStageBytes);
        load_w(i, st);
        load_x(i, st);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(kLnTile, NX, false);
      const int NS = p.stages;
      int seg = 0;
      for (int i = b; i < e; ++i) {
        const int j = i - b, st = j % NS, kb = i % p.KB;
        const bool first = (i == b) || kb == 0;
        const bool last = (i == e - 1) || kb == p.KB - 1;
        const int buf = seg & 1;
        if (first && seg >= 2) mbar_wait(&acc_empty[buf], ((seg >> 1) - 1) & 1);
        mbar_wait(&full_bar[st], (j / NS) & 1);
        tc_fence_after();
        const uint32_t waddr = smem_addr(base + st * C::kStageBytes);
        const uint32_t xaddr = waddr + KSUB * C::kWBytes;
        const uint32_t d = tmem_base + buf * NX;
#pragma unroll
        for (int u = 0; u < KSUB; ++u)
#pragma unroll
          for (int k = 0; k < kLnKB / 16; ++k)
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
  } else {
    // ------------------------------------------------------------------ epilogue
    pdl_wait();  // y / workspace / counters are touched only after the predecessor is done
    const int quad = warp & 3;
    const int nl = quad * 32 + lane;  // weight row within the tile = TMEM lane
    const int et = tid - 64;          // 0..127
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int seg = 0;
    // output rows are handled in chunks of RC: split activations pair TMEM column r (hi half)
    // with NX/2 + r (lo half); at NX 16 both halves come from one 16-column load
    constexpr int RC = NX == 16 ? 8 : 16;
    const int rows_half = p.split ? NX / 2 : NX;  // output rows the accumulator holds
    for (int t = b / p.KB; t * p.KB < e; ++t, ++seg) {
      const int buf = seg & 1;
      const int lo = t * p.KB, hi = lo + p.KB;
      const int c_lo = ln_owner(lo, p.iters, p.grid), c_hi = ln_owner(hi - 1, p.iters, p.grid);
      mbar_wait(&acc_full[buf], (seg >> 1) & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + lane_off + buf * NX;
      // raw accumulator columns of chunk r0: a = rows r0.. (hi half), bb = NX/2 + r0.. (lo)
      auto ld_chunk = [&](int r0, float* a, float* bb) {
        if (NX == 16) {
          float t16[16];
          tmem_ld16(tb, t16);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < RC; ++i) {
            a[i] = p.split ? t16[i] : t16[r0 + i];
            bb[i] = p.split ? t16[8 + i] : 0.f;
          }
        } else {
          tmem_ld16(tb + r0, a);
          if (p.split) tmem_ld16(tb + NX / 2 + r0, bb);
          tmem_wait_ld();
          if (!p.split) {
#pragma unroll
            for (int i = 0; i < RC; ++i) bb[i] = 0.f;
          }
        }
      };
      const int n = t * kLnTile + nl;
      const bool cut = c_lo != c_hi;
      if (cut) {
        // piece of a tile cut between CTAs: park it (hi + lo halves summed: rows_half rows x
        // 128, the layout k7_get reads); the last piece reduces in CTA order
        const int slot = (b >= lo) ? 0 : 1;
        float* w = p.ws + ((size_t)(c * 2 + slot) * rows_half) * kLnTile + nl;
        for (int r0 = 0; r0 < rows_half; r0 += RC) {
          float a[16], bb[16];
          ld_chunk(r0, a, bb);
#pragma unroll
          for (int i = 0; i < RC; ++i) w[(r0 + i) * kLnTile] = p.split ? a[i] + bb[i] : a[i];
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
        if (p.defer) continue;  // the consumer sums the pieces (k7_get)
        // the group's barrier orders the 128 threads' partial stores before thread 0's
        // GPU-scope release (one fence per piece instead of one per thread); the last piece
        // acquires the others the same way before reading them
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (et == 0) {
          asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
          const int old = atomicAdd(&p.counters[t], 1);
          s_last = old == c_hi - c_lo;
          if (s_last) asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (!s_last) continue;
        if (et == 0) p.counters[t] = 0;
      }
      // final rows of chunk r0 -> v: the pieces summed in CTA order (the order k7_get uses,
      // so deferred and reduced outputs are bit-identical), 4 pieces' loads in flight
      auto final_chunk = [&](int r0, float* v) {
        if (!cut) {
          float a[16], bb[16];
          ld_chunk(r0, a, bb);
#pragma unroll
          for (int i = 0; i < RC; ++i) v[i] = p.split ? a[i] + bb[i] : a[i];
          return;
        }
#pragma unroll
        for (int i = 0; i < RC; ++i) v[i] = 0.f;
        for (int c0 = c_lo; c0 <= c_hi; c0 += 4) {
          float pv[4][RC];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int cc = c0 + jj;
            if (cc <= c_hi) {
              const int sl = (ln_begin(cc, p.iters, p.grid) >= lo) ? 0 : 1;
              const float* r = p.ws + ((size_t)(cc * 2 + sl) * rows_half + r0) * kLnTile + nl;
#pragma unroll
              for (int i = 0; i < RC; ++i) pv[jj][i] = __ldcg(r + i * kLnTile);
            }
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (c0 + jj <= c_hi) {
#pragma unroll
              for (int i = 0; i < RC; ++i) v[i] += pv[jj][i];
            }
        }
      };
      if (p.silu_f) {
        // lanes 0-63 hold gate, 64-127 up of the same 64 ffn columns: exchange through smem
        // in chunks, then act = silu(g) * u (the formula of choreo_silu_mul) as bf16
        // (hi/lo rows r and out_rows + r when split)
        const int j = t * 64 + (nl & 63);
        __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(p.y);
        const int64_t lo_off = (int64_t)p.out_rows * p.silu_f;
        for (int r0 = 0; r0 < rows_half; r0 += RC) {
          float v[16];
          final_chunk(r0, v);
          asm volatile("bar.sync 1, 128;\n" ::: "memory");  // s_xch free
          if (nl >= 64) {
#pragma unroll
            for (int i = 0; i < RC; ++i) s_xch[i * 64 + (nl - 64)] = v[i];
          }
          asm volatile("bar.sync 1, 128;\n" ::: "memory");
          if (nl < 64) {
#pragma unroll
            for (int i = 0; i < RC; ++i) {
              const int r = r0 + i;
              if (r < p.out_rows) {
                const float g = v[i];
                const float vv = g / (1.0f + expf(-g)) * s_xch[i * 64 + nl];
                const __nv_bfloat16 h = __float2bfloat16_rn(vv);
                act[(int64_t)r * p.silu_f + j] = h;
                if (p.split) act[lo_off + (int64_t)r * p.silu_f + j] = __float2bfloat16_rn(vv - __bfloat162float(h));
              }
            }
          }
        }
      } else {
        // every lane runs final_chunk: tcgen05.ld is warp-collective (columns past N too)
        for (int r0 = 0; r0 < rows_half && r0 < p.out_rows; r0 += RC) {
          float v[16];
          final_chunk(r0, v);
          if (n < p.N) {
#pragma unroll
            for (int i = 0; i < RC; ++i)
              if (r0 + i < p.out_rows) p.y[(size_t)(r0 + i) * p.N + n] = v[i];
          }
        }
      }
      if (!cut) {
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, C::kTmemCols);
}

// ---------------------------------------------------------------- host side
// row-major [rows][cols] bf16, box = 64 cols x box_rows rows, SW128 (cached, tmap.cuh)
static bool ln_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, int box_rows,
                   CUtensorMapL2promotion l2) {
  return tmap_bf16_2d(m, ptr, rows, cols, 64, (uint32_t)box_rows, l2);
}

template <int NX, int KSUB>
static int launch_linear(const LinearParams& p, const void* x, int x_rows, const void* w, int N,
                         int K, cudaStream_t s) {
  CUtensorMap mw, mx;
  if (!ln_map(&mw, w, (uint64_t)(p.silu_f ? 2 * p.silu_f : N), (uint64_t)K,
              p.silu_f ? 64 : kLnTile, CU_TENSOR_MAP_L2_PROMOTION_L2_256B) ||
      !ln_map(&mx, x, (uint64_t)x_rows, (uint64_t)K, p.split ? NX / 2 : NX,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B))
    return CHOREO_ELAUNCH;
  using C = LnCfg<NX, KSUB>;
  const int smem = C::smem(p.stages);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(linear_skinny_sm100<NX, KSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::smem(C::kStages));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(kLnThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, linear_skinny_sm100<NX, KSUB>, p, mw, mx);
  return launch_status("choreo_linear_skinny");
}

}  // namespace choreo

using namespace choreo;

static int linear_impl(const void* x, int x_rows, int split, const void* w, int n, int k, void* y,
                       float* workspace, int* tile_counters, int grid_ctas, int silu_f,
                       void* stream, ChoreoK7Pieces* pieces = nullptr) {
  if (!x || !w || !y || !workspace || !tile_counters || x_rows <= 0 || n <= 0 || k <= 0 ||
      (split && (x_rows & 1)))
    return CHOREO_EINVAL;
  if (x_rows > 256 || (!split && x_rows > 128) || k % 8) return CHOREO_EUNSUPPORTED;
  if (silu_f && silu_f % 64) return CHOREO_EUNSUPPORTED;
  const int R = split ? x_rows / 2 : x_rows;  // output rows
  const int xr = split ? 2 * R : R;
  const int NX = xr <= 16 ? 16 : xr <= 32 ? 32 : xr <= 64 ? 64 : xr <= 128 ? 128 : 256;
  const int n_tiles = silu_f ? silu_f / 64 : (n + kLnTile - 1) / kLnTile;
  // k-blocks per ring stage: 2 (1 at 256 activation rows, whose X block alone is 32 KB)
  const int ks = NX == 256 ? 1 : 2;
  const int KB = (k + kLnKB * ks - 1) / (kLnKB * ks);  // iteration = ks k-blocks
  const int iters = n_tiles * KB;
  int grid = grid_ctas > 0 ? grid_ctas : 148;
  if (grid > iters) grid = iters;
  static int max_smem = -1;  // CHOREO_K7_SMEM_KB: cap the ring's shared memory (co-residency)
  if (max_smem < 0) {
    const char* e = getenv("CHOREO_K7_SMEM_KB");
    max_smem = e ? atoi(e) * 1024 : 0;
  }
  LinearParams p{reinterpret_cast<float*>(y), workspace, tile_counters, n, KB, iters, grid,
                 split ? x_rows / 2 : x_rows, split, silu_f, pieces ? 1 : 0, 0};
  if (pieces) {
    if (silu_f) return CHOREO_EINVAL;
    *pieces = ChoreoK7Pieces{reinterpret_cast<const float*>(y), workspace, n, KB, iters, grid, NX,
                             split};
  }
  auto s = as_stream(stream);
  auto stages_for = [&](int full, int stage_bytes) {
    int st = full;
    if (max_smem > 0) st = (max_smem - 1024) / stage_bytes;
    return st < 2 ? 2 : st > full ? full : st;
  };
#define LN_STAGES(nx, ks) \
  (p.stages = stages_for(LnCfg<nx, ks>::kStages, LnCfg<nx, ks>::kStageBytes), p)
#define LN_CASE(nx) return launch_linear<nx, 2>(LN_STAGES(nx, 2), x, x_rows, w, n, k, s);
  switch (NX) {
    case 16: LN_CASE(16)
    case 32: LN_CASE(32)
    case 64: LN_CASE(64)
    case 128: LN_CASE(128)
    default:  // 256 activation rows: one k-block per stage (48 KB)
      return launch_linear<256, 1>(LN_STAGES(256, 1), x, x_rows, w, n, k, s);
  }
#undef LN_CASE
#undef LN_STAGES
}

extern "C" int choreo_linear_skinny(const void* x, int x_rows, int split, const void* w, int n,
                                    int k, float* y, float* workspace, int* tile_counters,
                                    int grid_ctas, void* stream) {
  return linear_impl(x, x_rows, split, w, n, k, y, workspace, tile_counters, grid_ctas, 0, stream);
}

extern "C" int choreo_linear_gate_up_silu(const void* x, int x_rows, int split, const void* w_gu,
                                          int f, int d, void* act, float* workspace,
                                          int* tile_counters, void* stream) {
  if (f <= 0) return CHOREO_EINVAL;
  return linear_impl(x, x_rows, split, w_gu, f, d, act, workspace, tile_counters, 0, f, stream);
}

extern "C" int choreo_linear_skinny_pieces(const void* x, int x_rows, int split, const void* w,
                                           int n, int k, float* y, float* workspace,
                                           int* tile_counters, int grid_ctas,
                                           ChoreoK7Pieces* pieces, void* stream) {
  if (!pieces) return CHOREO_EINVAL;
  return linear_impl(x, x_rows, split, w, n, k, y, workspace, tile_counters, grid_ctas, 0, stream,
                     pieces);
}
