// Diagnostics: a one-CTA tcgen05 GEMM that exercises exactly the primitives K4 uses
// (TMEM alloc, SW128 K-major and MN-major UMMA smem descriptors, kind::f16 MMA,
// commit -> mbarrier, tcgen05.ld).  C1 = A * B1^T (B1 K-major), C2 = A * B2 (B2 MN-major).
#include "common.cuh"
#include "sm100.cuh"

namespace choreo {

__global__ void __launch_bounds__(128) umma_selftest_kernel(const __nv_bfloat16* __restrict__ A,
                                                            const __nv_bfloat16* __restrict__ B1,
                                                            const __nv_bfloat16* __restrict__ B2,
                                                            float* __restrict__ C1,
                                                            float* __restrict__ C2,
                                                            float* __restrict__ C3) {
  using namespace sm100;
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB1[64 * 128];
  __shared__ __align__(1024) uint8_t sB2[2 * 64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A [128][64] and B1 [64][64] (rows = M / N, 64 K elements) -> K-major SW128
  for (int c = tid; c < 128 * 8; c += 128) {
    const int r = c >> 3, ch = c & 7;
    *reinterpret_cast<uint4*>(sA + sw128_offset(r, ch * 8)) =
        *reinterpret_cast<const uint4*>(A + r * 64 + ch * 8);
  }
  for (int c = tid; c < 64 * 8; c += 128) {
    const int r = c >> 3, ch = c & 7;
    *reinterpret_cast<uint4*>(sB1 + sw128_offset(r, ch * 8)) =
        *reinterpret_cast<const uint4*>(B1 + r * 64 + ch * 8);
  }
  // B2 [64 K][128 N] row-major -> MN-major SW128: two 64-wide N blocks of [64 K rows][128 B]
  for (int c = tid; c < 64 * 16; c += 128) {
    const int k = c >> 4, ch = c & 15;
    const int blk = ch >> 3;
    *reinterpret_cast<uint4*>(sB2 + blk * 8192 + sw128_offset(k, (ch & 7) * 8)) =
        *reinterpret_cast<const uint4*>(B2 + k * 128 + ch * 8);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t a0 = smem_addr(sA), b10 = smem_addr(sB1), b20 = smem_addr(sB2);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = umma_desc_sw128(a0 + k * 32, 16, 1024);
      umma_bf16(tm, ad, umma_desc_sw128(b10 + k * 32, 16, 1024), umma_idesc_bf16(128, 64, false), k > 0);
      umma_bf16(tm + 128, ad, umma_desc_sw128(b20 + k * 2048, 8192, 1024),
                umma_idesc_bf16(128, 128, true), k > 0);
    }
    umma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  // C3 = A (staged in TMEM cols [256, 288) as packed bf16 pairs) * B2 (MN-major smem)
  {
    const int r = warp * 32 + lane;
    uint32_t pk[16];
    for (int half = 0; half < 2; ++half) {
      for (int i = 0; i < 16; ++i) {
        __nv_bfloat162 h = __halves2bfloat162(A[r * 64 + half * 32 + 2 * i], A[r * 64 + half * 32 + 2 * i + 1]);
        pk[i] = *reinterpret_cast<uint32_t*>(&h);
      }
      tmem_st16u(tm + ((uint32_t)(warp * 32) << 16) + 256 + half * 16, pk);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t b20 = smem_addr(sB2);
    for (int k = 0; k < 4; ++k)
      umma_bf16_tmem_a(tm + 384, tm + 256 + k * 8, umma_desc_sw128(b20 + k * 2048, 8192, 1024),
                       umma_idesc_bf16(128, 128, true), k > 0);
    umma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 1);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t lane_addr = tm + ((uint32_t)(warp * 32) << 16);
  float v[16];
  for (int c0 = 0; c0 < 64; c0 += 16) {
    tmem_ld16(lane_addr + c0, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) C1[row * 64 + c0 + i] = v[i];
  }
  for (int c0 = 0; c0 < 128; c0 += 16) {
    tmem_ld16(lane_addr + 128 + c0, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) C2[row * 128 + c0 + i] = v[i];
  }
  for (int c0 = 0; c0 < 128; c0 += 16) {
    tmem_ld16(lane_addr + 384 + c0, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) C3[row * 128 + c0 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

}  // namespace choreo

extern "C" int choreo_selftest_umma(const void* a, const void* b1, const void* b2, float* c1,
                                    float* c2, float* c3, void* stream) {
  if (!a || !b1 || !b2 || !c1 || !c2 || !c3) return CHOREO_EINVAL;
  choreo::umma_selftest_kernel<<<1, 128, 0, choreo::as_stream(stream)>>>(
      (const __nv_bfloat16*)a, (const __nv_bfloat16*)b1, (const __nv_bfloat16*)b2, c1, c2, c3);
  return choreo::launch_status("choreo_selftest_umma");
}
