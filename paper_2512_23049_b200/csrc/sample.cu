// K6b nucleus (temperature + top-p) selection on the device, the reference's algorithm in
// f64 step for step (engine.py:374-392), so sampled decoding needs no logits round trip:
//   z = logits / T over the generatable ids {0..255, 257} (others -inf); p = exp(z - max);
//   p /= sum(p)                          (NumPy's pairwise summation order)
//   order = lexsort((id, -p)); csum = cumsum(p[order]); cut = searchsorted(csum, top_p, left)
//   kept = order[:cut + 1]; kcs = cumsum(p[kept] / sum(p[kept]))
//   u = Philox4x64-10 draw, counter (sel, msg_id, 0, 0), key (engine_seed, sampling_seed):
//       the first output of the counter incremented once, (x >> 11) * 2^-53 (NumPy's
//       Generator(Philox).random())
//   token = kept[min(searchsorted(kcs, u, right), len(kept) - 1)]
// One CTA per row.  Sums follow NumPy's pairwise order (blocks of <= 128 with 8 partial
// accumulators, halving at multiples of 8); exp is the device f64 exp (<= 1 ulp from the
// host's), so tokens match the host sampler except on knife-edge boundaries.
#include <math.h>

#include "common.cuh"

namespace choreo {

constexpr int kNucThreads = 288;  // >= 257 candidates
constexpr int kNCand = 257;

__device__ __forceinline__ int cand_id(int c) { return c < 256 ? c : 257; }

// NumPy pairwise_sum over a virtual array: value(i) for i in [lo, lo + n)
template <typename F>
__device__ double np_pairwise(F value, long long lo, long long n) {
  // explicit stack of (lo, n, partial) frames
  struct Frame { long long lo, n; int state; double left; };
  Frame st[48];
  int sp = 0;
  st[0] = {lo, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n < 8) {
      double r = 0.0;
      for (long long i = 0; i < f.n; ++i) r += value(f.lo + i);
      ret = r;
      --sp;
    } else if (f.n <= 128) {
      double r[8];
      for (int j = 0; j < 8; ++j) r[j] = value(f.lo + j);
      long long i = 8;
      for (; i < f.n - (f.n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += value(f.lo + i + j);
      double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < f.n; ++i) res += value(f.lo + i);
      ret = res;
      --sp;
    } else {
      long long n2 = f.n / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        st[++sp] = {f.lo, n2, 0, 0.0};
      } else if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        st[++sp] = {f.lo + n2, f.n - n2, 0, 0.0};
      } else {
        ret = f.left + ret;
        --sp;
      }
    }
  }
  return ret;
}

__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

__device__ double philox_uniform(uint64_t c0, uint64_t c1, uint64_t k0, uint64_t k1) {
  uint64_t v0 = c0 + 1, v1 = c1 + (c0 + 1 == 0 ? 1 : 0), v2 = 0, v3 = 0;  // counter++ first
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, v0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ull, v2, hi1, lo1);
    const uint64_t n0 = hi1 ^ v1 ^ k0, n2 = hi0 ^ v3 ^ k1;
    v0 = n0;
    v1 = lo1;
    v2 = n2;
    v3 = lo0;
  }
  return (double)(v0 >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void __launch_bounds__(kNucThreads) select_nucleus_kernel(
    const float* __restrict__ logits, int64_t ld, int vocab, const double* __restrict__ params,
    const uint64_t* __restrict__ keys, int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, tid = threadIdx.x;
  const float* lr = logits + row * ld;
  const double T = params[2 * row], top_p = params[2 * row + 1];
  __shared__ double s_p[kNCand], s_sorted[kNCand];
  __shared__ int s_id[kNCand];
  __shared__ double s_red[kNucThreads / 32];
  __shared__ double s_max, s_sum;
  __shared__ int s_npos;
  // z and its max over the generatable ids
  double z = -INFINITY;
  if (tid < kNCand) z = (double)lr[cand_id(tid)] / T;
  double m = z;
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) s_red[tid >> 5] = m;
  __syncthreads();
  if (tid == 0) {
    double mm = -INFINITY;
    for (int i = 0; i < kNucThreads / 32; ++i) mm = fmax(mm, s_red[i]);
    s_max = mm;
  }
  __syncthreads();
  if (tid < kNCand) s_p[tid] = exp(z - s_max);
  __syncthreads();
  if (tid == 0) {  // NumPy's pairwise sum over the V-long array (zeros off the candidates)
    auto val = [&](long long i) -> double {
      return i < 256 ? s_p[i] : (i == 257 ? s_p[256] : 0.0);
    };
    s_sum = np_pairwise(val, 0, (long long)vocab);
  }
  __syncthreads();
  double p = 0.0;
  if (tid < kNCand) {
    p = s_p[tid] / s_sum;
    s_p[tid] = p;
  }
  __syncthreads();
  // rank by (p desc, id asc); only p > 0 candidates are ranked, zero-probability ids (all
  // non-candidates included) follow in ascending id order
  if (tid < kNCand && p > 0.0) {
    const int my = cand_id(tid);
    int rank = 0;
    for (int c = 0; c < kNCand; ++c) {
      const double q = s_p[c];
      rank += (q > p) || (q == p && cand_id(c) < my);
    }
    s_sorted[rank] = p;
    s_id[rank] = my;
  }
  if (tid == 0) {
    int np_ = 0;
    for (int c = 0; c < kNCand; ++c) np_ += s_p[c] > 0.0;
    s_npos = np_;
  }
  __syncthreads();
  if (tid != 0) return;
  const int npos = s_npos;
  // kept[j]: the j-th entry of the full sorted order
  auto zero_id = [&](int j) -> int {  // j-th smallest id with p == 0 (candidates or not)
    int id = -1;
    for (int k = 0; k <= j; ++k) {
      ++id;
      while (id < vocab) {
        bool pos = false;
        if (id < 256 || id == 257) pos = s_p[id < 256 ? id : 256] > 0.0;
        if (!pos) break;
        ++id;
      }
    }
    return id;
  };
  double csum = 0.0;
  int cut = vocab - 1;
  for (int j = 0; j < vocab; ++j) {
    csum += j < npos ? s_sorted[j] : 0.0;
    if (csum >= top_p) {
      cut = j;
      break;
    }
  }
  const int kept_n = cut + 1;
  auto kval = [&](long long j) -> double { return j < npos ? s_sorted[j] : 0.0; };
  const double ksum = np_pairwise(kval, 0, kept_n);
  const uint64_t* kk = keys + 4 * row;
  const double u = philox_uniform(kk[3], kk[2], kk[0], kk[1]);
  double kcs = 0.0;
  int pick = kept_n - 1;
  for (int j = 0; j < kept_n; ++j) {
    kcs += kval(j) / ksum;
    if (kcs > u) {
      pick = j;
      break;
    }
  }
  out[row] = pick < npos ? s_id[pick] : zero_id(pick - npos);
}

}  // namespace choreo

using namespace choreo;

extern "C" int choreo_select_nucleus(const float* logits, int n_rows, int ld, int vocab,
                                     const double* params, const uint64_t* keys, int32_t* out_tok,
                                     void* stream) {
  if (!logits || !params || !keys || !out_tok || n_rows < 0 || vocab < 258 || ld < vocab)
    return CHOREO_EINVAL;
  if (n_rows == 0) return CHOREO_OK;
  launch_k(select_nucleus_kernel, n_rows, kNucThreads, 0, as_stream(stream), logits, (int64_t)ld,
           vocab, params, keys, out_tok);
  return launch_status("choreo_select_nucleus");
}
