// K3 assemble: prompt assembly on device.
//
// For every call of a step it emits the visible page list — the parents' pages in
// parent order, then the call's own pages up to its last row — and splits each
// row block's prefix of that list into split-KV work items.  This is the page-level
// form of the reference's visibility (masking.py:36-53: a query sees all tokens of
// every parent, plus its own message's tokens with j <= its own j) and of the
// engine's per-call layout (engine.py:203-245, 277, 317).  Because every page holds
// tokens of exactly one message, the visible set of a call is an exact page subset
// plus a causal cut inside the own message; pages of the own message wholly after a
// block's last row are skipped (whole-tile skip).
#include "common.cuh"

namespace choreo {

constexpr int kMaxCalls = 1024;
constexpr int kCallFields = 5;  // msg, par_off, par_cnt, row_off, row_cnt

struct CallPlan {
  int parent_pages;  // pages of all parents
  int vis;           // parent pages + own pages up to the call's last row
  int items;
  int parts;
};

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

__device__ void plan_call(const int32_t* call, const int32_t* call_parents,
                          const int32_t* msg_len, const int32_t* row_t, int P, int rpb, int ppi,
                          CallPlan& cp) {
  const int par_off = call[1], par_cnt = call[2], row_off = call[3], row_cnt = call[4];
  int pp = 0;
  for (int i = 0; i < par_cnt; ++i) pp += cdiv(msg_len[call_parents[par_off + i]], P);
  cp.parent_pages = pp;
  cp.vis = cp.items = cp.parts = 0;
  if (row_cnt <= 0) return;
  cp.vis = pp + row_t[row_off + row_cnt - 1] / P + 1;
  for (int b = 0; b * rpb < row_cnt; ++b) {
    const int nr = min(rpb, row_cnt - b * rpb);
    const int t_hi = row_t[row_off + b * rpb + nr - 1];
    const int chunks = cdiv(pp + t_hi / P + 1, ppi);
    cp.items += chunks;
    cp.parts += chunks * nr;
  }
}

__global__ void assemble_kernel(const int32_t* __restrict__ msg_len,
                                const int32_t* __restrict__ msg_pt, int32_t* __restrict__ page_table,
                                const int32_t* __restrict__ calls,
                                const int32_t* __restrict__ call_parents, int n_calls,
                                const int32_t* __restrict__ row_t, const int32_t* __restrict__ patch,
                                int n_patch, int P, int rpb, int ppi, int32_t* __restrict__ vis_page,
                                int32_t* __restrict__ vis_len, int32_t* __restrict__ vis_own,
                                int32_t* __restrict__ items, int32_t* __restrict__ row_part,
                                int32_t* __restrict__ counts, int cap_pages, int cap_items,
                                int cap_parts) {
  __shared__ CallPlan plan[kMaxCalls];
  __shared__ int base_vis[kMaxCalls], base_item[kMaxCalls], base_part[kMaxCalls];
  __shared__ int overflow;

  for (int i = threadIdx.x; i < n_patch; i += blockDim.x) page_table[patch[2 * i]] = patch[2 * i + 1];
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();

  for (int c = threadIdx.x; c < n_calls; c += blockDim.x)
    plan_call(calls + kCallFields * c, call_parents, msg_len, row_t, P, rpb, ppi, plan[c]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int v = 0, it = 0, pa = 0;
    for (int c = 0; c < n_calls; ++c) {
      base_vis[c] = v;
      base_item[c] = it;
      base_part[c] = pa;
      v += plan[c].vis;
      it += plan[c].items;
      pa += plan[c].parts;
    }
    overflow = (v > cap_pages) || (it > cap_items) || (pa > cap_parts);
    counts[0] = v;
    counts[1] = overflow ? 0 : it;  // an overflowing plan launches no attention work
    counts[2] = pa;
    counts[3] = overflow ? -1 : 0;
  }
  __syncthreads();
  if (overflow) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, n_warps = blockDim.x >> 5;
  for (int c = warp; c < n_calls; c += n_warps) {
    const int32_t* call = calls + kCallFields * c;
    const int own_msg = call[0], par_off = call[1], par_cnt = call[2], row_off = call[3],
              row_cnt = call[4];
    if (row_cnt <= 0) continue;
    // visible page list: parents in order, then own pages
    int w = base_vis[c];
    for (int i = 0; i < par_cnt; ++i) {
      const int p = call_parents[par_off + i];
      const int len = msg_len[p], pt = msg_pt[p], np = cdiv(len, P);
      for (int j = lane; j < np; j += 32) {
        vis_page[w + j] = page_table[pt + j];
        vis_len[w + j] = min(P, len - j * P);
        vis_own[w + j] = -1;
      }
      w += np;
    }
    const int t_max = row_t[row_off + row_cnt - 1];
    const int own_pages = t_max / P + 1, opt = msg_pt[own_msg];
    for (int j = lane; j < own_pages; j += 32) {
      vis_page[w + j] = page_table[opt + j];
      vis_len[w + j] = min(P, t_max + 1 - j * P);
      vis_own[w + j] = j * P;
    }
    // row blocks -> split-KV items; partials of a block are [chunk][row]
    const int pp = plan[c].parent_pages;
    int it = base_item[c], pa = base_part[c];
    const int n_blocks = cdiv(row_cnt, rpb);
    for (int b = 0; b < n_blocks; ++b) {
      const int r0 = row_off + b * rpb, nr = min(rpb, row_cnt - b * rpb);
      const int nvis = pp + row_t[r0 + nr - 1] / P + 1;
      const int chunks = cdiv(nvis, ppi);
      for (int k = lane; k < chunks; k += 32) {
        int32_t* item = items + 6 * (it + k);
        item[0] = r0;
        item[1] = nr;
        item[2] = base_vis[c] + k * ppi;
        item[3] = min(ppi, nvis - k * ppi);
        item[4] = pa + k * nr;
        item[5] = c;
      }
      for (int r = lane; r < nr; r += 32) {
        row_part[3 * (r0 + r)] = pa + r;
        row_part[3 * (r0 + r) + 1] = nr;
        row_part[3 * (r0 + r) + 2] = chunks;
      }
      it += chunks;
      pa += chunks * nr;
    }
  }
}

}  // namespace choreo

using namespace choreo;

extern "C" int choreo_assemble(const int32_t* msg_len, const int32_t* msg_pt, int32_t* page_table,
                               const int32_t* calls, const int32_t* call_parents, int n_calls,
                               const int32_t* row_t, int n_rows, const int32_t* patch,
                               int n_patch, int page_size, int rows_per_block, int pages_per_item,
                               int32_t* vis_page, int32_t* vis_len, int32_t* vis_own,
                               int32_t* items, int32_t* row_part, int32_t* counts,
                               int cap_pages, int cap_items, int cap_parts, void* stream) {
  if (!msg_len || !msg_pt || !page_table || !calls || !row_t || !vis_page || !vis_len ||
      !vis_own || !items || !row_part || !counts)
    return CHOREO_EINVAL;
  if (n_calls < 0 || n_calls > kMaxCalls || n_rows < 0 || page_size <= 0 ||
      rows_per_block <= 0 || pages_per_item <= 0 || (n_patch > 0 && !patch))
    return CHOREO_EINVAL;
  assemble_kernel<<<1, 256, 0, as_stream(stream)>>>(
      msg_len, msg_pt, page_table, calls, call_parents, n_calls, row_t, patch, n_patch,
      page_size, rows_per_block, pages_per_item, vis_page, vis_len, vis_own, items, row_part,
      counts, cap_pages, cap_items, cap_parts);
  return launch_status("choreo_assemble");
}
