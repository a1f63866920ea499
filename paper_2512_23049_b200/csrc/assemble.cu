// K3 assemble: prompt assembly on device, page-centric.
//
// A step encodes new-token rows for several calls (messages).  The reference's
// visibility (masking.py:36-53) says a row of call c sees every token of every
// parent of c, plus the tokens of its own message up to its own j.  Since each
// page holds tokens of one message, that is an exact page subset plus a causal
// cut inside the own pages.  This kernel turns the step's calls into split-KV
// work items that read each parent message ONCE per step for all the rows that
// can see it (agents of a parallel decode share most parents):
//
//   group  = one distinct parent message p and its viewers (the rows of every call
//            that lists p), split into blocks of <= rows_per_block rows;
//   own    = one call's rows against its own pages (causal), same blocking;
//   item   = (row block, run of <= pages_per_item pages of the group's / own list).
//
// Outputs: the visible page lists (each distinct parent's pages once, then each
// call's own pages up to its last row), the row list of every block, the items,
// and per row the list of partial-result slots the combine step merges.
// Single CTA: steps have at most a few thousand (parent, call) pairs.
#include "common.cuh"

namespace choreo {

constexpr int kMaxCalls = 1024;
constexpr int kMaxPairs = 4096;
constexpr int kCallFields = 5;  // msg, par_off, par_cnt, row_off, row_cnt
constexpr int kThreads3 = 512;

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

struct K3Params {
  const int32_t* msg_len;
  const int32_t* msg_pt;
  int32_t* page_table;
  const int32_t* calls;
  const int32_t* call_parents;
  int n_calls;
  const int32_t* row_t;
  int n_rows;
  const int32_t* patch;
  int n_patch;
  int P, rpb, ppi;
  int32_t* vis_page;
  int32_t* vis_len;
  int32_t* vis_own;
  int32_t* blk_rows;
  int32_t* items;
  int32_t* row_part_off;  // [n_rows + 1]
  int32_t* row_part;      // partial slots, CSR by row
  int32_t* counts;
  int cap_vis, cap_blk_rows, cap_items, cap_parts;
  int32_t* fat;  // optional self-contained item records (kFatInts each), see write_fat
  int32_t* order;  // optional: item indices by page count, descending (stable), see order_items
  int tag;         // != 0: counts[4] = tag once every output is written (mode 0), see stamp
};

// counts[4..5] = {tag, n_items} (one 64-bit release store) after every output of the step
// is written and visible device-wide: a later kernel that finds its step's tag there may
// read the (step-static) K3 outputs before its programmatic-dependency wait (K5 v2 does, to
// overlap its first lookups), the item count coming with the tag in one round trip.
__device__ void stamp(const K3Params& p) {
  if (!p.tag) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t v = ((uint64_t)(uint32_t)p.counts[1] << 32) | (uint32_t)p.tag;
    asm volatile("st.release.gpu.global.b64 [%0], %1;\n" ::"l"(p.counts + 4), "l"(v) : "memory");
  }
}

// Self-contained item record for the latency-bound decode kernel: one 256-byte load gives
// a CTA everything it needs (no dependent lookups of rows, row_t or page descriptors).
//   [0] n_rows  [1] n_pages  [2] partial base  [3] first vis index
//   [4..19] row ids   [20..35] row_t   [36..43] page  [44..51] page_len  [52..59] own_base
// Requires n_rows <= kFatRows and n_pages <= kFatPages (the host sizes items that way).
constexpr int kFatInts = 64, kFatRows = 16, kFatPages = 8;

__device__ void write_fat(const K3Params& p, int n_items) {
  for (int i = threadIdx.x; i < n_items; i += blockDim.x) {
    const int32_t* it = p.items + 6 * i;
    int32_t* f = p.fat + kFatInts * i;
    const int nr = min(it[1], kFatRows), nv = min(it[3], kFatPages);
    f[0] = nr;
    f[1] = nv;
    f[2] = it[4];
    f[3] = it[2];  // first vis index (K5 v2's loader reads the page lengths from there)
    for (int r = 0; r < kFatRows; ++r) {
      const int rid = r < nr ? p.blk_rows[it[0] + r] : 0;
      f[4 + r] = rid;
      f[20 + r] = r < nr ? p.row_t[rid] : -1;
    }
    for (int k = 0; k < kFatPages; ++k) {
      const bool ok = k < nv;
      f[36 + k] = ok ? p.vis_page[it[2] + k] : 0;
      f[44 + k] = ok ? p.vis_len[it[2] + k] : 0;
      f[52 + k] = ok ? p.vis_own[it[2] + k] : -1;
    }
  }
}

// Item indices sorted by page count, descending, ties in item order (a stable counting sort
// over the 32 possible counts).  K5 v2 deals the (item, kv head) units of a multi-wave step
// to its persistent CTAs in this order, snaking across the grid (longest-first), so no CTA
// is left with several long units while others idle.  Only the schedule changes: every
// unit writes the same partial slots, so the results are bitwise independent of the order.
__device__ void order_items(const int32_t* items, int n, int32_t* order) {
  __shared__ int start[32];
  __shared__ int wcnt[kThreads3 / 32][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  auto key = [&](int i) { return 32 - min(max(items[6 * i + 3], 1), 32); };  // 0: longest
  if (tid < 32) start[tid] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) atomicAdd(&start[key(i)], 1);
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int k = 0; k < 32; ++k) {
      const int c = start[k];
      start[k] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + tid;
    const int k = i < n ? key(i) : -1;
    wcnt[warp][lane] = 0;
    __syncwarp();
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (k >= 0 && rank == 0) wcnt[warp][k] = __popc(peers);
    __syncthreads();
    if (k >= 0) {
      int o = start[k] + rank;
      for (int w = 0; w < warp; ++w) o += wcnt[w][k];
      order[o] = i;
    }
    __syncthreads();
    if (tid < 32) {
      int t = 0;
      for (int w = 0; w < nw; ++w) t += wcnt[w][tid];
      start[tid] += t;
    }
    __syncthreads();
  }
}

// smem-resident plan
struct Shared {
  uint32_t key[kMaxPairs];  // (parent << 11 | call) sorted
  int n_pairs;
  int n_groups;
  int g_first[kMaxPairs + 1];  // first pair index of group g
  int g_vis[kMaxPairs], g_rows[kMaxPairs], g_item[kMaxPairs], g_part[kMaxPairs];
  int c_vis[kMaxCalls], c_rows[kMaxCalls], c_item[kMaxCalls], c_part[kMaxCalls];
  int tot_vis, tot_rows, tot_items, tot_parts, overflow;
};

__global__ void __launch_bounds__(kThreads3) assemble_kernel(K3Params p) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ unsigned char smem_raw[];
  Shared& S = *reinterpret_cast<Shared*>(smem_raw);
  const int tid = threadIdx.x;
  for (int i = tid; i < p.n_patch; i += blockDim.x) p.page_table[p.patch[2 * i]] = p.patch[2 * i + 1];
  // ---- (parent, call) pairs, sorted by parent then call ----
  if (tid == 0) {
    int n = 0;
    for (int c = 0; c < p.n_calls; ++c) n += p.calls[kCallFields * c + 2];
    S.n_pairs = n;
    S.overflow = n > kMaxPairs;
  }
  __syncthreads();
  if (S.overflow) {
    if (tid == 0) { p.counts[1] = 0; p.counts[3] = -2; }
    return;
  }
  const int NP = S.n_pairs;
  for (int c = tid; c < p.n_calls; c += blockDim.x) {
    const int32_t* cl = p.calls + kCallFields * c;
    for (int i = 0; i < cl[2]; ++i)
      S.key[cl[1] + i] = ((uint32_t)p.call_parents[cl[1] + i] << 11) | (uint32_t)c;
  }
  int np2 = 1;
  while (np2 < NP) np2 <<= 1;
  for (int i = NP + tid; i < np2; i += blockDim.x) S.key[i] = 0xffffffffu;
  __syncthreads();
  for (int k = 2; k <= np2; k <<= 1)  // bitonic sort
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < np2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t a = S.key[i], b = S.key[l];
          if (((i & k) == 0) == (a > b)) { S.key[i] = b; S.key[l] = a; }
        }
      }
      __syncthreads();
    }
  // ---- groups and per-group / per-call sizes ----
  if (tid == 0) {
    int g = 0;
    for (int i = 0; i < NP; ++i)
      if (i == 0 || (S.key[i] >> 11) != (S.key[i - 1] >> 11)) S.g_first[g++] = i;
    S.g_first[g] = NP;
    S.n_groups = g;
  }
  __syncthreads();
  const int NG = S.n_groups;
  for (int g = tid; g < NG; g += blockDim.x) {
    const int msg = S.key[S.g_first[g]] >> 11;
    int rows = 0;
    for (int i = S.g_first[g]; i < S.g_first[g + 1]; ++i) rows += p.calls[kCallFields * (S.key[i] & 2047) + 4];
    const int pages = cdiv(p.msg_len[msg], p.P);
    const int chunks = cdiv(pages, p.ppi);
    S.g_vis[g] = pages;
    S.g_rows[g] = rows;
    S.g_item[g] = rows ? cdiv(rows, p.rpb) * chunks : 0;
    S.g_part[g] = rows ? chunks * rows : 0;
  }
  for (int c = tid; c < p.n_calls; c += blockDim.x) {
    const int32_t* cl = p.calls + kCallFields * c;
    const int row_off = cl[3], row_cnt = cl[4];
    S.c_vis[c] = S.c_rows[c] = S.c_item[c] = S.c_part[c] = 0;
    if (row_cnt <= 0) continue;
    S.c_vis[c] = p.row_t[row_off + row_cnt - 1] / p.P + 1;
    S.c_rows[c] = row_cnt;
    for (int b = 0; b * p.rpb < row_cnt; ++b) {
      const int nr = min(p.rpb, row_cnt - b * p.rpb);
      const int ch = cdiv(p.row_t[row_off + b * p.rpb + nr - 1] / p.P + 1, p.ppi);
      S.c_item[c] += ch;
      S.c_part[c] += ch * nr;
    }
  }
  __syncthreads();
  // ---- exclusive scans (serial: groups + calls are small) ----
  if (tid == 0) {
    int v = 0, r = 0, it = 0, pa = 0;
    for (int g = 0; g < NG; ++g) {
      int t;
      t = S.g_vis[g]; S.g_vis[g] = v; v += t;
      t = S.g_rows[g]; S.g_rows[g] = r; r += t;
      t = S.g_item[g]; S.g_item[g] = it; it += t;
      t = S.g_part[g]; S.g_part[g] = pa; pa += t;
    }
    for (int c = 0; c < p.n_calls; ++c) {
      int t;
      t = S.c_vis[c]; S.c_vis[c] = v; v += t;
      t = S.c_rows[c]; S.c_rows[c] = r; r += t;
      t = S.c_item[c]; S.c_item[c] = it; it += t;
      t = S.c_part[c]; S.c_part[c] = pa; pa += t;
    }
    S.tot_vis = v; S.tot_rows = r; S.tot_items = it; S.tot_parts = pa;
    S.overflow = v > p.cap_vis || r > p.cap_blk_rows || it > p.cap_items || pa > p.cap_parts;
    p.counts[0] = v;
    p.counts[1] = S.overflow ? 0 : it;
    p.counts[2] = pa;
    p.counts[3] = S.overflow ? -1 : 0;
  }
  __syncthreads();
  if (S.overflow) return;
  // ---- per-row partial counts -> CSR offsets ----
  // row r of call c: sum over parents p of chunks(p) + own chunks of its block
  for (int c = tid; c < p.n_calls; c += blockDim.x) {
    const int32_t* cl = p.calls + kCallFields * c;
    int par_chunks = 0;
    for (int i = 0; i < cl[2]; ++i) par_chunks += cdiv(cdiv(p.msg_len[p.call_parents[cl[1] + i]], p.P), p.ppi);
    for (int b = 0; b * p.rpb < cl[4]; ++b) {
      const int nr = min(p.rpb, cl[4] - b * p.rpb);
      const int ch = cdiv(p.row_t[cl[3] + b * p.rpb + nr - 1] / p.P + 1, p.ppi);
      for (int j = 0; j < nr; ++j) p.row_part_off[cl[3] + b * p.rpb + j + 1] = par_chunks + ch;
    }
  }
  __syncthreads();
  if (tid == 0) {
    p.row_part_off[0] = 0;
    for (int r = 0; r < p.n_rows; ++r) p.row_part_off[r + 1] += p.row_part_off[r];
  }
  __syncthreads();
  // fill cursor per row: reuse g_* / c_* are still needed; keep a per-row running
  // position in the row_part array by walking groups in order (one warp per call
  // would race), so groups are filled serially per row below.
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  // ---- groups: pages, block rows, items, partial slots ----
  for (int g = warp; g < NG; g += nw) {
    const int msg = S.key[S.g_first[g]] >> 11;
    const int len = p.msg_len[msg], pt = p.msg_pt[msg], pages = cdiv(len, p.P);
    const int vb = S.g_vis[g];
    for (int j = lane; j < pages; j += 32) {
      p.vis_page[vb + j] = p.page_table[pt + j];
      p.vis_len[vb + j] = min(p.P, len - j * p.P);
      p.vis_own[vb + j] = -1;
    }
    // block rows: concatenated row ranges of the viewer calls (ascending call)
    int rb = S.g_rows[g], w = 0;
    for (int i = S.g_first[g]; i < S.g_first[g + 1]; ++i) {
      const int32_t* cl = p.calls + kCallFields * (S.key[i] & 2047);
      for (int j = lane; j < cl[4]; j += 32) p.blk_rows[rb + w + j] = cl[3] + j;
      w += cl[4];
    }
    const int rows = w, chunks = cdiv(pages, p.ppi), nb = cdiv(rows, p.rpb);
    for (int k = lane; k < nb * chunks; k += 32) {
      const int b = k / chunks, ch = k % chunks;
      const int nr = min(p.rpb, rows - b * p.rpb);
      int32_t* it = p.items + 6 * (S.g_item[g] + k);
      it[0] = rb + b * p.rpb;
      it[1] = nr;
      it[2] = vb + ch * p.ppi;
      it[3] = min(p.ppi, pages - ch * p.ppi);
      it[4] = S.g_part[g] + ch * rows + b * p.rpb;
      it[5] = g;
    }
  }
  // ---- own pages, rows, items ----
  for (int c = warp; c < p.n_calls; c += nw) {
    const int32_t* cl = p.calls + kCallFields * c;
    const int row_off = cl[3], row_cnt = cl[4];
    if (row_cnt <= 0) continue;
    const int t_max = p.row_t[row_off + row_cnt - 1];
    const int own_pages = t_max / p.P + 1, opt = p.msg_pt[cl[0]], vb = S.c_vis[c];
    for (int j = lane; j < own_pages; j += 32) {
      p.vis_page[vb + j] = p.page_table[opt + j];
      p.vis_len[vb + j] = min(p.P, t_max + 1 - j * p.P);
      p.vis_own[vb + j] = j * p.P;
    }
    const int rb = S.c_rows[c];
    for (int j = lane; j < row_cnt; j += 32) p.blk_rows[rb + j] = row_off + j;
    if (lane == 0) {
      int it = S.c_item[c], pa = S.c_part[c];
      for (int b = 0; b * p.rpb < row_cnt; ++b) {
        const int nr = min(p.rpb, row_cnt - b * p.rpb);
        const int nvis = p.row_t[row_off + b * p.rpb + nr - 1] / p.P + 1;
        const int chunks = cdiv(nvis, p.ppi);
        for (int ch = 0; ch < chunks; ++ch) {
          int32_t* item = p.items + 6 * (it + ch);
          item[0] = rb + b * p.rpb;
          item[1] = nr;
          item[2] = vb + ch * p.ppi;
          item[3] = min(p.ppi, nvis - ch * p.ppi);
          item[4] = pa + ch * nr;
          item[5] = -1 - c;
        }
        it += chunks;
        pa += chunks * nr;
      }
    }
  }
  __syncthreads();
  // ---- per-row partial slot lists (CSR) ----
  // Row r (call c, local index j in its call) gets, in order: for each group g
  // viewing c (ascending parent id) its chunks' slots, then its own chunks' slots.
  for (int c = warp; c < p.n_calls; c += nw) {
    const int32_t* cl = p.calls + kCallFields * c;
    const int row_off = cl[3], row_cnt = cl[4];
    for (int j = lane; j < row_cnt; j += 32) {
      const int r = row_off + j;
      int w = p.row_part_off[r];
      for (int g = 0; g < NG; ++g) {
        // is call c a viewer of group g, and at which row index within the group?
        int base = 0, found = -1;
        for (int i = S.g_first[g]; i < S.g_first[g + 1]; ++i) {
          const int cc = S.key[i] & 2047;
          if (cc == c) { found = base; break; }
          base += p.calls[kCallFields * cc + 4];
        }
        if (found < 0) continue;
        const int msg = S.key[S.g_first[g]] >> 11;
        const int chunks = cdiv(cdiv(p.msg_len[msg], p.P), p.ppi);
        const int rows_g = (g + 1 < NG ? S.g_rows[g + 1] : S.c_rows[0]) - S.g_rows[g];
        for (int ch = 0; ch < chunks; ++ch) p.row_part[w++] = S.g_part[g] + ch * rows_g + found + j;
      }
      const int b = j / p.rpb, nr = min(p.rpb, row_cnt - b * p.rpb);
      int pa = S.c_part[c];
      for (int bb = 0; bb < b; ++bb) {
        const int nrb = min(p.rpb, row_cnt - bb * p.rpb);
        pa += cdiv(p.row_t[row_off + bb * p.rpb + nrb - 1] / p.P + 1, p.ppi) * nrb;
      }
      const int chunks = cdiv(p.row_t[row_off + b * p.rpb + nr - 1] / p.P + 1, p.ppi);
      for (int ch = 0; ch < chunks; ++ch) p.row_part[w++] = pa + ch * nr + (j - b * p.rpb);
    }
  }
  if (p.fat) {
    __syncthreads();
    write_fat(p, S.tot_items);
  }
  if (p.order) {
    __syncthreads();
    order_items(p.items, S.tot_items, p.order);
  }
  stamp(p);
}

// Per-call mode (prefill-sized steps): each call's visible list is its parents' pages
// in parent order followed by its own pages up to its last row; a row block's items are
// chunks of that list (pages past the block's last row are skipped).  A 128-row M tile
// already comes from one call here, so sharing pages across calls would not enlarge it.
__global__ void __launch_bounds__(kThreads3) assemble_percall_kernel(K3Params p) {
  pdl_trigger();
  pdl_wait();
  __shared__ int c_pp[kMaxCalls], c_vis[kMaxCalls], c_rows[kMaxCalls], c_item[kMaxCalls],
      c_part[kMaxCalls];
  __shared__ int overflow;
  const int tid = threadIdx.x;
  for (int i = tid; i < p.n_patch; i += blockDim.x) p.page_table[p.patch[2 * i]] = p.patch[2 * i + 1];
  __syncthreads();
  for (int c = tid; c < p.n_calls; c += blockDim.x) {
    const int32_t* cl = p.calls + kCallFields * c;
    int pp = 0;
    for (int i = 0; i < cl[2]; ++i) pp += cdiv(p.msg_len[p.call_parents[cl[1] + i]], p.P);
    c_pp[c] = pp;
    c_vis[c] = c_rows[c] = c_item[c] = c_part[c] = 0;
    if (cl[4] <= 0) continue;
    c_vis[c] = pp + p.row_t[cl[3] + cl[4] - 1] / p.P + 1;
    c_rows[c] = cl[4];
    for (int b = 0; b * p.rpb < cl[4]; ++b) {
      const int nr = min(p.rpb, cl[4] - b * p.rpb);
      const int ch = cdiv(pp + p.row_t[cl[3] + b * p.rpb + nr - 1] / p.P + 1, p.ppi);
      c_item[c] += ch;
      c_part[c] += ch * nr;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int v = 0, r = 0, it = 0, pa = 0;
    for (int c = 0; c < p.n_calls; ++c) {
      int t;
      t = c_vis[c]; c_vis[c] = v; v += t;
      t = c_rows[c]; c_rows[c] = r; r += t;
      t = c_item[c]; c_item[c] = it; it += t;
      t = c_part[c]; c_part[c] = pa; pa += t;
    }
    overflow = v > p.cap_vis || r > p.cap_blk_rows || it > p.cap_items || pa > p.cap_parts;
    p.counts[0] = v;
    p.counts[1] = overflow ? 0 : it;
    p.counts[2] = pa;
    p.counts[3] = overflow ? -1 : 0;
    p.row_part_off[p.n_rows] = pa;
  }
  __syncthreads();
  if (overflow) return;
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < p.n_calls; c += nw) {
    const int32_t* cl = p.calls + kCallFields * c;
    const int row_off = cl[3], row_cnt = cl[4];
    if (row_cnt <= 0) continue;
    int w = c_vis[c];
    for (int i = 0; i < cl[2]; ++i) {
      const int msg = p.call_parents[cl[1] + i];
      const int len = p.msg_len[msg], pt = p.msg_pt[msg], np = cdiv(len, p.P);
      for (int j = lane; j < np; j += 32) {
        p.vis_page[w + j] = p.page_table[pt + j];
        p.vis_len[w + j] = min(p.P, len - j * p.P);
        p.vis_own[w + j] = -1;
      }
      w += np;
    }
    const int t_max = p.row_t[row_off + row_cnt - 1];
    const int opt = p.msg_pt[cl[0]];
    for (int j = lane; j <= t_max / p.P; j += 32) {
      p.vis_page[w + j] = p.page_table[opt + j];
      p.vis_len[w + j] = min(p.P, t_max + 1 - j * p.P);
      p.vis_own[w + j] = j * p.P;
    }
    const int rb = c_rows[c];
    for (int j = lane; j < row_cnt; j += 32) p.blk_rows[rb + j] = row_off + j;
    int it = c_item[c], pa = c_part[c];
    for (int b = 0; b * p.rpb < row_cnt; ++b) {
      const int nr = min(p.rpb, row_cnt - b * p.rpb);
      const int nvis = c_pp[c] + p.row_t[row_off + b * p.rpb + nr - 1] / p.P + 1;
      const int chunks = cdiv(nvis, p.ppi);
      for (int k = lane; k < chunks; k += 32) {
        int32_t* item = p.items + 6 * (it + k);
        item[0] = rb + b * p.rpb;
        item[1] = nr;
        item[2] = c_vis[c] + k * p.ppi;
        item[3] = min(p.ppi, nvis - k * p.ppi);
        item[4] = pa + k * nr;
        item[5] = -1 - c;
      }
      // rows are contiguous per call and calls are in order, so row r's CSR entries
      // start at this block's partial base + j * chunks
      for (int j = lane; j < nr; j += 32) {
        const int r = row_off + b * p.rpb + j;
        const int o = pa + j * chunks;
        p.row_part_off[r] = o;
        for (int k = 0; k < chunks; ++k) p.row_part[o + k] = pa + k * nr + j;
      }
      it += chunks;
      pa += chunks * nr;
    }
  }
  if (p.fat) {
    __syncthreads();
    write_fat(p, p.counts[1]);
  }
  if (p.order) {
    __syncthreads();
    order_items(p.items, p.counts[1], p.order);
  }
}

}  // namespace choreo

using namespace choreo;

extern "C" int choreo_assemble_ex(const int32_t* msg_len, const int32_t* msg_pt, int32_t* page_table,
                               const int32_t* calls, const int32_t* call_parents, int n_calls,
                               const int32_t* row_t, int n_rows, const int32_t* patch,
                               int n_patch, int page_size, int rows_per_block, int pages_per_item,
                               int32_t* vis_page, int32_t* vis_len, int32_t* vis_own,
                               int32_t* blk_rows, int32_t* items, int32_t* row_part_off,
                               int32_t* row_part, int32_t* counts, int cap_vis, int cap_blk_rows,
                               int cap_items, int cap_parts, int mode, int32_t* fat, int32_t* item_order,
                               int step_tag, void* stream) {
  if (!msg_len || !msg_pt || !page_table || !calls || !row_t || !vis_page || !vis_len ||
      !vis_own || !blk_rows || !items || !row_part_off || !row_part || !counts)
    return CHOREO_EINVAL;
  if (n_calls < 0 || n_calls > kMaxCalls || n_rows < 0 || page_size <= 0 ||
      rows_per_block <= 0 || pages_per_item <= 0 || (n_patch > 0 && !patch))
    return CHOREO_EINVAL;
  K3Params p{msg_len, msg_pt, page_table, calls, call_parents, n_calls, row_t, n_rows, patch,
             n_patch, page_size, rows_per_block, pages_per_item, vis_page, vis_len, vis_own,
             blk_rows, items, row_part_off, row_part, counts, cap_vis, cap_blk_rows, cap_items,
             cap_parts, fat, item_order, mode == 0 ? step_tag : 0};
  if (mode == 1) {
    launch_k(assemble_percall_kernel, 1, kThreads3, 0, as_stream(stream), p);
    return launch_status("choreo_assemble");
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(Shared));
    attr = true;
  }
  launch_k(assemble_kernel, 1, kThreads3, sizeof(Shared), as_stream(stream), p);
  return launch_status("choreo_assemble");
}

extern "C" int choreo_assemble(const int32_t* msg_len, const int32_t* msg_pt, int32_t* page_table,
                               const int32_t* calls, const int32_t* call_parents, int n_calls,
                               const int32_t* row_t, int n_rows, const int32_t* patch,
                               int n_patch, int page_size, int rows_per_block, int pages_per_item,
                               int32_t* vis_page, int32_t* vis_len, int32_t* vis_own,
                               int32_t* blk_rows, int32_t* items, int32_t* row_part_off,
                               int32_t* row_part, int32_t* counts, int cap_vis, int cap_blk_rows,
                               int cap_items, int cap_parts, int mode, int32_t* fat,
                               void* stream) {
  return choreo_assemble_ex(msg_len, msg_pt, page_table, calls, call_parents, n_calls, row_t,
                            n_rows, patch, n_patch, page_size, rows_per_block, pages_per_item,
                            vis_page, vis_len, vis_own, blk_rows, items, row_part_off, row_part,
                            counts, cap_vis, cap_blk_rows, cap_items, cap_parts, mode, fat,
                            nullptr, 0, stream);
}
