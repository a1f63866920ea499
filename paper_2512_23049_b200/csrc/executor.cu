// Native decode-step executor: the per-layer launch sequence of a decode-sized step
// (reference model.py:169-189, run for every layer) issued from C++ in one call, so a
// decode step costs one host->library crossing instead of ~11 Python launches per layer.
//
// Per layer, on `stream`:
//   residual_rmsnorm (x += delta; h = norm(x) as hi/lo bf16)
//   K7 qkv = h @ Wqkv^T                 (weights streamed; PDL prefetch under the norm;
//                                        cut tiles left as pieces for RoPE, ChoreoK7Pieces)
//   K1 rope_append (q rotated to f32, K/V written into the message pages)
//   K5 v2 decode attention over the K3 page-centric items (+ LSE combine)
//   K7 ao = attn @ Wo^T
//   residual_rmsnorm (x += ao; h = norm(x))
//   K7 act = silu(h @ Wg^T) * (h @ Wu^T) (SwiGLU in the epilogue) ; K7 delta = act @ Wdown^T
// The final residual add, norm and head stay with the caller (they depend on which rows
// need logits).  Every kernel is one of the library's C-ABI entry points, so results are
// bit-identical to the Python-driven sequence.
#include <math.h>

#include "common.cuh"

using namespace choreo;

static bool k7_defer_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CHOREO_K7_DEFER");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

extern "C" int choreo_decode_layers(const ChoreoDecodeStep* s, void* stream) {
  if (!s || !s->attn_norm || !s->w_qkv || !s->wo || !s->ffn_norm || !s->w_gu || !s->w_down ||
      s->n_layers <= 0 || s->n_rows <= 0)
    return CHOREO_EINVAL;
  const int R = s->n_rows, sp = s->split, d = s->d, H = s->n_heads, Hk = s->n_kv;
  const int hd = s->head_dim, F = s->ffn_dim;
  const int x_rows = sp ? 2 * R : R;
  const int n_qkv = (H + 2 * Hk) * hd;
  cudaEvent_t* ev = reinterpret_cast<cudaEvent_t*>(s->attn_events);
  cudaEvent_t* lev = reinterpret_cast<cudaEvent_t*>(s->linear_events);
  cudaStream_t cs = as_stream(stream);
#define LIN_EV(i) \
  if (lev) cudaEventRecord(lev[8 * l + (i)], cs)
  int rc;
#define CHK(call)          \
  do {                     \
    rc = (call);           \
    if (rc != 0) return rc; \
  } while (0)
  const int l0 = s->layer_begin, l1 = s->layer_end > 0 ? s->layer_end : s->n_layers;
  if (l0 < 0 || l1 > s->n_layers || l0 >= l1 || s->part < 0 || s->part > 2) return CHOREO_EINVAL;
  // K7 outputs consumed inside this call are left deferred (ChoreoK7Pieces): the consumer
  // (RoPE / residual+norm) sums the cut tiles, the GEMM skips its cross-CTA fix-up.  Outputs
  // the caller reads (the last down_proj, the TP halves' o_proj / down_proj) are reduced.
  if (s->chain_ws && s->part == 0 && l0 == 0 && l1 == s->n_layers) {
    // K8 path: prologue, qkv(0), then per layer attention + combine + one chain launch
    if (!s->h_b || !s->ssq_a || !s->ssq_b || !s->chain_counters || !s->chain_done)
      return CHOREO_EINVAL;
    cudaEvent_t* cev = reinterpret_cast<cudaEvent_t*>(s->chain_events);
    ChoreoLayerChain c{};
    c.n_rows = R;
    c.split = sp;
    c.d = d;
    c.n_heads = H;
    c.n_kv = Hk;
    c.head_dim = hd;
    c.ffn_dim = F;
    c.eps = s->eps;
    c.x = s->x;
    c.attn = s->attn;
    c.h_a = s->h;
    c.act = s->act;
    c.h_b = s->h_b;
    c.ssq_a = s->ssq_a;
    c.ssq_b = s->ssq_b;
    c.q = s->q;
    c.k_pool = s->k_pool;
    c.v_pool = s->v_pool;
    c.n_pages = s->n_pages;
    c.page_size = s->page_size;
    c.pos = s->pos;
    c.page = s->page;
    c.slot = s->slot;
    c.cos_t = s->cos_t;
    c.sin_t = s->sin_t;
    c.max_delta = s->max_delta;
    c.ws = s->chain_ws;
    c.counters = s->chain_counters;
    c.done = s->chain_done;
    CHK(choreo_chain_prologue(s->x, s->delta_in, R, d, s->attn_norm[0], s->h_b, sp, s->ssq_b,
                              stream));
    c.phases = 8;
    c.w_qkv = s->w_qkv[0];
    c.layer_qkv = 0;
    if (cev) cudaEventRecord(cev[0], cs);
    CHK(choreo_layer_chain(&c, stream));
    if (cev) cudaEventRecord(cev[1], cs);
    for (int l = 0; l < s->n_layers; ++l) {
      if (ev) cudaEventRecord(ev[2 * l], cs);
      CHK(choreo_decode_attn_v2(s->q, s->k_pool, s->v_pool, s->n_layers, l, Hk, s->n_pages,
                                s->page_size, H, hd, s->row_t, s->vis_page, s->vis_len,
                                s->vis_own, s->blk_rows, s->items, s->counts, s->n_items,
                                s->part_o, s->part_lse, s->fat, 0, stream));
      if (ev) cudaEventRecord(ev[2 * l + 1], cs);
      CHK(choreo_attn_combine(s->part_o, s->part_lse, s->row_part_off, s->row_part, R, H, hd,
                              s->attn, CHOREO_BF16, sp, stream));
      const bool more = l + 1 < s->n_layers;
      c.phases = 1 | 2 | 4 | (more ? 8 : 0);
      c.wo = s->wo[l];
      c.ffn_norm = s->ffn_norm[l];
      c.w_gu = s->w_gu[l];
      c.w_down = s->w_down[l];
      c.attn_norm_next = more ? s->attn_norm[l + 1] : nullptr;
      c.w_qkv = more ? s->w_qkv[l + 1] : nullptr;
      c.layer_qkv = l + 1;
      if (cev) cudaEventRecord(cev[2 * (l + 1)], cs);
      CHK(choreo_layer_chain(&c, stream));
      if (cev) cudaEventRecord(cev[2 * (l + 1) + 1], cs);
    }
    return CHOREO_OK;
  }
  const bool defer = k7_defer_enabled();
  ChoreoK7Pieces pk{}, po{}, pd{};
  bool pd_valid = false;
  for (int l = l0; l < l1; ++l) {
   if (s->part != 2) {
    // delta: previous layer's down_proj output (K7 output, hi/lo already summed)
    if (pd_valid && l > l0)
      CHK(choreo_residual_rmsnorm_pieces(s->x, &pd, s->attn_norm[l], CHOREO_BF16, R, d, s->eps,
                                         s->h, CHOREO_BF16, sp, stream));
    else
      CHK(choreo_residual_rmsnorm(s->x, l > l0 ? s->delta : s->delta_in, CHOREO_F32, 0,
                                  s->attn_norm[l], CHOREO_BF16, R, d, s->eps, s->h, CHOREO_BF16,
                                  sp, nullptr, 0, stream));
    pd_valid = false;
    LIN_EV(0);
    if (defer) {
      CHK(choreo_linear_skinny_pieces(s->h, x_rows, sp, s->w_qkv[l], n_qkv, d, s->qkv, s->k7_ws,
                                      s->k7_cnt, 0, &pk, stream));
      LIN_EV(1);
      CHK(choreo_rope_append_pieces_ex(&pk, R, s->pos, s->page, s->slot, s->q, s->k_pool,
                                       s->v_pool, CHOREO_BF16, l, Hk, s->n_pages, s->page_size, H,
                                       hd, s->cos_t, s->sin_t, s->max_delta, s->q_k5,
                                       1.4426950408889634f / sqrtf((float)hd), stream));
    } else {
      CHK(choreo_linear_skinny(s->h, x_rows, sp, s->w_qkv[l], n_qkv, d, s->qkv, s->k7_ws,
                               s->k7_cnt, 0, stream));
      LIN_EV(1);
      CHK(choreo_rope_append(s->qkv, CHOREO_F32, n_qkv, R, 0, s->pos, s->page, s->slot, s->q,
                             s->k_pool, s->v_pool, CHOREO_BF16, l, Hk, s->n_pages, s->page_size,
                             H, hd, s->cos_t, s->sin_t, s->max_delta, stream));
    }
    if (ev) cudaEventRecord(ev[2 * l], as_stream(stream));
    CHK(choreo_decode_attn_v2_ex(s->q, s->k_pool, s->v_pool, s->n_layers, l, Hk, s->n_pages,
                                 s->page_size, H, hd, s->row_t, s->vis_page, s->vis_len,
                                 s->vis_own, s->blk_rows, s->items, s->counts, s->n_items,
                                 s->part_o, s->part_lse, s->fat, 0,
                                 defer ? s->q_k5 : nullptr, s->item_order, s->k3_tag, stream));
    if (ev) cudaEventRecord(ev[2 * l + 1], as_stream(stream));
    CHK(choreo_attn_combine(s->part_o, s->part_lse, s->row_part_off, s->row_part, R, H, hd,
                            s->attn, CHOREO_BF16, sp, stream));
    LIN_EV(2);
    if (defer && s->part == 0)
      CHK(choreo_linear_skinny_pieces(s->attn, x_rows, sp, s->wo[l], d, H * hd, s->ao, s->k7_ws,
                                      s->k7_cnt, 0, &po, stream));
    else
      CHK(choreo_linear_skinny(s->attn, x_rows, sp, s->wo[l], d, H * hd, s->ao, s->k7_ws,
                               s->k7_cnt, 0, stream));
    LIN_EV(3);
   }
   if (s->part != 1) {
    if (defer && s->part == 0)
      CHK(choreo_residual_rmsnorm_pieces(s->x, &po, s->ffn_norm[l], CHOREO_BF16, R, d, s->eps,
                                         s->h, CHOREO_BF16, sp, stream));
    else
      CHK(choreo_residual_rmsnorm(s->x, s->ao, CHOREO_F32, 0, s->ffn_norm[l], CHOREO_BF16, R, d,
                                  s->eps, s->h, CHOREO_BF16, sp, nullptr, 0, stream));
    LIN_EV(4);
    if (F % 64 == 0) {
      CHK(choreo_linear_gate_up_silu(s->h, x_rows, sp, s->w_gu[l], F, d, s->act, s->k7_ws,
                                     s->k7_cnt, stream));
    } else {
      CHK(choreo_linear_skinny(s->h, x_rows, sp, s->w_gu[l], 2 * F, d, s->gu, s->k7_ws,
                               s->k7_cnt, 0, stream));
      CHK(choreo_silu_mul(s->gu, CHOREO_F32, 0, R, F, s->act, CHOREO_BF16, sp, stream));
    }
    LIN_EV(5);
    LIN_EV(6);
    if (defer && s->part == 0 && l < l1 - 1) {
      CHK(choreo_linear_skinny_pieces(s->act, x_rows, sp, s->w_down[l], d, F, s->delta,
                                      s->k7_ws, s->k7_cnt, 0, &pd, stream));
      pd_valid = true;
    } else {
      CHK(choreo_linear_skinny(s->act, x_rows, sp, s->w_down[l], d, F, s->delta, s->k7_ws,
                               s->k7_cnt, 0, stream));
    }
    LIN_EV(7);
   }
  }
#undef CHK
#undef LIN_EV
  return CHOREO_OK;
}

// Timing events for the executor's K5 brackets (the bench reads the K5 launch durations
// recorded on the launching stream).
extern "C" int choreo_events_create(void** evs, int n) {
  for (int i = 0; i < n; ++i) {
    cudaEvent_t e;
    cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) {
      set_last_error("choreo_events_create", err);
      return CHOREO_ELAUNCH;
    }
    evs[i] = e;
  }
  return CHOREO_OK;
}

extern "C" int choreo_events_elapsed(void* const* evs, int n_pairs, float* ms) {
  for (int i = 0; i < n_pairs; ++i) {
    cudaError_t err = cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(evs[2 * i + 1]));
    if (err == cudaSuccess)
      err = cudaEventElapsedTime(&ms[i], reinterpret_cast<cudaEvent_t>(evs[2 * i]),
                                 reinterpret_cast<cudaEvent_t>(evs[2 * i + 1]));
    if (err != cudaSuccess) {
      set_last_error("choreo_events_elapsed", err);
      return CHOREO_ELAUNCH;
    }
  }
  return CHOREO_OK;
}

extern "C" int choreo_events_destroy(void* const* evs, int n) {
  for (int i = 0; i < n; ++i) cudaEventDestroy(reinterpret_cast<cudaEvent_t>(evs[i]));
  return CHOREO_OK;
}
