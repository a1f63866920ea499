/*
 * choreo_b200.h — C-ABI of the B200-native choreographed-attention hot path.
 *
 * The reference (/root/reference/pkg, pure Python/NumPy) has no FFI layer; its
 * hot path sits behind Python objects.  Each entry point below replaces one
 * reference function on that path (file:line relative to
 * /root/reference/pkg/src/choreo/) and is what a binding for the reference's
 * Engine would call (see INTEGRATION.md for the ctypes binding).
 *
 * Conventions (every function):
 *   - plain device pointers + sizes; no torch / C++ types; never allocates or
 *     frees device memory (the caller owns every buffer);
 *   - `stream` is a cudaStream_t passed as void*; all work is asynchronous on it;
 *   - returns 0 on success, a negative CHOREO_E* code otherwise; never throws;
 *   - dtype codes: CHOREO_F32 (0) and CHOREO_BF16 (1).
 *
 * KV pool layout (one pool for K, one for V):
 *   pool[layer][kv_head][page][slot][head_dim], pages of `page_size` slots.
 * Every page belongs to exactly one message; a message's tokens fill its page
 * chain in within-message order.  Keys are stored post-rotation at the
 * message's current logical position (reference cache.py:3-7).
 */
#ifndef CHOREO_B200_H
#define CHOREO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHOREO_F32 0
#define CHOREO_BF16 1

#define CHOREO_OK 0
#define CHOREO_EINVAL (-1)   /* bad argument (shape, dtype, null pointer) */
#define CHOREO_ELAUNCH (-2)  /* CUDA launch / runtime failure */
#define CHOREO_EUNSUPPORTED (-3)

/* ABI version (major*100 + minor). */
int choreo_abi_version(void);

/* Last CUDA error string recorded by this library (thread-local, never NULL). */
const char* choreo_last_error(void);

/* x[r, :] = embed[ids[r], :] as f32.  Replaces model.py:162 (`weights.embed[ids]`). */
int choreo_embed(const void* embed, int embed_dtype, int d, const int32_t* ids, int n_rows,
                 float* x, void* stream);

/* choreo_embed where row r takes sel_src[sel[r]] instead of ids[r] when sel[r] >= 0: the
 * token a device selection (choreo_select_greedy / _nucleus output) of the previous step
 * left in device memory, so a pipelined decode step needs no host round trip for its
 * input ids. */
int choreo_embed_select(const void* embed, int embed_dtype, int d, const int32_t* ids,
                        const int32_t* sel, const int32_t* sel_src, int n_rows, float* x,
                        void* stream);

/* Split activations ("*_split" flags): a bf16 activation row y is emitted as the pair
 * hi = bf16(y) at row r and lo = bf16(y - hi) at row n + r of a stacked [2n][.] buffer;
 * a bf16 GEMM over the 2n rows then a sum of the two output halves sees y with ~16
 * mantissa bits.  Consumers of such a stacked f32 GEMM output take *_split = 1 and
 * add rows r and n + r.  Decode GEMMs are weight-bandwidth bound, so the extra rows
 * are free there. */

/* Pre-norm residual step: if delta != NULL, x += delta (f32 residual stream; with
 * delta_split, delta rows r and n_rows + r are both added);
 * out = x / sqrt(mean(x^2) + eps) * w, written in out_dtype (hi/lo pair if out_split).
 * out == NULL: residual add only.  row_map (optional): out row i normalises x row
 * row_map[i], no residual add (used to pick logit rows).
 * Replaces model.py:171,185-186,189 (residual adds + tensor.py:78-80 rms_norm). */
int choreo_residual_rmsnorm(float* x, const void* delta, int delta_dtype, int delta_split,
                            const void* w, int w_dtype, int n_rows, int d, float eps, void* out,
                            int out_dtype, int out_split, const int32_t* row_map, int n_out,
                            void* stream);

/* out[r, i] = silu(gu[r, i]) * gu[r, f + i]  (gate | up concatenated).
 * Replaces model.py:187 and tensor.py:83-84. */
int choreo_silu_mul(const void* gu, int gu_dtype, int in_split, int n_rows, int f, void* out,
                    int out_dtype, int out_split, void* stream);

/* K1 rope_append: for each new-token row r at logical position pos[r],
 *   q_out[r, h, :]   = rotate(qkv[r, q_h], pos[r])           (f32)
 *   K[layer][h][dst_page[r]][dst_slot[r]] = rotate(qkv[r, k_h], pos[r])
 *   V[layer][h][dst_page[r]][dst_slot[r]] = qkv[r, v_h]
 * with qkv rows laid out [q (n_heads*hd) | k (n_kv*hd) | v (n_kv*hd)].
 * Rotation is the reference's interleaved-pair RoPE read from the f64-derived
 * table cos/sin[(pos + W) * (hd/2) + i] (tensor.py:87-143).
 * Replaces model.py:172-176 + cache.py:98-135 (append_tokens) fused. */
int choreo_rope_append(const void* qkv, int qkv_dtype, int ld_qkv, int n_rows, int qkv_split,
                       const int32_t* pos, const int32_t* dst_page, const int32_t* dst_slot,
                       float* q_out, void* k_pool, void* v_pool, int pool_dtype, int layer,
                       int n_kv, int n_pages, int page_size, int n_heads, int head_dim,
                       const float* cos_t, const float* sin_t, int max_delta, void* stream);

/* K2 rerotate: in-place rotation of cached keys by a per-page delta, all layers:
 *   for l, h, i < n_list, s < page_len[i]:  K[l][h][pages[i]][s] = rotate(., delta[i])
 * |delta| <= max_delta.  V is never touched.  delta == 0 pages are skipped.
 * Replaces cache.py:139-160 (reposition_message) + tensor.py:115-122. */
int choreo_rerotate(void* k_pool, int pool_dtype, int n_layers, int n_kv, int n_pages,
                    int page_size, int head_dim, const int32_t* pages, const int32_t* page_len,
                    const int32_t* delta, int n_list, const float* cos_t, const float* sin_t,
                    int max_delta, void* stream);

/* K3 assemble: page-centric prompt assembly on device.  Inputs (device int32):
 *   msg_len[m], msg_pt[m] (offset of message m's page chain in page_table), page_table[]
 *   calls[5*c..]: {own msg, parent offset, parent count, row offset, row count}
 *   call_parents[]: parent message ids, in the call's parent order
 *   row_t[r]: the row's within-message token index (rows grouped by call, ascending t);
 *             the row sees its own message's tokens 0..t
 *   patch[2*i], patch[2*i+1]: page_table[patch[2i]] = patch[2i+1], applied first
 * Work is grouped page-centrically: every distinct parent message of the step is one
 * group whose viewers are all rows of all calls listing it (read once for all of
 * them); each call's own pages form a causal group for its own rows.  Groups are
 * split into items of <= rows_per_block rows x <= pages_per_item pages.
 * Outputs (device int32):
 *   vis_page[], vis_len[], vis_own[]: visible pages (each distinct parent once, in
 *       ascending message id, vis_own = -1; then each call's own pages up to its last
 *       row, vis_own = own token index of slot 0)
 *   blk_rows[]: row ids of every row block
 *   items[6*i..]: {blk_rows offset, n_rows, vis offset, n_pages, partial base, group}
 *       (group >= 0: parent group index; -1-c: own pages of call c)
 *   row_part_off[n_rows + 1], row_part[]: per-row CSR list of the partial slots to merge
 *   counts[0..3] = {n_vis_pages, n_items, n_partials, status (0 ok, <0 over capacity)}
 * fat (optional, int32 [n_items][64]): self-contained item records for choreo_decode_attn_v2:
 *   {n_rows, n_pages, partial base, 0, row ids[16], row_t[16], page[8], page_len[8],
 *    own_base[8], pad[4]}; requires rows_per_block <= 16 and pages_per_item <= 8.
 * mode 0 = page-centric groups (decode-sized steps); mode 1 = per-call lists (prefill-sized
 * steps: each call's parents' pages in parent order, then its own pages, items are row
 * blocks x page chunks of that list; group field = -1-call).
 * Visibility is exactly reference masking.py:36-53 (parents' tokens + own tokens with
 * j <= query j) at page granularity; tests expand it to token level against the oracle.
 * Replaces engine.py:203-245 layout + masking.py:43-53 visible_cache_indices. */
int choreo_assemble(const int32_t* msg_len, const int32_t* msg_pt, int32_t* page_table,
                    const int32_t* calls, const int32_t* call_parents, int n_calls,
                    const int32_t* row_t, int n_rows, const int32_t* patch, int n_patch,
                    int page_size, int rows_per_block, int pages_per_item, int32_t* vis_page,
                    int32_t* vis_len, int32_t* vis_own, int32_t* blk_rows, int32_t* items,
                    int32_t* row_part_off, int32_t* row_part, int32_t* counts, int cap_vis,
                    int cap_blk_rows, int cap_items, int cap_parts, int mode, int32_t* fat,
                    void* stream);

/* choreo_assemble plus item_order (optional, int32 [n_items]): the item indices sorted by
 * page count, descending, ties in item order.  choreo_decode_attn_v2_ex deals a multi-wave
 * step's units to its persistent CTAs longest-first in this order (schedule only: results
 * are bitwise the same with or without it).  step_tag != 0 (mode 0; counts must then hold 6
 * ints, 8-byte aligned): counts[4..5] = {step_tag, n_items} (one 64-bit release store, device
 * scope) once every output is written, so a later kernel of the step may read them before
 * its programmatic-dependency wait. */
int choreo_assemble_ex(const int32_t* msg_len, const int32_t* msg_pt, int32_t* page_table,
                       const int32_t* calls, const int32_t* call_parents, int n_calls,
                       const int32_t* row_t, int n_rows, const int32_t* patch, int n_patch,
                       int page_size, int rows_per_block, int pages_per_item, int32_t* vis_page,
                       int32_t* vis_len, int32_t* vis_own, int32_t* blk_rows, int32_t* items,
                       int32_t* row_part_off, int32_t* row_part, int32_t* counts, int cap_vis,
                       int cap_blk_rows, int cap_items, int cap_parts, int mode, int32_t* fat,
                       int32_t* item_order, int step_tag, void* stream);

/* K5 split-KV attention over assembled work items (prefill and decode rows alike).
 * q: f32 [n_rows][n_heads][hd] (already rotated, K1).  For each item and KV head writes
 * per-(row, q-head) partials: part_o f32 [n_partials][n_heads][hd] (normalised) and
 * part_lse f32 [n_partials][n_heads] (natural-log sum-exp; -inf if nothing visible).
 * The generic path: SIMT with f32 math over f32 or bf16 pages, any head_dim in
 * {8,16,32,64,128}; the f32 parity variant and the shapes K4 / K5 v2 do not take run here.
 * grid_ctas = persistent CTAs (0 = auto).  Replaces model.py:177-184 + tensor.py:65-75
 * (gather, concat, scores, masked softmax, P.V). */
int choreo_attn_split(const float* q, const void* k_pool, const void* v_pool, int pool_dtype,
                      int layer, int n_kv, int n_pages, int page_size, int n_heads, int head_dim,
                      const int32_t* row_t, const int32_t* vis_page, const int32_t* vis_len,
                      const int32_t* vis_own, const int32_t* blk_rows, const int32_t* items,
                      const int32_t* counts, int max_items, float* part_o, float* part_lse,
                      int grid_ctas, void* stream);

/* K4 choreographed prefill attention on tcgen05 tensor cores (bf16 pools, page_size 64,
 * head_dim 64 or 128).  Same items / partials contract as choreo_attn_split, with items
 * built for rows_per_block = 256 / (n_heads / n_kv): two 128-vector M tiles of (row, head)
 * query vectors per item that share every K/V page and ping-pong on the tensor core.  Pages arrive by TMA (SW128 tensor maps over the pool, built
 * here), S = Q K^T and O += P V accumulate in TMEM, the masked online softmax runs in
 * registers, one query vector per TMEM lane.  Pool rows (layers*kv*pages*64) must fit in
 * int32.  out (optional, bf16 [n_rows (x2 if out_split)][n_heads*head_dim]): when every row
 * has exactly one item, write the final normalised rows there (hi/lo pair if out_split)
 * instead of partials, so no combine pass is needed.
 * Replaces model.py:177-184 for prefill-sized steps. */
int choreo_prefill_attn(const float* q, const void* k_pool, const void* v_pool, int pool_dtype,
                        int n_layers, int layer, int n_kv, int n_pages, int page_size,
                        int n_heads, int head_dim, const int32_t* row_t, const int32_t* vis_page,
                        const int32_t* vis_len, const int32_t* vis_own, const int32_t* blk_rows,
                        const int32_t* items, const int32_t* counts, int max_items, float* part_o,
                        float* part_lse, int grid_ctas, void* out, int out_split, int n_rows,
                        void* stream);

/* choreo_decode_attn_v2 reading Q from q_k5 (choreo_rope_append_pieces_ex's output) with
 * one 1-D bulk copy per vector half instead of per-lane loads and conversion (NULL: q), and
 * (item_order, optional: choreo_assemble_ex's output) dealing the units of a step with more
 * units than CTAs longest-first, snaking across the grid (NULL: unit w to CTA w mod grid).
 * k3_tag != 0: the step_tag given to choreo_assemble_ex; once counts[4] holds it the loader
 * and producer warps read the step's K3 outputs before the programmatic-dependency wait. */
int choreo_decode_attn_v2_ex(const float* q, const void* k_pool, const void* v_pool,
                             int n_layers, int layer, int n_kv, int n_pages, int page_size,
                             int n_heads, int head_dim, const int32_t* row_t,
                             const int32_t* vis_page, const int32_t* vis_len,
                             const int32_t* vis_own, const int32_t* blk_rows,
                             const int32_t* items, const int32_t* counts, int max_items,
                             float* part_o, float* part_lse, const int32_t* fat_items,
                             int grid_ctas, const void* q_k5, const int32_t* item_order,
                             int k3_tag, void* stream);

/* Combine each row's partials (CSR row_part_off / row_part, <= 512 per row) into
 * out[r][h][:] (out_dtype; hi/lo pair if out_split) with the LSE merge. */
int choreo_attn_combine(const float* part_o, const float* part_lse, const int32_t* row_part_off,
                        const int32_t* row_part, int n_rows, int n_heads, int head_dim, void* out,
                        int out_dtype, int out_split, void* stream);

/* K6 select: greedy argmax over generatable ids {0..255, 257} with first-index
 * tie-break, one row per logits row (engine.py:371, tokenizer.py:39-44). */
int choreo_select_greedy(const float* logits, int n_rows, int ld, int vocab, int split,
                         int32_t* out_tok, void* stream);

/* K5 v2 decode attention over K3 page-centric items (bf16 pools, page_size 64, head_dim
 * 64/128, n_heads / n_kv <= 32, items built with rows_per_block <= 32 / G): persistent CTAs
 * (grid_ctas <= 0: min(148, items * n_kv)), a TMA producer warp streaming K/V pages into a
 * 5-slot shared-memory ring and 8 mma.sync consumer warps (4 key slices x 2 m16 tiles);
 * Q as a hi/lo bf16 pair, P bf16, f32 accumulation.  Writes one normalised partial + LSE per
 * (block row, head) like choreo_attn_split; merge with choreo_attn_combine.
 * n_layers sizes the pool's TMA view.  fat_items (optional, the `fat` output of
 * choreo_assemble; used when 32 / G <= 16) lets the loader read a unit's rows in the same
 * round trip as its item.  Replaces model.py:177-184 for decode steps. */
int choreo_decode_attn_v2(const float* q, const void* k_pool, const void* v_pool, int n_layers,
                          int layer, int n_kv, int n_pages, int page_size, int n_heads,
                          int head_dim, const int32_t* row_t, const int32_t* vis_page,
                          const int32_t* vis_len, const int32_t* vis_own, const int32_t* blk_rows,
                          const int32_t* items, const int32_t* counts, int max_items,
                          float* part_o, float* part_lse, const int32_t* fat_items,
                          int grid_ctas, void* stream);

/* Deferred K7 output ("pieces"): tiles owned by one CTA are complete in y ([rows][n] f32);
 * tiles cut between CTAs (stream-K) are left as per-CTA partials in the workspace and summed
 * by the consuming kernel in the order the K7 reducer uses, so the values are bit-identical
 * to choreo_linear_skinny's y while the GEMM skips its cross-CTA fix-up (a GPU-scope
 * atomic and a second pass over the partials at the end of the launch). */
typedef struct {
  const float* y;
  const float* ws;
  int n, kb, iters, grid, nx, split;
} ChoreoK7Pieces;

/* K7 decode-sized linear layer (weight streaming, tcgen05 + TMA, stream-K):
 *   y[r][n] = sum_k x[r][k] * w[n][k]      x: bf16 [x_rows][k], w: bf16 [n][k] (out, in),
 *                                          y: f32 [x_rows / (1 + split)][n].
 * split = 1: x rows r and x_rows/2 + r are the hi/lo halves of one activation row and
 * y row r is their sum.  x_rows <= 256 when split (<= 128 output rows), else <= 128; k % 8 == 0.
 * workspace: f32 [148 * 2 * NX * 128] partial tiles (NX = x_rows rounded up to 16/32/64/128/256); tile_counters: int32 [ceil(n/128)],
 * zero on entry, left zero on exit.  grid_ctas <= 0: one CTA per SM (148).
 * Replaces the x @ W projections of model.py:172-174, 185-189 and the head at 193 for
 * decode-sized steps (the reference runs them as NumPy matmuls). */
int choreo_linear_skinny(const void* x, int x_rows, int split, const void* w, int n, int k,
                         float* y, float* workspace, int* tile_counters, int grid_ctas,
                         void* stream);

/* choreo_linear_skinny that leaves cut tiles as pieces (see ChoreoK7Pieces, filled in
 * `pieces`); consumers: choreo_rope_append_pieces, choreo_residual_rmsnorm_pieces. */
int choreo_linear_skinny_pieces(const void* x, int x_rows, int split, const void* w, int n, int k,
                                float* y, float* workspace, int* tile_counters, int grid_ctas,
                                ChoreoK7Pieces* pieces, void* stream);

/* choreo_rope_append (f32 qkv) reading a deferred K7 qkv projection. */
int choreo_rope_append_pieces(const ChoreoK7Pieces* qkv, int n_rows, const int32_t* pos,
                              const int32_t* dst_page, const int32_t* dst_slot, float* q_out,
                              void* k_pool, void* v_pool, int pool_dtype, int layer, int n_kv,
                              int n_pages, int page_size, int n_heads, int head_dim,
                              const float* cos_t, const float* sin_t, int max_delta, void* stream);

/* choreo_rope_append_pieces that also writes q_k5 (bf16 [n_rows][n_heads][2][head_dim]): each
 * rotated query vector times q_scale as a hi/lo bf16 pair -- the record format K5 v2 stages
 * with bulk copies (choreo_decode_attn_v2_ex, q_scale = log2(e) / sqrt(head_dim)). */
int choreo_rope_append_pieces_ex(const ChoreoK7Pieces* qkv, int n_rows, const int32_t* pos,
                                 const int32_t* dst_page, const int32_t* dst_slot, float* q_out,
                                 void* k_pool, void* v_pool, int pool_dtype, int layer, int n_kv,
                                 int n_pages, int page_size, int n_heads, int head_dim,
                                 const float* cos_t, const float* sin_t, int max_delta,
                                 void* q_k5, float q_scale, void* stream);

/* choreo_residual_rmsnorm with delta = a deferred K7 projection (x += delta; out = norm(x)).
 * bf16 outputs with d a multiple of 1024 (<= 4096) run one 8-CTA cluster of 128 threads per
 * row (DSMEM reduction in the single-CTA kernel's order: bit-identical results);
 * CHOREO_NORM_CLUSTER=0 selects the single-CTA kernel (A/B timing). */
int choreo_residual_rmsnorm_pieces(float* x, const ChoreoK7Pieces* delta, const void* w,
                                   int w_dtype, int n_rows, int d, float eps, void* out,
                                   int out_dtype, int out_split, void* stream);

/* K7 for the gate|up projection with the SwiGLU product fused into its epilogue:
 * act[r][i] = silu(g) * u, g = x[r] . w_gu[i], u = x[r] . w_gu[f + i] (w_gu = [gate; up],
 * (2f, d)), written as bf16 act [out_rows][f] (+ the lo halves at rows out_rows + r when
 * split) — choreo_linear_skinny followed by choreo_silu_mul in one launch (each tile pairs
 * 64 gate rows with the matching 64 up rows).  f % 64 == 0.  Replaces model.py:186-187. */
int choreo_linear_gate_up_silu(const void* x, int x_rows, int split, const void* w_gu, int f,
                               int d, void* act, float* workspace, int* tile_counters,
                               void* stream);

/* Native decode-step executor: every layer of a decode-sized bf16 step (split hi/lo
 * activations or plain bf16; page_size 64; K5 v2 items from choreo_assemble, page-centric
 * mode) issued in one call — per layer: residual_rmsnorm, K7 qkv, K1 rope_append,
 * K5 v2 decode attention, combine, K7 o_proj, residual_rmsnorm, K7 gate|up (+SwiGLU),
 * K7 down.  Replaces the per-layer loop of model.py:169-189.  Weight arrays are HOST
 * arrays of n_layers DEVICE pointers (bf16, (out, in) layout).  On return `delta` holds
 * the last layer's down_proj output (the caller adds it and runs the final norm / head).
 * attn_events: optional host array of 2 * n_layers cudaEvent_t recorded around each K5. */
typedef struct {
  int n_layers, d, n_heads, n_kv, head_dim, ffn_dim;
  const void* const* attn_norm;
  const void* const* w_qkv;
  const void* const* wo;
  const void* const* ffn_norm;
  const void* const* w_gu;
  const void* const* w_down;
  float eps;
  void* k_pool;
  void* v_pool;
  int n_pages, page_size;
  const float* cos_t;
  const float* sin_t;
  int max_delta;
  int n_rows, split, n_items;
  const int32_t* pos;
  const int32_t* page;
  const int32_t* slot;
  const int32_t* fat;
  const int32_t* counts;
  const int32_t* row_part_off;
  const int32_t* row_part;
  float* x;
  const float* delta_in; /* added to x before layer 0's norm (NULL: none) */
  void* h;
  float* qkv;
  float* q;
  float* part_o;
  float* part_lse;
  void* attn;
  float* ao;
  float* gu;
  void* act;
  float* delta;
  float* k7_ws;
  int* k7_cnt;
  void** attn_events;
  /* K3 arrays K5 v2 reads (choreo_assemble outputs) */
  const int32_t* row_t;
  const int32_t* vis_page;
  const int32_t* vis_len;
  const int32_t* vis_own;
  const int32_t* blk_rows;
  const int32_t* items;
  /* optional host array of 8 * n_layers cudaEvent_t recorded around the layer's four K7
   * launches (qkv, o_proj, gate|up, down); NULL: none */
  void** linear_events;
  /* layers [layer_begin, layer_end) (layer_end 0: n_layers) and which part of each:
   * 0 whole layers; 1 the attention half (first norm takes delta_in, ends with o_proj in
   * `ao`); 2 the MLP half (norm of x += ao, ends with down_proj in `delta`).  Tensor
   * parallel callers run part 1, all-reduce ao, part 2, all-reduce delta, per layer. */
  int layer_begin, layer_end, part;
  /* K8 chain path (part 0 with every layer): when chain_ws != NULL each step runs
   * choreo_chain_prologue, one choreo_layer_chain (qkv of layer 0), then per layer K5 v2 +
   * combine + one choreo_layer_chain (o_proj, gate|up, down, qkv of the next layer); the
   * last layer's down_proj is added into x (delta is not written).  h_b: bf16 [2 n_rows][d];
   * ssq_a / ssq_b f32 [ceil(d/128)][128]; chain_ws / chain_counters / chain_done as
   * choreo_layer_chain.
   * chain_events: optional host array of 2 * (n_layers + 1) cudaEvent_t recorded around
   * each chain launch. */
  void* h_b;
  float* ssq_a;
  float* ssq_b;
  float* chain_ws;
  int* chain_counters;
  int* chain_done;
  void** chain_events;
  /* optional bf16 [n_rows][n_heads][2][head_dim]: RoPE writes K5 v2's Q record format there and
   * K5 v2 stages it with bulk copies (choreo_rope_append_pieces_ex / _decode_attn_v2_ex) */
  void* q_k5;
  /* optional int32 [n_items]: choreo_assemble_ex's item_order (K5 v2 unit schedule) */
  const int32_t* item_order;
  /* the step_tag given to choreo_assemble_ex (0: none), see choreo_decode_attn_v2_ex */
  int k3_tag;
} ChoreoDecodeStep;

int choreo_decode_layers(const ChoreoDecodeStep* step, void* stream);

/* K8 layer chain: the weight-streaming projections between two attentions of a decode-sized
 * bf16 step in ONE persistent launch (tcgen05 + TMA, one CTA per SM, stream-K per phase,
 * per-tile dataflow flags between phases instead of kernel boundaries).  Phases (bits of
 * `phases`, run in this order):
 *   1 o_proj : x += attn @ wo^T; h_a = hi/lo(x * ffn_norm); ssq_a = per-128-column sums of x^2
 *   2 gate|up: act = silu(r g) * (r u), r = rsqrt(mean(x^2) + eps) from ssq_a (hi/lo bf16)
 *   4 down   : x += act @ w_down^T; if attn_norm_next: h_b = hi/lo(x * attn_norm_next), ssq_b
 *   8 qkv    : r * (h_b @ w_qkv^T) with r from ssq_b -> RoPE(q, k) at pos[row]; q (f32
 *              [n_rows][n_heads][head_dim]) out, k / v (bf16) written to pool slot
 *              (page[row], slot[row]) of layer layer_qkv  (K1's contract)
 * RMSNorm is applied as a per-row scale of the next GEMM's output (norm(x) w @ W^T =
 * r ((x w) @ W^T)).  Activations: split = 1 carries every GEMM input as hi/lo bf16 rows r and
 * n_rows + r (n_rows <= 128), else plain bf16 (n_rows <= 128).  Buffers: x f32 [n_rows][d];
 * attn, h_a, h_b bf16 [2 n_rows][.] ; act bf16 [2 n_rows][ffn_dim]; ssq_a / ssq_b f32
 * [ceil(d/128)][128]; ws f32 [4][148][2][128][128]; counters int32 [4][1024] and done int32
 * [8] (per-phase completion counters), zero before the first launch and left zero.
 * d, n_heads*head_dim, ffn_dim multiples of 64.
 * Replaces model.py:169-189 (everything after attention of layer l up to the attention of
 * layer l+1) for decode-sized steps. */
typedef struct {
  int n_rows, split, d, n_heads, n_kv, head_dim, ffn_dim;
  float eps;
  int phases;
  const void* wo;
  const void* ffn_norm;
  const void* w_gu;
  const void* w_down;
  const void* attn_norm_next;
  const void* w_qkv;
  int layer_qkv;
  float* x;
  const void* attn;
  void* h_a;
  void* act;
  void* h_b;
  float* ssq_a;
  float* ssq_b;
  float* q;
  void* k_pool;
  void* v_pool;
  int n_pages, page_size;
  const int32_t* pos;
  const int32_t* page;
  const int32_t* slot;
  const float* cos_t;
  const float* sin_t;
  int max_delta;
  float* ws;
  int* counters;
  int* done;
} ChoreoLayerChain;

int choreo_layer_chain(const ChoreoLayerChain* chain, void* stream);

/* Start of a chained step: x (+= delta when non-NULL); h = hi/lo(x * gamma) (bf16 [2n][d]
 * when split); ssq f32 [ceil(d/128)][128] = per-128-column sums of x^2 per row (n_rows <=
 * 128).  Feeds the first choreo_layer_chain (qkv phase only). */
int choreo_chain_prologue(float* x, const float* delta, int n_rows, int d, const void* gamma,
                          void* h, int split, float* ssq, void* stream);

/* Timing-event helpers for attn_events (cudaEvent_t as void*). */
int choreo_events_create(void** events, int n);
int choreo_events_elapsed(void* const* events, int n_pairs, float* ms_out);
int choreo_events_destroy(void* const* events, int n);

/* K6b nucleus selection (temperature + top-p) on the device, the reference's f64 algorithm
 * step for step (engine.py:374-392): one row per logits row; params = (temperature, top_p)
 * per row (f64); keys = (engine_seed, sampling_seed, msg_id, sel_index) per row (u64), the
 * Philox4x64-10 stream NumPy's Generator(Philox(counter=[sel, msg_id, 0, 0],
 * key=[engine_seed, sampling_seed])).random() draws from.  vocab >= 258. */
int choreo_select_nucleus(const float* logits, int n_rows, int ld, int vocab,
                          const double* params, const uint64_t* keys, int32_t* out_tok,
                          void* stream);

/* Diagnostics: one-CTA tcgen05 GEMM over the UMMA primitives K4 uses.
 * a: bf16 [128][64], b1: bf16 [64][64] (N x K), b2: bf16 [64][128] (K x N);
 * c1 = a * b1^T (f32 [128][64]), c2 = a * b2 (f32 [128][128]) with both operands in shared
 * memory, c3 = a * b2 with a staged in tensor memory (A-from-TMEM MMA form). */
int choreo_selftest_umma(const void* a, const void* b1, const void* b2, float* c1, float* c2,
                         float* c3, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CHOREO_B200_H */
