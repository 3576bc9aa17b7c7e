/*
 * sparseft_b200.h — C-ABI of the B200-native Long Exposure hot path.
 *
 * The drop-in boundary for the reference `sparseft` package
 * (/root/reference/pkg/src/sparseft, cited as sf/<file>:<line>). Each entry
 * point replaces the reference function(s) named in its comment; the Python
 * host layer (paper_2510_15964_b200/*.py) keeps the reference's names and
 * argument meaning and binds these symbols with ctypes.
 *
 * Conventions
 *   - plain device pointers + sizes; no torch types. bf16 = uint16_t storage.
 *   - every call is stream-ordered on `stream` and never synchronises the host.
 *   - the library allocates nothing; callers pass workspaces.
 *   - return 0 on success, else an LX_ERR_* code; lx_last_error() describes it.
 *     The host shim maps codes to the reference exception types
 *     (ShapeError, LayoutError, MaskError, PatternError).
 *   - deterministic at a fixed launch configuration (no float atomics).
 */
#ifndef SPARSEFT_B200_H
#define SPARSEFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lx_stream_t;

#define LX_OK 0
#define LX_ERR_SHAPE 1       /* sf/tensor_core.py:15 ShapeError   */
#define LX_ERR_LAYOUT 2      /* sf/block_sparse.py:18 LayoutError */
#define LX_ERR_MASK 3        /* sf/neuron_ops.py:18 MaskError     */
#define LX_ERR_PATTERN 4     /* sf/patterns.py:20 PatternError    */
#define LX_ERR_CUDA 5
#define LX_ERR_UNSUPPORTED 6 /* shape outside the sm_100a kernels' envelope */

const char* lx_last_error(void);
int lx_abi_version(void);
int lx_device_sm_count(void);
/* GEMM engine variant for the dense / item-packed modes: 0 (default) = single-CTA 128 x 256 tiles,
 * 1 = CTA pairs (tcgen05.mma.cta_group::2) with 256 x 256 tiles, 2 = CTA pairs with 256 x 128 tiles.
 * Returns the previous value. */
int lx_gemm_set_cta_pair(int mode);
/* Debug only: per-CTA clock64 phase stamps of the GEMM engine into buf [grid][32]; NULL disables. */
int lx_debug_set_gemm_trace(unsigned long long* buf);

/* ------------------------------------------------------------------ generic
 * C[M,N] (fp32 or bf16) = A[M,K] * B[N,K]^T, bf16 inputs, tcgen05 path.
 * a_k_split > 0 (a multiple of 64): A's K coordinate k maps to k - a_k_split for k >= a_k_split, so with
 * B = [W_hi | W_lo] (bf16 hi/lo split of an fp32 W, segments a_k_split wide) one GEMM returns A (W_hi + W_lo),
 * i.e. the product with W at ~2^-16 relative precision. Used by the predictor projections (split terms) and
 * by tests of the GEMM engine. */
int lx_gemm_bf16_tn(const uint16_t* a, int lda, const uint16_t* b, int ldb, void* c, int ldc, int c_is_f32, int M, int N,
                    int K, int a_k_split, lx_stream_t stream);

/* lora_linear_forward / lora_linear_backward's dense products (sf/model.py:292-304,
 * sf/autograd.py:48-58) with the bias, LoRA and residual fused in the epilogue:
 *   out[M,N] = (resid) + A[M,K] * B[N,K]^T + bias[N] + scaling * lora_x[M,r] . w(:, n)
 *   w(q, n) = lora_w[q*w_sr + n*w_sc]; out fp32 (out_f32, optional resid) or bf16. */
int lx_linear(const uint16_t* a, int lda, const uint16_t* b_t, int ldb, int M, int N, int K, void* out, int ldo,
              int out_f32, const float* resid, const float* bias, const float* lora_x, const float* lora_w,
              long long w_sr, long long w_sc, int r, float scaling, lx_stream_t stream);
/* Same with the weight as stored for x @ W (torch.addmm layout): b [K, N] row-major, row stride ldb.
 * The frozen Q/K/V/O projections and the LM head's input-grad (sf/model.py:340-342,354,449-450;
 * sf/autograd.py:127-162) run on this and on lx_linear (the input-grads take W itself as b_t). */
int lx_linear_kn(const uint16_t* a, int lda, const uint16_t* b, int ldb, int M, int N, int K, void* out, int ldo,
                 int out_f32, const float* resid, const float* bias, const float* lora_x, const float* lora_w,
                 long long w_sr, long long w_sc, int r, float scaling, lx_stream_t stream);

/* ------------------------------------------------------------------ K1 mask build
 * approx_mlp_scores + predict_mlp_mask + active_columns
 *   (sf/predictor.py:121-139, sf/neuron_ops.py:67-72)
 * h:      bf16 [n_items*s, d] post-LN2 MLP input (one item = one sequence)
 * wa_t:   bf16 [n_blk, k_terms*d]  (Wa_hat transposed: each block's scoring vector contiguous)
 * k_terms: precision of S_hat = h Wa_hat (the reference computes it in float32, sf/predictor.py:121-125):
 *          1: wa_t = bf16(W) (bf16 scores);
 *          2: wa_t = [W_hi | W_lo] (bf16 hi/lo split of the fp32 weights): h W exact to ~2^-16 for a bf16 h
 *             (the fine-tune step: h is the bf16 LN output);
 *          3: h = [x_hi | x_lo] bf16 [n_items*s, 2d] and wa_t = [W_hi | W_lo | W_hi]: an fp32 x and fp32 W
 *             (the reference-API call on host float32 inputs). Split terms need d % 64 == 0.
 * scope_batch: 0 = per-item masks (sf/harness.py:204-211), 1 = OR over items (sf/predictor.py:132-136)
 * bits_ws: uint32 [n_items, ceil(s/32), ceil(n_blk/32)] workspace: one word per (32-token group, 32 blocks), each
 *          stored exactly once by the scoring GEMM (no memset, no atomics); the compaction ORs the groups
 * counts: int32 [n_items]; ids: int32 [n_items, n_blk] ascending active block ids;
 * pos:    int32 [n_items, n_blk] packed position of each block or -1
 * scores_dump: optional fp32 [n_items*s, n_blk] copy of S_hat (parity tests) */
int lx_predict_mlp_mask(const uint16_t* h, int n_items, int s, int d, const uint16_t* wa_t, int n_blk, int k_terms,
                        float threshold, int scope_batch, uint32_t* bits_ws, int32_t* counts, int32_t* ids, int32_t* pos,
                        float* scores_dump, lx_stream_t stream);

/* Compaction only: bitmask words -> counts/ids/pos (used when masks come from a provider). */
int lx_mask_compact(const uint32_t* bits, int n_items, int n_blk, int scope_batch, int32_t* counts, int32_t* ids,
                    int32_t* pos, lx_stream_t stream);

/* predict_attention_patterns + select_pattern_by_coverage
 *   (sf/predictor.py:62-118, sf/exposer.py:71-85)
 * x_small: bf16 [n_items*m, d] downsampled rows (m = ceil(sqrt(s)), rows min(i*s//m, s-1))
 *          ([x_hi | x_lo] [n_items*m, 2d] for k_terms 3)
 * wqk_t:   bf16 [2*H*r, k_terms*d]: rows [h*r,(h+1)*r) = Wq_hat[h]^T, rows [(H+h)*r, ...) = Wk_hat[h]^T,
 *          as k_terms bf16 segments (see lx_predict_mlp_mask: 2 = [W_hi | W_lo], 3 = [W_hi | W_lo | W_hi])
 * pool_kind/pool_param: pool in reference order (kind 0 blockdiag,1 band,2 causal,3 global,4 strided,5 dense)
 * proj_ws: fp32 [n_items*m, 2*H*r] workspace; pattern_idx: int32 [n_items(or 1), H] pool index
 * scores_dump: optional fp32 [n_items, H, m, m] */
int lx_predict_attention_patterns(const uint16_t* x_small, int n_items, int m, int d, const uint16_t* wqk_t, int H,
                                  int r, int k_terms, float threshold_frac, double tau, int n_b, const int32_t* pool_kind,
                                  const int32_t* pool_param, int n_pool, int scope_batch, float* proj_ws,
                                  int32_t* pattern_idx, float* scores_dump, lx_stream_t stream);

/* ------------------------------------------------------------------ K2 neuron-sparse MLP
 * Layout: w1_t bf16 [d_ff, d] (= W1 column-major, sf/neuron_ops.py:31-45), w2 bf16 [d_ff, d].
 * w*_packed (optional, from lx_pack_active_rows): the item-packed active rows of the same weight;
 * when given, the GEMM streams them with one TMA box per 256 rows / 64x64 tile instead of one per block.
 * Hidden tensors are packed per item: row t of item b holds its active columns
 * [0, counts[b]*blk) in ascending block order, row stride ld_h (>= d_ff).
 * LoRA factors are fp32 (trainable); pass NULL to skip a term. */

/* neuron_matmul_fwd1 + b1 + scaling*(x A1) B1[:,cols] (+ ReLU if apply_relu)
 *   (sf/neuron_ops.py:75-82, sf/model.py:376-386)
 * ax1: fp32 [M, r] = x A1 (from lx_rowproj); b1_lora: fp32 [r, d_ff]
 * relu_bits (optional, apply_relu, ld_h % 16 == 0): also writes relu'(z) = (bf16 a > 0) as bits, uint16 [M, ld_h/16]
 * (bit j%16 of word j/16 of a row = packed column j), the mask mlp_backward applies (sf/autograd.py:101). */
int lx_neuron_fc1(const uint16_t* x, int n_items, int s, int d, int d_ff, int blk, const uint16_t* w1_t,
                  const int32_t* counts, const int32_t* ids, const float* b1, const float* ax1, const float* b1_lora,
                  int r, float scaling, int apply_relu, uint16_t* a_out, int ld_h, const uint16_t* w1_packed,
                  uint16_t* relu_bits, lx_stream_t stream);

/* neuron_matmul_fwd2 + b2 + scaling*(a A2[cols]) B2   (sf/neuron_ops.py:85-95, sf/model.py:388-395)
 * ax2: fp32 [M, r]; b2_lora: fp32 [r, d]. out bf16, or fp32 (out_f32) with optional fused residual
 * (out = resid + mlp, the block's y + MLP(LN(y)), sf/model.py:427). */
int lx_neuron_fc2(const uint16_t* a, int ld_h, int n_items, int s, int d, int d_ff, int blk, const uint16_t* w2,
                  const int32_t* counts, const int32_t* ids, const float* b2, const float* ax2, const float* b2_lora,
                  int r, float scaling, void* out, int out_f32, const float* resid, const uint16_t* w2_packed,
                  lx_stream_t stream);

/* mlp_backward input-grad through fc2 and ReLU   (sf/autograd.py:97-106)
 * dz = (dO W2[cols]^T + dax2 A2[cols]^T) * (a > 0); dax2 fp32 [M,r] (already scaled); a2: fp32 [d_ff, r]
 * relu_bits (optional): lx_neuron_fc1's bits of (a > 0), read instead of the bf16 a (16x fewer epilogue bytes). */
int lx_neuron_fc2_dgrad(const uint16_t* d_out, int n_items, int s, int d, int d_ff, int blk, const uint16_t* w2,
                        const int32_t* counts, const int32_t* ids, const float* dax2, const float* a2_lora, int r,
                        const uint16_t* a, uint16_t* dz, int ld_h, const uint16_t* w2_packed, const uint16_t* relu_bits,
                        lx_stream_t stream);

/* mlp_backward input-grad through fc1   (sf/autograd.py:112-120)
 * dx = dz W1[:,cols]^T + dax1 A1^T; dax1 fp32 [M,r] (already scaled); a1: fp32 [d, r] */
int lx_neuron_fc1_dgrad(const uint16_t* dz, int ld_h, int n_items, int s, int d, int d_ff, int blk,
                        const uint16_t* w1_t, const int32_t* counts, const int32_t* ids, const float* dax1,
                        const float* a1_lora, int r, void* dx, int out_f32, const uint16_t* w1_packed,
                        lx_stream_t stream);

/* Copy each item's active neuron-block rows of a [d_ff, d] weight (W1^T or W2), in ascending block
 * order, into packed [n_items, d_ff, d] rows [0, counts[b]*blk) (sf/neuron_ops.py:67-72 columns). */
int lx_pack_active_rows(const uint16_t* w, int d_ff, int d, int blk, int n_items, const int32_t* counts,
                        const int32_t* ids, uint16_t* packed, lx_stream_t stream);
/* The same for two weights with the same masks (W1^T and W2 of one layer) in one launch; w_b / packed_b may be NULL. */
int lx_pack_active_rows2(const uint16_t* w_a, const uint16_t* w_b, int d_ff, int d, int blk, int n_items,
                         const int32_t* counts, const int32_t* ids, uint16_t* packed_a, uint16_t* packed_b,
                         lx_stream_t stream);

/* Skinny LoRA row projection: Y[M, r] (row stride ldy) = scale * X[M, K] W, K optionally gathered per item.
 *   X bf16 row stride ldx; W(k, q) = w[k_orig*w_sk + q*w_sq]; k_orig = k (dense, counts==NULL) or
 *   ids[b][k/blk]*blk + k%blk over the item's packed K = counts[b]*blk.  (x A1, a A2[cols], dO B2^T, dz B1[:,cols]^T) */
int lx_rowproj(const uint16_t* x, int ldx, int n_items, int s, int K, const float* w, long long w_sk, long long w_sq,
               int r, float scale, const int32_t* counts, const int32_t* ids, int blk, float* y, int ldy, void* wpack_ws,
               lx_stream_t stream);
/* lx_rowproj over a pre-packed W (lx_pack_params): wpack = [2][RP][K_full] bf16 (hi rows, then lo rows),
 * W(k, q) = hi[q][k] + lo[q][k]; RP = 8 or 16 (r <= RP). Gathered (counts != NULL): packed k of item b maps to
 * column ids[b][k/blk]*blk + k%blk of the full pack. yb (optional): bf16 copy of Y with row stride ldyb — the
 * LoRA columns of a K-extended projection operand (lora_linear_forward's x A, sf/model.py:296-300). */
int lx_rowproj_packed(const uint16_t* x, int ldx, int n_items, int s, int K, const uint16_t* wpack, int K_full, int RP,
                      int r, float scale, const int32_t* counts, const int32_t* ids, int blk, float* y, int ldy,
                      uint16_t* yb, int ldyb, lx_stream_t stream);

/* lx_rowproj_packed over n_seg independent dense-K problems in one launch (segment k: x + k*x_seg, wpack +
 * k*w_seg, y + k*y_seg, yb + k*yb_seg, element offsets; n_rows rows each). The q/k/v LoRA input-grad projections
 * dAx_t = dqkv[:, slot_t] B_t^T of one layer (lora_linear_backward, sf/autograd.py:48-58), whose slots, packs and
 * output columns are equally spaced. K <= 4096. */
int lx_rowproj_packed_seg(const uint16_t* x, int ldx, long long x_seg, int n_rows, int K, const uint16_t* wpack,
                          long long w_seg, int K_full, int RP, int r, float scale, float* y, int ldy, int y_seg, uint16_t* yb,
                          int ldyb, int yb_seg, int n_seg, lx_stream_t stream);

/* Parameter packing after the optimizer step (sf/autograd.py:203-225 updates the fp32 trainables):
 *   dst[i*dst_sr + j*dst_sc] = bf16(scale * src[i*src_sr + j*src_sc]),  i < rows, j < cols (element strides);
 *   lo_off != 0 also writes the bf16 residual at dst + lo_off (hi/lo split of an fp32 factor).
 * segs is a DEVICE array of n_segs segments (built once; the pointers stay valid across steps). */
typedef struct lx_pack_segment {
  const float* src;
  long long src_sr;
  long long src_sc;
  int rows;
  int cols;
  uint16_t* dst;
  long long dst_sr;
  long long dst_sc;
  long long lo_off;
  float scale;
  int pad_;
} lx_pack_segment;
int lx_pack_params(const lx_pack_segment* segs, int n_segs, lx_stream_t stream);

/* Workspace for lx_rowproj's tensor-core path: W packed as bf16 hi/lo [items][2][R'][K] (gathered per item). */
long long lx_rowproj_ws_bytes(int n_items, int K, int r, int gathered);

/* Skinny LoRA / BitFit gradient reductions over tokens, up to 8 per launch (one sublayer's backward):
 *   G(q, c) = scale * sum_rows P[row, q] X[row, c]     c = original column
 * replacing lora_linear_backward's xᵀ·dAx / axᵀ·dz and mlp_backward's dB2, dA2[cols], dB1[:,cols], dA1
 * (sf/autograd.py:50-58,97-120) and BitFit's column sums (p == NULL, r = 1; sf/autograd.py:56-57,95-96,107-111).
 *   P fp32 [n_items*s, >= r] row stride ldp (r <= 16); X bf16 row stride ldx (16B-aligned rows).
 *   pos == NULL: X columns are the original columns [0, ncols).
 *   pos != NULL: X holds each item's active neuron blocks packed in ascending order; pos[b][block] is the
 *                block's packed index or -1 (NeuronMasks.pos); inactive columns of G are written 0.
 *   G(q, c) = g[q*g_sq + c*g_sc]. Summed over items in a fixed order: deterministic.
 *   ws: fp32 workspace of lx_colgrad_group_ws_floats floats (split partials). */
typedef struct lx_colgrad_problem {
  const float* p;
  int ldp;
  const uint16_t* x;
  int ldx;
  int ncols;
  int r;
  float scale;
  const int32_t* pos;
  int blk;
  float* g;
  long long g_sq;
  long long g_sc;
} lx_colgrad_problem;
long long lx_colgrad_group_ws_floats(const lx_colgrad_problem* probs, int n_probs, int n_items, int s);
int lx_colgrad_group(const lx_colgrad_problem* probs, int n_probs, int n_items, int s, float* ws, lx_stream_t stream);

/* ------------------------------------------------------------------ K3 block-sparse attention
 * One implementation: tcgen05 flash kernels (csrc/attn_sm100.cu), hd 64 or 128 (other head dims are
 * zero-padded to 64 / 128 by the Python shim, block_sparse.py), non-causal, explicit scale.
 * qkv: the fused projection output bf16 [n_items*s, ld] with q | k | v column blocks of H*hd each
 * (head h at columns h*hd of each block). pattern_idx: int32 [n_items, H] pool index per (item, head)
 * (or [1, H] with item_stride 0).
 * tables128: gathered 128-tile tables (patterns.tables128_from_grids): per pattern, CSR over 128-query
 * tiles and CSC over 128-key tiles whose entries each stack 128 / gather_rows units of gather_rows
 * consecutive tokens (gather_rows = gcd(attn_blk, 128)) with a 64-bit mask of active 16x16 cells, so
 * the MMA work is proportional to the active blocks (sf/block_sparse.py:47-137 computes exactly the
 * layout's blocks).
 * fwd = sdd -> sparse_softmax -> dsd (sf/block_sparse.py:47-126, sf/model.py:343-353); o bf16 with row
 * stride ldo, lse fp32 [n_items, H, s]. */
int lx_bsattn_fwd_tc(const uint16_t* qkv, int ld, int n_items, int s, int H, int hd, const int32_t* pattern_idx,
                     int item_stride, const int32_t* tables128, int gather_rows, float scale, uint16_t* o, int ldo,
                     float* lse, lx_stream_t stream);
/* Backward (dsd_backward -> sparse_softmax_backward -> sdd_backward, sf/block_sparse.py:63-137;
 * replaces mha_backward's per-head loop, sf/autograd.py:149-156): dqkv [n_items*s, ld_d] (same fused
 * layout as qkv) from d_o [n_items*s, ld_o] and the forward's o / lse; delta_ws fp32 [n_items, H, s];
 * ws fp32 [n_items * H * (hd + 8 * ceil(s/128))]: the per-(item, head) mean key (used by dQ to cancel the
 * bf16 row-sum residual of dS against the keys' common mode) and the per-unit work descriptors, all
 * written by the backward's prologue kernel. dK/dV walk the CSC of each 128-key tile, dQ the CSR of each
 * 128-query tile. */
int lx_bsattn_bwd_tc(const uint16_t* qkv, int ld, int ld_d, const uint16_t* o, const uint16_t* d_o, int ld_o, int n_items, int s,
                     int H, int hd, const int32_t* pattern_idx, int item_stride, const int32_t* tables128, int gather_rows,
                     float scale, const float* lse, float* delta_ws, float* ws, uint16_t* dqkv, lx_stream_t stream);
/* Debug only: per-CTA clock64 phase stamps of the tcgen05 attention kernels into buf
 * [n_ctas][32] (slot 31 = SM id); NULL disables. Used by tools/attn_trace.py. */
int lx_debug_set_attn_trace(unsigned long long* buf);

/* ------------------------------------------------------------------ Adapter
 * adapter_forward / adapter_backward (sf/model.py:76-83,315-319; sf/autograd.py:69-75), fp32 like the reference.
 * x fp32 [M, d] (row stride ldx), w_down [d, r], b_down [r], w_up [r, d], b_up [d]; r in {8, 16}.
 * fwd: out = x + relu(x w_down + b_down) w_up + b_up (row stride ldo); z = x w_down + b_down fp32 [M, r] is kept
 *      for the backward. resid (optional, fp32, row stride ldr): out = resid + (that), the block's residual add
 *      (sf/model.py:420-427) fused.
 * bwd: dh = (dy w_up^T) * (z > 0) (fp32 [M, r] out), dx = dy + dh w_down^T (row stride lddx); the gradients of
 *      w_down, b_down, w_up, b_up summed over the rows (fixed order) times `scale`; ws: lx_adapter_ws_floats(d, r)
 *      floats. */
long long lx_adapter_ws_floats(int d, int r);
int lx_adapter_fwd(const float* x, int ldx, int M, int d, int r, const float* w_down, const float* b_down, const float* w_up,
                   const float* b_up, float* z, float* out, int ldo, const float* resid, int ldr, lx_stream_t stream);
int lx_adapter_bwd(const float* dy, int ldy, const float* x, int ldx, int M, int d, int r, const float* z,
                   const float* w_down, const float* w_up, float* dh, float* dx, int lddx, float* ws, float scale,
                   float* g_w_down, float* g_b_down, float* g_w_up, float* g_b_up, lx_stream_t stream);

/* ------------------------------------------------------------------ glue (fused neighbours)
 * layernorm_forward (sf/model.py:307-312), fp32 residual in, bf16 out; saves mean/inv_std.
 * Optionally also writes the predictor's downsampled rows (sf/predictor.py:62-71) to x_small. */
int lx_layernorm_fwd(const float* x, const uint16_t* delta, float* resid_out, int M, int d, const float* gamma,
                     const float* beta, float eps, uint16_t* y, int ldy, float* mean, float* inv_std, int s, int m_small,
                     uint16_t* x_small, lx_stream_t stream);
/* (delta != NULL: fused residual add — resid_out = x + delta (fp32) is normalised and returned.) */
/* optimizer_step (sf/autograd.py:203-225) over the flat trainable buffer: float64 moments m, v, fp32 params,
 * fp32 mean gradients; step t (>= 1) gives the bias corrections 1 - b1^t, 1 - b2^t. One pass. */
int lx_adam_step(float* params, const float* grads, double* m, double* v, long long n, double lr, double b1, double b2,
                 double eps, int t, lx_stream_t stream);
/* loss_forward + loss_backward over rows of fp32 logits (sf/model.py:454-472): row_loss[r] =
 * logsumexp(l_r) - l_r[t_r]; grad_bf16[r] = (softmax(l_r) - onehot(t_r)) * inv_s (inv_s = 1/seq_len). */
int lx_cross_entropy(const float* logits, int rows, int V, const int64_t* targets, float inv_s, float* row_loss,
                     uint16_t* grad_bf16, lx_stream_t stream);

/* The tied LM head + loss_forward + loss_backward without fp32 logits (sf/model.py:449-472): a tcgen05 logits GEMM
 * hf [rows, d] x emb^T (emb bf16 [V, d]) whose epilogue keeps, per row and 256-column segment, m = max l and
 * z = sum exp(l - m), stores bf16 exp(l - m) into g [rows, ldg] and the target's fp32 logit; a combine kernel forms
 * row_loss[r] = logsumexp(l_r) - l_r[t_r] and the per-segment factors; a rescale pass turns g in place into
 * bf16((softmax(l_r) - onehot(t_r)) * inv_s) -- the operand of the d_hf = g emb GEMM.
 * stats_ws: float [rows, 2 * nseg]; coef_ws: float [rows, nseg]; tl_ws: float [rows]; nseg = lx_lm_head_ce_nseg(V). */
int lx_lm_head_ce_nseg(int V);
int lx_lm_head_ce(const uint16_t* hf, int ld_hf, int rows, int d, const uint16_t* emb, int V, const int64_t* targets,
                  float inv_s, uint16_t* g, int ldg, float* stats_ws, float* coef_ws, float* tl_ws, float* row_loss,
                  lx_stream_t stream);

/* layernorm_backward (sf/autograd.py:61-66): dx_accum += LN'(dy), dy bf16 or fp32 (dy_is_f32);
 * optionally also writes bf16(dx_accum) to dx_bf16 (the next GEMM's operand). */
int lx_layernorm_bwd(const void* dy, int dy_is_f32, const float* x, const float* gamma, const float* mean,
                     const float* inv_std, int M, int d, float* dx_accum, uint16_t* dx_bf16, lx_stream_t stream);


/* ------------------------------------------------------------------ exposer oracle mode (verification)
 * exact_attention + block_mass (sf/exposer.py:47-68): q, k fp32 rows [n_items*s, ld] (head h at columns
 * h*hd; the frozen projections x W_Q + b_Q, x W_K + b_K, no LoRA). mass: float64 [n_items, H, n_b, n_b],
 * the per-head softmax probabilities (float64, like the reference) summed over each block. */
size_t lx_exact_mass_smem(int s, int hd);
int lx_exact_block_mass(const float* q, const float* k, int ld, int n_items, int s, int H, int hd, int n_b,
                        double* mass, lx_stream_t stream);
/* select_pattern_by_coverage per grid (sf/exposer.py:71-91, OracleProvider._attn sf/harness.py:165-167);
 * head_sum = 1 sums the heads' grids first (ShadowyProvider._attn sf/harness.py:183-187) and writes the
 * one choice to every head. pattern_idx int32 [n_items, H]. */
int lx_select_by_coverage(const double* mass, int n_items, int H, int n_b, const int32_t* pool_kind,
                          const int32_t* pool_param, int n_pool, double tau, int head_sum, int32_t* pattern_idx,
                          lx_stream_t stream);
/* block_importance (sf/exposer.py:94-98): imp fp32 [n_items, ceil(n_cols/blk)] = max over the item's s
 * rows and the block's columns of |relu(z)|; z fp32 rows [n_items*s, ldz]. */
int lx_block_importance(const float* z, int ldz, int n_items, int s, int n_cols, int blk, float* imp,
                        lx_stream_t stream);
/* filter_neuron_blocks (sf/exposer.py:101-111) per item: bit b of bits [n_items, ceil(n_blk/32)] set iff
 * (double)imp[b] > theta * peak; all-zero importance -> no bits. Lower with lx_mask_compact. */
int lx_filter_neuron_blocks(const float* imp, int n_items, int n_blk, double theta, uint32_t* bits,
                            lx_stream_t stream);


/* ------------------------------------------------------------------ offline predictor pipeline
 * mlp_truth_labels (sf/predictor.py:251-259): bits [rows, ceil(ceil(n_cols/blk)/32)], bit b of row t set
 * iff some z[t, c] > 0 with c in block b; z fp32 rows [rows, ldz]. */
int lx_block_activity(const float* z, int ldz, int rows, int n_cols, int blk, uint32_t* bits, lx_stream_t stream);
/* the weighted logistic loss of train_mlp_predictor (sf/predictor.py:281-289) on fp32 logits [rows, ld]
 * against label bits (lx_block_activity layout): d_logits fp32 [rows, ldd] = dL/dlogits / (rows*n_blk),
 * row_loss float64 [rows] = the row's summed loss (mean = sum(row_loss) / (rows*n_blk)). */
int lx_weighted_bce(const float* logits, int ld, int rows, int n_blk, const uint32_t* labels, float pos_w,
                    float* d_logits, int ldd, double* row_loss, lx_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
