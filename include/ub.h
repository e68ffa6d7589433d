/*
 * ub.h -- C ABI of the unpadded-BERT data-parallel hot path for NVIDIA B200 (sm_100a).
 *
 * Paper: "Boosting Distributed Training Performance of the Unpadded BERT Model",
 * arXiv 2208.08124.  Citations "P:<n>" are lines of the paper text;
 * readings "R<k>" are listed in DESIGN.md §2.
 *
 * Conventions (all entry points):
 *   - Plain C types only.  Device pointers are CUDA device addresses; "h_" pointers are
 *     host memory.  `stream` is a cudaStream_t handle passed as void* (NULL = legacy
 *     default stream).
 *   - Ownership: the caller allocates and frees every buffer and keeps it alive until
 *     the work enqueued on `stream` has completed.  The library never allocates caller
 *     memory; the only library-owned object is `ub_comm`.
 *   - Asynchrony: device entry points only enqueue work on `stream` and never
 *     synchronise the host (the method exists to avoid host<->device syncs).
 *     The exceptions are ub_balance_exchange / ub_exchange_finish (documented there).
 *   - Errors: arguments are validated on the host before anything is launched; on a
 *     non-OK status nothing was enqueued and ub_last_error() returns a thread-local
 *     message.  Device-resident data (cu_seqlens monotonicity, lengths <= max_seqlen)
 *     is NOT validated on the fast path: that would need a sync.
 *   - Packed ("unpadded") layout (Fig. fig-storage): the batch and sequence
 *     dimensions are merged and only valid tokens are stored; cu_seqlens (the paper's
 *     batch_offset) is the int32 prefix sum [B+1] with cu[0] = 0, cu[B] = T.
 */
#ifndef UB_H_
#define UB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  UB_OK = 0,
  UB_ERR_INVALID_ARG = 1,  /* null pointer, bad enum, empty batch, length < 1, scale <= 0, p outside [0,1) */
  UB_ERR_INVALID_MASK = 2, /* non-prefix input_mask row */
  UB_ERR_CAPACITY = 3,     /* a length exceeds max_seqlen / padded capacity */
  UB_ERR_SHAPE = 4,        /* inconsistent sizes (W*B lengths, row_bytes <= 0, T mismatch) */
  UB_ERR_UNSUPPORTED = 5,  /* dtype / head_dim / device (needs sm_100) / mode limits */
  UB_ERR_CUDA = 6,         /* a CUDA runtime call failed */
  UB_ERR_NCCL = 7          /* an NCCL call failed */
} ub_status;

typedef enum { UB_BF16 = 0, UB_FP32 = 1 } ub_dtype;

/* Thread-local message describing the last non-OK status of this thread ("" if none). */
const char* ub_last_error(void);
/* Library build string (arch, version). */
const char* ub_version(void);

/* Measurement hook (bench / profiling only): record the given cudaEvent_t handles
 * immediately before and after every subsequent launch of one internal kernel, on the
 * stream it is launched on, so its device time can be read inside a larger step.
 * kernel_id: 0 = FMHA forward main kernel, 1 = FMHA backward main kernel, 2 = pad,
 * 3 = unpad.  NULL events clear the hook.  Process-wide; not thread-safe. */
ub_status ub_profile_events(int32_t kernel_id, void* start_event, void* stop_event);

/* ------------------------------------------------------------------------------------
 * batch_offset / cu_seqlens ("a prefix sum array ... to record the token number
 * of each sequence").  Host helper.
 *   h_lengths [B] int32, each 1 <= L <= max_seqlen (else UB_ERR_INVALID_ARG / _CAPACITY);
 *   h_cu [B+1] int32 output, exclusive prefix sum with trailing total.
 *   The total must fit in int32 (else UB_ERR_SHAPE).
 */
ub_status ub_cu_seqlens(const int32_t* h_lengths, int32_t B, int32_t max_seqlen, int32_t* h_cu);

/* Lengths from a padded input_mask [B, S] int32 (0/1) on the host ("The valid input
 * token number can be obtained from the input tensor input_mask").  A row that is not a
 * prefix of ones followed by zeros -> UB_ERR_INVALID_MASK. */
ub_status ub_lengths_from_mask(const int32_t* h_mask, int32_t B, int32_t S, int32_t* h_lengths);

/* ------------------------------------------------------------------------------------
 * Unpad = gather ("input data are compressed to the unpad format ... obtained by
 * the gather operator").  padded [B, S, row_bytes] -> packed [T, row_bytes]:
 *   packed[cu[b] + i] = padded[b][i]  for i < cu[b+1]-cu[b].
 * Rows are opaque row_bytes-wide records (int32 ids, bf16 hidden rows, ...).
 * d_cu: device [B+1].  T must equal cu[B] (not checked: device-resident).
 * 16-B vector path when row_bytes % 16 == 0 and both pointers are 16-B aligned,
 * else a 4-B or 1-B path (not an error).
 */
ub_status ub_unpad(const void* padded, void* packed, const int32_t* d_cu, int32_t B, int32_t S,
                   int64_t T, int64_t row_bytes, void* stream);

/* Pad = scatter ("uncompressed to the padding format by using a scatter operator").
 * packed [T, row_bytes] -> padded [B, S, row_bytes]; positions i >= L_b receive the
 * row_bytes pattern at d_pad_row (device), or zeros when d_pad_row is NULL. */
ub_status ub_pad(const void* packed, void* padded, const int32_t* d_cu, int32_t B, int32_t S,
                 int64_t T, int64_t row_bytes, const void* d_pad_row, void* stream);

/* ------------------------------------------------------------------------------------
 * Varlen fused multi-head attention, Eq. (1):
 *     O = softmax(scale * Q K^T) V   per sequence b and head h, within the sequence only
 * (unpadded FMHA over packed tokens; no cross-sequence attention, R2), with
 * optional inverted dropout on the probabilities (R4) from the counter-based Philox
 * mask of R5 keyed by (seed, offset): 8-bit decisions, 16 keys per Philox call.  The drop
 * rate APPLIED is p_eff = floor(256 p) / 256 (p = 0.1 drops 25/256 = 0.0977 of the
 * probabilities; ub_dropout_effective_p returns it) and kept values are scaled by the exact
 * inverse keep probability 1 / (1 - p_eff), so E[P~] = P.  0 < p < 1/256 (p_eff = 0: no
 * dropout would happen) is rejected with UB_ERR_INVALID_ARG.
 *
 * Work is grouped by length: a device-side plan buckets sequences by their number of
 * 128-token tiles -- the paper's groups (0,128] (128,256] (256,384] (384,512]
 * -- and one persistent launch processes the buckets longest-first, in place of the
 * paper's one-kernel-per-group multi-stream launch.
 *
 * Layouts: qkv [T, 3, H, D] (the QKV GEMM output [T, 3*H*D]); out, dout [T, H, D];
 * lse [H, T] fp32 natural log (LSE_t = max + log sum exp, before dropout);
 * dqkv [T, 3, H, D].  dtype UB_BF16 (tcgen05 tensor-core path, D == 64) or UB_FP32
 * (exact-fp32 CUDA-core path, D <= 128, for tiny checks).
 * ws: device workspace of ub_fmha_workspace_bytes() bytes, 256-B aligned, owned by the
 * caller; contents need no initialisation and are scratch between calls (one call at a
 * time per workspace).
 */
typedef struct {
  int32_t B;          /* number of sequences (>= 1) */
  int64_t T;          /* total valid tokens = cu[B] (>= 1) */
  int32_t max_seqlen; /* >= every length; bounds the per-sequence tile count */
  int32_t heads;      /* H >= 1 */
  int32_t head_dim;   /* D: 64 for UB_BF16; 1..128 for UB_FP32 */
  float scale;        /* > 0; 1/sqrt(D) in BERT (R1) */
  float p_dropout;    /* 0 (disables the RNG entirely) or in [1/256, 1); applied as
                         floor(256 p) / 256 (R5), see ub_dropout_effective_p */
  uint64_t seed;      /* Philox key (R5) */
  uint64_t offset;    /* Philox counter word 3 (low 32 bits used) */
  int32_t dtype;      /* ub_dtype */
  int32_t num_ctas;   /* persistent grid size; 0 = one CTA per SM.  Set below the SM count to
                         leave SMs to concurrent side-stream work (the overlapped exchange) */
  const void* dropout_mask; /* p > 0 only: the keep bits ub_dropout_mask wrote for these params and
                         cu_seqlens (device, ub_dropout_mask_bytes), read by the forward and the
                         backward; NULL = the kernels regenerate them by Philox as they go (the
                         same bits: results are bitwise identical either way) */
  const int32_t* schedule; /* device, NULL = the kernels' own snake deal of the length-bucketed
                         work items; else the ub_fmha_schedule result for THIS call's direction,
                         lengths, heads, max_seqlen and grid (results are bitwise identical; only
                         the makespan changes).  Ignored above 512 sequences; a schedule built for
                         another grid size falls back to the snake deal */
} ub_fmha_params;

size_t ub_fmha_workspace_bytes(const ub_fmha_params* prm, int is_bwd);

/* Static schedule of the persistent forward / backward grids (an input-only operator, P:402:
 * it needs the batch's lengths only, which the padding-exchange planner holds one step ahead,
 * P:376-381).  Longest-processing-time-first list scheduling of the work items -- backward:
 * (sequence, head); forward: (sequence, head, pair of 128-row query tiles) -- by an estimated
 * cost (backward nt^2 + 0.3 nt + 0.5 tile pairs for nt = ceil(L / 128); forward 1.0 (two tiles)
 * or 0.7 (one) per key step + 0.3), each to the least-loaded of `grid` CTAs (ties: lowest
 * id), in place of the kernels' snake deal (items longest first, round r dealt in alternating
 * direction).  Pure host function; deterministic.
 * h_lengths [B] host (the post-exchange lengths in cu_seqlens order, 0 <= L <= max_seqlen
 * <= 2048, else UB_ERR_CAPACITY / UB_ERR_UNSUPPORTED); grid = the launch's CTA count (num_ctas,
 * or the SM count); is_bwd selects the item kind.  Output h_sched (host, int32): [0] = grid,
 * [1 .. grid+1] = offsets (CTA c owns entries off[c] .. off[c+1] - 1), then the entries:
 * backward b*H + h, forward (b*H + h)*8 + g (query tiles 2g, 2g+1).  cap_ints >=
 * ub_fmha_schedule_ints(...) else UB_ERR_SHAPE; a CTA with more than 63 items (the kernels'
 * table) -> UB_ERR_UNSUPPORTED.  Copy it to the device and pass it as prm->schedule. */
size_t ub_fmha_schedule_ints(int32_t B, int32_t heads, int32_t max_seqlen, int32_t grid, int32_t is_bwd);
ub_status ub_fmha_schedule(const int32_t* h_lengths, int32_t B, int32_t heads, int32_t max_seqlen, int32_t grid,
                           int32_t is_bwd, int32_t* h_sched, size_t cap_ints);

/* The attention-dropout keep mask of R5 materialised as bits (an input-only operator, P:402:
 * it needs cu_seqlens, seed and offset only, so it can be produced while the batch is still
 * being exchanged, once per step for both directions).  Writes two layouts into d_mask
 * (device, ub_dropout_mask_bytes(prm) bytes, 16-B aligned), MT = ceil(max_seqlen / 128),
 * 32-bit words with the packed row innermost (coalesced):
 *   query-major [H][MT][4][T]: bit e of word [h][kt][w][t] = keep(query row t, key 128 kt + 32 w + e)
 *   key-major   [H][MT][4][T]: bit e of word [h][it][c][t] = keep(query 128 it + 32 c + e, key row t)
 * (t packed rows, keys / queries counted inside the sequence; words of rows past a sequence
 * end are left unwritten).  Needs 1/256 <= p < 1 (UB_ERR_INVALID_ARG); bf16 path.  Async. */
size_t ub_dropout_mask_bytes(const ub_fmha_params* prm);
ub_status ub_dropout_mask(const ub_fmha_params* prm, const int32_t* d_cu, void* d_mask, void* stream);
/* ub_dropout_mask with flags.  UB_MASK_OVERLAP_PREVIOUS: launched as a programmatic dependent of
 * the kernel before it on the stream and never waiting for it, so its CTAs fill the SMs that
 * kernel's tail leaves idle -- the CALLER guarantees that the previous kernel neither writes
 * d_cu nor reads or writes d_mask (e.g. the previous step's backward reading the other one of
 * two mask buffers).  Unknown bits -> UB_ERR_INVALID_ARG. */
#define UB_MASK_OVERLAP_PREVIOUS 1
ub_status ub_dropout_mask_ex(const ub_fmha_params* prm, const int32_t* d_cu, void* d_mask, int32_t flags,
                             void* stream);

/* The attention-dropout rate the FMHA kernels apply for a requested p (R5): floor(256 p) / 256
 * with p taken as float32; 0 for p <= 0.  (The Dropout_Add_LayerNorm kernels use 16-bit
 * decisions: floor(65536 p) / 65536, see ub_dal_fwd.)  Pure host function. */
double ub_dropout_effective_p(float p_dropout, int32_t bits);

ub_status ub_varlen_fmha_fwd(const ub_fmha_params* prm, const void* qkv, const int32_t* d_cu,
                             void* out, float* lse, void* ws, void* stream);

/* Forward with the padding scatter fused in (a7 + a9): as ub_varlen_fmha_fwd, and the
 * epilogue also writes O to padded [B, S, H, 64] bf16 at row b*S + i, with zeros in rows
 * i >= L_b (the ub_pad result for a NULL pad row), from the same staged tiles -- the separate
 * pad pass (a read of O and a write of the padded tensor) disappears.  S >= max_seqlen and
 * S % 32 == 0 else UB_ERR_SHAPE; bf16 only (UB_ERR_UNSUPPORTED). */
ub_status ub_varlen_fmha_fwd_pad(const ub_fmha_params* prm, const void* qkv, const int32_t* d_cu, void* out,
                                 float* lse, void* padded, int32_t S, void* ws, void* stream);

/* Backward: given dO, returns dQ, dK, dV (R4/R5 dropout replayed from the same key):
 *   Delta_i = sum_d dO_id O_id;  dV = P~^T dO;  dP = (dO V^T) * M/(1-p);
 *   dS = P * (dP - Delta);  dQ = scale dS K;  dK = scale dS^T Q. */
ub_status ub_varlen_fmha_bwd(const ub_fmha_params* prm, const void* qkv, const void* out,
                             const float* lse, const void* dout, const int32_t* d_cu,
                             void* dqkv, void* ws, void* stream);

/* ------------------------------------------------------------------------------------
 * Dropout_Add_LayerNorm (§IV-C-1 kernel fusion; SURVEY §8(f) NEXT-1 piece): one
 * forward kernel, two backward kernels, on packed rows (no padding).
 *   z = res + a * keep / (1 - p_eff),  y = (z - mean) * rstd * gamma + beta,  rstd = 1/sqrt(var + eps)
 *   keep: Philox4x32-10, key = seed, counter = (col >> 3, row, 0xDA100000, offset),
 *   16-bit half (col & 1) of word ((col & 7) >> 1) >= thr = floor(p * 65536)   (reading R21);
 *   p_eff = thr / 65536 is the applied drop rate (ub_dropout_effective_p(p, 16)), so the
 *   scale is the exact inverse keep probability; 0 < p < 1/65536 is UB_ERR_INVALID_ARG
 * Layouts (device, caller-allocated, 16-B aligned): a, res, y, dy, da, dres [T, E] bf16;
 * gamma, beta [E] bf16; mean, rstd [T] fp32 (written by the forward, read by the backward);
 * dgamma, dbeta [E] fp32.  E a multiple of 8 in [8, 2048] else UB_ERR_UNSUPPORTED;
 * p in [0, 1), eps > 0 else UB_ERR_INVALID_ARG.  The mask is regenerated, never stored.
 * Backward workspace: ub_dal_bwd_workspace_bytes(T, E) bytes (per-CTA partial sums; the
 * reduction order is fixed, so dgamma / dbeta are bitwise deterministic).  Async on stream. */
ub_status ub_dal_fwd(const void* a, const void* res, const void* gamma, const void* beta, int64_t T, int32_t E,
                     float p_dropout, float eps, uint64_t seed, uint64_t offset, void* y, float* mean, float* rstd,
                     void* stream);
size_t ub_dal_bwd_workspace_bytes(int64_t T, int32_t E);
ub_status ub_dal_bwd(const void* dy, const void* a, const void* res, const void* gamma, const float* mean,
                     const float* rstd, int64_t T, int32_t E, float p_dropout, uint64_t seed, uint64_t offset,
                     void* da, void* dres, float* dgamma, float* dbeta, void* ws, void* stream);

/* ------------------------------------------------------------------------------------
 * Unpadded BERT embedding (P:525-535 embedding backward with packed atomics;
 * SURVEY §8(f) NEXT-4), on packed tokens (reading R23):
 *   ub_embedding_fwd: out[t] = W_word[ids[t]] + W_pos[pos[t]] + W_type[seg[t]]  (bf16 [T, E])
 *   ub_embedding_bwd: dW_word[ids[t]] += dout[t], dW_pos[pos[t]] += dout[t],
 *                     dW_type[seg[t]] += dout[t]  -- ACCUMULATES into the caller's dW
 *                     (zero them first); grad_dtype UB_FP32 (16-B fp32 vector reductions)
 *                     or UB_BF16 (bf16x2 vector reductions, the paper's packed-atomic form,
 *                     P:535; less precise for frequent tokens).  Summation order is not
 *                     fixed (atomics): results agree with the oracle within rounding.  The
 *                     rows of each CTA's most frequent word ids (up to 4, found among its
 *                     first 128 tokens) are summed in shared memory first and reduced to
 *                     dW_word once per CTA (skewed vocabularies contend on those rows).
 * ids / pos / seg: int32 [T] device, values in range (not validated on the device, like
 * cu_seqlens); tables bf16 [rows, E]; E a multiple of 8 in [8, 2048] else UB_ERR_UNSUPPORTED;
 * n_type (token-type rows) in [1, 2]; 16-B aligned arrays.  Async on stream. */
ub_status ub_embedding_fwd(const int32_t* ids, const int32_t* pos, const int32_t* seg, const void* w_word,
                           const void* w_pos, const void* w_type, int64_t T, int32_t E, void* out, void* stream);
ub_status ub_embedding_bwd(const void* dout, const int32_t* ids, const int32_t* pos, const int32_t* seg, int64_t T,
                           int32_t E, int32_t n_type, int32_t grad_dtype, void* dw_word, void* dw_pos, void* dw_type,
                           void* stream);

/* ------------------------------------------------------------------------------------
 * Linear layers (P:410 Linear fusion through cuBLASLt; P:416 residual gradient through the
 * GEMM's beta), row-major packed rows, bf16 activations / weights, fp32 accumulation:
 *   ub_linear_fwd: y[T,N] = x[T,K] W[N,K]^T + b[N]    (b may be NULL; bias in the epilogue)
 *   ub_linear_bwd: dx[T,K] = dy[T,N] W[N,K] (+ res_grad[T,K] if non-NULL, beta = 1);
 *                  dW[N,K] = dy^T x (fp32), db[N] = sum_t dy (fp32, bias-gradient epilogue);
 *                  dx or dW may be NULL to skip that GEMM; db needs dW.
 * K, N multiples of 8; T >= 1 else UB_ERR_SHAPE.  ws: ub_linear_workspace_bytes() bytes
 * (cuBLASLt workspace).  No algorithm for the shape -> UB_ERR_UNSUPPORTED. */
size_t ub_linear_workspace_bytes(void);
ub_status ub_linear_fwd(const void* x, const void* W, const void* b, int64_t T, int32_t K, int32_t N, void* y,
                        void* ws, void* stream);
ub_status ub_linear_bwd(const void* dy, const void* x, const void* W, const void* res_grad, int64_t T, int32_t K,
                        int32_t N, void* dx, float* dW, float* db, void* ws, void* stream);

/* ------------------------------------------------------------------------------------
 * Unpadded encoder attention sub-layer (BASELINE config 4), packed rows:
 *   qkv = x Wqkv^T + bqkv;  ctx = varlen_fmha(qkv) (p_attn, R5);  a = ctx Wo^T + bo;
 *   y = LayerNorm(x + dropout(a)) (p_hidden, R21)
 * Layouts: x, y, dy, dx, ctx, a [T, hidden] bf16; qkv [T, 3*hidden] bf16 (= [T, 3, H, 64]);
 * Wqkv [3*hidden, hidden], Wo [hidden, hidden], bqkv [3*hidden], bo, gamma, beta [hidden]
 * bf16; lse [H, T], mean, rstd [T] fp32; weight / bias / LN gradients fp32.  qkv, ctx, lse,
 * a, mean, rstd are written by the forward and read by the backward (caller-owned).
 * hidden / heads must be 64 and hidden <= 2048 (else UB_ERR_UNSUPPORTED).  ws:
 * ub_encoder_attn_workspace_bytes(prm, is_bwd) bytes, 256-B aligned. */
typedef struct {
  int32_t B;          /* sequences */
  int64_t T;          /* tokens = cu[B] */
  int32_t max_seqlen;
  int32_t hidden;     /* 1024 for BERT-large */
  int32_t heads;      /* 16 for BERT-large */
  float p_attn;       /* attention-probability dropout */
  float p_hidden;     /* hidden dropout before the residual add */
  float eps;          /* LayerNorm epsilon (1e-12 in BERT) */
  uint64_t seed, offset;
  int32_t num_ctas;   /* FMHA persistent grid, 0 = all SMs */
} ub_encoder_params;
size_t ub_encoder_attn_workspace_bytes(const ub_encoder_params* prm, int is_bwd);
ub_status ub_encoder_attn_fwd(const ub_encoder_params* prm, const void* x, const int32_t* d_cu, const void* w_qkv,
                              const void* b_qkv, const void* w_o, const void* b_o, const void* gamma,
                              const void* beta, void* qkv, void* ctx, float* lse, void* a, float* mean, float* rstd,
                              void* y, void* ws, void* stream);
ub_status ub_encoder_attn_bwd(const ub_encoder_params* prm, const void* x, const int32_t* d_cu, const void* w_qkv,
                              const void* w_o, const void* gamma, const void* qkv, const void* ctx, const float* lse,
                              const void* a, const float* mean, const float* rstd, const void* dy, void* dx,
                              float* dw_qkv, float* db_qkv, float* dw_o, float* db_o, float* dgamma, float* dbeta,
                              void* ws, void* stream);

/* ------------------------------------------------------------------------------------
 * Padding-exchange balancer (§IV-B-1).  Pure host function: deterministic,
 * byte-identical on every rank given the same all-gathered lengths.
 *   h_all_lengths [W*B]: rank-major all-gather of the valid lengths, global id g = r*B+k.
 *   UB_BAL_PAPER: sort ids by (length asc, id asc) (R11), rank i takes sorted
 *     positions i, i+W, i+2W, ... in that order (R12).
 *   UB_BAL_SNAKE: same sort, round r dealt to ranks 0..W-1 (r even) or W-1..0 (r odd).
 *   UB_BAL_EXACT_SMALL: exhaustive min-max search over equal-cardinality partitions,
 *     W*B <= 12 else UB_ERR_UNSUPPORTED; ties -> lexicographically smallest perm (R15).
 *   UB_BAL_LPT: cardinality-constrained longest-processing-time greedy on tokens with
 *     (max, min) swap refinement, never worse than UB_BAL_PAPER (it falls back to the
 *     paper's plan when that has a strictly smaller maximum); samples on a rank listed by
 *     (length asc, id asc).  A beyond-the-paper variant of P:359 (
 *     steps in DESIGN.md and oracle/balance.py balance_lpt).
 *   UB_BAL_STAY (reading R25, NEXT-2 locality-aware): every rank starts with its own samples
 *     and UB_BAL_LPT's swap refinement balances the tokens, so only the swapped samples move
 *     (a few per cent of the tokens instead of (W-1)/W); ranks list samples by (length, id).
 *   | UB_BAL_LOCALITY (flag, OR-ed into any mode; reading R24, NEXT-2 beyond the paper): the
 *     mode's W groups are then handed to the ranks so that the most tokens stay on their
 *     source rank (group i -> rank sigma[i] maximising the kept tokens; exact, ties ->
 *     lexicographically smallest sigma; see ub_balance_relabel).  Loads are unchanged.
 * Outputs (host, caller-allocated):
 *   h_perm [W*B]         perm[r*B + k] = global id of the k-th sample placed on rank r
 *   h_rank_tokens [W]    tokens per rank after the exchange (may be NULL)
 *   h_send_samples [W*W] samples moving src -> dst, index src*W + dst (may be NULL)
 *   h_send_tokens [W*W]  tokens moving src -> dst (may be NULL)
 * Errors: W < 1, B < 1, a length < 1 -> INVALID_ARG; length > max_seqlen -> CAPACITY.
 */
typedef enum { UB_BAL_PAPER = 0, UB_BAL_SNAKE = 1, UB_BAL_EXACT_SMALL = 2, UB_BAL_LPT = 3, UB_BAL_STAY = 4 } ub_bal_mode;
#define UB_BAL_LOCALITY 0x100

ub_status ub_balance_plan(const int32_t* h_all_lengths, int32_t W, int32_t B, int32_t max_seqlen,
                          int32_t mode, int32_t* h_perm, int64_t* h_rank_tokens,
                          int32_t* h_send_samples, int64_t* h_send_tokens);

/* Locality relabeling of a plan (reading R24): the W groups of h_perm
 * (rank r's block perm[r*B .. r*B+B-1]) keep their contents and order but move to the ranks
 * sigma[0..W-1] that maximise the tokens staying home, sum_i M[i][sigma[i]] with M[i][r] =
 * tokens of group i whose source rank (g / B) is r -- an assignment problem solved exactly
 * by dynamic programming over rank subsets; ties -> lexicographically smallest sigma.
 * h_perm is rewritten in place; h_kept_before / h_kept_after (may be NULL) = kept tokens.
 * W <= 20 (2^W states) else UB_ERR_UNSUPPORTED; a perm that is not a permutation -> SHAPE. */
ub_status ub_balance_relabel(const int32_t* h_all_lengths, int32_t W, int32_t B, int32_t* h_perm,
                             int64_t* h_kept_before, int64_t* h_kept_after);

/* Cost-aware balancing (NEXT-2): UB_BAL_LPT's steps on the integer per-sample cost
 * alpha*L + beta*L^2 -- the linear layers grow with L, attention with L^2 (Eq. 1).
 * For BERT-large one layer's fwd flops per sample are ~ 4096*L*(2048 + L), i.e.
 * alpha = 2048, beta = 1.  h_rank_cost [W] (may be NULL) = summed cost per rank.
 * Errors: as ub_balance_plan; alpha < 0, beta < 0, both 0 or above 2^30 -> INVALID_ARG. */
ub_status ub_balance_plan_weighted(const int32_t* h_all_lengths, int32_t W, int32_t B, int32_t max_seqlen,
                                   int64_t alpha, int64_t beta, int32_t* h_perm, int64_t* h_rank_cost);

/* ------------------------------------------------------------------------------------
 * Exchange data movement (P:355-359 steps 1 and 3, without the padded all-gather: only
 * lengths are all-gathered; each sample's packed token records then travel once).
 *
 * ub_exchange_tables (host): copy table for rank `rank`, from the all-gathered lengths
 * and the plan.  h_tab [5*B] int64 = {src_tok[B], len[B], dst_tok[B], src_smp[B], dst_smp[B]}
 * (token offsets in records, sample offsets in records).
 *   is_unpack == 0 (pack): source = this rank's packed batch (sample k at its cu[k]);
 *     destination = the send buffer, grouped by destination rank ascending, each group
 *     in the destination's perm order.  h_counts [W] (may be NULL) = token records sent
 *     to each destination; h_scounts [W] = samples sent to each destination.
 *   is_unpack == 1 (unpack): source = the receive buffer (per-source chunks, source rank
 *     ascending, each chunk in this rank's perm order); destination = perm order.
 *     h_counts [W] = token records received from each source; h_scounts [W] samples.
 *   *h_total_tokens (may be NULL) = tokens packed (pack) / received (unpack).
 * ub_exchange_copy (device): for each of the B table entries copies len*rec_bytes from
 *   src_tokens + src_tok*rec_bytes to dst_tokens + dst_tok*rec_bytes and srec_bytes from
 *   src_samples + src_smp*srec_bytes to dst_samples + dst_smp*srec_bytes.  d_tab is the
 *   table in device memory.  srec_bytes may be 0 (then sample pointers may be NULL).
 */
ub_status ub_exchange_tables(const int32_t* h_all_lengths, const int32_t* h_perm, int32_t W,
                             int32_t B, int32_t rank, int32_t is_unpack, int64_t* h_tab,
                             int64_t* h_counts, int64_t* h_scounts, int64_t* h_total_tokens);
ub_status ub_exchange_copy(const void* src_tokens, void* dst_tokens, const void* src_samples,
                           void* dst_samples, const int64_t* d_tab, int32_t B, int64_t rec_bytes,
                           int64_t srec_bytes, void* stream);

/* ------------------------------------------------------------------------------------
 * Checked mode (SURVEY §8(b) "Errors": device-resident data is not validated on the fast
 * path; a debug switch validates it on the device and reports after a sync -- tests only).
 *
 * ub_validate_cu_seqlens (device, async): one CTA checks the device cu_seqlens [B+1] and
 *   writes *d_flag (device int32): 0 valid, 1 cu[0] != 0, 2 not monotone, 3 a length >
 *   max_seqlen, 4 cu[B] > T.  The caller reads the flag after synchronising.
 * ub_set_checked (host): on != 0 makes ub_unpad / ub_pad (max_seqlen = S) and the FMHA
 *   entry points run that check first, synchronise the stream and return CAPACITY (code 3)
 *   or INVALID_ARG (codes 1, 2, 4) instead of launching.  Also switched on by UB_CHECKED=1
 *   in the environment.  Off by default: it costs a host synchronisation per call.
 */
ub_status ub_validate_cu_seqlens(const int32_t* d_cu, int32_t B, int32_t max_seqlen, int64_t T,
                                 int32_t* d_flag, void* stream);
ub_status ub_set_checked(int32_t on);

/* ------------------------------------------------------------------------------------
 * Pull-based exchange (the data movement of P:355-359 step 3 done as
 * one gather): every rank copies its perm-ordered samples directly out of the peers'
 * packed token buffers, mapped into its address space by CUDA IPC -- the all-to-all-v
 * (a4) and the reorder (a5) in one kernel, no staging buffers, no NCCL kernels.
 *
 * ub_ipc_export (host): writes UB_IPC_HANDLE_BYTES bytes describing the device buffer that
 *   starts at d_ptr (the CUDA IPC handle of its allocation plus d_ptr's offset in it), to be
 *   sent to the other ranks (e.g. over torch.distributed).  d_ptr must come from cudaMalloc
 *   (directly or through a caching allocator).  Errors: not device memory -> INVALID_ARG.
 * ub_ipc_import (host): maps a peer's exported buffer; *d_ptr = the buffer in this process,
 *   *d_base = the mapping to pass to ub_ipc_close when done.  A handle exported by this
 *   process cannot be imported by it (CUDA returns an error -> UB_ERR_CUDA).
 * ub_exchange_pull_table (host): for rank `rank`, from the all-gathered lengths and the plan
 *   (perm as ub_balance_plan writes it), h_tab [6*B] int64 = {src_rank[B], src_tok[B],
 *   len[B], dst_tok[B], src_smp[B], dst_smp[B]}: output sample k (perm order) is local
 *   sample src_smp of rank src_rank, whose token records start at record src_tok of that
 *   rank's packed buffer (its local cu_seqlens); it lands at record dst_tok.
 *   *h_total_tokens (may be NULL) = records this rank receives.  Errors: perm not a
 *   permutation -> SHAPE; negative length -> INVALID_ARG.
 * ub_exchange_pull (device, async on `stream`): d_peer_tokens / d_peer_samples are DEVICE
 *   arrays of W pointers (this rank's own buffers at its own index); 16-B aligned bases take
 *   the vector path when rec_bytes % 16 == 0, a misaligned peer base is detected per sample
 *   on the device and copied bytewise (slower, never a fault); d_tab is the pull table in
 *   device memory.  One CTA per output
 *   sample.  d_ready (may be NULL): DEVICE array of W pointers to the ranks' "buffer
 *   published" flags (IPC-mapped); each CTA first waits, with system-scope acquire, until
 *   the flag of its source rank is >= wait_value, so the host never waits.  Without flags
 *   the caller orders the peers' writes before the call (a barrier).
 * ub_signal (device, async): after every earlier write of `stream`, stores `value` to the
 *   uint32 flag with system-scope release (a rank publishes its buffer, or its completed
 *   pull, to the other processes).
 * ub_wait_flags (device, async): `stream` waits until each of the n flags (DEVICE array of
 *   pointers) is >= value, e.g. before overwriting a buffer the peers may still be reading.
 *   Flags are monotone counters (a step number); the waits spin on the GPU, one CTA.
 */
#define UB_IPC_HANDLE_BYTES 128
ub_status ub_ipc_export(const void* d_ptr, void* h_handle);
ub_status ub_ipc_import(const void* h_handle, void** d_ptr, void** d_base);
ub_status ub_ipc_close(void* d_base);
ub_status ub_exchange_pull_table(const int32_t* h_all_lengths, const int32_t* h_perm, int32_t W,
                                 int32_t B, int32_t rank, int64_t* h_tab, int64_t* h_total_tokens);
ub_status ub_exchange_pull(const void* const* d_peer_tokens, const void* const* d_peer_samples,
                           const uint32_t* const* d_ready, uint32_t wait_value, const int64_t* d_tab,
                           int32_t B, int64_t rec_bytes, int64_t srec_bytes, void* dst_tokens,
                           void* dst_samples, void* stream);
ub_status ub_signal(uint32_t* d_flag, uint32_t value, void* stream);
ub_status ub_wait_flags(const uint32_t* const* d_flags, int32_t n, uint32_t value, void* stream);

/* NCCL communicator (NCCL over NVLink 5 / NVSwitch).  nccl_unique_id: the 128-byte
 * ncclUniqueId produced by ub_comm_unique_id() on rank 0 and broadcast by the caller
 * (e.g. over a torch.distributed process group).  Must be called with the CUDA device
 * of this rank current. */
ub_status ub_comm_unique_id(void* out_id_128);
ub_status ub_comm_init(void** out_comm, const void* nccl_unique_id, int32_t W, int32_t rank);
ub_status ub_comm_destroy(void* comm);

/* Options of a communicator (host, between exchanges).  UB_COMM_FORCE_NCCL: the part of the
 * exchange a rank keeps for itself, and a one-rank all-gather, also travel through NCCL
 * (ncclAllGather; ncclSend / ncclRecv to itself inside the step's group) instead of device
 * copies -- the collective data plane of P:355-359 then runs even on a one-GPU box (tests);
 * the default (0) copies the self chunk on the device.  Also set by UB_EXCHANGE_FORCE_NCCL=1
 * at ub_comm_init.  Unknown bits -> UB_ERR_INVALID_ARG. */
#define UB_COMM_FORCE_NCCL 1
/* UB_COMM_HOST_PROFILE: accumulate the host time ub_exchange_finish spends per phase (read back
 * by ub_comm_host_profile; setting it restarts the accumulation).  Also on with
 * UB_EXCHANGE_TRACE=1, which prints the per-finish means when the communicator is destroyed. */
#define UB_COMM_HOST_PROFILE 2
ub_status ub_comm_set_options(void* comm, int32_t flags);
/* Host microseconds accumulated over the finishes since profiling started, per phase, in
 * out_us[0..n_out): 0 wait for this slot's lengths (the one host wait: the GPU's pace, not
 * host work), 1 plan, 2 wait for the previous finish's staging copies, 3 tables,
 * 4 pack launch, 5 NCCL send/recv enqueue, 6 gather + cu_seqlens launch; *out_finishes = the
 * number of finishes.  Host-only, no synchronisation. */
ub_status ub_comm_host_profile(void* comm, double* out_us, int32_t n_out, int64_t* out_finishes);
/* Number of NCCL calls (all-gathers, sends, receives) this communicator has enqueued so far
 * (host counter; evidence that the collective data plane ran). */
ub_status ub_comm_nccl_ops(void* comm, int64_t* out);

/* All-gather of B int32 lengths (P:355 step 1, lengths only): d_my_lengths [B] ->
 * d_all_lengths [W*B] rank-major, on `stream`. */
ub_status ub_allgather_lengths(void* comm, const int32_t* d_my_lengths, int32_t* d_all_lengths,
                               int32_t B, void* stream);

/* The whole exchange for one step, on `side_stream` (one mini-batch ahead,
 * overlapped with the compute stream):
 *   1. all-gather lengths (NCCL), 2. D2H of the W*B lengths and a host wait on the side
 *   stream only (send/recv counts must be known on the host -- the single host sync of
 *   the library; it never waits on the compute stream), 3. ub_balance_plan, 4. pack,
 *   5. grouped ncclSend/ncclRecv (all-to-all-v of packed token records and sample
 *   records), 6. unpack into perm order, 7. H2D of the new cu_seqlens.
 * Inputs: d_my_lengths [B]; d_my_tokens [T_mine, rec]; d_my_samples [B, srec].
 * Outputs: d_out_tokens [capacity_tokens, rec]; d_out_samples [B, srec]; d_out_cu [B+1];
 *   h_perm [W*B] (may be NULL); *h_out_T.  Capacity: out tokens must fit
 *   capacity_tokens (else UB_ERR_CAPACITY, nothing moved).
 * ws: device workspace of ub_exchange_workspace_bytes(W, B, capacity_tokens, rec, srec).
 */
size_t ub_exchange_workspace_bytes(int32_t W, int32_t B, int64_t capacity_tokens, int64_t rec_bytes,
                                   int64_t srec_bytes);
ub_status ub_balance_exchange(void* comm, int32_t mode, int32_t B, int32_t max_seqlen,
                              const int32_t* d_my_lengths, const void* d_my_tokens,
                              const void* d_my_samples, int64_t rec_bytes, int64_t srec_bytes,
                              int64_t capacity_tokens, void* d_out_tokens, void* d_out_samples,
                              int32_t* d_out_cu, int32_t* h_perm, int64_t* h_out_T, void* ws,
                              void* side_stream);

/* The same exchange split in two so that the host never waits on work it has just
 * enqueued (the balancing of mini-batch n+1 runs while n computes).
 * ub_balance_exchange == ub_exchange_begin + ub_exchange_finish on an internal slot.
 *
 * ub_exchange_begin (device, no host wait): step 1 -- all-gather of d_my_lengths [B] into
 *   slot `slot` (0 <= slot < UB_EXCHANGE_SLOTS) of the communicator's pinned ring, D2H on
 *   `stream`, and an event recorded behind it.  The slot must not hold an unfinished
 *   begin (UB_ERR_INVALID_ARG).  ws as for ub_balance_exchange (only its front is used).
 * ub_exchange_finish: waits (host) for that slot's event only, then steps 3-7 exactly as
 *   ub_balance_exchange on `stream`, and frees the slot.  B must equal the begin's B.
 *   Issue the begin of step n+1 one step before its finish: by then its event has fired
 *   and the wait is free.  Outputs, capacity and errors as ub_balance_exchange.
 * Collective calls: every rank issues the same begin/finish sequence. */
#define UB_EXCHANGE_SLOTS 8
ub_status ub_exchange_begin(void* comm, int32_t slot, int32_t B, const int32_t* d_my_lengths, void* ws,
                            void* stream);
ub_status ub_exchange_finish(void* comm, int32_t slot, int32_t mode, int32_t B, int32_t max_seqlen,
                             const void* d_my_tokens, const void* d_my_samples, int64_t rec_bytes,
                             int64_t srec_bytes, int64_t capacity_tokens, void* d_out_tokens,
                             void* d_out_samples, int32_t* d_out_cu, int32_t* h_perm, int64_t* h_out_T,
                             void* ws, void* stream);
/* The W*B all-gathered lengths (rank-major, global id r*B + k) of slot `slot`'s last finished
 * exchange, copied to h_out (host, W*B int32) -- valid until that slot's next begin.  With the
 * finish's perm, a rank's post-exchange lengths are h_out[perm[rank*B + k]]: the input of
 * ub_fmha_schedule for the batch the exchange delivered.  A slot with an unfinished begin, or
 * B above the communicator's staging, -> UB_ERR_INVALID_ARG / UB_ERR_SHAPE.  Host only. */
ub_status ub_exchange_slot_lengths(void* comm, int32_t slot, int32_t B, int32_t* h_out);
/* ub_fmha_schedule of the batch slot `slot`'s last finished exchange delivered to this rank
 * (lengths h_all[h_perm[rank*B + k]], h_perm = that finish's perm), written to h_sched (host,
 * pinned if d_sched is given) and, if d_sched is not NULL, copied to d_sched (device,
 * ub_fmha_schedule_ints ints) on `stream` -- the exchange planner emitting the schedule of the
 * batch it delivers, one call per direction.  B <= 4096.  Errors as ub_fmha_schedule and
 * ub_exchange_slot_lengths. */
ub_status ub_exchange_fmha_schedule(void* comm, int32_t slot, const int32_t* h_perm, int32_t B, int32_t heads,
                                    int32_t max_seqlen, int32_t grid, int32_t is_bwd, int32_t* h_sched,
                                    size_t cap_ints, int32_t* d_sched, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* UB_H_ */
