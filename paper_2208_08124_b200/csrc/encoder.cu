// The unpadded BERT encoder's attention sub-layer (BASELINE config 4),
// forward and backward, on packed rows [T, hidden] (the whole encoder runs on
// unpadded tokens):
//   qkv = x Wqkv^T + bqkv                 Linear, bias in the cuBLASLt epilogue
//   ctx = varlen_fmha(qkv)                 this library's tcgen05 kernel
//   a   = ctx Wo^T + bo                    Linear
//   y   = LayerNorm(x + dropout(a))        fused Dropout_Add_LayerNorm
// backward: DAL (2 kernels), Linear (data GEMM + weight GEMM with the bias-gradient
// epilogue), varlen FMHA backward, Linear with the residual gradient of x added by the data
// GEMM's beta.  Attention dropout keeps its mask (R5), hidden dropout its own (R21);
// both come from (seed, offset).
#include "ub_internal.h"

namespace ub {
ub_status linear_fwd(const void* x, const void* W, const void* b, int64_t T, int32_t K, int32_t N, void* y, void* ws,
                     cudaStream_t s);
ub_status linear_bwd(const void* dy, const void* x, const void* W, const void* res_grad, int64_t T, int32_t K,
                     int32_t N, void* dx, float* dW, float* db, void* ws, cudaStream_t s);
size_t linear_workspace_bytes();

namespace {

ub_fmha_params fmha_of(const ub_encoder_params& p) {
  ub_fmha_params f{};
  f.B = p.B;
  f.T = p.T;
  f.max_seqlen = p.max_seqlen;
  f.heads = p.heads;
  f.head_dim = p.hidden / p.heads;
  f.scale = 1.f / sqrtf((float)f.head_dim);
  f.p_dropout = p.p_attn;
  f.seed = p.seed;
  f.offset = p.offset;
  f.dtype = UB_BF16;
  f.num_ctas = p.num_ctas;
  return f;
}

struct Ws {
  char* lt;
  char* fmha;
  char* dal;
  char* da;      // [T, hidden] bf16 (backward)
  char* dres;
  char* dctx;
  char* dqkv;    // [T, 3 hidden] bf16
};

size_t layout(const ub_encoder_params& p, int is_bwd, char* base, Ws* w) {
  const ub_fmha_params f = fmha_of(p);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* ptr = base ? base + off : nullptr;
    off += align_up(bytes, 256);
    return ptr;
  };
  Ws tmp{};
  tmp.lt = take(linear_workspace_bytes());
  tmp.fmha = take(ub_fmha_workspace_bytes(&f, is_bwd));
  if (is_bwd) {
    const size_t row = (size_t)p.T * p.hidden * 2;
    tmp.dal = take(ub_dal_bwd_workspace_bytes(p.T, p.hidden));
    tmp.da = take(row);
    tmp.dres = take(row);
    tmp.dctx = take(row);
    tmp.dqkv = take(3 * row);
  }
  if (w) *w = tmp;
  return off;
}

ub_status check(const ub_encoder_params* p) {
  UB_REQUIRE(p, UB_ERR_INVALID_ARG, "null params");
  UB_REQUIRE(p->B >= 1 && p->T >= 1 && p->heads >= 1 && p->hidden >= 8, UB_ERR_INVALID_ARG, "bad sizes");
  UB_REQUIRE(p->hidden % p->heads == 0 && p->hidden / p->heads == 64, UB_ERR_UNSUPPORTED,
             "hidden / heads must be 64 (the bf16 FMHA's head_dim)");
  UB_REQUIRE(p->hidden <= 2048, UB_ERR_UNSUPPORTED, "hidden <= 2048 (the LayerNorm kernel keeps a row in registers)");
  UB_REQUIRE(p->p_attn >= 0.f && p->p_attn < 1.f && p->p_hidden >= 0.f && p->p_hidden < 1.f && p->eps > 0.f,
             UB_ERR_INVALID_ARG, "dropout probabilities in [0, 1), eps > 0");
  return UB_OK;
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" size_t ub_encoder_attn_workspace_bytes(const ub_encoder_params* p, int is_bwd) {
  if (!p) return 0;
  return layout(*p, is_bwd, nullptr, nullptr);
}

extern "C" ub_status ub_encoder_attn_fwd(const ub_encoder_params* p, const void* x, const int32_t* d_cu,
                                         const void* w_qkv, const void* b_qkv, const void* w_o, const void* b_o,
                                         const void* gamma, const void* beta, void* qkv, void* ctx, float* lse,
                                         void* a, float* mean, float* rstd, void* y, void* ws, void* stream) {
  clear_error();
  ub_status st = check(p);
  if (st != UB_OK) return st;
  UB_REQUIRE(x && d_cu && w_qkv && b_qkv && w_o && b_o && gamma && beta && qkv && ctx && lse && a && mean && rstd && y &&
                 ws,
             UB_ERR_INVALID_ARG, "null pointer");
  Ws w;
  layout(*p, 0, static_cast<char*>(ws), &w);
  cudaStream_t s = as_stream(stream);
  const int32_t Hd = p->hidden;
  const ub_fmha_params f = fmha_of(*p);
  if ((st = linear_fwd(x, w_qkv, b_qkv, p->T, Hd, 3 * Hd, qkv, w.lt, s)) != UB_OK) return st;
  if ((st = ub_varlen_fmha_fwd(&f, qkv, d_cu, ctx, lse, w.fmha, s)) != UB_OK) return st;
  if ((st = linear_fwd(ctx, w_o, b_o, p->T, Hd, Hd, a, w.lt, s)) != UB_OK) return st;
  return ub_dal_fwd(a, x, gamma, beta, p->T, Hd, p->p_hidden, p->eps, p->seed, p->offset, y, mean, rstd, s);
}

extern "C" ub_status ub_encoder_attn_bwd(const ub_encoder_params* p, const void* x, const int32_t* d_cu,
                                         const void* w_qkv, const void* w_o, const void* gamma, const void* qkv,
                                         const void* ctx, const float* lse, const void* a, const float* mean,
                                         const float* rstd, const void* dy, void* dx, float* dw_qkv, float* db_qkv,
                                         float* dw_o, float* db_o, float* dgamma, float* dbeta, void* ws,
                                         void* stream) {
  clear_error();
  ub_status st = check(p);
  if (st != UB_OK) return st;
  UB_REQUIRE(x && d_cu && w_qkv && w_o && gamma && qkv && ctx && lse && a && mean && rstd && dy && dx && dw_qkv && db_qkv &&
                 dw_o && db_o && dgamma && dbeta && ws,
             UB_ERR_INVALID_ARG, "null pointer");
  Ws w;
  layout(*p, 1, static_cast<char*>(ws), &w);
  cudaStream_t s = as_stream(stream);
  const int32_t Hd = p->hidden;
  const ub_fmha_params f = fmha_of(*p);
  // DAL backward: da (through the dropout) and the residual branch's gradient dres
  if ((st = ub_dal_bwd(dy, a, x, gamma, mean, rstd, p->T, Hd, p->p_hidden, p->seed, p->offset, w.da, w.dres, dgamma,
                       dbeta, w.dal, s)) != UB_OK)
    return st;
  // out-projection: dctx = da Wo, dWo = da^T ctx, dbo = sum da
  if ((st = linear_bwd(w.da, ctx, w_o, nullptr, p->T, Hd, Hd, w.dctx, dw_o, db_o, w.lt, s)) != UB_OK) return st;
  // attention
  if ((st = ub_varlen_fmha_bwd(&f, qkv, ctx, lse, w.dctx, d_cu, w.dqkv, w.fmha, s)) != UB_OK) return st;
  // QKV projection: dx = dqkv Wqkv + dres (residual gradient through beta)
  return linear_bwd(w.dqkv, x, w_qkv, w.dres, p->T, Hd, 3 * Hd, dx, dw_qkv, db_qkv, w.lt, s);
}
