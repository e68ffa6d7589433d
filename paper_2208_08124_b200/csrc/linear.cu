// Linear layers of the unpadded encoder through cuBLASLt ("Linear Fusion": the GEMM
// and its bias add in one call forward, the GEMM and the bias-gradient reduction in one call
// backward; "Fusion of Residual Grad": the residual gradient enters the data-gradient
// GEMM through its beta).  Plain library GEMMs on packed [T, features] rows -- no padding
// rows are ever multiplied.
//
// Row-major operands are handed to the column-major cuBLASLt as their transposes:
//   y[T,N]  = x[T,K] W[N,K]^T + b   ->  y^T(N x T)  = W^T'(op T on the K x N view) x^T(K x T)
//   dx[T,K] = dy[T,N] W[N,K] (+ r)  ->  dx^T(K x T) = W^T(K x N, op N) dy^T(N x T)
//   dW[N,K] = dy^T x                ->  dW^T(K x N) = x^T(K x T, op N) dy(T x N, op T),  db = sum_k B
#include <cublasLt.h>

#include <mutex>

#include "ub_internal.h"

namespace ub {
namespace {

constexpr size_t kLtWorkspace = 32u << 20;

cublasLtHandle_t lt_handle() {
  static cublasLtHandle_t h = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { cublasLtCreate(&h); });
  return h;
}

#define UB_CHECK_LT(expr)                                                                    \
  do {                                                                                       \
    cublasStatus_t _s = (expr);                                                              \
    if (_s != CUBLAS_STATUS_SUCCESS) return set_error(UB_ERR_CUDA, "%s failed: cublasLt status %d", #expr, (int)_s); \
  } while (0)

struct Mm {
  cublasOperation_t ta, tb;
  int m, n, k;
  const void* A; cudaDataType at; int lda;
  const void* B; cudaDataType bt; int ldb;
  const void* C; cudaDataType ct; int ldc;
  void* D; cudaDataType dt; int ldd;
  float beta;
  cublasLtEpilogue_t epi;
  const void* bias;
};

ub_status lt_matmul(const Mm& q, void* ws, cudaStream_t s) {
  cublasLtHandle_t h = lt_handle();
  UB_REQUIRE(h != nullptr, UB_ERR_CUDA, "cublasLtCreate failed");
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr, ld = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  ub_status st = UB_OK;
  auto body = [&]() -> ub_status {
    UB_CHECK_LT(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    UB_CHECK_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &q.ta, sizeof(q.ta)));
    UB_CHECK_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &q.tb, sizeof(q.tb)));
    UB_CHECK_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &q.epi, sizeof(q.epi)));
    if (q.bias) UB_CHECK_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &q.bias, sizeof(q.bias)));
    const int ar = q.ta == CUBLAS_OP_N ? q.m : q.k, ac = q.ta == CUBLAS_OP_N ? q.k : q.m;
    const int br = q.tb == CUBLAS_OP_N ? q.k : q.n, bc = q.tb == CUBLAS_OP_N ? q.n : q.k;
    UB_CHECK_LT(cublasLtMatrixLayoutCreate(&la, q.at, ar, ac, q.lda));
    UB_CHECK_LT(cublasLtMatrixLayoutCreate(&lb, q.bt, br, bc, q.ldb));
    UB_CHECK_LT(cublasLtMatrixLayoutCreate(&lc, q.ct, q.m, q.n, q.ldc));
    UB_CHECK_LT(cublasLtMatrixLayoutCreate(&ld, q.dt, q.m, q.n, q.ldd));
    UB_CHECK_LT(cublasLtMatmulPreferenceCreate(&pref));
    size_t wsb = kLtWorkspace;
    UB_CHECK_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)));
    cublasLtMatmulHeuristicResult_t res{};
    int n_res = 0;
    UB_CHECK_LT(cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, ld, pref, 1, &res, &n_res));
    UB_REQUIRE(n_res > 0, UB_ERR_UNSUPPORTED, "cublasLt: no algorithm for this GEMM (epilogue %d)", (int)q.epi);
    const float alpha = 1.f;
    UB_CHECK_LT(cublasLtMatmul(h, op, &alpha, q.A, la, q.B, lb, &q.beta, q.C ? q.C : q.D, lc, q.D, ld, &res.algo, ws,
                               kLtWorkspace, s));
    return UB_OK;
  };
  st = body();
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (ld) cublasLtMatrixLayoutDestroy(ld);
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  return st;
}

}  // namespace

size_t linear_workspace_bytes() { return kLtWorkspace; }

ub_status linear_fwd(const void* x, const void* W, const void* b, int64_t T, int32_t K, int32_t N, void* y, void* ws,
                     cudaStream_t s) {
  Mm q{};
  q.ta = CUBLAS_OP_T; q.tb = CUBLAS_OP_N;
  q.m = N; q.n = (int)T; q.k = K;
  q.A = W; q.at = CUDA_R_16BF; q.lda = K;
  q.B = x; q.bt = CUDA_R_16BF; q.ldb = K;
  q.C = nullptr; q.ct = CUDA_R_16BF; q.ldc = N;
  q.D = y; q.dt = CUDA_R_16BF; q.ldd = N;
  q.beta = 0.f;
  q.epi = b ? CUBLASLT_EPILOGUE_BIAS : CUBLASLT_EPILOGUE_DEFAULT;
  q.bias = b;
  return lt_matmul(q, ws, s);
}

ub_status linear_bwd(const void* dy, const void* x, const void* W, const void* res_grad, int64_t T, int32_t K,
                     int32_t N, void* dx, float* dW, float* db, void* ws, cudaStream_t s) {
  ub_status st;
  if (dx) {                                     // dx^T = W^T dy^T (+ r^T, beta = 1: P:416)
    Mm q{};
    q.ta = CUBLAS_OP_N; q.tb = CUBLAS_OP_N;
    q.m = K; q.n = (int)T; q.k = N;
    q.A = W; q.at = CUDA_R_16BF; q.lda = K;
    q.B = dy; q.bt = CUDA_R_16BF; q.ldb = N;
    q.C = res_grad; q.ct = CUDA_R_16BF; q.ldc = K;
    q.D = dx; q.dt = CUDA_R_16BF; q.ldd = K;
    q.beta = res_grad ? 1.f : 0.f;
    q.epi = CUBLASLT_EPILOGUE_DEFAULT;
    if ((st = lt_matmul(q, ws, s)) != UB_OK) return st;
  }
  if (dW) {                                     // dW^T = x^T dy, db = sum over T of dy (BGRADB)
    Mm q{};
    q.ta = CUBLAS_OP_N; q.tb = CUBLAS_OP_T;
    q.m = K; q.n = N; q.k = (int)T;
    q.A = x; q.at = CUDA_R_16BF; q.lda = K;
    q.B = dy; q.bt = CUDA_R_16BF; q.ldb = N;
    q.C = nullptr; q.ct = CUDA_R_32F; q.ldc = K;
    q.D = dW; q.dt = CUDA_R_32F; q.ldd = K;
    q.beta = 0.f;
    q.epi = db ? CUBLASLT_EPILOGUE_BGRADB : CUBLASLT_EPILOGUE_DEFAULT;
    q.bias = db;
    if ((st = lt_matmul(q, ws, s)) != UB_OK) return st;
  }
  return UB_OK;
}

}  // namespace ub

using namespace ub;

extern "C" size_t ub_linear_workspace_bytes(void) { return linear_workspace_bytes(); }

extern "C" ub_status ub_linear_fwd(const void* x, const void* W, const void* b, int64_t T, int32_t K, int32_t N, void* y,
                                   void* ws, void* stream) {
  clear_error();
  UB_REQUIRE(x && W && y && ws, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(T >= 1 && K >= 1 && N >= 1 && K % 8 == 0 && N % 8 == 0, UB_ERR_SHAPE, "need T >= 1, K, N multiples of 8");
  return linear_fwd(x, W, b, T, K, N, y, ws, as_stream(stream));
}

extern "C" ub_status ub_linear_bwd(const void* dy, const void* x, const void* W, const void* res_grad, int64_t T,
                                   int32_t K, int32_t N, void* dx, float* dW, float* db, void* ws, void* stream) {
  clear_error();
  UB_REQUIRE(dy && ws && (dx || dW), UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(!dx || W, UB_ERR_INVALID_ARG, "dx needs W");
  UB_REQUIRE(!dW || x, UB_ERR_INVALID_ARG, "dW needs x");
  UB_REQUIRE(!db || dW, UB_ERR_INVALID_ARG, "db is produced with dW");
  UB_REQUIRE(T >= 1 && K >= 1 && N >= 1 && K % 8 == 0 && N % 8 == 0, UB_ERR_SHAPE, "need T >= 1, K, N multiples of 8");
  return linear_bwd(dy, x, W, res_grad, T, K, N, dx, dW, db, ws, as_stream(stream));
}
