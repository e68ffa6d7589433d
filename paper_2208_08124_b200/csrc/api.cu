// C-ABI entry points: validation, error reporting, dispatch.  See include/ub.h.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "ub_internal.h"

namespace ub {

static thread_local std::string g_last_error;

ub_status set_error(ub_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}
void clear_error() { g_last_error.clear(); }

ub_status require_sm100() {
  static int cached[64];
  static std::once_flag once;
  std::call_once(once, [] { for (int& c : cached) c = -1; });
  int dev = 0;
  UB_CHECK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return set_error(UB_ERR_UNSUPPORTED, "device index %d", dev);
  if (cached[dev] < 0) {
    int maj = 0, min = 0;
    UB_CHECK_CUDA(cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev));
    UB_CHECK_CUDA(cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev));
    cached[dev] = maj * 10 + min;
  }
  if (cached[dev] != 100)
    return set_error(UB_ERR_UNSUPPORTED, "this library is built for sm_100a (B200); device is sm_%d", cached[dev]);
  return UB_OK;
}

ub_status smem_attr_once(const void* func, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  UB_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : done)
    if (e.first == func && e.second == dev) return UB_OK;
  UB_CHECK_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.emplace_back(func, dev);
  return UB_OK;
}

static cudaEvent_t g_prof[kProfCount][2] = {};

void prof_record(int kernel_id, int which, cudaStream_t s) {
  cudaEvent_t e = g_prof[kernel_id][which];
  if (e) cudaEventRecord(e, s);
}

}  // namespace ub

using namespace ub;

extern "C" ub_status ub_profile_events(int32_t kernel_id, void* start_event, void* stop_event) {
  clear_error();
  UB_REQUIRE(kernel_id >= 0 && kernel_id < kProfCount, UB_ERR_INVALID_ARG, "bad kernel id %d", kernel_id);
  UB_REQUIRE((start_event == nullptr) == (stop_event == nullptr), UB_ERR_INVALID_ARG, "give both events or none");
  g_prof[kernel_id][0] = static_cast<cudaEvent_t>(start_event);
  g_prof[kernel_id][1] = static_cast<cudaEvent_t>(stop_event);
  return UB_OK;
}

extern "C" double ub_dropout_effective_p(float p_dropout, int32_t bits) {
  if (!(p_dropout > 0.f) || (bits != 8 && bits != 16)) return 0.0;
  const double levels = bits == 8 ? 256.0 : 65536.0;
  return std::floor((double)p_dropout * levels) / levels;
}

extern "C" const char* ub_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* ub_version(void) {
  return "ubert 0.2 (sm_100a; tcgen05/TMEM/TMA FMHA; NCCL all-gather + send/recv exchange)";
}

extern "C" ub_status ub_cu_seqlens(const int32_t* h_lengths, int32_t B, int32_t max_seqlen, int32_t* h_cu) {
  clear_error();
  UB_REQUIRE(h_lengths && h_cu, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1, UB_ERR_INVALID_ARG, "empty batch (B=%d)", B);
  UB_REQUIRE(max_seqlen >= 1, UB_ERR_INVALID_ARG, "max_seqlen < 1");
  int64_t acc = 0;
  h_cu[0] = 0;
  for (int32_t b = 0; b < B; ++b) {
    const int32_t L = h_lengths[b];
    UB_REQUIRE(L >= 1, UB_ERR_INVALID_ARG, "length[%d] = %d < 1", b, L);
    UB_REQUIRE(L <= max_seqlen, UB_ERR_CAPACITY, "length[%d] = %d > max_seqlen %d", b, L, max_seqlen);
    acc += L;
    UB_REQUIRE(acc <= INT32_MAX, UB_ERR_SHAPE, "total tokens overflow int32");
    h_cu[b + 1] = static_cast<int32_t>(acc);
  }
  return UB_OK;
}

extern "C" ub_status ub_lengths_from_mask(const int32_t* h_mask, int32_t B, int32_t S, int32_t* h_lengths) {
  clear_error();
  UB_REQUIRE(h_mask && h_lengths, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1 && S >= 1, UB_ERR_INVALID_ARG, "empty mask");
  for (int32_t b = 0; b < B; ++b) {
    const int32_t* row = h_mask + (int64_t)b * S;
    int32_t L = 0;
    while (L < S && row[L] != 0) ++L;
    for (int32_t i = L; i < S; ++i)
      UB_REQUIRE(row[i] == 0, UB_ERR_INVALID_MASK, "mask row %d is not a prefix", b);
    h_lengths[b] = L;
  }
  return UB_OK;
}

// ------------------------------------------------------------------------------ FMHA
static ub_status check_fmha(const ub_fmha_params* p) {
  UB_REQUIRE(p != nullptr, UB_ERR_INVALID_ARG, "null params");
  UB_REQUIRE(p->B >= 1, UB_ERR_INVALID_ARG, "B < 1");
  UB_REQUIRE(p->T >= 1, UB_ERR_INVALID_ARG, "T < 1");
  UB_REQUIRE(p->T <= INT32_MAX, UB_ERR_SHAPE, "T exceeds int32");
  UB_REQUIRE(p->heads >= 1, UB_ERR_INVALID_ARG, "heads < 1");
  UB_REQUIRE(p->max_seqlen >= 1, UB_ERR_INVALID_ARG, "max_seqlen < 1");
  UB_REQUIRE(std::isfinite(p->scale) && p->scale > 0.f, UB_ERR_INVALID_ARG, "scale must be > 0");
  UB_REQUIRE(p->p_dropout >= 0.f && p->p_dropout < 1.f, UB_ERR_INVALID_ARG, "p_dropout outside [0,1)");
  UB_REQUIRE(p->p_dropout == 0.f || ub_dropout_effective_p(p->p_dropout, 8) > 0.0, UB_ERR_INVALID_ARG,
             "p_dropout %g < 1/256: the 8-bit keep decisions (R5) would drop nothing", (double)p->p_dropout);
  if (p->dtype == UB_BF16) {
    UB_REQUIRE(p->head_dim == 64, UB_ERR_UNSUPPORTED, "bf16 tensor-core path supports head_dim 64 (got %d)", p->head_dim);
  } else if (p->dtype == UB_FP32) {
    UB_REQUIRE(p->head_dim >= 1 && p->head_dim <= 128, UB_ERR_UNSUPPORTED, "fp32 path supports head_dim 1..128");
  } else {
    return set_error(UB_ERR_INVALID_ARG, "bad dtype %d", p->dtype);
  }
  return UB_OK;
}

extern "C" size_t ub_fmha_workspace_bytes(const ub_fmha_params* p, int is_bwd) {
  if (!p || p->B < 1) return 0;
  size_t n = align_up(fmha_plan_bytes(p->B), 256);
  if (is_bwd) {
    if (p->dtype == UB_BF16) n += fmha_bwd_sm100_ws_bytes(*p);
    else n += align_up((size_t)p->T * p->heads * sizeof(float), 256);   // Delta
  }
  return n;
}

extern "C" ub_status ub_varlen_fmha_fwd(const ub_fmha_params* p, const void* qkv, const int32_t* d_cu,
                                        void* out, float* lse, void* ws, void* stream) {
  clear_error();
  ub_status st = check_fmha(p);
  if (st != UB_OK) return st;
  UB_REQUIRE(qkv && d_cu && out && lse, UB_ERR_INVALID_ARG, "null pointer");
  if ((st = require_sm100()) != UB_OK) return st;
  if ((st = checked_cu(d_cu, p->B, p->max_seqlen, p->T, as_stream(stream))) != UB_OK) return st;
  if (p->dtype == UB_BF16) {
    UB_REQUIRE(ws, UB_ERR_INVALID_ARG, "null workspace");
    UB_REQUIRE(((uintptr_t)qkv & 15) == 0 && ((uintptr_t)out & 15) == 0, UB_ERR_INVALID_ARG,
               "qkv/out must be 16-B aligned");
    return fmha_fwd_sm100(*p, qkv, d_cu, out, lse, nullptr, 0, ws, as_stream(stream));
  }
  return fmha_fwd_simt(*p, static_cast<const float*>(qkv), d_cu, static_cast<float*>(out), lse, as_stream(stream));
}

extern "C" ub_status ub_varlen_fmha_fwd_pad(const ub_fmha_params* p, const void* qkv, const int32_t* d_cu,
                                            void* out, float* lse, void* padded, int32_t S, void* ws, void* stream) {
  clear_error();
  ub_status st = check_fmha(p);
  if (st != UB_OK) return st;
  UB_REQUIRE(qkv && d_cu && out && lse && padded && ws, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(p->dtype == UB_BF16, UB_ERR_UNSUPPORTED, "the fused pad is on the bf16 path");
  UB_REQUIRE(S >= p->max_seqlen && S % 32 == 0, UB_ERR_SHAPE, "S = %d: need S >= max_seqlen and S %% 32 == 0", S);
  UB_REQUIRE((((uintptr_t)qkv | (uintptr_t)out | (uintptr_t)padded) & 15) == 0, UB_ERR_INVALID_ARG,
             "qkv/out/padded must be 16-B aligned");
  if ((st = require_sm100()) != UB_OK) return st;
  if ((st = checked_cu(d_cu, p->B, p->max_seqlen, p->T, as_stream(stream))) != UB_OK) return st;
  return fmha_fwd_sm100(*p, qkv, d_cu, out, lse, padded, S, ws, as_stream(stream));
}

extern "C" ub_status ub_varlen_fmha_bwd(const ub_fmha_params* p, const void* qkv, const void* out,
                                        const float* lse, const void* dout, const int32_t* d_cu,
                                        void* dqkv, void* ws, void* stream) {
  clear_error();
  ub_status st = check_fmha(p);
  if (st != UB_OK) return st;
  UB_REQUIRE(qkv && out && lse && dout && d_cu && dqkv && ws, UB_ERR_INVALID_ARG, "null pointer");
  if ((st = require_sm100()) != UB_OK) return st;
  if ((st = checked_cu(d_cu, p->B, p->max_seqlen, p->T, as_stream(stream))) != UB_OK) return st;
  if (p->dtype == UB_BF16) {
    UB_REQUIRE(((uintptr_t)qkv & 15) == 0 && ((uintptr_t)dout & 15) == 0 && ((uintptr_t)dqkv & 15) == 0,
               UB_ERR_INVALID_ARG, "qkv/dout/dqkv must be 16-B aligned");
    return fmha_bwd_sm100(*p, qkv, out, lse, dout, d_cu, dqkv, ws, as_stream(stream));
  }
  float* delta = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up(fmha_plan_bytes(p->B), 256));
  return fmha_bwd_simt(*p, static_cast<const float*>(qkv), static_cast<const float*>(out), lse,
                       static_cast<const float*>(dout), d_cu, static_cast<float*>(dqkv), delta,
                       as_stream(stream));
}
