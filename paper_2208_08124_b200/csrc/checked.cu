// Checked mode (SURVEY §8(b) conventions: device-resident data is not validated on the fast
// path; a debug switch validates it on the device and reports through a flag read after a
// sync -- tests only).  ub_validate_cu_seqlens is the check itself (async, result in a
// caller-provided device flag); with checked mode on (ub_set_checked(1) or UB_CHECKED=1 in
// the environment) the unpad / pad / FMHA entry points run it first, synchronise the stream
// and fail with the matching status instead of launching on bad offsets.
#include <atomic>
#include <cstdlib>
#include <mutex>

#include "ub_internal.h"

namespace ub {

// flag: 0 ok, 1 cu[0] != 0, 2 cu not monotone, 3 a length > max_seqlen, 4 cu[B] > T
__global__ void validate_cu_kernel(const int32_t* __restrict__ cu, int32_t B, int32_t max_seqlen, int64_t T,
                                   int32_t* __restrict__ flag) {
  int32_t code = 0;
  for (int32_t b = threadIdx.x; b < B; b += blockDim.x) {
    const int32_t L = cu[b + 1] - cu[b];
    if (L < 0) code = max(code, 2);
    else if (L > max_seqlen) code = max(code, 3);
  }
  if (threadIdx.x == 0) {
    if (cu[0] != 0) code = max(code, 1);
    if ((int64_t)cu[B] > T) code = max(code, 4);
  }
  code = __reduce_max_sync(0xffffffffu, (unsigned)code);
  __shared__ int32_t warp_code[32];
  if ((threadIdx.x & 31) == 0) warp_code[threadIdx.x >> 5] = code;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t c = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c = max(c, warp_code[w]);
    *flag = c;
  }
}

__device__ int32_t g_check_flag;
static std::atomic<int> g_checked{-1};           // -1: not read from the environment yet
// One device flag serves every checked call: the validate launch, the flag's D2H copy and the
// stream sync run under this lock, so two checked calls on different streams / host threads
// cannot read each other's result.
static std::mutex g_check_mu;

bool checked_mode() {
  int v = g_checked.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("UB_CHECKED");
    int want = (e && e[0] == '1') ? 1 : 0;
    g_checked.compare_exchange_strong(v, want);
    v = g_checked.load();
  }
  return v == 1;
}

ub_status checked_cu(const int32_t* d_cu, int32_t B, int32_t max_seqlen, int64_t T, cudaStream_t s) {
  if (!checked_mode()) return UB_OK;
  std::lock_guard<std::mutex> lock(g_check_mu);
  int32_t* flag = nullptr;
  UB_CHECK_CUDA(cudaGetSymbolAddress(reinterpret_cast<void**>(&flag), g_check_flag));
  validate_cu_kernel<<<1, 256, 0, s>>>(d_cu, B, max_seqlen, T, flag);
  UB_CHECK_LAUNCH();
  int32_t code = 0;
  UB_CHECK_CUDA(cudaMemcpyAsync(&code, flag, sizeof(code), cudaMemcpyDeviceToHost, s));
  UB_CHECK_CUDA(cudaStreamSynchronize(s));
  if (code == 3) return set_error(UB_ERR_CAPACITY, "checked mode: a sequence is longer than max_seqlen %d", max_seqlen);
  if (code != 0)
    return set_error(UB_ERR_INVALID_ARG, "checked mode: cu_seqlens invalid (%s)",
                     code == 1 ? "cu[0] != 0" : code == 2 ? "not monotone" : "cu[B] > T");
  return UB_OK;
}

}  // namespace ub

using namespace ub;

extern "C" ub_status ub_set_checked(int32_t on) {
  clear_error();
  g_checked.store(on ? 1 : 0);
  return UB_OK;
}

extern "C" ub_status ub_validate_cu_seqlens(const int32_t* d_cu, int32_t B, int32_t max_seqlen, int64_t T,
                                            int32_t* d_flag, void* stream) {
  clear_error();
  UB_REQUIRE(d_cu && d_flag && B >= 1 && max_seqlen >= 1 && T >= 0, UB_ERR_INVALID_ARG, "bad arguments");
  validate_cu_kernel<<<1, 256, 0, as_stream(stream)>>>(d_cu, B, max_seqlen, T, d_flag);
  UB_CHECK_LAUNCH();
  return UB_OK;
}
