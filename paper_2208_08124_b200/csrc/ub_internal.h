// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <utility>

#include "../../include/ub.h"

namespace ub {

ub_status set_error(ub_status st, const char* fmt, ...);
void clear_error();

// Capability check: device of the current context must be sm_100 (cached per device).
ub_status require_sm100();

// Measurement hook (ub_profile_events): events recorded around one internal kernel.
enum ProfKernel { kProfFwd = 0, kProfBwd = 1, kProfPad = 2, kProfUnpad = 3, kProfDalFwd = 4, kProfDalBwd = 5, kProfCount = 6 };
void prof_record(int kernel_id, int which, cudaStream_t s);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device).
ub_status smem_attr_once(const void* func, int bytes);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define UB_CHECK_CUDA(expr)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return ::ub::set_error(UB_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                             __FILE__, __LINE__);                                        \
  } while (0)

#define UB_CHECK_LAUNCH()                                                                \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return ::ub::set_error(UB_ERR_CUDA, "launch: %s (%s:%d)", cudaGetErrorString(e_),   \
                             __FILE__, __LINE__);                                        \
  } while (0)

#define UB_REQUIRE(cond, status, ...)                                                    \
  do {                                                                                   \
    if (!(cond)) return ::ub::set_error((status), __VA_ARGS__);                          \
  } while (0)

// ---- FMHA internals (fmha_*.cu) ------------------------------------------------------
constexpr int kTile = 128;  // query / key tile (rows) of the tensor-core path and of the plan

struct FmhaPlanView {   // device views into the workspace, filled by the plan kernel
  int32_t* seq_order;   // [B] sequences sorted by tile count desc (then id asc)
  int32_t* item_prefix; // [B+1] prefix of items along seq_order
  int32_t* pad_c0;      // [B+1] per sequence (original order): sum of 128 * tiles of the earlier ones
  int32_t* counters;    // [4] scheduler counters
};

size_t fmha_plan_bytes(int32_t B);
FmhaPlanView fmha_plan_view(void* ws, int32_t B);
ub_status launch_fmha_plan(const int32_t* d_cu, int32_t B, int32_t H, int32_t max_tiles, int32_t tiles_per_item,
                           FmhaPlanView v, cudaStream_t s);

ub_status fmha_fwd_sm100(const ub_fmha_params& p, const void* qkv, const int32_t* d_cu, void* out, float* lse,
                         void* padded, int32_t S_pad, void* ws, cudaStream_t s);
ub_status fmha_bwd_sm100(const ub_fmha_params& p, const void* qkv, const void* out, const float* lse,
                         const void* dout, const int32_t* d_cu, void* dqkv, void* ws, cudaStream_t s);
size_t fmha_bwd_sm100_ws_bytes(const ub_fmha_params& p);
size_t fmha_schedule_ints(int32_t B, int32_t H, int32_t max_seqlen, int32_t grid, int32_t is_bwd);

// dropout_mask.cu: R5's keep bits, query-major half then key-major half
size_t dropout_mask_bytes(const ub_fmha_params& p);
int32_t mask_tiles(const ub_fmha_params& p);
uint32_t dropout_threshold(float p);
ub_status launch_dropout_mask(const ub_fmha_params& p, const int32_t* d_cu, void* mask, cudaStream_t s,
                              bool overlap_previous = false);

ub_status fmha_fwd_simt(const ub_fmha_params& p, const float* qkv, const int32_t* d_cu, float* out,
                        float* lse, cudaStream_t s);
ub_status fmha_bwd_simt(const ub_fmha_params& p, const float* qkv, const float* out, const float* lse,
                        const float* dout, const int32_t* d_cu, float* dqkv, float* ws, cudaStream_t s);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Programmatic dependent launch (sm_90+): the kernel may be scheduled while the previous
// kernel in the stream drains; it calls pdl_wait() before touching memory that kernel (or
// anything ordered before it) produces.  Hides the launch latency and the prologue (barrier
// init, TMEM allocation) behind the previous kernel's tail.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// exchange copy (unpad_pad.cu): n entries of a {src_tok, len, dst_tok, src_smp, dst_smp} table with
// row stride B; d_sel (row of n, may be NULL) picks src_b / ssrc_b for entries != 0; cu_dst (may be
// NULL) receives ncu int32 from cu_src in the same launch.
ub_status exchange_gather(const void* src_a, const void* src_b, void* dst, const void* ssrc_a, const void* ssrc_b,
                          void* sdst, const int64_t* d_tab, const int64_t* d_sel, int32_t n, int32_t B, int64_t rec,
                          int64_t srec, const int32_t* cu_src, int32_t* cu_dst, int32_t ncu, cudaStream_t s);

// checked mode (checked.cu): validate device cu_seqlens before a launch (sync; tests only)
bool checked_mode();
ub_status checked_cu(const int32_t* d_cu, int32_t B, int32_t max_seqlen, int64_t T, cudaStream_t s);

}  // namespace ub
