// Pull-based exchange: every rank gathers its perm-ordered samples
// straight out of the peers' packed token buffers -- a4 (all-to-all-v) and a5 (reorder)
// as one copy kernel reading peer memory, with no send buffer, no receive buffer and no
// NCCL kernels competing for SMs with the FMHA.  The peers' buffers are mapped into this
// process by CUDA IPC (over NVLink P2P between GPUs; the same mechanism maps a buffer of
// another process on the same GPU, which is how it is tested on one device).
//
// Plan (host): output sample k of rank r is global id g = perm[r*B + k], held by
// rank s = g / B as its local sample g % B, whose records start at that rank's cu.
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "sm100.cuh"
#include "ub_internal.h"

namespace ub {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_ge(const uint32_t* p, uint32_t v) {
  while (ld_acquire_sys(p) < v) __nanosleep(256);
}

// One CTA per output sample: len * rec bytes of token records from the source rank's
// buffer, srec bytes of its sample record.  tab = {src_rank, src_tok, len, dst_tok,
// src_smp, dst_smp} x B.  With ready flags, a CTA first waits (acquire, system scope) until
// its source rank has published the buffer (ready[src] >= wait_value): a sample moves as soon
// as its own source is ready.
template <typename Vec>
__global__ void __launch_bounds__(256) exchange_pull_kernel(const uint8_t* const* __restrict__ peer_tok,
                                                            const uint8_t* const* __restrict__ peer_smp,
                                                            const uint32_t* const* __restrict__ ready,
                                                            uint32_t wait_value, uint8_t* __restrict__ dt,
                                                            uint8_t* __restrict__ ds, const int64_t* __restrict__ tab,
                                                            int32_t B, int64_t rec, int64_t srec) {
  const int e = blockIdx.x;
  const int64_t src = tab[e], src_tok = tab[B + e], len = tab[2 * B + e], dst_tok = tab[3 * B + e];
  if (ready != nullptr) {
    if (threadIdx.x == 0) spin_until_ge(ready[src], wait_value);
    __syncthreads();
  }
  const uint8_t* sb = peer_tok[src] + src_tok * rec;
  uint8_t* db = dt + dst_tok * rec;
  const int64_t stride = (int64_t)gridDim.y * blockDim.x;
  if (((uintptr_t)sb & (sizeof(Vec) - 1)) == 0) {
    const Vec* s = reinterpret_cast<const Vec*>(sb);
    Vec* d = reinterpret_cast<Vec*>(db);
    const int64_t nv = len * rec / (int64_t)sizeof(Vec);
    // gridDim.y CTAs share a sample (large records): interleaved 256-vector blocks
    for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < nv; i += stride) d[i] = s[i];
  } else {
    // a peer base the caller mapped at an offset not aligned to the vector width (the host
    // cannot see the device pointer table): byte copy for this sample instead of a fault
    for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < len * rec; i += stride) db[i] = sb[i];
  }
  if (srec > 0 && blockIdx.y == 0) {
    const uint8_t* ss = peer_smp[src] + tab[4 * B + e] * srec;
    uint8_t* dd = ds + tab[5 * B + e] * srec;
    for (int64_t i = threadIdx.x; i < srec; i += blockDim.x) dd[i] = ss[i];
  }
}

// publish: every earlier write of this stream is visible system-wide before the flag
__global__ void signal_kernel(uint32_t* flag, uint32_t value) {
  __threadfence_system();
  st_release_sys(flag, value);
}
// wait until flags[i] >= value for all i < n (one thread per flag)
__global__ void wait_flags_kernel(const uint32_t* const* __restrict__ flags, int32_t n, uint32_t value) {
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) spin_until_ge(flags[i], value);
  __syncthreads();
  __threadfence_system();
}

// export: the CUDA IPC handle of the allocation holding ptr, plus ptr's offset in it (a
// caching allocator hands out sub-ranges of larger cudaMalloc blocks)
struct IpcHandle {
  cudaIpcMemHandle_t mem;
  int64_t offset;
};
static_assert(sizeof(IpcHandle) <= UB_IPC_HANDLE_BYTES, "IPC handle size");

static PFN_cuMemGetAddressRange_v3020 get_range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

}  // namespace ub

using namespace ub;

extern "C" ub_status ub_ipc_export(const void* d_ptr, void* h_handle) {
  clear_error();
  UB_REQUIRE(d_ptr && h_handle, UB_ERR_INVALID_ARG, "null pointer");
  auto range = get_range_fn();
  UB_REQUIRE(range != nullptr, UB_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  UB_REQUIRE(range(&base, &size, (CUdeviceptr)(uintptr_t)d_ptr) == CUDA_SUCCESS, UB_ERR_INVALID_ARG,
             "pointer is not device memory");
  IpcHandle h{};
  UB_CHECK_CUDA(cudaIpcGetMemHandle(&h.mem, reinterpret_cast<void*>(base)));
  h.offset = (int64_t)((uintptr_t)d_ptr - (uintptr_t)base);
  std::memset(h_handle, 0, UB_IPC_HANDLE_BYTES);
  std::memcpy(h_handle, &h, sizeof(h));
  return UB_OK;
}

extern "C" ub_status ub_ipc_import(const void* h_handle, void** d_ptr, void** d_base) {
  clear_error();
  UB_REQUIRE(h_handle && d_ptr && d_base, UB_ERR_INVALID_ARG, "null pointer");
  IpcHandle h;
  std::memcpy(&h, h_handle, sizeof(h));
  void* base = nullptr;
  UB_CHECK_CUDA(cudaIpcOpenMemHandle(&base, h.mem, cudaIpcMemLazyEnablePeerAccess));
  *d_base = base;
  *d_ptr = static_cast<char*>(base) + h.offset;
  return UB_OK;
}

extern "C" ub_status ub_ipc_close(void* d_base) {
  clear_error();
  UB_REQUIRE(d_base, UB_ERR_INVALID_ARG, "null pointer");
  UB_CHECK_CUDA(cudaIpcCloseMemHandle(d_base));
  return UB_OK;
}

extern "C" ub_status ub_exchange_pull_table(const int32_t* a, const int32_t* perm, int32_t W, int32_t B, int32_t rank,
                                            int64_t* tab, int64_t* total_tokens) {
  clear_error();
  UB_REQUIRE(a && perm && tab, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(W >= 1 && B >= 1 && rank >= 0 && rank < W, UB_ERR_INVALID_ARG, "bad W/B/rank");
  // each rank's local cu_seqlens (its packed batch, samples in local order)
  std::vector<int64_t> cu((size_t)W * (B + 1), 0);
  for (int32_t s = 0; s < W; ++s)
    for (int32_t k = 0; k < B; ++k) {
      UB_REQUIRE(a[(size_t)s * B + k] >= 0, UB_ERR_INVALID_ARG, "negative length");
      cu[(size_t)s * (B + 1) + k + 1] = cu[(size_t)s * (B + 1) + k] + a[(size_t)s * B + k];
    }
  std::vector<char> seen((size_t)W * B, 0);
  int64_t off = 0;
  for (int32_t k = 0; k < B; ++k) {
    const int32_t g = perm[(size_t)rank * B + k];
    UB_REQUIRE(g >= 0 && g < W * B && !seen[g], UB_ERR_SHAPE, "perm is not a permutation");
    seen[g] = 1;
    const int32_t s = g / B, kk = g % B;
    tab[k] = s;
    tab[B + k] = cu[(size_t)s * (B + 1) + kk];
    tab[2 * B + k] = a[g];
    tab[3 * B + k] = off;
    tab[4 * B + k] = kk;
    tab[5 * B + k] = k;
    off += a[g];
  }
  if (total_tokens) *total_tokens = off;
  return UB_OK;
}

extern "C" ub_status ub_exchange_pull(const void* const* d_peer_tokens, const void* const* d_peer_samples,
                                      const uint32_t* const* d_ready, uint32_t wait_value, const int64_t* d_tab,
                                      int32_t B, int64_t rec_bytes, int64_t srec_bytes, void* dst_tokens,
                                      void* dst_samples, void* stream) {
  clear_error();
  UB_REQUIRE(d_peer_tokens && d_tab && dst_tokens, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1 && rec_bytes > 0 && srec_bytes >= 0, UB_ERR_SHAPE, "bad sizes");
  UB_REQUIRE(srec_bytes == 0 || (d_peer_samples && dst_samples), UB_ERR_INVALID_ARG, "null sample pointer");
  cudaStream_t s = as_stream(stream);
  auto* pt = reinterpret_cast<const uint8_t* const*>(d_peer_tokens);
  auto* ps = reinterpret_cast<const uint8_t* const*>(d_peer_samples);
  auto* dt = static_cast<uint8_t*>(dst_tokens);
  auto* ds = static_cast<uint8_t*>(dst_samples);
  // the vector width follows rec and dst; a peer base that is not aligned to it is detected
  // per sample on the device (byte-copy path), since the pointer table is device memory.
  // Large records (a hidden row per token): 16 CTAs per sample, else one.
  const dim3 grid(B, rec_bytes >= 256 ? 16 : 1);
  if (rec_bytes % 16 == 0 && ((uintptr_t)dst_tokens & 15) == 0)
    exchange_pull_kernel<int4><<<grid, 256, 0, s>>>(pt, ps, d_ready, wait_value, dt, ds, d_tab, B, rec_bytes, srec_bytes);
  else if (rec_bytes % 4 == 0 && ((uintptr_t)dst_tokens & 3) == 0)
    exchange_pull_kernel<uint32_t><<<grid, 256, 0, s>>>(pt, ps, d_ready, wait_value, dt, ds, d_tab, B, rec_bytes,
                                                      srec_bytes);
  else
    exchange_pull_kernel<uint8_t><<<grid, 256, 0, s>>>(pt, ps, d_ready, wait_value, dt, ds, d_tab, B, rec_bytes,
                                                     srec_bytes);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

extern "C" ub_status ub_signal(uint32_t* d_flag, uint32_t value, void* stream) {
  clear_error();
  UB_REQUIRE(d_flag, UB_ERR_INVALID_ARG, "null pointer");
  signal_kernel<<<1, 1, 0, as_stream(stream)>>>(d_flag, value);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

extern "C" ub_status ub_wait_flags(const uint32_t* const* d_flags, int32_t n, uint32_t value, void* stream) {
  clear_error();
  UB_REQUIRE(d_flags && n >= 1, UB_ERR_INVALID_ARG, "bad flags");
  wait_flags_kernel<<<1, 32, 0, as_stream(stream)>>>(d_flags, n, value);
  UB_CHECK_LAUNCH();
  return UB_OK;
}
