// Unpadded BERT embedding forward and backward ("Embedding Operator
// Optimization"), on packed tokens (no padding rows are looked up).
//   forward : out[t] = W_word[ids[t]] + W_pos[pos[t]] + W_type[seg[t]]      (reading R23)
//   backward: dW_x[idx[t]] += dout[t] for the three tables
// The paper resolves the backward's write conflicts with atomics, packing two fp16 values
// per atomic (half2) and spreading the work over many light blocks.  On B200
// the same idea goes one step further: 16-byte vector reductions (red.global.add.v4.f32, or
// .v4.bf16x2 for bf16 gradients -- 8 values per instruction), one warp per token row, a grid
// sized to the SM count.  The two-row token-type table, which every token hits, is first
// reduced per CTA in shared memory (one vector reduction per column per CTA instead of one
// per token); the segment ids must be < n_type <= 2.
#include <cuda_bf16.h>

#include "sm100.cuh"
#include "ub_internal.h"

namespace ub {
namespace emb {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxVec = 8;                    // E <= 32 * 8 * 8 = 2048
constexpr int kHot = 4;                       // hot word ids cached per CTA (backward)
constexpr int kScan = 128;                    // tokens scanned per CTA to find them

__device__ __forceinline__ void add8(float (&acc)[8], const uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    acc[2 * e] += __uint_as_float(w[e] << 16);
    acc[2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void red_v4_f32(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red_v4_bf16x2(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("red.global.add.noftz.v4.bf16x2 [%0], {%1, %2, %3, %4};" :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

template <int NV>
__global__ void __launch_bounds__(kThreads) embedding_fwd_kernel(const int32_t* __restrict__ ids,
                                                                 const int32_t* __restrict__ pos,
                                                                 const int32_t* __restrict__ seg,
                                                                 const uint4* __restrict__ w_word,
                                                                 const uint4* __restrict__ w_pos,
                                                                 const uint4* __restrict__ w_type,
                                                                 uint4* __restrict__ out, int64_t T, int32_t V) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); t < T; t += warps) {
    const int64_t iw = __ldg(ids + t), ip = __ldg(pos + t), is = __ldg(seg + t);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < V) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        add8(acc, __ldg(w_word + iw * V + v));
        add8(acc, __ldg(w_pos + ip * V + v));
        add8(acc, __ldg(w_type + is * V + v));
        __stcs(out + t * V + v, make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]),
                                           pack_bf16(acc[4], acc[5]), pack_bf16(acc[6], acc[7])));
      }
    }
  }
}

// dW accumulation: kF32 -> fp32 gradients (v4.f32 reductions), else bf16 (v4.bf16x2).
// Token-type rows (n_type <= 2 here: BERT's two segments) are summed per lane in registers,
// per CTA in shared memory, then one vector reduction per column per CTA.
template <int NV, bool kF32>
__global__ void __launch_bounds__(kThreads) embedding_bwd_kernel(const uint4* __restrict__ dout,
                                                                 const int32_t* __restrict__ ids,
                                                                 const int32_t* __restrict__ pos,
                                                                 const int32_t* __restrict__ seg, void* dw_word,
                                                                 void* dw_pos, void* dw_type, int64_t T, int32_t V,
                                                                 int32_t n_type) {
  extern __shared__ float type_acc[];           // [kWarps][2][E], then hot_acc [kHot][E], hot ids [kHot]
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = V * 8;
  float* hot_acc = type_acc + (size_t)kWarps * 2 * E;
  int32_t* hot_id = reinterpret_cast<int32_t*>(hot_acc + (size_t)kHot * E);
  const int64_t warps = (int64_t)gridDim.x * kWarps;
  // Hot word ids of this CTA's tokens (skewed vocabularies: a few ids take a large share of
  // the batch): up to kHot ids occurring at least twice among the CTA's first kScan tokens
  // are summed in shared memory and reduced to global memory once per CTA -- the reductions
  // that serialise on one row in L2 drop from one per token to one per CTA.
  if (warp == 0) {
    int64_t n_cta = (T - (int64_t)blockIdx.x * kWarps + warps - 1) / warps * kWarps;   // upper bound
    if (n_cta < 0) n_cta = 0;
    const int n = n_cta < kScan ? (int)n_cta : kScan;
    auto tok = [&](int j) { return (int64_t)blockIdx.x * kWarps + (j % kWarps) + (int64_t)(j / kWarps) * warps; };
    int32_t my_id[kScan / 32], my_cnt[kScan / 32];
#pragma unroll
    for (int q = 0; q < kScan / 32; ++q) {
      const int j = lane + 32 * q;
      my_id[q] = (j < n && tok(j) < T) ? __ldg(ids + tok(j)) : -1;
      my_cnt[q] = 0;
    }
    for (int i = 0; i < n; ++i) {
      const int32_t x = tok(i) < T ? __ldg(ids + tok(i)) : -2;
#pragma unroll
      for (int q = 0; q < kScan / 32; ++q) my_cnt[q] += (my_id[q] >= 0 && my_id[q] == x) ? 1 : 0;
    }
    for (int h = 0; h < kHot; ++h) {
      int best = 1, best_id = -1;                 // count >= 2 to be worth caching
#pragma unroll
      for (int q = 0; q < kScan / 32; ++q)
        if (my_cnt[q] > best || (my_cnt[q] == best && best > 1 && my_id[q] < best_id)) {
          best = my_cnt[q];
          best_id = my_id[q];
        }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, off), oi = __shfl_xor_sync(0xffffffffu, best_id, off);
        if (ob > best || (ob == best && oi < best_id && oi >= 0)) { best = ob; best_id = oi; }
      }
      if (lane == 0) hot_id[h] = best > 1 ? best_id : -1;
#pragma unroll
      for (int q = 0; q < kScan / 32; ++q)
        if (my_id[q] == best_id) my_cnt[q] = 0;
    }
  }
  for (int i = threadIdx.x; i < kHot * E; i += kThreads) hot_acc[i] = 0.f;
  __syncthreads();
  int32_t hid[kHot];
#pragma unroll
  for (int h = 0; h < kHot; ++h) hid[h] = hot_id[h];
  float ta[2][NV][8];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int e = 0; e < 8; ++e) ta[q][k][e] = 0.f;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < T; t += warps) {
    const int64_t iw = __ldg(ids + t), ip = __ldg(pos + t);
    const int is = __ldg(seg + t);
    int hot = -1;
#pragma unroll
    for (int h = 0; h < kHot; ++h)
      if (hid[h] >= 0 && iw == hid[h]) hot = h;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < V) {
        const uint4 g = __ldcs(dout + t * V + v);
        float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        add8(f, g);
        if (hot >= 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) atomicAdd(&hot_acc[(size_t)hot * E + 8 * v + e], f[e]);
        }
        if (kF32) {
          float* pw = static_cast<float*>(dw_word) + iw * E + 8 * v;
          float* pp = static_cast<float*>(dw_pos) + ip * E + 8 * v;
          if (hot < 0) {
            red_v4_f32(pw, f[0], f[1], f[2], f[3]);
            red_v4_f32(pw + 4, f[4], f[5], f[6], f[7]);
          }
          red_v4_f32(pp, f[0], f[1], f[2], f[3]);
          red_v4_f32(pp + 4, f[4], f[5], f[6], f[7]);
        } else {
          if (hot < 0) red_v4_bf16x2(static_cast<__nv_bfloat16*>(dw_word) + iw * E + 8 * v, g.x, g.y, g.z, g.w);
          red_v4_bf16x2(static_cast<__nv_bfloat16*>(dw_pos) + ip * E + 8 * v, g.x, g.y, g.z, g.w);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          ta[0][k][e] += is == 0 ? f[e] : 0.f;
          ta[1][k][e] += is == 1 ? f[e] : 0.f;
        }
      }
    }
  }
  // per-warp partials -> shared memory -> one reduction per column per CTA (warp order fixed)
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < V)
#pragma unroll
        for (int e = 0; e < 8; ++e) type_acc[((size_t)warp * 2 + q) * E + 8 * v + e] = ta[q][k][e];
    }
  __syncthreads();
  // the hot rows: one reduction per column per CTA
  for (int i = threadIdx.x; i < kHot * V; i += kThreads) {
    const int h = i / V, v = i - h * V;
    if (hid[h] < 0) continue;
    const float* a = hot_acc + (size_t)h * E + 8 * v;
    if (kF32) {
      float* p = static_cast<float*>(dw_word) + (int64_t)hid[h] * E + 8 * v;
      red_v4_f32(p, a[0], a[1], a[2], a[3]);
      red_v4_f32(p + 4, a[4], a[5], a[6], a[7]);
    } else {
      red_v4_bf16x2(static_cast<__nv_bfloat16*>(dw_word) + (int64_t)hid[h] * E + 8 * v, pack_bf16(a[0], a[1]),
                    pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
    }
  }
  for (int i = threadIdx.x; i < n_type * V; i += kThreads) {
    const int q = i / V, v = i - q * V;
    float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int w = 0; w < kWarps; ++w)
#pragma unroll
      for (int e = 0; e < 8; ++e) s8[e] += type_acc[((size_t)w * 2 + q) * E + 8 * v + e];
    if (kF32) {
      float* p = static_cast<float*>(dw_type) + (size_t)q * E + 8 * v;
      red_v4_f32(p, s8[0], s8[1], s8[2], s8[3]);
      red_v4_f32(p + 4, s8[4], s8[5], s8[6], s8[7]);
    } else {
      red_v4_bf16x2(static_cast<__nv_bfloat16*>(dw_type) + (size_t)q * E + 8 * v, pack_bf16(s8[0], s8[1]),
                    pack_bf16(s8[2], s8[3]), pack_bf16(s8[4], s8[5]), pack_bf16(s8[6], s8[7]));
    }
  }
}

int grid_for(int64_t T) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((T + kWarps - 1) / kWarps, (int64_t)sms * 4));
}

}  // namespace emb
}  // namespace ub

using namespace ub;

extern "C" ub_status ub_embedding_fwd(const int32_t* ids, const int32_t* pos, const int32_t* seg, const void* w_word,
                                      const void* w_pos, const void* w_type, int64_t T, int32_t E, void* out,
                                      void* stream) {
  clear_error();
  UB_REQUIRE(ids && pos && seg && w_word && w_pos && w_type && out, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(T >= 0, UB_ERR_INVALID_ARG, "T < 0");
  UB_REQUIRE(E >= 8 && E % 8 == 0 && E <= 32 * emb::kMaxVec * 8, UB_ERR_UNSUPPORTED, "E = %d: multiple of 8 in [8, 2048]",
             E);
  UB_REQUIRE((((uintptr_t)w_word | (uintptr_t)w_pos | (uintptr_t)w_type | (uintptr_t)out) & 15) == 0,
             UB_ERR_INVALID_ARG, "bf16 arrays must be 16-B aligned");
  if (T == 0) return UB_OK;
  const int V = E / 8, nv = (V + 31) / 32;
  auto k = nv <= 4 ? emb::embedding_fwd_kernel<4> : emb::embedding_fwd_kernel<8>;
  launch_pdl(k, dim3(emb::grid_for(T)), dim3(emb::kThreads), 0, as_stream(stream), ids, pos, seg,
             static_cast<const uint4*>(w_word), static_cast<const uint4*>(w_pos), static_cast<const uint4*>(w_type),
             static_cast<uint4*>(out), T, (int32_t)V);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

extern "C" ub_status ub_embedding_bwd(const void* dout, const int32_t* ids, const int32_t* pos, const int32_t* seg,
                                      int64_t T, int32_t E, int32_t n_type, int32_t grad_dtype, void* dw_word,
                                      void* dw_pos, void* dw_type, void* stream) {
  clear_error();
  UB_REQUIRE(dout && ids && pos && seg && dw_word && dw_pos && dw_type, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(T >= 0 && n_type >= 1 && n_type <= 2, UB_ERR_INVALID_ARG, "T < 0 or n_type not in [1, 2]");
  UB_REQUIRE(E >= 8 && E % 8 == 0 && E <= 32 * emb::kMaxVec * 8, UB_ERR_UNSUPPORTED, "E = %d: multiple of 8 in [8, 2048]",
             E);
  UB_REQUIRE(grad_dtype == UB_FP32 || grad_dtype == UB_BF16, UB_ERR_INVALID_ARG, "bad gradient dtype");
  UB_REQUIRE((((uintptr_t)dout | (uintptr_t)dw_word | (uintptr_t)dw_pos | (uintptr_t)dw_type) & 15) == 0,
             UB_ERR_INVALID_ARG, "arrays must be 16-B aligned");
  if (T == 0) return UB_OK;
  const int V = E / 8, nv = (V + 31) / 32;
  const bool f32 = grad_dtype == UB_FP32;
  auto k = f32 ? (nv <= 4 ? emb::embedding_bwd_kernel<4, true> : emb::embedding_bwd_kernel<8, true>)
               : (nv <= 4 ? emb::embedding_bwd_kernel<4, false> : emb::embedding_bwd_kernel<8, false>);
  const int smem = (emb::kWarps * 2 + emb::kHot) * E * (int)sizeof(float) + emb::kHot * (int)sizeof(int32_t);
  // the attribute is set once per kernel: the largest E the kernel supports
  smem_attr_once(reinterpret_cast<const void*>(k), (emb::kWarps * 2 + emb::kHot) * (32 * emb::kMaxVec * 8) *
                                                       (int)sizeof(float) + emb::kHot * (int)sizeof(int32_t));
  launch_pdl(k, dim3(emb::grid_for(T)), dim3(emb::kThreads), (size_t)smem, as_stream(stream),
             static_cast<const uint4*>(dout), ids, pos, seg, dw_word, dw_pos, dw_type, T, (int32_t)V, n_type);
  UB_CHECK_LAUNCH();
  return UB_OK;
}
