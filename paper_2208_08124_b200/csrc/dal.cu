// Dropout_Add_LayerNorm (§IV-C-1 "Kernel Fusion"): one forward kernel, two backward
// kernels (the paper's Table table:kernel-fusion, 3 -> 1 and 5 -> 2), on packed (unpadded)
// rows [T, E], bf16 activations, fp32 statistics.  Formulas and the dropout mask: reading R21
// (oracle/dal.py follows the same equations in fp64).
//
// HBM-bound (fwd 3 x 2 B per element, bwd 5 x 2 B): one warp per row, each lane owning the
// 16-B vectors v = lane + 32 k of the row (coalesced 512-B warp accesses), the row held in
// registers between the two reductions (warp shuffles, no shared memory).  gamma / beta stay
// in registers across the rows a warp walks.  The dropout mask is regenerated in the
// backward from the Philox key (one call per 8 columns, coordinate-pure), never stored.
// dgamma / dbeta: per-lane fp32 partials over a fixed set of rows, summed in a fixed order
// per CTA into the workspace, then across CTAs by the second kernel (deterministic).
#include <cuda_bf16.h>

#include "sm100.cuh"
#include "ub_internal.h"

namespace ub {
namespace dal {

constexpr int kThreads = 256;                 // 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kMaxVec = 8;                    // E <= 32 * 8 * 8 = 2048 (row held in registers)
constexpr uint32_t kSalt = 0xDA100000u;

struct Params {
  int64_t T;
  int32_t E, V;                               // V = E / 8 vectors per row
  float eps, rp;                              // rp = 1 / (1 - thr / 65536)
  uint32_t thr, k0, k1, off;
};

__device__ __forceinline__ void unpack8(const uint4 v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}
// keep bits of columns 8v .. 8v+7 of row t (R21)
__device__ __forceinline__ uint32_t keep8(uint32_t v, uint32_t t, const Params& p) {
  const U4 w = philox4x32_10(v, t, kSalt, p.off, p.k0, p.k1);
  const uint32_t words[4] = {w.x, w.y, w.z, w.w};
  uint32_t bits = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) bits |= (((words[e >> 1] >> (16 * (e & 1))) & 0xFFFFu) >= p.thr ? 1u : 0u) << e;
  return bits;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int NV, bool kDrop>
__global__ void __launch_bounds__(kThreads, 3) dal_fwd_kernel(const uint4* __restrict__ a, const uint4* __restrict__ res,
                                                           const uint4* __restrict__ gamma, const uint4* __restrict__ beta,
                                                           uint4* __restrict__ y, float* __restrict__ mean,
                                                           float* __restrict__ rstd, const Params p) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); t < p.T; t += warps) {
    if (t + warps < p.T) {                         // warm L2 with this warp's next row
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (lane + 32 * k < p.V) {
          prefetch_l2(a + (t + warps) * p.V + lane + 32 * k);
          prefetch_l2(res + (t + warps) * p.V + lane + 32 * k);
        }
    }
    float z[NV][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < p.V) {
        float av[8], rv[8];
        unpack8(__ldcs(a + t * p.V + v), av);
        unpack8(__ldcs(res + t * p.V + v), rv);
        const uint32_t keep = kDrop ? keep8((uint32_t)v, (uint32_t)t, p) : 0xFFu;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          z[k][e] = rv[e] + (((keep >> e) & 1u) ? av[e] * p.rp : 0.f);
          s += z[k][e];
        }
      }
    }
    const float mu = warp_sum(s) / (float)p.E;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (lane + 32 * k < p.V)
#pragma unroll
        for (int e = 0; e < 8; ++e) q += (z[k][e] - mu) * (z[k][e] - mu);
    const float rs = rsqrtf(warp_sum(q) / (float)p.E + p.eps);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < p.V) {
        float o[8], g[8], b[8];
        unpack8(__ldg(gamma + v), g);                    // L1-resident across rows
        unpack8(__ldg(beta + v), b);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (z[k][e] - mu) * rs * g[e] + b[e];
        __stcs(y + t * p.V + v, pack8(o));
      }
    }
    if (lane == 0) {
      mean[t] = mu;
      rstd[t] = rs;
    }
  }
}

// Backward 1/2: da, dres per row; per-CTA partial dgamma / dbeta into ws [gridDim][2][E].
// For E <= 1024 each lane sums its columns' dgamma / dbeta over the warp's rows in registers
// (one CTA per SM for the registers; against per-row read-modify-writes of a per-warp smem
// slice at two CTAs per SM: 52.2 -> 51.3 us at p = 0, 54.3 -> 52.4 at p = 0.1 on the config-2
// rows) and writes the warp's slice to shared memory once; wider rows keep the per-row smem
// slice (the register sums would spill).  The slices are summed in warp order (no atomics).
template <int NV> __host__ __device__ constexpr bool bwd_regacc() { return NV <= 4; }   // E <= 1024: register sums
template <int NV> __host__ __device__ constexpr int bwd_per_sm() { return bwd_regacc<NV>() ? 1 : 2; }
template <int NV, bool kDrop>
__global__ void __launch_bounds__(kThreads, bwd_per_sm<NV>()) dal_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ a,
                                                              const uint4* __restrict__ res, const uint4* __restrict__ gamma,
                                                              const float* __restrict__ mean, const float* __restrict__ rstd,
                                                              uint4* __restrict__ da, uint4* __restrict__ dres,
                                                              float* __restrict__ part, const Params p) {
  extern __shared__ float4 acc4[];                // [kWarps][2][E / 4]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t warps = (int64_t)gridDim.x * kWarps;
  const int E4 = p.E / 4;
  float4* my_g = acc4 + (size_t)warp * 2 * E4;    // this warp's dgamma slice, then dbeta
  float4* my_b = my_g + E4;
  constexpr bool kRegAcc = bwd_regacc<NV>();
  if (!kRegAcc) {
    for (int i = lane; i < 2 * E4; i += 32) my_g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
  }
  float ag[kRegAcc ? NV : 1][8], ab[kRegAcc ? NV : 1][8];   // this lane's dgamma / dbeta columns, over its rows
  if (kRegAcc) {
#pragma unroll
    for (int k = 0; k < (kRegAcc ? NV : 1); ++k)
#pragma unroll
      for (int e = 0; e < 8; ++e) ag[k][e] = ab[k][e] = 0.f;
  }
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) ag[k][e] = ab[k][e] = 0.f;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < p.T; t += warps) {
    if (t + warps < p.T) {                         // warm L2 with this warp's next row
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (lane + 32 * k < p.V) {
          prefetch_l2(a + (t + warps) * p.V + lane + 32 * k);
          prefetch_l2(res + (t + warps) * p.V + lane + 32 * k);
          prefetch_l2(dy + (t + warps) * p.V + lane + 32 * k);
        }
    }
    const float mu = mean[t], rs = rstd[t];
    float xh[NV][8], gy[NV][8];
    uint32_t keepv[NV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < p.V) {
        float av[8], rv[8], dv[8], g[8];
        unpack8(__ldcs(a + t * p.V + v), av);
        unpack8(__ldcs(res + t * p.V + v), rv);
        unpack8(__ldcs(dy + t * p.V + v), dv);
        unpack8(__ldg(gamma + v), g);
        keepv[k] = kDrop ? keep8((uint32_t)v, (uint32_t)t, p) : 0xFFu;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float z = rv[e] + (((keepv[k] >> e) & 1u) ? av[e] * p.rp : 0.f);
          xh[k][e] = (z - mu) * rs;
          gy[k][e] = dv[e] * g[e];
          s1 += gy[k][e];
          s2 += gy[k][e] * xh[k][e];
        }
        if constexpr (kRegAcc) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            ag[k][e] += dv[e] * xh[k][e];
            ab[k][e] += dv[e];
          }
        } else {                                     // E > 1024: the warp's smem slice, per row
          float4* pg = my_g + 2 * v;                 // columns 8v .. 8v+7
          float4* pb = my_b + 2 * v;
          const float4 g0 = pg[0], g1 = pg[1], b0 = pb[0], b1 = pb[1];
          pg[0] = make_float4(g0.x + dv[0] * xh[k][0], g0.y + dv[1] * xh[k][1], g0.z + dv[2] * xh[k][2], g0.w + dv[3] * xh[k][3]);
          pg[1] = make_float4(g1.x + dv[4] * xh[k][4], g1.y + dv[5] * xh[k][5], g1.z + dv[6] * xh[k][6], g1.w + dv[7] * xh[k][7]);
          pb[0] = make_float4(b0.x + dv[0], b0.y + dv[1], b0.z + dv[2], b0.w + dv[3]);
          pb[1] = make_float4(b1.x + dv[4], b1.y + dv[5], b1.z + dv[6], b1.w + dv[7]);
        }
      }
    }
    const float m1 = warp_sum(s1) / (float)p.E, m2 = warp_sum(s2) / (float)p.E;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = lane + 32 * k;
      if (v < p.V) {
        float dz[8], dav[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dz[e] = rs * (gy[k][e] - m1 - xh[k][e] * m2);
          dav[e] = ((keepv[k] >> e) & 1u) ? dz[e] * p.rp : 0.f;
        }
        __stcs(dres + t * p.V + v, pack8(dz));
        __stcs(da + t * p.V + v, pack8(dav));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < (kRegAcc ? NV : 0); ++k) {  // (register sums) the warp's slice once, at the end
    const int v = lane + 32 * k;
    if (v < p.V) {
      my_g[2 * v] = make_float4(ag[k][0], ag[k][1], ag[k][2], ag[k][3]);
      my_g[2 * v + 1] = make_float4(ag[k][4], ag[k][5], ag[k][6], ag[k][7]);
      my_b[2 * v] = make_float4(ab[k][0], ab[k][1], ab[k][2], ab[k][3]);
      my_b[2 * v + 1] = make_float4(ab[k][4], ab[k][5], ab[k][6], ab[k][7]);
    }
  }
  __syncthreads();
  // CTA partials: the warps' slices summed in warp order (deterministic)
  for (int c = threadIdx.x; c < 2 * E4; c += kThreads) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float4 x = acc4[(size_t)w * 2 * E4 + c];
      s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
    }
    reinterpret_cast<float4*>(part)[(size_t)blockIdx.x * 2 * E4 + c] = s;
  }
}

// Backward 2/2: dgamma[c] = sum over CTAs of the partials, in CTA order (deterministic).
__global__ void __launch_bounds__(256) dal_bwd_reduce_kernel(const float* __restrict__ part, int32_t nparts, int32_t E,
                                                             float* __restrict__ dgamma, float* __restrict__ dbeta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= 2 * E) return;
  const int which = c / E, col = c - which * E;
  float acc = 0.f;
  for (int b = 0; b < nparts; ++b) acc += part[((int64_t)b * 2 + which) * E + col];
  (which ? dbeta : dgamma)[col] = acc;
}

static int grid_for(int64_t T, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (T + kWarps - 1) / kWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * per_sm));
}
constexpr int kFwdPerSm = 3, kBwdPerSm = 2;   // resident CTAs per SM (launch bounds; the backward's largest)
// The backward workspace holds one partial per CTA.  Its size must not depend on whichever
// device is current when it is queried: it is sized for the largest grid any device can get
// (kMaxSms SMs), and the launch never exceeds it.
constexpr int kMaxSms = 256;
static int64_t max_bwd_grid(int64_t T) {
  return std::max<int64_t>(1, std::min<int64_t>((T + kWarps - 1) / kWarps, (int64_t)kMaxSms * kBwdPerSm));
}

static Params make_params(int64_t T, int32_t E, float p, float eps, uint64_t seed, uint64_t offset) {
  Params q{};
  q.T = T;
  q.E = E;
  q.V = E / 8;
  q.eps = eps;
  q.thr = p > 0.f ? (uint32_t)floor((double)p * 65536.0) : 0u;        // R21: 16-bit decisions
  q.rp = p > 0.f ? (float)(1.0 / (1.0 - q.thr / 65536.0)) : 1.f;        // exact inverse keep probability
  q.k0 = (uint32_t)(seed & 0xFFFFFFFFull);
  q.k1 = (uint32_t)(seed >> 32);
  q.off = (uint32_t)(offset & 0xFFFFFFFFull);
  return q;
}

template <int NV>
static void launch_fwd(bool drop, int grid, cudaStream_t s, const void* a, const void* res, const void* gamma,
                       const void* beta, void* y, float* mean, float* rstd, const Params& q) {
  auto k = drop ? dal_fwd_kernel<NV, true> : dal_fwd_kernel<NV, false>;
  k<<<grid, kThreads, 0, s>>>(static_cast<const uint4*>(a), static_cast<const uint4*>(res),
                              static_cast<const uint4*>(gamma), static_cast<const uint4*>(beta), static_cast<uint4*>(y),
                              mean, rstd, q);
}
template <int NV>
static void launch_bwd(bool drop, int grid, cudaStream_t s, const void* dy, const void* a, const void* res,
                       const void* gamma, const float* mean, const float* rstd, void* da, void* dres, float* part,
                       const Params& q) {
  auto k = drop ? dal_bwd_kernel<NV, true> : dal_bwd_kernel<NV, false>;
  const int smem = kWarps * 2 * q.E * (int)sizeof(float);
  // the attribute is set once per kernel: the largest E the kernel supports
  smem_attr_once(reinterpret_cast<const void*>(k), kWarps * 2 * (32 * kMaxVec * 8) * (int)sizeof(float));
  k<<<grid, kThreads, smem, s>>>(static_cast<const uint4*>(dy), static_cast<const uint4*>(a),
                              static_cast<const uint4*>(res), static_cast<const uint4*>(gamma), mean, rstd,
                              static_cast<uint4*>(da), static_cast<uint4*>(dres), part, q);
}

static ub_status check_args(int64_t T, int32_t E, float p, float eps) {
  UB_REQUIRE(T >= 0, UB_ERR_INVALID_ARG, "T < 0");
  UB_REQUIRE(E >= 8 && E % 8 == 0 && E <= 32 * kMaxVec * 8, UB_ERR_UNSUPPORTED,
             "E = %d: need a multiple of 8 in [8, 2048]", E);
  UB_REQUIRE(p >= 0.f && p < 1.f, UB_ERR_INVALID_ARG, "p_dropout %f not in [0, 1)", (double)p);
  UB_REQUIRE(p == 0.f || floor((double)p * 65536.0) >= 1.0, UB_ERR_INVALID_ARG,
             "p_dropout %g < 1/65536: the 16-bit keep decisions (R21) would drop nothing", (double)p);
  UB_REQUIRE(eps > 0.f, UB_ERR_INVALID_ARG, "eps <= 0");
  return UB_OK;
}

}  // namespace dal
}  // namespace ub

using namespace ub;

extern "C" ub_status ub_dal_fwd(const void* a, const void* res, const void* gamma, const void* beta, int64_t T, int32_t E,
                                float p_dropout, float eps, uint64_t seed, uint64_t offset, void* y, float* mean,
                                float* rstd, void* stream) {
  clear_error();
  ub_status st = dal::check_args(T, E, p_dropout, eps);
  if (st != UB_OK) return st;
  UB_REQUIRE(a && res && gamma && beta && y && mean && rstd, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE((((uintptr_t)a | (uintptr_t)res | (uintptr_t)gamma | (uintptr_t)beta | (uintptr_t)y) & 15) == 0,
             UB_ERR_INVALID_ARG, "bf16 arrays must be 16-B aligned");
  if (T == 0) return UB_OK;
  const dal::Params q = dal::make_params(T, E, p_dropout, eps, seed, offset);
  const int grid = dal::grid_for(T, dal::kFwdPerSm);
  const bool drop = p_dropout > 0.f;
  cudaStream_t s = as_stream(stream);
  const int nv = (q.V + 31) / 32;
  prof_record(kProfDalFwd, 0, s);
  if (nv <= 4) dal::launch_fwd<4>(drop, grid, s, a, res, gamma, beta, y, mean, rstd, q);
  else dal::launch_fwd<8>(drop, grid, s, a, res, gamma, beta, y, mean, rstd, q);
  UB_CHECK_LAUNCH();
  prof_record(kProfDalFwd, 1, s);
  return UB_OK;
}

extern "C" size_t ub_dal_bwd_workspace_bytes(int64_t T, int32_t E) {
  return (size_t)dal::max_bwd_grid(T) * 2 * (size_t)(E > 0 ? E : 0) * sizeof(float);
}

extern "C" ub_status ub_dal_bwd(const void* dy, const void* a, const void* res, const void* gamma, const float* mean,
                                const float* rstd, int64_t T, int32_t E, float p_dropout, uint64_t seed, uint64_t offset,
                                void* da, void* dres, float* dgamma, float* dbeta, void* ws, void* stream) {
  clear_error();
  ub_status st = dal::check_args(T, E, p_dropout, 1.f);
  if (st != UB_OK) return st;
  UB_REQUIRE(dy && a && res && gamma && mean && rstd && da && dres && dgamma && dbeta && ws, UB_ERR_INVALID_ARG,
             "null pointer");
  UB_REQUIRE((((uintptr_t)dy | (uintptr_t)a | (uintptr_t)res | (uintptr_t)gamma | (uintptr_t)da | (uintptr_t)dres) & 15) ==
                 0,
             UB_ERR_INVALID_ARG, "bf16 arrays must be 16-B aligned");
  const dal::Params q = dal::make_params(T, E, p_dropout, 1.f, seed, offset);
  const int nv = (q.V + 31) / 32;
  const int per_sm = nv <= 4 ? dal::bwd_per_sm<4>() : dal::bwd_per_sm<8>();
  const int grid = (int)std::min<int64_t>(dal::grid_for(T, per_sm), dal::max_bwd_grid(T));
  const bool drop = p_dropout > 0.f;
  cudaStream_t s = as_stream(stream);
  float* part = static_cast<float*>(ws);
  prof_record(kProfDalBwd, 0, s);
  if (T > 0) {
    if (nv <= 4) dal::launch_bwd<4>(drop, grid, s, dy, a, res, gamma, mean, rstd, da, dres, part, q);
    else dal::launch_bwd<8>(drop, grid, s, dy, a, res, gamma, mean, rstd, da, dres, part, q);
    UB_CHECK_LAUNCH();
  } else {
    UB_CHECK_CUDA(cudaMemsetAsync(part, 0, (size_t)grid * 2 * E * sizeof(float), s));
  }
  dal::dal_bwd_reduce_kernel<<<(2 * E + 255) / 256, 256, 0, s>>>(part, grid, E, dgamma, dbeta);
  UB_CHECK_LAUNCH();
  prof_record(kProfDalBwd, 1, s);
  return UB_OK;
}
