// Dev microbenchmark: cycles per 64-element row of the backward's P / dS math (8 warps per
// SM = 2 per SMSP, as in fmha_bwd_kernel), isolated from TMEM, MMA and barriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2208_08124_b200/csrc -o /tmp/ubm scripts/ubench_bwd_math.cu
#include <cstdio>
#include "sm100.cuh"
using namespace ub;
template <int kPoly>
__global__ void k(uint32_t* sink, long long* cyc, float seed, int iters) {
  __shared__ __align__(16) float lse[128], dl[128];
  if (threadIdx.x < 128) { lse[threadIdx.x] = -0.3f * threadIdx.x; dl[threadIdx.x] = 0.01f * threadIdx.x; }
  __syncthreads();
  uint32_t sr[64], dr[64];
#pragma unroll
  for (int e = 0; e < 64; ++e) { sr[e] = __float_as_uint(seed * (e + threadIdx.x)); dr[e] = __float_as_uint(seed * (e - 3.f)); }
  const float c = 0.18f; const uint64_t c2 = f2pack(c, c);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pp[32], pd[32];
    const int x = (threadIdx.x >> 7) & 1;
#pragma unroll
    for (int e = 0; e < 64; e += 4) {
      const float4 l4 = *reinterpret_cast<const float4*>(&lse[x * 64 + e]);
      const float4 d4 = *reinterpret_cast<const float4*>(&dl[x * 64 + e]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ee = e + 2 * u;
        float pa, pb;
        f2unpack(ffma2(f2pack(__uint_as_float(sr[ee]), __uint_as_float(sr[ee + 1])), c2, u ? f2pack(l4.z, l4.w) : f2pack(l4.x, l4.y)), pa, pb);
        if (kPoly && ((ee >> 1) & 3) == 3) f2unpack(ex2_poly2(pa, pb), pa, pb);
        else { pa = ex2f(pa); pb = ex2f(pb); }
        float da, db;
        f2unpack(fmul2(f2pack(pa, pb), fadd2(f2pack(__uint_as_float(dr[ee]), __uint_as_float(dr[ee + 1])), u ? f2pack(d4.z, d4.w) : f2pack(d4.x, d4.y))), da, db);
        pp[ee / 2] = pack_bf16(pa, pb);
        pd[ee / 2] = pack_bf16(da, db);
      }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) acc ^= pp[e] + pd[e];
#pragma unroll
    for (int e = 0; e < 64; ++e) sr[e] ^= (acc & 1);   // loop-carried: keep the math inside
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  uint32_t* sink; long long* cyc; cudaMalloc(&sink, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  for (int th : {128, 256, 512}) {
    for (int poly = 0; poly < 2; ++poly) {
      auto kern = poly ? k<1> : k<0>;
      kern<<<148, th>>>(sink, cyc, 1.0001f, iters); kern<<<148, th>>>(sink, cyc, 1.0001f, iters);
      cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
      printf("warps/SM %2d poly %d: %.0f cycles per 64-element row iteration\n", th / 32, poly, m / iters);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
