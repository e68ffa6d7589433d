// Dev microbenchmark: MUFU throughput of ex2.approx.f32 vs ex2.approx.f16x2 (results per
// clock per SM), 16 warps per SM, independent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ube scripts/ubench_ex2.cu && /tmp/ube
#include <cstdio>
#include <cuda_fp16.h>
template <int kMode>
__global__ void k(unsigned* sink, long long* cyc, float seed, int iters) {
  unsigned r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { __half2 h = __floats2half2_rn(-seed * (i + 1) * 0.01f, -seed * i * 0.02f); r[i] = *reinterpret_cast<unsigned*>(&h); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (kMode == 0) { float x = __uint_as_float(r[i]); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x)); r[i] = __float_as_uint(x); }
      else asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= r[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  unsigned* sink; long long* cyc; cudaMalloc(&sink, 148 * 512 * 4); cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 512>>>(sink, cyc, 1.f, iters); else k<1><<<148, 512>>>(sink, cyc, 1.f, iters);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double results = 512.0 * iters * 16 * (mode ? 2 : 1);
    printf("%s: %.2f results/clk/SM, %.2f instr/clk/SM\n", mode ? "ex2.f16x2" : "ex2.f32", results / c, 512.0 * iters * 16 / c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
