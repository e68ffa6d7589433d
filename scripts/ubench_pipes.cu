// Dev microbenchmark: issue throughput (ops / clock / SM) of MUFU.EX2, the bf16x2 pack
// conversion (F2FP), the integer pack, FFMA2, and ex2+cvt mixed -- do EX2 and F2FP share a
// pipe on sm_100a?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub scripts/ubench_pipes.cu
#include <cstdio>
#include <cstdint>

#define N_IT 4096
#define CH 8

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t cvt2(float lo, float hi) {
  uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r;
}
__device__ __forceinline__ uint32_t ipack(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("mad.lo.u32 %0, %0, 1, 32768;" : "+r"(a));
  asm volatile("mad.lo.u32 %0, %0, 1, 32768;" : "+r"(b));
  asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

template <int MODE>
__global__ void k(float* out, long long* cyc, float seed) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-6f - 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0) v[c] = ex2f(v[c]);
      if (MODE == 1) v[c] = __uint_as_float(cvt2(v[c], v[c] + 1.f) & 0x3FFFFFFFu);
      if (MODE == 2) { v[c] = ex2f(v[c]); v[c] = __uint_as_float(cvt2(v[c], v[(c + 1) % CH]) & 0x3FFFFFFFu); }
      if (MODE == 3) v[c] = __uint_as_float(ipack(__float_as_uint(v[c]), __float_as_uint(v[(c + 1) % CH])) & 0x3FFFFFFFu);
      if (MODE == 4) v[c] = fmaf(v[c], 0.999f, 0.001f);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 1024;
  float* out; long long* cyc; cudaMalloc(&out, sizeof(float) * sms * threads); cudaMalloc(&cyc, sizeof(long long) * sms);
  const char* names[] = {"ex2", "cvt.bf16x2", "ex2+cvt", "int-pack(2 IMAD+PRMT)", "ffma"};
  void (*ks[])(float*, long long*, float) = {k<0>, k<1>, k<2>, k<3>, k<4>};
  for (int m = 0; m < 5; ++m) {
    ks[m]<<<sms, threads>>>(out, cyc, 1.f);
    ks[m]<<<sms, threads>>>(out, cyc, 1.f);
    cudaDeviceSynchronize();
    long long h[1024]; cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < sms; ++i) mean += h[i]; mean /= sms;
    const double ops = (double)threads * N_IT * CH;  // per SM (one block per SM)
    printf("%-24s %8.2f ops/clk/SM (%s)\n", names[m], ops / mean, m == 2 ? "pairs of ex2+cvt" : "");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
