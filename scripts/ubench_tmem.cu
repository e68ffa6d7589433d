// Dev microbenchmark: TMEM load / store throughput per SM (tcgen05.ld / st .32x32b, each warp
// its lane quadrant).  One iteration per warp: NLD loads of 32 fp32 columns + wait, then NST
// stores of 32 columns (other columns), as the backward's compute phases do.  kSplit: the
// first half of the warps only load, the second half only store.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2208_08124_b200/csrc -o /tmp/ubt scripts/ubench_tmem.cu
#include <cstdio>
#include "sm100.cuh"
using namespace ub;
template <int NLD, int NST, bool kStWait, bool kSplit>
__global__ void k(uint32_t* sink, long long* cyc, int iters) {
  __shared__ uint32_t base;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;
  if (warp == 0) tmem_alloc(&base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t_row = base + (((warp & 3) * 32) << 16);
  const bool do_ld = !kSplit || warp < nw / 2, do_st = !kSplit || warp >= nw / 2;
  uint32_t acc = 0;
  uint32_t r[32], q[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) { r[e] = e; q[e] = 3 * e + threadIdx.x; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (NLD > 0 && do_ld) {
#pragma unroll
      for (int l = 0; l < NLD; ++l) {
        tmem_ld32(t_row + 32 * l, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += r[e];
      }
    }
    if (NST > 0 && do_st) {
#pragma unroll
      for (int l = 0; l < NST; ++l) {
        q[l] += acc;
        tmem_st32(t_row + 256 + 32 * l, q);
      }
      if (kStWait) tmem_st_wait();
    }
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + q[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(base, 512); }
}
template <int NLD, int NST, bool W, bool S>
void run(const char* name, uint32_t* sink, long long* cyc) {
  const int iters = 2000;
  for (int th : {128, 256, 512}) {
    k<NLD, NST, W, S><<<148, th>>>(sink, cyc, iters);
    k<NLD, NST, W, S><<<148, th>>>(sink, cyc, iters);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
    const double wl = S ? th / 64 : th / 32, ws = S ? th / 64 : th / 32;
    printf("%-34s warps %2d: %6.0f cyc/iter  ld %4.0f B/cyc  st %4.0f B/cyc\n", name, th / 32, m / iters,
           wl * 32 * 128.0 * NLD / (m / iters), ws * 32 * 128.0 * NST / (m / iters));
  }
}
int main() {
  uint32_t* sink; long long* cyc; cudaMalloc(&sink, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  run<2, 0, false, false>("ld x2", sink, cyc);
  run<0, 1, true, false>("st x1 +wait", sink, cyc);
  run<0, 1, false, false>("st x1", sink, cyc);
  run<2, 1, false, false>("ld x2, st x1 (same warp)", sink, cyc);
  run<2, 1, true, false>("ld x2, st x1 +wait (same warp)", sink, cyc);
  run<4, 1, false, false>("ld x4, st x1 (same warp)", sink, cyc);
  run<2, 2, false, false>("ld x2, st x2 (same warp)", sink, cyc);
  run<2, 1, false, true>("ld x2 | st x1 (split warps)", sink, cyc);
  run<2, 1, true, true>("ld x2 | st x1 +wait (split warps)", sink, cyc);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
