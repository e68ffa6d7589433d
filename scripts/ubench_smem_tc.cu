// Dev microbenchmark: do tcgen05 SS-MMA operand reads and LSU shared-memory traffic share
// bandwidth?  One thread issues a stream of SS MMAs (M128 N128 or N64, K16 slices, bf16) from
// smem into TMEM; 8 other warps run an STS.128 (or LDS.128) loop on another smem region.
// Reports cycles per MMA and bytes/cycle of the LSU loop, alone and together.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2208_08124_b200/csrc -o /tmp/ubs scripts/ubench_smem_tc.cu
#include <cstdio>
#include "sm100.cuh"
using namespace ub;

struct __align__(1024) Sm {
  uint8_t a[128 * 128];   // 16 KB A (128 x 64 bf16, SW128)
  uint8_t b[128 * 128];   // 16 KB B
  uint8_t lsu[9][16384];  // LSU traffic region (8 warps x 16 KB ... )
  uint64_t bar;
  uint32_t tmem;
};
template <int kMode, int kNmma>   // mode: 0 MMA only, 1 STS only, 2 both, 3 LDS only, 4 MMA + LDS
__global__ void __launch_bounds__(288, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t raw[];
  Sm& sm = *reinterpret_cast<Sm*>(raw);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&sm.tmem, 256);
  if (threadIdx.x == 32) { mbar_init(&sm.bar, 1); fence_mbar_init(); }
  for (uint32_t i = threadIdx.x; i < sizeof(sm.a) / 16; i += blockDim.x) {
    st_shared_v4(smem_u32(sm.a) + 16 * i, 0x3c003c00u, 0, 0, 0);
    st_shared_v4(smem_u32(sm.b) + 16 * i, 0x3c003c00u, 0, 0, 0);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  long long t0 = clock64();
  const bool do_mma = kMode == 0 || kMode == 2 || kMode == 4;
  const bool do_lsu = kMode >= 1 && kMode != 0;
  if (warp == 8) {
    if (do_mma && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, kNmma, 0, 0);
      const uint32_t a = smem_u32(sm.a), b = smem_u32(sm.b);
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (uint32_t kk = 0; kk < 4; ++kk)
          umma_bf16_ss(tmem, sdesc_sw128(a + kk * 32, 16, 1024), sdesc_sw128(b + kk * 32, 16, 1024), idesc, 1);
        if ((i & 15) == 15) {                     // bound the queue: wait every 16 tiles
          umma_commit(&sm.bar);
          mbar_wait(&sm.bar, (i >> 4) & 1);
        }
      }
      umma_commit(&sm.bar);
      mbar_wait(&sm.bar, (iters >> 4) & 1);
      out[blockIdx.x * 4 + 0] = clock64() - t0;
    }
  } else if (do_lsu && kMode != 0) {
    const uint32_t base = smem_u32(sm.lsu[warp]) + lane * 16;
    uint32_t acc = 0;
    const int n = iters * 2;
    for (int i = 0; i < n; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t addr = base + ((u * 512 + i * 64) & 16383);
        if (kMode == 3 || kMode == 4) {
          uint32_t x, y, z, w;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
          acc += x ^ y ^ z ^ w;
        } else {
          st_shared_v4(addr, acc + i, u, i, lane);
        }
      }
    }
    if (lane == 0) out[blockIdx.x * 4 + 1 + (warp & 1)] = clock64() - t0;
    if (acc == 12345) out[3] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}
template <int M, int N>
void run(const char* name, long long* d, int iters) {
  cudaFuncSetAttribute(k<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Sm));
  k<M, N><<<148, 288, sizeof(Sm)>>>(d, iters);
  k<M, N><<<148, 288, sizeof(Sm)>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mma = 0, lsu = 0;
  for (int i = 0; i < 148; ++i) { mma += h[4 * i]; lsu += h[4 * i + 1]; }
  mma /= 148; lsu /= 148;
  const double mma_bytes = (double)iters * 4 * (128 * 16 * 2 + N * 16 * 2);   // A + B slices
  const double lsu_bytes = (double)iters * 2 * 8 * 512 * 8;                    // 8 warps x 8 x 512 B per i
  printf("%-22s N=%3d: MMA %s  LSU %s\n", name, N,
         (M == 0 || M == 2 || M == 4) ? "" : "-", (M >= 1) ? "" : "-");
  if (M == 0 || M == 2 || M == 4)
    printf("   MMA: %.1f cyc per K16 MMA, operand reads %.0f B/cyc\\n", mma / (iters * 4.0), mma_bytes / mma);
  if (M >= 1) printf("   LSU: %.0f B/cyc (8 warps)\\n", lsu_bytes / lsu);
  memset(h, 0, sizeof(h));
  cudaMemset(d, 0, sizeof(h));
}
int main() {
  long long* d; cudaMalloc(&d, 148 * 4 * 8); cudaMemset(d, 0, 148 * 4 * 8);
  const int iters = 2048;
  run<0, 128>("MMA only", d, iters);
  run<0, 64>("MMA only", d, iters);
  run<1, 128>("STS only", d, iters);
  run<3, 128>("LDS only", d, iters);
  run<2, 128>("MMA + STS", d, iters);
  run<2, 64>("MMA + STS", d, iters);
  run<4, 128>("MMA + LDS", d, iters);
  run<4, 64>("MMA + LDS", d, iters);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
