// Varlen FMHA backward on B200 tensor cores (tcgen05 + TMEM + TMA), bf16 in, fp32 accumulate.
//
// Chain rule of Eq. (1) per sequence and head; dropout replayed from the Philox
// key (R4/R5):
//   Delta_i = sum_d dO_id O_id                               (prologue kernel)
//   S = Q K^T, P = exp(scale S - LSE), dP~ = dO V^T            (recompute, TMEM)
//   P~ = P M/(1-p), dP = dP~ M/(1-p), dS = P (dP - Delta)      (registers)
//   dV += P~^T dO,  dK += dS^T Q  (TMEM, per key tile),  dQ += dS K  (fp32 atomics)
//   dK *= scale, dQ *= scale                                  (epilogues)
//
// Work item = (sequence, head, 128-key tile) along the length-bucketed plan; the CTA
// walks the sequence's query tiles.  Warp roles as in the forward: warp 0 TMA, warp 1
// MMA (one thread), warp 2 TMEM allocator, warps 4-7 "softmax" (thread r owns query row
// r of S/dP, and key row r of dK/dV).  P~ and dS are written once to smem ([q][key],
// UMMA SW128 K-major) and read by three MMAs each through K-major or MN-major descriptors:
//   dV: A = P~^T (MN-major view), B = dO (MN-major)      M128 N64 K128
//   dK: A = dS^T (MN-major view), B = Q  (MN-major)      M128 N64 K128
//   dQ: A = dS   (K-major),       B = K  (MN-major)      M128 N64 K128
// TMEM: S 128 + dP 128 + dQ 64 + dK 64 + dV 64 = 448 of 512 columns.
#include <cmath>

#include "fmha_common.cuh"

namespace ub {
namespace bwd {

constexpr int kD = 64;
constexpr uint32_t kTileBytes = kTile * kD * 2;   // 16 KB
constexpr uint32_t kPBytes = kTile * kTile * 2;   // 32 KB
constexpr int kThreads = 256;
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColDK = 320, kColDV = 384;

struct Smem {
  uint8_t k[kTileBytes];
  uint8_t v[kTileBytes];
  uint8_t q[2][kTileBytes];
  uint8_t dO[2][kTileBytes];
  uint8_t p[kPBytes];
  uint8_t ds[kPBytes];
  uint64_t kv_full, kv_empty;
  uint64_t qdo_full[2], qdo_empty[2];
  uint64_t s_full, s_free, ds_full, pds_empty, dq_full, dq_free, dkv_full, dkv_free;
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

struct Params {
  const int32_t* cu;
  FmhaPlanView plan;
  const float* lse;     // [H, T]
  const float* delta;   // [H, T]
  float* dq_acc;        // [T, H, 64] fp32
  __nv_bfloat16* dqkv;  // [T, 3, H, 64]
  int32_t B, H;
  int64_t T;
  float scale, scale_log2;
  float rp;
  uint32_t thr, k0, k1, off;
};

constexpr uint32_t kIdescS = idesc_bf16_f32(128, 128, 0, 0);     // S, dP: K-major x K-major
constexpr uint32_t kIdescT = idesc_bf16_f32(128, 64, 1, 1);      // dV, dK: A MN-major, B MN-major
constexpr uint32_t kIdescQ = idesc_bf16_f32(128, 64, 0, 1);      // dQ: A K-major, B MN-major

__global__ void __launch_bounds__(kThreads, 1)
fmha_bwd_kernel(const __grid_constant__ CUtensorMap tmap_qkv, const __grid_constant__ CUtensorMap tmap_do,
                const Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_qkv);
    tma_prefetch_desc(&tmap_do);
    mbar_init(&sm.kv_full, 1);
    mbar_init(&sm.kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.qdo_full[s], 1);
      mbar_init(&sm.qdo_empty[s], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_free, 4);
    mbar_init(&sm.ds_full, 4);
    mbar_init(&sm.pds_empty, 1);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_free, 4);
    mbar_init(&sm.dkv_full, 1);
    mbar_init(&sm.dkv_free, 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&sm.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int32_t H = prm.H;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t kv_uses = 0, qit = 0;
      WorkItem it;
      for (int32_t w = blockIdx.x; decode_item(w, prm.plan, prm.cu, prm.B, H, it); w += gridDim.x) {
        mbar_wait(&sm.kv_empty, (kv_uses & 1) ^ 1);
        mbar_expect_tx(&sm.kv_full, 2 * kTileBytes);
        const int32_t krow = it.c0 + it.tile * kTile;
        tma_load_2d(sm.k, &tmap_qkv, &sm.kv_full, (H + it.h) * kD, krow);
        tma_load_2d(sm.v, &tmap_qkv, &sm.kv_full, (2 * H + it.h) * kD, krow);
        ++kv_uses;
        for (int32_t i = 0; i < it.nt; ++i, ++qit) {
          const uint32_t st = qit & 1, ph = (qit >> 1) & 1;
          mbar_wait(&sm.qdo_empty[st], ph ^ 1);
          mbar_expect_tx(&sm.qdo_full[st], 2 * kTileBytes);
          tma_load_2d(sm.q[st], &tmap_qkv, &sm.qdo_full[st], it.h * kD, it.c0 + i * kTile);
          tma_load_2d(sm.dO[st], &tmap_do, &sm.qdo_full[st], it.h * kD, it.c0 + i * kTile);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t kv_uses = 0, qit = 0, s_uses = 0, g_uses = 0, items = 0;
      const uint32_t k_addr = smem_u32(sm.k), v_addr = smem_u32(sm.v);
      const uint32_t p_addr = smem_u32(sm.p), ds_addr = smem_u32(sm.ds);
      auto issue_grads = [&](uint32_t st, bool first) {
        mbar_wait(&sm.ds_full, g_uses & 1);
        mbar_wait(&sm.dq_free, (g_uses & 1) ^ 1);
        if (first) mbar_wait(&sm.dkv_free, (items & 1) ^ 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sm.q[st]), do_addr = smem_u32(sm.dO[st]);
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k) {        // K = query rows, 16 per MMA
          const uint64_t pa = sdesc_sw128(p_addr + k * 2048, kTile * 128, 1024);     // P~^T, MN-major
          const uint64_t da = sdesc_sw128(ds_addr + k * 2048, kTile * 128, 1024);    // dS^T, MN-major
          const uint64_t ob = sdesc_sw128(do_addr + k * 2048, 8192, 1024);           // dO, MN-major
          const uint64_t qb = sdesc_sw128(q_addr + k * 2048, 8192, 1024);            // Q, MN-major
          const uint32_t acc = (first && k == 0) ? 0u : 1u;
          umma_bf16_ss(tmem + kColDV, pa, ob, kIdescT, acc);
          umma_bf16_ss(tmem + kColDK, da, qb, kIdescT, acc);
        }
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k) {        // K = key rows, 16 per MMA
          const uint64_t a = sdesc_sw128(ds_addr + (k >> 2) * (kTile * 128) + (k & 3) * 32, 16, 1024);  // dS, K-major
          const uint64_t b = sdesc_sw128(k_addr + k * 2048, 8192, 1024);                              // K, MN-major
          umma_bf16_ss(tmem + kColDQ, a, b, kIdescQ, k > 0);
        }
        umma_commit(&sm.dq_full);
        umma_commit(&sm.pds_empty);
        umma_commit(&sm.qdo_empty[st]);
        ++g_uses;
      };
      WorkItem it;
      for (int32_t w = blockIdx.x; decode_item(w, prm.plan, prm.cu, prm.B, H, it); w += gridDim.x) {
        mbar_wait(&sm.kv_full, kv_uses & 1);
        uint32_t prev_st = 0;
        for (int32_t i = 0; i < it.nt; ++i, ++qit) {
          const uint32_t st = qit & 1, ph = (qit >> 1) & 1;
          mbar_wait(&sm.qdo_full[st], ph);
          mbar_wait(&sm.s_free, (s_uses & 1) ^ 1);
          tc_fence_after();
          const uint32_t q_addr = smem_u32(sm.q[st]), do_addr = smem_u32(sm.dO[st]);
#pragma unroll
          for (uint32_t k = 0; k < kD / 16; ++k) {
            umma_bf16_ss(tmem + kColS, sdesc_sw128(q_addr + k * 32, 16, 1024), sdesc_sw128(k_addr + k * 32, 16, 1024),
                         kIdescS, k > 0);
            umma_bf16_ss(tmem + kColDP, sdesc_sw128(do_addr + k * 32, 16, 1024),
                         sdesc_sw128(v_addr + k * 32, 16, 1024), kIdescS, k > 0);
          }
          umma_commit(&sm.s_full);
          ++s_uses;
          if (i > 0) issue_grads(prev_st, i == 1);
          prev_st = st;
        }
        issue_grads(prev_st, it.nt == 1);
        umma_commit(&sm.kv_empty);
        umma_commit(&sm.dkv_full);
        ++kv_uses;
        ++items;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax-grad + epilogues
    const uint32_t r = threadIdx.x - 128;
    const uint32_t t_row = tmem + (((warp & 3) * 32) << 16);
    const float c = prm.scale_log2;
    const uint32_t p_addr = smem_u32(sm.p), ds_addr = smem_u32(sm.ds);
    uint32_t s_uses = 0, g_uses = 0, dq_uses = 0, items = 0;
    WorkItem it;
    for (int32_t w = blockIdx.x; decode_item(w, prm.plan, prm.cu, prm.B, H, it); w += gridDim.x) {
      const int32_t kbase = it.tile * kTile;               // first key of this item
      int32_t prev_row = -1;

      auto consume_dq = [&](int32_t row) {
        mbar_wait(&sm.dq_full, dq_uses & 1);
        tc_fence_after();
        uint32_t a0[32], a1[32];
        tmem_ld32(t_row + kColDQ, a0);
        tmem_ld32(t_row + kColDQ + 32, a1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.dq_free);
        ++dq_uses;
        if (row < it.L) {
          float4* dst = reinterpret_cast<float4*>(prm.dq_acc + ((int64_t)(it.c0 + row) * H + it.h) * kD);
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            atomicAdd(dst + g, make_float4(__uint_as_float(a0[4 * g]), __uint_as_float(a0[4 * g + 1]),
                                           __uint_as_float(a0[4 * g + 2]), __uint_as_float(a0[4 * g + 3])));
            atomicAdd(dst + 8 + g, make_float4(__uint_as_float(a1[4 * g]), __uint_as_float(a1[4 * g + 1]),
                                               __uint_as_float(a1[4 * g + 2]), __uint_as_float(a1[4 * g + 3])));
          }
        }
      };

      for (int32_t i = 0; i < it.nt; ++i) {
        const int32_t row = i * kTile + (int32_t)r;          // query row inside the sequence
        const bool row_ok = row < it.L;
        const uint32_t t_glob = (uint32_t)(it.c0 + row);
        const float lse2 = row_ok ? prm.lse[(int64_t)it.h * prm.T + t_glob] * 1.4426950408889634f : INFINITY;
        const float dl = row_ok ? prm.delta[(int64_t)it.h * prm.T + t_glob] : 0.f;
        mbar_wait(&sm.s_full, s_uses & 1);
        tc_fence_after();
        mbar_wait(&sm.pds_empty, (g_uses & 1) ^ 1);
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t sr[32], dr[32];
          tmem_ld32(t_row + kColS + ch * 32, sr);
          tmem_ld32(t_row + kColDP + ch * 32, dr);
          tmem_ld_wait();
          const int32_t key0 = kbase + ch * 32;
          uint32_t keep = 0xFFFFFFFFu;
          if (prm.thr != 0) {
            keep = 0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
              keep |= keep_bits8(key0 + g * 8, t_glob, it.h, prm.off, prm.k0, prm.k1, prm.thr) << (8 * g);
          }
          float pd[32], ds[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const bool kv = key0 + e < it.L;
            const float P = kv ? ex2f(fmaf(__uint_as_float(sr[e]), c, -lse2)) : 0.f;
            const bool kp = (keep >> e) & 1u;
            const float dp = kp ? __uint_as_float(dr[e]) * prm.rp : 0.f;
            pd[e] = kp ? P * prm.rp : 0.f;
            ds[e] = P * (dp - dl);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t unit = (ch & 1) * 4 + u, region = (ch >> 1) * (kTile * 128);
            const uint32_t off = region + sw128_off(r, unit);
            st_shared_v4(p_addr + off, pack_bf16(pd[8 * u], pd[8 * u + 1]), pack_bf16(pd[8 * u + 2], pd[8 * u + 3]),
                         pack_bf16(pd[8 * u + 4], pd[8 * u + 5]), pack_bf16(pd[8 * u + 6], pd[8 * u + 7]));
            st_shared_v4(ds_addr + off, pack_bf16(ds[8 * u], ds[8 * u + 1]), pack_bf16(ds[8 * u + 2], ds[8 * u + 3]),
                         pack_bf16(ds[8 * u + 4], ds[8 * u + 5]), pack_bf16(ds[8 * u + 6], ds[8 * u + 7]));
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sm.s_free);
          mbar_arrive(&sm.ds_full);
        }
        ++s_uses;
        ++g_uses;
        if (i > 0) consume_dq(prev_row);
        prev_row = row;
      }
      consume_dq(prev_row);

      // dK, dV epilogue: thread r owns key row kbase + r
      mbar_wait(&sm.dkv_full, items & 1);
      tc_fence_after();
      uint32_t kr[32], vr[32];
      const int32_t key = kbase + (int32_t)r;
      const int64_t t = (int64_t)it.c0 + key;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        tmem_ld32(t_row + kColDK + half * 32, kr);
        tmem_ld32(t_row + kColDV + half * 32, vr);
        tmem_ld_wait();
        if (key < it.L) {
          uint4* dk = reinterpret_cast<uint4*>(prm.dqkv + ((t * 3 + 1) * H + it.h) * kD + half * 32);
          uint4* dv = reinterpret_cast<uint4*>(prm.dqkv + ((t * 3 + 2) * H + it.h) * kD + half * 32);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float s = prm.scale;
            dk[g] = make_uint4(pack_bf16(__uint_as_float(kr[8 * g]) * s, __uint_as_float(kr[8 * g + 1]) * s),
                               pack_bf16(__uint_as_float(kr[8 * g + 2]) * s, __uint_as_float(kr[8 * g + 3]) * s),
                               pack_bf16(__uint_as_float(kr[8 * g + 4]) * s, __uint_as_float(kr[8 * g + 5]) * s),
                               pack_bf16(__uint_as_float(kr[8 * g + 6]) * s, __uint_as_float(kr[8 * g + 7]) * s));
            dv[g] = make_uint4(pack_bf16(__uint_as_float(vr[8 * g]), __uint_as_float(vr[8 * g + 1])),
                               pack_bf16(__uint_as_float(vr[8 * g + 2]), __uint_as_float(vr[8 * g + 3])),
                               pack_bf16(__uint_as_float(vr[8 * g + 4]), __uint_as_float(vr[8 * g + 5])),
                               pack_bf16(__uint_as_float(vr[8 * g + 6]), __uint_as_float(vr[8 * g + 7])));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dkv_free);
      ++items;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Prologue: Delta[h, t] = sum_d O[t,h,d] dO[t,h,d]; dq_acc[t,h,:] = 0.  Block 0 / warp 0
// additionally builds the length-bucketed plan (fmha_plan.cu semantics).
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ out,
                                                      const __nv_bfloat16* __restrict__ dout, float* __restrict__ delta,
                                                      float* __restrict__ dq_acc, int64_t T, int32_t H) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // row (t, h)
  if (idx >= T * H) return;
  const uint4* o = reinterpret_cast<const uint4*>(out + idx * kD);
  const uint4* g = reinterpret_cast<const uint4*>(dout + idx * kD);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kD / 8; ++k) {
    const uint4 a = o[k], b = g[k];
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s = fmaf(__uint_as_float(av[e] << 16), __uint_as_float(bv[e] << 16), s);
      s = fmaf(__uint_as_float(av[e] & 0xFFFF0000u), __uint_as_float(bv[e] & 0xFFFF0000u), s);
    }
  }
  const int64_t t = idx / H;
  const int32_t h = (int32_t)(idx - t * H);
  delta[(int64_t)h * T + t] = s;
  float4* acc = reinterpret_cast<float4*>(dq_acc + idx * kD);
#pragma unroll
  for (int k = 0; k < kD / 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Epilogue: dQ (bf16) = scale * dq_acc into dqkv[:, 0].
__global__ void __launch_bounds__(256) bwd_dq_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                                                     int64_t T, int32_t H, float scale) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (t, h, 8-wide group)
  if (idx >= T * H * (kD / 8)) return;
  const int64_t row = idx / (kD / 8);
  const int32_t g = (int32_t)(idx - row * (kD / 8));
  const int64_t t = row / H;
  const int32_t h = (int32_t)(row - t * H);
  const float4* a = reinterpret_cast<const float4*>(dq_acc + row * kD + g * 8);
  const float4 x = a[0], y = a[1];
  uint4 v = make_uint4(pack_bf16(x.x * scale, x.y * scale), pack_bf16(x.z * scale, x.w * scale),
                       pack_bf16(y.x * scale, y.y * scale), pack_bf16(y.z * scale, y.w * scale));
  *reinterpret_cast<uint4*>(dqkv + ((t * 3 + 0) * H + h) * kD + g * 8) = v;
}

}  // namespace bwd

size_t fmha_bwd_sm100_ws_bytes(const ub_fmha_params& p) {
  return align_up((size_t)p.T * p.heads * 4, 256) + align_up((size_t)p.T * p.heads * 64 * 4, 256);
}

ub_status fmha_bwd_sm100(const ub_fmha_params& p, const void* qkv, const void* out, const float* lse, const void* dout,
                         const int32_t* d_cu, void* dqkv, void* ws, cudaStream_t s) {
  UB_CHECK_CUDA(cudaFuncSetAttribute(bwd::fmha_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)bwd::kSmemBytes));
  CUtensorMap tq, tdo;
  ub_status st = make_tmap_bf16(&tq, qkv, (uint64_t)3 * p.heads * bwd::kD, (uint64_t)p.T,
                                (uint64_t)3 * p.heads * bwd::kD * 2);
  if (st != UB_OK) return st;
  if ((st = make_tmap_bf16(&tdo, dout, (uint64_t)p.heads * bwd::kD, (uint64_t)p.T, (uint64_t)p.heads * bwd::kD * 2)) !=
      UB_OK)
    return st;
  char* base = static_cast<char*>(ws);
  FmhaPlanView v = fmha_plan_view(base, p.B);
  char* extra = base + align_up(fmha_plan_bytes(p.B), 256);
  float* delta = reinterpret_cast<float*>(extra);
  float* dq_acc = reinterpret_cast<float*>(extra + align_up((size_t)p.T * p.heads * 4, 256));
  const int32_t max_tiles = (p.max_seqlen + kTile - 1) / kTile;
  if ((st = launch_fmha_plan(d_cu, p.B, p.heads, max_tiles, v, s)) != UB_OK) return st;
  const int64_t rows = p.T * p.heads;
  bwd::bwd_pre_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), delta, dq_acc, p.T, p.heads);
  UB_CHECK_LAUNCH();

  bwd::Params prm{};
  prm.cu = d_cu;
  prm.plan = v;
  prm.lse = lse;
  prm.delta = delta;
  prm.dq_acc = dq_acc;
  prm.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  prm.B = p.B;
  prm.H = p.heads;
  prm.T = p.T;
  prm.scale = p.scale;
  prm.scale_log2 = p.scale * 1.4426950408889634f;
  prm.rp = 1.f / (1.f - p.p_dropout);
  prm.thr = p.p_dropout > 0.f ? (uint32_t)floor((double)p.p_dropout * 65536.0) : 0u;
  prm.k0 = (uint32_t)(p.seed & 0xFFFFFFFFull);
  prm.k1 = (uint32_t)(p.seed >> 32);
  prm.off = (uint32_t)(p.offset & 0xFFFFFFFFull);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t max_items = (int64_t)p.heads * (p.B + p.T / kTile + 1);
  const int ctas = p.num_ctas > 0 ? std::min(p.num_ctas, sms) : sms;
  const int grid = (int)std::min<int64_t>(ctas, max_items);
  prof_record(kProfBwd, 0, s);
  bwd::fmha_bwd_kernel<<<grid, bwd::kThreads, bwd::kSmemBytes, s>>>(tq, tdo, prm);
  UB_CHECK_LAUNCH();
  prof_record(kProfBwd, 1, s);
  const int64_t n = rows * (bwd::kD / 8);
  bwd::bwd_dq_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dq_acc, static_cast<__nv_bfloat16*>(dqkv), p.T,
                                                                  p.heads, p.scale);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

}  // namespace ub
