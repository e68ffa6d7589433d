// Varlen FMHA forward on B200 tensor cores (tcgen05 + TMEM + TMA), bf16 in, fp32 accumulate.
//
// Eq. (1) of the paper per sequence and head on cu_seqlens-packed tokens (P:302,
// P:313).  One persistent launch walks the length-bucketed plan (fmha_plan.cu).
//
// CTA = 8 warps, warp-specialised:
//   warp 0      TMA producer: Q tile (128 x 64) once per item; K_j, V_j tiles (128 x 64)
//               through a 2-stage ring, straight from the packed qkv [T, 3*H*64] matrix.
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T  (M128 N128 K64, K-major x K-major)
//               into TMEM (double-buffered), then O_j = P_j V_j (M128 N64 K128, P from
//               smem K-major, V MN-major) into TMEM (double-buffered).
//   warp 2      TMEM allocator.
//   warps 4-7   softmax: thread r owns query row r; tcgen05.ld its S row, masks keys past
//               the sequence end, online max / exp2 / row sum in registers, writes P (bf16)
//               to smem in the UMMA SW128 layout, and accumulates the per-tile O_j
//               (relative to the running max) in registers; epilogue writes O and LSE.
// Boxes that run past a sequence end read the next sequence's rows: those keys are
// masked to -inf and those query rows are never stored.
#include <cmath>

#include "fmha_common.cuh"

namespace ub {
namespace fwd {

constexpr int kD = 64;
constexpr int kStages = 2;
constexpr uint32_t kTileBytes = kTile * kD * 2;          // 16 KB
constexpr uint32_t kPBytes = kTile * kTile * 2;          // 32 KB (2 chunks of 64 keys)
constexpr int kThreads = 256;

struct Smem {
  uint8_t q[kTileBytes];
  uint8_t k[kStages][kTileBytes];
  uint8_t v[kStages][kTileBytes];
  uint8_t p[2][kPBytes];
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages], v_full[kStages], kv_empty[kStages];
  uint64_t s_full[2], s_free[2], p_full[2], p_empty[2], o_full[2], o_free[2];
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

struct Params {
  const int32_t* cu;
  FmhaPlanView plan;
  __nv_bfloat16* out;
  float* lse;
  int32_t B, H;
  int64_t T;
  float scale, scale_log2;
  float rp;           // 1 / (1 - p)
  uint32_t thr, k0, k1, off;
};

constexpr uint32_t kIdescS = idesc_bf16_f32(128, 128, 0, 0);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 64, 0, 1);

__global__ void __launch_bounds__(kThreads, 1)
fmha_fwd_kernel(const __grid_constant__ CUtensorMap tmap_qkv, const Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_qkv);
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], 4);
      mbar_init(&sm.p_full[s], 4);
      mbar_init(&sm.p_empty[s], 1);
      mbar_init(&sm.o_full[s], 1);
      mbar_init(&sm.o_free[s], 4);
    }
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
      uint32_t q_uses = 0, kv_it = 0;
      WorkItem it;
      for (int32_t w = blockIdx.x; decode_item(w, prm.plan, prm.cu, prm.B, H, it); w += gridDim.x) {
        mbar_wait(&sm.q_empty, (q_uses & 1) ^ 1);
        mbar_expect_tx(&sm.q_full, kTileBytes);
        tma_load_2d(sm.q, &tmap_qkv, &sm.q_full, it.h * kD, it.c0 + it.tile * kTile);
        ++q_uses;
        for (int32_t j = 0; j < it.nt; ++j, ++kv_it) {
          const uint32_t st = kv_it % kStages, ph = (kv_it / kStages) & 1;
          mbar_wait(&sm.kv_empty[st], ph ^ 1);
          mbar_expect_tx(&sm.k_full[st], kTileBytes);
          tma_load_2d(sm.k[st], &tmap_qkv, &sm.k_full[st], (H + it.h) * kD, it.c0 + j * kTile);
          mbar_expect_tx(&sm.v_full[st], kTileBytes);
          tma_load_2d(sm.v[st], &tmap_qkv, &sm.v_full[st], (2 * H + it.h) * kD, it.c0 + j * kTile);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t q_uses = 0, kv_it = 0, s_it = 0, p_it = 0, o_it = 0;
      const uint32_t q_addr = smem_u32(sm.q);
      auto issue_pv = [&](uint32_t st, uint32_t vph) {
        const uint32_t pb = p_it & 1, ob = o_it & 1;
        mbar_wait(&sm.p_full[pb], (p_it >> 1) & 1);
        mbar_wait(&sm.v_full[st], vph);
        mbar_wait(&sm.o_free[ob], ((o_it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(sm.p[pb]), v_addr = smem_u32(sm.v[st]);
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k) {
          const uint64_t a = sdesc_sw128(p_addr + (k >> 2) * (kTile * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(v_addr + k * 2048, 8192, 1024);
          umma_bf16_ss(tmem + 256 + ob * 64, a, bd, kIdescPV, k > 0);
        }
        umma_commit(&sm.o_full[ob]);
        umma_commit(&sm.p_empty[pb]);
        umma_commit(&sm.kv_empty[st]);
        ++p_it;
        ++o_it;
      };
      WorkItem it;
      for (int32_t w = blockIdx.x; decode_item(w, prm.plan, prm.cu, prm.B, H, it); w += gridDim.x) {
        mbar_wait(&sm.q_full, q_uses & 1);
        tc_fence_after();
        uint32_t prev_st = 0, prev_ph = 0;
        for (int32_t j = 0; j < it.nt; ++j, ++kv_it) {
          const uint32_t st = kv_it % kStages, ph = (kv_it / kStages) & 1;
          mbar_wait(&sm.k_full[st], ph);
          const uint32_t sb = s_it & 1;
          mbar_wait(&sm.s_free[sb], ((s_it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sm.k[st]);
#pragma unroll
          for (uint32_t k = 0; k < kD / 16; ++k) {
            const uint64_t a = sdesc_sw128(q_addr + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(k_addr + k * 32, 16, 1024);
            umma_bf16_ss(tmem + sb * 128, a, bd, kIdescS, k > 0);
          }
          umma_commit(&sm.s_full[sb]);
          ++s_it;
          if (j == it.nt - 1) umma_commit(&sm.q_empty);
          if (j > 0) issue_pv(prev_st, prev_ph);
          prev_st = st;
          prev_ph = ph;
        }
        issue_pv(prev_st, prev_ph);
        ++q_uses;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const uint32_t r = threadIdx.x - 128;                 // query row inside the tile
    const uint32_t lane_base = (warp & 3) * 32;           // TMEM sub-partition of this warp
    const uint32_t t_row = tmem + (lane_base << 16);
    const float c = prm.scale_log2;
    uint32_t s_it = 0, p_it = 0, o_it = 0;
    WorkItem it;
    for (int32_t w = blockIdx.x; decode_item(w, prm.plan, prm.cu, prm.B, H, it); w += gridDim.x) {
      const int32_t row = it.tile * kTile + (int32_t)r;
      const uint32_t t_glob = (uint32_t)(it.c0 + row);
      float m = -INFINITY, l = 0.f, m_acc = -INFINITY, m_tile = -INFINITY;
      float acc[kD];
#pragma unroll
      for (int d = 0; d < kD; ++d) acc[d] = 0.f;

      auto consume_o = [&](float mj) {
        const uint32_t ob = o_it & 1;
        mbar_wait(&sm.o_full[ob], (o_it >> 1) & 1);
        tc_fence_after();
        uint32_t o0[32], o1[32];
        tmem_ld32(t_row + 256 + ob * 64, o0);
        tmem_ld32(t_row + 256 + ob * 64 + 32, o1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.o_free[ob]);
        ++o_it;
        const float f = ex2f((m_acc - mj) * c);
#pragma unroll
        for (int d = 0; d < 32; ++d) {
          acc[d] = fmaf(acc[d], f, __uint_as_float(o0[d]));
          acc[32 + d] = fmaf(acc[32 + d], f, __uint_as_float(o1[d]));
        }
        m_acc = mj;
      };

      for (int32_t j = 0; j < it.nt; ++j) {
        const uint32_t sb = s_it & 1;
        mbar_wait(&sm.s_full[sb], (s_it >> 1) & 1);
        tc_fence_after();
        float s[kTile];
        {
          uint32_t raw[32];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            tmem_ld32(t_row + sb * 128 + q * 32, raw);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) s[q * 32 + e] = __uint_as_float(raw[e]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[sb]);
        ++s_it;

        const int32_t kvalid = it.L - j * kTile;
        if (kvalid < kTile) {
#pragma unroll
          for (int e = 0; e < kTile; ++e)
            if (e >= kvalid) s[e] = -INFINITY;
        }
        float mt = s[0];
#pragma unroll
        for (int e = 1; e < kTile; ++e) mt = fmaxf(mt, s[e]);
        const float m_new = fmaxf(m, mt);
        const float alpha = ex2f((m - m_new) * c);
        const float neg = -m_new * c;
        float rs = 0.f;
#pragma unroll
        for (int e = 0; e < kTile; ++e) {
          s[e] = ex2f(fmaf(s[e], c, neg));
          rs += s[e];
        }
        l = fmaf(l, alpha, rs);
        m = m_new;
        if (prm.thr != 0) {
#pragma unroll
          for (int g = 0; g < kTile / 8; ++g) {
            const uint32_t bits = keep_bits8(j * kTile + g * 8, t_glob, it.h, prm.off, prm.k0, prm.k1, prm.thr);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (!((bits >> e) & 1u)) s[g * 8 + e] = 0.f;
          }
        }
        // P (bf16) -> smem, K-major SW128: chunk g holds keys 8g..8g+7
        const uint32_t pb = p_it & 1;
        mbar_wait(&sm.p_empty[pb], ((p_it >> 1) & 1) ^ 1);
        const uint32_t p_addr = smem_u32(sm.p[pb]);
#pragma unroll
        for (int g = 0; g < kTile / 8; ++g) {
          const uint32_t addr = p_addr + (g >> 3) * (kTile * 128) + sw128_off(r, g & 7);
          st_shared_v4(addr, pack_bf16(s[g * 8 + 0], s[g * 8 + 1]), pack_bf16(s[g * 8 + 2], s[g * 8 + 3]),
                       pack_bf16(s[g * 8 + 4], s[g * 8 + 5]), pack_bf16(s[g * 8 + 6], s[g * 8 + 7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[pb]);
        ++p_it;
        if (j > 0) consume_o(m_tile);
        m_tile = m;
      }
      consume_o(m_tile);

      if (row < it.L) {
        const float inv = prm.rp / l;
        uint4* op = reinterpret_cast<uint4*>(prm.out + ((int64_t)t_glob * H + it.h) * kD);
#pragma unroll
        for (int g = 0; g < kD / 8; ++g) {
          uint4 v;
          v.x = pack_bf16(acc[g * 8 + 0] * inv, acc[g * 8 + 1] * inv);
          v.y = pack_bf16(acc[g * 8 + 2] * inv, acc[g * 8 + 3] * inv);
          v.z = pack_bf16(acc[g * 8 + 4] * inv, acc[g * 8 + 5] * inv);
          v.w = pack_bf16(acc[g * 8 + 6] * inv, acc[g * 8 + 7] * inv);
          op[g] = v;
        }
        prm.lse[(int64_t)it.h * prm.T + t_glob] = m * prm.scale + logf(l);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace fwd

ub_status fmha_fwd_sm100(const ub_fmha_params& p, const void* qkv, const int32_t* d_cu, void* out, float* lse,
                         void* ws, cudaStream_t s) {
  UB_CHECK_CUDA(cudaFuncSetAttribute(fwd::fmha_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)fwd::kSmemBytes));
  CUtensorMap tmap;
  ub_status st = make_tmap_bf16(&tmap, qkv, (uint64_t)3 * p.heads * fwd::kD, (uint64_t)p.T,
                                (uint64_t)3 * p.heads * fwd::kD * 2);
  if (st != UB_OK) return st;
  FmhaPlanView v = fmha_plan_view(ws, p.B);
  const int32_t max_tiles = (p.max_seqlen + kTile - 1) / kTile;
  if ((st = launch_fmha_plan(d_cu, p.B, p.heads, max_tiles, v, s)) != UB_OK) return st;

  fwd::Params prm{};
  prm.cu = d_cu;
  prm.plan = v;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.lse = lse;
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
  // upper bound on items: H * (B + T/128); one CTA per SM, persistent
  const int64_t max_items = (int64_t)p.heads * (p.B + p.T / kTile + 1);
  const int ctas = p.num_ctas > 0 ? std::min(p.num_ctas, sms) : sms;
  const int grid = (int)std::min<int64_t>(ctas, max_items);
  prof_record(kProfFwd, 0, s);
  fwd::fmha_fwd_kernel<<<grid, fwd::kThreads, fwd::kSmemBytes, s>>>(tmap, prm);
  UB_CHECK_LAUNCH();
  prof_record(kProfFwd, 1, s);
  return UB_OK;
}

}  // namespace ub
