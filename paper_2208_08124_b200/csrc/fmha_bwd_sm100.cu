// Varlen FMHA backward on B200 tensor cores (tcgen05 + TMEM + TMA), bf16 in, fp32 accumulate.
//
// Chain rule of Eq. (1) per sequence and head; dropout replayed from the Philox
// key (R4/R5):
//   Delta_i = sum_d dO_id O_id                                   (prologue kernel)
//   S^T = K Q^T, P^T = exp(scale S^T - LSE), dP~^T = V dO^T       (recompute, TMEM)
//   P~ = P M/(1-p), dP = dP~ M/(1-p), dS = P (dP - Delta)          (registers)
//   dV += P~^T dO, dK += dS^T Q   (TMEM, per key tile)             dQ += dS K (TMA reduce-add)
//   dK *= scale (epilogue), dQ *= scale (finalize kernel)
//
// Work item = (sequence, head, 128-key tile) along the length-bucketed plan; the CTA walks
// the sequence's query tiles.  The transposed products put the key on the TMEM lane, so
// P~^T and dS^T are already the A operands of dV and dK and never leave TMEM (TS MMA); only
// dS goes to smem, for dQ.
//
// CTA = 16 warps (1 per SM), four warpgroups:
//   warps 0-7   two compute warpgroups: thread r of warpgroup x owns key row r and query
//               columns [64x, 64x+64) of S^T / dP^T
//   warps 8-11  epilogue warpgroup: dQ_i out of TMEM into the fp32 accumulator, and dK / dV
//               of the finished item, so the compute warps never leave the exp/dS loop
//   warp 12     producer of Q, dO per query tile (2 stages) by TMA; the tile's LSE / Delta
//               vectors by the 32 lanes into smem
//   warp 13     TMEM allocator, then MMA issuer (one thread)
//   warp 14     producer of K, V per item (double-buffered); warp 15 idle
// Registers: 128 per thread at launch; setmaxnreg moves them to the compute warpgroups
// (168) from the others (88): per SMSP 2 x 168 + 2 x 88 = 512 = 4 x 128.
// TMEM columns: S^T 0..127, dP^T 128..255, P~^T 256..319 (bf16 pairs), dS^T 320..383
// (bf16 pairs; dQ_i = dS K is written over it after dK_i has read it -- tcgen05.mma ops of
// one thread execute in issue order), dV 384..447, dK 448..511.
// The MMA issues S_{i+1}, dP_{i+1} as soon as the compute warps have loaded S_i, dP_i, so
// the exp/dS phase of tile i overlaps the tensor work of tile i+1; the compute warps write
// P~_{i+1} / dS_{i+1} once the epilogue has read dQ_i out (which implies grads_i are done).
// dQ_i leaves through per-warp smem staging (128-B swizzle) and cp.reduce.async.bulk.tensor
// add into an fp32 [H*T, 64] accumulator (two TMA ops per warp instead of 8192 atomics);
// dK / dV of whole warps leave by TMA store from the same staging.
#include <cmath>

#include "fmha_common.cuh"

namespace ub {
namespace bwd {

#ifdef UB_TRACE
__device__ uint64_t g_trace[16 * 1024];
#define TR(ev)                                                                                          \
  do {                                                                                                  \
    if (blockIdx.x == 0 && lane == 0 && tr_n < 1024)                                                    \
      g_trace[warp * 1024 + tr_n++] = ((uint64_t)(ev) << 48) | ((uint64_t)clock64() & 0xFFFFFFFFFFFFull); \
  } while (0)
#else
#define TR(ev) do {} while (0)
#endif

constexpr int kD = 64;
constexpr uint32_t kTileBytes = kTile * kD * 2;   // 16 KB
constexpr uint32_t kPBytes = kTile * kTile * 2;   // 32 KB
constexpr int kThreads = 512;
constexpr uint32_t kQStages = 3;                  // Q / dO / LSE / Delta pipeline depth
constexpr uint32_t kColS = 0, kColDP = 128, kColP = 256, kColDS = 320, kColDQ = 320, kColDV = 384, kColDK = 448;

struct Smem {
  uint8_t k[2][kTileBytes];
  uint8_t v[2][kTileBytes];
  uint8_t q[kQStages][kTileBytes];
  uint8_t dO[kQStages][kTileBytes];
  uint8_t ds[kPBytes];              // dS^T [key][query], 2 x 64-query SW128 regions
  uint8_t stage[4][4096];           // per epilogue warp: [32 rows][128 B], 128-B swizzle: half of
                                    // dQ (32 fp32 columns), or dK, or dV (64 bf16)
  float lse[kQStages][kTile];       // LSE of the query tile's rows (natural log)
  float delta[kQStages][kTile];
  uint64_t kv_full[2], kv_empty[2];
  uint64_t qdo_full[kQStages], qdo_empty[kQStages];
  uint64_t s_full, s_free, pds_full, dq_full, dq_empty, dkv_full, dkv_free;
  uint32_t tmem_base;
  PlanSmem plan;
};
constexpr size_t kSmemBytes = sizeof(Smem);

struct Params {
  const int32_t* cu;
  FmhaPlanView plan;
  const float* lse;     // [H, T]
  const float* delta;   // [H, T]
  __nv_bfloat16* dqkv;  // [T, 3, H, 64]
  int32_t B, H, max_tiles;
  int64_t T;
  float scale, scale_log2;
  float rp;
  uint32_t thr, k0, k1, off;
};

constexpr uint32_t kIdescS = idesc_bf16_f32(128, 128, 0, 0);     // S^T, dP^T: K-major x K-major
constexpr uint32_t kIdescTS = idesc_bf16_f32(128, 64, 0, 1);     // dV, dK: A in TMEM, B MN-major
constexpr uint32_t kIdescQ = idesc_bf16_f32(128, 64, 1, 1);      // dQ: A MN-major, B MN-major

// keep bits of 8 query columns [q0, q0+8) for this thread's key (lane-cooperative Philox):
// lane l computes the mask word of key group (l/8) at column q0 + (l%8); lanes then gather
// bit (l%8) of their group's 8 words.
__device__ __forceinline__ uint32_t keep8_cols(uint32_t key_grp_j0, uint32_t t_q0, uint32_t h, const Params& prm,
                                               uint32_t lane) {
  const uint32_t word = keep_bits8(key_grp_j0, t_q0 + (lane & 7), h, prm.off, prm.k0, prm.k1, prm.thr);
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t w = __shfl_sync(0xffffffffu, word, (lane & ~7u) + k);
    bits |= ((w >> (lane & 7)) & 1u) << k;
  }
  return bits;
}

template <bool kDropout, bool kBigB>
__global__ void __launch_bounds__(kThreads, 1)
fmha_bwd_kernel(const __grid_constant__ CUtensorMap tmap_qkv, const __grid_constant__ CUtensorMap tmap_do,
                const __grid_constant__ CUtensorMap tmap_dq, const __grid_constant__ CUtensorMap tmap_dkv,
                const Params prm) {
  // Taken straight from the __shared__ array so that every access compiles to LDS/STS (a
  // generic pointer would turn them into long-latency generic loads); the dynamic smem
  // window starts 1024-B aligned (checked), as the 128-B swizzle atoms require.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();
  uint32_t tr_n = 0;
  (void)tr_n;

  if (warp == 12 && lane == 0) {
    tma_prefetch_desc(&tmap_qkv);
    tma_prefetch_desc(&tmap_do);
    tma_prefetch_desc(&tmap_dq);
    tma_prefetch_desc(&tmap_dkv);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (uint32_t s = 0; s < kQStages; ++s) {
      mbar_init(&sm.qdo_full[s], 1);
      mbar_init(&sm.qdo_empty[s], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_free, 8);
    mbar_init(&sm.pds_full, 8);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_empty, 4);
    mbar_init(&sm.dkv_full, 1);
    mbar_init(&sm.dkv_free, 4);
    fence_mbar_init();
  }
  if (!kBigB && warp == 12) build_plan_smem(sm.plan, prm.cu, prm.B, prm.H, prm.max_tiles, 1, lane);
  if (warp == 13) tmem_alloc(&sm.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int32_t H = prm.H;
  // each role re-sizes its registers at its entry, inside its branch (ptxas takes the
  // minimum where paths merge); setmaxnreg is warpgroup-uniform

  if (warp >= 12) {
    regs_dec<88>();
  }
  if (warp == 14) {
    // ------------------------------------------------------------ K / V producer (per item)
    if (lane == 0) {
      uint32_t items = 0;
      WorkItem it;
      for (int32_t w = blockIdx.x; decode_item_smem<kBigB>(w, sm.plan, prm.plan, prm.cu, prm.B, H, 1, it);
           w += gridDim.x, ++items) {
        const uint32_t kvs = items & 1;
        TR(20);
        mbar_wait(&sm.kv_empty[kvs], ((items >> 1) & 1) ^ 1);
        TR(21);
        mbar_expect_tx(&sm.kv_full[kvs], 2 * kTileBytes);
        const int32_t krow = it.c0 + it.tile * kTile;
        tma_load_2d(sm.k[kvs], &tmap_qkv, &sm.kv_full[kvs], (H + it.h) * kD, krow);
        tma_load_2d(sm.v[kvs], &tmap_qkv, &sm.kv_full[kvs], (2 * H + it.h) * kD, krow);
      }
    }
  } else if (warp == 12) {
    // ------------------------------------------------------------ Q / dO producer (per pair)
    uint32_t qit = 0;
    WorkItem it;
    for (int32_t w = blockIdx.x; decode_item_smem<kBigB>(w, sm.plan, prm.plan, prm.cu, prm.B, H, 1, it);
         w += gridDim.x) {
      for (int32_t i = 0; i < it.nt; ++i, ++qit) {
        const uint32_t st = qit % kQStages, ph = (qit / kQStages) & 1;
        const int32_t q0 = it.c0 + i * kTile;
        // LSE / Delta loads are issued before the stage wait so their latency hides behind it
        float lv[4], dv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t k = (int32_t)lane + 32 * u;
          const bool ok = i * kTile + k < it.L;
          const int64_t idx = (int64_t)it.h * prm.T + q0 + k;
          lv[u] = ok ? __ldg(prm.lse + idx) : 0.f;
          dv[u] = ok ? __ldg(prm.delta + idx) : 0.f;
        }
        TR(22);
        mbar_wait(&sm.qdo_empty[st], ph ^ 1);
        TR(23);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          sm.lse[st][lane + 32 * u] = lv[u];
          sm.delta[st][lane + 32 * u] = dv[u];
        }
        __syncwarp();
        if (lane == 0) {
          mbar_expect_tx(&sm.qdo_full[st], 2 * kTileBytes);
          tma_load_2d(sm.q[st], &tmap_qkv, &sm.qdo_full[st], it.h * kD, q0);
          tma_load_2d(sm.dO[st], &tmap_do, &sm.qdo_full[st], it.h * kD, q0);
          if (i + 1 < it.nt) {                       // warm L2 for the next stage's tile
            tma_prefetch_2d(&tmap_qkv, it.h * kD, q0 + kTile);
            tma_prefetch_2d(&tmap_do, it.h * kD, q0 + kTile);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------------ MMA issuer
    // One pipeline over all (item, query tile) pairs: S_p, dP_p are issued before the grads of
    // pair p-1, also across item boundaries, so the compute warps never wait for the previous
    // item's last grads before they can start on the next item.
    if (lane == 0) {
      uint32_t items = 0, qit = 0, s_cnt = 0, g_cnt = 0;
      const uint32_t ds_addr = smem_u32(sm.ds);
      bool pend = false, p_first = false, p_last = false;    // the pair whose grads are pending
      uint32_t p_st = 0, p_kaddr = 0, p_kvs = 0, p_item = 0;
      auto grads = [&]() {
        mbar_wait(&sm.pds_full, g_cnt & 1);
        if (p_first) mbar_wait(&sm.dkv_free, (p_item & 1) ^ 1);
        TR(12);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sm.q[p_st]), do_addr = smem_u32(sm.dO[p_st]);
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k)        // K = query rows, 16 per MMA
          umma_bf16_ts(tmem + kColDV, tmem + kColP + k * 8, sdesc_sw128(do_addr + k * 2048, 8192, 1024), kIdescTS,
                       (p_first && k == 0) ? 0u : 1u);
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k)
          umma_bf16_ts(tmem + kColDK, tmem + kColDS + k * 8, sdesc_sw128(q_addr + k * 2048, 8192, 1024), kIdescTS,
                       (p_first && k == 0) ? 0u : 1u);
        umma_commit(&sm.qdo_empty[p_st]);              // Q_i / dO_i no longer needed
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k)        // K = key rows, 16 per MMA
          umma_bf16_ss(tmem + kColDQ, sdesc_sw128(ds_addr + k * 2048, kTile * 128, 1024),
                       sdesc_sw128(p_kaddr + k * 2048, 8192, 1024), kIdescQ, k > 0);
        umma_commit(&sm.dq_full);                      // grads_i done; dQ_i in TMEM
        ++g_cnt;
        if (p_last) {                                  // the item's K, V and dK, dV are final
          umma_commit(&sm.kv_empty[p_kvs]);
          umma_commit(&sm.dkv_full);
        }
      };
      WorkItem it;
      for (int32_t w = blockIdx.x; decode_item_smem<kBigB>(w, sm.plan, prm.plan, prm.cu, prm.B, H, 1, it); w += gridDim.x, ++items) {
        const uint32_t kvs = items & 1;
        const uint32_t k_addr = smem_u32(sm.k[kvs]), v_addr = smem_u32(sm.v[kvs]);
        TR(16);
        mbar_wait(&sm.kv_full[kvs], (items >> 1) & 1);
        TR(17);
        for (int32_t i = 0; i < it.nt; ++i, ++qit) {
          const uint32_t st = qit % kQStages;
          mbar_wait(&sm.qdo_full[st], (qit / kQStages) & 1);
          TR(18);
          mbar_wait(&sm.s_free, (s_cnt & 1) ^ 1);
          TR(10);
          tc_fence_after();
          const uint32_t q_addr = smem_u32(sm.q[st]), do_addr = smem_u32(sm.dO[st]);
#pragma unroll
          for (uint32_t k = 0; k < kD / 16; ++k) {
            umma_bf16_ss(tmem + kColS, sdesc_sw128(k_addr + k * 32, 16, 1024), sdesc_sw128(q_addr + k * 32, 16, 1024),
                         kIdescS, k > 0);
            umma_bf16_ss(tmem + kColDP, sdesc_sw128(v_addr + k * 32, 16, 1024),
                         sdesc_sw128(do_addr + k * 32, 16, 1024), kIdescS, k > 0);
          }
          umma_commit(&sm.s_full);
          ++s_cnt;
          if (pend) grads();
          pend = true;
          p_st = st; p_kaddr = k_addr; p_kvs = kvs; p_item = items;
          p_first = i == 0;
          p_last = i == it.nt - 1;
        }
      }
      if (pend) grads();
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ compute warpgroups
    regs_inc<168>();
    const uint32_t x = warp >> 2;                           // query-column half
    const uint32_t r = threadIdx.x & 127u;                  // key row (TMEM lane)
    const uint32_t t_row = tmem + (((warp & 3) * 32) << 16);
    const float c = prm.scale_log2;
    const uint64_t c2 = f2pack(c, c);
    const uint64_t nl2e2 = f2pack(-1.4426950408889634f, -1.4426950408889634f);
    const uint32_t ds_addr = smem_u32(sm.ds) + x * (kTile * 128);
    uint32_t s_cnt = 0, g_cnt = 0, qit = 0, items = 0;
    WorkItem it;

    for (int32_t w = blockIdx.x; decode_item_smem<kBigB>(w, sm.plan, prm.plan, prm.cu, prm.B, H, 1, it); w += gridDim.x, ++items) {
      const int32_t key = it.tile * kTile + (int32_t)r;
      const bool key_ok = key < it.L;
      const uint32_t grp_j0 = (uint32_t)(it.tile * kTile) + (warp & 3) * 32 + (lane & ~7u);
      for (int32_t i = 0; i < it.nt; ++i, ++qit) {
        const uint32_t st = qit % kQStages;
        const int32_t qvalid = it.L - i * kTile;          // query rows of this tile inside the sequence
        TR(1);
        mbar_wait(&sm.qdo_full[st], (qit / kQStages) & 1);   // LSE / Delta of this query tile
        mbar_wait(&sm.s_full, s_cnt & 1);
        TR(2);
        tc_fence_after();
        uint32_t sr[2][32], dr[2][32];
        tmem_ld32(t_row + kColS + x * 64, sr[0]);
        tmem_ld32(t_row + kColS + x * 64 + 32, sr[1]);
        tmem_ld32(t_row + kColDP + x * 64, dr[0]);
        tmem_ld32(t_row + kColDP + x * 64 + 32, dr[1]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free);
        ++s_cnt;
        TR(3);

        uint32_t pp[32], pd[32];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          const int q0 = (int)x * 64 + ch * 32;
          uint32_t keep = 0xFFFFFFFFu;
          if (kDropout) {
            keep = 0;
            const uint32_t tq = (uint32_t)(it.c0 + i * kTile + q0);
#pragma unroll
            for (int b8 = 0; b8 < 4; ++b8) keep |= keep8_cols(grp_j0, tq + 8 * b8, it.h, prm, lane) << (8 * b8);
          }
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 l2 = *reinterpret_cast<const float2*>(&sm.lse[st][q0 + e]);
            const float2 dl = *reinterpret_cast<const float2*>(&sm.delta[st][q0 + e]);
            float pa, pb;
            f2unpack(ffma2(f2pack(__uint_as_float(sr[ch][e]), __uint_as_float(sr[ch][e + 1])), c2,
                           fmul2(f2pack(l2.x, l2.y), nl2e2)), pa, pb);
            pa = (key_ok && q0 + e < qvalid) ? ex2f(pa) : 0.f;
            pb = (key_ok && q0 + e + 1 < qvalid) ? ex2f(pb) : 0.f;
            float dpa = __uint_as_float(dr[ch][e]), dpb = __uint_as_float(dr[ch][e + 1]);
            float qa = pa, qb = pb;
            if (kDropout) {
              const bool ka = (keep >> e) & 1u, kb = (keep >> (e + 1)) & 1u;
              qa = ka ? pa * prm.rp : 0.f;
              qb = kb ? pb * prm.rp : 0.f;
              dpa = ka ? dpa * prm.rp : 0.f;
              dpb = kb ? dpb * prm.rp : 0.f;
            }
            float da, db;
            f2unpack(fmul2(f2pack(pa, pb), fadd2(f2pack(dpa, dpb), f2pack(-dl.x, -dl.y))), da, db);
            pp[ch * 16 + e / 2] = pack_bf16(qa, qb);
            pd[ch * 16 + e / 2] = pack_bf16(da, db);
          }
        }
        // dQ_{i-1} read out of TMEM by the epilogue => grads_{i-1} done: P~^T / dS^T TMEM
        // and the dS smem tile are free
        TR(4);
        mbar_wait(&sm.dq_empty, (g_cnt & 1) ^ 1);
        TR(5);
        tc_fence_after();
        tmem_st32(t_row + kColP + x * 32, pp);
        tmem_st32(t_row + kColDS + x * 32, pd);
#pragma unroll
        for (int g = 0; g < 8; ++g)
          st_shared_v4(ds_addr + sw128_off(r, g), pd[4 * g], pd[4 * g + 1], pd[4 * g + 2], pd[4 * g + 3]);
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pds_full);
        ++g_cnt;
        TR(7);
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ epilogue warpgroup
    regs_dec<88>();
    const uint32_t qd = warp & 3;                           // TMEM lane quadrant
    const uint32_t t_row = tmem + ((qd * 32) << 16);
    uint8_t* stage = sm.stage[qd];
    const uint32_t stage_addr = smem_u32(stage);
    uint32_t e_cnt = 0, items = 0;
    auto stage_free = [&]() {                               // this warp's previous bulk op read it
      if (lane == 0) bulk_wait_group_read0();
      __syncwarp();
    };
    WorkItem it;
    for (int32_t w = blockIdx.x; decode_item_smem<kBigB>(w, sm.plan, prm.plan, prm.cu, prm.B, H, 1, it); w += gridDim.x, ++items) {
      for (int32_t i = 0; i < it.nt; ++i, ++e_cnt) {
        // dQ_i (query rows 32qd.. of the tile, 64 fp32 columns) -> accumulator (TMA reduce-add)
        uint32_t d0[32], d1[32];
        TR(30);
        mbar_wait(&sm.dq_full, e_cnt & 1);
        TR(31);
        tc_fence_after();
        tmem_ld32(t_row + kColDQ, d0);
        tmem_ld32(t_row + kColDQ + 32, d1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.dq_empty);
        const int32_t row0 = (int32_t)((int64_t)it.h * prm.T + it.c0 + i * kTile) + (int32_t)qd * 32;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint32_t* d = half ? d1 : d0;
          stage_free();
#pragma unroll
          for (int g = 0; g < 8; ++g)
            st_shared_v4(stage_addr + sw128_off(lane, g), d[4 * g], d[4 * g + 1], d[4 * g + 2], d[4 * g + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_reduce_add_2d(&tmap_dq, stage, half * 32, row0);
            bulk_commit_group();
          }
        }
        TR(32);
      }
      // dK, dV of this key tile (key rows 32qd.., 64 columns each), one after the other
      TR(33);
      mbar_wait(&sm.dkv_full, items & 1);
      TR(34);
      tc_fence_after();
      const int32_t wrow0 = it.tile * kTile + (int32_t)qd * 32;      // first key row of this warp
      const bool full = wrow0 + 32 <= it.L;                           // whole warp inside the sequence
      const int64_t t = (int64_t)it.c0 + wrow0 + lane;
#pragma unroll 1
      for (int m = 0; m < 2; ++m) {                                   // 0: dK (x scale), 1: dV
        uint32_t a[32], b[32], pk[32];
        tmem_ld32(t_row + (m ? kColDV : kColDK), a);
        tmem_ld32(t_row + (m ? kColDV : kColDK) + 32, b);
        tmem_ld_wait();
        if (m == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.dkv_free);
        }
        const float sc = m ? 1.f : prm.scale;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          pk[e] = pack_bf16(__uint_as_float(a[2 * e]) * sc, __uint_as_float(a[2 * e + 1]) * sc);
          pk[16 + e] = pack_bf16(__uint_as_float(b[2 * e]) * sc, __uint_as_float(b[2 * e + 1]) * sc);
        }
        if (full) {
          stage_free();
#pragma unroll
          for (int g = 0; g < 8; ++g)
            st_shared_v4(stage_addr + sw128_off(lane, g), pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmap_dkv, stage, ((1 + m) * H + it.h) * kD, it.c0 + wrow0);
            bulk_commit_group();
          }
        } else if (wrow0 + (int32_t)lane < it.L) {
          uint4* dst = reinterpret_cast<uint4*>(prm.dqkv + ((t * 3 + 1 + m) * H + it.h) * kD);
#pragma unroll
          for (int g = 0; g < 8; ++g) dst[g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        }
      }
    }
    if (lane == 0) bulk_wait_group0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Prologue: Delta[h, t] = sum_d O[t,h,d] dO[t,h,d]  (8 threads per (t, h) row, 16-B loads)
// and dq_acc = 0 (grid-stride float4 stores).
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ out,
                                                      const __nv_bfloat16* __restrict__ dout, float* __restrict__ delta,
                                                      float4* __restrict__ dq_acc, int64_t T, int32_t H, int64_t n_acc4) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gtid >> 3;                   // (t, h) row
  const int part = (int)(gtid & 7);
  if (row < T * H) {
    const uint4 a = reinterpret_cast<const uint4*>(out + row * kD)[part];
    const uint4 b = reinterpret_cast<const uint4*>(dout + row * kD)[part];
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s = fmaf(__uint_as_float(av[e] << 16), __uint_as_float(bv[e] << 16), s);
      s = fmaf(__uint_as_float(av[e] & 0xFFFF0000u), __uint_as_float(bv[e] & 0xFFFF0000u), s);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (part == 0) {
      const int64_t t = row / H;
      const int32_t h = (int32_t)(row - t * H);
      delta[(int64_t)h * T + t] = s;
    }
  }
  for (int64_t k = gtid; k < n_acc4; k += (int64_t)gridDim.x * blockDim.x) dq_acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Finalize: dqkv[t, 0, h, :] = bf16(scale * dq_acc[h * T + t, :]).
__global__ void __launch_bounds__(256) bwd_dq_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                                                     int64_t T, int32_t H, float scale) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (h, t, 8-wide group)
  if (idx >= T * H * (kD / 8)) return;
  const int64_t row = idx >> 3;                  // h * T + t
  const int32_t g = (int32_t)(idx & 7);
  const int32_t h = (int32_t)(row / T);
  const int64_t t = row - (int64_t)h * T;
  const float4* a = reinterpret_cast<const float4*>(dq_acc + row * kD + g * 8);
  const float4 x = a[0], y = a[1];
  uint4 v = make_uint4(pack_bf16(x.x * scale, x.y * scale), pack_bf16(x.z * scale, x.w * scale),
                       pack_bf16(y.x * scale, y.y * scale), pack_bf16(y.z * scale, y.w * scale));
  *reinterpret_cast<uint4*>(dqkv + ((t * 3 + 0) * H + h) * kD + g * 8) = v;
}

}  // namespace bwd

#ifdef UB_TRACE
extern "C" __attribute__((visibility("default"))) int ub_debug_bwd_trace(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, bwd::g_trace, bytes < sizeof(bwd::g_trace) ? bytes : sizeof(bwd::g_trace));
}
#endif

size_t fmha_bwd_sm100_ws_bytes(const ub_fmha_params& p) {
  return align_up((size_t)p.T * p.heads * 4, 256) + align_up((size_t)p.T * p.heads * 64 * 4, 256);
}

ub_status fmha_bwd_sm100(const ub_fmha_params& p, const void* qkv, const void* out, const float* lse, const void* dout,
                         const int32_t* d_cu, void* dqkv, void* ws, cudaStream_t s) {
  const bool drop = p.p_dropout > 0.f;
  const bool big = p.B > kPlanCap;
  auto kern = drop ? (big ? bwd::fmha_bwd_kernel<true, true> : bwd::fmha_bwd_kernel<true, false>)
                   : (big ? bwd::fmha_bwd_kernel<false, true> : bwd::fmha_bwd_kernel<false, false>);
  {
    const ub_status sa = smem_attr_once(reinterpret_cast<const void*>(kern), (int)bwd::kSmemBytes);
    if (sa != UB_OK) return sa;
  }
  char* base = static_cast<char*>(ws);
  FmhaPlanView v = fmha_plan_view(base, p.B);
  char* extra = base + align_up(fmha_plan_bytes(p.B), 256);
  float* delta = reinterpret_cast<float*>(extra);
  float* dq_acc = reinterpret_cast<float*>(extra + align_up((size_t)p.T * p.heads * 4, 256));
  CUtensorMap tq, tdo, tdq, tdkv;
  ub_status st = make_tmap_bf16(&tq, qkv, (uint64_t)3 * p.heads * bwd::kD, (uint64_t)p.T,
                                (uint64_t)3 * p.heads * bwd::kD * 2);
  if (st != UB_OK) return st;
  if ((st = make_tmap_bf16(&tdo, dout, (uint64_t)p.heads * bwd::kD, (uint64_t)p.T, (uint64_t)p.heads * bwd::kD * 2)) !=
      UB_OK)
    return st;
  if ((st = make_tmap_f32(&tdq, dq_acc, bwd::kD, (uint64_t)p.T * p.heads, bwd::kD * 4, 32, 32)) != UB_OK) return st;
  if ((st = make_tmap_bf16(&tdkv, dqkv, (uint64_t)3 * p.heads * bwd::kD, (uint64_t)p.T,
                           (uint64_t)3 * p.heads * bwd::kD * 2, 64, 32, 128)) != UB_OK)
    return st;
  const int32_t max_tiles = (p.max_seqlen + kTile - 1) / kTile;
  if (p.B > kPlanCap && (st = launch_fmha_plan(d_cu, p.B, p.heads, max_tiles, 1, v, s)) != UB_OK) return st;
  const int64_t rows = p.T * p.heads;
  const int64_t n_acc4 = rows * bwd::kD / 4;
  bwd::bwd_pre_kernel<<<(unsigned)((rows * 8 + 255) / 256), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), delta,
      reinterpret_cast<float4*>(dq_acc), p.T, p.heads, n_acc4);
  UB_CHECK_LAUNCH();

  bwd::Params prm{};
  prm.cu = d_cu;
  prm.plan = v;
  prm.lse = lse;
  prm.delta = delta;
  prm.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  prm.B = p.B;
  prm.H = p.heads;
  prm.max_tiles = max_tiles;
  prm.T = p.T;
  prm.scale = p.scale;
  prm.scale_log2 = p.scale * 1.4426950408889634f;
  prm.rp = 1.f / (1.f - p.p_dropout);
  prm.thr = drop ? (uint32_t)floor((double)p.p_dropout * 65536.0) : 0u;
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
  kern<<<grid, bwd::kThreads, bwd::kSmemBytes, s>>>(tq, tdo, tdq, tdkv, prm);
  UB_CHECK_LAUNCH();
  prof_record(kProfBwd, 1, s);
  const int64_t n = rows * (bwd::kD / 8);
  bwd::bwd_dq_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dq_acc, static_cast<__nv_bfloat16*>(dqkv), p.T,
                                                                  p.heads, p.scale);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

}  // namespace ub
