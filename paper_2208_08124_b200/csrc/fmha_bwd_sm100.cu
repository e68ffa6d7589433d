// Varlen FMHA backward on B200 tensor cores (tcgen05 + TMEM + TMA), bf16 in, fp32 accumulate.
//
// Chain rule of Eq. (1) per sequence and head; dropout replayed from R5's keep bits,
// read from the mask ub_dropout_mask materialised (key-major: 2 words per thread and pair) or
// regenerated here by Philox (R4/R5):
//   Delta_i = sum_d dO_id O_id                                   (prologue kernel)
//   S^T = K Q^T, P^T = exp(scale S^T - LSE), dP~^T = V dO^T       (recompute, TMEM)
//   P~ = P M/(1-p), dP = dP~ M/(1-p), dS = P (dP - Delta)          (registers)
//   (with dropout as P' = P/(1-p) from the exp2 argument, P~ = P' M by a packed-pair mask,
//    dS = P' (dP~ M - Delta (1-p)): no per-element multiply by 1/(1-p))
//   dV += P~^T dO, dK += dS^T Q   (TMEM, per key tile)             dQ_i = sum_kt dS K
//   dK *= scale, dQ *= scale (epilogues)
//
// Work item = (sequence, head) along the length-bucketed plan (longest first), dealt to
// the CTAs in snake order (round r: CTA c takes item rG + c, or rG + G-1-c on odd rounds).
// The CTA makes one pass per 128-key tile kt (K_kt, V_kt loaded once) over the sequence's
// query tiles i.  The transposed products put the key on the TMEM lane, so P~^T is the A
// operand of dV straight from TMEM (TS MMA); dS^T goes to smem once and is the A operand of
// both dK (K-major) and dQ (MN-major).
// dQ_i of pass kt leaves TMEM through the epilogue warpgroup: pass 0 stores it (fp32) to a
// scratch row block, middle passes reduce-add into it (TMA), the last pass reads it back,
// adds its own part, scales and writes bf16 dQ -- one sequence never needs a zeroed
// accumulator or a finalize kernel, and the summation order is fixed (deterministic dQ).
//
// CTA = 16 warps (1 per SM), four warpgroups:
//   warps 0-7   two compute warpgroups: thread r of warpgroup x owns key row r and query
//               columns [64x, 64x+64) of S^T / dP^T; per pair two phases:
//                 A: S^T -> P (exp2), P~ (dropout) -> bf16 over its own S^T columns
//                 B: dP^T -> dS = P (dP~ M/(1-p) - Delta) -> bf16 over its own dP^T columns
//                    and into smem (the A operand of dQ)
//   warps 8-11  epilogue warpgroup: dQ_i out of TMEM (two buffers), dK / dV at a pass end
//   warp 12     producer of Q, dO per query tile (3 stages) by TMA; the tile's LSE / Delta
//               vectors by the 32 lanes into smem
//   warp 13     TMEM allocator, then MMA issuer (one thread)
//   warp 14     producer of K, V per pass (double-buffered); warp 15 idle
// Registers: 128 per thread at launch; setmaxnreg moves them to the compute warpgroups
// (168) and the epilogue (112) from the producer / MMA warps (64): 2 x 168 + 112 + 64 = 4 x 128.
// TMEM columns: S^T 0..127 (P~^T bf16 pairs over it: warpgroup x at 64x..64x+31), dP^T
// 128..255 (dS^T bf16 pairs over it: 128+64x..+31), dQ two buffers 256..319 / 320..383,
// dV 384..447, dK 448..511.
// MMA order per pair p (one thread, tcgen05 ops execute in issue order):
//     dV_p += P~_p^T dO_p (TS) | S_{p+1} | dK_p += dS_p^T Q_p (TS) | dQ_p = dS_p K (SS) | dP_{p+1}
// S_{p+1} overwrites the P~_p columns only after dV_p has read them and dP_{p+1} the dS_p
// columns only after dK_p (issue order); a completion commit after dP_{p+1} also covers dQ_p,
// so the compute warps' next dS store to smem never races dQ_p's read.  Phase A of pair
// p+1 (the exp2 work) runs while the tensor core does dK_p, dQ_p, dP_{p+1}; phase B of pair p
// while it does dV_p, S_{p+1}.
#include <cmath>

#include "fmha_common.cuh"

namespace ub {
namespace bwd {

#ifdef UB_TRACE
__device__ uint64_t g_trace[16 * 1024];
__device__ uint64_t g_cta_time[2 * 1024];   // per-CTA start / end globaltimer (trace builds)
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
#ifndef UB_BWD_POLY
#define UB_BWD_POLY 0
#endif
constexpr int kPolyPairs = UB_BWD_POLY;           // exp2 pairs of every 8 on the FMA pipe (phase A); measured 0 / 1 / 2 / 3 -> 106.5 / 107.1 / 107.2 / 108.2 us: MUFU does not bind
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColDV = 384, kColDK = 448;   // dQ: 2 x 64
// TMEM column of the k-th K=16 slice of a TS MMA's A operand held as bf16 pairs over the
// S^T / dP^T block at `base`: queries 0..63 sit at base+0..31 (warpgroup 0), 64..127 at
// base+64..95 (warpgroup 1), so that each warpgroup overwrites only its own fp32 columns
__device__ __forceinline__ uint32_t a_col(uint32_t base, uint32_t k) { return base + (k < 4 ? k * 8 : 64 + (k - 4) * 8); }

struct Smem {
  uint8_t k[2][kTileBytes];
  uint8_t v[2][kTileBytes];
  uint8_t q[kQStages][kTileBytes];
  uint8_t dO[kQStages][kTileBytes];
  uint8_t ds[kPBytes];              // dS^T [key][query], 2 x 64-query SW128 regions
  uint8_t stage[4][4096];           // per epilogue warp: [32 rows][128 B], 128-B swizzle: half of
                                    // dQ (32 fp32 columns), or dK, or dV (64 bf16)
  float lse[kQStages][kTile];       // -LSE * log2(e) of the query tile's rows; -inf past the sequence
  float delta[kQStages][kTile];
  uint64_t kv_full[2], kv_empty[2];
  uint64_t qdo_full[kQStages], qdo_empty[kQStages];
  uint64_t s_full, dp_full, p_full, ds_full, dq_full[2], dq_empty[2], dkv_full, dkv_free;
  uint32_t tmem_base;
  PlanSmem plan;
  ItemTable items;                  // this CTA's items, decoded once
};
constexpr size_t kSmemBytes = sizeof(Smem);
static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");

struct Params {
  const int32_t* cu;
  FmhaPlanView plan;
  const float* lse;     // [H, T]
  const float* delta;   // [H, T]
  float* dq_acc;        // [H * T, 64] fp32 partial dQ of sequences with more than one key tile
  __nv_bfloat16* dqkv;  // [T, 3, H, 64]
  int32_t B, H, max_tiles;
  int64_t T;
  float scale, scale_log2;
  float rp;
  uint32_t thr, k0, k1, off;
  const uint32_t* mk;   // dropout keep bits, key-major [H][MT][4][T] words
  int32_t MT;
  const int32_t* sched; // host LPT schedule (ub_fmha_schedule), NULL = snake deal
};

constexpr uint32_t kIdescS = idesc_bf16_f32(128, 128, 0, 0);     // S^T, dP^T: K-major x K-major
constexpr uint32_t kIdescTS = idesc_bf16_f32(128, 64, 0, 1);     // dV, dK: A in TMEM, B MN-major
constexpr uint32_t kIdescQ = idesc_bf16_f32(128, 64, 1, 1);      // dQ: A MN-major, B MN-major

// keep bits of 16 query columns [q0, q0+16) for this thread's key (lane-cooperative Philox):
// the warp's 32 keys are two 16-key Philox blocks; lane l computes the block (l / 16) word
// set of query column q0 + (l % 16), then every lane gathers bit (l % 16) of the 16 words of
// its block.
__device__ __forceinline__ uint32_t keep16_cols(uint32_t warp_j0, uint32_t t_q0, uint32_t h, const Params& prm,
                                                uint32_t lane) {
  const uint32_t word = keep_bits16(warp_j0 + (lane & 16u), t_q0 + (lane & 15u), h, prm.off, prm.k0, prm.k1, prm.thr);
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t w = __shfl_sync(0xffffffffu, word, (lane & 16u) + k);
    bits |= ((w >> (lane & 15u)) & 1u) << k;
  }
  return bits;
}

// kDrop: 0 no dropout, 1 keep bits regenerated by Philox in the kernel (lane-cooperative),
// 2 keep bits read from the materialised mask (ub_dropout_mask, key-major)
template <int kDrop, bool kBigB>
__global__ void __launch_bounds__(kThreads, 1)
fmha_bwd_kernel(const __grid_constant__ CUtensorMap tmap_qkv, const __grid_constant__ CUtensorMap tmap_do,
                const __grid_constant__ CUtensorMap tmap_dq, const __grid_constant__ CUtensorMap tmap_dqkv,
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

#ifdef UB_TRACE
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_cta_time[2 * blockIdx.x] = t;
  }
#endif
  pdl_launch_dependents();
  if (warp == 12 && lane == 0) {
    tma_prefetch_desc(&tmap_qkv);
    tma_prefetch_desc(&tmap_do);
    tma_prefetch_desc(&tmap_dq);
    tma_prefetch_desc(&tmap_dqkv);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (uint32_t s = 0; s < kQStages; ++s) {
      mbar_init(&sm.qdo_full[s], 2);                // expect_tx arrival + LSE / Delta stores
      mbar_init(&sm.qdo_empty[s], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.dp_full, 1);
    mbar_init(&sm.p_full, 8);
    mbar_init(&sm.ds_full, 8);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.dq_full[b], 1);
      mbar_init(&sm.dq_empty[b], 4);
    }
    mbar_init(&sm.dkv_full, 1);
    mbar_init(&sm.dkv_free, 4);
    fence_mbar_init();
  }
  if (warp == 13) tmem_alloc(&sm.tmem_base, 512);
  // the plan reads only cu_seqlens, which the preceding kernel (bwd_pre) does not write: it is
  // built before the programmatic-dependency wait, overlapping bwd_pre's tail
  if (!kBigB && warp == 12) {
    build_plan_smem(sm.plan, prm.cu, prm.B, prm.H, prm.max_tiles, 0, lane);
    __syncwarp();
    if (!(prm.sched && build_item_table_sched(sm.items, prm.sched, prm.cu, prm.H, 0, (int32_t)blockIdx.x,
                                              (int32_t)gridDim.x, lane)))
      build_item_table(sm.items, sm.plan, prm.cu, prm.B, prm.H, 0, (int32_t)blockIdx.x, (int32_t)gridDim.x, lane);
  }
  pdl_wait();                                            // everything below may read / write global memory
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int32_t H = prm.H;
  const int32_t G = (int32_t)gridDim.x, cta = (int32_t)blockIdx.x;
#define UB_ITEMS(r, it) \
  for (int32_t r = 0; next_item<kBigB>(r, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 0, cta, G, it); ++r)
  constexpr bool kDropout = kDrop != 0;
  // each role re-sizes its registers at its entry, inside its branch (ptxas takes the
  // minimum where paths merge); setmaxnreg is warpgroup-uniform

  if (warp >= 12) {
    regs_dec<64>();
  }
  if (warp == 14) {
    // ------------------------------------------------------------ K / V producer (per pass)
    if (lane == 0) {
      uint32_t pass = 0;
      WorkItem it;
      UB_ITEMS(r, it) {
        for (int32_t kt = 0; kt < it.nt; ++kt, ++pass) {
          const uint32_t kvs = pass & 1;
          TR(20);
          mbar_wait(&sm.kv_empty[kvs], ((pass >> 1) & 1) ^ 1);
          TR(21);
          mbar_expect_tx(&sm.kv_full[kvs], 2 * kTileBytes);
          const int32_t krow = it.c0 + kt * kTile;
          tma_load_2d(sm.k[kvs], &tmap_qkv, &sm.kv_full[kvs], (H + it.h) * kD, krow);
          tma_load_2d(sm.v[kvs], &tmap_qkv, &sm.kv_full[kvs], (2 * H + it.h) * kD, krow);
        }
      }
    }
  } else if (warp == 12) {
    // ------------------------------------------------------------ Q / dO producer (per pair)
    uint32_t qit = 0;
    WorkItem it;
    // with dropout the compute warps work with P' = P / (1-p) = exp2(scale_log2 S - LSE log2 e
    // + log2(1/(1-p))) and Delta' = Delta (1-p): P~ = P' M and dS = P' (dP~ M - Delta')
    const float lse_add = kDropout ? log2f(prm.rp) : 0.f, delta_mul = kDropout ? 1.f / prm.rp : 1.f;
    UB_ITEMS(r, it) {
      for (int32_t kt = 0; kt < it.nt; ++kt) {
        for (int32_t i = 0; i < it.nt; ++i, ++qit) {
          const uint32_t st = qit % kQStages, ph = (qit / kQStages) & 1;
          const int32_t q0 = it.c0 + i * kTile;
          // LSE / Delta loads are issued before the stage wait so their latency hides behind it
          // stored as -LSE * log2(e) (the compute warps' exp2 argument is scale_log2 * S + this),
          // and -inf / 0 for query rows past the sequence end: their P = exp2(-inf) = 0 and dS = 0
          // without any per-element mask in the compute warps
          float lv[4], dv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int32_t k = (int32_t)lane + 32 * u;
            const bool ok = i * kTile + k < it.L;
            const int64_t idx = (int64_t)it.h * prm.T + q0 + k;
            lv[u] = ok ? fmaf(-1.4426950408889634f, __ldg(prm.lse + idx), lse_add) : -INFINITY;
            dv[u] = ok ? __ldg(prm.delta + idx) * delta_mul : 0.f;
          }
          TR(22);
          mbar_wait(&sm.qdo_empty[st], ph ^ 1);
          TR(23);
          if (lane == 0) {
            mbar_expect_tx(&sm.qdo_full[st], 2 * kTileBytes);
            tma_load_2d(sm.q[st], &tmap_qkv, &sm.qdo_full[st], it.h * kD, q0);
            tma_load_2d(sm.dO[st], &tmap_do, &sm.qdo_full[st], it.h * kD, q0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            sm.lse[st][lane + 32 * u] = lv[u];
            sm.delta[st][lane + 32 * u] = dv[u];
          }
          // the lanes' LSE / Delta stores precede the arrival that completes the phase
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.qdo_full[st]);
          TR(24);
        }
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------------ MMA issuer
    // One pipeline over all (item, pass, query tile) pairs of the CTA, also across pass and
    // item boundaries: dV_p | S_{p+1} | dK_p | dQ_p | dP_{p+1} (see the header).
    if (lane == 0) {
      const uint32_t ds_addr = smem_u32(sm.ds);
      // the pair sequence, walked one pair ahead of issue
      struct Pair { int32_t kt, i, nt; uint32_t q, st, kvs, pass; bool first, last; };
      WorkItem it;
      int32_t r = 0, kt = 0, i = 0;
      uint32_t qit = 0, pass = 0;
      bool have = next_item<kBigB>(0, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 0, cta, G, it);
      auto advance = [&](Pair& pr) -> bool {           // the next pair in CTA order, or false
        if (!have) return false;
        pr.kt = kt; pr.i = i; pr.nt = it.nt; pr.q = qit; pr.st = qit % kQStages; pr.kvs = pass & 1; pr.pass = pass;
        pr.first = i == 0; pr.last = i == it.nt - 1;
        ++qit;
        if (++i == it.nt) {
          i = 0; ++pass;
          if (++kt == it.nt) {
            kt = 0;
            have = next_item<kBigB>(++r, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 0, cta, G, it);
          }
        }
        return true;
      };
      auto issue_s_dp = [&](const Pair& pr, bool s_part) {  // S^T = K Q^T or dP~^T = V dO^T
        const uint32_t a = smem_u32(s_part ? sm.k[pr.kvs] : sm.v[pr.kvs]);
        const uint32_t b = smem_u32(s_part ? sm.q[pr.st] : sm.dO[pr.st]);
#pragma unroll
        for (uint32_t k = 0; k < kD / 16; ++k)
          umma_bf16_ss(tmem + (s_part ? kColS : kColDP), sdesc_sw128(a + k * 32, 16, 1024),
                       sdesc_sw128(b + k * 32, 16, 1024), kIdescS, k > 0);
      };
      auto wait_inputs = [&](const Pair& pr) {          // K/V of its pass, Q/dO of its tile
        if (pr.first) mbar_wait(&sm.kv_full[pr.kvs], (pr.pass >> 1) & 1);
        mbar_wait(&sm.qdo_full[pr.st], (pr.q / kQStages) & 1);
      };
      Pair cur, nxt;
      uint32_t p = 0;
      bool has_cur = advance(cur);
      if (has_cur) {
        wait_inputs(cur);
        tc_fence_after();
        issue_s_dp(cur, true);
        umma_commit(&sm.s_full);
        issue_s_dp(cur, false);
        umma_commit(&sm.dp_full);
      }
      while (has_cur) {
        const uint32_t q_addr = smem_u32(sm.q[cur.st]), do_addr = smem_u32(sm.dO[cur.st]);
        const uint32_t k_addr = smem_u32(sm.k[cur.kvs]);
        // dV_p += P~_p^T dO_p (A = P~^T bf16 pairs over the S^T columns)
        mbar_wait(&sm.p_full, p & 1);
        if (cur.first) mbar_wait(&sm.dkv_free, (cur.pass & 1) ^ 1);   // previous pass's dK / dV drained
        TR(12);
        tc_fence_after();
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k)
          umma_bf16_ts(tmem + kColDV, tmem + a_col(kColS, k), sdesc_sw128(do_addr + k * 2048, 8192, 1024), kIdescTS,
                       (cur.first && k == 0) ? 0u : 1u);
        // S_{p+1} (its Q / K inputs)
        const bool has_nxt = advance(nxt);
        if (has_nxt) {
          wait_inputs(nxt);
          tc_fence_after();
          issue_s_dp(nxt, true);
          umma_commit(&sm.s_full);
        }
        TR(10);
        // dK_p += dS_p^T Q_p (A = dS^T bf16 pairs over the dP^T columns), dQ_p = dS_p K
        mbar_wait(&sm.ds_full, p & 1);
        tc_fence_after();
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k)
          umma_bf16_ts(tmem + kColDK, tmem + a_col(kColDP, k), sdesc_sw128(q_addr + k * 2048, 8192, 1024), kIdescTS,
                       (cur.first && k == 0) ? 0u : 1u);
        umma_commit(&sm.qdo_empty[cur.st]);              // Q_p / dO_p / LSE / Delta no longer needed
        const uint32_t b = p & 1;
        mbar_wait(&sm.dq_empty[b], ((p >> 1) & 1) ^ 1);  // the epilogue has drained this dQ buffer
        tc_fence_after();
#pragma unroll
        for (uint32_t k = 0; k < kTile / 16; ++k)
          umma_bf16_ss(tmem + kColDQ + 64 * b, sdesc_sw128(ds_addr + k * 2048, kTile * 128, 1024),
                       sdesc_sw128(k_addr + k * 2048, 8192, 1024), kIdescQ, k > 0);
        umma_commit(&sm.dq_full[b]);
        if (cur.last) {                                  // the pass's K, V and dK, dV are final
          umma_commit(&sm.kv_empty[cur.kvs]);
          umma_commit(&sm.dkv_full);
        }
        TR(19);
        // dP~_{p+1} (overwrites dS_p's columns after dK_p in issue order)
        if (has_nxt) {
          issue_s_dp(nxt, false);
          umma_commit(&sm.dp_full);
        }
        ++p;
        cur = nxt;
        has_cur = has_nxt;
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ compute warpgroups
    regs_inc<168>();
    const uint32_t x = warp >> 2;                           // query-column half
    const uint32_t r = threadIdx.x & 127u;                  // key row (TMEM lane)
    const uint32_t t_row = tmem + (((warp & 3) * 32) << 16);
    const float c = prm.scale_log2;
    const uint64_t c2 = f2pack(c, c);
    const uint32_t ds_addr = smem_u32(sm.ds) + x * (kTile * 128);
    uint32_t p = 0, qit = 0;
    WorkItem it;

    UB_ITEMS(ri, it) {
      // keep bits of key row kt*128 + r for the warpgroup's 64 query columns of query tile i:
      // words c = 2x, 2x+1 at ((h MT + i) 4 + c) T + t (a warp's 32 key rows read 128 contiguous
      // bytes per word), loaded one pair ahead within the item
      auto load_kw = [&](int32_t kt_, int32_t i_) {
        const int32_t key_ = kt_ * kTile + (int32_t)r;
        if (key_ >= it.L) return make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
        const uint32_t* m0 = prm.mk + (((int64_t)it.h * prm.MT + i_) * 4 + 2 * x) * prm.T + it.c0 + key_;
        return make_uint2(__ldg(m0), __ldg(m0 + prm.T));
      };
      uint2 kw_next = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
      if (kDrop == 2) kw_next = load_kw(0, 0);
      for (int32_t kt = 0; kt < it.nt; ++kt) {
        const int32_t key = kt * kTile + (int32_t)r;
        const bool key_ok = key < it.L;
        const bool warp_partial = __any_sync(0xffffffffu, !key_ok);     // a sequence's last key tile
        for (int32_t i = 0; i < it.nt; ++i, ++qit, ++p) {
          const uint32_t st = qit % kQStages;
          // ---- phase A: P = exp2(scale_log2 S - LSE log2 e), P~ = P M / (1-p) -> bf16 over S^T
          const uint2 kw = kw_next;
          if (kDrop == 2) {
            if (i + 1 < it.nt) kw_next = load_kw(kt, i + 1);
            else if (kt + 1 < it.nt) kw_next = load_kw(kt + 1, 0);
          }
          TR(1);
          mbar_wait(&sm.qdo_full[st], (qit / kQStages) & 1);   // LSE / Delta of this query tile
          mbar_wait(&sm.s_full, p & 1);
          TR(2);
          tc_fence_after();
          if (i * kTile + (int32_t)x * 64 >= it.L) {
            // this warpgroup's 64 query columns are all past the sequence end (x = 1 on a last
            // query tile of <= 64 rows): P~ = dS = 0 there, written as zeros over its S^T / dP^T
            // columns once the MMAs have written them (the A operands of dV / dK); the dQ rows
            // of these queries are never stored, so the smem dS half is not needed
            uint32_t z[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) z[e] = 0u;
            tmem_st32(t_row + kColS + x * 64, z);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full);
            mbar_wait(&sm.dp_full, p & 1);
            tc_fence_after();
            tmem_st32(t_row + kColDP + x * 64, z);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.ds_full);
            continue;
          }
          float pf[64];                                     // P (fp32), kept for phase B
          {
            uint32_t sr[2][32];
            tmem_ld32(t_row + kColS + x * 64, sr[0]);
            tmem_ld32(t_row + kColS + x * 64 + 32, sr[1]);
            tmem_ld_wait();
#pragma unroll
            for (int ch = 0; ch < 2; ++ch)
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                // -LSE log2(e) of the two query columns (broadcast smem loads); the producer's
                // -inf for columns past the sequence end makes P = dS = 0 there
                const float2 l2 = *reinterpret_cast<const float2*>(&sm.lse[st][x * 64 + ch * 32 + e]);
                float a, b;
                f2unpack(ffma2(f2pack(__uint_as_float(sr[ch][e]), __uint_as_float(sr[ch][e + 1])), c2,
                               f2pack(l2.x, l2.y)), a, b);
                if (kPolyPairs > 0 && ((e >> 1) & 7) < kPolyPairs) {
                  f2unpack(ex2_poly2(a, b), a, b);          // FMA pipe: MUFU is phase A's bound
                } else {
                  a = ex2f(a);
                  b = ex2f(b);
                }
                pf[ch * 32 + e] = a;
                pf[ch * 32 + e + 1] = b;
              }
          }
          TR(3);
          uint32_t keep[2] = {kw.x, kw.y};                  // bit e: query 64x + 32ch + e of the tile
          if (kDrop == 1) {
            const uint32_t warp_j0 = (uint32_t)(kt * kTile) + (warp & 3) * 32;   // the warp's first key
#pragma unroll
            for (int ch = 0; ch < 2; ++ch) {
              const uint32_t tq = (uint32_t)(it.c0 + i * kTile + (int)x * 64 + ch * 32);
              keep[ch] = keep16_cols(warp_j0, tq, it.h, prm, lane) | (keep16_cols(warp_j0, tq + 16, it.h, prm, lane) << 16);
            }
          }
          {
            uint32_t pp[32];
            // pair jj = 4m + i of chunk ch, walked i-major so that each shifted copy of the keep
            // word keep_mask2 reads is live for 4 consecutive pairs only
#pragma unroll
            for (int ch = 0; ch < 2; ++ch)
#pragma unroll
              for (int i4 = 0; i4 < 4; ++i4)
#pragma unroll
                for (int m4 = 0; m4 < 4; ++m4) {
                  const int jj = 4 * m4 + i4, e = ch * 32 + 2 * jj;
                  pp[e / 2] = pack_bf16(pf[e], pf[e + 1]);    // P' (dropout) or P
                  if (kDropout) pp[e / 2] &= keep_mask2(keep[ch], jj);   // P~ = P' M
                }
            if (warp_partial) {                            // key rows past the sequence end
#pragma unroll
              for (int e = 0; e < 32; ++e) pp[e] = key_ok ? pp[e] : 0u;
            }
            tmem_st32(t_row + kColS + x * 64, pp);        // over this warpgroup's own S^T columns
            tmem_st_wait();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.p_full);
          TR(4);
          // ---- phase B: dS = P (dP~ M / (1-p) - Delta) = P' (dP~ M - Delta') -> bf16 over dP^T and into smem
          mbar_wait(&sm.dp_full, p & 1);
          TR(5);
          tc_fence_after();
          {
            uint32_t dr[2][32];
            tmem_ld32(t_row + kColDP + x * 64, dr[0]);
            tmem_ld32(t_row + kColDP + x * 64 + 32, dr[1]);
            tmem_ld_wait();
            uint32_t pd[32];
#pragma unroll
            for (int ch = 0; ch < 2; ++ch)
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float2 dl = *reinterpret_cast<const float2*>(&sm.delta[st][x * 64 + ch * 32 + e]);
                float dpa = __uint_as_float(dr[ch][e]), dpb = __uint_as_float(dr[ch][e + 1]);
                if (kDropout) {                             // dS = P' (dP~ M - Delta')
                  dpa = ((keep[ch] >> e) & 1u) ? dpa : 0.f;
                  dpb = ((keep[ch] >> (e + 1)) & 1u) ? dpb : 0.f;
                }
                float da, db;
                f2unpack(fmul2(f2pack(pf[ch * 32 + e], pf[ch * 32 + e + 1]), fadd2(f2pack(dpa, dpb), f2pack(-dl.x, -dl.y))),
                         da, db);
                pd[ch * 16 + e / 2] = pack_bf16(da, db);
              }
            if (warp_partial) {
#pragma unroll
              for (int e = 0; e < 32; ++e) pd[e] = key_ok ? pd[e] : 0u;
            }
            tmem_st32(t_row + kColDP + x * 64, pd);       // dS^T: A operand of dK (TS)
#pragma unroll
            for (int g = 0; g < 8; ++g)                    // dS^T [key][query]: A operand of dQ (MN-major)
              st_shared_v4(ds_addr + sw128_off(r, g), pd[4 * g], pd[4 * g + 1], pd[4 * g + 2], pd[4 * g + 3]);
            tmem_st_wait();
          }
          fence_proxy_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.ds_full);
          TR(7);
        }
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ epilogue warpgroup
    regs_dec<112>();
    const uint32_t qd = warp & 3;                           // TMEM lane quadrant
    const uint32_t t_row = tmem + ((qd * 32) << 16);
    uint8_t* stage = sm.stage[qd];
    const uint32_t stage_addr = smem_u32(stage);
    uint32_t e_cnt = 0, pass = 0;
    uint32_t ng = 0;                                        // bulk groups committed by this warp (lane 0)
    uint32_t gq[4] = {0, 0, 0, 0};                          // group count after tile i's last dQ op
    auto stage_free = [&]() {                               // this warp's previous bulk op read it
      if (lane == 0) bulk_wait_group_read0();
      __syncwarp();
    };
    auto stage_bf16 = [&](const uint32_t (&pk)[32]) {
      stage_free();
#pragma unroll
      for (int g = 0; g < 8; ++g)
        st_shared_v4(stage_addr + sw128_off(lane, g), pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
      fence_proxy_async_smem();
      __syncwarp();
    };
    WorkItem it;
    UB_ITEMS(ri, it) {
      for (int32_t kt = 0; kt < it.nt; ++kt, ++pass) {
        const bool first = kt == 0, last = kt == it.nt - 1;
        for (int32_t i = 0; i < it.nt; ++i, ++e_cnt) {
          // dQ_i partial of this pass: query rows 32qd.. of the tile, 64 fp32 columns
          const int32_t wrow0 = i * kTile + (int32_t)qd * 32;          // first query row of this warp
          const bool full = wrow0 + 32 <= it.L;
          const bool row_ok = wrow0 + (int32_t)lane < it.L;
          const int32_t arow0 = (int32_t)((int64_t)it.h * prm.T + it.c0 + wrow0);   // accumulator row
          float* acc = prm.dq_acc + ((int64_t)arow0 + lane) * kD;
          // this pass's op on tile i follows the previous pass's one (async TMA ops of this
          // warp complete in any order: wait for that group); the last pass re-reads the
          // partial, which is warmed into L1 before dQ is even ready
          if (!first && full) {
            if (lane == 0) {
              bulk_wait_group_n((int)(ng - gq[i]));
              if (last) fence_proxy_async_global();
            }
            __syncwarp();
          }
          if (last && !first && row_ok) {
            asm volatile("prefetch.global.L1 [%0];" :: "l"(acc) : "memory");
            asm volatile("prefetch.global.L1 [%0];" :: "l"(acc + 32) : "memory");
          }
          TR(30);
          const uint32_t qb = e_cnt & 1;                    // this pair's dQ buffer
          mbar_wait(&sm.dq_full[qb], (e_cnt >> 1) & 1);
          TR(31);
          tc_fence_after();
          if (i == it.nt - 1) {
            // pass end: dK, dV of the key tile are final (committed with this pair's dQ).  They
            // leave TMEM first, so the next pass's first grads are not held up by dQ's stores.
            mbar_wait(&sm.dkv_full, pass & 1);
            tc_fence_after();
            uint32_t pkk[32], pkv[32];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t a[32];
              tmem_ld32(t_row + kColDK + q * 32, a);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e)
                pkk[q * 16 + e] = pack_bf16(__uint_as_float(a[2 * e]) * prm.scale, __uint_as_float(a[2 * e + 1]) * prm.scale);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t a[32];
              tmem_ld32(t_row + kColDV + q * 32, a);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e) pkv[q * 16 + e] = pack_bf16(__uint_as_float(a[2 * e]), __uint_as_float(a[2 * e + 1]));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.dkv_free);
            const int32_t krow0 = kt * kTile + (int32_t)qd * 32;     // first key row of this warp
            const bool kfull = krow0 + 32 <= it.L;                      // whole warp inside the sequence
#pragma unroll
            for (int m = 0; m < 2; ++m) {                               // 0: dK (x scale), 1: dV
              const uint32_t(&pk)[32] = m ? pkv : pkk;
              if (kfull) {
                stage_bf16(pk);
                if (lane == 0) {
                  tma_store_2d(&tmap_dqkv, stage, ((1 + m) * H + it.h) * kD, it.c0 + krow0);
                  bulk_commit_group();
                  ++ng;
                }
              } else if (krow0 + (int32_t)lane < it.L) {
                uint4* dst = reinterpret_cast<uint4*>(prm.dqkv + ((((int64_t)it.c0 + krow0 + lane) * 3 + 1 + m) * H + it.h) * kD);
#pragma unroll
                for (int g = 0; g < 8; ++g) dst[g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
              }
            }
          }
          uint32_t d[64];
          tmem_ld32(t_row + kColDQ + 64 * qb, *reinterpret_cast<uint32_t(*)[32]>(&d[0]));
          tmem_ld32(t_row + kColDQ + 64 * qb + 32, *reinterpret_cast<uint32_t(*)[32]>(&d[32]));
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.dq_empty[qb]);     // this TMEM dQ buffer is free again
          if (last) {
            // final: (partial +) this pass's part, x scale -> bf16 dQ
            if (!first && row_ok) {
              const float4* src = reinterpret_cast<const float4*>(acc);
#pragma unroll
              for (int g = 0; g < 16; ++g) {
                const float4 v = src[g];
                d[4 * g] = __float_as_uint(__uint_as_float(d[4 * g]) + v.x);
                d[4 * g + 1] = __float_as_uint(__uint_as_float(d[4 * g + 1]) + v.y);
                d[4 * g + 2] = __float_as_uint(__uint_as_float(d[4 * g + 2]) + v.z);
                d[4 * g + 3] = __float_as_uint(__uint_as_float(d[4 * g + 3]) + v.w);
              }
            }
            uint32_t pk[32];
#pragma unroll
            for (int e = 0; e < 32; ++e)
              pk[e] = pack_bf16(__uint_as_float(d[2 * e]) * prm.scale, __uint_as_float(d[2 * e + 1]) * prm.scale);
            if (full) {
              stage_bf16(pk);
              if (lane == 0) {
                tma_store_2d(&tmap_dqkv, stage, it.h * kD, it.c0 + wrow0);
                bulk_commit_group();
                ++ng;
              }
            } else if (row_ok) {
              uint4* dst = reinterpret_cast<uint4*>(prm.dqkv + (((int64_t)(it.c0 + wrow0 + lane) * 3) * H + it.h) * kD);
#pragma unroll
              for (int g = 0; g < 8; ++g) dst[g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
            }
          } else {
            // pass 0 stores the fp32 partial, middle passes add to it
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              if (full) {
                stage_free();
#pragma unroll
                for (int g = 0; g < 8; ++g)
                  st_shared_v4(stage_addr + sw128_off(lane, g), d[half * 32 + 4 * g], d[half * 32 + 4 * g + 1],
                               d[half * 32 + 4 * g + 2], d[half * 32 + 4 * g + 3]);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  if (first) tma_store_2d(&tmap_dq, stage, half * 32, arow0);
                  else tma_reduce_add_2d(&tmap_dq, stage, half * 32, arow0);
                  bulk_commit_group();
                  ++ng;
                }
              } else if (row_ok) {
                float4* dst = reinterpret_cast<float4*>(acc + half * 32);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                  const float4 v = make_float4(__uint_as_float(d[half * 32 + 4 * g]), __uint_as_float(d[half * 32 + 4 * g + 1]),
                                               __uint_as_float(d[half * 32 + 4 * g + 2]), __uint_as_float(d[half * 32 + 4 * g + 3]));
                  if (first) dst[g] = v;
                  else atomicAdd(dst + g, v);
                }
              }
            }
            if (i == 0) gq[0] = ng; else if (i == 1) gq[1] = ng; else if (i == 2) gq[2] = ng; else gq[3] = ng;
          }
          TR(32);
        }
      }
    }
    if (lane == 0) bulk_wait_group0();
  }
#undef UB_ITEMS

  tc_fence_before();
  __syncthreads();
#ifdef UB_TRACE
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_cta_time[2 * blockIdx.x + 1] = t;
  }
#endif
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Prologue: Delta[h, t] = sum_d O[t,h,d] dO[t,h,d]  (8 threads per (t, h) row, 16-B loads,
// kPreRows rows per thread group so that several loads per thread are in flight).
constexpr int kPreRows = 4;
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ out,
                                                      const __nv_bfloat16* __restrict__ dout, float* __restrict__ delta,
                                                      int64_t T, int32_t H) {
  pdl_launch_dependents();
  pdl_wait();                                      // O comes from the forward
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int part = (int)(gtid & 7);
  const int64_t g = gtid >> 3;                     // row group: rows base + g + k * n_groups
  const int64_t rows = T * H, n_groups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  // grid-stride over blocks of kPreRows * n_groups rows: a one-wave grid (host) keeps every SM
  // streaming to the end instead of a partial last wave
  for (int64_t base = 0; base < rows; base += kPreRows * n_groups) {
    uint4 a[kPreRows], b[kPreRows];
#pragma unroll
    for (int k = 0; k < kPreRows; ++k) {
      const int64_t row = base + g + k * n_groups;
      a[k] = b[k] = make_uint4(0, 0, 0, 0);
      if (row < rows) {
        a[k] = __ldcs(reinterpret_cast<const uint4*>(out + row * kD) + part);
        b[k] = __ldcs(reinterpret_cast<const uint4*>(dout + row * kD) + part);
      }
    }
#pragma unroll
    for (int k = 0; k < kPreRows; ++k) {
      const int64_t row = base + g + k * n_groups;
      const uint32_t av[4] = {a[k].x, a[k].y, a[k].z, a[k].w}, bv[4] = {b[k].x, b[k].y, b[k].z, b[k].w};
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s = fmaf(__uint_as_float(av[e] << 16), __uint_as_float(bv[e] << 16), s);
        s = fmaf(__uint_as_float(av[e] & 0xFFFF0000u), __uint_as_float(bv[e] & 0xFFFF0000u), s);
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (part == 0 && row < rows) {
        const int64_t t = row / H;
        const int32_t h = (int32_t)(row - t * H);
        delta[(int64_t)h * T + t] = s;
      }
    }
  }
}

}  // namespace bwd

#ifdef UB_TRACE
extern "C" __attribute__((visibility("default"))) int ub_debug_bwd_cta_times(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, bwd::g_cta_time, bytes < sizeof(bwd::g_cta_time) ? bytes : sizeof(bwd::g_cta_time));
}
extern "C" __attribute__((visibility("default"))) int ub_debug_bwd_trace(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, bwd::g_trace, bytes < sizeof(bwd::g_trace) ? bytes : sizeof(bwd::g_trace));
}
#endif

size_t fmha_bwd_sm100_ws_bytes(const ub_fmha_params& p) {
  return align_up((size_t)p.T * p.heads * 4, 256) + align_up((size_t)p.T * p.heads * 64 * 4, 256);
}

ub_status fmha_bwd_sm100(const ub_fmha_params& p, const void* qkv, const void* out, const float* lse, const void* dout,
                         const int32_t* d_cu, void* dqkv, void* ws, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t max_items = (int64_t)p.heads * p.B;
  const int ctas = p.num_ctas > 0 ? std::min(p.num_ctas, sms) : sms;
  const int grid = (int)std::min<int64_t>(ctas, max_items);
  const bool drop = p.p_dropout > 0.f;
  // plan and item table in shared memory, else the global plan decoded per item
  const bool big = !item_table_fits(p.B, max_items, grid);
  // dropout bits: read from the caller's materialised mask (one pass per step shared by both
  // directions), else regenerated by Philox inside the kernel (cheaper than materialising it
  // for a single call)
  const int mode = !drop ? 0 : (p.dropout_mask != nullptr ? 2 : 1);
  using KernT = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, bwd::Params);
  static const KernT table[6] = {bwd::fmha_bwd_kernel<0, false>, bwd::fmha_bwd_kernel<0, true>,
                                 bwd::fmha_bwd_kernel<1, false>, bwd::fmha_bwd_kernel<1, true>,
                                 bwd::fmha_bwd_kernel<2, false>, bwd::fmha_bwd_kernel<2, true>};
  const KernT kern = table[mode * 2 + (big ? 1 : 0)];
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
  if (big && (st = launch_fmha_plan(d_cu, p.B, p.heads, max_tiles, 0, v, s)) != UB_OK) return st;
  const void* mask = p.dropout_mask;
  const int64_t rows = p.T * p.heads;
#ifndef UB_PRE_WAVES
#define UB_PRE_WAVES 1
#endif
  // Delta's grid: UB_PRE_WAVES full waves of resident CTAs (grid-stride), 0 = one CTA per 256 x kPreRows rows
  static const int pre_per_sm = [] {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bwd::bwd_pre_kernel, 256, 0);
    return nb > 0 ? nb : 1;
  }();
  const int64_t pre_need = (rows * 8 + 256 * bwd::kPreRows - 1) / (256 * bwd::kPreRows);
  const int64_t pre_grid =
      UB_PRE_WAVES > 0 ? std::min<int64_t>(pre_need, (int64_t)sms * pre_per_sm * UB_PRE_WAVES) : pre_need;
  launch_pdl(bwd::bwd_pre_kernel, dim3((unsigned)pre_grid), dim3(256), 0, s,
             static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), delta, p.T, p.heads);
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
  prm.max_tiles = max_tiles;
  prm.T = p.T;
  prm.scale = p.scale;
  prm.scale_log2 = p.scale * 1.4426950408889634f;
  prm.thr = drop ? (uint32_t)floor((double)p.p_dropout * 256.0) : 0u;   // R5: 8-bit decisions
  prm.rp = 1.f / (1.f - (float)prm.thr / 256.f);
  prm.k0 = (uint32_t)(p.seed & 0xFFFFFFFFull);
  prm.k1 = (uint32_t)(p.seed >> 32);
  prm.off = (uint32_t)(p.offset & 0xFFFFFFFFull);
  prm.mk = reinterpret_cast<const uint32_t*>(static_cast<const char*>(mask) + (mask ? dropout_mask_bytes(p) / 2 : 0));
  prm.MT = mask_tiles(p);
  prm.sched = big ? nullptr : p.schedule;
  prof_record(kProfBwd, 0, s);
  launch_pdl(kern, dim3(grid), dim3(bwd::kThreads), bwd::kSmemBytes, s, tq, tdo, tdq, tdkv, prm);
  UB_CHECK_LAUNCH();
  prof_record(kProfBwd, 1, s);
  return UB_OK;
}

}  // namespace ub
