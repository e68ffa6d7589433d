// Varlen FMHA forward on B200 tensor cores (tcgen05 + TMEM + TMA), bf16 in, fp32 accumulate.
//
// Eq. (1) of the paper per sequence and head on cu_seqlens-packed tokens (P:302,
// P:313).  One persistent launch walks the length-bucketed plan (fmha_plan.cu);
// a work item is (sequence, head, pair of 128-row query tiles) so the two query tiles
// share every K/V tile load.
//
// CTA = 12 warps (1 per SM), warp-specialised (warps 10-11 idle: setmaxnreg needs whole warpgroups):
//   warps 0-3   softmax warpgroup 0: query tile A (thread r owns row r)
//   warps 4-7   softmax warpgroup 1: query tile B
//   warp 8      TMA producer: Q_A, Q_B (double-buffered across items), K_j / V_j through a
//               3-stage ring, straight from the packed qkv [T, 3*H*64] matrix (128-B swizzle)
//   warp 9      TMEM allocator, then MMA issuer (one thread):
//                 S_x(j) = Q_x K_j^T   M128 N128 K64, smem x smem       -> TMEM S_x
//                 O_x   += P_x(j) V_j  M128 N64 K128, P from TMEM (TS) -> TMEM O_x
//               issue order S_A(j+1), PV_A(j), S_B(j+1), PV_B(j) over one stream of key tiles
//               that runs across items (at an item's last tile the look-ahead S is the next
//               item's first), so the softmax never waits for an item boundary
//   warps 10-11 idle (the third warpgroup is whole so that setmaxnreg can move registers
//               from it to the softmax warpgroups: 208 vs 88 per thread)
// Each softmax warpgroup defers its epilogue (O / l -> bf16 -> TMA store, LSE) into the first key tile of its
// next item, after that tile's P has been handed to the MMA.
// TMEM (512 columns): per warpgroup x: S at 256x (128 cols fp32), P at 256x+128 (64 cols,
// bf16 pairs), O at 256x+192 (64 cols fp32).
// Softmax per tile: tcgen05.ld the S row, mask keys past the sequence end, 3-input max
// tree, exp2 (MUFU, a fraction on the FMA pipe by polynomial), packed f32x2 sums,
// P -> TMEM by tcgen05.st.  O stays in TMEM; it is rescaled (ld/scale/st) only when the
// running max grows by more than 2^8 (lazy rescale: P is bounded by 256, exact in the end
// because l uses the same reference max).
// Boxes that run past a sequence end read the next sequence's rows: those keys are
// masked to -inf and those query rows are never stored.
#include <cmath>
#include <cstdlib>

#include "fmha_common.cuh"

namespace ub {
namespace fwd {

#ifdef UB_TRACE
// Debug timeline (trace builds only): CTA 0, lane 0 of every warp records (event, clock64).
__device__ uint64_t g_trace[10 * 1024];
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
constexpr int kStages = 3;
constexpr uint32_t kTileBytes = kTile * kD * 2;   // 16 KB
constexpr int kThreads = 384;                     // 3 warpgroups (setmaxnreg is per warpgroup)
constexpr float kRescaleThreshold = 8.0f;         // log2 units

struct Smem {
  uint8_t q[2][2][kTileBytes];                    // [item slot][warpgroup]
  uint8_t k[kStages][kTileBytes];
  uint8_t v[kStages][kTileBytes];
  uint8_t ostage[8][32 * 128];                    // per softmax warp: 32 output rows, SW128
  uint8_t zeros[32 * 128];                        // a zero 32-row block: padded rows by TMA store
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[kStages], v_full[kStages], kv_empty[kStages];
  uint64_t s_full[2], s_free[2], p_full[2], o_done[2];   // per warpgroup
  uint32_t tmem_base;
  PlanSmem plan;
  ItemTable items;                                // this CTA's items, decoded once
};
constexpr size_t kSmemBytes = sizeof(Smem);
static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");

struct Params {
  const int32_t* cu;
  FmhaPlanView plan;
  __nv_bfloat16* out;
  float* lse;
  __nv_bfloat16* padded;   // fused a9: O also written to [B, S_pad, H, 64], zeros past L; NULL = off
  int32_t S_pad;
  int32_t B, H, max_tiles;
  int64_t T;
  float scale, scale_log2;
  float rp;           // 1 / (1 - p_eff)
  uint32_t thr, k0, k1, off;
  const int32_t* sched;   // host LPT schedule (ub_fmha_schedule), NULL = snake deal
};

constexpr uint32_t kIdescS = idesc_bf16_f32(128, 128, 0, 0);   // Q (K-major) x K (K-major)
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, 64, 0, 1);   // P (TMEM) x V (MN-major)
__host__ __device__ constexpr uint32_t col_s(int x) { return 256u * x; }
__host__ __device__ constexpr uint32_t col_p(int x) { return 256u * x + 128u; }
__host__ __device__ constexpr uint32_t col_o(int x) { return 256u * x + 192u; }

// kPoly: number of column pairs out of every 8 whose exp2 runs on the FMA pipe (ex2_poly2).
// kPack: 0 = bf16 packing by cvt (XU pipe), 1 = integer rounding + byte permute.
// kDropout: compile the Philox mask in (p > 0) or out (p == 0: no RNG code at all, so the
// compiler cannot hoist it into the exp loop).  kBigB: batch larger than the smem plan cache.
// kDrop: 0 no dropout, 1 keep bits by Philox in the softmax loop, 2 keep bits read from the
// mask ub_dropout_mask materialised (query-major, 16 bytes per thread and key tile)
template <int kPoly, int kPack, int kDrop, bool kBigB>
__global__ void __launch_bounds__(kThreads, 1)
fmha_fwd_kernel(const __grid_constant__ CUtensorMap tmap_qkv, const __grid_constant__ CUtensorMap tmap_out,
                const __grid_constant__ CUtensorMap tmap_pad, const Params prm,
                const uint32_t* __restrict__ mq,   // dropout keep bits, query-major [H][MT][4][T] words
                int32_t MT) {
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
  constexpr bool kDropout = kDrop != 0;

#ifdef UB_TRACE
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_cta_time[2 * blockIdx.x] = t;
  }
#endif
  pdl_launch_dependents();
  if (warp == 10) {                                      // idle warps: the zero block for padded rows
    for (uint32_t i = lane; i < sizeof(sm.zeros) / 16; i += 32) st_shared_v4(smem_u32(sm.zeros) + 16 * i, 0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmap_qkv);
    tma_prefetch_desc(&tmap_out);
    if (prm.padded) tma_prefetch_desc(&tmap_pad);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], 1);
      mbar_init(&sm.q_empty[s], 1);
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], 4);
      mbar_init(&sm.p_full[s], 4);
      mbar_init(&sm.o_done[s], 1);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(&sm.tmem_base, 512);
  pdl_wait();                                            // everything below may read / write global memory
  if (!kBigB && warp == 8) {
    build_plan_smem(sm.plan, prm.cu, prm.B, prm.H, prm.max_tiles, 2, lane);
    __syncwarp();
    if (!(prm.sched && build_item_table_sched(sm.items, prm.sched, prm.cu, prm.H, 2, (int32_t)blockIdx.x,
                                              (int32_t)gridDim.x, lane)))
      build_item_table(sm.items, sm.plan, prm.cu, prm.B, prm.H, 2, (int32_t)blockIdx.x, (int32_t)gridDim.x, lane);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int32_t H = prm.H;
  // registers: 168 per thread at launch; the producer / MMA warpgroup (warps 8-11, of which
  // 10-11 idle) gives them to the softmax warpgroups: the pool is the launch allocation: 8 x 40 = 4 x 80 extra per thread
  // (each role re-sizes at its entry, inside its branch: ptxas takes the minimum where paths merge)

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    regs_dec<88>();
    if (lane == 0) {
      uint32_t items = 0, kv_it = 0;
      WorkItem it;
      for (int32_t r = 0; next_item<kBigB, !kDropout>(r, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 2, (int32_t)blockIdx.x, (int32_t)gridDim.x, it); ++r, ++items) {
        const uint32_t slot = items & 1;
        TR(20);
        mbar_wait(&sm.q_empty[slot], ((items >> 1) & 1) ^ 1);
        TR(21);
        mbar_expect_tx(&sm.q_full[slot], kTileBytes * it.ntile);
        for (int x = 0; x < it.ntile; ++x)
          tma_load_2d(sm.q[slot][x], &tmap_qkv, &sm.q_full[slot], it.h * kD, it.c0 + (it.tile + x) * kTile);
        for (int32_t j = 0; j < it.nt; ++j, ++kv_it) {
          const uint32_t st = kv_it % kStages, ph = (kv_it / kStages) & 1;
          mbar_wait(&sm.kv_empty[st], ph ^ 1);
          TR(22);
          mbar_expect_tx(&sm.k_full[st], kTileBytes);
          tma_load_2d(sm.k[st], &tmap_qkv, &sm.k_full[st], (H + it.h) * kD, it.c0 + j * kTile);
          mbar_expect_tx(&sm.v_full[st], kTileBytes);
          tma_load_2d(sm.v[st], &tmap_qkv, &sm.v_full[st], (2 * H + it.h) * kD, it.c0 + j * kTile);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    regs_dec<88>();
    if (lane == 0) {
      // One stream of key tiles across items: the S of the next tile -- the next item's first
      // tile at an item's last -- is issued before the PV of the current one, so a softmax
      // warpgroup finds its next S ready, also across item boundaries.
      uint32_t s_cnt[2] = {0, 0}, p_cnt[2] = {0, 0};
      auto issue_s = [&](int x, uint32_t qslot, uint32_t kst) {
        mbar_wait(&sm.s_free[x], (s_cnt[x] & 1) ^ 1);
        TR(10 + x);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sm.q[qslot][x]), k_addr = smem_u32(sm.k[kst]);
#pragma unroll
        for (uint32_t k = 0; k < kD / 16; ++k)
          umma_bf16_ss(tmem + col_s(x), sdesc_sw128(q_addr + k * 32, 16, 1024), sdesc_sw128(k_addr + k * 32, 16, 1024),
                       kIdescS, k > 0);
        umma_commit(&sm.s_full[x]);
        ++s_cnt[x];
      };
      WorkItem it, nit;
      int32_t r = 0;                                      // this CTA's item round (snake order)
      bool have = next_item<kBigB, !kDropout>(0, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 2, (int32_t)blockIdx.x, (int32_t)gridDim.x, it);
      uint32_t items = 0, kv_it = 0;
      if (have) {
        mbar_wait(&sm.q_full[0], 0);
        mbar_wait(&sm.k_full[0], 0);
        tc_fence_after();
#pragma unroll
        for (int x = 0; x < 2; ++x)
          if (x < it.ntile) issue_s(x, 0, 0);
      }
      while (have) {
        const uint32_t slot = items & 1;
        const int nx = it.ntile;
        TR(16);
        bool have_next_item = false;
        for (int32_t j = 0; j < it.nt; ++j) {
          const uint32_t cur = kv_it + j, st = cur % kStages, ph = (cur / kStages) & 1;
          const uint32_t nst = (cur + 1) % kStages;
          // target of the look-ahead S: (this item, j+1) or (next item, 0)
          int nxt_tiles = 0;
          uint32_t nslot = slot;
          if (j + 1 < it.nt) {
            nxt_tiles = nx;
          } else {
            have_next_item = next_item<kBigB, !kDropout>(r + 1, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 2, (int32_t)blockIdx.x, (int32_t)gridDim.x, nit);
            if (have_next_item) {
              nxt_tiles = nit.ntile;
              nslot = slot ^ 1u;
              mbar_wait(&sm.q_full[nslot], ((items + 1) >> 1) & 1);
            }
          }
          TR(14);
          if (nxt_tiles > 0) {
            mbar_wait(&sm.k_full[nst], ((cur + 1) / kStages) & 1);
            tc_fence_after();
          }
          mbar_wait(&sm.v_full[st], ph);
          TR(15);
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (x < nxt_tiles) issue_s(x, nslot, nst);
            if (x < nx) {
              mbar_wait(&sm.p_full[x], p_cnt[x] & 1);   // (at j = 0 also: the previous O was read)
              TR(12 + x);
              tc_fence_after();
              const uint32_t v_addr = smem_u32(sm.v[st]);
#pragma unroll
              for (uint32_t k = 0; k < kTile / 16; ++k)
                umma_bf16_ts(tmem + col_o(x), tmem + col_p(x) + k * 8, sdesc_sw128(v_addr + k * 2048, 8192, 1024),
                             kIdescPV, (j > 0 || k > 0) ? 1u : 0u);
              umma_commit(&sm.o_done[x]);
              ++p_cnt[x];
            }
          }
          umma_commit(&sm.kv_empty[st]);
        }
        umma_commit(&sm.q_empty[slot]);
        kv_it += it.nt;
        ++items;
        ++r;
        have = have_next_item;
        it = nit;
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax warpgroups
    regs_inc<208>();
    const int x = (int)(warp >> 2);                       // warpgroup / query tile of the pair
    const uint32_t r = threadIdx.x - 128u * x;            // row inside the tile
    const uint32_t t_row = tmem + (((warp & 3) * 32) << 16);
    const float c = prm.scale_log2;
    const uint64_t c2 = f2pack(c, c);
    uint32_t s_cnt = 0, pv_cnt = 0;
    // The epilogue of an item is deferred into the first key tile of the warpgroup's next
    // item: its O is read out of TMEM once that tile's P is ready (the next PV overwrites O),
    // and scaled / stored after P is handed to the MMA -- the softmax never idles on the
    // last PV of an item.
    bool have_prev = false;
    float l_prev = 0.f, m_prev = 0.f;
    WorkItem pit{};
    // previous item's O / l -> bf16 pairs (read 32 columns at a time: registers)
    auto read_o = [&](uint32_t (&opk)[32]) {
      mbar_wait(&sm.o_done[x], pv_cnt & 1);             // the previous item's last PV
      ++pv_cnt;
      tc_fence_after();
      const float inv = prm.rp / l_prev;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t o[32];
        tmem_ld32(t_row + col_o(x) + q * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) opk[q * 16 + e] = pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
      }
    };
    auto epilogue = [&](const uint32_t (&pk)[32]) {
      TR(8);
      const int32_t row = (pit.tile + x) * kTile + (int32_t)r;
      const uint32_t t_glob = (uint32_t)(pit.c0 + row);
      const int32_t wrow0 = (pit.tile + x) * kTile + (int32_t)(warp & 3) * 32;   // first row of this warp
      if (wrow0 + 32 <= pit.L) {
        // whole warp inside the sequence: stage 32 rows (128-B swizzle) and TMA-store them
        uint8_t* stage = sm.ostage[warp];
        const uint32_t sa = smem_u32(stage);
        if (lane == 0) bulk_wait_group_read0();          // previous store of this warp has read it
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 8; ++g)
          st_shared_v4(sa + sw128_off(lane, g), pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmap_out, stage, pit.h * kD, pit.c0 + wrow0);
          if (prm.padded) tma_store_2d(&tmap_pad, stage, pit.h * kD, pit.b * prm.S_pad + wrow0);
          bulk_commit_group();
        }
      } else if (row < pit.L) {
        uint4* op = reinterpret_cast<uint4*>(prm.out + ((int64_t)t_glob * H + pit.h) * kD);
#pragma unroll
        for (int g = 0; g < 8; ++g) op[g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        if (prm.padded) {
          uint4* pp = reinterpret_cast<uint4*>(prm.padded + (((int64_t)pit.b * prm.S_pad + row) * H + pit.h) * kD);
#pragma unroll
          for (int g = 0; g < 8; ++g) pp[g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        }
      }
      if (row < pit.L) prm.lse[(int64_t)pit.h * prm.T + t_glob] = m_prev * prm.scale + logf(l_prev);
      if (prm.padded && pit.tile + x == pit.nt - 1) {
        // the sequence's last tile: zero its head's padded rows [L, S) -- lanes up to the
        // tile end, then whole 32-row blocks from the zero tile, dealt over the 4 warps
        if (row >= pit.L && row < prm.S_pad) {
          uint4* pp = reinterpret_cast<uint4*>(prm.padded + (((int64_t)pit.b * prm.S_pad + row) * H + pit.h) * kD);
#pragma unroll
          for (int g = 0; g < 8; ++g) pp[g] = make_uint4(0, 0, 0, 0);
        }
        if (lane == 0) {
          for (int32_t blk = pit.nt * (kTile / 32) + (int32_t)(warp & 3); blk * 32 < prm.S_pad; blk += 4)
            tma_store_2d(&tmap_pad, sm.zeros, pit.h * kD, pit.b * prm.S_pad + blk * 32);
          bulk_commit_group();
        }
      }
      TR(9);
    };
    WorkItem it;
    for (int32_t ri = 0; next_item<kBigB, !kDropout>(ri, sm.items, sm.plan, prm.plan, prm.cu, prm.B, H, 2, (int32_t)blockIdx.x, (int32_t)gridDim.x, it); ++ri) {
      if (x >= it.ntile) continue;
      const int32_t row = (it.tile + x) * kTile + (int32_t)r;
      const uint32_t t_glob = (uint32_t)(it.c0 + row);
      float m_run = -INFINITY, l = 0.f;
      // keep bits of key tile j's 128 keys: word w (keys 32w..32w+31 of the tile) at
      // ((h MT + j) 4 + w) T + t, a warp's 32 rows read 128 contiguous bytes per word; loaded one
      // key tile ahead (an L2 load takes longer than the S wait it used to hide behind)
      auto load_kw = [&](int32_t j, uint32_t (&w4)[4]) {
        const uint32_t* m0 = mq + ((int64_t)it.h * MT + j) * 4 * prm.T + t_glob;
#pragma unroll
        for (int w = 0; w < 4; ++w) w4[w] = row < it.L ? __ldg(m0 + (int64_t)w * prm.T) : 0xFFFFFFFFu;
      };
      uint32_t kw_next[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
      if constexpr (kDrop == 2) load_kw(0, kw_next);
      for (int32_t j = 0; j < it.nt; ++j) {
        uint32_t kw[4] = {kw_next[0], kw_next[1], kw_next[2], kw_next[3]};
        if constexpr (kDrop == 2) {
          if (j + 1 < it.nt) load_kw(j + 1, kw_next);
        }
        TR(1);
        mbar_wait(&sm.s_full[x], s_cnt & 1);
        TR(2);
        tc_fence_after();
        float s[kTile];
        {
          uint32_t raw[4][32];
#pragma unroll
          for (int q = 0; q < 4; ++q) tmem_ld32(t_row + col_s(x) + q * 32, raw[q]);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int e = 0; e < 32; ++e) s[q * 32 + e] = __uint_as_float(raw[q][e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[x]);
        ++s_cnt;
        TR(3);

        const int32_t kvalid = it.L - j * kTile;
        if (kvalid < kTile) {
#pragma unroll
          for (int e = 0; e < kTile; ++e)
            if (e >= kvalid) s[e] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float a = fmax3(s[g * 16 + 0], s[g * 16 + 1], s[g * 16 + 2]);
#pragma unroll
          for (int e = 3; e < 15; e += 2) a = fmax3(a, s[g * 16 + e], s[g * 16 + e + 1]);
          mx[g] = fmaxf(a, s[g * 16 + 15]);
        }
        const float mt = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmaxf(fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        const float m_new = fmaxf(m_run, mt);
        const bool need = (m_new - m_run) * c > kRescaleThreshold;   // m_run = -inf -> true
        const float m_ref = need ? m_new : m_run;
        const float alpha = need ? ex2f((m_run - m_new) * c) : 1.f;
        const bool rescale_warp = __any_sync(0xffffffffu, need) && j > 0;
        const float negm = -m_ref * c;
        const uint64_t neg2 = f2pack(negm, negm);
        uint64_t acc2[4] = {0, 0, 0, 0};
        uint32_t pk[kTile / 2];
        uint32_t bits16 = 0;
        (void)bits16;
#pragma unroll
        for (int g = 0; g < kTile / 8; ++g) {          // 8 keys at a time: exp2, sum, dropout, pack
          float e8[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e2 = g * 4 + u;
            float a, b;
            f2unpack(ffma2(f2pack(s[2 * e2], s[2 * e2 + 1]), c2, neg2), a, b);
            if (kPoly > 0 && (e2 & 7) < kPoly) {
              f2unpack(ex2_poly2(a, b), a, b);
            } else {
              a = ex2f(a);
              b = ex2f(b);
            }
            acc2[u] = fadd2(acc2[u], f2pack(a, b));
            e8[2 * u] = a;
            e8[2 * u + 1] = b;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            pk[g * 4 + u] = kPack ? pack_bf16_int(e8[2 * u], e8[2 * u + 1]) : pack_bf16(e8[2 * u], e8[2 * u + 1]);
          if constexpr (kDropout) {                       // P~ = P M on the packed pairs (l sums P)
            if constexpr (kDrop == 2) {
#pragma unroll
              for (int u = 0; u < 4; ++u) pk[g * 4 + u] &= keep_mask2(kw[g >> 2], (g & 3) * 4 + u);
            } else {
              if ((g & 1) == 0) bits16 = keep_bits16(j * kTile + g * 8, t_glob, it.h, prm.off, prm.k0, prm.k1, prm.thr);
#pragma unroll
              for (int u = 0; u < 4; ++u) pk[g * 4 + u] &= keep_mask2(bits16, (g & 1) * 4 + u);
            }
          }
        }
        float rs;
        {
          float a0, a1;
          f2unpack(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])), a0, a1);
          rs = a0 + a1;
        }

        TR(4);
        const bool defer = j == 0 && have_prev;
        uint32_t opk[32];
        if (defer) {
          read_o(opk);                                     // previous item's O, before PV(0) overwrites it
        } else if (j > 0) {
          // PV_x(j-1) must have finished reading P and accumulating into O
          mbar_wait(&sm.o_done[x], pv_cnt & 1);
          ++pv_cnt;
          tc_fence_after();
        }
        if (rescale_warp) {                              // rare: running max grew by > 2^8
          const uint64_t al2 = f2pack(alpha, alpha);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t o[32];
            tmem_ld32(t_row + col_o(x) + q * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              float a, b;
              f2unpack(fmul2(f2pack(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), al2), a, b);
              o[e] = __float_as_uint(a);
              o[e + 1] = __float_as_uint(b);
            }
            tmem_st32(t_row + col_o(x) + q * 32, o);
          }
        }
        TR(5);
        l = fmaf(l, alpha, rs);
        m_run = m_ref;
        tmem_st32(t_row + col_p(x), *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
        tmem_st32(t_row + col_p(x) + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[x]);
        TR(6);
        if (defer) epilogue(opk);                        // overlaps this item's first PV
      }
      have_prev = true;
      l_prev = l;
      m_prev = m_run;
      pit = it;
    }
    if (have_prev) {
      TR(7);
      uint32_t opk[32];
      read_o(opk);
      epilogue(opk);
    }
  } else {
    regs_dec<88>();                // warps 10-11: otherwise idle
    if (warp == 10 && prm.padded) {
      // fused pad of EMPTY sequences (L = 0 has no work item, so no epilogue zeroes its
      // padded block): CTA c zero-fills [b, 0:S, h, :] of b = c, c + G, ... with TMA stores
      // of the zero block, one (head, 32-row block) per lane -- the ub_pad result
      const int32_t nblk = prm.S_pad / 32;
      bool issued = false;
      for (int32_t b = (int32_t)blockIdx.x; b < prm.B; b += (int32_t)gridDim.x) {
        if (prm.cu[b + 1] - prm.cu[b] != 0) continue;
        for (int32_t w = (int32_t)lane; w < H * nblk; w += 32) {
          const int32_t h = w / nblk, blk = w - h * nblk;
          tma_store_2d(&tmap_pad, sm.zeros, h * kD, b * prm.S_pad + blk * 32);
          issued = true;
        }
      }
      if (issued) {
        bulk_commit_group();
        bulk_wait_group0();
      }
    }
  }

  if (warp < 8 && lane == 0) bulk_wait_group0();        // output stores complete before exit
  tc_fence_before();
  __syncthreads();
#ifdef UB_TRACE
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_cta_time[2 * blockIdx.x + 1] = t;
  }
#endif
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace fwd

#ifdef UB_TRACE
extern "C" __attribute__((visibility("default"))) int ub_debug_fwd_cta_times(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, fwd::g_cta_time, bytes < sizeof(fwd::g_cta_time) ? bytes : sizeof(fwd::g_cta_time));
}
extern "C" __attribute__((visibility("default"))) int ub_debug_fwd_trace(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, fwd::g_trace, bytes < sizeof(fwd::g_trace) ? bytes : sizeof(fwd::g_trace));
}
#endif

static int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = std::getenv(name);
  int v = e ? std::atoi(e) : dflt;
  return (v < lo || v > hi) ? dflt : v;
}

using FwdKern = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, fwd::Params, const uint32_t*, int32_t);
template <int P>
static FwdKern pick_fwd(int mode, bool big) {
  static const FwdKern t[6] = {fwd::fmha_fwd_kernel<P, 0, 0, false>, fwd::fmha_fwd_kernel<P, 0, 0, true>,
                               fwd::fmha_fwd_kernel<P, 0, 1, false>, fwd::fmha_fwd_kernel<P, 0, 1, true>,
                               fwd::fmha_fwd_kernel<P, 0, 2, false>, fwd::fmha_fwd_kernel<P, 0, 2, true>};
  return t[mode * 2 + (big ? 1 : 0)];
}

ub_status fmha_fwd_sm100(const ub_fmha_params& p, const void* qkv, const int32_t* d_cu, void* out, float* lse,
                         void* padded, int32_t S_pad, void* ws, cudaStream_t s) {
  // fraction (x/8) of exp2 pairs on the FMA pipe, 0 or 2.  Measured on config 2 without
  // dropout: 0 -> 64.5 us, 2 -> 58.4, 3 -> 62.2, 4 -> 68.4 (issue-bound beyond 2/8); with
  // dropout the Philox integer work already loads the FMA pipe: 0 -> 92.3 us, 2 -> 99.5.
  // UB_FWD_POLY = 0 / 2 forces one for both.
  static const int poly_env = env_int("UB_FWD_POLY", -1, -1, 4);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t max_items = (int64_t)p.heads * (p.B + p.T / (2 * kTile) + 1);   // >= sum_b ceil(nt_b / 2) * H
  const int ctas = p.num_ctas > 0 ? std::min(p.num_ctas, sms) : sms;
  const int grid = (int)std::min<int64_t>(ctas, max_items);
  // plan and item table in shared memory, else the global plan decoded per item
  const bool drop = p.p_dropout > 0.f, big = !item_table_fits(p.B, max_items, grid);
  const int poly = poly_env < 0 ? (drop ? 0 : 2) : (poly_env >= 2 ? 2 : 0);
  // dropout bits: read from the caller's materialised mask, else regenerated by Philox in
  // the softmax loop (cheaper than materialising them for a single call)
  const int mode = !drop ? 0 : (p.dropout_mask != nullptr ? 2 : 1);
  const FwdKern kern = poly == 2 ? pick_fwd<2>(mode, big) : pick_fwd<0>(mode, big);
  {
    const ub_status sa = smem_attr_once(reinterpret_cast<const void*>(kern), (int)fwd::kSmemBytes);
    if (sa != UB_OK) return sa;
  }
  CUtensorMap tmap;
  ub_status st = make_tmap_bf16(&tmap, qkv, (uint64_t)3 * p.heads * fwd::kD, (uint64_t)p.T,
                                (uint64_t)3 * p.heads * fwd::kD * 2);
  if (st != UB_OK) return st;
  CUtensorMap tmap_out;
  if ((st = make_tmap_bf16(&tmap_out, out, (uint64_t)p.heads * fwd::kD, (uint64_t)p.T, (uint64_t)p.heads * fwd::kD * 2,
                           64, 32, 128)) != UB_OK)
    return st;
  CUtensorMap tmap_pad = tmap_out;                       // (unused when padded is NULL)
  if (padded && (st = make_tmap_bf16(&tmap_pad, padded, (uint64_t)p.heads * fwd::kD, (uint64_t)p.B * S_pad,
                                     (uint64_t)p.heads * fwd::kD * 2, 64, 32, 128)) != UB_OK)
    return st;
  FmhaPlanView v = fmha_plan_view(ws, p.B);
  const int32_t max_tiles = (p.max_seqlen + kTile - 1) / kTile;
  if (big && (st = launch_fmha_plan(d_cu, p.B, p.heads, max_tiles, 2, v, s)) != UB_OK) return st;
  const void* mask = p.dropout_mask;

  fwd::Params prm{};
  prm.padded = static_cast<__nv_bfloat16*>(padded);
  prm.S_pad = S_pad;
  prm.cu = d_cu;
  prm.plan = v;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.lse = lse;
  prm.B = p.B;
  prm.H = p.heads;
  prm.max_tiles = max_tiles;
  prm.T = p.T;
  prm.scale = p.scale;
  prm.scale_log2 = p.scale * 1.4426950408889634f;
  prm.thr = p.p_dropout > 0.f ? (uint32_t)floor((double)p.p_dropout * 256.0) : 0u;   // R5: 8-bit decisions
  prm.rp = 1.f / (1.f - (float)prm.thr / 256.f);                                       // exact keep probability
  prm.k0 = (uint32_t)(p.seed & 0xFFFFFFFFull);
  prm.k1 = (uint32_t)(p.seed >> 32);
  prm.off = (uint32_t)(p.offset & 0xFFFFFFFFull);
  prm.sched = big ? nullptr : p.schedule;

  prof_record(kProfFwd, 0, s);
  launch_pdl(kern, dim3(grid), dim3(fwd::kThreads), fwd::kSmemBytes, s, tmap, tmap_out, tmap_pad, prm,
             static_cast<const uint32_t*>(mask), mask_tiles(p));
  UB_CHECK_LAUNCH();
  prof_record(kProfFwd, 1, s);
  return UB_OK;
}

}  // namespace ub
