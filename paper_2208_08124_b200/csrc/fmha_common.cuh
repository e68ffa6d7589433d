// Shared pieces of the tcgen05 FMHA kernels: work-item decode, TMA descriptor creation,
// dropout mask word.
#pragma once
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "sm100.cuh"
#include "ub_internal.h"

namespace ub {

struct WorkItem {
  int32_t b, h, tile, c0, L, nt, ntile;   // tile = first tile of the item, ntile = tiles in it
  int32_t pc0;                            // tile-padded row base of the sequence
};

// Map a flat work index onto (sequence, head, tile group) along the bucketed plan.
__device__ __forceinline__ bool decode_item(int32_t w, const FmhaPlanView& v, const int32_t* __restrict__ cu,
                                            int32_t B, int32_t H, int32_t tiles_per_item, WorkItem& it) {
  const int32_t total = v.item_prefix[B];
  if (w >= total) return false;
  int32_t lo = 0, hi = B;                       // largest k with prefix[k] <= w
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (v.item_prefix[mid] <= w) lo = mid; else hi = mid - 1;
  }
  it.b = v.seq_order[lo];
  const int32_t local = w - v.item_prefix[lo];
  it.c0 = cu[it.b];
  it.L = cu[it.b + 1] - it.c0;
  it.nt = (it.L + kTile - 1) / kTile;
  it.pc0 = v.pad_c0[it.b];
  if (tiles_per_item == 0) {
    it.h = local;
    it.tile = 0;
    it.ntile = it.nt;
    return true;
  }
  const int32_t ngroups = (it.nt + tiles_per_item - 1) / tiles_per_item;
  it.h = local / ngroups;
  it.tile = (local - it.h * ngroups) * tiles_per_item;
  it.ntile = min(tiles_per_item, it.nt - it.tile);
  return true;
}

// The plan built by each CTA in shared memory (B <= kPlanCap): one warp buckets the
// sequences by 128-token tile count exactly like fmha_plan_kernel and writes the item
// prefix, so the persistent kernels need no separate planning launch and decode a work
// item with a few shared loads.  Larger batches use fmha_plan_kernel + global decode.
constexpr int kPlanCap = 512;
struct PlanSmem {
  int32_t prefix[kPlanCap + 1];  // item prefix along the bucketed order
  int32_t seq[kPlanCap];         // sequence id
  int32_t c0[kPlanCap];          // cu_seqlens[seq]
  int32_t len[kPlanCap];         // length of seq
};

// executed by all 32 lanes of one warp
__device__ __forceinline__ void build_plan_smem(PlanSmem& ps, const int32_t* __restrict__ cu, int32_t B, int32_t H,
                                                int32_t max_tiles, int32_t tiles_per_item, uint32_t lane) {
  const uint32_t lt = (1u << lane) - 1u;
  int32_t base = 0;
  for (int32_t c = max_tiles; c >= 0; --c) {
    for (int32_t b0 = 0; b0 < B; b0 += 32) {
      const int32_t b = b0 + (int32_t)lane;
      int32_t bucket = -1, a = 0, L = 0;
      if (b < B) {
        a = cu[b];
        L = cu[b + 1] - a;
        const int32_t nt = (L + kTile - 1) / kTile;
        bucket = nt < max_tiles ? (nt < 0 ? 0 : nt) : max_tiles;
      }
      const bool flag = bucket == c;
      const uint32_t bal = __ballot_sync(0xffffffffu, flag);
      if (flag) {
        const int32_t pos = base + __popc(bal & lt);
        ps.seq[pos] = b;
        ps.c0[pos] = a;
        ps.len[pos] = L;
      }
      base += __popc(bal);
    }
  }
  __syncwarp();
  int32_t running = 0;
  for (int32_t k0 = 0; k0 < B; k0 += 32) {
    const int32_t k = k0 + (int32_t)lane;
    int32_t items = 0;
    if (k < B) {
      const int32_t L = ps.len[k];
      const int32_t nt = L > 0 ? (L + kTile - 1) / kTile : 0;
      items = (tiles_per_item > 0 ? (nt + tiles_per_item - 1) / tiles_per_item : (nt > 0 ? 1 : 0)) * H;
    }
    int32_t incl = items;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    if (k < B) ps.prefix[k] = running + incl - items;
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) ps.prefix[B] = running;
}

// kBigB selects the global-memory decode at compile time: with a runtime branch the compiler
// hoists the global loads of the fallback above it and every decode pays an L2 round trip.
template <bool kBigB>
__device__ __forceinline__ bool decode_item_smem(int32_t w, const PlanSmem& ps, const FmhaPlanView& v,
                                                 const int32_t* __restrict__ cu, int32_t B, int32_t H,
                                                 int32_t tiles_per_item, WorkItem& it) {
  if (kBigB) return decode_item(w, v, cu, B, H, tiles_per_item, it);
  if (w >= ps.prefix[B]) return false;
  int32_t lo = 0, hi = B;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (ps.prefix[mid] <= w) lo = mid; else hi = mid - 1;
  }
  it.b = ps.seq[lo];
  const int32_t local = w - ps.prefix[lo];
  it.c0 = ps.c0[lo];
  it.L = ps.len[lo];
  it.pc0 = 0;
  it.nt = (it.L + kTile - 1) / kTile;
  if (tiles_per_item == 0) {
    it.h = local;
    it.tile = 0;
    it.ntile = it.nt;
    return true;
  }
  const int32_t ngroups = (it.nt + tiles_per_item - 1) / tiles_per_item;
  it.h = local / ngroups;
  it.tile = (local - it.h * ngroups) * tiles_per_item;
  it.ntile = min(tiles_per_item, it.nt - it.tile);
  return true;
}

// r-th work item of CTA c out of G along the plan, dealt in snake order (round r goes
// 0..G-1 on even rounds, G-1..0 on odd ones): with items sorted longest first this keeps
// the per-CTA totals within about one item of each other.
__device__ __forceinline__ int32_t snake_item(int32_t r, int32_t c, int32_t G) {
  return r * G + ((r & 1) ? (G - 1 - c) : c);
}

// The CTA's work items, decoded once at kernel start (one warp) into shared memory: the
// persistent loops then fetch item r with two shared loads instead of running the plan
// decode (binary search + divisions) at every item boundary -- code that executes once per
// item and so is rarely in the instruction cache.  The host guarantees that every CTA's
// items fit (item_table_fits); otherwise it launches the kBigB form, which decodes per item.
constexpr int kItemCap = 64;
struct ItemTable {
  int32_t n;                                   // this CTA's items
  WorkItem it[kItemCap];
};
// host: every CTA's share in snake order (at most ceil(items / grid)) fits the table;
// max_items is an upper bound of the plan's items
inline bool item_table_fits(int32_t B, int64_t max_items, int32_t grid) {
  return B <= kPlanCap && (max_items + grid - 1) / grid <= kItemCap;
}

__device__ __forceinline__ void build_item_table(ItemTable& t, const PlanSmem& ps, const int32_t* __restrict__ cu,
                                                 int32_t B, int32_t H, int32_t tiles_per_item, int32_t cta, int32_t G,
                                                 uint32_t lane) {
  const FmhaPlanView none{};
  int32_t count = 0;
  for (int32_t r0 = 0; r0 < kItemCap; r0 += 32) {
    const int32_t r = r0 + (int32_t)lane;
    WorkItem it;
    const bool ok = decode_item_smem<false>(snake_item(r, cta, G), ps, none, cu, B, H, tiles_per_item, it);
    if (ok) t.it[r] = it;
    count += __popc(__ballot_sync(0xffffffffu, ok));     // ok is monotone in r
  }
  if (lane == 0) t.n = count;
}

// The table from a host schedule (ub_fmha_schedule): sched[0] = grid, sched[1 + c] .. sched[2 + c]
// the CTA's entry range, entries b*H + h (tiles_per_item 0) or (b*H + h)*8 + g (tile pair g).
// Returns false (the caller falls back to the snake deal) when the schedule was built for
// another grid size.  Executed by all 32 lanes of one warp.
__device__ __forceinline__ bool build_item_table_sched(ItemTable& t, const int32_t* __restrict__ sched,
                                                       const int32_t* __restrict__ cu, int32_t H, int32_t tiles_per_item,
                                                       int32_t cta, int32_t G, uint32_t lane) {
  if (__ldg(sched) != G) return false;
  const int32_t o0 = __ldg(sched + 1 + cta), n = min(__ldg(sched + 2 + cta) - o0, kItemCap - 1);
  const int32_t* ent = sched + 2 + G + o0;
  for (int32_t r = (int32_t)lane; r < n; r += 32) {
    const int32_t e = __ldg(ent + r);
    const int32_t bh = tiles_per_item == 0 ? e : (e >> 3), g = tiles_per_item == 0 ? 0 : (e & 7);
    WorkItem it;
    it.b = bh / H;
    it.h = bh - it.b * H;
    it.c0 = cu[it.b];
    it.L = cu[it.b + 1] - it.c0;
    it.nt = (it.L + kTile - 1) / kTile;
    it.pc0 = 0;
    it.tile = tiles_per_item == 0 ? 0 : 2 * g;
    it.ntile = tiles_per_item == 0 ? it.nt : min(2, it.nt - 2 * g);
    t.it[r] = it;
  }
  if (lane == 0) t.n = n;
  return true;
}

// item r of this CTA: from the table, or (kBigB) decoded from the global plan.  kTail adds
// a smem-plan decode for items past a full table -- unreachable while item_table_fits holds,
// but it changes how ptxas allocates the caller's registers: measured 3.6 % faster for the
// forward without dropout (55.8 vs 57.9 us on config 2) and slower with dropout (spills),
// so the forward sets it for p = 0 only.
template <bool kBigB, bool kTail = false>
__device__ __forceinline__ bool next_item(int32_t r, const ItemTable& t, const PlanSmem& ps, const FmhaPlanView& v,
                                          const int32_t* __restrict__ cu, int32_t B, int32_t H, int32_t tiles_per_item,
                                          int32_t cta, int32_t G, WorkItem& it) {
  if (kBigB) return decode_item(snake_item(r, cta, G), v, cu, B, H, tiles_per_item, it);
  if (r < t.n) {
    it = t.it[r];
    return true;
  }
  if (!kTail || t.n < kItemCap) return false;
  return decode_item_smem<false>(snake_item(r, cta, G), ps, v, cu, B, H, tiles_per_item, it);
}

// Dropout keep bits for 16 consecutive keys j0..j0+15 (j0 % 16 == 0) of packed row t (R5):
// bit e set <=> byte e of the Philox block (word e >> 2, byte e & 3) >= thr (8-bit threshold).
__device__ __forceinline__ uint32_t keep_bits16(uint32_t j0, uint32_t t, uint32_t h, uint32_t off, uint32_t k0,
                                                uint32_t k1, uint32_t thr) {
  const U4 w = philox4x32_10(j0 >> 4, t, h, off, k0, k1);
  const uint32_t words[4] = {w.x, w.y, w.z, w.w};
  // SWAR r8 >= thr on the 4 bytes of a word, half of it on the FMA pipe (the ALU pipe carries
  // Philox's XORs): d's byte msb = [r8 & 0x7F >= thr & 0x7F] (bytes (r8 & 0x7F) + 0x80 -
  // (thr & 0x7F) never borrow); with the msb of r8 and thr that decides r8 >= thr; the four
  // msbs (bits 7, 15, 23, 31) land on bits 28..31 of one multiply.  Checked against the byte
  // compare for every (byte, thr) pair.
  const uint32_t c1 = 0x80808080u - (thr & 0x7Fu) * 0x01010101u;
  uint32_t bits = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t d = (words[q] & 0x7F7F7F7Fu) + c1;
    const uint32_t r = (thr & 0x80u) ? (words[q] & d & 0x80808080u) : ((words[q] | d) & 0x80808080u);
    bits += ((r * 0x00204081u) >> 28) * (1u << (4 * q));
  }
  return bits;
}

// Host: 2-D bf16 tensor map over a row-major [rows, cols] matrix with row pitch
// `pitch_bytes`, box {64 cols, 128 rows}, 128-B swizzle (matches sdesc_sw128).
ub_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                         uint32_t box_cols = 64, uint32_t box_rows = 128, int swizzle_bytes = 128);
// Host: 2-D fp32 tensor map (row-major [rows, cols]), box {box_cols, box_rows}, swizzle of
// box_cols * 4 bytes (128 or 64).
// Host: 1-D fp32 tensor map over n elements, box of `box` elements (no swizzle).
ub_status make_tmap_f32_1d(CUtensorMap* map, const void* base, uint64_t n, uint32_t box);
ub_status make_tmap_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                        uint32_t box_cols, uint32_t box_rows, int swizzle_bytes = 128);

}  // namespace ub
