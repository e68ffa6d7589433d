// Length-bucketed work plan for the persistent FMHA kernels (P:330 grouping).
//
// The paper groups sequences into (0,128] (128,256] (256,384] (384,512] and launches one
// kernel per group on its own stream.  Here a one-warp device kernel buckets sequences
// by their number of 128-token tiles (the same groups for 128-wide tiles, reading R19),
// longest bucket first (LPT order: the costliest work items start first), and writes
// a flat item list that one persistent launch walks.  cu_seqlens stays on the device:
// no host sync, no D2H of the lengths.
//
// Work item = (sequence, head, group of `tiles_per_item` 128-row tiles; 0 = all of them).
// Forward: pairs of query tiles (the two softmax warpgroups share K/V), cost = 2 x #key
// tiles.  Backward: the whole (sequence, head), cost = #tiles^2.  Costs grow with the
// sequence's tile count, so bucketing by tile count orders items longest-first.
// pad_c0: row base of each sequence in a tile-padded layout (backward dQ accumulator).
#include "ub_internal.h"

namespace ub {

size_t fmha_plan_bytes(int32_t B) {
  return align_up((size_t)B * 4, 256) + 2 * align_up((size_t)(B + 1) * 4, 256) + 256;
}

FmhaPlanView fmha_plan_view(void* ws, int32_t B) {
  char* p = static_cast<char*>(ws);
  FmhaPlanView v;
  v.seq_order = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)B * 4, 256);
  v.item_prefix = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)(B + 1) * 4, 256);
  v.pad_c0 = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)(B + 1) * 4, 256);
  v.counters = reinterpret_cast<int32_t*>(p);
  return v;
}

__global__ void __launch_bounds__(32) fmha_plan_kernel(const int32_t* __restrict__ cu, int32_t B, int32_t H,
                                                       int32_t max_tiles, int32_t tiles_per_item, FmhaPlanView v) {
  const uint32_t lane = threadIdx.x;
  if (lane < 4) v.counters[lane] = 0;
  const uint32_t lt = (1u << lane) - 1u;
  int32_t base = 0;
  // bucket c = min(tiles, max_tiles), c = max_tiles .. 0 (0 = empty sequences, no work)
  for (int32_t c = max_tiles; c >= 0; --c) {
    for (int32_t b0 = 0; b0 < B; b0 += 32) {
      const int32_t b = b0 + (int32_t)lane;
      int32_t bucket = -1;
      if (b < B) {
        const int32_t L = cu[b + 1] - cu[b];
        const int32_t nt = (L + kTile - 1) / kTile;
        bucket = nt < max_tiles ? (nt < 0 ? 0 : nt) : max_tiles;
      }
      const bool flag = bucket == c;
      const uint32_t bal = __ballot_sync(0xffffffffu, flag);
      if (flag) v.seq_order[base + __popc(bal & lt)] = b;
      base += __popc(bal);
    }
  }
  __syncwarp();
  int32_t running = 0;
  for (int32_t k0 = 0; k0 < B; k0 += 32) {
    const int32_t k = k0 + (int32_t)lane;
    int32_t items = 0;
    if (k < B) {
      const int32_t b = v.seq_order[k];
      const int32_t L = cu[b + 1] - cu[b];
      const int32_t nt = L > 0 ? (L + kTile - 1) / kTile : 0;
      items = (tiles_per_item > 0 ? (nt + tiles_per_item - 1) / tiles_per_item : (nt > 0 ? 1 : 0)) * H;
    }
    int32_t incl = items;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    if (k < B) v.item_prefix[k] = running + incl - items;
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) v.item_prefix[B] = running;
  // padded row bases in the original sequence order (each sequence rounded up to whole tiles)
  int32_t pad = 0;
  for (int32_t b0 = 0; b0 < B; b0 += 32) {
    const int32_t b = b0 + (int32_t)lane;
    int32_t rows = 0;
    if (b < B) {
      const int32_t L = cu[b + 1] - cu[b];
      rows = (L > 0 ? (L + kTile - 1) / kTile : 0) * kTile;
    }
    int32_t incl = rows;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    if (b < B) v.pad_c0[b] = pad + incl - rows;
    pad += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) v.pad_c0[B] = pad;
}

ub_status launch_fmha_plan(const int32_t* d_cu, int32_t B, int32_t H, int32_t max_tiles, int32_t tiles_per_item,
                           FmhaPlanView v, cudaStream_t s) {
  fmha_plan_kernel<<<1, 32, 0, s>>>(d_cu, B, H, max_tiles, tiles_per_item, v);
  UB_CHECK_LAUNCH();
  return UB_OK;
}

}  // namespace ub
