// Host-side static schedule of the persistent FMHA grids' work items (include/ub.h,
// ub_fmha_schedule).  The schedule only depends on the batch's lengths -- an input-only
// operator in the sense of P:402, computed while the padding exchange (whose planner holds the
// post-exchange lengths one step ahead) is still running -- and replaces the
// kernels' built-in snake deal (round r of G items, alternating direction) by longest-
// processing-time-first list scheduling: items in decreasing estimated cost, each to the CTA
// with the least estimated load so far (ties: lowest CTA id).  Each CTA's list keeps
// assignment order, i.e. decreasing cost, like the snake deal.  Results of the kernels do not
// depend on the schedule (each item's arithmetic and summation order are fixed); only the
// makespan does.
#include <algorithm>
#include <vector>

#include "ub_internal.h"

namespace ub {
namespace {

constexpr int32_t kSchedTile = 128;   // kTile of the tensor-core path
constexpr int32_t kSchedItemCap = 63; // < the kernels' per-CTA item table (kItemCap = 64)

// Estimated cost of a work item (x10 below), in units of one (query tile, key tile) step of two
// busy softmax / compute warpgroups.  Backward item (sequence, head): nt passes of nt pairs,
// plus a pass's K/V load and dK/dV drain and an item's setup: nt^2 + 0.3 nt + 0.5.  Forward item
// (sequence, head, query-tile pair): nt key steps, one tile alone about 0.7 of a pair's step
// (one warpgroup idles, the other runs faster alone), + 0.3.

}  // namespace

size_t fmha_schedule_ints(int32_t B, int32_t H, int32_t max_seqlen, int32_t grid, int32_t is_bwd) {
  const int64_t mt = (max_seqlen + kSchedTile - 1) / kSchedTile;
  const int64_t per_seq = is_bwd ? H : (int64_t)H * ((mt + 1) / 2);
  return (size_t)(2 + grid + (int64_t)B * per_seq);
}

}  // namespace ub

using namespace ub;

extern "C" size_t ub_fmha_schedule_ints(int32_t B, int32_t heads, int32_t max_seqlen, int32_t grid, int32_t is_bwd) {
  if (B < 1 || heads < 1 || max_seqlen < 1 || grid < 1) return 0;
  return fmha_schedule_ints(B, heads, max_seqlen, grid, is_bwd);
}

extern "C" ub_status ub_fmha_schedule(const int32_t* h_lengths, int32_t B, int32_t heads, int32_t max_seqlen,
                                      int32_t grid, int32_t is_bwd, int32_t* h_sched, size_t cap_ints) {
  clear_error();
  UB_REQUIRE(h_lengths && h_sched, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(B >= 1 && heads >= 1 && grid >= 1 && max_seqlen >= 1, UB_ERR_INVALID_ARG, "bad sizes");
  UB_REQUIRE(max_seqlen <= 8 * 2 * kSchedTile, UB_ERR_UNSUPPORTED, "max_seqlen %d above 2048", max_seqlen);
  UB_REQUIRE((int64_t)B * heads < (1ll << 27), UB_ERR_UNSUPPORTED, "batch too large for the schedule encoding");
  UB_REQUIRE(cap_ints >= fmha_schedule_ints(B, heads, max_seqlen, grid, is_bwd), UB_ERR_SHAPE,
             "schedule buffer of %zu ints, need %zu", cap_ints, fmha_schedule_ints(B, heads, max_seqlen, grid, is_bwd));
  // Items come in a few cost classes (nt = 1..16 tiles; forward: pair or single tile), each in
  // (sequence, head, group) order: walk the classes in decreasing cost (a counting sort) --
  // the stable order of a sort by cost -- with integer costs (x10) and a binary min-heap of
  // (load, CTA) for the least-loaded CTA.
  constexpr int kMaxNt = 16;
  int32_t cls_count[2 * kMaxNt + 2] = {};
  for (int32_t b = 0; b < B; ++b) {
    const int32_t L = h_lengths[b];
    UB_REQUIRE(L >= 0 && L <= max_seqlen, UB_ERR_CAPACITY, "length %d of sequence %d outside [0, %d]", L, b, max_seqlen);
  }
  // class id -> integer cost (x10); forward classes: 2 nt + (ntile == 2)
  auto cost10 = [is_bwd](int32_t cls) -> int64_t {
    if (is_bwd) return 10ll * cls * cls + 3ll * cls + 5;
    const int32_t nt = cls >> 1;
    return (cls & 1) ? 10ll * nt + 3 : 7ll * nt + 3;
  };
  std::vector<int32_t> keys;
  std::vector<int32_t> cls_of;
  keys.reserve((size_t)B * heads * (is_bwd ? 1 : 8));
  for (int32_t b = 0; b < B; ++b) {
    const int32_t nt = (h_lengths[b] + kSchedTile - 1) / kSchedTile;
    for (int32_t h = 0; h < heads && nt > 0; ++h) {
      const int32_t bh = b * heads + h;
      if (is_bwd) {
        keys.push_back(bh);
        cls_of.push_back(nt);
      } else {
        for (int32_t g = 0; 2 * g < nt; ++g) {
          keys.push_back(bh * 8 + g);
          cls_of.push_back(2 * nt + (nt - 2 * g >= 2 ? 1 : 0));
        }
      }
    }
  }
  const int32_t n = (int32_t)keys.size();
  const int ncls = 2 * kMaxNt + 2;
  for (int32_t i = 0; i < n; ++i) ++cls_count[cls_of[i]];
  // classes in decreasing cost, ties by class id descending (deterministic)
  int32_t order[2 * kMaxNt + 2];
  for (int c = 0; c < ncls; ++c) order[c] = c;
  std::sort(order, order + ncls, [&](int32_t x, int32_t y) {
    const int64_t cx = cost10(x), cy = cost10(y);
    return cx != cy ? cx > cy : x > y;
  });
  std::vector<int32_t> start(ncls + 1, 0), pos(ncls);
  {
    int32_t acc = 0;
    for (int k = 0; k < ncls; ++k) {
      pos[order[k]] = acc;
      acc += cls_count[order[k]];
    }
  }
  std::vector<int32_t> sorted(n);
  for (int32_t i = 0; i < n; ++i) sorted[pos[cls_of[i]]++] = i;
  // LPT over the sorted items, one cost class at a time: with equal costs the greedy's choices
  // are the merge of the CTAs sorted by (load, id) with the queue of CTAs it has just loaded
  // (appended in non-decreasing load order) -- O(m + G log G) per class instead of a heap
  // operation per item; the same assignment as a (load, id) min-heap.
  std::vector<int64_t> load(grid, 0);
  std::vector<int32_t> owner(n), A(grid), A2(grid), Q((size_t)n + grid);
  for (int32_t x = 0; x < grid; ++x) A[x] = x;             // CTAs by (load, id): all loads 0
  auto before = [&](int32_t x, int32_t y) { return load[x] != load[y] ? load[x] < load[y] : x < y; };
  int32_t k = 0;
  for (int ci = 0; ci < ncls; ++ci) {
    const int32_t cls = order[ci], m = cls_count[cls];
    if (m == 0) continue;
    const int64_t c = cost10(cls);
    int32_t ia = 0, qh = 0, qt = 0;
    for (int32_t t = 0; t < m; ++t, ++k) {
      const bool from_a = ia < grid && (qh == qt || before(A[ia], Q[qh]));
      const int32_t cta = from_a ? A[ia++] : Q[qh++];
      owner[k] = cta;
      load[cta] += c;
      Q[qt++] = cta;
    }
    // the next class's order: merge the untouched CTAs with the queue's live entries (both
    // sorted by (load, id); together every CTA once)
    int32_t o = 0;
    while (ia < grid || qh < qt) {
      if (ia < grid && (qh == qt || before(A[ia], Q[qh]))) A2[o++] = A[ia++];
      else A2[o++] = Q[qh++];
    }
    A.swap(A2);
  }
  // per-CTA lists in assignment order (a counting sort by owner)
  std::vector<int32_t> cnt(grid + 1, 0);
  for (int32_t k = 0; k < n; ++k) ++cnt[owner[k] + 1];
  h_sched[0] = grid;
  for (int32_t c = 0; c < grid; ++c) {
    UB_REQUIRE(cnt[c + 1] <= kSchedItemCap, UB_ERR_UNSUPPORTED,
               "CTA %d would hold %d items (table holds %d): run without a schedule", c, cnt[c + 1], kSchedItemCap);
    cnt[c + 1] += cnt[c];
  }
  for (int32_t c = 0; c <= grid; ++c) h_sched[1 + c] = cnt[c];
  for (int32_t k = 0; k < n; ++k) h_sched[2 + grid + cnt[owner[k]]++] = keys[sorted[k]];
  return UB_OK;
}
