// Host-side padding-exchange planner (§IV-B-1) and exchange copy tables.
// Pure functions of the all-gathered lengths: every rank computes byte-identical output.
#include <algorithm>
#include <numeric>
#include <vector>

#include "ub_internal.h"

namespace ub {
namespace {

// Step 2: order global ids by (valid tokens asc, id asc) -- R11.
std::vector<int32_t> sorted_ids(const int32_t* a, int32_t n) {
  std::vector<int32_t> ids(n);
  std::iota(ids.begin(), ids.end(), 0);
  std::stable_sort(ids.begin(), ids.end(), [a](int32_t x, int32_t y) { return a[x] < a[y]; });
  return ids;
}

struct ExactSearch {  // exhaustive min-max partition search for W*B <= 12 (R15 (iii))
  const int32_t* a;
  int32_t W, B, n;
  std::vector<std::vector<int32_t>> cur, best_groups;
  int64_t best_val = -1;
  std::vector<int32_t> best_perm;

  void canon(std::vector<int32_t>& g) const {
    std::sort(g.begin(), g.end(), [this](int32_t x, int32_t y) { return a[x] != a[y] ? a[x] < a[y] : x < y; });
  }
  void evaluate() {
    int64_t val = 0;
    for (auto& g : cur) {
      int64_t s = 0;
      for (int32_t x : g) s += a[x];
      val = std::max(val, s);
    }
    if (best_val >= 0 && val > best_val) return;
    std::vector<std::vector<int32_t>> groups = cur;
    for (auto& g : groups) canon(g);
    std::sort(groups.begin(), groups.end());
    std::vector<int32_t> perm;
    for (auto& g : groups) perm.insert(perm.end(), g.begin(), g.end());
    if (best_val < 0 || val < best_val || perm < best_perm) {
      best_val = val;
      best_perm = perm;
      best_groups = groups;
    }
  }
  // take the smallest remaining id, choose its B-1 companions, recurse
  void rec(std::vector<int32_t>& rem) {
    if (rem.empty()) { evaluate(); return; }
    const int32_t first = rem[0];
    std::vector<int32_t> rest(rem.begin() + 1, rem.end());
    const int m = (int)rest.size(), k = B - 1;
    std::vector<int> idx(k);
    std::iota(idx.begin(), idx.end(), 0);
    while (true) {
      std::vector<int32_t> grp{first};
      std::vector<char> used(m, 0);
      for (int j : idx) { grp.push_back(rest[j]); used[j] = 1; }
      std::vector<int32_t> left;
      for (int j = 0; j < m; ++j) if (!used[j]) left.push_back(rest[j]);
      cur.push_back(grp);
      rec(left);
      cur.pop_back();
      // next combination
      int i = k - 1;
      while (i >= 0 && idx[i] == m - k + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int j = i + 1; j < k; ++j) idx[j] = idx[j - 1] + 1;
    }
  }
};

// R20 step 2 (also R25 step 2): repeat (at most 4*W*B times): M = most loaded rank, m = least
// loaded (lowest index on ties); among pairs x in M, y in m with d = c[x] - c[y] > 0 take the
// one minimising max(load[M] - d, load[m] + d), ties by (x, y) ascending; stop unless that is
// < load[M]; swap x and y.
void swap_refine(const std::vector<int64_t>& c, int32_t W, int32_t B, std::vector<std::vector<int32_t>>& grp,
                 std::vector<int64_t>& load) {
  const int32_t n = W * B;
  for (int32_t iter = 0; iter < 4 * n && W > 1; ++iter) {
    int32_t M = 0, m = 0;
    for (int32_t r = 1; r < W; ++r) {
      if (load[r] > load[M]) M = r;
      if (load[r] < load[m]) m = r;
    }
    if (M == m) break;
    int64_t best_val = load[M];
    int32_t bx = -1, by = -1, bi = -1, bj = -1;
    for (int32_t i = 0; i < B; ++i)
      for (int32_t j = 0; j < B; ++j) {
        const int32_t x = grp[M][i], y = grp[m][j];
        const int64_t d = c[x] - c[y];
        if (d <= 0) continue;
        const int64_t v = std::max(load[M] - d, load[m] + d);
        if (v < best_val || (v == best_val && bx >= 0 && (x < bx || (x == bx && y < by)))) {
          best_val = v; bx = x; by = y; bi = i; bj = j;
        }
      }
    if (bx < 0) break;
    const int64_t d = c[bx] - c[by];
    grp[M][bi] = by;
    grp[m][bj] = bx;
    load[M] -= d;
    load[m] += d;
  }
}

// Cardinality-constrained LPT with (max, min) swap refinement on an integer per-sample cost
// (NEXT-2 of SURVEY §8(f)).  Steps, as oracle/balance.py:
//   1. ids by (cost desc, id asc); each goes to the open rank (fewer than B samples) with the
//      least load, lowest rank on ties;
//   2. repeat (at most 4*W*B times): M = most loaded rank, m = least loaded (lowest index on
//      ties); among pairs x in M, y in m with d = c[x] - c[y] > 0 take the one minimising
//      max(load[M] - d, load[m] + d), ties by (x, y) ascending; stop unless that is < load[M];
//   3. if the paper's interleave (same cost) has a strictly smaller maximum, use it instead;
//   4. each rank lists its samples by (length asc, id asc), the paper's order (R12).
void plan_lpt(const int32_t* a, const std::vector<int64_t>& c, int32_t W, int32_t B, int32_t* perm) {
  const int32_t n = W * B;
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&c](int32_t x, int32_t y) { return c[x] > c[y]; });
  std::vector<std::vector<int32_t>> grp(W);
  std::vector<int64_t> load(W, 0);
  for (int32_t g : order) {
    int32_t best = -1;
    for (int32_t r = 0; r < W; ++r)
      if ((int32_t)grp[r].size() < B && (best < 0 || load[r] < load[best])) best = r;
    grp[best].push_back(g);
    load[best] += c[g];
  }
  swap_refine(c, W, B, grp, load);
  // the paper's interleave as a floor
  const auto ids = sorted_ids(a, n);
  int64_t paper_max = 0, lpt_max = 0;
  for (int32_t r = 0; r < W; ++r) {
    int64_t t = 0;
    for (int32_t k = 0; k < B; ++k) t += c[ids[r + k * W]];
    paper_max = std::max(paper_max, t);
    lpt_max = std::max(lpt_max, load[r]);
  }
  if (paper_max < lpt_max) {
    for (int32_t i = 0; i < W; ++i)
      for (int32_t k = 0; k < B; ++k) perm[i * B + k] = ids[i + k * W];
    return;
  }
  for (int32_t r = 0; r < W; ++r) {
    std::sort(grp[r].begin(), grp[r].end(), [a](int32_t x, int32_t y) { return a[x] != a[y] ? a[x] < a[y] : x < y; });
    for (int32_t k = 0; k < B; ++k) perm[r * B + k] = grp[r][k];
  }
}

// Reading R24: hand the W groups to the ranks maximising the tokens kept at home.  g[mask] =
// best kept tokens of groups popcount(mask)..W-1 placed on the ranks outside mask; the
// reconstruction takes, group by group, the smallest rank that attains the optimum, which
// yields the lexicographically smallest optimal sigma (the oracle's first maximum in
// lexicographic permutation order).
// Reading R25 (NEXT-2, locality-aware): every rank starts with its own samples, R20's swap
// refinement on tokens balances them, each rank lists its ids by (length asc, id asc).
void plan_stay(const int32_t* a, int32_t W, int32_t B, int32_t* perm) {
  std::vector<int64_t> c(a, a + (size_t)W * B);
  std::vector<std::vector<int32_t>> grp(W);
  std::vector<int64_t> load(W, 0);
  for (int32_t r = 0; r < W; ++r)
    for (int32_t k = 0; k < B; ++k) {
      grp[r].push_back(r * B + k);
      load[r] += a[r * B + k];
    }
  swap_refine(c, W, B, grp, load);
  for (int32_t r = 0; r < W; ++r) {
    std::sort(grp[r].begin(), grp[r].end(), [a](int32_t x, int32_t y) { return a[x] != a[y] ? a[x] < a[y] : x < y; });
    for (int32_t k = 0; k < B; ++k) perm[r * B + k] = grp[r][k];
  }
}

void relabel_groups(const int32_t* a, int32_t W, int32_t B, int32_t* perm, int64_t* before, int64_t* after) {
  std::vector<int64_t> M((size_t)W * W, 0);
  int64_t kept0 = 0;
  for (int32_t i = 0; i < W; ++i)
    for (int32_t k = 0; k < B; ++k) {
      const int32_t g = perm[i * B + k];
      M[(size_t)i * W + g / B] += a[g];
      if (g / B == i) kept0 += a[g];
    }
  const uint32_t full = (W >= 32) ? 0xFFFFFFFFu : ((1u << W) - 1u);
  std::vector<int64_t> best((size_t)full + 1, 0);
  for (int64_t mask = (int64_t)full - 1; mask >= 0; --mask) {
    const int32_t i = __builtin_popcount((uint32_t)mask);
    int64_t v = -1;
    for (int32_t r = 0; r < W; ++r)
      if (!((uint32_t)mask >> r & 1u)) v = std::max(v, M[(size_t)i * W + r] + best[(size_t)mask | (1u << r)]);
    best[(size_t)mask] = v;
  }
  std::vector<int32_t> sigma(W);
  uint32_t mask = 0;
  for (int32_t i = 0; i < W; ++i)
    for (int32_t r = 0; r < W; ++r)
      if (!(mask >> r & 1u) && M[(size_t)i * W + r] + best[mask | (1u << r)] == best[mask]) {
        sigma[i] = r;
        mask |= 1u << r;
        break;
      }
  std::vector<int32_t> old(perm, perm + (size_t)W * B);
  for (int32_t i = 0; i < W; ++i)
    std::copy(old.begin() + (size_t)i * B, old.begin() + (size_t)(i + 1) * B, perm + (size_t)sigma[i] * B);
  if (before) *before = kept0;
  if (after) *after = best[0];
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" ub_status ub_balance_relabel(const int32_t* a, int32_t W, int32_t B, int32_t* perm, int64_t* kept_before,
                                        int64_t* kept_after) {
  clear_error();
  UB_REQUIRE(a && perm, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(W >= 1 && B >= 1, UB_ERR_INVALID_ARG, "W=%d B=%d", W, B);
  UB_REQUIRE(W <= 20, UB_ERR_UNSUPPORTED, "locality relabeling needs W <= 20 (got %d)", W);
  std::vector<char> seen((size_t)W * B, 0);
  for (int32_t i = 0; i < W * B; ++i) {
    UB_REQUIRE(perm[i] >= 0 && perm[i] < W * B && !seen[perm[i]], UB_ERR_SHAPE, "perm is not a permutation");
    seen[perm[i]] = 1;
    UB_REQUIRE(a[perm[i]] >= 0, UB_ERR_INVALID_ARG, "negative length");
  }
  relabel_groups(a, W, B, perm, kept_before, kept_after);
  return UB_OK;
}

extern "C" ub_status ub_balance_plan(const int32_t* a, int32_t W, int32_t B, int32_t max_seqlen, int32_t mode,
                                     int32_t* perm, int64_t* rank_tokens, int32_t* send_samples,
                                     int64_t* send_tokens) {
  clear_error();
  UB_REQUIRE(a && perm, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(W >= 1 && B >= 1, UB_ERR_INVALID_ARG, "W=%d B=%d", W, B);
  UB_REQUIRE((int64_t)W * B <= (1 << 30), UB_ERR_SHAPE, "W*B too large");
  const int32_t n = W * B;
  for (int32_t g = 0; g < n; ++g) {
    UB_REQUIRE(a[g] >= 1, UB_ERR_INVALID_ARG, "length[%d] = %d < 1", g, a[g]);
    UB_REQUIRE(a[g] <= max_seqlen, UB_ERR_CAPACITY, "length[%d] = %d > max_seqlen %d", g, a[g], max_seqlen);
  }
  const bool locality = (mode & UB_BAL_LOCALITY) != 0;
  mode &= ~UB_BAL_LOCALITY;
  UB_REQUIRE(!locality || W <= 20, UB_ERR_UNSUPPORTED, "UB_BAL_LOCALITY needs W <= 20 (got %d)", W);
  if (mode == UB_BAL_PAPER) {
    const auto ids = sorted_ids(a, n);
    for (int32_t i = 0; i < W; ++i)                 // worker i takes i, i+W, i+2W, ...
      for (int32_t k = 0; k < B; ++k) perm[i * B + k] = ids[i + k * W];
  } else if (mode == UB_BAL_SNAKE) {
    const auto ids = sorted_ids(a, n);
    for (int32_t r = 0; r < B; ++r)
      for (int32_t s = 0; s < W; ++s) {
        const int32_t dst = (r % 2 == 0) ? s : W - 1 - s;
        perm[dst * B + r] = ids[r * W + s];
      }
  } else if (mode == UB_BAL_LPT) {
    std::vector<int64_t> c(a, a + n);
    plan_lpt(a, c, W, B, perm);
  } else if (mode == UB_BAL_STAY) {
    plan_stay(a, W, B, perm);
  } else if (mode == UB_BAL_EXACT_SMALL) {
    UB_REQUIRE(n <= 12, UB_ERR_UNSUPPORTED, "UB_BAL_EXACT_SMALL needs W*B <= 12 (got %d)", n);
    ExactSearch es{a, W, B, n};
    std::vector<int32_t> rem(n);
    std::iota(rem.begin(), rem.end(), 0);
    es.rec(rem);
    for (int32_t i = 0; i < n; ++i) perm[i] = es.best_perm[i];
  } else {
    return set_error(UB_ERR_INVALID_ARG, "bad balance mode %d", mode);
  }
  if (locality) relabel_groups(a, W, B, perm, nullptr, nullptr);
  if (rank_tokens)
    for (int32_t r = 0; r < W; ++r) {
      int64_t t = 0;
      for (int32_t k = 0; k < B; ++k) t += a[perm[r * B + k]];
      rank_tokens[r] = t;
    }
  if (send_samples) std::fill(send_samples, send_samples + (int64_t)W * W, 0);
  if (send_tokens) std::fill(send_tokens, send_tokens + (int64_t)W * W, 0);
  for (int32_t dst = 0; dst < W; ++dst)
    for (int32_t k = 0; k < B; ++k) {
      const int32_t g = perm[dst * B + k], src = g / B;
      if (send_samples) send_samples[src * W + dst] += 1;
      if (send_tokens) send_tokens[src * W + dst] += a[g];
    }
  return UB_OK;
}

extern "C" ub_status ub_balance_plan_weighted(const int32_t* a, int32_t W, int32_t B, int32_t max_seqlen,
                                              int64_t alpha, int64_t beta, int32_t* perm, int64_t* rank_cost) {
  clear_error();
  UB_REQUIRE(a && perm, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(W >= 1 && B >= 1, UB_ERR_INVALID_ARG, "W=%d B=%d", W, B);
  UB_REQUIRE((int64_t)W * B <= (1 << 30), UB_ERR_SHAPE, "W*B too large");
  UB_REQUIRE(alpha >= 0 && beta >= 0 && (alpha > 0 || beta > 0), UB_ERR_INVALID_ARG, "need alpha, beta >= 0, not both 0");
  UB_REQUIRE(alpha <= (1ll << 30) && beta <= (1ll << 30), UB_ERR_INVALID_ARG, "weights above 2^30");
  const int32_t n = W * B;
  std::vector<int64_t> c(n);
  for (int32_t g = 0; g < n; ++g) {
    UB_REQUIRE(a[g] >= 1, UB_ERR_INVALID_ARG, "length[%d] = %d < 1", g, a[g]);
    UB_REQUIRE(a[g] <= max_seqlen, UB_ERR_CAPACITY, "length[%d] = %d > max_seqlen %d", g, a[g], max_seqlen);
    c[g] = alpha * a[g] + beta * (int64_t)a[g] * a[g];
  }
  plan_lpt(a, c, W, B, perm);
  if (rank_cost)
    for (int32_t r = 0; r < W; ++r) {
      int64_t t = 0;
      for (int32_t k = 0; k < B; ++k) t += c[perm[r * B + k]];
      rank_cost[r] = t;
    }
  return UB_OK;
}

extern "C" ub_status ub_exchange_tables(const int32_t* a, const int32_t* perm, int32_t W, int32_t B, int32_t rank,
                                        int32_t is_unpack, int64_t* tab, int64_t* counts, int64_t* scounts,
                                        int64_t* total_tokens) {
  clear_error();
  UB_REQUIRE(a && perm && tab, UB_ERR_INVALID_ARG, "null pointer");
  UB_REQUIRE(W >= 1 && B >= 1 && rank >= 0 && rank < W, UB_ERR_INVALID_ARG, "bad W/B/rank");
  int64_t* src_tok = tab;
  int64_t* len = tab + B;
  int64_t* dst_tok = tab + 2 * B;
  int64_t* src_smp = tab + 3 * B;
  int64_t* dst_smp = tab + 4 * B;
  std::vector<int64_t> cnt(W, 0), scnt(W, 0);
  if (!is_unpack) {
    // source: this rank's packed batch; cu of local samples
    std::vector<int64_t> cu(B + 1, 0);
    for (int32_t k = 0; k < B; ++k) cu[k + 1] = cu[k] + a[rank * B + k];
    int64_t off = 0;
    int32_t q = 0;
    for (int32_t dst = 0; dst < W; ++dst)
      for (int32_t k = 0; k < B; ++k) {
        const int32_t g = perm[dst * B + k];
        if (g / B != rank) continue;
        const int32_t kk = g % B;
        UB_REQUIRE(q < B, UB_ERR_SHAPE, "perm is not a permutation");
        src_tok[q] = cu[kk]; len[q] = a[g]; dst_tok[q] = off; src_smp[q] = kk; dst_smp[q] = q;
        off += a[g]; cnt[dst] += a[g]; scnt[dst] += 1; ++q;
      }
    UB_REQUIRE(q == B, UB_ERR_SHAPE, "rank %d sends %d samples, expected %d", rank, q, B);
    if (total_tokens) *total_tokens = off;
  } else {
    // receive buffer: chunks per source rank ascending, each in this rank's perm order
    for (int32_t k = 0; k < B; ++k) {
      const int32_t g = perm[rank * B + k];
      cnt[g / B] += a[g];
      scnt[g / B] += 1;
    }
    std::vector<int64_t> base(W, 0), sbase(W, 0);
    for (int32_t s = 1; s < W; ++s) { base[s] = base[s - 1] + cnt[s - 1]; sbase[s] = sbase[s - 1] + scnt[s - 1]; }
    int64_t off = 0;
    for (int32_t k = 0; k < B; ++k) {
      const int32_t g = perm[rank * B + k], s = g / B;
      src_tok[k] = base[s]; len[k] = a[g]; dst_tok[k] = off; src_smp[k] = sbase[s]; dst_smp[k] = k;
      base[s] += a[g]; sbase[s] += 1; off += a[g];
    }
    if (total_tokens) *total_tokens = off;
  }
  if (counts) for (int32_t r = 0; r < W; ++r) counts[r] = cnt[r];
  if (scounts) for (int32_t r = 0; r < W; ++r) scounts[r] = scnt[r];
  return UB_OK;
}
