"""Padding-exchange load balancer (§IV-B-1, Fig. fig-exchange-padding).
ORACLE: test infrastructure only.  Plain Python.

The paper's three steps, on the valid-token counts the all-gather makes
identical on every worker:
  1. all-gather: global sample id g = r*B + k (rank-major concatenation).
  2. "Sort the all-gathered input sequences ... according to the valid token number"
     (P:357); ties broken by global id ascending (reading R11).
  3. "Interleave slicing": worker i takes sorted positions i, i+W, i+2W, ...,
     in that order (reading R12).

Also here (reading R15): the snake (boustrophedon) deal, and a brute-force search
for the min-max-tokens partition with equal cardinality B, by two independent
enumerators, with the canonical tie-break "lexicographically smallest perm vector".
Beyond the paper (reading R20, NEXT-2): cardinality-constrained LPT with swap refinement
on an integer cost alpha*L + beta*L^2, floored by the paper's plan.

Beyond the paper (reading R24, NEXT-2): relabel_locality -- the plan's W groups handed to the
ranks so that the most tokens stay home (exhaustive over the W! labelings); (reading R25)
balance_stay -- start from "every rank keeps its samples" and balance by R20's swaps.

Outputs use the library's layout: perm[r*B + k] = global id of the k-th sample on
rank r; rank_tokens[r]; send_samples[src*W + dst]; send_tokens[src*W + dst].

Pins (tests/test_oracle_balance.py): SPEC worked examples (S:316 tie order, S:326 W=2
positions 0,2,4, S:336 [[512,512],[64,64]] -> 576/576), permutation + cardinality,
spread <= Lmax - Lmin, brute force agreement of the two enumerators, the
counterexample [1,2,3,4] (paper 4/6 vs optimum 5/5), W=1 and B=1 special cases.
LPT: never above the paper's maximum (by construction, checked), equal to the brute-force
optimum where the greedy provably is (B = 1: one sample per rank; all lengths equal), a
hand-worked instance, and max <= OPT + Lmax on random tiny inputs.  relabel_locality: a
hand-worked instance, the optimum equals scipy's linear_sum_assignment (Hungarian method, an
independent library routine) on the same W x W matrix, every rank's load and sample order
unchanged up to the labeling, never fewer kept tokens than the identity labeling.
balance_stay: hand-worked instance, W = 1 / equal-lengths special cases (no swap), cardinality,
max load never above the unbalanced maximum, every moved sample belongs to a swap pair.  Parity pinned.
"""
from __future__ import annotations

import itertools

import numpy as np


def _check(all_lengths, W, B):
    a = [int(x) for x in all_lengths]
    if W < 1 or B < 1 or len(a) != W * B:
        raise ValueError("shape: need W*B lengths")
    if any(x < 1 for x in a):
        raise ValueError("length must be >= 1")
    return a


def sort_by_valid_tokens(all_lengths):
    """Global ids ordered by (valid tokens asc, id asc) -- P:357 + R11."""
    a = list(all_lengths)
    return sorted(range(len(a)), key=lambda g: (a[g], g))


def plan_from_groups(all_lengths, W, B, groups):
    """perm / rank_tokens / send matrices for a list of W per-rank id lists."""
    a = list(all_lengths)
    perm = np.zeros(W * B, dtype=np.int64)
    rank_tokens = np.zeros(W, dtype=np.int64)
    send_samples = np.zeros(W * W, dtype=np.int64)
    send_tokens = np.zeros(W * W, dtype=np.int64)
    for dst in range(W):
        assert len(groups[dst]) == B
        for k, g in enumerate(groups[dst]):
            perm[dst * B + k] = g
            rank_tokens[dst] += a[g]
            src = g // B
            send_samples[src * W + dst] += 1
            send_tokens[src * W + dst] += a[g]
    return {"perm": perm, "rank_tokens": rank_tokens,
            "send_samples": send_samples, "send_tokens": send_tokens}


def balance_paper(all_lengths, W, B):
    """NVIDIA/paper padding exchange: sort + interleave slice."""
    a = _check(all_lengths, W, B)
    order = sort_by_valid_tokens(a)
    groups = [[order[i + k * W] for k in range(B)] for i in range(W)]
    return plan_from_groups(a, W, B, groups)


def balance_snake(all_lengths, W, B):
    """Snake deal of the same sorted list: round r goes to ranks 0..W-1 when r is even
    and W-1..0 when r is odd (a variant of P:359, reading R15(iv))."""
    a = _check(all_lengths, W, B)
    order = sort_by_valid_tokens(a)
    groups = [[] for _ in range(W)]
    for r in range(B):
        for s in range(W):
            dst = s if r % 2 == 0 else W - 1 - s
            groups[dst].append(order[r * W + s])
    return plan_from_groups(a, W, B, groups)


def balance_lpt(all_lengths, W, B, alpha=1, beta=0):
    """Beyond the paper (reading R20): cardinality-constrained
    LPT with (max, min) swap refinement on the integer cost c = alpha*L + beta*L^2, floored by
    the paper's interleave.  Written as the four steps of DESIGN.md R20, in order:
      1. ids by (cost desc, id asc); each to the open rank (< B samples) with the least
         load, lowest rank on ties;
      2. up to 4*W*B times: M = most loaded rank, m = least loaded (lowest index on ties);
         over x in M, y in m with d = c[x] - c[y] > 0 take the pair minimising
         max(load[M] - d, load[m] + d), ties by (x, y) ascending; stop unless it beats
         load[M]; swap;
      3. if the paper's plan has a strictly smaller maximum cost, return the paper's plan;
      4. each rank lists its ids by (length asc, id asc).
    Returns the plan dict of plan_from_groups plus "rank_cost"."""
    a = _check(all_lengths, W, B)
    n = W * B
    c = [alpha * x + beta * x * x for x in a]
    order = sorted(range(n), key=lambda g: (-c[g], g))
    groups = [[] for _ in range(W)]
    load = [0] * W
    for g in order:
        open_ranks = [r for r in range(W) if len(groups[r]) < B]
        r = min(open_ranks, key=lambda q: (load[q], q))
        groups[r].append(g)
        load[r] += c[g]
    for _ in range(4 * n):
        if W == 1:
            break
        M = max(range(W), key=lambda q: (load[q], -q))
        m = min(range(W), key=lambda q: (load[q], q))
        if M == m:
            break
        best = None
        for x in groups[M]:
            for y in groups[m]:
                d = c[x] - c[y]
                if d <= 0:
                    continue
                key = (max(load[M] - d, load[m] + d), x, y)
                if best is None or key < best:
                    best = key
        if best is None or best[0] >= load[M]:
            break
        _, x, y = best
        d = c[x] - c[y]
        groups[M][groups[M].index(x)] = y
        groups[m][groups[m].index(y)] = x
        load[M] -= d
        load[m] += d
    paper = balance_paper(a, W, B)
    paper_groups = [list(paper["perm"][r * B:(r + 1) * B]) for r in range(W)]
    paper_max = max(sum(c[g] for g in grp) for grp in paper_groups)
    if paper_max < max(load):
        groups = paper_groups
    else:
        groups = [sorted(grp, key=lambda g: (a[g], g)) for grp in groups]
    out = plan_from_groups(a, W, B, groups)
    out["rank_cost"] = np.array([sum(c[g] for g in grp) for grp in groups], dtype=np.int64)
    return out


def _canon_group(a, grp):
    return tuple(sorted(grp, key=lambda g: (a[g], g)))


def partitions_recursive(n, W, B):
    """Enumerator 1: unlabeled partitions of range(n) into W groups of B, by taking the
    smallest remaining id and choosing its B-1 companions."""
    def rec(rem):
        if not rem:
            yield []
            return
        first, rest = rem[0], rem[1:]
        for comp in itertools.combinations(rest, B - 1):
            left = [x for x in rest if x not in comp]
            for tail in rec(left):
                yield [(first,) + comp] + tail
    yield from rec(list(range(n)))


def partitions_labelings(n, W, B):
    """Enumerator 2: all W**n labelings, keep those with exactly B per label, dedupe to
    unlabeled partitions.  Only for tiny W**n."""
    seen = set()
    for lab in itertools.product(range(W), repeat=n):
        counts = [0] * W
        for x in lab:
            counts[x] += 1
        if any(c != B for c in counts):
            continue
        groups = [tuple(i for i in range(n) if lab[i] == r) for r in range(W)]
        key = tuple(sorted(groups))
        if key not in seen:
            seen.add(key)
            yield [list(g) for g in key]


def balance_opt(all_lengths, W, B, enumerator="recursive"):
    """Brute-force optimum: minimise the max per-rank token count over all equal-
    cardinality partitions; among optima return the lexicographically smallest perm
    vector (groups laid out in (length, id) order inside a rank)."""
    a = _check(all_lengths, W, B)
    n = W * B
    gen = partitions_recursive(n, W, B) if enumerator == "recursive" else partitions_labelings(n, W, B)
    best_val, best_perm, best_groups = None, None, None
    for part in gen:
        val = max(sum(a[g] for g in grp) for grp in part)
        if best_val is not None and val > best_val:
            continue
        groups = sorted(_canon_group(a, grp) for grp in part)   # lexicographic labelling
        perm = [g for grp in groups for g in grp]
        if best_val is None or val < best_val or perm < best_perm:
            best_val, best_perm, best_groups = val, perm, groups
    out = plan_from_groups(a, W, B, [list(g) for g in best_groups])
    out["opt_max_tokens"] = best_val
    return out


def balance_stay(all_lengths, W, B):
    """Beyond the paper (reading R25, NEXT-2 "locality-aware"): balance by moving as few
    samples as possible.  The steps, in order:
      1. every rank keeps its own samples (group r = ids r*B .. r*B + B - 1);
      2. R20's step 2 on tokens (c = L), unchanged: up to 4*W*B times, M = most loaded rank
         (lowest index on ties), m = least loaded (lowest index on ties); over x in M, y in m
         with d = L[x] - L[y] > 0 take the pair minimising max(load[M] - d, load[m] + d), ties
         by (x, y) ascending; stop unless it beats load[M]; swap x and y;
      3. each rank lists its ids by (length asc, id asc).
    Every swap moves two samples; no floor by the paper's plan (that would move ~all tokens)."""
    a = _check(all_lengths, W, B)
    groups = [list(range(r * B, (r + 1) * B)) for r in range(W)]
    load = [sum(a[g] for g in grp) for grp in groups]
    for _ in range(4 * W * B):
        if W == 1:
            break
        M = max(range(W), key=lambda q: (load[q], -q))
        m = min(range(W), key=lambda q: (load[q], q))
        if M == m:
            break
        best = None
        for x in groups[M]:
            for y in groups[m]:
                d = a[x] - a[y]
                if d <= 0:
                    continue
                key = (max(load[M] - d, load[m] + d), x, y)
                if best is None or key < best:
                    best = key
        if best is None or best[0] >= load[M]:
            break
        _, x, y = best
        d = a[x] - a[y]
        groups[M][groups[M].index(x)] = y
        groups[m][groups[m].index(y)] = x
        load[M] -= d
        load[m] += d
    return plan_from_groups(a, W, B, [sorted(grp, key=lambda g: (a[g], g)) for grp in groups])


def kept_tokens(all_lengths, perm, W, B) -> int:
    """Tokens that stay on their source rank under a plan: sum of L_g over samples g that rank
    g // B keeps (the all-to-all-v moves every other token)."""
    a = list(all_lengths)
    return int(sum(a[int(perm[r * B + k])] for r in range(W) for k in range(B) if int(perm[r * B + k]) // B == r))


def relabel_locality(all_lengths, perm, W, B):
    """NEXT-2 beyond the paper (reading R24): the W groups of a plan (rank r's samples
    perm[r*B : r*B+B]) may be handed to the ranks in any order without changing any rank's
    load -- P:359's "worker i takes slice i" is one of W! labelings.  Choose the labeling that
    keeps the most tokens on their source rank: group i goes to rank sigma[i], maximising
    sum_i M[i][sigma[i]] with M[i][r] = tokens of group i whose source rank (g // B) is r.
    Exhaustive over all W! labelings in lexicographic order of sigma (itertools), the first
    maximum wins (ties -> lexicographically smallest sigma).  Returns the new perm (rank
    sigma[i] lists group i in its original order)."""
    a = list(all_lengths)
    M = [[0] * W for _ in range(W)]
    for i in range(W):
        for k in range(B):
            g = int(perm[i * B + k])
            M[i][g // B] += a[g]
    best, best_sigma = -1, None
    for sigma in itertools.permutations(range(W)):
        v = sum(M[i][sigma[i]] for i in range(W))
        if v > best:
            best, best_sigma = v, sigma
    out = np.zeros(W * B, dtype=np.int64)
    for i in range(W):
        r = best_sigma[i]
        out[r * B:(r + 1) * B] = [int(x) for x in perm[i * B:(i + 1) * B]]
    return out


def cu_seqlens_for_rank(all_lengths, perm, W, B, rank):
    """batch_offset of rank's post-exchange batch (P:302 on the rebalanced samples)."""
    a = list(all_lengths)
    out = [0]
    for k in range(B):
        out.append(out[-1] + a[int(perm[rank * B + k])])
    return np.asarray(out, dtype=np.int64)


def imbalance(rank_tokens) -> float:
    """max_r / mean_r - 1 (reading R14; S:296 defines max/mean)."""
    t = np.asarray(rank_tokens, dtype=np.float64)
    return float(t.max() / t.mean() - 1.0)
