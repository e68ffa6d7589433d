"""Pins for oracle.balance and oracle.exchange -- CPU only."""
import itertools

import numpy as np
import pytest

from oracle import balance, exchange, varlen
import synth


def test_spec_worked_examples(golden):
    g = golden["spec_worked_examples"]
    ex = g["sort_by_valid_tokens"][0]
    assert balance.sort_by_valid_tokens(ex["counts"]) == ex["order"], ex["cite"]
    ex = g["interleave_slice"][0]
    lens = list(range(1, ex["n"] + 1))                 # already sorted: position == id
    plan = balance.balance_paper(lens, ex["W"], ex["n"] // ex["W"])
    B = ex["n"] // ex["W"]
    assert plan["perm"][ex["worker"] * B:(ex["worker"] + 1) * B].tolist() == ex["positions"]
    ex = g["exchange_padding"][0]
    flat = [x for r in ex["lengths"] for x in r]
    plan = balance.balance_paper(flat, ex["W"], ex["B"])
    assert plan["rank_tokens"].tolist() == ex["rank_tokens"], ex["cite"]


def _invariants(plan, a, W, B):
    perm = plan["perm"]
    assert sorted(perm.tolist()) == list(range(W * B))                  # permutation
    for r in range(W):
        grp = perm[r * B:(r + 1) * B]
        assert len(grp) == B                                            # cardinality
        assert plan["rank_tokens"][r] == sum(a[g] for g in grp)
    ss = plan["send_samples"].reshape(W, W)
    assert np.all(ss.sum(axis=1) == B) and np.all(ss.sum(axis=0) == B)
    st = plan["send_tokens"].reshape(W, W)
    assert np.array_equal(st.sum(axis=0), plan["rank_tokens"])


def test_paper_mode_invariants_and_spread_bound():
    for W, B, seed in [(2, 56, 0), (4, 56, 1), (8, 56, 2), (3, 5, 3), (8, 1, 4), (1, 9, 5)]:
        a = synth.gen_lengths("mlperf_like_v0", W * B, seed).tolist()
        plan = balance.balance_paper(a, W, B)
        _invariants(plan, a, W, B)
        t = plan["rank_tokens"]
        assert t.max() - t.min() <= max(a) - min(a)                     # S:353 telescoping bound
        # interleave order inside a rank is ascending length (R12)
        for r in range(W):
            lens = [a[g] for g in plan["perm"][r * B:(r + 1) * B]]
            assert lens == sorted(lens)
        # determinism
        assert np.array_equal(balance.balance_paper(a, W, B)["perm"], plan["perm"])


def test_paper_mode_imbalance_gate_at_8():
    """BASELINE gate: max-over-ranks imbalance <= 5% at 8 GPUs, B=56 (proof bound 3.2%)."""
    for step in range(20):
        a = synth.skewed_rank_lengths(8, 56, step, "sorted-block").reshape(-1)
        plan = balance.balance_paper(a, 8, 56)
        assert balance.imbalance(plan["rank_tokens"]) <= 0.05


def test_two_enumerators_agree():
    rng = np.random.default_rng(0)
    for W, B in [(2, 2), (2, 3), (3, 2), (2, 4), (3, 3), (2, 5), (4, 2)]:
        n = W * B
        if W ** n > 300000:
            continue
        for _ in range(3):
            a = rng.integers(1, 20, size=n).tolist()
            r1 = balance.balance_opt(a, W, B, "recursive")
            r2 = balance.balance_opt(a, W, B, "labelings")
            assert r1["opt_max_tokens"] == r2["opt_max_tokens"]
            assert np.array_equal(r1["perm"], r2["perm"])


def test_opt_is_optimal_by_plain_search():
    """Independent check of the optimum: plain search over all permutations of the ids."""
    rng = np.random.default_rng(1)
    for W, B in [(2, 2), (2, 3), (3, 2)]:
        a = rng.integers(1, 50, size=W * B).tolist()
        best = min(max(sum(a[g] for g in perm[r * B:(r + 1) * B]) for r in range(W))
                   for perm in itertools.permutations(range(W * B)))
        assert balance.balance_opt(a, W, B)["opt_max_tokens"] == best


def test_counterexample_and_bounds_vs_opt():
    plan = balance.balance_paper([1, 2, 3, 4], 2, 2)
    assert sorted(plan["rank_tokens"].tolist()) == [4, 6]               # the paper's rule
    assert balance.balance_opt([1, 2, 3, 4], 2, 2)["opt_max_tokens"] == 5   # the optimum
    rng = np.random.default_rng(2)
    for _ in range(60):
        W, B = [(2, 2), (2, 3), (3, 2), (2, 4), (3, 3), (4, 2), (2, 5)][rng.integers(0, 7)]
        a = rng.integers(1, 513, size=W * B).tolist()
        opt = balance.balance_opt(a, W, B)["opt_max_tokens"]
        pm = balance.balance_paper(a, W, B)["rank_tokens"].max()
        sn = balance.balance_snake(a, W, B)["rank_tokens"].max()
        assert opt <= sn <= pm                                          # snake never worse than paper
        assert pm - opt <= (W - 1) / W * (max(a) - min(a)) + 1e-9
        if B <= 2:
            assert sn == opt                                            # snake optimal for B <= 2


def test_special_cases():
    a = [9, 3, 5]
    assert balance.balance_paper(a, 1, 3)["perm"].tolist() == [1, 2, 0]   # W=1: sorted order
    assert balance.balance_opt(a, 1, 3)["opt_max_tokens"] == 17
    p = balance.balance_paper([4, 1, 3], 3, 1)                            # B=1: one per rank
    assert p["perm"].tolist() == [1, 2, 0]
    with pytest.raises(ValueError):
        balance.balance_paper([1, 2, 3], 2, 2)                            # W*B not full (R13)
    with pytest.raises(ValueError):
        balance.balance_paper([1, 0], 2, 1)


def test_exchange_simulation():
    W, B, rec, srec = 3, 4, 16, 4
    lens = synth.gen_lengths("uniform", W * B, 11, max_seqlen=32).reshape(W, B)
    toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 20 + r).reshape(-1, rec) for r in range(W)]
    smps = [synth.gen_bytes(B * srec, 30 + r).reshape(B, srec) for r in range(W)]
    plan = balance.balance_paper(lens.reshape(-1), W, B)
    out = exchange.exchange(lens, toks, smps, plan["perm"], W, B)
    offs = [varlen.batch_offset(lens[r]) for r in range(W)]
    all_rows = sorted(bytes(x) for r in range(W) for x in toks[r])
    got_rows = sorted(bytes(x) for d in range(W) for x in out[d]["tokens"])
    assert all_rows == got_rows                                            # multiset preserved
    for d in range(W):
        assert out[d]["cu"][-1] == plan["rank_tokens"][d]
        # the rank's post-exchange batch_offset from the plan alone equals the offsets of the
        # records the simulation actually moved
        assert np.array_equal(balance.cu_seqlens_for_rank(lens.reshape(-1), plan["perm"], W, B, d), out[d]["cu"])
        for k in range(B):
            g = int(plan["perm"][d * B + k]); s, kk = divmod(g, B)
            a0, a1 = out[d]["cu"][k], out[d]["cu"][k + 1]
            assert np.array_equal(out[d]["tokens"][a0:a1], toks[s][offs[s][kk]:offs[s][kk + 1]])
            assert np.array_equal(out[d]["samples"][k], smps[s][kk])


# ---------------------------------------------------------------- LPT (reading R20, NEXT-2)
def test_lpt_hand_worked_instances():
    """Worked by hand from the four steps of R20."""
    # [1,2,3,4], W=2: greedy 4->r0, 3->r1, 2->r1, 1->r0 => {1,4} {2,3}: 5/5 (the optimum;
    # the paper's interleave gives 4/6)
    plan = balance.balance_lpt([1, 2, 3, 4], 2, 2)
    assert list(plan["perm"]) == [0, 3, 1, 2] and list(plan["rank_tokens"]) == [5, 5]
    # [5,1,1,1,4,2], W=2, B=3: 5->r0, 4->r1, 2->r1, 1->r0, 1->r0 (tie -> r0), 1->r1 (r0 full)
    plan = balance.balance_lpt([5, 1, 1, 1, 4, 2], 2, 3)
    assert list(plan["perm"]) == [1, 2, 0, 3, 5, 4] and list(plan["rank_tokens"]) == [7, 7]


def test_lpt_invariants_floor_and_optimality_cases():
    rng = np.random.default_rng(20)
    for _ in range(300):
        W = int(rng.integers(1, 5)); B = int(rng.integers(1, 4))
        a = rng.integers(1, 40, size=W * B).tolist()
        plan = balance.balance_lpt(a, W, B)
        perm = plan["perm"]
        assert sorted(perm.tolist()) == list(range(W * B))                        # a permutation
        assert plan["rank_tokens"].max() <= balance.balance_paper(a, W, B)["rank_tokens"].max()   # floor
        for r in range(W):                                                        # order within a rank
            grp = perm[r * B:(r + 1) * B]
            assert [(a[g], g) for g in grp] == sorted((a[g], g) for g in grp)
        if W * B <= 9:
            opt = balance.balance_opt(a, W, B)["opt_max_tokens"]
            assert plan["rank_tokens"].max() <= opt + max(a)                      # LPT bound
            if B == 1:
                assert plan["rank_tokens"].max() == opt                           # one sample per rank
    # all lengths equal: perfect balance
    plan = balance.balance_lpt([7] * 12, 4, 3)
    assert set(plan["rank_tokens"].tolist()) == {21}
    # W = 1: everything on rank 0, ascending
    plan = balance.balance_lpt([3, 1, 2], 1, 3)
    assert list(plan["perm"]) == [1, 2, 0]


def test_lpt_weighted_cost():
    """alpha*L + beta*L^2: with beta = 0 it is the token LPT scaled; with a quadratic cost the
    rank costs are what the plan's groups sum to."""
    rng = np.random.default_rng(21)
    for _ in range(50):
        W, B = 4, 5
        a = rng.integers(1, 512, size=W * B).tolist()
        p1 = balance.balance_lpt(a, W, B)
        p3 = balance.balance_lpt(a, W, B, alpha=3, beta=0)
        assert np.array_equal(p1["perm"], p3["perm"]) and np.array_equal(3 * p1["rank_tokens"], p3["rank_cost"])
        q = balance.balance_lpt(a, W, B, alpha=2048, beta=1)
        c = [2048 * x + x * x for x in a]
        assert [sum(c[g] for g in q["perm"][r * B:(r + 1) * B]) for r in range(W)] == q["rank_cost"].tolist()


def test_lpt_balances_far_better_at_8():
    """SURVEY Appendix A simulation: mean imbalance 1.6% (paper) vs ~0.01% (LPT) at W=8."""
    from synth import gen_lengths
    imb_p, imb_l = [], []
    for s in range(10):
        a = gen_lengths("mlperf_like_v0", 8 * 56, 100 + s)
        imb_p.append(balance.imbalance(balance.balance_paper(a, 8, 56)["rank_tokens"]))
        imb_l.append(balance.imbalance(balance.balance_lpt(a, 8, 56)["rank_tokens"]))
    assert np.mean(imb_l) < 0.002 < np.mean(imb_p)


# ---------------------------------------------------------------- locality relabeling (R24, NEXT-2)
def test_relabel_locality_hand_worked():
    """W=2, B=2, lengths rank0 = [5, 1], rank1 = [2, 9] (ids 0..3).  Paper plan: sorted
    ids by length = [1(1), 2(2), 0(5), 3(9)]; rank0 <- [1, 0], rank1 <- [2, 3].  Group 0
    = {1, 0} is all rank-0 data (6 tokens), group 1 = {2, 3} all rank-1 data (11): the
    identity labeling keeps all 17 tokens, the swap keeps 0 -> identity stays."""
    a = [5, 1, 2, 9]
    plan = balance.balance_paper(a, 2, 2)
    assert plan["perm"].tolist() == [1, 0, 2, 3]
    assert balance.relabel_locality(a, plan["perm"], 2, 2).tolist() == [1, 0, 2, 3]
    assert balance.kept_tokens(a, plan["perm"], 2, 2) == 17
    # rank0 = [9, 2], rank1 = [1, 5]: sorted [2(1), 1(2), 3(5), 0(9)] -> group0 {2, 3} (rank-1
    # data, 6), group1 {1, 0} (rank-0 data, 11): identity keeps 0, the swap keeps 17
    a = [9, 2, 1, 5]
    plan = balance.balance_paper(a, 2, 2)
    assert plan["perm"].tolist() == [2, 3, 1, 0]
    assert balance.kept_tokens(a, plan["perm"], 2, 2) == 0
    r = balance.relabel_locality(a, plan["perm"], 2, 2)
    assert r.tolist() == [1, 0, 2, 3] and balance.kept_tokens(a, r, 2, 2) == 17


@pytest.mark.parametrize("W", [2, 3, 4, 5, 6])
def test_relabel_locality_vs_hungarian_and_invariants(W):
    from scipy.optimize import linear_sum_assignment
    for seed in range(12):
        B = 7
        a = synth.skewed_rank_lengths(W, B, seed, "iid" if seed % 2 else "sorted-block").reshape(-1)
        for mode in ("paper", "snake", "lpt"):
            plan = {"paper": balance.balance_paper, "snake": balance.balance_snake,
                    "lpt": balance.balance_lpt}[mode](a, W, B)
            perm = plan["perm"]
            r = balance.relabel_locality(a, perm, W, B)
            # the optimum of the assignment problem, by an independent routine
            M = np.zeros((W, W))
            for i in range(W):
                for k in range(B):
                    g = int(perm[i * B + k])
                    M[i, g // B] += a[g]
            rows, cols = linear_sum_assignment(M, maximize=True)
            assert balance.kept_tokens(a, r, W, B) == int(M[rows, cols].sum())
            assert balance.kept_tokens(a, r, W, B) >= balance.kept_tokens(a, perm, W, B)
            # every group survives intact (same ids, same order), only its rank changes
            groups = sorted(tuple(int(x) for x in perm[i * B:(i + 1) * B]) for i in range(W))
            assert sorted(tuple(int(x) for x in r[i * B:(i + 1) * B]) for i in range(W)) == groups
            assert sorted(balance.plan_from_groups(a, W, B, [list(r[i * B:(i + 1) * B]) for i in range(W)])
                          ["rank_tokens"].tolist()) == sorted(plan["rank_tokens"].tolist())


# ---------------------------------------------------------------- stay-home balancing (R25, NEXT-2)
def test_balance_stay_hand_worked():
    """W=2, B=2: rank0 = [10, 2] (ids 0, 1), rank1 = [1, 3] (ids 2, 3); loads 12 / 4.
    Pairs x in rank0, y in rank1 with d > 0: (0,2) d=9 -> max(3, 13) = 13; (0,3) d=7 ->
    max(5, 11) = 11; (1,2) d=1 -> max(11, 5) = 11.  Best value 11, tie (0,3) vs (1,2) ->
    (0,3) first.  11 < 12: swap -> rank0 {3, 1} = 5, rank1 {2, 0} = 11.  Next: M = rank1,
    m = rank0: pairs x in {2, 0}, y in {3, 1}: (0,3) d=7 -> max(4, 12); (0,1) d=8 -> max(3,
    13); none beats 11.  Stop.  Sorted: rank0 [1 (2), 3 (3)], rank1 [2 (1), 0 (10)]."""
    p = balance.balance_stay([10, 2, 1, 3], 2, 2)
    assert p["perm"].tolist() == [1, 3, 2, 0]
    assert p["rank_tokens"].tolist() == [5, 11]


def test_balance_stay_invariants():
    for W in (1, 2, 3, 8):
        for seed in range(6):
            B = 56 if W == 8 else 9
            a = synth.skewed_rank_lengths(W, B, seed, "iid").reshape(-1)
            p = balance.balance_stay(a, W, B)
            perm = [int(x) for x in p["perm"]]
            assert sorted(perm) == list(range(W * B))                        # a permutation
            before = [int(a[r * B:(r + 1) * B].sum()) for r in range(W)]
            assert max(p["rank_tokens"]) <= max(before)                      # never worse than not moving
            moved = [g for r in range(W) for g in perm[r * B:(r + 1) * B] if g // B != r]
            assert len(moved) % 2 == 0 or W > 2                              # swaps move samples in pairs
            for r in range(W):                                               # rank order: (length, id)
                blk = perm[r * B:(r + 1) * B]
                assert blk == sorted(blk, key=lambda g: (a[g], g))
            if W == 1:
                assert moved == []
    # all lengths equal: nothing to balance, nothing moves
    p = balance.balance_stay([5] * 12, 3, 4)
    assert all(int(g) // 4 == r for r in range(3) for g in p["perm"][r * 4:(r + 1) * 4])
