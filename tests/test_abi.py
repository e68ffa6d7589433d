"""The C-ABI library loads, exports every symbol include/ub.h declares, and its host-side
functions (no GPU needed) match the oracle bit-exactly.  CPU only."""
import os
import re

import numpy as np
import pytest

from oracle import balance as obal
from oracle import exchange as oex
from oracle import varlen as ovar
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ub():
    from paper_2208_08124_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2208_08124_b200 import build
        build.build()
    return _lib


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ub.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ub_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(ub):
    L = ub.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
        assert name in ub.SIGNATURES, f"binding lacks {name}"
    assert "sm_100a" in L.ub_version().decode()


def test_dropout_effective_p(ub):
    """The applied drop rates (R5 8-bit, R21 16-bit) agree with the oracle's thresholds."""
    from oracle import dal as odal
    from oracle import philox
    from paper_2208_08124_b200 import api
    for p in (0.0, 0.1, 0.25, 0.5, 1.0 / 3.0, 0.9):
        assert api.dropout_effective_p(p, 8) == philox.dropout_threshold(p) / 256.0
        assert api.dropout_effective_p(p, 16) == (odal.dal_threshold(p) / 65536.0 if p > 0 else 0.0)
    assert api.dropout_effective_p(0.001, 8) == 0.0      # rejected by the FMHA entry points


def test_cu_seqlens_and_errors(ub, golden):
    from paper_2208_08124_b200 import api
    for ex in golden["spec_worked_examples"]["batch_offset"]:
        assert api.cu_seqlens(ex["lengths"], 512).tolist() == ex["offsets"]
    L = synth.gen_lengths("mlperf_like_v0", 300, 4)
    assert np.array_equal(api.cu_seqlens(L, 512), ovar.batch_offset(L))
    with pytest.raises(ub.UbError) as e:
        api.cu_seqlens([3, 0], 512)
    assert e.value.status == 1
    with pytest.raises(ub.UbError) as e:
        api.cu_seqlens([3, 600], 512)
    assert e.value.status == 3
    with pytest.raises(ub.UbError):
        api.cu_seqlens([], 512)


def test_lengths_from_mask(ub, golden):
    from paper_2208_08124_b200 import api
    ex = golden["spec_worked_examples"]["unpad"][0]
    assert api.lengths_from_mask(ex["mask"]).tolist() == [2, 3]
    with pytest.raises(ub.UbError) as e:
        api.lengths_from_mask([[1, 0, 1]])
    assert e.value.status == 2


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_balance_plan_paper_and_snake_bit_exact(ub, W):
    from paper_2208_08124_b200 import api
    for step in range(5):
        for skew in ("iid", "sorted-block"):
            a = synth.skewed_rank_lengths(W, 56, step, skew).reshape(-1)
            for mode, ref in (("paper", obal.balance_paper), ("snake", obal.balance_snake)):
                got = api.balance_plan(a, W, 56, 512, mode)
                exp = ref(a, W, 56)
                for k in ("perm", "rank_tokens", "send_samples", "send_tokens"):
                    assert np.array_equal(got[k], exp[k]), (mode, k)


def test_balance_plan_exact_small_bit_exact(ub):
    from paper_2208_08124_b200 import api
    rng = np.random.default_rng(0)
    for W, B in [(1, 4), (2, 1), (2, 2), (2, 3), (3, 2), (2, 4), (3, 3), (4, 2), (2, 5), (4, 3), (3, 4), (6, 2)]:
        for _ in range(3):
            a = rng.integers(1, 40, size=W * B)
            got = api.balance_plan(a, W, B, 512, "exact_small")
            exp = obal.balance_opt(a, W, B)
            assert np.array_equal(got["perm"], exp["perm"]), (W, B, a)
            assert got["rank_tokens"].max() == exp["opt_max_tokens"]
    with pytest.raises(ub.UbError) as e:
        api.balance_plan(np.ones(13, np.int32), 13, 1, 512, "exact_small")
    assert e.value.status == 5
    with pytest.raises(ub.UbError) as e:
        api.balance_plan([1, 2, 0, 4], 2, 2, 512)
    assert e.value.status == 1
    with pytest.raises(ub.UbError) as e:
        api.balance_plan([1, 2, 513, 4], 2, 2, 512)
    assert e.value.status == 3


def test_balance_plan_lpt_bit_exact(ub):
    """UB_BAL_LPT and ub_balance_plan_weighted vs oracle balance_lpt (R20), bit-exact."""
    from paper_2208_08124_b200 import api
    rng = np.random.default_rng(5)
    for W in (1, 2, 3, 8):
        for B in (1, 2, 7, 56):
            for _ in range(3):
                a = rng.integers(1, 513, size=W * B).astype(np.int32)
                got = api.balance_plan(a, W, B, 512, "lpt")
                exp = obal.balance_lpt(a, W, B)
                for k in ("perm", "rank_tokens", "send_samples", "send_tokens"):
                    assert np.array_equal(np.asarray(got[k], np.int64), np.asarray(exp[k], np.int64)), (W, B, k)
                gw = api.balance_plan_weighted(a, W, B, 512, 2048, 1)
                ew = obal.balance_lpt(a, W, B, alpha=2048, beta=1)
                assert np.array_equal(gw["perm"].astype(np.int64), ew["perm"]) and np.array_equal(gw["rank_cost"], ew["rank_cost"])
    from paper_2208_08124_b200 import UbError
    with pytest.raises(UbError):
        api.balance_plan_weighted([1, 2], 2, 1, 512, 0, 0)


def test_balance_plan_stay_bit_exact(ub):
    """UB_BAL_STAY vs oracle balance_stay (R25), bit-exact (perm, loads, send matrices)."""
    from paper_2208_08124_b200 import api
    rng = np.random.default_rng(13)
    for W in (1, 2, 3, 8):
        for B in (1, 2, 7, 56):
            for trial in range(3):
                a = rng.integers(1, 513, size=W * B).astype(np.int32) if trial < 2 else \
                    synth.skewed_rank_lengths(W, B, trial, "iid").reshape(-1).astype(np.int32)
                got = api.balance_plan(a, W, B, 512, "stay")
                exp = obal.balance_stay(a, W, B)
                for k in ("perm", "rank_tokens", "send_samples", "send_tokens"):
                    assert np.array_equal(np.asarray(got[k], np.int64), np.asarray(exp[k], np.int64)), (W, B, k)


def test_balance_relabel_locality_bit_exact(ub):
    """ub_balance_relabel (DP over rank subsets) and the UB_BAL_LOCALITY flag vs the oracle's
    exhaustive relabel_locality (R24), bit-exact, incl. ties (equal lengths everywhere)."""
    from paper_2208_08124_b200 import api
    rng = np.random.default_rng(9)
    for W in (1, 2, 3, 5, 8):
        for B in (1, 3, 56):
            for trial in range(3):
                a = (np.full(W * B, 7, np.int32) if trial == 2 else rng.integers(1, 513, size=W * B).astype(np.int32))
                if trial == 1:
                    a = synth.skewed_rank_lengths(W, B, 3, "sorted-block").reshape(-1).astype(np.int32)
                for mode in ("paper", "snake", "lpt"):
                    base = api.balance_plan(a, W, B, 512, mode)
                    exp = obal.relabel_locality(a, base["perm"], W, B)
                    got, kb, ka = api.balance_relabel(a, base["perm"], W, B)
                    assert np.array_equal(got.astype(np.int64), exp), (W, B, mode)
                    assert kb == obal.kept_tokens(a, base["perm"], W, B) and ka == obal.kept_tokens(a, exp, W, B)
                    flag = api.balance_plan(a, W, B, 512, mode + "+locality")
                    assert np.array_equal(flag["perm"].astype(np.int64), exp)
                    assert sorted(flag["rank_tokens"].tolist()) == sorted(base["rank_tokens"].tolist())
    from paper_2208_08124_b200 import UbError
    with pytest.raises(UbError) as e:
        api.balance_relabel(np.ones(4, np.int32), [0, 0, 1, 2], 2, 2)
    assert e.value.status == 4


def test_exchange_tables_reproduce_oracle_exchange(ub):
    """Apply the library's pack/unpack tables with plain numpy copies (the device kernel
    only follows the table) and compare the bytes every rank ends with to the oracle."""
    from paper_2208_08124_b200 import api
    W, B, rec, srec = 4, 7, 16, 4
    lens = synth.gen_lengths("mlperf_like_v0", W * B, 9).reshape(W, B)
    toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 50 + r).reshape(-1, rec) for r in range(W)]
    smps = [synth.gen_bytes(B * srec, 60 + r).reshape(B, srec) for r in range(W)]
    plan = api.balance_plan(lens.reshape(-1), W, B, 512, "paper")
    exp = oex.exchange(lens, toks, smps, plan["perm"], W, B)

    def apply(tab, src_t, src_s, T_out):
        dst_t = np.zeros((T_out, rec), np.uint8)
        dst_s = np.zeros((B, srec), np.uint8)
        for e in range(B):
            s0, n, d0, ss, ds = (int(tab[k * B + e]) for k in range(5))
            dst_t[d0:d0 + n] = src_t[s0:s0 + n]
            dst_s[ds] = src_s[ss]
        return dst_t, dst_s

    send = []
    for r in range(W):
        tab, cnt, scnt, tot = api.exchange_tables(lens.reshape(-1), plan["perm"], W, B, r, unpack=False)
        assert tot == lens[r].sum() and cnt.sum() == tot and scnt.sum() == B
        st, ss = apply(tab, toks[r], smps[r], tot)
        send.append((st, ss, cnt, scnt))
    for d in range(W):
        # transport: concatenation of every source's slice for d, sources ascending
        chunks_t, chunks_s = [], []
        for s in range(W):
            st, ss, cnt, scnt = send[s]
            o = int(cnt[:d].sum()); so = int(scnt[:d].sum())
            chunks_t.append(st[o:o + cnt[d]]); chunks_s.append(ss[so:so + scnt[d]])
        recv_t, recv_s = np.concatenate(chunks_t), np.concatenate(chunks_s)
        tab, cnt, scnt, tot = api.exchange_tables(lens.reshape(-1), plan["perm"], W, B, d, unpack=True)
        assert tot == plan["rank_tokens"][d]
        out_t, out_s = apply(tab, recv_t, recv_s, tot)
        assert np.array_equal(out_t, exp[d]["tokens"])
        assert np.array_equal(out_s, exp[d]["samples"])


@pytest.mark.parametrize("W,B", [(1, 5), (2, 7), (4, 7), (8, 3)])
def test_exchange_pull_table_reproduces_oracle_exchange(ub, W, B):
    """NEXT-3: apply the pull table (each output sample copied straight out of its source
    rank's packed batch) with numpy and compare every rank's bytes with the oracle."""
    from paper_2208_08124_b200 import api
    rec, srec = 16, 4
    lens = synth.gen_lengths("mlperf_like_v0", W * B, 10 + W).reshape(W, B)
    toks = [synth.gen_bytes(int(lens[r].sum()) * rec, 70 + r).reshape(-1, rec) for r in range(W)]
    smps = [synth.gen_bytes(B * srec, 80 + r).reshape(B, srec) for r in range(W)]
    plan = api.balance_plan(lens.reshape(-1), W, B, 512, "paper")
    exp = oex.exchange(lens, toks, smps, plan["perm"], W, B)
    for d in range(W):
        tab, tot = api.exchange_pull_table(lens.reshape(-1), plan["perm"], W, B, d)
        assert tot == plan["rank_tokens"][d]
        out_t = np.zeros((tot, rec), np.uint8)
        out_s = np.zeros((B, srec), np.uint8)
        for e in range(B):
            src, s0, n, d0, ss, ds = (int(tab[k * B + e]) for k in range(6))
            out_t[d0:d0 + n] = toks[src][s0:s0 + n]
            out_s[ds] = smps[src][ss]
        assert np.array_equal(out_t, exp[d]["tokens"]) and np.array_equal(out_s, exp[d]["samples"])
    from paper_2208_08124_b200 import UbError
    bad = plan["perm"].copy()
    bad[0] = bad[1]
    with pytest.raises(UbError):
        api.exchange_pull_table(lens.reshape(-1), bad, W, B, 0)
