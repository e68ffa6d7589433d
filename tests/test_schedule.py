"""ub_fmha_schedule (host LPT schedule of the persistent FMHA grids' work items): every item
exactly once, per-CTA lists in decreasing estimated cost, a makespan no worse than the kernels'
snake deal under the same cost model, determinism, argument checks.  (A performance-only
input: the GPU tests check that the kernels' results do not depend on it.)"""
import numpy as np
import pytest

import synth

H, S, G = 16, 512, 144


@pytest.fixture(scope="module")
def api():
    from paper_2208_08124_b200 import api
    return api


def _items(lengths, is_bwd):
    out = []
    for b, L in enumerate(lengths):
        nt = (int(L) + 127) // 128
        for h in range(H if nt else 0):
            if is_bwd:
                out.append(b * H + h)
            else:
                out += [(b * H + h) * 8 + g for g in range((nt + 1) // 2)]
    return out


def _cost(key, lengths, is_bwd):
    if is_bwd:
        nt = (int(lengths[key // H]) + 127) // 128
        return nt * nt + 0.3 * nt + 0.5
    bh, g = divmod(key, 8)
    nt = (int(lengths[bh // H]) + 127) // 128
    return (1.0 if nt - 2 * g >= 2 else 0.7) * nt + 0.3


def _lists(sched):
    g = int(sched[0])
    off = sched[1:g + 2]
    ent = sched[g + 2:]
    return [list(ent[off[c]:off[c + 1]]) for c in range(g)]


@pytest.mark.parametrize("is_bwd", [True, False])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_schedule_covers_every_item_once(api, is_bwd, seed):
    L = synth.gen_lengths("mlperf_like_v0", 56, seed)
    sched = api.fmha_schedule(L, H, S, G, is_bwd)
    lists = _lists(sched)
    assert int(sched[0]) == G and len(lists) == G
    got = sorted(k for lst in lists for k in lst)
    assert got == sorted(_items(L, is_bwd))
    for lst in lists:                                     # each CTA's items longest first
        c = [_cost(k, L, is_bwd) for k in lst]
        assert c == sorted(c, reverse=True)
        assert len(lst) <= 63


@pytest.mark.parametrize("is_bwd", [True, False])
def test_schedule_makespan_not_worse_than_snake(api, is_bwd):
    for seed in range(10):
        L = synth.gen_lengths("mlperf_like_v0", 56, seed)
        lists = _lists(api.fmha_schedule(L, H, S, G, is_bwd))
        lpt = max(sum(_cost(k, L, is_bwd) for k in lst) for lst in lists)
        # the kernels' deal: items longest first (stable), round r to CTA r*G + c or reversed
        items = sorted(_items(L, is_bwd), key=lambda k: -_cost(k, L, is_bwd))
        load = np.zeros(G)
        for i, k in enumerate(items):
            r, c = divmod(i, G)
            load[c if r % 2 == 0 else G - 1 - c] += _cost(k, L, is_bwd)
        assert lpt <= load.max() + 1e-9
        mean = sum(_cost(k, L, is_bwd) for k in items) / G
        assert lpt <= mean + max(_cost(k, L, is_bwd) for k in items)   # Graham's list-scheduling bound


def test_schedule_deterministic_and_edge_lengths(api):
    L = np.array([0, 1, 128, 129, 512, 0, 300], np.int32)
    a = api.fmha_schedule(L, 2, 512, 5, True)
    b = api.fmha_schedule(L, 2, 512, 5, True)
    assert np.array_equal(a, b)
    assert sorted(k for lst in _lists(a) for k in lst) == [b_ * 2 + h for b_ in (1, 2, 3, 4, 6) for h in range(2)]


def test_schedule_rejects(api):
    from paper_2208_08124_b200 import UbError
    with pytest.raises(UbError):                          # length above max_seqlen
        api.fmha_schedule([600], 2, 512, 4, True)
    with pytest.raises(UbError):                          # more than 63 items on a CTA
        api.fmha_schedule([128] * 400, 1, 128, 2, True)
    with pytest.raises(UbError):                          # buffer too small
        api.fmha_schedule([100], 2, 512, 4, True, out=np.zeros(3, np.int32))
