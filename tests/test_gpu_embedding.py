"""GPU parity of the unpadded embedding fwd/bwd (NEXT-4) vs the fp64 oracle."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import assert_close
from oracle import embedding as oemb
from oracle import varlen as ovar

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as m
    return m


def _batch(lengths, vocab, seed):
    """Zipf-like token ids (hot tokens hit the same gradient rows many times, as [CLS] /
    [SEP] and frequent words do), positions 0..L-1 per packed sequence, two segments."""
    rng = np.random.default_rng(seed)
    off = ovar.batch_offset(np.asarray(lengths, np.int32))
    T = int(off[-1])
    ids = np.minimum(rng.zipf(1.2, T) - 1, vocab - 1).astype(np.int32)
    ids[off[:-1]] = 101                                   # a [CLS]-like token opening every sequence
    pos = oemb.packed_positions(off).astype(np.int32)
    seg = (rng.random(T) < 0.5).astype(np.int32)
    return off, T, ids, pos, seg


@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_embedding_fwd_bwd(ub, gdt):
    lengths = synth.gen_lengths("mlperf_like_v0", 20, 3)
    V, P, E = 30522, 512, 1024
    off, T, ids, pos, seg = _batch(lengths, V, 1)
    w_word = (0.02 * synth.gen_normal((V, E), 2)).to(torch.bfloat16)
    w_pos = (0.02 * synth.gen_normal((P, E), 3)).to(torch.bfloat16)
    w_type = (0.02 * synth.gen_normal((2, E), 4)).to(torch.bfloat16)
    dout = synth.gen_normal((T, E), 5)
    d = lambda a: torch.from_numpy(a).cuda()
    out = ub.embedding_fwd(d(ids), d(pos), d(seg), w_word.cuda(), w_pos.cuda(), w_type.cuda())
    dw = [torch.zeros((n, E), dtype=gdt, device="cuda") for n in (V, P, 2)]
    ub.embedding_bwd(dout.cuda(), d(ids), d(pos), d(seg), *dw)
    torch.cuda.synchronize()
    f = lambda t: t.double().numpy()
    ref = oemb.embedding_fwd(ids, pos, seg, f(w_word), f(w_pos), f(w_type))
    assert_close(out.float().cpu().numpy(), ref, "out")
    DW = oemb.embedding_bwd(f(dout), ids, pos, seg, V, P, 2)
    for got, exp, name in zip(dw, DW, ("dW_word", "dW_pos", "dW_type")):
        g = got.float().cpu().numpy()
        rows = np.unique(np.concatenate([ids, pos, seg])) if name == "dW_word" else np.arange(exp.shape[0])
        if gdt == torch.float32:
            # fp32 sums of up to T bf16 rows: error ~ sqrt(count) * 2^-24 * |sum|
            assert np.max(np.abs(g - exp) / np.maximum(1.0, np.abs(exp))) < 1e-4, name
        else:
            # bf16 accumulation (the paper's packed-atomic form): every add rounds to bf16, so
            # the error grows like sqrt(adds) * 2^-9 (R23) -- the fp32 form is the accurate one
            idx = {"dW_word": ids, "dW_pos": pos, "dW_type": seg}[name]
            adds = np.bincount(idx).max()
            rel = np.linalg.norm(g - exp) / np.linalg.norm(exp)
            assert rel < 4 * 2.0 ** -9 * np.sqrt(adds), (name, rel, adds)
        untouched = np.setdiff1d(np.arange(exp.shape[0]), np.unique({"dW_word": ids, "dW_pos": pos, "dW_type": seg}[name]))
        assert np.all(g[untouched] == 0.0), name
