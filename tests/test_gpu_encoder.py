"""GPU parity of the Linear layers (cuBLASLt) and the unpadded encoder
attention sub-layer (NEXT-1) against the fp64 oracle."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import assert_close
from oracle import encoder as oenc
from oracle import varlen as ovar

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as m
    return m


def _close_scaled(got, exp, what):
    """Composed layer (reading R22): |got - exp| <= 2e-2 * max(1, |exp|) elementwise and
    rel-L2 <= 1e-2 -- four bf16-stored intermediates make the error relative to magnitude."""
    got = np.asarray(got, np.float64)
    e = float(np.max(np.abs(got - exp) / np.maximum(1.0, np.abs(exp))))
    r = _rel(got, exp)
    assert e <= 2e-2 and r <= 1e-2, f"{what}: scaled max {e:.3e} rel_l2 {r:.3e}"


def _rel(got, exp):
    return float(np.linalg.norm(np.asarray(got, np.float64) - exp) / max(np.linalg.norm(exp), 1e-30))


def test_linear_fwd_bwd(ub):
    T, K, N = 333, 256, 384
    x = synth.gen_normal((T, K), 1)
    W = (synth.gen_normal((N, K), 2) * (1.0 / np.sqrt(K))).to(torch.bfloat16)
    b = synth.gen_normal((N,), 3)
    dy = synth.gen_normal((T, N), 4)
    r = synth.gen_normal((T, K), 5)
    xd, Wd, bd, dyd, rd = x.cuda(), W.cuda(), b.cuda(), dy.cuda(), r.cuda()
    y = ub.linear_fwd(xd, Wd, bd)
    dx, dW, db = ub.linear_bwd(dyd, xd, Wd, rd)
    torch.cuda.synchronize()
    f = lambda t: t.double().numpy()
    assert_close(y.float().cpu().numpy(), f(x) @ f(W).T + f(b), "y")
    assert_close(dx.float().cpu().numpy(), f(dy) @ f(W) + f(r), "dx (+ residual via beta)")
    assert _rel(dW.cpu().numpy(), f(dy).T @ f(x)) < 1e-3
    assert _rel(db.cpu().numpy(), f(dy).sum(axis=0)) < 1e-4


@pytest.mark.parametrize("lengths,p_attn,p_hidden", [([3, 130, 64, 200], 0.0, 0.0), ([512, 1, 77, 300, 129], 0.1, 0.1)])
def test_encoder_attn_sublayer(ub, lengths, p_attn, p_hidden):
    lengths = np.asarray(lengths, np.int32)
    off = ovar.batch_offset(lengths)
    T, hid, H, S = int(off[-1]), 1024, 16, 512
    s = 1.0 / np.sqrt(hid)
    x = synth.gen_normal((T, hid), 10)
    wq = (synth.gen_normal((3 * hid, hid), 11) * s).to(torch.bfloat16)
    bq = (0.1 * synth.gen_normal((3 * hid,), 12)).to(torch.bfloat16)
    wo = (synth.gen_normal((hid, hid), 13) * s).to(torch.bfloat16)
    bo = (0.1 * synth.gen_normal((hid,), 14)).to(torch.bfloat16)
    g = (1.0 + 0.1 * synth.gen_normal((hid,), 15)).to(torch.bfloat16)
    b = (0.1 * synth.gen_normal((hid,), 16)).to(torch.bfloat16)
    dy = synth.gen_normal((T, hid), 17)
    seed, eps = 0x2208, 1e-12
    cu = torch.tensor(off.astype(np.int32)).cuda()
    dev = [t.cuda() for t in (x, wq, bq, wo, bo, g, b, dy)]
    y, saved = ub.encoder_attn_fwd(dev[0], cu, S, dev[1], dev[2], dev[3], dev[4], dev[5], dev[6], H, p_attn, p_hidden,
                                   eps, seed)
    grads = ub.encoder_attn_bwd(dev[7], dev[0], cu, S, dev[1], dev[3], dev[5], saved, H, p_attn, p_hidden, eps, seed)
    torch.cuda.synchronize()
    f = lambda t: t.double().numpy()
    Y, sv = oenc.encoder_attn_fwd(f(x), off, S, f(wq), f(bq), f(wo), f(bo), f(g), f(b), H, p_attn, p_hidden, eps, seed,
                                  round_bf16=True)
    G = oenc.encoder_attn_bwd(f(dy), f(x), off, S, f(wq), f(wo), f(g), sv, H, p_attn, p_hidden, eps, seed,
                              round_bf16=True)
    _close_scaled(saved["qkv"].float().cpu().numpy(), sv["qkv"], "qkv")
    _close_scaled(saved["ctx"].float().cpu().numpy(), sv["ctx"], "ctx")
    _close_scaled(y.float().cpu().numpy(), Y, "y")
    _close_scaled(grads["dx"].float().cpu().numpy(), G["dx"], "dx")
    for k in ("dw_qkv", "db_qkv", "dw_o", "db_o", "dgamma", "dbeta"):
        assert _rel(grads[k].cpu().numpy(), G[k]) < 2e-2, k
