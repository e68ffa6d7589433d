"""Pins for oracle.encoder (NEXT-1 encoder attention sub-layer) -- CPU only: torch fp64
autograd of the same composition from torch's own SDPA and layer_norm."""
import numpy as np
import torch

from oracle import dal as odal
from oracle import encoder as oenc
from oracle import varlen as ovar


def _params(hid, seed):
    rng = np.random.default_rng(seed)
    s = 1.0 / np.sqrt(hid)
    return (rng.standard_normal((3 * hid, hid)) * s, 0.1 * rng.standard_normal(3 * hid), rng.standard_normal((hid, hid)) * s,
            0.1 * rng.standard_normal(hid), 1.0 + 0.1 * rng.standard_normal(hid), 0.1 * rng.standard_normal(hid))


def test_matches_torch_autograd_composition():
    lengths = np.array([3, 7, 1, 5], np.int32)
    off = ovar.batch_offset(lengths)
    T, hid, H, S = int(off[-1]), 32, 4, 8
    D = hid // H
    rng = np.random.default_rng(1)
    x, dy = rng.standard_normal((T, hid)), rng.standard_normal((T, hid))
    wq, bq, wo, bo, g, b = _params(hid, 2)
    p_hidden, eps, seed = 0.2, 1e-12, 11
    y, saved = oenc.encoder_attn_fwd(x, off, S, wq, bq, wo, bo, g, b, H, 0.0, p_hidden, eps, seed)
    grads = oenc.encoder_attn_bwd(dy, x, off, S, wq, wo, g, saved, H, 0.0, p_hidden, eps, seed)

    t = {k: torch.tensor(v, requires_grad=True) for k, v in
         dict(x=x, wq=wq, bq=bq, wo=wo, bo=bo, g=g, b=b).items()}
    qkv = t["x"] @ t["wq"].T + t["bq"]
    ctx = []
    for i in range(len(lengths)):
        s, e = int(off[i]), int(off[i + 1])
        q, k, v = (qkv[s:e].reshape(e - s, 3, H, D)[:, j].transpose(0, 1) for j in range(3))
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, scale=1.0 / np.sqrt(D))
        ctx.append(o.transpose(0, 1).reshape(e - s, hid))
    a = torch.cat(ctx) @ t["wo"].T + t["bo"]
    keep = torch.tensor(odal.dal_keep_mask(seed, 0, T, hid, p_hidden), dtype=torch.float64)
    ty = torch.nn.functional.layer_norm(t["x"] + a * keep * odal.dal_dropout_scale(p_hidden), (hid,), t["g"], t["b"], eps)
    ty.backward(torch.tensor(dy))
    assert np.allclose(y, ty.detach().numpy(), atol=1e-10)
    for name, key in (("dx", "x"), ("dw_qkv", "wq"), ("db_qkv", "bq"), ("dw_o", "wo"), ("db_o", "bo"),
                      ("dgamma", "g"), ("dbeta", "b")):
        assert np.allclose(grads[name], t[key].grad.numpy(), atol=1e-9), name


def test_bf16_storage_rounding_only_perturbs():
    """round_bf16 models the device's storage precision: close to the exact composition, not equal."""
    lengths = np.array([20, 9], np.int32)
    off = ovar.batch_offset(lengths)
    T, hid, H = int(off[-1]), 64, 1
    rng = np.random.default_rng(3)
    x = rng.standard_normal((T, hid))
    wq, bq, wo, bo, g, b = _params(hid, 4)
    y0, _ = oenc.encoder_attn_fwd(x, off, 32, wq, bq, wo, bo, g, b, H)
    y1, _ = oenc.encoder_attn_fwd(x, off, 32, wq, bq, wo, bo, g, b, H, round_bf16=True)
    err = np.abs(y1 - y0).max()
    assert 0 < err < 5e-2
