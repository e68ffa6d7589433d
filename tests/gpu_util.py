"""Helpers for the -m gpu parity tests: seeded inputs (synth), oracle comparisons."""
import numpy as np
import torch

import synth
from oracle import attention as oatt
from oracle import varlen as ovar

TOL_MAX_ABS = 2e-2    # BASELINE north_star: max-abs-error 2e-2 ...
TOL_REL_L2 = 1e-2     # ... and relative-L2 1e-2 for bf16 attention
TOL_LSE = 1e-2        # our addition (R7)


def make_batch(lengths, H, D, dtype=torch.bfloat16, seed=1000):
    lengths = np.asarray(lengths, dtype=np.int32)
    off = ovar.batch_offset(lengths)
    T = int(off[-1])
    qkv = synth.gen_normal((T, 3, H, D), seed, dtype)
    dout = synth.gen_normal((T, H, D), seed + 1000, dtype)
    return lengths, off, qkv, dout


def to_dev(x):
    return x.cuda()


def errors(got, exp):
    got = np.asarray(got, dtype=np.float64)
    exp = np.asarray(exp, dtype=np.float64)
    max_abs = float(np.max(np.abs(got - exp))) if got.size else 0.0
    ne = np.linalg.norm(exp)
    # rel-L2 is undefined for an exactly-zero reference (e.g. dQ of a 1-token sequence):
    # there only the max-abs bound applies
    rel = float(np.linalg.norm(got - exp) / ne) if got.size and ne > 1e-6 else 0.0
    return max_abs, rel


def assert_close(got, exp, what, max_abs=TOL_MAX_ABS, rel_l2=TOL_REL_L2):
    a, r = errors(got, exp)
    assert a <= max_abs and r <= rel_l2, f"{what}: max_abs={a:.3e} rel_l2={r:.3e}"
    return a, r


def oracle_seq_slice(qkv_cpu, dout_cpu, off, seqs, scale, p=0.0, seed=0, offset=0, bwd=True):
    """Oracle on a subset of sequences (absolute dropout coordinates kept via t_base).
    Returns {b: (O [L,H,D], LSE [H,L], dqkv [L,3,H,D] or None)}."""
    out = {}
    q64 = qkv_cpu.double().numpy()
    g64 = dout_cpu.double().numpy() if dout_cpu is not None else None
    for b in seqs:
        s, e = int(off[b]), int(off[b + 1])
        sub_off = np.array([0, e - s])
        O, LSE = oatt.varlen_fwd(q64[s:e], sub_off, e - s, scale, p, seed, offset, t_base=s)
        d = oatt.varlen_bwd(q64[s:e], g64[s:e], sub_off, e - s, scale, p, seed, offset, t_base=s) if bwd else None
        out[b] = (O, LSE, d)
    return out
