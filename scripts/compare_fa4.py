"""Context only: time the image's FlashAttention-4 CuTe-DSL varlen kernels
(vllm.vllm_flash_attn.cute, library code) on the same config-2 batch as bench.py, beside this
library's kernels.  Never a dependency of the product or of any test.

    python scripts/compare_fa4.py            (on the GPU box)
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2208_08124_b200 as ub  # noqa: E402


def timeit(fn, iters=50, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts))


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    H, D, S = 16, 64, 512
    lengths = synth.gen_lengths("mlperf_like_v0", 56, 0)
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
    T = int(off[-1])
    cu = torch.from_numpy(off).to(dev)
    qkv = torch.randn(T, 3, H, D, device=dev, dtype=torch.bfloat16)
    dout = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)
    scale = 1.0 / math.sqrt(D)
    res = {"T": T, "sum_L2": int((lengths.astype(np.int64) ** 2).sum())}

    o, lse = ub.varlen_fmha_fwd(qkv, cu, S, scale, 0.0, 0, 0)
    res["ub_fwd_us"] = timeit(lambda: ub.varlen_fmha_fwd(qkv, cu, S, scale, 0.0, 0, 0))
    res["ub_bwd_us"] = timeit(lambda: ub.varlen_fmha_bwd(qkv, o, lse, dout, cu, S, scale, 0.0, 0, 0))

    try:
        from vllm.vllm_flash_attn.cute import interface as fa
        q, k, v = qkv[:, 0], qkv[:, 1], qkv[:, 2]
        kw = dict(cu_seqlens_q=cu, cu_seqlens_k=cu, max_seqlen_q=S, max_seqlen_k=S, softmax_scale=scale)
        out, lse4 = fa._flash_attn_fwd(q, k, v, return_lse=True, **kw)
        res["fa4_fwd_us"] = timeit(lambda: fa._flash_attn_fwd(q, k, v, return_lse=True, **kw))

        def bwd():
            return fa._flash_attn_bwd(q, k, v, out, dout, lse4, scale, False, 0.0, cu_seqlens_q=cu,
                                      cu_seqlens_k=cu, max_seqlen_q=S, max_seqlen_k=S)
        bwd()
        res["fa4_bwd_us"] = timeit(bwd)
        ref_o = o.float()
        res["fa4_vs_ub_fwd_maxabs"] = float((out.float() - ref_o).abs().max())
    except Exception as ex:  # context only
        res["fa4_error"] = repr(ex)[:400]
    try:
        from flash_attn import flash_attn_varlen_qkvpacked_func as fa2
        qkvr = qkv.clone().requires_grad_(True)

        def f2():
            return fa2(qkvr, cu, S, softmax_scale=scale)
        res["fa2_fwd_us"] = timeit(f2)
        y = f2()
        res["fa2_fwd_bwd_us"] = timeit(lambda: torch.autograd.grad(f2(), qkvr, dout))
    except Exception as ex:
        res["fa2_error"] = repr(ex)[:400]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
