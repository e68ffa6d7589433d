"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no prefix sums, no attention, no
balancing): it only draws random numbers with named generators, so that the oracle
(`oracle/`) and the CUDA path (`paper_2208_08124_b200/`) can be fed byte-identical
inputs without sharing any computation.  Recipes are stated in DESIGN.md §3.

Length distributions:
  * ``mlperf_like_v0`` -- P(L=512)=0.232 (the only number the paper prints about the
    Wikipedia length histogram, §III-C-1) and a linear ramp
    P(L)=0.768*(512-L)/130816 for L=1..511 (a synthetic stand-in: the figure's
    histogram is not in the text).  E[L]=250.1.
  * ``uniform``  -- L ~ U{1..512}.
  * ``bimodal``  -- exactly half 64, half 512 (shuffled).
All draws use numpy's PCG64 (``numpy.random.default_rng(seed)``) by inverse CDF.

Values: q, k, v, dO ~ N(0,1) drawn in fp32 by a seeded ``torch.Generator`` (CPU,
Philox-free mt19937) and rounded to bf16 (round-to-nearest-even) for the bf16 path.
"""
from __future__ import annotations

import numpy as np
import torch

MAX_SEQLEN = 512
DISTRIBUTIONS = ("mlperf_like_v0", "uniform", "bimodal")


def length_pmf(dist: str, max_seqlen: int = MAX_SEQLEN) -> np.ndarray:
    """Probability mass over L = 1..max_seqlen (index L-1)."""
    L = np.arange(1, max_seqlen + 1, dtype=np.float64)
    if dist == "mlperf_like_v0":
        if max_seqlen != 512:
            raise ValueError("mlperf_like_v0 is defined at max_seqlen 512")
        pmf = 0.768 * (512.0 - L) / 130816.0
        pmf[-1] = 0.232
    elif dist == "uniform":
        pmf = np.full(max_seqlen, 1.0 / max_seqlen)
    else:
        raise ValueError(f"no pmf for distribution {dist!r}")
    return pmf


def gen_lengths(dist: str, n: int, seed: int, max_seqlen: int = MAX_SEQLEN) -> np.ndarray:
    """n sequence lengths (int32, each in [1, max_seqlen]) drawn with PCG64(seed)."""
    rng = np.random.default_rng(seed)
    if dist == "bimodal":
        out = np.where(np.arange(n) < n // 2, 64, max_seqlen).astype(np.int32)
        rng.shuffle(out)
        return out
    pmf = length_pmf(dist, max_seqlen)
    cdf = np.cumsum(pmf)
    cdf[-1] = 1.0
    u = rng.random(n)
    return (np.searchsorted(cdf, u, side="right") + 1).astype(np.int32)


def gen_normal(shape, seed: int, dtype=torch.bfloat16) -> torch.Tensor:
    """N(0,1) fp32 draw with torch.Generator(seed) on CPU, cast (RNE) to ``dtype``."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return torch.randn(tuple(shape), generator=g, dtype=torch.float32).to(dtype)


def gen_bytes(nbytes: int, seed: int) -> np.ndarray:
    """Uniform random bytes (uint8) with PCG64(seed) -- opaque payload records."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=int(nbytes), dtype=np.uint8)


def gen_padded_mask(lengths, max_seqlen: int) -> np.ndarray:
    """[B, max_seqlen] 0/1 prefix mask (input_mask of PAPER.md:355) for given lengths."""
    lengths = np.asarray(lengths)
    return (np.arange(max_seqlen)[None, :] < lengths[:, None]).astype(np.int32)


def skewed_rank_lengths(world: int, batch: int, step: int, mode: str = "iid",
                        dist: str = "mlperf_like_v0") -> np.ndarray:
    """Per-rank lengths [world, batch] for the balanced-DP config (BASELINE config 3).

    ``iid``: every rank draws its own batch (seed 100+step).  ``sorted-block``: the
    world*batch draws are sorted and rank r receives block r (the worst case for
    unbalanced all-reduce, §III-C-2).
    """
    draws = gen_lengths(dist, world * batch, 100 + step)
    if mode == "sorted-block":
        draws = np.sort(draws, kind="stable")
    elif mode != "iid":
        raise ValueError(mode)
    return draws.reshape(world, batch).astype(np.int32)


def gen_normal_device(shape, seed: int, device, dtype=torch.bfloat16) -> torch.Tensor:
    """N(0,1) drawn on the GPU with a seeded torch CUDA generator (Philox), rounded to
    ``dtype`` -- for large benchmark buffers where a CPU draw would dominate set-up time.
    Parity tests use the CPU draw (gen_normal)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return torch.randn(tuple(shape), generator=g, device=device, dtype=torch.float32).to(dtype)
