"""ORACLE -- test infrastructure only.

A plain, slow, obviously-correct CPU implementation (numpy, fp64) of what the
unpadded-BERT hot path computes, written from the paper (arXiv 2208.08124,
`/root/reference/PAPER.md`, cited as P:<line>) and the readings listed in
DESIGN.md §2.  It shares no code with the CUDA path (`paper_2208_08124_b200/`)
and neither imports the other; only `synth/` (seeded random draws, no method
arithmetic) feeds both.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`.  The product path
never calls it: there is no CPU fallback.

Modules:
  varlen     -- batch_offset (cu_seqlens), unpad gather, pad scatter, nonzero_indices
                
  attention  -- padded-masked multi-head attention Eq. (1) forward, its analytic
                backward, and the per-sequence unpadded form
  philox     -- Philox4x32-10 counter-based RNG and the attention-dropout keep mask
                (our convention; the paper is silent -- DESIGN.md reading R5)
  balance    -- the padding-exchange balancer: sort by valid tokens + interleave slice
                (P:355-359), the snake variant, and brute-force optimal search
  exchange   -- in-process simulation of all-gather + redistribution of sample payloads
                

Parity status of every function is stated in its module header; every function is
pinned by a `-m "not gpu"` test in tests/test_oracle_*.py (none is "parity unpinned").
"""
