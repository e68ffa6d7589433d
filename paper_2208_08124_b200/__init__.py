"""Unpadded-BERT data-parallel hot path for NVIDIA B200 (sm_100a).

arXiv 2208.08124 ("Boosting Distributed Training Performance of the Unpadded BERT
Model"): unpad/pad gather-scatter, varlen fused multi-head attention forward
and backward grouped by length, and the padding-exchange load
balancer.  The compute lives in libub.so (include/ub.h); this package is
its argument-marshalling binding.
"""
from ._lib import UbError
from .api import (Comm, balance_plan, balance_plan_weighted, cu_seqlens, dal_bwd, dal_fwd, embedding_bwd, embedding_fwd, encoder_attn_bwd, encoder_attn_fwd, linear_bwd, linear_fwd, exchange_copy, exchange_pull, exchange_pull_table, exchange_tables, ipc_close, ipc_export, ipc_import, set_checked, signal, validate_cu_seqlens,
                  wait_flags,
                  lengths_from_mask, pad, unpad, varlen_fmha_bwd, varlen_fmha_fwd, version)

__all__ = ["UbError", "Comm", "balance_plan", "balance_plan_weighted", "dal_bwd", "dal_fwd", "embedding_bwd", "embedding_fwd", "encoder_attn_bwd", "encoder_attn_fwd", "linear_bwd", "linear_fwd", "cu_seqlens", "exchange_copy", "exchange_pull", "exchange_pull_table", "exchange_tables", "ipc_close", "ipc_export", "ipc_import", "set_checked", "signal", "validate_cu_seqlens", "wait_flags", "lengths_from_mask", "pad",
           "unpad", "varlen_fmha_bwd", "varlen_fmha_fwd", "version"]
