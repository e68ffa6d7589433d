"""ctypes loader for libub.so (the C ABI of include/ub.h).  Fails loudly if the library is
missing: there is no fallback implementation of anything."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UB_LIB", os.path.join(_HERE, "libub.so"))

UB_OK = 0
STATUS_NAMES = {0: "UB_OK", 1: "UB_ERR_INVALID_ARG", 2: "UB_ERR_INVALID_MASK", 3: "UB_ERR_CAPACITY",
                4: "UB_ERR_SHAPE", 5: "UB_ERR_UNSUPPORTED", 6: "UB_ERR_CUDA", 7: "UB_ERR_NCCL"}
UB_BF16, UB_FP32 = 0, 1
UB_IPC_HANDLE_BYTES = 128
UB_COMM_FORCE_NCCL = 1
UB_BAL_PAPER, UB_BAL_SNAKE, UB_BAL_EXACT_SMALL, UB_BAL_LPT, UB_BAL_STAY = 0, 1, 2, 3, 4

# every symbol include/ub.h declares, with (restype, argtypes)
i32, i64, u64, f32, vp, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_void_p, C.c_size_t
P_i32, P_i64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)


class FmhaParams(C.Structure):
    _fields_ = [("B", i32), ("T", i64), ("max_seqlen", i32), ("heads", i32), ("head_dim", i32),
                ("scale", f32), ("p_dropout", f32), ("seed", u64), ("offset", u64), ("dtype", i32),
                ("num_ctas", i32), ("dropout_mask", vp), ("schedule", vp)]


class EncoderParams(C.Structure):
    _fields_ = [("B", i32), ("T", i64), ("max_seqlen", i32), ("hidden", i32), ("heads", i32), ("p_attn", f32),
                ("p_hidden", f32), ("eps", f32), ("seed", u64), ("offset", u64), ("num_ctas", i32)]


SIGNATURES = {
    "ub_last_error": (C.c_char_p, []),
    "ub_version": (C.c_char_p, []),
    "ub_profile_events": (i32, [i32, vp, vp]),
    "ub_cu_seqlens": (i32, [vp, i32, i32, vp]),
    "ub_lengths_from_mask": (i32, [vp, i32, i32, vp]),
    "ub_unpad": (i32, [vp, vp, vp, i32, i32, i64, i64, vp]),
    "ub_pad": (i32, [vp, vp, vp, i32, i32, i64, i64, vp, vp]),
    "ub_fmha_workspace_bytes": (sz, [C.POINTER(FmhaParams), C.c_int]),
    "ub_fmha_schedule_ints": (sz, [i32, i32, i32, i32, i32]),
    "ub_fmha_schedule": (i32, [vp, i32, i32, i32, i32, i32, vp, sz]),
    "ub_exchange_slot_lengths": (i32, [vp, i32, i32, vp]),
    "ub_exchange_fmha_schedule": (i32, [vp, i32, vp, i32, i32, i32, i32, i32, vp, sz, vp, vp]),
    "ub_dropout_effective_p": (C.c_double, [f32, i32]),
    "ub_dropout_mask_bytes": (sz, [C.POINTER(FmhaParams)]),
    "ub_dropout_mask": (i32, [C.POINTER(FmhaParams), vp, vp, vp]),
    "ub_dropout_mask_ex": (i32, [C.POINTER(FmhaParams), vp, vp, i32, vp]),
    "ub_varlen_fmha_fwd": (i32, [C.POINTER(FmhaParams), vp, vp, vp, vp, vp, vp]),
    "ub_varlen_fmha_fwd_pad": (i32, [C.POINTER(FmhaParams), vp, vp, vp, vp, vp, i32, vp, vp]),
    "ub_varlen_fmha_bwd": (i32, [C.POINTER(FmhaParams), vp, vp, vp, vp, vp, vp, vp, vp]),
    "ub_dal_fwd": (i32, [vp, vp, vp, vp, i64, i32, f32, f32, u64, u64, vp, vp, vp, vp]),
    "ub_dal_bwd_workspace_bytes": (sz, [i64, i32]),
    "ub_dal_bwd": (i32, [vp, vp, vp, vp, vp, vp, i64, i32, f32, u64, u64, vp, vp, vp, vp, vp, vp]),
    "ub_embedding_fwd": (i32, [vp, vp, vp, vp, vp, vp, i64, i32, vp, vp]),
    "ub_embedding_bwd": (i32, [vp, vp, vp, vp, i64, i32, i32, i32, vp, vp, vp, vp]),
    "ub_linear_workspace_bytes": (sz, []),
    "ub_linear_fwd": (i32, [vp, vp, vp, i64, i32, i32, vp, vp, vp]),
    "ub_linear_bwd": (i32, [vp, vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp]),
    "ub_encoder_attn_workspace_bytes": (sz, [C.POINTER(EncoderParams), C.c_int]),
    "ub_encoder_attn_fwd": (i32, [C.POINTER(EncoderParams)] + [vp] * 17),
    "ub_encoder_attn_bwd": (i32, [C.POINTER(EncoderParams)] + [vp] * 21),
    "ub_balance_plan": (i32, [vp, i32, i32, i32, i32, vp, vp, vp, vp]),
    "ub_balance_plan_weighted": (i32, [vp, i32, i32, i32, i64, i64, vp, vp]),
    "ub_balance_relabel": (i32, [vp, i32, i32, vp, vp, vp]),
    "ub_exchange_tables": (i32, [vp, vp, i32, i32, i32, i32, vp, vp, vp, vp]),
    "ub_exchange_copy": (i32, [vp, vp, vp, vp, vp, i32, i64, i64, vp]),
    "ub_validate_cu_seqlens": (i32, [vp, i32, i32, i64, vp, vp]),
    "ub_set_checked": (i32, [i32]),
    "ub_ipc_export": (i32, [vp, vp]),
    "ub_ipc_import": (i32, [vp, vp, vp]),
    "ub_ipc_close": (i32, [vp]),
    "ub_exchange_pull_table": (i32, [vp, vp, i32, i32, i32, vp, vp]),
    "ub_exchange_pull": (i32, [vp, vp, vp, C.c_uint32, vp, i32, i64, i64, vp, vp, vp]),
    "ub_signal": (i32, [vp, C.c_uint32, vp]),
    "ub_wait_flags": (i32, [vp, i32, C.c_uint32, vp]),
    "ub_comm_unique_id": (i32, [vp]),
    "ub_comm_init": (i32, [C.POINTER(vp), vp, i32, i32]),
    "ub_comm_destroy": (i32, [vp]),
    "ub_comm_set_options": (i32, [vp, i32]),
    "ub_comm_nccl_ops": (i32, [vp, vp]),
    "ub_comm_host_profile": (i32, [vp, vp, i32, vp]),
    "ub_allgather_lengths": (i32, [vp, vp, vp, i32, vp]),
    "ub_exchange_workspace_bytes": (sz, [i32, i32, i64, i64, i64]),
    "ub_balance_exchange": (i32, [vp, i32, i32, i32, vp, vp, vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
    "ub_exchange_begin": (i32, [vp, i32, i32, vp, vp, vp]),
    "ub_exchange_finish": (i32, [vp, i32, i32, i32, i32, vp, vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]),
}

_lib = None


class UbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """The loaded library (raises if libub.so was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2208_08124_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    if status != UB_OK:
        raise UbError(status, lib().ub_last_error().decode())
