"""ctypes binding of libkvb.so (include/kvb.h). Fails loudly if the library is
missing: there is no CPU fallback anywhere in the product path."""

from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# KVB_LIB_TAG selects an experiment build libkvb_<tag>.so (build.py, same tag)
_TAG = os.environ.get("KVB_LIB_TAG", "")
LIB_PATH = os.path.join(_PKG, f"libkvb_{_TAG}.so" if _TAG else "libkvb.so")

KVB_OK, KVB_EINVAL, KVB_ECUDA, KVB_ENOMEM, KVB_ENCCL, KVB_EUNSUPPORTED = range(6)
KVB_F32, KVB_BF16 = 0, 1
KVB_LM_DENSE, KVB_LM_HIGGS = 0, 1
KVB_SLOW_NONE, KVB_SLOW_SVD, KVB_SLOW_FP8, KVB_SLOW_NVFP4 = 0, 1, 2, 3
KVB_TIER_HBM, KVB_TIER_HOST_MAPPED = 0, 1
KVB_AGG_SUM, KVB_AGG_MAX = 0, 1


class HiggsDesc(C.Structure):
    _fields_ = [("d", C.c_int32), ("n", C.c_int32), ("group", C.c_int32), ("seed", C.c_int32),
                ("codebook", C.POINTER(C.c_float)), ("signs", C.POINTER(C.c_float))]


class StoreDesc(C.Structure):
    _fields_ = [("batch", C.c_int32), ("n_tokens", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("chunk_size", C.c_int32), ("kv_dtype", C.c_int32),
                ("landmark_kind", C.c_int32), ("landmark_higgs", HiggsDesc),
                ("has_residual", C.c_int32), ("residual_higgs", HiggsDesc),
                ("slow_kind", C.c_int32), ("svd_rank", C.c_int32), ("svd_groups", C.c_int32),
                ("offload_tier", C.c_int32), ("max_resident", C.c_int32),
                ("capacity_tokens", C.c_int32)]


class StoreInfo(C.Structure):
    _fields_ = [("n_chunks", C.c_int32), ("n_groups_landmark", C.c_int32),
                ("n_groups_residual", C.c_int32), ("bytes_fast_tier", C.c_int64),
                ("bytes_offload_tier", C.c_int64)]


class SelectArgs(C.Structure):
    _fields_ = [("queries_per_head", C.c_int32), ("n_select", C.c_int32),
                ("aggregation", C.c_int32), ("rank_order", C.c_int32),
                ("token_capacity", C.c_int32), ("exact_scores", C.c_int32)]


class ResidualArgs(C.Structure):
    _fields_ = [("queries_per_head", C.c_int32), ("k_tokens", C.c_int32),
                ("n_candidates", C.c_int32), ("token_capacity", C.c_int32),
                ("exact_scores", C.c_int32)]


class AppendArgs(C.Structure):
    _fields_ = [("outlier_tokens", C.c_int32), ("local_window", C.c_int32)]


class AttendArgs(C.Structure):
    _fields_ = [("queries_per_head", C.c_int32), ("token_capacity", C.c_int32),
                ("k_path", C.c_int32)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64

# (name, restype, argtypes) -- every symbol declared in include/kvb.h
SIGNATURES = [
    ("kvb_last_error", C.c_char_p, []),
    ("kvb_abi_version", _I32, []),
    ("kvb_launch_count", _I64, []),
    ("kvb_trace_enable", _I32, [_I32]),
    ("kvb_trace_read", _I64, [_P, _I64]),
    ("kvb_store_create", _I32, [C.POINTER(StoreDesc), C.POINTER(_P)]),
    ("kvb_store_destroy", _I32, [_P]),
    ("kvb_store_get_info", _I32, [_P, C.POINTER(StoreInfo)]),
    ("kvb_store_landmark_ptr", _I32, [_P, C.POINTER(_P)]),
    ("kvb_build_landmarks", _I32, [_P, _P, _P]),
    ("kvb_build_residuals", _I32, [_P, _P, _P]),
    ("kvb_build_chunk_cosine", _I32, [_P, _P, _P, _P]),
    ("kvb_choose_outliers", _I32, [_P, _I32, _I32, _I32, _I32, _P, _P]),
    ("kvb_store_set_residency", _I32, [_P, _P, _P, _P, _P, _P]),
    ("kvb_store_set_offload", _I32, [_P, _P, _P, _P]),
    ("kvb_store_set_svd", _I32, [_P, _P, _P, _P]),
    ("kvb_store_set_landmarks_dense", _I32, [_P, _P, _P]),
    ("kvb_store_set_landmarks_higgs", _I32, [_P, _P, _P, _P]),
    ("kvb_store_set_residuals_higgs", _I32, [_P, _P, _P, _P]),
    ("kvb_landmarks_dequantized", _I32, [_P, _P, _P]),
    ("kvb_residuals_dequantized", _I32, [_P, _P, _P]),
    ("kvb_store_append", _I32, [_P, _P, _P, C.POINTER(AppendArgs), _P, _P, _P, _P]),
    ("kvb_gather_kv", _I32, [_P, _I32, _P, _I32, _I32, _P, _P, _P]),
    ("kvb_select", _I32, [_P, _P, C.POINTER(SelectArgs), _P, _P, _P, _P, _P, _I64, _P]),
    ("kvb_score_landmarks", _I32, [_P, _P, _I32, _I32, _P, _P]),
    ("kvb_select_workspace_bytes", _I64, [_P, C.POINTER(SelectArgs)]),
    ("kvb_select_residual", _I32, [_P, _P, C.POINTER(ResidualArgs), _P, _P, _P, _P, _P, _I64, _P]),
    ("kvb_select_residual_workspace_bytes", _I64, [_P, C.POINTER(ResidualArgs)]),
    ("kvb_attend", _I32, [_P, _P, C.POINTER(AttendArgs), _P, _P, _P, _P, _P, _I64, _P]),
    ("kvb_attend_workspace_bytes", _I64, [_P, C.POINTER(AttendArgs)]),
    ("kvb_decode_step", _I32, [_P, _P, C.POINTER(SelectArgs), C.POINTER(AttendArgs), _P, _P, _P,
                               _P, _P, _P, _I64, _P]),
    ("kvb_decode_workspace_bytes", _I64, [_P, C.POINTER(SelectArgs), C.POINTER(AttendArgs)]),
    ("kvb_select_candidates", _I32, [_P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _I64, _P]),
    ("kvb_select_candidates_workspace_bytes", _I64, [_P, _I32]),
    ("kvb_tokens_from_chunks", _I32, [_P, _P, _I32, _I32, _P, _P, _I32, _P]),
    ("kvb_merge_attention", _I32, [_P, _P, _I32, _I32, _I32, _P, _P, _P]),
    ("kvb_merge_topk", _I32, [_P, _P, _I32, _I32, _I32, _P, _P]),
    ("kvb_merge_topk_packed", _I32, [_P, _I32, _I32, _I32, _P, _P]),
    ("kvb_merge_attention_packed", _I32, [_P, _I32, _I32, _I32, _P, _P, _P]),
]

_lib = None


class KvbError(RuntimeError):
    pass


def load():
    """Load libkvb.so (building it is __graft_entry__.build()'s job)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 kernels are not built. Run "
            "`python -m paper_2604_08426_b200.build` (there is no CPU fallback).")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = "kvb"):
    """Map a kvb_status to the reference's exception types: EINVAL ->
    ValueError (same conditions as kvlab), the rest -> KvbError."""
    if status == KVB_OK:
        return
    msg = load().kvb_last_error().decode(errors="replace")
    if status == KVB_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if status == KVB_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise KvbError(f"{what}: status {status}: {msg}")
