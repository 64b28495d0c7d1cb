"""ctypes binding of libquestkv_b200.so (the C ABI declared in include/questkv_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2406_10774_b200/csrc``).  There is deliberately no fallback: if the library is
missing or fails to load, importing this module raises, so no Python or CPU path can
silently stand in for the CUDA kernels.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libquestkv_b200.so")
# Kernel A/B experiments point QK_LIB at another in-tree build (tools/ab_bench.sh).
LIB_PATH = os.environ.get("QK_LIB", LIB_PATH)

QK_OK = 0
QK_ERR_INVALID_ARGUMENT = 1
QK_ERR_OUT_OF_RANGE = 2
QK_ERR_CUDA = 3
QK_ERR_UNSUPPORTED = 4

QK_DTYPE_F32 = 0
QK_DTYPE_F16 = 1

QK_GROUP_MAX = 1
QK_GROUP_SUM = 2


class qk_cache_desc(ctypes.Structure):
    _fields_ = [
        ("head_dim", ctypes.c_uint32),
        ("page_size", ctypes.c_uint32),
        ("bytes_per_element", ctypes.c_uint32),
        ("num_layers", ctypes.c_uint32),
        ("max_batch", ctypes.c_uint32),
        ("num_q_heads", ctypes.c_uint32),
        ("num_kv_heads", ctypes.c_uint32),
        ("max_tokens", ctypes.c_uint32),
        ("device", ctypes.c_int32),
    ]


class qk_selection_cfg(ctypes.Structure):
    _fields_ = [
        ("token_budget", ctypes.c_uint32),
        ("force_include_recent", ctypes.c_int32),
        ("per_layer_enabled", ctypes.c_int32),
    ]


# Every symbol include/questkv_b200.h declares, with its ctypes signature.
_P = ctypes.c_void_p
_U32 = ctypes.c_uint32
_I32 = ctypes.c_int32
SIGNATURES = {
    "qk_last_error": (ctypes.c_char_p, []),
    "qk_abi_version": (ctypes.c_int, []),
    "qk_cache_create": (ctypes.c_int, [ctypes.POINTER(qk_cache_desc), ctypes.POINTER(_P)]),
    "qk_cache_destroy": (ctypes.c_int, [_P]),
    "qk_cache_describe": (ctypes.c_int, [_P, ctypes.POINTER(qk_cache_desc)]),
    "qk_cache_device_bytes": (ctypes.c_uint64, [_P]),
    "qk_cache_max_pages": (ctypes.c_uint32, [_P]),
    "qk_cache_reserve": (ctypes.c_int, [_P, ctypes.c_uint32]),
    "qk_host_alloc": (ctypes.c_void_p, [ctypes.c_size_t]),
    "qk_host_free": (None, [ctypes.c_void_p]),
    "qk_token_count": (ctypes.c_int, [_P, _U32, _U32, ctypes.POINTER(_U32)]),
    "qk_page_count": (ctypes.c_int, [_P, _U32, _U32, ctypes.POINTER(_U32)]),
    "qk_reset": (ctypes.c_int, [_P, _U32, _P]),
    "qk_append": (ctypes.c_int, [_P, _U32, _P, _P, _U32, _P]),
    "qk_prefill": (ctypes.c_int, [_P, _U32, _U32, _P, _P, _U32, _P]),
    "qk_read_metadata": (ctypes.c_int, [_P, _U32, _U32, _U32, _U32, _U32, _P, _P, _P]),
    "qk_read_kv": (ctypes.c_int, [_P, _U32, _U32, _U32, _U32, _U32, _P, _P, _P]),
    "qk_estimate": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P]),
    "qk_select_topk": (
        ctypes.c_int,
        [_P, _U32, _P, _U32, _U32, ctypes.POINTER(qk_selection_cfg), _P, _U32, _P, _P],
    ),
    "qk_sparse_attend": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _I32, _P, _P, _P]),
    "qk_dense_attend": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _I32, _P, _P, _P]),
    "qk_select_topk_pairs": (
        ctypes.c_int, [_P, _U32, _U32, _P, _P, _U32, ctypes.POINTER(qk_selection_cfg), _P, _U32, _P, _P],
    ),
    "qk_select_topk_pairs_host": (
        ctypes.c_int, [_P, _U32, _U32, _P, _P, _U32, ctypes.POINTER(qk_selection_cfg), _P, _U32, _P, _P],
    ),
    "qk_attend_tokens": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _I32, _P, _P, _P]),
    "qk_attention_logits": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _U32, _P]),
    "qk_softmax_weights": (ctypes.c_int, [_P, _P, _P, _U32, _U32, _U32, _P, _P]),
    "qk_decode_step": (
        ctypes.c_int,
        [_P, _U32, _P, _P, _P, _U32, ctypes.POINTER(qk_selection_cfg), _P, _I32, _P, _U32, _P, _P],
    ),
    "qk_decode_step_host": (
        ctypes.c_int,
        [_P, _U32, _P, _P, _P, _U32, ctypes.POINTER(qk_selection_cfg), _P, _P],
    ),
    "qk_check_status": (ctypes.c_int, [_P, _P]),
    "qk_sync_lengths": (ctypes.c_int, [_P, _P]),
    "qk_debug_probe": (ctypes.c_int, [_P, _P, _U32, _P]),
    "qk_debug_step_scores": (ctypes.c_int, [_P, _U32, _U32, _P, _U32, _P]),
    "qk_kernel_launches": (ctypes.c_uint64, [_P]),
    "qk_debug_keep_scores": (ctypes.c_int, [_P, _I32]),
    "qk_append_host": (ctypes.c_int, [_P, _U32, _P, _P, _U32, _P]),
    "qk_prefill_host": (ctypes.c_int, [_P, _U32, _U32, _P, _P, _U32, _P]),
    "qk_estimate_host": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P]),
    "qk_select_topk_host": (
        ctypes.c_int,
        [_P, _U32, _P, _U32, _U32, ctypes.POINTER(qk_selection_cfg), _P, _U32, _P, _P],
    ),
    "qk_sparse_attend_host": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _P, _P, _P]),
    "qk_dense_attend_host": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _P, _P, _P]),
    "qk_attend_tokens_host": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _P, _P, _P]),
    "qk_attention_logits_host": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _U32, _P]),
    "qk_softmax_weights_host": (ctypes.c_int, [_P, _U32, _P, _I32]),
    "qk_estimate_metadata_host": (ctypes.c_int, [_P, _P, _P, _U32, _U32, _P, _I32]),
    "qk_select_topk_grouped": (
        ctypes.c_int,
        [_P, _U32, _P, _U32, _U32, ctypes.POINTER(qk_selection_cfg), _I32, _P, _U32, _P, _P],
    ),
    "qk_sparse_attend_grouped": (ctypes.c_int, [_P, _U32, _P, _U32, _P, _U32, _P, _P, _I32, _P]),
    "qk_decode_step_grouped": (
        ctypes.c_int,
        [_P, _U32, _P, _P, _P, _U32, ctypes.POINTER(qk_selection_cfg), _I32, _P, _I32, _P, _U32,
         _P, _P],
    ),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the library once; raise loudly if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback for the Quest kernels)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (restype, argtypes) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


class QuestError(Exception):
    pass


def check(rc: int) -> None:
    """Map a qk_status to the Python analogue of the reference's exception type:
    std::invalid_argument -> ValueError, std::out_of_range -> IndexError."""
    if rc == QK_OK:
        return
    msg = load().qk_last_error().decode(errors="replace")
    if rc == QK_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == QK_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == QK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise QuestError(f"CUDA error: {msg}")
