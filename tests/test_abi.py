"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every symbol the
header declares, and validates arguments with the reference's error semantics before it
touches the GPU.  No compute call is made here (there is no GPU in this container)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "questkv_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"QK_API\s+[\w\s\*]+?\b(qk_\w+)\s*\(", text)))


def test_header_declares_the_operator_surface():
    syms = declared_symbols()
    for must in ("qk_cache_create", "qk_append", "qk_prefill", "qk_read_metadata", "qk_estimate",
                 "qk_select_topk", "qk_sparse_attend", "qk_dense_attend", "qk_decode_step",
                 "qk_attend_tokens", "qk_attention_logits", "qk_softmax_weights",
                 "qk_select_topk_pairs", "qk_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} lacks a ctypes signature"
    assert lib.qk_abi_version() == 2


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2406_10774_b200", "libquestkv_b200.so")
    out = os.popen(f"cuobjdump -lelf {so} 2>/dev/null").read()
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def _desc(**kw):
    from paper_2406_10774_b200._lib import qk_cache_desc

    base = dict(head_dim=128, page_size=16, bytes_per_element=2, num_layers=1, max_batch=1,
                num_q_heads=1, num_kv_heads=1, max_tokens=64, device=0)
    base.update(kw)
    return qk_cache_desc(*[base[f] for f, _ in qk_cache_desc._fields_])


@pytest.mark.parametrize("field,msg", [
    ("head_dim", "head_dim must be >= 1"),
    ("page_size", "page_size must be >= 1"),
    ("bytes_per_element", "bytes_per_element must be >= 1"),
])
def test_cache_config_validation_mirrors_reference(field, msg):
    # kv_store.cpp:8-13 messages, std::invalid_argument -> QK_ERR_INVALID_ARGUMENT
    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.qk_cache_create(ctypes.byref(_desc(**{field: 0})), ctypes.byref(h))
    assert rc == _lib.QK_ERR_INVALID_ARGUMENT
    assert msg in lib.qk_last_error().decode()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_unsupported_geometry_is_reported():
    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.qk_cache_create(ctypes.byref(_desc(head_dim=512)), ctypes.byref(h)) == \
        _lib.QK_ERR_UNSUPPORTED
    assert lib.qk_cache_create(ctypes.byref(_desc(bytes_per_element=4)), ctypes.byref(h)) == \
        _lib.QK_ERR_UNSUPPORTED
    assert lib.qk_cache_create(ctypes.byref(_desc(num_q_heads=3, num_kv_heads=2)),
                               ctypes.byref(h)) == _lib.QK_ERR_INVALID_ARGUMENT


def test_no_cpu_fallback_without_gpu():
    """Without a GPU the library refuses to create a cache (it has no CPU path)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.qk_cache_create(ctypes.byref(_desc()), ctypes.byref(h))
    assert rc == _lib.QK_ERR_CUDA
    assert "no CUDA device" in lib.qk_last_error().decode()


def test_null_handles_are_rejected():
    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    assert lib.qk_append(None, 0, None, None, 1, None) == _lib.QK_ERR_INVALID_ARGUMENT
    assert lib.qk_estimate(None, 0, None, 1, None, 0, None) == _lib.QK_ERR_INVALID_ARGUMENT
    assert lib.qk_cache_destroy(None) == _lib.QK_OK
    assert lib.qk_cache_reserve(None, 64) == _lib.QK_ERR_INVALID_ARGUMENT


def test_grouped_entry_points_reject_null_handles():
    """The GQA group-shared entry points validate before touching a device."""
    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    cfg = _lib.qk_selection_cfg(256, 1, 1)
    assert lib.qk_select_topk_grouped(None, 0, None, 0, 1, ctypes.byref(cfg), _lib.QK_GROUP_MAX,
                                      None, 0, None, None) == _lib.QK_ERR_INVALID_ARGUMENT
    assert "null argument" in lib.qk_last_error().decode()
    assert lib.qk_sparse_attend_grouped(None, 0, None, 1, None, 0, None, None, 0,
                                        None) == _lib.QK_ERR_INVALID_ARGUMENT
    assert lib.qk_decode_step_grouped(None, 0, None, None, None, 1, ctypes.byref(cfg),
                                      _lib.QK_GROUP_SUM, None, 0, None, 0, None,
                                      None) == _lib.QK_ERR_INVALID_ARGUMENT
    assert (_lib.QK_GROUP_MAX, _lib.QK_GROUP_SUM) == (1, 2)
