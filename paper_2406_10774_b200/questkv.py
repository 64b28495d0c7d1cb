"""Host-side mirror of the reference's ``questkv::`` operator API over the B200 kernels.

Two layers, both calling the C ABI (include/questkv_b200.h) through ``_lib``:

* :class:`QuestCache` -- the batched, device-resident cache a serving engine uses: every
  (layer, sequence, KV head) slice of a model in one object, operating on CUDA tensors
  (fp16 q/k/v, f64 scores, int32 page lists).
* The reference-shaped single-head API -- :class:`CacheConfig`, :class:`KvCache`,
  :func:`estimate_all`, :func:`select_top_k`, :func:`sparse_attention`,
  :func:`full_attention` ... -- with the same names, argument meaning and error behaviour
  as ``/root/reference/proj/core/include/questkv/{kv_store,criticality,attention}.hpp``
  (std::invalid_argument -> ValueError, std::out_of_range -> IndexError), so parity
  tests read like the reference's own tests.  Values cross the boundary as fp16 (the
  reference stores float; callers feed fp16-representable values for bitwise parity).

Torch is used only for device memory and streams.  Every compute call launches the
sm_100a kernels in libquestkv_b200.so; there is no CPU or PyTorch fallback.
"""

from __future__ import annotations

import ctypes
import math
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, qk_cache_desc, qk_selection_cfg

__all__ = [
    "QuestCache",
    "CacheConfig",
    "PageMetadata",
    "Page",
    "KvCache",
    "PageScore",
    "SelectionConfig",
    "AttentionOutput",
    "estimate_page_score",
    "estimate_all",
    "select_top_k",
    "sparse_attention",
    "full_attention",
    "attend_tokens",
    "attention_logits",
    "softmax_weights",
    "traffic_fraction",
]


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


def _sel_cfg(token_budget: int, force_include_recent: bool, per_layer_enabled: bool):
    return qk_selection_cfg(int(token_budget), int(bool(force_include_recent)),
                            int(bool(per_layer_enabled)))


def host_empty(shape, dtype) -> np.ndarray:
    """A numpy array in pinned, device-mapped host memory (qk_host_alloc), freed when the last
    view of it goes away.  decode_step_host reads and writes such arrays in place (no staging
    copy); other host arrays work too, through the cache's staging buffer."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    lib = _lib.load()
    p = lib.qk_host_alloc(max(nbytes, 1))
    if not p:
        check(_lib.QK_ERR_CUDA)
    block = (ctypes.c_uint8 * max(nbytes, 1)).from_address(p)
    weakref.finalize(block, lib.qk_host_free, p)
    return np.frombuffer(block, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


class QuestCache:
    """Batched paged KV cache with per-page min/max key metadata, resident in HBM.

    Mirrors ``questkv::KvCache`` (kv_store.hpp:41-65) for every (layer, sequence, KV head)
    slice at once.  ``num_q_heads`` may be a multiple of ``num_kv_heads`` (GQA); each query
    head selects its own pages.
    """

    def __init__(self, head_dim: int, page_size: int, *, num_layers: int = 1, max_batch: int = 1,
                 num_q_heads: int = 1, num_kv_heads: Optional[int] = None, max_tokens: int = 4096,
                 bytes_per_element: int = 2, device: Optional[int] = None):
        self._lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        num_kv_heads = num_q_heads if num_kv_heads is None else num_kv_heads
        desc = qk_cache_desc(head_dim, page_size, bytes_per_element, num_layers, max_batch,
                             num_q_heads, num_kv_heads, max_tokens, device)
        handle = ctypes.c_void_p()
        self._h = None
        check(self._lib.qk_cache_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._h = handle
        self.head_dim = head_dim
        self.page_size = page_size
        self.num_layers = num_layers
        self.max_batch = max_batch
        self.num_q_heads = num_q_heads
        self.num_kv_heads = num_kv_heads
        self.max_tokens = max_tokens
        self.device = torch.device("cuda", device)
        self.max_pages = int(self._lib.qk_cache_max_pages(self._h))

    def reserve(self, max_tokens: int) -> None:
        """Grow every slice to hold ``max_tokens`` tokens (qk_cache_reserve): the cached pages,
        metadata and lengths are kept.  Graphs captured before the call must be re-captured."""
        check(self._lib.qk_cache_reserve(self._h, int(max_tokens)))
        self.max_tokens = max(self.max_tokens, int(max_tokens))
        self.max_pages = int(self._lib.qk_cache_max_pages(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.qk_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- geometry ---------------------------------------------------------------------
    @property
    def device_bytes(self) -> int:
        return int(self._lib.qk_cache_device_bytes(self._h))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.qk_kernel_launches(self._h))

    def token_count(self, layer: int = 0, seq: int = 0) -> int:
        n = ctypes.c_uint32()
        check(self._lib.qk_token_count(self._h, layer, seq, ctypes.byref(n)))
        return n.value

    def page_count(self, layer: int = 0, seq: int = 0) -> int:
        n = ctypes.c_uint32()
        check(self._lib.qk_page_count(self._h, layer, seq, ctypes.byref(n)))
        return n.value

    def _check_half(self, t: torch.Tensor, shape, name: str) -> torch.Tensor:
        if t.dtype != torch.float16 or t.device != self.device:
            raise ValueError(f"{name} must be a float16 tensor on {self.device}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
        return t.contiguous()

    # -- writes -----------------------------------------------------------------------
    def reset(self, layer: Optional[int] = None, stream=None) -> None:
        check(self._lib.qk_reset(self._h, 0xFFFFFFFF if layer is None else layer,
                                 _stream_ptr(stream)))

    def append(self, layer: int, k: torch.Tensor, v: torch.Tensor, stream=None) -> None:
        """KvCache::append for sequences 0..batch-1; k, v: [batch, Hkv, head_dim] fp16."""
        batch = k.shape[0]
        k = self._check_half(k, (batch, self.num_kv_heads, self.head_dim), "k")
        v = self._check_half(v, (batch, self.num_kv_heads, self.head_dim), "v")
        check(self._lib.qk_append(self._h, layer, _ptr(k), _ptr(v), batch, _stream_ptr(stream)))

    def prefill(self, layer: int, seq: int, k: torch.Tensor, v: torch.Tensor, stream=None) -> None:
        """n successive appends for one sequence; k, v: [Hkv, n, head_dim] fp16."""
        n = k.shape[1]
        k = self._check_half(k, (self.num_kv_heads, n, self.head_dim), "k")
        v = self._check_half(v, (self.num_kv_heads, n, self.head_dim), "v")
        check(self._lib.qk_prefill(self._h, layer, seq, _ptr(k), _ptr(v), n, _stream_ptr(stream)))

    # -- reads (synchronous) ---------------------------------------------------------
    def read_metadata(self, layer: int, seq: int, kv_head: int, page0: int = 0,
                      n_pages: Optional[int] = None, stream=None):
        """(min, max) fp16 arrays [n_pages, head_dim] of KvCache::page_metadata."""
        if n_pages is None:
            n_pages = self.page_count(layer, seq) - page0
        mn = np.empty((max(n_pages, 0), self.head_dim), dtype=np.float16)
        mx = np.empty_like(mn)
        check(self._lib.qk_read_metadata(self._h, layer, seq, kv_head, page0, n_pages,
                                          mn.ctypes.data, mx.ctypes.data, _stream_ptr(stream)))
        return mn, mx

    def read_kv(self, layer: int, seq: int, kv_head: int, token0: int = 0,
                n_tokens: Optional[int] = None, stream=None):
        if n_tokens is None:
            n_tokens = self.token_count(layer, seq) - token0
        k = np.empty((max(n_tokens, 0), self.head_dim), dtype=np.float16)
        v = np.empty_like(k)
        check(self._lib.qk_read_kv(self._h, layer, seq, kv_head, token0, n_tokens,
                                    k.ctypes.data, v.ctypes.data, _stream_ptr(stream)))
        return k, v

    # -- the hot path -----------------------------------------------------------------
    def _check_q(self, q: torch.Tensor) -> torch.Tensor:
        return self._check_half(q, (q.shape[0], self.num_q_heads, self.head_dim), "q")

    def estimate(self, layer: int, q: torch.Tensor, scores: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
        """estimate_all for every (sequence, query head): f64 [batch, Hq, max_pages]."""
        q = self._check_q(q)
        batch = q.shape[0]
        if scores is None:
            scores = torch.zeros((batch, self.num_q_heads, self.max_pages), dtype=torch.float64,
                                 device=self.device)
        check(self._lib.qk_estimate(self._h, layer, _ptr(q), batch, _ptr(scores),
                                    scores.shape[-1], _stream_ptr(stream)))
        return scores

    def select_topk(self, layer: int, scores: torch.Tensor, token_budget: int,
                    force_include_recent: bool = True, per_layer_enabled: bool = True,
                    pages: Optional[torch.Tensor] = None, counts: Optional[torch.Tensor] = None,
                    stream=None):
        """select_top_k per (sequence, query head): (pages int32 [batch, Hq, stride], counts)."""
        batch = scores.shape[0]
        if pages is None:
            stride = self.max_pages
            if per_layer_enabled and token_budget >= self.page_size:
                stride = min(self.max_pages, token_budget // self.page_size)
            pages = torch.full((batch, self.num_q_heads, max(stride, 1)), -1, dtype=torch.int32,
                               device=self.device)
        if counts is None:
            counts = torch.zeros((batch, self.num_q_heads), dtype=torch.int32, device=self.device)
        cfg = _sel_cfg(token_budget, force_include_recent, per_layer_enabled)
        check(self._lib.qk_select_topk(self._h, layer, _ptr(scores), scores.shape[-1], batch,
                                       ctypes.byref(cfg), _ptr(pages), pages.shape[-1],
                                       _ptr(counts), _stream_ptr(stream)))
        return pages, counts

    def _attn_outputs(self, batch, out_dtype, want_lse, want_wsum):
        out = torch.empty((batch, self.num_q_heads, self.head_dim), dtype=out_dtype,
                          device=self.device)
        lse = torch.empty((batch, self.num_q_heads), dtype=torch.float32,
                          device=self.device) if want_lse else None
        wsum = torch.empty((batch, self.num_q_heads), dtype=torch.float64,
                           device=self.device) if want_wsum else None
        dt = _lib.QK_DTYPE_F32 if out_dtype == torch.float32 else _lib.QK_DTYPE_F16
        return out, lse, wsum, dt

    @staticmethod
    def _attn_result(out, lse, wsum):
        res = (out,) + ((lse,) if lse is not None else ()) + ((wsum,) if wsum is not None else ())
        return res[0] if len(res) == 1 else res

    def sparse_attend(self, layer: int, q: torch.Tensor, pages: torch.Tensor, counts: torch.Tensor,
                      out_dtype: torch.dtype = torch.float32, want_lse: bool = False,
                      want_weights_sum: bool = False, stream=None):
        """sparse_attention per (sequence, query head); returns out [, lse] [, weights_sum]."""
        q = self._check_q(q)
        batch = q.shape[0]
        out, lse, wsum, dt = self._attn_outputs(batch, out_dtype, want_lse, want_weights_sum)
        pages = pages.to(torch.int32).contiguous()
        counts = counts.to(torch.int32).contiguous()
        check(self._lib.qk_sparse_attend(self._h, layer, _ptr(q), batch, _ptr(pages),
                                         pages.shape[-1], _ptr(counts), _ptr(out), dt, _ptr(lse),
                                         _ptr(wsum), _stream_ptr(stream)))
        return self._attn_result(out, lse, wsum)

    def dense_attend(self, layer: int, q: torch.Tensor, out_dtype: torch.dtype = torch.float32,
                     want_lse: bool = False, want_weights_sum: bool = False, stream=None):
        """full_attention per (sequence, query head); returns out [, lse] [, weights_sum]."""
        q = self._check_q(q)
        batch = q.shape[0]
        out, lse, wsum, dt = self._attn_outputs(batch, out_dtype, want_lse, want_weights_sum)
        check(self._lib.qk_dense_attend(self._h, layer, _ptr(q), batch, _ptr(out), dt, _ptr(lse),
                                        _ptr(wsum), _stream_ptr(stream)))
        return self._attn_result(out, lse, wsum)

    def attend_tokens(self, layer: int, q: torch.Tensor, tokens: torch.Tensor,
                      counts: torch.Tensor, out_dtype: torch.dtype = torch.float32,
                      want_lse: bool = False, want_weights_sum: bool = False, stream=None):
        """attend_tokens (attention.cpp:69-84) per (sequence, query head) over explicit,
        strictly ascending token lists tokens [batch, Hq, stride] (counts [batch, Hq]);
        invalid lists surface at check_status()."""
        q = self._check_q(q)
        batch = q.shape[0]
        out, lse, wsum, dt = self._attn_outputs(batch, out_dtype, want_lse, want_weights_sum)
        tokens = tokens.to(torch.int32).contiguous()
        counts = counts.to(torch.int32).contiguous()
        check(self._lib.qk_attend_tokens(self._h, layer, _ptr(q), batch, _ptr(tokens),
                                         tokens.shape[-1], _ptr(counts), _ptr(out), dt, _ptr(lse),
                                         _ptr(wsum), _stream_ptr(stream)))
        return self._attn_result(out, lse, wsum)

    def attention_logits(self, layer: int, q: torch.Tensor, tokens: Optional[torch.Tensor] = None,
                         counts: Optional[torch.Tensor] = None, stride: Optional[int] = None,
                         stream=None) -> torch.Tensor:
        """attention_logits (attention.cpp:34-52): f64 [batch, Hq, stride], bitwise the
        reference's; tokens None -> every cached token (stride defaults to max_tokens)."""
        q = self._check_q(q)
        batch = q.shape[0]
        if tokens is not None:
            tokens = tokens.to(torch.int32).contiguous()
            counts = counts.to(torch.int32).contiguous()
            stride = tokens.shape[-1] if stride is None else stride
        elif stride is None:
            stride = self.max_tokens
        logits = torch.zeros((batch, self.num_q_heads, stride), dtype=torch.float64,
                             device=self.device)
        check(self._lib.qk_attention_logits(self._h, layer, _ptr(q), batch, _ptr(tokens),
                                            0 if tokens is None else tokens.shape[-1],
                                            _ptr(counts), _ptr(logits), stride,
                                            _stream_ptr(stream)))
        return logits

    def softmax_weights(self, logits: torch.Tensor, counts: Optional[torch.Tensor] = None,
                        stream=None) -> torch.Tensor:
        """softmax_weights (attention.cpp:54-67) over the rows of f64 logits [..., stride]
        (counts: valid entries per row; None = the whole row)."""
        lg = logits.to(torch.float64).contiguous()
        stride = lg.shape[-1]
        rows = lg.numel() // max(stride, 1)
        if counts is not None:
            counts = counts.to(torch.int32).contiguous()
        w = torch.zeros_like(lg)
        check(self._lib.qk_softmax_weights(self._h, _ptr(lg), _ptr(counts), stride, stride, rows,
                                           _ptr(w), _stream_ptr(stream)))
        return w

    def select_topk_pairs(self, layer: int, seq: int, page_index: torch.Tensor,
                          scores: torch.Tensor, token_budget: int, force_include_recent: bool = True,
                          per_layer_enabled: bool = True, stream=None):
        """select_top_k on an arbitrary PageScore vector (any order, repeats allowed):
        returns (pages int32 [capacity], count int32 [1])."""
        pi = page_index.to(torch.int32).contiguous()
        sc = scores.to(torch.float64).contiguous()
        cap = max(self.max_pages, token_budget // self.page_size, 1)
        pages = torch.full((cap,), -1, dtype=torch.int32, device=self.device)
        count = torch.zeros((1,), dtype=torch.int32, device=self.device)
        cfg = _sel_cfg(token_budget, force_include_recent, per_layer_enabled)
        check(self._lib.qk_select_topk_pairs(self._h, layer, seq, _ptr(pi), _ptr(sc), pi.numel(),
                                             ctypes.byref(cfg), _ptr(pages), cap, _ptr(count),
                                             _stream_ptr(stream)))
        return pages, count

    def decode_step(self, layer: int, q: torch.Tensor, k: Optional[torch.Tensor],
                    v: Optional[torch.Tensor], token_budget: int, force_include_recent: bool = True,
                    per_layer_enabled: bool = True, out: Optional[torch.Tensor] = None,
                    pages: Optional[torch.Tensor] = None, counts: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
        """append -> estimate -> top-K -> attend for one layer (qk_decode_step)."""
        q = self._check_q(q)
        batch = q.shape[0]
        if k is not None:
            k = self._check_half(k, (batch, self.num_kv_heads, self.head_dim), "k")
            v = self._check_half(v, (batch, self.num_kv_heads, self.head_dim), "v")
        if out is None:
            out = torch.empty((batch, self.num_q_heads, self.head_dim), dtype=torch.float32,
                              device=self.device)
        dt = _lib.QK_DTYPE_F32 if out.dtype == torch.float32 else _lib.QK_DTYPE_F16
        cfg = _sel_cfg(token_budget, force_include_recent, per_layer_enabled)
        check(self._lib.qk_decode_step(self._h, layer, _ptr(q), _ptr(k), _ptr(v), batch,
                                       ctypes.byref(cfg), _ptr(out), dt, _ptr(pages),
                                       0 if pages is None else pages.shape[-1], _ptr(counts),
                                       _stream_ptr(stream)))
        return out

    # -- GQA group-shared selection (opt-in, not the reference's
    #    per-head semantics -- see include/questkv_b200.h) ----------------------------------
    _GROUP_REDUCE = {"max": _lib.QK_GROUP_MAX, "sum": _lib.QK_GROUP_SUM}

    def _group_reduce(self, reduce: str) -> int:
        if reduce not in self._GROUP_REDUCE:
            raise ValueError("group_reduce must be 'max' or 'sum'")
        return self._GROUP_REDUCE[reduce]

    def _group_lists(self, batch, token_budget, per_layer_enabled, pages, counts):
        if pages is None:
            stride = self.max_pages
            if per_layer_enabled and token_budget >= self.page_size:
                stride = min(self.max_pages, token_budget // self.page_size)
            pages = torch.full((batch, self.num_kv_heads, max(stride, 1)), -1, dtype=torch.int32,
                               device=self.device)
        if counts is None:
            counts = torch.zeros((batch, self.num_kv_heads), dtype=torch.int32, device=self.device)
        return pages, counts

    def select_topk_grouped(self, layer: int, scores: torch.Tensor, token_budget: int,
                            group_reduce: str = "max", force_include_recent: bool = True,
                            per_layer_enabled: bool = True, pages: Optional[torch.Tensor] = None,
                            counts: Optional[torch.Tensor] = None, stream=None):
        """One page set per (sequence, KV head) from the group scores of estimate()'s per-head
        scores: (pages int32 [batch, Hkv, stride], counts [batch, Hkv])."""
        batch = scores.shape[0]
        pages, counts = self._group_lists(batch, token_budget, per_layer_enabled, pages, counts)
        cfg = _sel_cfg(token_budget, force_include_recent, per_layer_enabled)
        check(self._lib.qk_select_topk_grouped(
            self._h, layer, _ptr(scores), scores.shape[-1], batch, ctypes.byref(cfg),
            self._group_reduce(group_reduce), _ptr(pages), pages.shape[-1], _ptr(counts),
            _stream_ptr(stream)))
        return pages, counts

    def sparse_attend_grouped(self, layer: int, q: torch.Tensor, pages: torch.Tensor,
                              counts: torch.Tensor, out_dtype: torch.dtype = torch.float32,
                              stream=None) -> torch.Tensor:
        """Every query head attends over its KV group's page list (tensor-core kernel)."""
        q = self._check_q(q)
        batch = q.shape[0]
        out = torch.empty((batch, self.num_q_heads, self.head_dim), dtype=out_dtype,
                          device=self.device)
        dt = _lib.QK_DTYPE_F32 if out_dtype == torch.float32 else _lib.QK_DTYPE_F16
        pages = pages.to(torch.int32).contiguous()
        counts = counts.to(torch.int32).contiguous()
        check(self._lib.qk_sparse_attend_grouped(self._h, layer, _ptr(q), batch, _ptr(pages),
                                                 pages.shape[-1], _ptr(counts), _ptr(out), dt,
                                                 _stream_ptr(stream)))
        return out

    def decode_step_grouped(self, layer: int, q: torch.Tensor, k: Optional[torch.Tensor],
                            v: Optional[torch.Tensor], token_budget: int,
                            group_reduce: str = "max", force_include_recent: bool = True,
                            per_layer_enabled: bool = True, out: Optional[torch.Tensor] = None,
                            pages: Optional[torch.Tensor] = None,
                            counts: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """append -> estimate -> group top-K -> group attention (qk_decode_step_grouped)."""
        q = self._check_q(q)
        batch = q.shape[0]
        if k is not None:
            k = self._check_half(k, (batch, self.num_kv_heads, self.head_dim), "k")
            v = self._check_half(v, (batch, self.num_kv_heads, self.head_dim), "v")
        if out is None:
            out = torch.empty((batch, self.num_q_heads, self.head_dim), dtype=torch.float32,
                              device=self.device)
        dt = _lib.QK_DTYPE_F32 if out.dtype == torch.float32 else _lib.QK_DTYPE_F16
        cfg = _sel_cfg(token_budget, force_include_recent, per_layer_enabled)
        check(self._lib.qk_decode_step_grouped(
            self._h, layer, _ptr(q), _ptr(k), _ptr(v), batch, ctypes.byref(cfg),
            self._group_reduce(group_reduce), _ptr(out), dt, _ptr(pages),
            0 if pages is None else pages.shape[-1], _ptr(counts), _stream_ptr(stream)))
        return out

    def decode_step_host(self, layer: int, q: np.ndarray, k: Optional[np.ndarray],
                         v: Optional[np.ndarray], token_budget: int,
                         force_include_recent: bool = True, per_layer_enabled: bool = True,
                         out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
        """qk_decode_step_host: host fp16 arrays in, host fp32 output out (synchronous)."""
        def host(a, shape, dtype, name):
            if not isinstance(a, np.ndarray) or a.dtype != dtype:
                raise ValueError(f"{name} must be a numpy {np.dtype(dtype).name} array")
            if tuple(a.shape) != tuple(shape):
                raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(a.shape)}")
            if not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"{name} must be C-contiguous")
            return a

        if not isinstance(q, np.ndarray) or q.ndim != 3:
            raise ValueError("q must be a numpy float16 array [batch, num_q_heads, head_dim]")
        batch = q.shape[0]
        host(q, (batch, self.num_q_heads, self.head_dim), np.float16, "q")
        if (k is None) != (v is None):
            raise ValueError("k and v must both be given")
        if k is not None:
            host(k, (batch, self.num_kv_heads, self.head_dim), np.float16, "k")
            host(v, (batch, self.num_kv_heads, self.head_dim), np.float16, "v")
        if out is None:
            out = np.empty((batch, self.num_q_heads, self.head_dim), dtype=np.float32)
        host(out, (batch, self.num_q_heads, self.head_dim), np.float32, "out")
        if not out.flags["WRITEABLE"]:
            raise ValueError("out must be writeable")
        cfg = _sel_cfg(token_budget, force_include_recent, per_layer_enabled)
        check(self._lib.qk_decode_step_host(
            self._h, layer, q.ctypes.data, None if k is None else k.ctypes.data,
            None if v is None else v.ctypes.data, batch, ctypes.byref(cfg), out.ctypes.data,
            _stream_ptr(stream)))
        return out

    def keep_step_scores(self, on: bool = True) -> None:
        """Make decode_step estimate every page and keep the scores (parity diagnostics;
        by default the fused step skips scores the selection cannot use)."""
        check(self._lib.qk_debug_keep_scores(self._h, int(bool(on))))

    def step_scores(self, seq: int, q_head: int, n_pages: int, stream=None) -> np.ndarray:
        """Page scores the last decode_step computed for (seq, q_head) (diagnostics; needs
        keep_step_scores())."""
        out = np.empty(n_pages, dtype=np.float64)
        check(self._lib.qk_debug_step_scores(self._h, seq, q_head, out.ctypes.data, n_pages,
                                             _stream_ptr(stream)))
        return out

    def sync_lengths(self, stream=None) -> None:
        """Refresh the host-side token counts from the device (after CUDA-graph replays)."""
        check(self._lib.qk_sync_lengths(self._h, _stream_ptr(stream)))

    def check_status(self, stream=None) -> None:
        """Raise the error a kernel recorded on the device (bad page list, overflow)."""
        check(self._lib.qk_check_status(self._h, _stream_ptr(stream)))


# ---------------------------------------------------------------------------------------
# Reference-shaped single-head API (kv_store.hpp, criticality.hpp, attention.hpp).


@dataclass
class CacheConfig:
    """questkv::CacheConfig (kv_store.hpp:10-17)."""

    head_dim: int = 0
    page_size: int = 0
    bytes_per_element: int = 2

    def validate(self) -> None:
        """kv_store.cpp:8-13."""
        if self.head_dim == 0:
            raise ValueError("CacheConfig: head_dim must be >= 1")
        if self.page_size == 0:
            raise ValueError("CacheConfig: page_size must be >= 1")
        if self.bytes_per_element == 0:
            raise ValueError("CacheConfig: bytes_per_element must be >= 1")


@dataclass
class PageMetadata:
    min_key: List[float] = field(default_factory=list)
    max_key: List[float] = field(default_factory=list)


@dataclass
class Page:
    keys: List[float]
    values: List[float]
    metadata: PageMetadata
    length: int


def _as_half_row(x, dim: int, what: str) -> np.ndarray:
    a = np.asarray(x, dtype=np.float32).reshape(-1)
    if a.shape[0] != dim:
        raise ValueError(f"{what}: vector dimension mismatch")
    return a.astype(np.float16)


class KvCache:
    """questkv::KvCache (kv_store.hpp:41-65): one head's paged cache, held on the GPU.

    ``capacity`` is the initial allocation; like the reference's page vector it grows
    (doubling, qk_cache_reserve) when an append or extend needs more.
    """

    def __init__(self, config: CacheConfig, capacity: int = 8192, device: Optional[int] = None):
        config.validate()
        self._config = config
        self._qc = QuestCache(config.head_dim, config.page_size, max_tokens=capacity,
                              bytes_per_element=config.bytes_per_element, device=device)

    @property
    def quest_cache(self) -> QuestCache:
        return self._qc

    def config(self) -> CacheConfig:
        return self._config

    def token_count(self) -> int:
        return self._qc.token_count()

    def page_count(self) -> int:
        return self._qc.page_count()

    def append(self, key: Sequence[float], value: Sequence[float]) -> int:
        """kv_store.cpp:19-47; returns the token index."""
        d = self._config.head_dim
        k = _as_half_row(key, d, "KvCache::append")
        v = _as_half_row(value, d, "KvCache::append")
        t = self.token_count()
        self._ensure(t + 1)
        dev = self._qc.device
        self._qc.append(0, torch.from_numpy(k).to(dev).view(1, 1, d),
                        torch.from_numpy(v).to(dev).view(1, 1, d))
        return t

    def extend(self, keys, values) -> None:
        """Bulk append of [n, head_dim] rows (qk_prefill): same result as n appends."""
        d = self._config.head_dim
        k = np.asarray(keys, dtype=np.float32).reshape(-1, d).astype(np.float16)
        v = np.asarray(values, dtype=np.float32).reshape(-1, d).astype(np.float16)
        if k.shape != v.shape:
            raise ValueError("KvCache::extend: keys/values shape mismatch")
        self._ensure(self.token_count() + k.shape[0])
        dev = self._qc.device
        self._qc.prefill(0, 0, torch.from_numpy(k).to(dev).view(1, -1, d),
                         torch.from_numpy(v).to(dev).view(1, -1, d))

    def _ensure(self, tokens: int) -> None:
        if tokens > self._qc.max_tokens:
            cap = 16384 * self._config.page_size  # the ABI's page limit per slice
            self._qc.reserve(max(tokens, min(2 * self._qc.max_tokens, cap)))

    def page_metadata(self, page_index: int) -> PageMetadata:
        """kv_store.cpp:49-54 (IndexError == std::out_of_range)."""
        if page_index < 0 or page_index >= self.page_count():
            raise IndexError(f"KvCache::page_metadata: page index {page_index} out of range")
        mn, mx = self._qc.read_metadata(0, 0, 0, page_index, 1)
        return PageMetadata(mn[0].astype(np.float32).tolist(), mx[0].astype(np.float32).tolist())

    def page(self, page_index: int) -> Page:
        if page_index < 0 or page_index >= self.page_count():
            raise IndexError(f"KvCache::page: page index {page_index} out of range")
        S = self._config.page_size
        t0 = page_index * S
        n = min(S, self.token_count() - t0)
        k, v = self._qc.read_kv(0, 0, 0, t0, n)
        return Page(k.astype(np.float32).reshape(-1).tolist(), v.astype(np.float32).reshape(-1).tolist(),
                    self.page_metadata(page_index), n)

    def key(self, token: int) -> List[float]:
        if token < 0 or token >= self.token_count():
            raise IndexError(f"KvCache::key: token {token} out of range")
        k, _ = self._qc.read_kv(0, 0, 0, token, 1)
        return k[0].astype(np.float32).tolist()

    def value(self, token: int) -> List[float]:
        if token < 0 or token >= self.token_count():
            raise IndexError(f"KvCache::value: token {token} out of range")
        _, v = self._qc.read_kv(0, 0, 0, token, 1)
        return v[0].astype(np.float32).tolist()


@dataclass
class PageScore:
    """criticality.hpp:13-16."""

    page_index: int = 0
    score: float = 0.0


@dataclass
class SelectionConfig:
    """criticality.hpp:18-22."""

    token_budget: int = 0
    force_include_recent: bool = True
    per_layer_enabled: bool = True


@dataclass
class AttentionOutput:
    """attention.hpp:15-18.  weights_sum_check: the post-softmax mass of the weights the
    kernel applied (fp64 from its fp32 partials; 1 up to fp32 rounding of the normaliser)."""

    output: List[float]
    weights_sum_check: float = 0.0


def _query_dev(query, cache: KvCache) -> torch.Tensor:
    d = cache.config().head_dim
    q = _as_half_row(query, d, "attention: query")
    return torch.from_numpy(q).to(cache.quest_cache.device).view(1, 1, d)


def estimate_all(query, cache: KvCache) -> List[PageScore]:
    """criticality.cpp:25-34 -- one PageScore per page, bitwise the reference's doubles."""
    qc = cache.quest_cache
    d = cache.config().head_dim
    if cache.page_count() == 0:
        raise ValueError("estimate_all: empty cache")
    if len(np.asarray(query).reshape(-1)) != d:
        raise ValueError("estimate_page_score: dimension mismatch")
    scores = qc.estimate(0, _query_dev(query, cache))
    vals = scores[0, 0, : cache.page_count()].cpu().numpy()
    return [PageScore(i, float(s)) for i, s in enumerate(vals)]


def estimate_page_score(query, metadata: PageMetadata) -> float:
    """criticality.cpp:9-23 on explicit metadata: a one-page GPU cache whose two keys are
    min_key and max_key has exactly that metadata (min <= max channel-wise)."""
    d = len(metadata.min_key)
    if d == 0 or len(np.asarray(query).reshape(-1)) != d or len(metadata.max_key) != d:
        raise ValueError("estimate_page_score: dimension mismatch")
    tmp = KvCache(CacheConfig(head_dim=d, page_size=2), capacity=2)
    tmp.extend(np.stack([np.asarray(metadata.min_key), np.asarray(metadata.max_key)]),
               np.zeros((2, d), dtype=np.float32))
    return estimate_all(query, tmp)[0].score


def select_top_k(scores: Sequence[PageScore], config: SelectionConfig,
                 cache: KvCache) -> List[int]:
    """criticality.cpp:36-81 on the GPU.  estimate_all's form (one score per page, in page
    order) takes the radix top-K kernel; any other PageScore vector (any order, repeated
    pages) takes the pair-sorting kernel, with the reference's exact semantics."""
    P = cache.page_count()
    if not config.per_layer_enabled:
        return list(range(P))
    if config.token_budget < cache.config().page_size:
        raise ValueError("select_top_k: token_budget below page_size")
    if len(scores) == 0:
        raise ValueError("select_top_k: no scores")
    for s in scores:
        if s.page_index >= P:
            raise IndexError("select_top_k: score for nonexistent page")
    qc = cache.quest_cache
    if [s.page_index for s in scores] == list(range(P)):
        dev = torch.tensor([s.score for s in scores], dtype=torch.float64, device=qc.device)
        pages, counts = qc.select_topk(0, dev.view(1, 1, -1), config.token_budget,
                                       config.force_include_recent, config.per_layer_enabled)
        n = int(counts[0, 0])
        return pages[0, 0, :n].cpu().tolist()
    pi = np.array([s.page_index for s in scores], dtype=np.uint32)
    sc = np.array([s.score for s in scores], dtype=np.float64)
    cap = max(P, config.token_budget // cache.config().page_size, 1)
    out = np.zeros(cap, dtype=np.int32)
    cnt = ctypes.c_int32()
    cfg = _sel_cfg(config.token_budget, config.force_include_recent, config.per_layer_enabled)
    check(qc._lib.qk_select_topk_pairs_host(qc._h, 0, 0, pi.ctypes.data, sc.ctypes.data, len(pi),
                                            ctypes.byref(cfg), out.ctypes.data, cap,
                                            ctypes.byref(cnt), None))
    return out[: cnt.value].tolist()


def sparse_attention(query, cache: KvCache, selected_pages: Sequence[int]) -> AttentionOutput:
    """attention.cpp:94-116: any order accepted; empty -> ValueError, duplicate ->
    ValueError, out of range -> IndexError."""
    if len(selected_pages) == 0:
        raise ValueError("sparse_attention: empty page selection")
    pages = sorted(int(p) for p in selected_pages)
    P = cache.page_count()
    for i, p in enumerate(pages):
        if p < 0 or p >= P:
            raise IndexError("sparse_attention: page index out of range")
        if i > 0 and p == pages[i - 1]:
            raise ValueError("sparse_attention: duplicate page index")
    qc = cache.quest_cache
    pl = torch.tensor(pages, dtype=torch.int32, device=qc.device).view(1, 1, -1)
    cnt = torch.tensor([[len(pages)]], dtype=torch.int32, device=qc.device)
    out, ws = qc.sparse_attend(0, _query_dev(query, cache), pl, cnt, want_weights_sum=True)
    qc.check_status()
    return AttentionOutput(out[0, 0].double().cpu().tolist(), float(ws[0, 0]))


def full_attention(query, cache: KvCache) -> AttentionOutput:
    """attention.cpp:86-92 (empty cache -> ValueError)."""
    if cache.token_count() == 0:
        raise ValueError("full_attention: empty cache")
    out, ws = cache.quest_cache.dense_attend(0, _query_dev(query, cache), want_weights_sum=True)
    return AttentionOutput(out[0, 0].double().cpu().tolist(), float(ws[0, 0]))


def _check_token_set(cache: KvCache, tokens: Sequence[int]) -> List[int]:
    """check_token_set (attention.cpp:19-30), same errors (ValueError / IndexError)."""
    toks = [int(t) for t in tokens]
    if not toks:
        raise ValueError("attention: empty token set")
    n = cache.token_count()
    for i, t in enumerate(toks):
        if t < 0 or t >= n:
            raise IndexError("attention: token index out of range")
        if i > 0 and t <= toks[i - 1]:
            raise ValueError("attention: token set must be strictly ascending")
    return toks


def attend_tokens(query, cache: KvCache, tokens: Sequence[int]) -> AttentionOutput:
    """attention.cpp:69-84: attention over an explicit strictly ascending token set."""
    toks = _check_token_set(cache, tokens)
    if len(np.asarray(query).reshape(-1)) != cache.config().head_dim:
        raise ValueError("attention_logits: query dimension mismatch")
    qc = cache.quest_cache
    tl = torch.tensor(toks, dtype=torch.int32, device=qc.device).view(1, 1, -1)
    cnt = torch.tensor([[len(toks)]], dtype=torch.int32, device=qc.device)
    out, ws = qc.attend_tokens(0, _query_dev(query, cache), tl, cnt, want_weights_sum=True)
    qc.check_status()
    return AttentionOutput(out[0, 0].double().cpu().tolist(), float(ws[0, 0]))


def attention_logits(query, cache: KvCache, token_subset: Optional[Sequence[int]] = None):
    """attention.cpp:34-52 (both overloads): logits q.k/sqrt(d) in ascending token order,
    bitwise the reference's doubles."""
    if token_subset is None:
        toks = list(range(cache.token_count()))
        if not toks:
            raise ValueError("attention: empty token set")
    else:
        toks = _check_token_set(cache, token_subset)
    if len(np.asarray(query).reshape(-1)) != cache.config().head_dim:
        raise ValueError("attention_logits: query dimension mismatch")
    qc = cache.quest_cache
    tl = torch.tensor(toks, dtype=torch.int32, device=qc.device).view(1, 1, -1)
    cnt = torch.tensor([[len(toks)]], dtype=torch.int32, device=qc.device)
    lg = qc.attention_logits(0, _query_dev(query, cache), tl, cnt)
    qc.check_status()
    return lg[0, 0, : len(toks)].cpu().tolist()


def softmax_weights(logits: Sequence[float], device: Optional[int] = None) -> List[float]:
    """attention.cpp:54-67 on the GPU (empty -> ValueError)."""
    lg = np.ascontiguousarray(np.asarray(logits, dtype=np.float64).reshape(-1))
    if lg.size == 0:
        raise ValueError("softmax_weights: empty logits")
    w = np.empty_like(lg)
    lib = _lib.load()
    dev = torch.cuda.current_device() if device is None else device
    check(lib.qk_softmax_weights_host(lg.ctypes.data, lg.size, w.ctypes.data, dev))
    return w.tolist()


def traffic_fraction(page_size: int, token_count: int, token_budget: int) -> float:
    """metrics.cpp:54-66 -- the byte model the roofline uses (host arithmetic only)."""
    if page_size == 0:
        raise ValueError("traffic_fraction: zero page_size")
    if token_count == 0 or token_budget == 0:
        raise ValueError("traffic_fraction: counts must be positive")
    if token_budget > token_count:
        raise ValueError("traffic_fraction: budget exceeds token count")
    k = token_budget // page_size
    return 1.0 / page_size + (k * page_size) / token_count


def quest_step_bytes(head_dim: int, n_pages: int, attended_tokens: int,
                     bytes_per_element: int = 2) -> int:
    """metrics.cpp:105-106: metadata 2*d*bpe per page + K/V 2*d*bpe per attended token."""
    vec = head_dim * bytes_per_element
    return 2 * vec * n_pages + 2 * vec * attended_tokens
