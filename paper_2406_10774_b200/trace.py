"""QKVTRACE decode traces and the recall / traffic metrics over the GPU decode path.

A trace is one attention head's decode history: per step a key, a value and a query
(float32, head_dim each).  The binary format is the reference's (R/core/src/workloads.cpp
:151-196, R = /root/reference/proj):

    "QKVTRACE" (8 bytes) | version u8 = 1 | head_dim u32 LE | length u32 LE |
    length x (key f32[d] | value f32[d] | query f32[d])  (little-endian IEEE-754)

`read_trace` raises `TraceFormatError` for a bad magic, an unsupported version, a zero
head_dim or trailing bytes, and `TraceTruncatedError` (a subclass) for a short file, as the
reference throws trace_format_error / trace_truncated_error (workloads.hpp:66-78).

`recall_at_n` is the reference's metric (R/core/src/metrics.cpp:12-38): the fraction of the
n tokens with the largest exact logits (fp64 dot products accumulated in ascending channel
order, divided by sqrt(d), attention.cpp:13-46; ties to the older token) that the
selection attends.  `replay_quest` drives a trace through the B200 decode step one token at
a time (append, estimate, top-K, attend: the fused kernel) and reports per-step recall,
the reference's counted traffic ratio (cmd_recall.cpp:76-88: pages + attended tokens over
tokens) and the output error against dense attention (metrics.cpp:155-168), as the
reference's `recall` command does for the Quest policy.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

MAGIC = b"QKVTRACE"
VERSION = 1


class TraceFormatError(ValueError):
    """A malformed trace (the reference's trace_format_error)."""


class TraceTruncatedError(TraceFormatError):
    """A trace shorter than its header promises (trace_truncated_error)."""


@dataclass
class DecodeTrace:
    """keys / values / queries: float32 [length, head_dim]."""

    head_dim: int
    keys: np.ndarray
    values: np.ndarray
    queries: np.ndarray

    @property
    def length(self) -> int:
        return int(self.keys.shape[0])

    def __eq__(self, other) -> bool:  # payload equality, as DecodeTrace::operator==
        return (isinstance(other, DecodeTrace) and self.head_dim == other.head_dim
                and np.array_equal(self.keys.view(np.uint32), other.keys.view(np.uint32))
                and np.array_equal(self.values.view(np.uint32), other.values.view(np.uint32))
                and np.array_equal(self.queries.view(np.uint32), other.queries.view(np.uint32)))


def make_trace(keys, values, queries) -> DecodeTrace:
    k, v, q = (np.ascontiguousarray(a, dtype=np.float32) for a in (keys, values, queries))
    if k.ndim != 2 or k.shape != v.shape or k.shape != q.shape:
        raise ValueError("make_trace: keys, values and queries must share one [length, d] shape")
    return DecodeTrace(int(k.shape[1]), k, v, q)


def write_trace(path, trace: DecodeTrace) -> None:
    """Serialise `trace` (byte-identical to the reference's write_trace)."""
    n, d = trace.length, trace.head_dim
    body = np.empty((n, 3, d), dtype="<f4")
    body[:, 0], body[:, 1], body[:, 2] = trace.keys, trace.values, trace.queries
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(bytes([VERSION]))
        f.write(struct.pack("<II", d, n))
        f.write(body.tobytes())


def read_trace(path) -> DecodeTrace:
    """Parse a QKVTRACE file; errors as the reference's read_trace."""
    try:
        data = open(path, "rb").read()
    except OSError as e:
        raise TraceFormatError(f"cannot open trace file: {path}") from e
    if len(data) < len(MAGIC):
        raise TraceTruncatedError("trace file truncated")
    if data[:8] != MAGIC:
        raise TraceFormatError("bad trace magic")
    if len(data) < 9:
        raise TraceTruncatedError("trace file truncated")
    if data[8] != VERSION:
        raise TraceFormatError("unsupported trace version")
    if len(data) < 13:
        raise TraceTruncatedError("trace file truncated")
    (d,) = struct.unpack_from("<I", data, 9)
    if d == 0:
        raise TraceFormatError("trace head_dim is zero")
    if len(data) < 17:
        raise TraceTruncatedError("trace file truncated")
    (n,) = struct.unpack_from("<I", data, 13)
    need = 17 + n * 3 * d * 4
    if len(data) < need:
        raise TraceTruncatedError("trace file truncated")
    if len(data) > need:
        raise TraceFormatError("trailing bytes after trace payload")
    body = np.frombuffer(data, dtype="<f4", count=n * 3 * d, offset=17).reshape(n, 3, d)
    body = body.astype(np.float32)
    return DecodeTrace(d, np.ascontiguousarray(body[:, 0]), np.ascontiguousarray(body[:, 1]),
                       np.ascontiguousarray(body[:, 2]))


def exact_logits(query, keys) -> np.ndarray:
    """attention_logits: sum_i double(q_i) * double(k_i) in ascending i (a separate multiply
    and add per channel, as the reference compiles without contraction), / sqrt(d)."""
    q = np.asarray(query, dtype=np.float32).astype(np.float64)
    k = np.asarray(keys, dtype=np.float32).astype(np.float64)
    acc = np.zeros(k.shape[0], dtype=np.float64)
    for i in range(k.shape[1]):
        acc = acc + q[i] * k[:, i]
    return acc / math.sqrt(float(k.shape[1]))


def recall_at_n(selected_tokens, query, keys, n: int) -> float:
    """The reference's recall_at_n over the first len(keys) tokens of a cache."""
    count = int(np.asarray(keys).shape[0])
    if n == 0:
        raise ValueError("recall_at_n: n must be >= 1")
    if n > count:
        raise ValueError("recall_at_n: n exceeds token count")
    sel = np.asarray(selected_tokens, dtype=np.int64)
    if sel.size and (sel.min() < 0 or sel.max() >= count):
        raise IndexError("recall_at_n: selected token out of range")
    logits = exact_logits(query, keys)
    order = np.lexsort((np.arange(count), -logits))[:n]  # logit desc, then older token
    chosen = np.zeros(count, dtype=bool)
    chosen[sel] = True
    return float(chosen[order].sum()) / float(n)


def output_error(sparse, full) -> float:
    """metrics.cpp:155-168: ||sparse - full|| / (||full|| + 1e-12)."""
    s, f = np.asarray(sparse, np.float64), np.asarray(full, np.float64)
    if s.shape != f.shape:
        raise ValueError("output_error: dimension mismatch")
    return float(np.sqrt(((s - f) ** 2).sum()) / (np.sqrt((f * f).sum()) + 1e-12))


@dataclass
class StepRow:
    step: int
    recall: float
    traffic: float
    error: float
    pages: List[int]


@dataclass
class RecallReport:
    budget: int
    top_n: int
    rows: List[StepRow]

    @property
    def mean_recall(self) -> float:
        return float(np.mean([r.recall for r in self.rows])) if self.rows else 0.0

    @property
    def mean_traffic(self) -> float:
        return float(np.mean([r.traffic for r in self.rows])) if self.rows else 0.0

    @property
    def mean_error(self) -> float:
        return float(np.mean([r.error for r in self.rows])) if self.rows else 0.0


def replay_quest(trace: DecodeTrace, budget: int, top_n: int, page_size: int = 16,
                 force_include_recent: bool = True, device: Optional[int] = None) -> RecallReport:
    """Replay `trace` through the GPU decode step (QuestCache, one head): per step append the
    key/value, estimate, select and attend (one fused launch), then score the selection as the
    reference's `recall` command does for the Quest policy (cmd_recall.cpp:57-99).  The trace
    values are stored as fp16 on the GPU; recall and the dense comparator use the fp16-rounded
    keys/values the GPU actually holds."""
    import torch

    from .questkv import QuestCache

    if budget < page_size:
        raise ValueError("select_top_k: token_budget below page_size")
    if budget > trace.length:
        raise ValueError(f"budget {budget} exceeds trace length {trace.length}")
    d = trace.head_dim
    qc = QuestCache(d, page_size, num_q_heads=1, num_kv_heads=1, max_tokens=trace.length + 1,
                    device=device)
    dev = qc.device
    k16 = trace.keys.astype(np.float16)
    v16 = trace.values.astype(np.float16)
    q16 = trace.queries.astype(np.float16)
    kf, vf = k16.astype(np.float32), v16.astype(np.float32)
    P = (trace.length + page_size - 1) // page_size
    pages = torch.full((1, 1, P), -1, dtype=torch.int32, device=dev)
    counts = torch.zeros((1, 1), dtype=torch.int32, device=dev)
    rows: List[StepRow] = []
    try:
        for t in range(trace.length):
            q = torch.from_numpy(q16[t]).to(dev).view(1, 1, d)
            k = torch.from_numpy(k16[t]).to(dev).view(1, 1, d)
            v = torch.from_numpy(v16[t]).to(dev).view(1, 1, d)
            out = qc.decode_step(0, q, k, v, budget, force_include_recent, True, pages=pages,
                                 counts=counts)
            if t + 1 < top_n:
                continue
            n_sel = int(counts[0, 0].item())
            sel_pages = pages[0, 0, :n_sel].cpu().numpy().astype(np.int64)
            count = t + 1
            tokens = np.concatenate([np.arange(p * page_size, min((p + 1) * page_size, count))
                                     for p in sel_pages]) if n_sel else np.zeros(0, np.int64)
            rec = recall_at_n(tokens, q16[t].astype(np.float32), kf[:count], top_n)
            n_pages = (count + page_size - 1) // page_size
            traffic = float(n_pages + tokens.size) / float(count)
            ref = qc.dense_attend(0, q).cpu().numpy().reshape(-1)  # the dense comparator
            err = output_error(out.cpu().numpy().reshape(-1), ref)
            rows.append(StepRow(t, rec, traffic, err, sel_pages.tolist()))
    finally:
        qc.close()
    return RecallReport(budget, top_n, rows)
