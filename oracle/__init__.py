"""Python bindings of the parity checkers (TEST INFRASTRUCTURE ONLY).

* :class:`Oracle` -- oracle/liboracle.so, the C restatement (questkv_oracle.c).
* :class:`Reference` -- oracle/_ref/libquestkv_ref.so, the unmodified reference library
  compiled from /root/reference by oracle/Makefile, behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) may
import this package.  The product (paper_2406_10774_b200/) never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libquestkv_ref.so")

OK, INVALID_ARGUMENT, OUT_OF_RANGE = 0, 1, 2

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u32 = ctypes.c_uint32


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and _ref/ when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _raise(rc: int, what: str) -> None:
    if rc == OK:
        return
    if rc == INVALID_ARGUMENT:
        raise ValueError(what)
    if rc == OUT_OF_RANGE:
        raise IndexError(what)
    raise RuntimeError(f"{what}: status {rc}")


class Oracle:
    """The C restatement; arrays are float32 [n, dim] (keys/values), float32 [dim] (q)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.qo_build_metadata.argtypes = [_f32p, _u32, _u32, _u32, _f32p, _f32p]
        L.qo_estimate_all.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _f64p]
        L.qo_estimate_page_score.argtypes = [_f32p, _f32p, _f32p, _u32]
        L.qo_estimate_page_score.restype = ctypes.c_double
        L.qo_select_top_k.argtypes = [_f64p, _u32, _u32, _u32, ctypes.c_int, ctypes.c_int, _u32p,
                                      ctypes.POINTER(_u32)]
        L.qo_sparse_attention.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32, _u32p, _u32,
                                          _f64p, ctypes.POINTER(ctypes.c_double)]
        L.qo_full_attention.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _f64p,
                                        ctypes.POINTER(ctypes.c_double)]
        L.qo_naive_attention.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32p, _u32, _f64p]
        L.qo_traffic_fraction.argtypes = [_u32, ctypes.c_uint64, ctypes.c_uint64]
        L.qo_traffic_fraction.restype = ctypes.c_double
        L.qo_quest_step_bytes.argtypes = [_u32, _u32, _u32, ctypes.c_uint64]
        L.qo_quest_step_bytes.restype = ctypes.c_uint64
        L.qo_validate_config.argtypes = [_u32, _u32, _u32]
        self.lib = L

    def validate_config(self, head_dim, page_size, bpe=2):
        _raise(self.lib.qo_validate_config(head_dim, page_size, bpe), "CacheConfig")

    def metadata(self, keys, page_size: int) -> Tuple[np.ndarray, np.ndarray]:
        k = _f32(keys)
        n, d = k.shape
        P = (n + page_size - 1) // page_size
        mn = np.zeros((P, d), np.float32)
        mx = np.zeros((P, d), np.float32)
        self.lib.qo_build_metadata(k, n, d, page_size, mn, mx)
        return mn, mx

    def estimate_page_score(self, q, mn, mx) -> float:
        q = _f32(q)
        return float(self.lib.qo_estimate_page_score(q, _f32(mn), _f32(mx), q.shape[0]))

    def estimate_all(self, q, mn, mx) -> np.ndarray:
        mn = _f32(mn).reshape(-1, len(q))
        P = mn.shape[0]
        out = np.zeros(max(P, 1), np.float64)
        _raise(self.lib.qo_estimate_all(_f32(q), mn, _f32(mx), P, len(q), out), "estimate_all")
        return out[:P]

    def select_top_k(self, scores, page_size: int, budget: int, force: bool = True,
                     enabled: bool = True) -> np.ndarray:
        s = np.ascontiguousarray(np.asarray(scores, dtype=np.float64))
        P = s.shape[0]
        out = np.zeros(max(P, 1), np.uint32)
        cnt = _u32()
        _raise(self.lib.qo_select_top_k(s, P, page_size, budget, int(force), int(enabled), out,
                                        ctypes.byref(cnt)), "select_top_k")
        return out[: cnt.value].copy()

    def sparse_attention(self, q, keys, values, page_size: int, pages) -> np.ndarray:
        k, v, q = _f32(keys), _f32(values), _f32(q)
        n, d = k.shape
        p = np.ascontiguousarray(np.asarray(pages, dtype=np.uint32))
        out = np.zeros(d, np.float64)
        w = ctypes.c_double()
        _raise(self.lib.qo_sparse_attention(q, k, v, n, d, page_size, p, p.shape[0], out,
                                            ctypes.byref(w)), "sparse_attention")
        return out

    def full_attention(self, q, keys, values) -> np.ndarray:
        k, v, q = _f32(keys), _f32(values), _f32(q)
        n, d = k.shape
        out = np.zeros(d, np.float64)
        w = ctypes.c_double()
        _raise(self.lib.qo_full_attention(q, k, v, n, d, out, ctypes.byref(w)), "full_attention")
        return out

    def naive_attention(self, q, keys, values, tokens) -> np.ndarray:
        k, v, q = _f32(keys), _f32(values), _f32(q)
        n, d = k.shape
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
        out = np.zeros(d, np.float64)
        _raise(self.lib.qo_naive_attention(q, k, v, n, d, t, t.shape[0], out), "naive_attention")
        return out

    def quest_step(self, q, keys, values, page_size: int, budget: int, force: bool = True,
                   enabled: bool = True):
        """(scores, pages, output) of one estimate -> select -> sparse step."""
        k = _f32(keys)
        mn, mx = self.metadata(k, page_size)
        scores = self.estimate_all(q, mn, mx)
        pages = self.select_top_k(scores, page_size, budget, force, enabled)
        out = self.sparse_attention(q, k, values, page_size, pages)
        return scores, pages, out

    def group_quest_step(self, qs, keys, values, page_size: int, budget: int,
                         reduce: str = "max", force: bool = True, enabled: bool = True):
        """Checker of the GQA group-shared variant (not a reference
        function -- composed from the restated ones): per query head g, estimate_all
        (criticality.cpp:25-34) on the shared KV head's metadata; the group score of a page
        is max_g (exact) or the fp64 sum in head order ((s_0 + s_1) + s_2) + ...; ONE
        select_top_k (criticality.cpp:36-81) on the group scores; every head's
        sparse_attention (attention.cpp:94-116) over that page set.
        Returns (group_scores, pages, outputs [G][d])."""
        qs = _f32(qs)
        k = _f32(keys)
        mn, mx = self.metadata(k, page_size)
        per_head = [self.estimate_all(q, mn, mx) for q in qs]
        group = per_head[0].copy()
        for s in per_head[1:]:
            group = np.maximum(group, s) if reduce == "max" else group + s  # IEEE fp64 adds
        pages = self.select_top_k(group, page_size, budget, force, enabled)
        outs = np.stack([self.sparse_attention(q, k, values, page_size, pages) for q in qs])
        return group, pages, outs

    def traffic_fraction(self, page_size, token_count, budget) -> float:
        return float(self.lib.qo_traffic_fraction(page_size, token_count, budget))

    def quest_step_bytes(self, dim, bpe, n_pages, attended) -> int:
        return int(self.lib.qo_quest_step_bytes(dim, bpe, n_pages, attended))


class Reference:
    """The unmodified reference library (oracle/_ref), same call shapes as Oracle."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (build with make -C oracle ref)")
        L = ctypes.CDLL(path)
        L.ref_validate_config.argtypes = [_u32, _u32, _u32]
        L.ref_metadata.argtypes = [_f32p, _f32p, _u32, _u32, _u32, _f32p, _f32p]
        L.ref_estimate_all.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32, _f64p]
        L.ref_select_top_k.argtypes = [_f64p, _u32, _u32, _u32, _u32, ctypes.c_int, ctypes.c_int,
                                       _u32p, ctypes.POINTER(_u32)]
        L.ref_sparse_attention.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32, _u32p, _u32,
                                           _f64p, ctypes.POINTER(ctypes.c_double)]
        L.ref_full_attention.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32, _f64p,
                                         ctypes.POINTER(ctypes.c_double)]
        L.ref_naive_attention.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32p, _u32, _f64p]
        L.ref_quest_step.argtypes = [_f32p, _f32p, _f32p, _u32, _u32, _u32, _u32, ctypes.c_int,
                                     ctypes.c_int, _f64p, _u32p, ctypes.POINTER(_u32), _f64p]
        L.ref_traffic_fraction.argtypes = [_u32, ctypes.c_uint64, ctypes.c_uint64]
        L.ref_traffic_fraction.restype = ctypes.c_double
        L.ref_layer_create.argtypes = [_f32p, _f32p, _u32, _u32, _u32, _u32]
        L.ref_layer_create.restype = ctypes.c_void_p
        L.ref_layer_destroy.argtypes = [ctypes.c_void_p]
        L.ref_layer_step.argtypes = [ctypes.c_void_p, _f32p, _u32, ctypes.c_int, _u32, _u32, _u32,
                                     ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double), _f64p]
        L.ref_write_trace.argtypes = [ctypes.c_char_p, _u32, _u32, _f32p, _f32p, _f32p]
        L.ref_read_trace.argtypes = [ctypes.c_char_p, ctypes.POINTER(_u32), ctypes.POINTER(_u32),
                                     _f32p, _f32p, _f32p, _u32]
        L.ref_recall_at_n.argtypes = [_u32p, _u32, _f32p, _f32p, _f32p, _u32, _u32, _u32, _u32,
                                      ctypes.POINTER(ctypes.c_double)]
        self.lib = L

    def write_trace(self, path, keys, values, queries):
        """The reference's write_trace (workloads.cpp) of float32 [n, d] arrays."""
        k, v, q = (np.ascontiguousarray(a, np.float32) for a in (keys, values, queries))
        n, d = k.shape
        _raise(self.lib.ref_write_trace(str(path).encode(), d, n, k, v,
                                        q), "write_trace")

    def read_trace(self, path, cap=1 << 16):
        """The reference's read_trace: (head_dim, keys, values, queries); raises ValueError
        on trace_format_error (status 4)."""
        d, n = _u32(0), _u32(0)
        e = np.zeros(0, np.float32)
        st = self.lib.ref_read_trace(str(path).encode(), ctypes.byref(d), ctypes.byref(n), e, e, e, 0)
        if st:
            raise ValueError(f"read_trace: status {st}")
        k = np.zeros((n.value, d.value), np.float32)
        v, q = np.zeros_like(k), np.zeros_like(k)
        _raise(self.lib.ref_read_trace(str(path).encode(), ctypes.byref(d), ctypes.byref(n), k,
                                       v, q, n.value), "read_trace")
        return d.value, k, v, q

    def recall_at_n(self, selected, query, keys, values, page_size, top_n):
        sel = np.ascontiguousarray(selected, np.uint32)
        k, v = np.ascontiguousarray(keys, np.float32), np.ascontiguousarray(values, np.float32)
        q = np.ascontiguousarray(query, np.float32)
        r = ctypes.c_double(0.0)
        _raise(self.lib.ref_recall_at_n(sel, len(sel), q, k, v,
                                        k.shape[0], k.shape[1], page_size, top_n, ctypes.byref(r)),
               "recall_at_n")
        return r.value

    def validate_config(self, head_dim, page_size, bpe=2):
        _raise(self.lib.ref_validate_config(head_dim, page_size, bpe), "CacheConfig")

    def metadata(self, keys, page_size: int):
        k = _f32(keys)
        n, d = k.shape
        P = (n + page_size - 1) // page_size
        mn = np.zeros((P, d), np.float32)
        mx = np.zeros((P, d), np.float32)
        _raise(self.lib.ref_metadata(k, k, n, d, page_size, mn, mx), "metadata")
        return mn, mx

    def estimate_all(self, q, keys, page_size: int) -> np.ndarray:
        k = _f32(keys)
        n, d = k.shape
        P = (n + page_size - 1) // page_size
        out = np.zeros(max(P, 1), np.float64)
        _raise(self.lib.ref_estimate_all(_f32(q), k, k, n, d, page_size, out), "estimate_all")
        return out[:P]

    def select_top_k(self, scores, page_size: int, budget: int, force: bool = True,
                     enabled: bool = True, n_pages: Optional[int] = None) -> np.ndarray:
        s = np.ascontiguousarray(np.asarray(scores, dtype=np.float64))
        P = s.shape[0] if n_pages is None else n_pages
        out = np.zeros(max(P, 1), np.uint32)
        cnt = _u32()
        _raise(self.lib.ref_select_top_k(s if s.size else np.zeros(1), s.shape[0], P, page_size,
                                         budget, int(force), int(enabled), out, ctypes.byref(cnt)),
               "select_top_k")
        return out[: cnt.value].copy()

    def sparse_attention(self, q, keys, values, page_size: int, pages):
        k, v = _f32(keys), _f32(values)
        n, d = k.shape
        p = np.ascontiguousarray(np.asarray(pages, dtype=np.uint32))
        out = np.zeros(d, np.float64)
        w = ctypes.c_double()
        _raise(self.lib.ref_sparse_attention(_f32(q), k, v, n, d, page_size,
                                             p if p.size else np.zeros(1, np.uint32), p.shape[0],
                                             out, ctypes.byref(w)), "sparse_attention")
        return out, w.value

    def full_attention(self, q, keys, values, page_size: int = 16):
        k, v = _f32(keys), _f32(values)
        n, d = k.shape
        out = np.zeros(d, np.float64)
        w = ctypes.c_double()
        _raise(self.lib.ref_full_attention(_f32(q), k, v, n, d, page_size, out, ctypes.byref(w)),
               "full_attention")
        return out, w.value

    def naive_attention(self, q, keys, values, tokens) -> np.ndarray:
        k, v = _f32(keys), _f32(values)
        n, d = k.shape
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
        out = np.zeros(d, np.float64)
        _raise(self.lib.ref_naive_attention(_f32(q), k, v, n, d, t, t.shape[0], out),
               "naive_attention")
        return out

    def quest_step(self, q, keys, values, page_size: int, budget: int, force: bool = True,
                   enabled: bool = True):
        k, v = _f32(keys), _f32(values)
        n, d = k.shape
        P = (n + page_size - 1) // page_size
        scores = np.zeros(max(P, 1), np.float64)
        pages = np.zeros(max(P, 1), np.uint32)
        cnt = _u32()
        out = np.zeros(d, np.float64)
        _raise(self.lib.ref_quest_step(_f32(q), k, v, n, d, page_size, budget, int(force),
                                       int(enabled), scores, pages, ctypes.byref(cnt), out),
               "quest_step")
        return scores[:P], pages[: cnt.value].copy(), out

    # CPU baseline: one layer of independent heads timed like cmd_bench.
    def layer(self, keys, values, page_size: int) -> "RefLayer":
        return RefLayer(self, keys, values, page_size)


class RefLayer:
    def __init__(self, ref: Reference, keys, values, page_size: int):
        k, v = _f32(keys), _f32(values)  # [H, n, d]
        self.ref = ref
        self.H, self.n, self.d = k.shape
        self.h = ref.lib.ref_layer_create(k, v, self.H, self.n, self.d, page_size)

    def step(self, queries, budget: int, dense: bool = False, threads: int = 1, warmup: int = 1,
             reps: int = 3):
        """Returns (mean_ns, min_ns, outputs [H, d])."""
        q = _f32(queries)
        out = np.zeros((self.H, self.d), np.float64)
        mean, best = ctypes.c_double(), ctypes.c_double()
        _raise(self.ref.lib.ref_layer_step(self.h, q, budget, 1 if dense else 0, threads, warmup,
                                           reps, ctypes.byref(mean), ctypes.byref(best), out),
               "ref_layer_step")
        return mean.value, best.value, out

    def close(self):
        if self.h:
            self.ref.lib.ref_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
