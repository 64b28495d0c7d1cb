"""Generate tests/golden/golden_v1.npz from the UNMODIFIED reference library.

Run in the dev container (needs /root/reference to build oracle/_ref):

    make -C oracle && python tests/golden/make_golden.py

Every case stores fp16-representable inputs (as float32) and the reference's outputs:
page metadata (KvCache::page_metadata), estimate_all scores, select_top_k pages for several
selection configs, and sparse/full attention outputs (fp64).  The file is committed so the
GPU box (which has no /root/reference) can check against it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def half(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)


def gaussian_case(rng, n, d, sd):
    k = half(rng.standard_normal((n, d)) * sd)
    v = half(rng.standard_normal((n, d)) * sd)
    q = half(rng.standard_normal(d) * sd)
    return q, k, v


def main() -> None:
    ref = Reference()
    rng = np.random.default_rng(20240611)
    cases = {}

    def add(name, q, k, v, S, budgets):
        P = (k.shape[0] + S - 1) // S
        mn, mx = ref.metadata(k, S)
        scores = ref.estimate_all(q, k, S)
        full, _ = ref.full_attention(q, k, v, S)
        entry = dict(q=q.astype(np.float16), k=k.astype(np.float16), v=v.astype(np.float16),
                     S=np.int64(S), meta_min=mn.astype(np.float16), meta_max=mx.astype(np.float16),
                     scores=scores,
                     full=full)
        sel_rows = []
        for (budget, force, enabled) in budgets:
            try:
                pages = ref.select_top_k(scores, S, budget, force, enabled)
                out, _ = ref.sparse_attention(q, k, v, S, pages)
                status = 0
            except ValueError:
                pages, out, status = np.zeros(0, np.uint32), np.zeros(k.shape[1]), 1
            sel_rows.append((budget, int(force), int(enabled), status, pages, out))
        entry["sel_cfg"] = np.array([[b, f, e, s] for (b, f, e, s, _, _) in sel_rows], np.int64)
        width = max(P, 1)
        pages_mat = np.full((len(sel_rows), width), -1, np.int64)
        outs = np.zeros((len(sel_rows), k.shape[1]), np.float64)
        for i, (_, _, _, _, pages, out) in enumerate(sel_rows):
            pages_mat[i, : len(pages)] = pages
            outs[i] = out
        entry["sel_pages"] = pages_mat
        entry["sel_out"] = outs
        for key, val in entry.items():
            cases[f"{name}/{key}"] = val

    budget_sweep = lambda S, L: [  # noqa: E731
        (S, True, True), (S, False, True), (S * 2, True, True), (S * 4, False, True),
        (max(S, (L // 4) // S * S), True, True), (L + S, True, True), (S - 1 if S > 1 else 0, True, True),
        (S * 3, True, False)]

    # Llama-shaped heads (d=128, S=16) at several lengths incl. partial last pages.
    for L in (1, 15, 16, 17, 257, 1000, 2047):
        q, k, v = gaussian_case(rng, L, 128, 1.0 / np.sqrt(128))
        add(f"llama_L{L}", q, k, v, 16, budget_sweep(16, L))
    # Other geometries (padding paths: d < 64, d = 64, odd S).
    for (d, S, L) in ((2, 4, 37), (3, 8, 100), (16, 8, 200), (64, 16, 700), (100, 7, 300)):
        q, k, v = gaussian_case(rng, L, d, 1.0)
        add(f"geom_d{d}_S{S}_L{L}", q, k, v, S, budget_sweep(S, L))
    # Tie stress: keys from a tiny value set -> many equal page scores.
    vals = np.array([-1.0, -0.5, 0.0, 0.5, 1.0], np.float32)
    k = vals[rng.integers(0, 5, size=(640, 8))]
    v = half(rng.standard_normal((640, 8)))
    q = np.array([1, 1, 0, 0, -1, 0, 0, 1], np.float32)
    add("ties_d8_S4", q, k, v, 4, budget_sweep(4, 640))
    # Signed zeros in keys (first-seen sign kept in metadata).
    k = np.zeros((64, 4), np.float32)
    k[::2] = -0.0
    k[1::3, 1] = -0.0
    k[5, 2] = 1.0
    v = half(rng.standard_normal((64, 4)))
    add("zeros_d4_S8", np.array([1, -1, 0.5, -0.5], np.float32), k, v, 8, budget_sweep(8, 64))

    names = sorted({key.split("/")[0] for key in cases})
    cases["__names__"] = np.array(names)
    np.savez_compressed(OUT, **cases)
    print(f"wrote {OUT}: {len(names)} cases, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
