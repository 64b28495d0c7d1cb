"""Generate the QKVTRACE / recall golden fixtures from the UNMODIFIED reference library.

Run in the dev container (needs /root/reference to build oracle/_ref):

    make -C oracle && python tests/golden/make_trace_golden.py

Writes
  tests/golden/trace_ref_v1.qkvtrace  -- a 96-step, d=32 trace serialised by the reference's
                                         write_trace (workloads.cpp:151-164); its payload is
                                         trace_payload() below (seeded, fp16-representable).
  tests/golden/recall_v1.npz          -- recall_at_n (metrics.cpp:12-38) of the reference for
                                         a set of (selection, query, cache prefix, n) cases,
                                         including exact logit ties.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def trace_payload():
    rng = np.random.default_rng(20240614)
    n, d = 96, 32
    f = lambda: rng.standard_normal((n, d)).astype(np.float16).astype(np.float32)  # noqa: E731
    return f(), f(), f()


def recall_cases():
    rng = np.random.default_rng(7)
    cases = []
    for n_tok, d, n, n_sel in [(64, 16, 8, 20), (200, 32, 16, 48), (37, 8, 5, 5), (128, 16, 32, 128)]:
        k = rng.standard_normal((n_tok, d)).astype(np.float16).astype(np.float32)
        v = rng.standard_normal((n_tok, d)).astype(np.float16).astype(np.float32)
        q = rng.standard_normal(d).astype(np.float16).astype(np.float32)
        sel = np.sort(rng.choice(n_tok, size=n_sel, replace=False)).astype(np.uint32)
        cases.append((sel, q, k, v, n))
    # exact ties: repeated keys -> equal logits, the older token ranks first
    k = np.tile(np.eye(8, dtype=np.float32)[:4], (10, 1))
    q = np.ones(8, np.float32)
    cases.append((np.arange(0, 40, 2, dtype=np.uint32), q, k, k.copy(), 10))
    return cases


def main() -> None:
    ref = Reference()
    k, v, q = trace_payload()
    ref.write_trace(os.path.join(HERE, "trace_ref_v1.qkvtrace"), k, v, q)
    out = {}
    for i, (sel, qq, kk, vv, n) in enumerate(recall_cases()):
        out[f"c{i}/sel"] = sel
        out[f"c{i}/q"] = qq
        out[f"c{i}/k"] = kk
        out[f"c{i}/v"] = vv
        out[f"c{i}/n"] = np.int64(n)
        out[f"c{i}/recall"] = np.float64(ref.recall_at_n(sel, qq, kk, vv, 16, n))
    np.savez_compressed(os.path.join(HERE, "recall_v1.npz"), **out)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
