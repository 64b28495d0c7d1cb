"""QKVTRACE I/O and the recall metric (paper_2406_10774_b200/trace.py) against the
reference: a trace file written by the reference's write_trace (tests/golden/
trace_ref_v1.qkvtrace, tests/golden/make_trace_golden.py), byte-identical writing, the
reference's error classes, and recall_at_n equal to the reference's on golden and live
cases."""

import os

import numpy as np
import pytest

from paper_2406_10774_b200 import trace as tr

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TRACE = os.path.join(GOLD, "trace_ref_v1.qkvtrace")


def payload():
    rng = np.random.default_rng(20240614)  # tests/golden/make_trace_golden.py:trace_payload
    n, d = 96, 32
    f = lambda: rng.standard_normal((n, d)).astype(np.float16).astype(np.float32)  # noqa: E731
    return f(), f(), f()


def test_read_reference_written_trace():
    t = tr.read_trace(TRACE)
    k, v, q = payload()
    assert t.head_dim == 32 and t.length == 96
    assert t == tr.make_trace(k, v, q)


def test_write_is_byte_identical_to_reference(tmp_path):
    p = tmp_path / "t.qkvtrace"
    tr.write_trace(p, tr.make_trace(*payload()))
    assert p.read_bytes() == open(TRACE, "rb").read()


def test_roundtrip_empty_and_small(tmp_path):
    for n, d in [(0, 4), (1, 1), (5, 128)]:
        rng = np.random.default_rng(n + d)
        t = tr.make_trace(*(rng.standard_normal((n, d)).astype(np.float32) for _ in range(3)))
        p = tmp_path / f"t{n}_{d}.qkvtrace"
        tr.write_trace(p, t)
        assert tr.read_trace(p) == t


def _corrupt(kind):
    data = bytearray(open(TRACE, "rb").read())
    if kind == "magic":
        data[0:1] = b"X"
    elif kind == "version":
        data[8] = 2
    elif kind == "head_dim":
        data[9:13] = b"\0\0\0\0"
    elif kind.startswith("cut"):
        data = data[: int(kind[3:])]
    elif kind == "trailing":
        data += b"\0"
    return bytes(data)


@pytest.mark.parametrize("kind,err", [
    ("magic", tr.TraceFormatError), ("version", tr.TraceFormatError),
    ("head_dim", tr.TraceFormatError), ("trailing", tr.TraceFormatError),
    ("cut4", tr.TraceTruncatedError), ("cut8", tr.TraceTruncatedError),
    ("cut12", tr.TraceTruncatedError), ("cut16", tr.TraceTruncatedError),
    ("cut500", tr.TraceTruncatedError),
])
def test_read_errors_match_reference(tmp_path, kind, err, request):
    p = tmp_path / f"bad_{kind}.qkvtrace"
    p.write_bytes(_corrupt(kind))
    with pytest.raises(err):
        tr.read_trace(p)
    from oracle import REF_SO
    if os.path.exists(REF_SO):  # the reference's reader rejects it too (trace_format_error)
        ref = request.getfixturevalue("reference")
        with pytest.raises(ValueError):
            ref.read_trace(p)


def test_recall_matches_reference_golden():
    z = np.load(os.path.join(GOLD, "recall_v1.npz"))
    i = 0
    while f"c{i}/sel" in z.files:
        got = tr.recall_at_n(z[f"c{i}/sel"], z[f"c{i}/q"], z[f"c{i}/k"], int(z[f"c{i}/n"]))
        assert got == float(z[f"c{i}/recall"]), i
        i += 1
    assert i >= 5


def test_recall_errors():
    k = np.ones((4, 8), np.float32)
    with pytest.raises(ValueError):
        tr.recall_at_n([0], np.ones(8, np.float32), k, 0)
    with pytest.raises(ValueError):
        tr.recall_at_n([0], np.ones(8, np.float32), k, 5)
    with pytest.raises(IndexError):
        tr.recall_at_n([4], np.ones(8, np.float32), k, 2)


def test_recall_vs_reference_live(reference):
    rng = np.random.default_rng(3)
    for _ in range(20):
        n_tok, d = int(rng.integers(8, 300)), int(rng.choice([8, 32, 128]))
        k = rng.standard_normal((n_tok, d)).astype(np.float16).astype(np.float32)
        q = rng.standard_normal(d).astype(np.float16).astype(np.float32)
        n = int(rng.integers(1, n_tok + 1))
        sel = np.sort(rng.choice(n_tok, size=int(rng.integers(1, n_tok + 1)), replace=False))
        want = reference.recall_at_n(sel.astype(np.uint32), q, k, k, 16, n)
        assert tr.recall_at_n(sel, q, k, n) == want
