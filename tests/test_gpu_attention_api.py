"""GPU parity of the rest of the reference's attention.hpp surface (attention.cpp:19-84):
attention_logits (both overloads, bitwise), softmax_weights, attend_tokens (token-granular,
check_token_set errors), weights_sum_check -- restating R/tests/test_attention.cpp:51-120
and :248-257 -- plus select_top_k on arbitrary PageScore vectors (criticality.cpp:36-81
literally: any order, repeated pages, -0 == +0) against the C oracle's rule."""

import math

import numpy as np
import pytest
import torch

from conftest import half

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qk():
    from paper_2406_10774_b200 import questkv

    return questkv


def cache_of(qk, d, S, keys, vals):
    c = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=max(len(keys), 1) + 16)
    for k, v in zip(keys, vals):
        c.append(k, v)
    return c


def ref_logits(q, keys):
    """attention.cpp:34-46 in numpy: exact fp64 products summed sequentially (cumsum is
    sequential), divided by sqrt(d)."""
    prods = np.asarray(keys, np.float64) * np.asarray(q, np.float64)[None, :]
    return np.cumsum(prods, axis=1)[:, -1] / math.sqrt(len(q))


def test_logit_worked_examples(qk):
    # test_attention.cpp:51-61
    c = cache_of(qk, 4, 4, [[1, 1, 1, 1]], [[0] * 4])
    assert qk.attention_logits([1, 1, 1, 1], c) == [2.0]
    o = cache_of(qk, 2, 2, [[1, 0]], [[0, 0]])
    assert qk.attention_logits([0, 1], o) == [0.0]


@pytest.mark.parametrize("d,S,L", [(3, 2, 5), (64, 16, 1000), (128, 16, 777), (100, 8, 300)])
def test_logits_bitwise(qk, d, S, L):
    rng = np.random.default_rng(d + L)
    keys = half(rng.standard_normal((L, d)))
    vals = half(rng.standard_normal((L, d)))
    q = half(rng.standard_normal(d))
    c = cache_of(qk, d, S, keys, vals)
    got = np.array(qk.attention_logits(q, c))
    want = ref_logits(q, keys)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    sub = list(range(1, L, 3))
    got = np.array(qk.attention_logits(q, c, sub))
    assert np.array_equal(got.view(np.uint64), want[sub].view(np.uint64))


def test_logit_subset_validation(qk):
    # test_attention.cpp:73-83
    rng = np.random.default_rng(6)
    c = cache_of(qk, 2, 2, half(rng.standard_normal((4, 2))), half(rng.standard_normal((4, 2))))
    q = half(rng.standard_normal(2))
    with pytest.raises(IndexError):
        qk.attention_logits(q, c, [0, 4])
    with pytest.raises(ValueError):
        qk.attention_logits(q, c, [2, 1])
    with pytest.raises(ValueError):
        qk.attention_logits(q, c, [1, 1])
    empty = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2), capacity=4)
    with pytest.raises(ValueError):
        qk.attention_logits(q, empty)


def test_device_logits_and_token_list_errors(qk):
    """The batched device entry points validate lists on the device (check_token_set)."""
    qc = qk.QuestCache(64, 16, num_q_heads=2, max_tokens=512)
    k = (torch.randn((2, 300, 64), device="cuda") / 8).half()
    qc.prefill(0, 0, k, k)
    q = (torch.randn((1, 2, 64), device="cuda") / 8).half()
    toks = torch.tensor([[[0, 5, 9], [1, 2, 300]]], dtype=torch.int32, device="cuda")
    cnt = torch.tensor([[3, 3]], dtype=torch.int32, device="cuda")
    qc.attention_logits(0, q, toks, cnt)
    with pytest.raises(IndexError):
        qc.check_status()
    toks[0, 1, 2] = 1
    qc.attend_tokens(0, q, toks, cnt)
    with pytest.raises(ValueError):
        qc.check_status()
    toks[0, 1, 2] = 299
    out, ws = qc.attend_tokens(0, q, toks, cnt, want_weights_sum=True)
    qc.check_status()
    assert torch.isfinite(out).all() and torch.allclose(ws, torch.ones_like(ws), atol=1e-6)
    lg = qc.attention_logits(0, q)  # every token
    qc.check_status()
    kh = k.float().cpu().numpy()
    for h in range(2):
        want = ref_logits(q[0, h].float().cpu().numpy(), kh[h])
        assert np.array_equal(lg[0, h, :300].cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_softmax_worked_examples(qk):
    # test_attention.cpp:86-95
    assert qk.softmax_weights([0.0, 0.0]) == [0.5, 0.5]
    assert qk.softmax_weights([1000.0, 1000.0]) == [0.5, 0.5]
    w = qk.softmax_weights([0.0, math.log(3.0)])
    assert w[0] == pytest.approx(0.25, rel=1e-12) and w[1] == pytest.approx(0.75, rel=1e-12)
    with pytest.raises(ValueError):
        qk.softmax_weights([])


def test_softmax_extreme_logits_and_monotone(qk):
    # test_attention.cpp:97-120
    rng = np.random.default_rng(17)
    for _ in range(100):
        logits = (rng.random(1 + rng.integers(64)) * 2 - 1) * 1e4
        w = np.array(qk.softmax_weights(logits.tolist()))
        assert abs(w.sum() - 1.0) <= 1e-6
        w2 = np.array(qk.softmax_weights((logits + (rng.random() - 0.5) * 100).tolist()))
        assert np.max(np.abs(w2 - w)) <= 1e-6
        e = np.exp(logits - logits.max())
        np.testing.assert_allclose(w, e / e.sum(), rtol=1e-13, atol=1e-300)
    w = qk.softmax_weights([-1.0, 0.5, 0.4, 2.0])
    assert w[3] > w[1] > w[2] > w[0]


def test_device_softmax_rows(qk):
    qc = qk.QuestCache(64, 16, max_tokens=64)
    lg = torch.randn((3, 50), dtype=torch.float64, device="cuda") * 20
    cnt = torch.tensor([50, 7, 1], dtype=torch.int32, device="cuda")
    w = qc.softmax_weights(lg, cnt)
    qc.check_status()
    for r, n in enumerate([50, 7, 1]):
        x = lg[r, :n].cpu().numpy()
        e = np.exp(x - x.max())
        np.testing.assert_allclose(w[r, :n].cpu().numpy(), e / e.sum(), rtol=1e-13)
    qc.softmax_weights(lg, torch.tensor([50, 0, 1], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        qc.check_status()


@pytest.mark.parametrize("d,S,L", [(64, 16, 1000), (128, 16, 2500), (32, 4, 97)])
def test_attend_tokens_vs_oracle(qk, oracle_c, d, S, L):
    rng = np.random.default_rng(L)
    sd = 1 / np.sqrt(d)
    keys = half(rng.standard_normal((L, d)) * sd)
    vals = half(rng.standard_normal((L, d)) * sd)
    q = half(rng.standard_normal(d) * sd)
    c = cache_of(qk, d, S, keys, vals)
    for toks in (sorted(rng.choice(L, size=L // 3, replace=False).tolist()), [L - 1], [0, L - 1]):
        got = qk.attend_tokens(q, c, toks)
        want = oracle_c.naive_attention(q, keys, vals, np.array(toks, np.uint32))
        err = np.linalg.norm(np.array(got.output) - want) / np.linalg.norm(want)
        assert err <= 1e-5
        assert abs(got.weights_sum_check - 1.0) <= 1e-6
    # every token in order == full_attention, bitwise (same chunking as the pages)
    allt = qk.attend_tokens(q, c, list(range(L)))
    full = qk.full_attention(q, c)
    assert allt.output == full.output
    assert abs(full.weights_sum_check - 1.0) <= 1e-6


def test_attend_tokens_rejects_malformed_sets(qk):
    # test_attention.cpp:248-257
    rng = np.random.default_rng(777)
    c = cache_of(qk, 2, 2, half(rng.standard_normal((4, 2))), half(rng.standard_normal((4, 2))))
    q = half(rng.standard_normal(2))
    with pytest.raises(ValueError):
        qk.attend_tokens(q, c, [])
    with pytest.raises(ValueError):
        qk.attend_tokens(q, c, [3, 2])
    with pytest.raises(IndexError):
        qk.attend_tokens(q, c, [9])


def test_sparse_weights_sum_check(qk, oracle_c):
    rng = np.random.default_rng(3)
    d, S, L = 64, 16, 2000
    keys = half(rng.standard_normal((L, d)) / 8)
    vals = half(rng.standard_normal((L, d)) / 8)
    q = half(rng.standard_normal(d) / 8)
    c = cache_of(qk, d, S, keys, vals)
    out = qk.sparse_attention(q, c, [0, 5, 17, 124])
    assert abs(out.weights_sum_check - 1.0) <= 1e-6
    want = oracle_c.sparse_attention(q, keys, vals, S, [0, 5, 17, 124])
    assert np.linalg.norm(np.array(out.output) - want) / np.linalg.norm(want) <= 1e-5


def ref_select_pairs(pairs, P, S, budget, force, enabled):
    """criticality.cpp:36-81 literally (python sorted is stable; ties by page index)."""
    if not enabled:
        return list(range(P))
    k = budget // S
    if k >= len(pairs):
        return list(range(P))
    order = sorted(range(len(pairs)), key=lambda i: (-pairs[i][1], pairs[i][0]))
    sel = [pairs[i][0] for i in order[:k]]
    if force and (P - 1) not in sel:
        sel[-1] = P - 1
    return sorted(sel)


@pytest.mark.parametrize("seed", range(6))
def test_select_top_k_arbitrary_pagescore_vectors(qk, seed):
    rng = np.random.default_rng(seed)
    S, P = 4, 1 + int(rng.integers(1, 300))
    c = cache_of(qk, 2, S, half(rng.standard_normal((P * S - 1, 2))), half(rng.standard_normal((P * S - 1, 2))))
    n = int(rng.integers(1, 2 * P + 2))
    pages = rng.integers(0, P, size=n)
    vals = rng.choice(np.array([0.0, -0.0, 1.0, -2.5, 3.0]), size=n) if seed % 2 else rng.standard_normal(n)
    pairs = [(int(p), float(v)) for p, v in zip(pages, vals)]
    for budget in (S, 3 * S, 17 * S, 10_000):
        for force in (True, False):
            want = ref_select_pairs(pairs, P, S, budget, force, True)
            got = qk.select_top_k([qk.PageScore(p, v) for p, v in pairs], qk.SelectionConfig(budget, force), c)
            assert got == want, (budget, force)
    with pytest.raises(IndexError):
        qk.select_top_k([qk.PageScore(P, 1.0)], qk.SelectionConfig(S), c)


def test_select_top_k_zero_signs_tie(qk):
    """-0.0 and +0.0 are equal in the reference's comparator (ties to the lower page), in
    the page-ordered fast path as well."""
    c = cache_of(qk, 2, 1, [[0, 0]] * 6, [[0, 0]] * 6)
    scores = [qk.PageScore(i, v) for i, v in enumerate([0.0, -0.0, -0.0, 0.0, -1.0, -0.0])]
    assert qk.select_top_k(scores, qk.SelectionConfig(2, False), c) == [0, 1]
    assert qk.select_top_k(scores, qk.SelectionConfig(3, True), c) == [0, 1, 5]
