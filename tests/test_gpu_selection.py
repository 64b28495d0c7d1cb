"""GPU parity: criticality estimate (K2, bitwise fp64) and top-K selection (K3, exact pages).

Restates /root/reference/proj/tests/test_criticality.cpp against the CUDA path and adds the
GPU fixtures of SURVEY.md section 8(c): tie stress, signed zeros, partial last page,
K = 1 / P-1 / >= P, force on/off, selection disabled, budget < S."""

import numpy as np
import pytest
import torch

from conftest import half
from test_oracle import sorted_top_k_pages

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qk():
    from paper_2406_10774_b200 import questkv

    return questkv


def geometry_cache(qk, pages, page_size):
    """test_criticality.cpp geometry_cache: only the page count matters."""
    c = qk.KvCache(qk.CacheConfig(head_dim=1, page_size=page_size), capacity=pages * page_size)
    c.extend(np.zeros((pages * page_size, 1)), np.zeros((pages * page_size, 1)))
    return c


def as_scores(qk, values):
    return [qk.PageScore(i, float(v)) for i, v in enumerate(values)]


def test_worked_score_example(qk):
    # test_criticality.cpp:60-64
    assert qk.estimate_page_score([1, -2], qk.PageMetadata([0, -1], [3, 2])) == 5.0


def test_zero_query_scores_zero(qk):
    # test_criticality.cpp:66-69
    assert qk.estimate_page_score([0, 0, 0], qk.PageMetadata([-4, 1, 0], [2, 5, 9])) == 0.0


def test_singleton_page_collapses_to_exact_dot(qk):
    # test_criticality.cpp:71-79 (+ estimate_all shape :87-101)
    rng = np.random.default_rng(11)
    for _ in range(20):
        keys = half(rng.standard_normal((3, 16)))
        q = half(rng.standard_normal(16))
        c = qk.KvCache(qk.CacheConfig(head_dim=16, page_size=1))
        c.extend(keys, np.zeros_like(keys))
        scores = qk.estimate_all(q, c)
        assert [s.page_index for s in scores] == [0, 1, 2]
        for p in range(3):
            dot = 0.0
            for a, b in zip(q.astype(np.float64), keys[p].astype(np.float64)):
                dot += a * b
            assert scores[p].score == dot


def test_estimate_all_errors(qk):
    c = qk.KvCache(qk.CacheConfig(head_dim=4, page_size=1))
    with pytest.raises(ValueError):
        qk.estimate_all([1, 2, 3, 4], c)
    c.append([1, 2, 3, 4], [0, 0, 0, 0])
    with pytest.raises(ValueError):
        qk.estimate_all([1, 2, 3], c)


def test_golden_vectors_through_gpu(qk, golden):
    """Metadata, scores and pages bitwise equal to the real reference's (golden_v1.npz);
    outputs within the fp32-accumulate tolerance."""
    for name in golden.names:
        g = golden.case(name)
        S, d = g["S"], g["k"].shape[1]
        c = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=g["k"].shape[0])
        c.extend(g["k"], g["v"])
        mn, mx = c.quest_cache.read_metadata(0, 0, 0)
        assert np.array_equal(mn.astype(np.float32).view(np.uint32), g["meta_min"].view(np.uint32)), name
        assert np.array_equal(mx.astype(np.float32).view(np.uint32), g["meta_max"].view(np.uint32)), name
        scores = qk.estimate_all(g["q"], c)
        got = np.array([s.score for s in scores])
        assert np.array_equal(got.view(np.uint64), g["scores"].view(np.uint64)), name
        full = np.array(qk.full_attention(g["q"], c).output)
        assert np.linalg.norm(full - g["full"]) <= 1e-5 * np.linalg.norm(g["full"]) + 1e-7, name
        for row, (budget, force, enabled, status) in enumerate(g["sel_cfg"]):
            cfg = qk.SelectionConfig(int(budget), bool(force), bool(enabled))
            if status:
                with pytest.raises(ValueError):
                    qk.select_top_k(scores, cfg, c)
                continue
            pages = qk.select_top_k(scores, cfg, c)
            want = g["sel_pages"][row]
            assert pages == want[want >= 0].tolist(), (name, row)
            out = np.array(qk.sparse_attention(g["q"], c, pages).output)
            ref = g["sel_out"][row]
            assert np.linalg.norm(out - ref) <= 1e-5 * np.linalg.norm(ref) + 1e-7, (name, row)


@pytest.mark.parametrize("values,budget,force,enabled,want", [
    ([5, 9, 9, 1], 8, False, True, [1, 2]),
    ([3, 3, 3], 4, False, True, [0]),
    ([1, 2, 3], 1000, True, True, [0, 1, 2]),
    ([9, 8, 1], 8, True, True, [0, 2]),
    ([9, 8, 1], 8, False, True, [0, 1]),
    ([5, 9, 9, 1], 4, True, False, [0, 1, 2, 3]),
])
def test_select_top_k_worked_examples(qk, values, budget, force, enabled, want):
    # test_criticality.cpp:121-160
    c = geometry_cache(qk, len(values), 4)
    cfg = qk.SelectionConfig(budget, force, enabled)
    assert qk.select_top_k(as_scores(qk, values), cfg, c) == want


def test_budget_below_page_size_rejected(qk):
    # test_criticality.cpp:161-165
    c = geometry_cache(qk, 2, 8)
    with pytest.raises(ValueError):
        qk.select_top_k(as_scores(qk, [1, 2]), qk.SelectionConfig(4), c)


def test_selection_matches_sort_oracle_exhaustive(qk):
    # test_criticality.cpp:169-186: pages 1..8, integer scores force ties
    rng = np.random.default_rng(555)
    caches = {p: geometry_cache(qk, p, 4) for p in range(1, 9)}
    for pages in range(1, 9):
        for _ in range(8):
            vals = rng.integers(0, 4, size=pages).astype(np.float64)
            for k in range(1, pages + 1):
                for force in (False, True):
                    got = qk.select_top_k(as_scores(qk, vals), qk.SelectionConfig(k * 4, force),
                                          caches[pages])
                    assert got == sorted_top_k_pages(list(vals), k, force)


def test_batched_selection_random_ties_large(qk, oracle_c):
    """Many (sequence, head) rows at once, up to 8192 pages, integer and float scores,
    force on/off, every K regime -- against the oracle's std::sort-equivalent selection."""
    rng = np.random.default_rng(99)
    S = 16
    for P, H in ((1, 4), (2, 4), (37, 8), (512, 8), (2048, 4), (8192, 2)):
        qc = qk.QuestCache(1, S, num_q_heads=H, max_tokens=P * S)
        z = torch.zeros((H, P * S, 1), dtype=torch.float16, device="cuda")
        qc.prefill(0, 0, z, z)
        for kind in ("int", "float", "const"):
            if kind == "int":
                vals = rng.integers(0, 9, size=(H, P)).astype(np.float64)
            elif kind == "float":
                vals = rng.standard_normal((H, P))
            else:
                vals = np.full((H, P), 0.25)
            scores = torch.from_numpy(vals).cuda().view(1, H, P)
            for K in sorted({1, 2, max(1, P // 16), max(1, P - 1), P, P + 3}):
                for force in (False, True):
                    pages, counts = qc.select_topk(0, scores, K * S, force)
                    pages, counts = pages.cpu().numpy(), counts.cpu().numpy()
                    for h in range(H):
                        want = oracle_c.select_top_k(vals[h], S, K * S, force)
                        got = pages[0, h, : counts[0, h]]
                        assert got.tolist() == want.tolist(), (P, kind, K, force, h)


def test_partial_last_page_lengths(qk, oracle_c):
    """L = 32767 / 32768 / 32769 around a page boundary: metadata of the partial last page
    and the selection (force keeps the partial page) are exact."""
    rng = np.random.default_rng(5)
    for L in (32767, 32768, 32769):
        d, S = 128, 16
        keys = half(rng.standard_normal((L, d)) / np.sqrt(d))
        vals = half(rng.standard_normal((L, d)) / np.sqrt(d))
        q = half(rng.standard_normal(d) / np.sqrt(d))
        c = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=L)
        c.extend(keys, vals)
        scores = qk.estimate_all(q, c)
        mn, mx = oracle_c.metadata(keys, S)
        want_scores = oracle_c.estimate_all(q, mn, mx)
        got = np.array([s.score for s in scores])
        assert np.array_equal(got.view(np.uint64), want_scores.view(np.uint64))
        for force in (True, False):
            pages = qk.select_top_k(scores, qk.SelectionConfig(2048, force), c)
            assert pages == oracle_c.select_top_k(want_scores, S, 2048, force).tolist()


def test_scale_covariance(qk):
    # test_criticality.cpp:201-230: power-of-two query scales scale scores exactly
    rng = np.random.default_rng(99)
    keys = half(rng.standard_normal((64, 8)))
    q = half(rng.standard_normal(8))
    c = qk.KvCache(qk.CacheConfig(head_dim=8, page_size=4))
    c.extend(keys, np.zeros_like(keys))
    base = qk.estimate_all(q, c)
    cfg = qk.SelectionConfig(16)
    base_pick = qk.select_top_k(base, cfg, c)
    for s in (0.25, 2.0, 64.0):
        scaled = qk.estimate_all(q * s, c)
        assert [x.score for x in scaled] == [s * x.score for x in base]
        assert qk.select_top_k(scaled, cfg, c) == base_pick


def test_determinism(qk):
    # test_criticality.cpp:232-245
    rng = np.random.default_rng(7)
    keys = half(rng.standard_normal((128, 16)))
    q = half(rng.standard_normal(16))
    c = qk.KvCache(qk.CacheConfig(head_dim=16, page_size=8))
    c.extend(keys, np.zeros_like(keys))
    a, b = qk.estimate_all(q, c), qk.estimate_all(q, c)
    assert [x.score for x in a] == [x.score for x in b]
    cfg = qk.SelectionConfig(32)
    assert qk.select_top_k(a, cfg, c) == qk.select_top_k(b, cfg, c)


def test_gqa_estimate_reads_shared_metadata(qk, oracle_c):
    """GQA: every query head of a group is scored on its KV head's metadata, bitwise."""
    rng = np.random.default_rng(17)
    for G in (2, 4, 8):
        Hkv, d, S, L = 2, 128, 16, 1500
        qc = qk.QuestCache(d, S, num_q_heads=Hkv * G, num_kv_heads=Hkv, max_tokens=L)
        keys = half(rng.standard_normal((Hkv, L, d)) / np.sqrt(d))
        kt = torch.from_numpy(keys).half().cuda()
        qc.prefill(0, 0, kt, kt)
        q = half(rng.standard_normal((1, Hkv * G, d)) / np.sqrt(d))
        scores = qc.estimate(0, torch.from_numpy(q).half().cuda()).cpu().numpy()
        P = (L + S - 1) // S
        for h in range(Hkv * G):
            mn, mx = oracle_c.metadata(keys[h // G], S)
            want = oracle_c.estimate_all(q[0, h], mn, mx)
            assert np.array_equal(scores[0, h, :P].view(np.uint64), want.view(np.uint64)), (G, h)


@pytest.mark.parametrize("Hq,Hkv,B", [(32, 8, 19), (16, 8, 20), (16, 2, 75)])
def test_wide_gqa_estimate_bitwise(qk, Hq, Hkv, B):
    """Wide GQA launches (more (sequence, KV head) units than SMs, the shape the decode step
    sends to the separate kernels): scores of sampled (sequence, query head) rows bitwise equal
    to the oracle, across ragged lengths (partial page blocks, partial pages) and special
    values (subnormals, signed zeros, +-65504)."""
    import torch
    from oracle import Oracle

    rng = np.random.default_rng(Hq * 100 + B)
    d, S = 128, 16
    lens = [int(x) for x in rng.integers(300, 9000, size=B)]
    qc = qk.QuestCache(d, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv, max_tokens=max(lens))
    keys = []
    specials = np.array([0.0, -0.0, 6e-8, -6e-8, 65504.0, -65504.0, 1e-5], np.float32)
    for b, L in enumerate(lens):
        k = (rng.standard_normal((Hkv, L, d)) / np.sqrt(d)).astype(np.float32)
        mask = rng.random(k.shape) < 0.002
        k[mask] = rng.choice(specials, size=int(mask.sum()))
        k16 = k.astype(np.float16)
        qc.prefill(0, b, torch.from_numpy(k16).cuda(), torch.from_numpy(k16).cuda())
        keys.append(k16.astype(np.float32))
    q = (rng.standard_normal((B, Hq, d)) / np.sqrt(d)).astype(np.float16)
    q[0, 0, :4] = np.array([0.0, -0.0, 6e-8, -65504.0], np.float16)
    scores = qc.estimate(0, torch.from_numpy(q).cuda()).cpu().numpy()
    orc = Oracle()
    G = Hq // Hkv
    for b in list(range(0, B, max(1, B // 6))) + [B - 1]:
        for h in (0, Hq - 1, int(rng.integers(0, Hq))):
            mn, mx = orc.metadata(keys[b][h // G], S)
            want = orc.estimate_all(q[b, h].astype(np.float32), mn, mx)
            got = scores[b, h, : len(want)]
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (b, h)
