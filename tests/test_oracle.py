"""CPU tests: pin the C restatement (oracle/) before trusting it as the GPU checker.

1. The reference's own known-answer tests, restated (cited file:line in
   /root/reference/proj/tests/).
2. The golden vectors tests/golden/golden_v1.npz produced by the real reference.
3. Randomised agreement with the real reference library (oracle/_ref) when it is built.
"""

import numpy as np
import pytest

from conftest import half


# ---- 1. reference known-answer tests ---------------------------------------------------

def test_config_validation(oracle_c):
    # test_kv_store.cpp:22-28
    with pytest.raises(ValueError):
        oracle_c.validate_config(0, 16)
    with pytest.raises(ValueError):
        oracle_c.validate_config(4, 0)
    with pytest.raises(ValueError):
        oracle_c.validate_config(4, 4, 0)
    oracle_c.validate_config(128, 16)


def test_metadata_worked_example(oracle_c):
    # test_kv_store.cpp:39-51: keys [1,5],[3,2] -> min [1,2], max [3,5]
    mn, mx = oracle_c.metadata([[1, 5], [3, 2]], 4)
    assert mn.tolist() == [[1, 2]] and mx.tolist() == [[3, 5]]


def test_first_key_seeds_metadata(oracle_c):
    # test_kv_store.cpp:53-59
    mn, mx = oracle_c.metadata([[-2.5, 0.0, 7.25]], 8)
    assert mn.tolist() == [[-2.5, 0.0, 7.25]] and mx.tolist() == [[-2.5, 0.0, 7.25]]


def test_paging_arithmetic(oracle_c):
    # test_kv_store.cpp:30-37,61-73: page size 1 and 2
    mn, _ = oracle_c.metadata([[1, 2], [3, 4]], 1)
    assert mn.shape == (2, 2)
    mn, _ = oracle_c.metadata([[0, 0], [1, 0], [2, 0]], 2)
    assert mn.shape == (2, 2) and mn[1, 0] == 2.0


def test_metadata_equals_rescan_property(oracle_c):
    # test_kv_store.cpp:89-113 (1000 sequences instead of 10^4)
    rng = np.random.default_rng(20240811)
    for _ in range(1000):
        d, S, L = rng.integers(1, 9), rng.integers(1, 9), rng.integers(1, 33)
        k = rng.standard_normal((L, d)).astype(np.float32)
        mn, mx = oracle_c.metadata(k, S)
        P = (L + S - 1) // S
        assert mn.shape == (P, d)
        for p in range(P):
            rows = k[p * S:(p + 1) * S]
            assert np.array_equal(mn[p], rows.min(axis=0))
            assert np.array_equal(mx[p], rows.max(axis=0))


def test_signed_zero_first_seen(oracle_c):
    # kv_store.cpp:40-43 strict compares: +0 then -0 keeps +0; -0 then +0 keeps -0
    mn, mx = oracle_c.metadata([[0.0], [-0.0]], 4)
    assert not np.signbit(mn[0, 0]) and not np.signbit(mx[0, 0])
    mn, mx = oracle_c.metadata([[-0.0], [0.0]], 4)
    assert np.signbit(mn[0, 0]) and np.signbit(mx[0, 0])


def test_score_worked_examples(oracle_c):
    # test_criticality.cpp:60-64 and :66-69
    assert oracle_c.estimate_page_score([1, -2], [0, -1], [3, 2]) == 5.0
    assert oracle_c.estimate_page_score([0, 0, 0], [-4, 1, 0], [2, 5, 9]) == 0.0


def test_singleton_page_is_exact_dot(oracle_c):
    # test_criticality.cpp:71-79
    rng = np.random.default_rng(11)
    for _ in range(200):
        k = rng.standard_normal((1, 16)).astype(np.float32)
        q = rng.standard_normal(16).astype(np.float32)
        mn, mx = oracle_c.metadata(k, 8)
        dot = 0.0
        for a, b in zip(q.astype(np.float64), k[0].astype(np.float64)):
            dot += a * b
        assert oracle_c.estimate_all(q, mn, mx)[0] == dot


def test_estimate_all_empty_throws(oracle_c):
    # test_criticality.cpp:87-101
    with pytest.raises(ValueError):
        oracle_c.estimate_all(np.zeros(4, np.float32), np.zeros((0, 4)), np.zeros((0, 4)))


def test_upper_bound_property(oracle_c):
    # test_criticality.cpp:104-119 (2000 trials)
    rng = np.random.default_rng(31337)
    for trial in range(2000):
        d = 16 if trial % 2 == 0 else 64
        S = 1 + trial % 16
        k = rng.standard_normal((S, d)).astype(np.float32)
        q = rng.standard_normal(d).astype(np.float32)
        mn, mx = oracle_c.metadata(k, S)
        score = oracle_c.estimate_all(q, mn, mx)[0]
        exact = k.astype(np.float64) @ q.astype(np.float64)
        assert (exact <= score + 1e-6 * (1 + abs(score))).all()


@pytest.mark.parametrize("scores,budget,force,enabled,want", [
    ([5, 9, 9, 1], 8, False, True, [1, 2]),       # test_criticality.cpp:122-129
    ([3, 3, 3], 4, False, True, [0]),             # :130-136 three-way tie -> oldest
    ([1, 2, 3], 1000, True, True, [0, 1, 2]),     # :137-142 budget covers cache
    ([9, 8, 1], 8, True, True, [0, 2]),           # :143-150 forced recent
    ([9, 8, 1], 8, False, True, [0, 1]),          # :151-153
    ([5, 9, 9, 1], 4, True, False, [0, 1, 2, 3]),  # :154-160 selection disabled
])
def test_select_top_k_worked_examples(oracle_c, scores, budget, force, enabled, want):
    assert oracle_c.select_top_k(scores, 4, budget, force, enabled).tolist() == want


def test_select_top_k_budget_below_page_size(oracle_c):
    # test_criticality.cpp:161-165
    with pytest.raises(ValueError):
        oracle_c.select_top_k([1, 2], 8, 4)


def sorted_top_k_pages(values, k, force_last):
    """tests/oracles.hpp:52-72, restated."""
    P = len(values)
    order = sorted(range(P), key=lambda i: (-values[i], i))
    if k >= P:
        return list(range(P))
    picked = order[:k]
    if force_last and (P - 1) not in picked:
        picked[-1] = P - 1
    return sorted(picked)


def test_selection_matches_sort_oracle(oracle_c):
    # test_criticality.cpp:169-199 (exhaustive small + random with integer ties)
    rng = np.random.default_rng(555)
    for pages in range(1, 9):
        for _ in range(50):
            vals = rng.integers(0, 4, size=pages).astype(np.float64)
            for k in range(1, pages + 1):
                for force in (False, True):
                    got = oracle_c.select_top_k(vals, 4, k * 4, force).tolist()
                    assert got == sorted_top_k_pages(list(vals), k, force)
    for _ in range(300):
        pages = int(rng.integers(9, 65))
        vals = rng.integers(0, 7, size=pages).astype(np.float64)
        k = int(rng.integers(1, pages + 1))
        for force in (False, True):
            got = oracle_c.select_top_k(vals, 2, k * 2, force).tolist()
            assert got == sorted_top_k_pages(list(vals), k, force)


def test_attention_worked_examples(oracle_c):
    # test_attention.cpp:125-146
    out = oracle_c.full_attention([1, 0], [[1, 2]], [[5.5, -3.25]])
    assert out.tolist() == [5.5, -3.25]
    out = oracle_c.full_attention([3, -1], [[1, 1], [1, 1]], [[2, 0], [4, 6]])
    assert out == pytest.approx([3.0, 3.0], rel=1e-12)
    with pytest.raises(ValueError):
        oracle_c.full_attention([1, 0], np.zeros((0, 2)), np.zeros((0, 2)))


def test_sparse_attention_worked_examples(oracle_c):
    # test_attention.cpp:148-192
    rng = np.random.default_rng(8)
    k = rng.standard_normal((37, 8)).astype(np.float32) * 0.5
    v = rng.standard_normal((37, 8)).astype(np.float32) * 0.5
    q = rng.standard_normal(8).astype(np.float32) * 0.5
    dense = oracle_c.full_attention(q, k, v)
    sparse = oracle_c.sparse_attention(q, k, v, 4, list(range(10)))
    assert np.array_equal(dense, sparse)  # bit for bit
    out = oracle_c.sparse_attention([1, 1], [[1, 0], [0, 1]], [[9, 9], [-1.5, 4]], 1, [1])
    assert out.tolist() == [-1.5, 4.0]
    with pytest.raises(ValueError):
        oracle_c.sparse_attention(q, k, v, 4, [])
    with pytest.raises(ValueError):
        oracle_c.sparse_attention(q, k, v, 4, [0, 0])
    with pytest.raises(IndexError):
        oracle_c.sparse_attention(q, k, v, 4, [10])


def test_naive_oracle_agreement(oracle_c):
    # test_attention.cpp:227-246 (1e-5 relative L2)
    rng = np.random.default_rng(666)
    for _ in range(100):
        d = int(rng.integers(1, 65))
        L = int(rng.integers(1, 513))
        sd = 1.0 / np.sqrt(d)
        k = (rng.standard_normal((L, d)) * sd).astype(np.float32)
        v = (rng.standard_normal((L, d)) * sd).astype(np.float32)
        q = (rng.standard_normal(d) * sd).astype(np.float32)
        got = oracle_c.full_attention(q, k, v)
        want = oracle_c.naive_attention(q, k, v, np.arange(L))
        assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want) + 1e-12


def test_traffic_model(oracle_c):
    # test_metrics.cpp:175-185, acceptance_main.cpp:176-195: 0.125 exactly
    assert oracle_c.traffic_fraction(16, 65536, 4096) == 0.125
    # acceptance_main.cpp:366-385 accounting: L=32K, B=2048, S=16, d=16 -> 262,144 B
    assert oracle_c.quest_step_bytes(16, 2, 2048, 2048) == 262144
    assert oracle_c.quest_step_bytes(16, 2, 0, 32768) == 2097152


# ---- 2. golden vectors from the real reference -------------------------------------------

def test_golden_vectors(oracle_c, golden):
    assert len(golden.names) >= 10
    for name in golden.names:
        g = golden.case(name)
        S = g["S"]
        mn, mx = oracle_c.metadata(g["k"], S)
        assert np.array_equal(mn.view(np.uint32), g["meta_min"].view(np.uint32)), name
        assert np.array_equal(mx.view(np.uint32), g["meta_max"].view(np.uint32)), name
        scores = oracle_c.estimate_all(g["q"], mn, mx)
        assert np.array_equal(scores.view(np.uint64), g["scores"].view(np.uint64)), name
        assert np.array_equal(oracle_c.full_attention(g["q"], g["k"], g["v"]), g["full"]), name
        for row, (budget, force, enabled, status) in enumerate(g["sel_cfg"]):
            if status:
                with pytest.raises(ValueError):
                    oracle_c.select_top_k(scores, S, int(budget), bool(force), bool(enabled))
                continue
            pages = oracle_c.select_top_k(scores, S, int(budget), bool(force), bool(enabled))
            want = g["sel_pages"][row]
            assert pages.tolist() == want[want >= 0].tolist(), (name, row)
            out = oracle_c.sparse_attention(g["q"], g["k"], g["v"], S, pages)
            assert np.array_equal(out, g["sel_out"][row]), (name, row)


# ---- 3. randomised agreement with the real reference -------------------------------------

def test_oracle_matches_reference_random(oracle_c, reference):
    rng = np.random.default_rng(7)
    for trial in range(40):
        d = int(rng.choice([2, 16, 64, 128]))
        S = int(rng.choice([1, 4, 16]))
        L = int(rng.integers(1, 600))
        sd = 1.0 if trial % 2 else 1 / np.sqrt(d)
        k, v = half(rng.standard_normal((L, d)) * sd), half(rng.standard_normal((L, d)) * sd)
        q = half(rng.standard_normal(d) * sd)
        budget = int(rng.integers(S, 8 * S + 1))
        force = bool(trial % 3)
        s_ref, p_ref, o_ref = reference.quest_step(q, k, v, S, budget, force)
        s_or, p_or, o_or = oracle_c.quest_step(q, k, v, S, budget, force)
        assert np.array_equal(s_ref.view(np.uint64), s_or.view(np.uint64))
        assert p_ref.tolist() == p_or.tolist()
        assert np.array_equal(o_ref, o_or)


def test_group_quest_step_composes_the_reference(oracle_c, reference):
    """The checker of the GQA group-shared variant (Oracle.group_quest_step) equals the same
    composition of the unmodified reference's functions: per-head estimate_all, the group
    score (max / fp64 sum in head order), one select_top_k, each head's sparse_attention."""
    rng = np.random.default_rng(17)
    for trial in range(12):
        d, S, G = int(rng.choice([16, 64, 128])), int(rng.choice([4, 16])), int(rng.choice([2, 4, 8]))
        L = int(rng.integers(S, 500))
        sd = 1 / np.sqrt(d)
        k, v = half(rng.standard_normal((L, d)) * sd), half(rng.standard_normal((L, d)) * sd)
        qs = half(rng.standard_normal((G, d)) * sd)
        budget = int(rng.integers(S, 8 * S + 1))
        reduce = "max" if trial % 2 else "sum"
        force = bool(trial % 3)
        group, pages, outs = oracle_c.group_quest_step(qs, k, v, S, budget, reduce, force)
        per_head = [reference.estimate_all(q, k, S) for q in qs]
        want = per_head[0].copy()
        for s_ in per_head[1:]:
            want = np.maximum(want, s_) if reduce == "max" else want + s_
        assert np.array_equal(group.view(np.uint64), want.view(np.uint64)), trial
        ref_pages = reference.select_top_k(want, S, budget, force)
        assert pages.tolist() == ref_pages.tolist(), trial
        for g in range(G):
            ref_out, _ = reference.sparse_attention(qs[g], k, v, S, ref_pages)
            assert np.array_equal(outs[g], ref_out), (trial, g)
