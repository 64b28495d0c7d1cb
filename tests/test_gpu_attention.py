"""GPU parity: split-KV sparse/dense paged attention (K4-K6) and the decode step.

Restates /root/reference/proj/tests/test_attention.cpp against the CUDA path.  The
reference accumulates in fp64; the kernels accumulate in fp32, so outputs are compared
with the reference's own oracle bar: relative L2 <= 1e-5 (acceptance_main.cpp:165) for
fp32 outputs and 1e-3 for fp16 outputs.  Full-budget degeneracy is bitwise on the GPU."""

import numpy as np
import pytest
import torch

from conftest import half

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
TOL_F16 = 1e-3


@pytest.fixture(scope="module")
def qk():
    from paper_2406_10774_b200 import questkv

    return questkv


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.linalg.norm(got - want) / (np.linalg.norm(want) + 1e-30)


def random_cache(qk, rng, d, S, L, sd):
    keys = half(rng.standard_normal((L, d)) * sd)
    vals = half(rng.standard_normal((L, d)) * sd)
    c = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=max(L, 1))
    c.extend(keys, vals)
    return c, keys, vals


def test_single_token_returns_its_value(qk):
    # test_attention.cpp:126-132
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2))
    c.append([1, 2], [5.5, -3.25])
    assert qk.full_attention([1, 0], c).output == [5.5, -3.25]


def test_equal_keys_average_the_values(qk):
    # test_attention.cpp:133-140
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2))
    c.append([1, 1], [2, 0])
    c.append([1, 1], [4, 6])
    assert qk.full_attention([3, -1], c).output == pytest.approx([3.0, 3.0], rel=1e-6)


def test_empty_cache_rejected(qk):
    # test_attention.cpp:141-145
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2))
    with pytest.raises(ValueError):
        qk.full_attention([1, 0], c)


def test_all_pages_reproduce_full_attention_bitwise(qk):
    # test_attention.cpp:151-158 and :194-207 (degeneracy across geometries), on the GPU
    rng = np.random.default_rng(444)
    for _ in range(30):
        d = int(rng.integers(1, 257))
        S = int(rng.integers(1, 65))
        L = int(rng.integers(1, 3000))
        c, _, _ = random_cache(qk, rng, d, S, L, 0.5)
        q = half(rng.standard_normal(d) * 0.5)
        dense = qk.full_attention(q, c).output
        sparse = qk.sparse_attention(q, c, list(range(c.page_count()))).output
        assert np.array_equal(np.array(dense), np.array(sparse)), (d, S, L)


def test_singleton_page_returns_that_tokens_value(qk):
    # test_attention.cpp:159-166
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=1))
    c.append([1, 0], [9, 9])
    c.append([0, 1], [-1.5, 4])
    assert qk.sparse_attention([1, 1], c, [1]).output == [-1.5, 4.0]


def test_page_set_validation(qk):
    # test_attention.cpp:167-176
    rng = np.random.default_rng(6)
    c, _, _ = random_cache(qk, rng, 2, 2, 6, 1.0)
    q = half(rng.standard_normal(2))
    with pytest.raises(ValueError):
        qk.sparse_attention(q, c, [])
    with pytest.raises(ValueError):
        qk.sparse_attention(q, c, [0, 0])
    with pytest.raises(IndexError):
        qk.sparse_attention(q, c, [3])
    # any order is accepted (attention.hpp:37)
    assert qk.sparse_attention(q, c, [2, 0]).output == qk.sparse_attention(q, c, [0, 2]).output


def test_device_page_list_validation(qk):
    """Device-side checks of qk_sparse_attend page lists surface as the reference's
    exception types through qk_check_status."""
    rng = np.random.default_rng(1)
    c, _, _ = random_cache(qk, rng, 64, 16, 100, 1.0)
    qc = c.quest_cache
    q = torch.from_numpy(half(rng.standard_normal((1, 1, 64)))).half().cuda()
    for bad, exc in (([0, 9], IndexError), ([3, 1], ValueError), ([2, 2], ValueError)):
        pl = torch.tensor([[bad]], dtype=torch.int32, device="cuda")
        cnt = torch.tensor([[2]], dtype=torch.int32, device="cuda")
        qc.sparse_attend(0, q, pl, cnt)
        with pytest.raises(exc):
            qc.check_status()
    qc.check_status()  # cleared


def test_subset_matches_reference_oracles(qk, oracle_c):
    # test_attention.cpp:177-191: pages {1,5,15} of 64 tokens, page size 4
    rng = np.random.default_rng(8)
    for _ in range(20):
        c, keys, vals = random_cache(qk, rng, 16, 4, 64, 0.25)
        q = half(rng.standard_normal(16) * 0.25)
        got = qk.sparse_attention(q, c, [1, 5, 15]).output
        tokens = [p * 4 + r for p in (1, 5, 15) for r in range(4)]
        naive = oracle_c.naive_attention(q, keys, vals, tokens)
        assert rel_l2(got, naive) <= TOL_F32
        assert rel_l2(got, oracle_c.sparse_attention(q, keys, vals, 4, [1, 5, 15])) <= TOL_F32


def test_output_is_convex_combination(qk):
    # test_attention.cpp:209-225
    rng = np.random.default_rng(555)
    for _ in range(20):
        c, _, vals = random_cache(qk, rng, 8, 4, 50, 1.0)
        q = half(rng.standard_normal(8))
        out = np.array(qk.full_attention(q, c).output)
        assert (out >= vals.min(axis=0) - 1e-6).all() and (out <= vals.max(axis=0) + 1e-6).all()


def test_agreement_with_naive_oracle(qk, oracle_c):
    # test_attention.cpp:227-246 (1e-5 relative L2)
    rng = np.random.default_rng(666)
    for _ in range(40):
        d = int(rng.integers(1, 129))
        L = int(rng.integers(1, 1025))
        sd = 1.0 / np.sqrt(d)
        c, keys, vals = random_cache(qk, rng, d, 16, L, sd)
        q = half(rng.standard_normal(d) * sd)
        got = qk.full_attention(q, c).output
        want = oracle_c.naive_attention(q, keys, vals, np.arange(L))
        assert rel_l2(got, want) <= TOL_F32


def test_fp16_output_and_lse(qk, oracle_c):
    rng = np.random.default_rng(12)
    d, S, L, H = 128, 16, 5000, 4
    qc = qk.QuestCache(d, S, num_q_heads=H, max_tokens=L)
    keys = half(rng.standard_normal((H, L, d)) / np.sqrt(d))
    vals = half(rng.standard_normal((H, L, d)) / np.sqrt(d))
    qc.prefill(0, 0, torch.from_numpy(keys).half().cuda(), torch.from_numpy(vals).half().cuda())
    q = half(rng.standard_normal((1, H, d)) / np.sqrt(d))
    qt = torch.from_numpy(q).half().cuda()
    o32, lse = qc.dense_attend(0, qt, want_lse=True)
    o16 = qc.dense_attend(0, qt, out_dtype=torch.float16)
    for h in range(H):
        want = oracle_c.full_attention(q[0, h], keys[h], vals[h])
        assert rel_l2(o32[0, h].cpu().numpy(), want) <= TOL_F32
        assert rel_l2(o16[0, h].float().cpu().numpy(), want) <= TOL_F16
        logits = keys[h].astype(np.float64) @ q[0, h].astype(np.float64) / np.sqrt(d)
        m = logits.max()
        assert abs(lse[0, h].item() - (m + np.log(np.exp(logits - m).sum()))) <= 1e-4


def _layer(qk, rng, B, Hq, Hkv, d, S, lens, max_tokens=None):
    qc = qk.QuestCache(d, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                       max_tokens=max_tokens or max(lens) + 8)
    keys, vals = [], []
    for b, L in enumerate(lens):
        k = half(rng.standard_normal((Hkv, L, d)) / np.sqrt(d))
        v = half(rng.standard_normal((Hkv, L, d)) / np.sqrt(d))
        qc.prefill(0, b, torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda())
        keys.append(k)
        vals.append(v)
    return qc, keys, vals


@pytest.mark.parametrize("Hq,Hkv,lens,budget", [
    (32, 32, [8192], 1024),          # BASELINE configs[0]: Llama-2-7B shape, 8K, budget 1024
    (8, 2, [3000, 17, 6001], 512),    # GQA, ragged batch, a 2-page sequence
    (4, 4, [16, 33], 16),             # K = 1 with force: only the newest page
])
def test_batched_quest_step_vs_oracle(qk, oracle_c, Hq, Hkv, lens, budget):
    """estimate -> select -> sparse attend for every (sequence, query head): scores and
    pages bitwise, outputs within 1e-5, against the oracle per query head on its KV
    head's cache (the reference's single-head semantics, GQA per query head)."""
    rng = np.random.default_rng(sum(lens) + Hq)
    d, S = 128, 16
    B = len(lens)
    qc, keys, vals = _layer(qk, rng, B, Hq, Hkv, d, S, lens)
    q = half(rng.standard_normal((B, Hq, d)) / np.sqrt(d))
    qt = torch.from_numpy(q).half().cuda()
    scores = qc.estimate(0, qt)
    pages, counts = qc.select_topk(0, scores, budget)
    out = qc.sparse_attend(0, qt, pages, counts)
    qc.check_status()
    scores, pages, counts, out = (x.cpu().numpy() for x in (scores, pages, counts, out))
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            k, v = keys[b][h // G], vals[b][h // G]
            s_want, p_want, o_want = oracle_c.quest_step(q[b, h], k, v, S, budget)
            P = len(s_want)
            assert np.array_equal(scores[b, h, :P].view(np.uint64), s_want.view(np.uint64))
            assert pages[b, h, : counts[b, h]].tolist() == p_want.tolist(), (b, h)
            assert rel_l2(out[b, h], o_want) <= TOL_F32, (b, h)


def test_decode_step_equals_separate_ops(qk):
    """qk_decode_step (the fused kernel: append + estimate + select + attend) == the four
    separate calls: same pages and counts bitwise, outputs equal up to fp32 reassociation
    of the split-KV merge (the two paths partition the pages differently)."""
    rng = np.random.default_rng(21)
    B, Hq, Hkv, d, S = 2, 8, 4, 128, 16
    lens = [2000, 777]
    a, keys, vals = _layer(qk, rng, B, Hq, Hkv, d, S, lens)
    b_, _, _ = _layer(qk, np.random.default_rng(21), B, Hq, Hkv, d, S, lens)
    for step in range(3):
        q = torch.from_numpy(half(rng.standard_normal((B, Hq, d)) / np.sqrt(d))).half().cuda()
        kn = torch.from_numpy(half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d))).half().cuda()
        vn = torch.from_numpy(half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d))).half().cuda()
        pages = torch.full((B, Hq, 64), -1, dtype=torch.int32, device="cuda")
        counts = torch.zeros((B, Hq), dtype=torch.int32, device="cuda")
        out_a = a.decode_step(0, q, kn, vn, 1024, pages=pages, counts=counts)
        b_.append(0, kn, vn)
        sc = b_.estimate(0, q)
        pb, cb = b_.select_topk(0, sc, 1024)
        out_b = b_.sparse_attend(0, q, pb, cb)
        assert torch.equal(counts, cb)
        for bb in range(B):
            for h in range(Hq):
                n = int(cb[bb, h])
                assert torch.equal(pages[bb, h, :n], pb[bb, h, :n])
        for bb in range(B):
            for h in range(Hq):
                assert rel_l2(out_a[bb, h].cpu().numpy(), out_b[bb, h].cpu().numpy()) <= 1e-6
        assert a.token_count(0, 0) == lens[0] + step + 1
        ka, va = a.read_kv(0, 0, 1)
        kb, vb = b_.read_kv(0, 0, 1)
        assert np.array_equal(ka.view(np.uint16), kb.view(np.uint16))
        ma, xa = a.read_metadata(0, 1, 3)
        mb, xb = b_.read_metadata(0, 1, 3)
        assert np.array_equal(ma.view(np.uint16), mb.view(np.uint16))
        assert np.array_equal(xa.view(np.uint16), xb.view(np.uint16))


def test_decode_step_host_matches_device(qk):
    rng = np.random.default_rng(5)
    B, H, d, S = 1, 4, 128, 16
    a, _, _ = _layer(qk, rng, B, H, H, d, S, [1000])
    b_, _, _ = _layer(qk, np.random.default_rng(5), B, H, H, d, S, [1000])
    q = half(rng.standard_normal((B, H, d)) / np.sqrt(d)).astype(np.float16)
    kn = half(rng.standard_normal((B, H, d)) / np.sqrt(d)).astype(np.float16)
    out_h = a.decode_step_host(0, q, kn, kn, 256)
    out_d = b_.decode_step(0, torch.from_numpy(q).cuda(), torch.from_numpy(kn).cuda(),
                           torch.from_numpy(kn).cuda(), 256)
    assert np.array_equal(out_h, out_d.cpu().numpy())  # same kernel, same inputs


def test_decode_step_host_consecutive_steps(qk):
    """The host step's completion word (the fused kernel's last unit publishes a sequence
    number the host spins on): eight consecutive host steps, batch 2, GQA 4, each equal to
    the device step on an identical cache."""
    rng = np.random.default_rng(8)
    B, Hq, Hkv, d, S = 2, 8, 2, 128, 16
    a, _, _ = _layer(qk, np.random.default_rng(9), B, Hq, Hkv, d, S, [3000, 41])
    b_, _, _ = _layer(qk, np.random.default_rng(9), B, Hq, Hkv, d, S, [3000, 41])
    for step in range(8):
        q = half(rng.standard_normal((B, Hq, d)) / np.sqrt(d)).astype(np.float16)
        kn = half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d)).astype(np.float16)
        vn = half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d)).astype(np.float16)
        out_h = a.decode_step_host(0, q, kn, vn, 512)
        out_d = b_.decode_step(0, torch.from_numpy(q).cuda(), torch.from_numpy(kn).cuda(),
                               torch.from_numpy(vn).cuda(), 512)
        assert np.array_equal(out_h, out_d.cpu().numpy()), step


@pytest.mark.parametrize("pin", ["all", "q_out", "kv"])
def test_decode_step_host_pinned_buffers_in_place(qk, pin):
    """Caller buffers from qk_host_alloc (questkv.host_empty) are read and written by the
    kernel in place; any mix with pageable or torch-pinned (staged) buffers, and a new
    buffer set every step (the host step's graph re-keys), gives the device step's output
    bitwise."""
    rng = np.random.default_rng(21)
    B, Hq, Hkv, d, S = 2, 8, 2, 128, 16
    a, _, _ = _layer(qk, np.random.default_rng(22), B, Hq, Hkv, d, S, [2500, 77])
    b_, _, _ = _layer(qk, np.random.default_rng(22), B, Hq, Hkv, d, S, [2500, 77])

    def buf(a_np, pinned):
        if not pinned:  # alternate pageable and torch-pinned (both staged)
            return torch.from_numpy(a_np.copy()).pin_memory().numpy() if step % 2 else a_np.copy()
        h = qk.host_empty(a_np.shape, a_np.dtype)
        h[...] = a_np
        return h

    for step in range(4):
        q = half(rng.standard_normal((B, Hq, d)) / np.sqrt(d)).astype(np.float16)
        kn = half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d)).astype(np.float16)
        vn = half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d)).astype(np.float16)
        out = buf(np.zeros((B, Hq, d), np.float32), pin in ("all", "q_out"))
        qh = buf(q, pin in ("all", "q_out"))
        kh, vh = buf(kn, pin in ("all", "kv")), buf(vn, pin in ("all", "kv"))
        got = a.decode_step_host(0, qh, kh, vh, 512, out=out)
        want = b_.decode_step(0, torch.from_numpy(q).cuda(), torch.from_numpy(kn).cuda(),
                              torch.from_numpy(vn).cuda(), 512)
        assert got is out
        assert np.array_equal(got, want.cpu().numpy()), step


def test_host_alloc_is_pinned_and_mapped(qk):
    import ctypes

    from paper_2406_10774_b200 import _lib

    lib = _lib.load()
    p = lib.qk_host_alloc(4096)
    assert p
    arr = (ctypes.c_uint8 * 4096).from_address(p)
    arr[0], arr[4095] = 7, 9
    assert arr[0] == 7 and arr[4095] == 9
    lib.qk_host_free(p)
    lib.qk_host_free(None)
    h = qk.host_empty((3, 5), np.float32)
    h[...] = 2.5
    assert h.shape == (3, 5) and float(h.sum()) == 37.5
