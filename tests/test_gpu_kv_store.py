"""GPU parity: KvCache append + fused metadata update (K1) and the bulk prefill.

Restates /root/reference/proj/tests/test_kv_store.cpp against the CUDA path (through the
C ABI via paper_2406_10774_b200.questkv) and checks metadata bitwise against the oracle."""

import numpy as np
import pytest
import torch

from conftest import half

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qk():
    from paper_2406_10774_b200 import questkv

    return questkv


def test_empty_construction(qk):
    # test_kv_store.cpp:16-20
    c = qk.KvCache(qk.CacheConfig(head_dim=128, page_size=16))
    assert c.token_count() == 0 and c.page_count() == 0


def test_invalid_configs_rejected(qk):
    # test_kv_store.cpp:22-28
    with pytest.raises(ValueError):
        qk.KvCache(qk.CacheConfig(head_dim=0, page_size=16))
    with pytest.raises(ValueError):
        qk.KvCache(qk.CacheConfig(head_dim=4, page_size=0))
    with pytest.raises(ValueError):
        qk.KvCache(qk.CacheConfig(head_dim=4, page_size=4, bytes_per_element=0))


def test_degenerate_page_size_of_one(qk):
    # test_kv_store.cpp:30-37
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=1))
    c.append([1, 2], [0, 0])
    c.append([3, 4], [0, 0])
    assert c.page_count() == 2
    assert c.page(0).length == 1 and c.page(1).length == 1


def test_append_maintains_min_max(qk):
    # test_kv_store.cpp:39-51
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=4))
    c.append([1, 5], [0, 0])
    c.append([3, 2], [0, 0])
    m = c.page_metadata(0)
    assert m.min_key == [1, 2] and m.max_key == [3, 5]


def test_first_key_seeds_metadata(qk):
    # test_kv_store.cpp:53-59
    c = qk.KvCache(qk.CacheConfig(head_dim=3, page_size=8))
    c.append([-2.5, 0.0, 7.25], [0, 0, 0])
    assert c.page_metadata(0).min_key == [-2.5, 0.0, 7.25]
    assert c.page_metadata(0).max_key == [-2.5, 0.0, 7.25]


def test_paging_arithmetic(qk):
    # test_kv_store.cpp:61-73
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2))
    for i in range(3):
        assert c.append([float(i), 0], [0, float(i)]) == i
    assert c.page_count() == 2
    assert c.page(0).length == 2 and c.page(1).length == 1
    assert c.key(2)[0] == 2.0 and c.value(2)[1] == 2.0


def test_dimension_mismatch_and_range_errors(qk):
    # test_kv_store.cpp:75-84
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2))
    with pytest.raises(ValueError):
        c.append([1], [1, 2])
    with pytest.raises(IndexError):
        c.page_metadata(0)
    c.append([1, 2], [3, 4])
    with pytest.raises(IndexError):
        c.page_metadata(1)
    with pytest.raises(IndexError):
        c.key(1)
    with pytest.raises(IndexError):
        c.value(7)


def test_kv_cache_grows_past_its_capacity(qk, oracle_c):
    """The reference's KvCache grows without bound (kv_store.cpp:24-29); the GPU KvCache starts
    at `capacity` and doubles through qk_cache_reserve, keeping pages and metadata bitwise."""
    rng = np.random.default_rng(3)
    d, S = 5, 3
    keys = half(rng.standard_normal((200, d)))
    vals = half(rng.standard_normal((200, d)))
    c = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=2)
    for t in range(70):  # 2 -> 4 -> ... -> 128
        assert c.append(keys[t], vals[t]) == t
    c.extend(keys[70:], vals[70:])  # one reserve for the bulk
    assert c.token_count() == 200 and c.page_count() == 67
    assert c.quest_cache.max_tokens >= 200
    mn, mx = c.quest_cache.read_metadata(0, 0, 0)
    omn, omx = oracle_c.metadata(keys, S)
    assert np.array_equal(mn.astype(np.float32).view(np.uint32), omn.view(np.uint32))
    assert np.array_equal(mx.astype(np.float32).view(np.uint32), omx.view(np.uint32))
    k, v = c.quest_cache.read_kv(0, 0, 0, 0, 200)
    assert np.array_equal(k, keys.astype(np.float16)) and np.array_equal(v, vals.astype(np.float16))


def test_kv_cache_growth_stops_at_the_page_limit(qk):
    c = qk.KvCache(qk.CacheConfig(head_dim=1, page_size=1), capacity=16)
    c.extend(np.ones((16384, 1)), np.ones((16384, 1)))
    assert c.token_count() == 16384
    with pytest.raises(NotImplementedError):
        c.append([1], [1])
    assert c.token_count() == 16384


def test_quest_cache_capacity_is_out_of_range(qk):
    """The batched cache never grows implicitly: a full slice raises until reserve()."""
    qc = qk.QuestCache(2, 2, max_tokens=2)
    one = torch.ones((1, 1, 2), dtype=torch.float16, device="cuda")
    qc.append(0, one, one)
    qc.append(0, one, one)
    with pytest.raises(IndexError):
        qc.append(0, one, one)
    qc.reserve(3)
    qc.append(0, one, one)
    assert qc.token_count() == 3


def test_reserve_keeps_every_slice_and_the_step_matches(qk, oracle_c):
    """Multi-layer, batched, GQA cache grown mid-sequence: every (layer, sequence, KV head)
    slice keeps its pages, metadata and length, and the fused step then equals the oracle."""
    rng = np.random.default_rng(11)
    Lyr, B, Hq, Hkv, d, S = 2, 2, 4, 2, 128, 16
    lens = [700, 333]
    qc = qk.QuestCache(d, S, num_layers=Lyr, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                       max_tokens=max(lens))
    keys = [[half(rng.standard_normal((Hkv, L, d)) / np.sqrt(d)) for L in lens] for _ in range(Lyr)]
    vals = [[half(rng.standard_normal((Hkv, L, d)) / np.sqrt(d)) for L in lens] for _ in range(Lyr)]
    for layer in range(Lyr):
        for b in range(B):
            qc.prefill(layer, b, torch.from_numpy(keys[layer][b]).half().cuda(),
                       torch.from_numpy(vals[layer][b]).half().cuda())
    bytes_before = qc._lib.qk_cache_device_bytes(qc._h)
    qc.reserve(5000)
    assert qc.max_tokens == 5000 and qc.max_pages == 313
    assert qc._lib.qk_cache_device_bytes(qc._h) > bytes_before
    for layer in range(Lyr):
        for b in range(B):
            assert qc.token_count(layer, b) == lens[b]
            for h in range(Hkv):
                mn, mx = qc.read_metadata(layer, b, h)
                omn, omx = oracle_c.metadata(keys[layer][b][h], S)
                assert np.array_equal(mn.astype(np.float32).view(np.uint32), omn.view(np.uint32))
                assert np.array_equal(mx.astype(np.float32).view(np.uint32), omx.view(np.uint32))
    # Steps on layer 1 after the growth: append, estimate, select, attend against the oracle.
    G = Hq // Hkv
    for _ in range(2):
        q = half(rng.standard_normal((B, Hq, d)) / np.sqrt(d))
        kn = half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d))
        vn = half(rng.standard_normal((B, Hkv, d)) / np.sqrt(d))
        for b in range(B):
            keys[1][b] = np.concatenate([keys[1][b], kn[b][:, None]], axis=1)
            vals[1][b] = np.concatenate([vals[1][b], vn[b][:, None]], axis=1)
        P = qc.max_pages
        pages = torch.full((B, Hq, P), -1, dtype=torch.int32, device="cuda")
        counts = torch.zeros((B, Hq), dtype=torch.int32, device="cuda")
        t = lambda a: torch.from_numpy(a).half().cuda()  # noqa: E731
        out = qc.decode_step(1, t(q), t(kn), t(vn), 256, pages=pages, counts=counts)
        qc.check_status()
        out, pages, counts = out.cpu().numpy(), pages.cpu().numpy(), counts.cpu().numpy()
        for b in range(B):
            for h in range(Hq):
                _, p_want, o_want = oracle_c.quest_step(q[b, h], keys[1][b][h // G],
                                                        vals[1][b][h // G], S, 256)
                assert pages[b, h, :counts[b, h]].tolist() == p_want.tolist()
                err = np.linalg.norm(out[b, h] - o_want) / np.linalg.norm(o_want)
                assert err <= 1e-5


def test_metadata_equals_rescan_property(qk, oracle_c):
    # test_kv_store.cpp:89-113, 150 random sequences through single-token appends
    rng = np.random.default_rng(20240811)
    for _ in range(150):
        d, S, L = int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 33))
        keys = half(rng.standard_normal((L, d)))
        c = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=64)
        for t in range(L):
            c.append(keys[t], np.zeros(d))
        assert c.token_count() == L and c.page_count() == (L + S - 1) // S
        mn, mx = c.quest_cache.read_metadata(0, 0, 0)
        omn, omx = oracle_c.metadata(keys, S)
        assert np.array_equal(mn.astype(np.float32).view(np.uint32), omn.view(np.uint32))
        assert np.array_equal(mx.astype(np.float32).view(np.uint32), omx.view(np.uint32))


def test_signed_zeros_keep_first_seen(qk):
    # kv_store.cpp:40-43: append(+0, -0) keeps +0; append(-0, +0) keeps -0
    for first, second in ((0.0, -0.0), (-0.0, 0.0)):
        c = qk.KvCache(qk.CacheConfig(head_dim=1, page_size=4))
        c.append([first], [0])
        c.append([second], [0])
        mn, mx = c.quest_cache.read_metadata(0, 0, 0)
        assert np.signbit(mn[0, 0]) == np.signbit(np.float16(first))
        assert np.signbit(mx[0, 0]) == np.signbit(np.float16(first))


def test_reads_are_pure(qk):
    # test_kv_store.cpp:115-125
    c = qk.KvCache(qk.CacheConfig(head_dim=2, page_size=2))
    c.append([1, 2], [3, 4])
    before = c.page_metadata(0)
    c.key(0), c.value(0), c.page(0)
    assert c.page_metadata(0) == before and c.token_count() == 1


@pytest.mark.parametrize("d,S", [(128, 16), (64, 16), (100, 7), (256, 8), (3, 1)])
def test_prefill_equals_appends_bitwise(qk, d, S):
    """qk_prefill (page-parallel) leaves exactly the pages and metadata of n appends,
    including a first page already partly filled and signed zeros."""
    rng = np.random.default_rng(d * 100 + S)
    L1, L2 = int(rng.integers(1, 3 * S)), int(rng.integers(1, 200))
    keys = half(rng.standard_normal((L1 + L2, d)) * 0.3)
    keys[rng.random(keys.shape) < 0.05] = -0.0
    keys[rng.random(keys.shape) < 0.05] = 0.0
    vals = half(rng.standard_normal((L1 + L2, d)))
    a = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=512)
    b = qk.KvCache(qk.CacheConfig(head_dim=d, page_size=S), capacity=512)
    for t in range(L1 + L2):
        a.append(keys[t], vals[t])
    b.extend(keys[:L1], vals[:L1])
    b.extend(keys[L1:], vals[L1:])
    ma, xa = a.quest_cache.read_metadata(0, 0, 0)
    mb, xb = b.quest_cache.read_metadata(0, 0, 0)
    assert np.array_equal(ma.view(np.uint16), mb.view(np.uint16))
    assert np.array_equal(xa.view(np.uint16), xb.view(np.uint16))
    ka, va = a.quest_cache.read_kv(0, 0, 0)
    kb, vb = b.quest_cache.read_kv(0, 0, 0)
    assert np.array_equal(ka.view(np.uint16), kb.view(np.uint16))
    assert np.array_equal(va.view(np.uint16), vb.view(np.uint16))
    assert np.array_equal(ka.astype(np.float32), keys)


def test_batched_append_all_heads(qk, oracle_c):
    """qk_append over a batch of sequences x KV heads x layers matches per-slice oracles."""
    rng = np.random.default_rng(3)
    L, B, H, d, S = 2, 3, 4, 128, 16
    qc = qk.QuestCache(d, S, num_layers=L, max_batch=B, num_q_heads=H, max_tokens=128)
    ks = half(rng.standard_normal((40, L, B, H, d)))
    for t in range(40):
        for layer in range(L):
            k = torch.from_numpy(ks[t, layer]).half().cuda()
            qc.append(layer, k, k)
    for layer in range(L):
        for b in range(B):
            assert qc.token_count(layer, b) == 40
            for h in range(H):
                mn, mx = qc.read_metadata(layer, b, h)
                omn, omx = oracle_c.metadata(ks[:, layer, b, h], S)
                assert np.array_equal(mn.astype(np.float32), omn)
                assert np.array_equal(mx.astype(np.float32), omx)
