"""GPU parity of the GQA group-shared variant (opt-in, not the
reference's per-head semantics): per (sequence, KV head) ONE page set chosen by
select_top_k's rule from the group score (max / fp64 sum of the exact per-head estimates),
then every query head attends over it on the tensor cores (mma.sync m16n8k16).

Checker: Oracle.group_quest_step, composed from the C restatements of estimate_all,
select_top_k and sparse_attention (criticality.cpp:25-81, attention.cpp:94-116) that are
pinned against the reference.  Bar: page sets bitwise, outputs relative L2 <= 1e-5 (fp32)
and <= 1e-3 (fp16 outputs), as the per-head path."""

import numpy as np
import pytest
import torch

from conftest import half

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def qk():
    from paper_2406_10774_b200 import questkv

    return questkv


def dev16(a):
    return torch.from_numpy(np.asarray(a, np.float16)).cuda()


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.linalg.norm(got - want) / (np.linalg.norm(want) + 1e-30)


def make(qk, rng, B, Hq, Hkv, d, S, lens, extra=8, keyset=None):
    qc = qk.QuestCache(d, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                       max_tokens=max(lens) + extra)
    keys, vals = [], []
    sd = 1 / np.sqrt(d)
    for b, L in enumerate(lens):
        if keyset is None:
            k = half(rng.standard_normal((Hkv, L, d)) * sd)
        else:  # tie stress: keys from a tiny value set
            k = half(rng.choice(keyset, size=(Hkv, L, d)))
        v = half(rng.standard_normal((Hkv, L, d)) * sd)
        qc.prefill(0, b, dev16(k), dev16(v))
        keys.append(k)
        vals.append(v)
    return qc, keys, vals


def check_step(orc, qc, keys, vals, q, pages, counts, out, S, budget, reduce, force=True,
               enabled=True, tol=TOL):
    B, Hq, d = q.shape
    Hkv = keys[0].shape[0]
    G = Hq // Hkv
    pages, counts, out = pages.cpu().numpy(), counts.cpu().numpy(), out.float().cpu().numpy()
    for b in range(B):
        for kvh in range(Hkv):
            qs = q[b, kvh * G:(kvh + 1) * G].astype(np.float32)
            _, want_pages, want_out = orc.group_quest_step(
                qs, keys[b][kvh].astype(np.float32), vals[b][kvh].astype(np.float32), S, budget,
                reduce, force, enabled)
            n = int(counts[b, kvh])
            assert pages[b, kvh, :n].tolist() == want_pages.tolist(), (b, kvh)
            for g in range(G):
                err = rel_l2(out[b, kvh * G + g], want_out[g])
                assert err <= tol, (b, kvh, g, err)


@pytest.mark.parametrize("Hq,Hkv,d,S,lens,budget,reduce,force", [
    (8, 2, 128, 16, [1000, 1777], 256, "max", True),
    (8, 2, 128, 16, [1000, 1777], 256, "sum", True),
    (16, 2, 128, 16, [3001], 512, "max", False),
    (8, 4, 64, 16, [640, 333, 1025], 128, "sum", False),
    (4, 2, 128, 32, [999], 256, "max", True),     # two 16-token chunks per page
    (4, 1, 128, 8, [515], 64, "sum", True),       # half-chunk pages (masked rows)
    (4, 4, 128, 16, [700], 128, "max", True),     # G = 1: the reference's per-head rule
    (32, 8, 128, 16, [4097, 2049], 2048, "max", True),  # cfg4 shape, two requests
    (4, 1, 128, 16, [200], 4096, "max", True),    # budget covers the cache: every page
])
def test_grouped_step_vs_oracle(qk, Hq, Hkv, d, S, lens, budget, reduce, force):
    from oracle import Oracle

    rng = np.random.default_rng(Hq * 1000 + sum(lens) + budget)
    B = len(lens)
    qc, keys, vals = make(qk, rng, B, Hq, Hkv, d, S, lens)
    sd = 1 / np.sqrt(d)
    q = half(rng.standard_normal((B, Hq, d)) * sd)
    kn = half(rng.standard_normal((B, Hkv, d)) * sd)
    vn = half(rng.standard_normal((B, Hkv, d)) * sd)
    for b in range(B):
        keys[b] = np.concatenate([keys[b], kn[b][:, None]], axis=1)
        vals[b] = np.concatenate([vals[b], vn[b][:, None]], axis=1)
    P = max((L + 1 + S - 1) // S for L in lens)
    pages = torch.full((B, Hkv, P), -1, dtype=torch.int32, device="cuda")
    counts = torch.zeros((B, Hkv), dtype=torch.int32, device="cuda")
    out = qc.decode_step_grouped(0, dev16(q), dev16(kn),
                                 dev16(vn), budget, reduce, force,
                                 pages=pages, counts=counts)
    qc.check_status()
    check_step(Oracle(), qc, keys, vals, q, pages, counts, out, S, budget, reduce, force)


def test_grouped_separable_ops_equal_the_step(qk):
    """estimate -> select_topk_grouped -> sparse_attend_grouped == decode_step_grouped
    (same kernels, bitwise), and the fp16 output is the fp32 one rounded."""
    from oracle import Oracle

    rng = np.random.default_rng(11)
    qc, keys, vals = make(qk, rng, 2, 16, 4, 128, 16, [2500, 1600])
    q = half(rng.standard_normal((2, 16, 128)) / np.sqrt(128))
    qd = dev16(q)
    scores = qc.estimate(0, qd)
    pages, counts = qc.select_topk_grouped(0, scores, 512, "sum")
    out = qc.sparse_attend_grouped(0, qd, pages, counts)
    out16 = qc.sparse_attend_grouped(0, qd, pages, counts, out_dtype=torch.float16)
    p2 = torch.full_like(pages, -1)
    c2 = torch.zeros_like(counts)
    step = qc.decode_step_grouped(0, qd, None, None, 512, "sum", pages=p2, counts=c2)
    qc.check_status()
    assert torch.equal(pages, p2) and torch.equal(counts, c2)
    assert torch.equal(out, step)
    assert torch.equal(out16, out.half())
    check_step(Oracle(), qc, keys, vals, q, pages, counts, out, 16, 512, "sum", True)
    check_step(Oracle(), qc, keys, vals, q, pages, counts, out16, 16, 512, "sum", True, tol=1e-3)


def test_grouped_heavy_ties_are_bitwise(qk):
    from oracle import Oracle

    rng = np.random.default_rng(5)
    qc, keys, vals = make(qk, rng, 1, 8, 2, 128, 16, [2048], keyset=[-0.5, 0.0, 0.25, 0.5])
    q = half(rng.choice([-1.0, 0.0, 1.0], size=(1, 8, 128)))
    qd = dev16(q)
    for reduce in ("max", "sum"):
        pages, counts = qc.select_topk_grouped(0, qc.estimate(0, qd), 256, reduce)
        out = qc.sparse_attend_grouped(0, qd, pages, counts)
        qc.check_status()
        check_step(Oracle(), qc, keys, vals, q, pages, counts, out, 16, 256, reduce, True)


def test_group_of_one_is_the_per_head_selection(qk):
    """G = 1: the group score is the head's score, so the page sets equal select_top_k's
    and the tensor-core attention equals the per-head kernel within fp32 rounding."""
    rng = np.random.default_rng(3)
    qc, keys, vals = make(qk, rng, 2, 4, 4, 128, 16, [1500, 900])
    q = dev16(half(rng.standard_normal((2, 4, 128)) / np.sqrt(128)))
    scores = qc.estimate(0, q)
    gp, gc = qc.select_topk_grouped(0, scores, 256)
    hp, hc = qc.select_topk(0, scores, 256)
    assert torch.equal(gp, hp) and torch.equal(gc, hc)
    got = qc.sparse_attend_grouped(0, q, gp, gc).cpu().numpy()
    want = qc.sparse_attend(0, q, hp, hc).cpu().numpy()
    assert rel_l2(got, want) <= 1e-6


def test_grouped_dense_budget_matches_dense_attention(qk):
    rng = np.random.default_rng(9)
    qc, keys, vals = make(qk, rng, 1, 8, 2, 128, 16, [3000])
    q = dev16(half(rng.standard_normal((1, 8, 128)) / np.sqrt(128)))
    pages, counts = qc.select_topk_grouped(0, qc.estimate(0, q), 1 << 20)
    assert counts.cpu().tolist() == [[188, 188]]
    got = qc.sparse_attend_grouped(0, q, pages, counts).cpu().numpy()
    want = qc.dense_attend(0, q).cpu().numpy()
    assert rel_l2(got, want) <= 1e-6


def test_grouped_errors(qk):
    rng = np.random.default_rng(1)
    qc, keys, vals = make(qk, rng, 1, 8, 2, 128, 16, [300])
    q = dev16(half(rng.standard_normal((1, 8, 128))))
    with pytest.raises(ValueError, match="group_reduce"):
        qc.decode_step_grouped(0, q, None, None, 64, "mean")
    with pytest.raises(ValueError, match="token_budget below page_size"):
        qc.decode_step_grouped(0, q, None, None, 8)
    bad = torch.tensor([[[3, 2, 7], [1, 2, 3]]], dtype=torch.int32, device="cuda")
    cnt = torch.tensor([[3, 3]], dtype=torch.int32, device="cuda")
    qc.sparse_attend_grouped(0, q, bad, cnt)
    with pytest.raises(ValueError):
        qc.check_status()
    oob = torch.tensor([[[0, 1, 99], [1, 2, 3]]], dtype=torch.int32, device="cuda")
    qc.sparse_attend_grouped(0, q, oob, cnt)
    with pytest.raises(IndexError):
        qc.check_status()


def test_grouped_graph_replay_grows_the_context(qk):
    """A CUDA graph of decode_step_grouped captured at one length replays correctly as the
    appends grow the cache (grids and shared memory are sized for the capacity)."""
    from oracle import Oracle

    rng = np.random.default_rng(21)
    Hq, Hkv, d, S, L0, steps, budget = 8, 2, 128, 16, 1000, 40, 256
    qc, keys, vals = make(qk, rng, 1, Hq, Hkv, d, S, [L0], extra=steps + 8)
    sd = 1 / np.sqrt(d)
    q = torch.zeros((1, Hq, d), dtype=torch.float16, device="cuda")
    kn = torch.zeros((1, Hkv, d), dtype=torch.float16, device="cuda")
    vn = torch.zeros_like(kn)
    out = torch.empty((1, Hq, d), dtype=torch.float32, device="cuda")
    P = (L0 + steps + S - 1) // S
    pages = torch.full((1, Hkv, P), -1, dtype=torch.int32, device="cuda")
    counts = torch.zeros((1, Hkv), dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    warm, _, _ = make(qk, rng, 1, Hq, Hkv, d, S, [64])
    warm.decode_step_grouped(0, q, kn, vn, budget, "max")  # load the kernels before capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        qc.decode_step_grouped(0, q, kn, vn, budget, "max", out=out, pages=pages, counts=counts,
                               stream=torch.cuda.current_stream())
    qc.sync_lengths()
    orc = Oracle()
    for t in range(steps):
        qh = half(rng.standard_normal((1, Hq, d)) * sd)
        kh = half(rng.standard_normal((1, Hkv, d)) * sd)
        vh = half(rng.standard_normal((1, Hkv, d)) * sd)
        q.copy_(dev16(qh))
        kn.copy_(dev16(kh))
        vn.copy_(dev16(vh))
        g.replay()
        torch.cuda.synchronize()
        keys[0] = np.concatenate([keys[0], kh[0][:, None]], axis=1)
        vals[0] = np.concatenate([vals[0], vh[0][:, None]], axis=1)
        if t % 13 == 0 or t == steps - 1:
            check_step(orc, qc, keys, vals, qh, pages, counts, out, S, budget, "max")
    qc.sync_lengths()
    assert qc.token_count(0, 0) == L0 + steps


@pytest.mark.parametrize("seed", range(16))
def test_grouped_step_random_geometry(qk, seed):
    """Seeded random sweep: batch, group, head_dim (padded ones too), page size, ragged
    lengths, budget, reduction and forced page.  Pages bitwise, outputs 1e-5 relative L2."""
    from oracle import Oracle

    rng = np.random.default_rng(5000 + seed)
    B = int(rng.integers(1, 4))
    Hkv = int(rng.choice([1, 2, 4]))
    G = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 80, 96, 128]))
    S = int(rng.choice([4, 8, 16, 16, 32, 64]))
    lens = [int(x) for x in rng.integers(1, 12000, size=B)]
    P = max((L + 1 + S - 1) // S for L in lens)
    budget = S * int(rng.integers(1, P + 4))
    reduce = str(rng.choice(["max", "sum"]))
    force = bool(rng.integers(0, 4) > 0)
    Hq = Hkv * G
    qc, keys, vals = make(qk, rng, B, Hq, Hkv, d, S, lens)
    sd = 1 / np.sqrt(d)
    q = half(rng.standard_normal((B, Hq, d)) * sd)
    kn = half(rng.standard_normal((B, Hkv, d)) * sd)
    vn = half(rng.standard_normal((B, Hkv, d)) * sd)
    for b in range(B):
        keys[b] = np.concatenate([keys[b], kn[b][:, None]], axis=1)
        vals[b] = np.concatenate([vals[b], vn[b][:, None]], axis=1)
    pages = torch.full((B, Hkv, P), -1, dtype=torch.int32, device="cuda")
    counts = torch.zeros((B, Hkv), dtype=torch.int32, device="cuda")
    out = qc.decode_step_grouped(0, dev16(q), dev16(kn), dev16(vn), budget, reduce, force,
                                 pages=pages, counts=counts)
    qc.check_status()
    check_step(Oracle(), qc, keys, vals, q, pages, counts, out, S, budget, reduce, force)
