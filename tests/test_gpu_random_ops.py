"""Seeded random-geometry sweep of the separate operator chain the reference's callers use
(estimate_all -> select_top_k -> sparse_attention, plus full_attention and attend_tokens),
through QuestCache against the oracle: batch, GQA group, head_dim (padded ones and > 128),
page size 1..64, ragged lengths, budget, forced page and the disabled mode.  Scores and page
sets bitwise, outputs within 1e-5 relative L2 (attention.cpp:94-116; criticality.cpp:9-81)."""

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


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.linalg.norm(got - want) / (np.linalg.norm(want) + 1e-30)


@pytest.mark.parametrize("seed", range(24))
def test_operator_chain_random_geometry(qk, oracle_c, seed):
    rng = np.random.default_rng(9000 + seed)
    B = int(rng.integers(1, 4))
    Hkv = int(rng.choice([1, 2, 4]))
    G = int(rng.choice([1, 2, 4, 8]))
    Hq = Hkv * G
    d = int(rng.choice([32, 64, 100, 128, 160, 256]))
    S = int(rng.choice([1, 2, 8, 16, 16, 32, 64]))
    lens = [int(x) for x in rng.integers(1, 3000 if S == 1 else 16000, size=B)]
    force = bool(rng.integers(0, 4) > 0)
    enabled = bool(rng.integers(0, 6) > 0)
    qc = qk.QuestCache(d, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                       max_tokens=max(lens) + 8)
    sd = 1 / np.sqrt(d)
    keys, vals = [], []
    for b, L in enumerate(lens):
        k = half(rng.standard_normal((Hkv, L, d)) * sd)
        v = half(rng.standard_normal((Hkv, L, d)) * sd)
        qc.prefill(0, b, torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda())
        keys.append(k)
        vals.append(v)
    P = max((L + S - 1) // S for L in lens)
    budget = S * int(rng.integers(1, P + 3))
    q = half(rng.standard_normal((B, Hq, d)) * sd)
    qd = torch.from_numpy(q).half().cuda()

    scores = qc.estimate(0, qd).cpu().numpy()
    pages, counts = qc.select_topk(0, torch.from_numpy(scores).cuda(), budget, force, enabled)
    out = qc.sparse_attend(0, qd, pages, counts).cpu().numpy()
    dense = qc.dense_attend(0, qd).cpu().numpy()
    pages, counts = pages.cpu().numpy(), counts.cpu().numpy()
    for b in range(B):
        Pb = (lens[b] + S - 1) // S
        for h in range(Hq):
            k, v = keys[b][h // G], vals[b][h // G]
            mn, mx = oracle_c.metadata(k, S)
            s_want = oracle_c.estimate_all(q[b, h], mn, mx)
            assert np.array_equal(scores[b, h, :Pb].view(np.uint64), s_want.view(np.uint64)), (b, h)
            p_want = oracle_c.select_top_k(s_want, S, budget, force, enabled)
            assert pages[b, h, :counts[b, h]].tolist() == p_want.tolist(), (b, h)
            o_want = oracle_c.sparse_attention(q[b, h], k, v, S, p_want)
            assert rel_l2(out[b, h], o_want) <= TOL, (b, h)
            assert rel_l2(dense[b, h], oracle_c.full_attention(q[b, h], k, v)) <= TOL, (b, h)

    # attend_tokens over a random ascending token subset of each row
    stride = max(lens)
    toks = np.zeros((B, Hq, stride), np.int32)
    tcnt = np.zeros((B, Hq), np.int32)
    for b in range(B):
        for h in range(Hq):
            n = int(rng.integers(1, lens[b] + 1))
            sel = np.sort(rng.choice(lens[b], size=n, replace=False)).astype(np.int32)
            toks[b, h, :n] = sel
            tcnt[b, h] = n
    got = qc.attend_tokens(0, qd, torch.from_numpy(toks).cuda(),
                           torch.from_numpy(tcnt).cuda()).cpu().numpy()
    for b in range(B):
        for h in range(Hq):
            k, v = keys[b][h // G], vals[b][h // G]
            want = oracle_c.naive_attention(q[b, h], k, v, toks[b, h, :tcnt[b, h]])
            assert rel_l2(got[b, h], want) <= TOL, (b, h)
