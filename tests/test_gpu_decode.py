"""GPU parity of the fused decode step (qk_decode_step, one kernel per layer step):
append -> estimate -> top-K -> sparse attend, against the oracle run per query head on its
KV head's cache.  Scores are not exposed by the fused kernel, so selection (bitwise) and
outputs (relative L2 <= 1e-5) are checked, across MHA/GQA, cluster sizes (1..8 CTAs per
KV head), ragged batches, selection modes and multi-step appends, plus CUDA-graph replay."""

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


class Layer:
    """A QuestCache layer plus a host mirror of every slice for the oracle."""

    def __init__(self, qk, rng, B, Hq, Hkv, d, S, lens, extra=16, keep_scores=True):
        self.qc = qk.QuestCache(d, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                                max_tokens=max(lens) + extra)
        # keep_scores: estimate every page and keep the scores for a bitwise check; off,
        # the production path skips the forced page's estimate (pages/outputs checked).
        self.keep_scores = keep_scores
        self.qc.keep_step_scores(keep_scores)
        self.B, self.Hq, self.Hkv, self.d, self.S = B, Hq, Hkv, d, S
        self.keys, self.vals = [], []
        sd = 1 / np.sqrt(d)
        for b, L in enumerate(lens):
            k = half(rng.standard_normal((Hkv, L, d)) * sd)
            v = half(rng.standard_normal((Hkv, L, d)) * sd)
            if L:
                self.qc.prefill(0, b, torch.from_numpy(k).half().cuda(),
                                torch.from_numpy(v).half().cuda())
            self.keys.append(k)
            self.vals.append(v)

    def step(self, rng, budget, force=True, enabled=True, append=True):
        B, Hq, Hkv, d = self.B, self.Hq, self.Hkv, self.d
        sd = 1 / np.sqrt(d)
        q = half(rng.standard_normal((B, Hq, d)) * sd)
        kn = half(rng.standard_normal((B, Hkv, d)) * sd)
        vn = half(rng.standard_normal((B, Hkv, d)) * sd)
        if append:
            for b in range(B):
                self.keys[b] = np.concatenate([self.keys[b], kn[b][:, None]], axis=1)
                self.vals[b] = np.concatenate([self.vals[b], vn[b][:, None]], axis=1)
        P = max(k.shape[1] for k in self.keys) // self.S + 1
        pages = torch.full((B, Hq, P), -1, dtype=torch.int32, device="cuda")
        counts = torch.zeros((B, Hq), dtype=torch.int32, device="cuda")
        t = lambda a: torch.from_numpy(a).half().cuda()  # noqa: E731
        out = self.qc.decode_step(0, t(q), t(kn) if append else None, t(vn) if append else None,
                                  budget, force, enabled, pages=pages, counts=counts)
        self.qc.check_status()
        return q, out.cpu().numpy(), pages.cpu().numpy(), counts.cpu().numpy()

    def check(self, oracle_c, q, out, pages, counts, budget, force=True, enabled=True):
        G = self.Hq // self.Hkv
        for b in range(self.B):
            for h in range(self.Hq):
                k, v = self.keys[b][h // G], self.vals[b][h // G]
                s_want, p_want, o_want = oracle_c.quest_step(q[b, h], k, v, self.S, budget,
                                                             force, enabled)
                if self.keep_scores:
                    s_got = self.qc.step_scores(b, h, len(s_want))
                    assert np.array_equal(s_got.view(np.uint64), s_want.view(np.uint64)), (b, h)
                got = pages[b, h, : counts[b, h]].tolist()
                assert got == p_want.tolist(), (b, h)
                assert rel_l2(out[b, h], o_want) <= TOL, (b, h)


@pytest.mark.parametrize("B,Hq,Hkv,d,lens,budget", [
    (1, 8, 8, 128, [32767], 2048),        # cfg2 length, the newest token opens page 2047
    (1, 32, 32, 128, [8191], 1024),       # cfg1 (Llama-2-7B layer, 8K, budget 1024)
    (3, 8, 2, 128, [5000, 100, 1], 512),  # GQA 4, ragged, a 1-token sequence
    (2, 16, 2, 128, [3001, 2047], 256),   # GQA 8
    (2, 4, 2, 64, [1500, 33], 128),       # head_dim 64, GQA 2
    (1, 2, 2, 128, [40000], 4096),        # long context, cluster of 8, K = 256
    (1, 4, 4, 100, [700], 64),            # padded head_dim
    (1, 4, 4, 128, [32800], 2048),        # 2051 pages: per-CTA tail pass, 256-thread select
    (1, 4, 4, 128, [65000], 2048),        # 4063 pages: two estimate passes per CTA
    (1, 2, 2, 128, [70000], 2048),        # 4375 pages: the 512-thread select
    (1, 80, 80, 64, [9300], 1024),        # cluster 1, 582 pages per CTA: pipelined passes, d=64
    (1, 40, 40, 128, [19000], 2048),      # cluster 2, 594 pages per CTA: pipelined passes
])
@pytest.mark.parametrize("keep", [True, False])
def test_fused_step_vs_oracle(qk, oracle_c, B, Hq, Hkv, d, lens, budget, keep):
    rng = np.random.default_rng(sum(lens) + 7 * Hq + d)
    layer = Layer(qk, rng, B, Hq, Hkv, d, 16, lens, keep_scores=keep)
    q, out, pages, counts = layer.step(rng, budget)
    layer.check(oracle_c, q, out, pages, counts, budget)


@pytest.mark.parametrize("keep", [True, False])
@pytest.mark.parametrize("budget,force,enabled", [
    (16, True, True),      # K = 1: only the newest page
    (16, False, True),     # K = 1 by score
    (512, False, True),    # no forced page
    (512, True, False),    # selection disabled: dense over every page
    (1 << 20, True, True),  # budget covers the cache
])
def test_fused_selection_modes(qk, oracle_c, budget, force, enabled, keep):
    rng = np.random.default_rng(budget + force)
    layer = Layer(qk, rng, 2, 4, 4, 128, 16, [2500, 97], keep_scores=keep)
    q, out, pages, counts = layer.step(rng, budget, force, enabled)
    layer.check(oracle_c, q, out, pages, counts, budget, force, enabled)


def test_fused_multi_step_appends(qk, oracle_c):
    """Five consecutive steps: every KV head of every sequence appends once per step (the
    length is bumped once, after all heads read it), pages open at the boundary."""
    rng = np.random.default_rng(77)
    layer = Layer(qk, rng, 2, 8, 4, 128, 16, [62, 1023])
    for step in range(5):
        q, out, pages, counts = layer.step(rng, 256)
        layer.check(oracle_c, q, out, pages, counts, 256)
        assert layer.qc.token_count(0, 0) == 63 + step
        assert layer.qc.token_count(0, 1) == 1024 + step
        for b in range(2):
            mn, mx = layer.qc.read_metadata(0, b, 3)
            omn, omx = oracle_c.metadata(layer.keys[b][3], 16)
            assert np.array_equal(mn.astype(np.float32), omn)
            assert np.array_equal(mx.astype(np.float32), omx)


@pytest.mark.parametrize("G", [1, 4])
def test_fused_scores_adversarial_values(qk, oracle_c, G):
    """Exactness of the fused estimate's fp16 -> f64 conversions (XU F2F on even channels,
    the integer 2^-1008-scaled path on odd ones): keys and queries drawn from fp16
    subnormals, +-0, the extremes +-65504 and ordinary values, mixed signs -- scores
    bitwise equal to the oracle."""
    rng = np.random.default_rng(31 + G)
    specials = np.array([0.0, -0.0, 2 ** -24, -(2 ** -24), 3 * 2 ** -24, -(1023 * 2 ** -24),
                         2 ** -14, -(2 ** -14), 65504.0, -65504.0, 1.0, -1.0, 0.5, -3.25],
                        np.float32)
    Hkv, d, S, L = 2, 128, 16, 1000
    qc = qk.QuestCache(d, S, num_q_heads=Hkv * G, num_kv_heads=Hkv, max_tokens=L + 1)
    qc.keep_step_scores(True)
    keys = half(rng.standard_normal((Hkv, L, d)))
    mask = rng.random(keys.shape) < 0.3
    keys[mask] = rng.choice(specials, size=mask.sum())
    vals = half(rng.standard_normal((Hkv, L, d)) * 0.1)
    qc.prefill(0, 0, torch.from_numpy(keys).half().cuda(), torch.from_numpy(vals).half().cuda())
    q = half(rng.standard_normal((1, Hkv * G, d)) * 1e-3)
    qmask = rng.random(q.shape) < 0.3
    q[qmask] = rng.choice(specials[:8], size=qmask.sum())  # keep products finite
    out = qc.decode_step(0, torch.from_numpy(q).half().cuda(), None, None, 256)
    qc.check_status()
    for h in range(Hkv * G):
        mn, mx = oracle_c.metadata(keys[h // G], S)
        want = oracle_c.estimate_all(q[0, h], mn, mx)
        got = qc.step_scores(0, h, len(want))
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), h
    assert torch.isfinite(out).all()


def test_fused_step_without_append(qk, oracle_c):
    rng = np.random.default_rng(5)
    layer = Layer(qk, rng, 1, 4, 4, 128, 16, [4000])
    q, out, pages, counts = layer.step(rng, 1024, append=False)
    layer.check(oracle_c, q, out, pages, counts, 1024)
    assert layer.qc.token_count(0, 0) == 4000


def test_fused_step_graph_replay(qk, oracle_c):
    """A CUDA graph of the step replayed 4 times equals 4 eager steps (device lengths
    advance on replay; qk_sync_lengths refreshes the host shadow)."""
    rng = np.random.default_rng(9)
    B, H, d, S, L = 1, 8, 128, 16, 3000
    eager = Layer(qk, np.random.default_rng(1), B, H, H, d, S, [L])
    graphed = Layer(qk, np.random.default_rng(1), B, H, H, d, S, [L])
    qs = [torch.from_numpy(half(rng.standard_normal((B, H, d)) / np.sqrt(d))).half().cuda()
          for _ in range(4)]
    ks = [torch.from_numpy(half(rng.standard_normal((B, H, d)) / np.sqrt(d))).half().cuda()
          for _ in range(4)]
    qb, kb, vb = qs[0].clone(), ks[0].clone(), ks[0].clone()
    out_g = torch.zeros((B, H, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    warm = Layer(qk, np.random.default_rng(2), B, H, H, d, S, [16])
    warm.qc.decode_step(0, qb, kb, vb, 512, stream=s)  # load the kernel before capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        graphed.qc.decode_step(0, qb, kb, vb, 512, out=out_g, stream=s)
    for i in range(4):
        with torch.cuda.stream(s):
            qb.copy_(qs[i])
            kb.copy_(ks[i])
            vb.copy_(ks[i])
            g.replay()
        s.synchronize()
        ref = eager.qc.decode_step(0, qs[i], ks[i], ks[i], 512)
        assert torch.equal(out_g, ref), i
    graphed.qc.sync_lengths()
    assert graphed.qc.token_count(0, 0) == L + 4 == eager.qc.token_count(0, 0)


def test_fused_graph_replay_outgrows_capture(qk, oracle_c):
    """A graph captured at 2047 pages replayed while the context grows past 2048 pages
    (per-CTA tail pass, 256-thread selection group): every replay equals the eager step
    bitwise, and the last one matches the oracle.  Guards the shared-memory key array
    being sized for the cache, not for the capture-time page count."""
    rng = np.random.default_rng(11)
    B, H, d, S, L, steps = 1, 4, 128, 16, 2047 * 16 - 4, 40
    eager = Layer(qk, np.random.default_rng(3), B, H, H, d, S, [L], extra=steps + 8)
    graphed = Layer(qk, np.random.default_rng(3), B, H, H, d, S, [L], extra=steps + 8)
    sd = 1 / np.sqrt(d)
    qs = [half(rng.standard_normal((B, H, d)) * sd) for _ in range(steps)]
    ks = [half(rng.standard_normal((B, H, d)) * sd) for _ in range(steps)]
    vs = [half(rng.standard_normal((B, H, d)) * sd) for _ in range(steps)]
    t = lambda a: torch.from_numpy(a).half().cuda()  # noqa: E731
    qb, kb, vb = t(qs[0]), t(ks[0]), t(vs[0])
    out_g = torch.zeros((B, H, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    warm = Layer(qk, np.random.default_rng(2), B, H, H, d, S, [16])
    warm.qc.decode_step(0, qb, kb, vb, 2048, stream=s)  # load the kernel before capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        graphed.qc.decode_step(0, qb, kb, vb, 2048, out=out_g, stream=s)
    for i in range(steps):
        with torch.cuda.stream(s):
            qb.copy_(t(qs[i]))
            kb.copy_(t(ks[i]))
            vb.copy_(t(vs[i]))
            g.replay()
        s.synchronize()
        ref = eager.qc.decode_step(0, t(qs[i]), t(ks[i]), t(vs[i]), 2048)
        assert torch.equal(out_g, ref), i
        eager.keys[0] = np.concatenate([eager.keys[0], ks[i][0][:, None]], axis=1)
        eager.vals[0] = np.concatenate([eager.vals[0], vs[i][0][:, None]], axis=1)
    graphed.qc.sync_lengths()
    assert graphed.qc.token_count(0, 0) == L + steps  # 2050 pages at the end
    out = out_g.cpu().numpy()
    for h in range(H):
        _, _, o_want = oracle_c.quest_step(qs[-1][0, h], eager.keys[0][h], eager.vals[0][h], S,
                                           2048, True, True)
        assert rel_l2(out[0, h], o_want) <= TOL, h


@pytest.mark.parametrize("Hq,Hkv,L,budget", [
    (4, 4, 8000, 1024),     # 500 pages: 128-thread group
    (4, 4, 32800, 2048),    # 2051 pages: 256-thread group
    (2, 2, 70000, 4096),    # 4375 pages: the 512-thread select
    (8, 2, 6000, 512),      # GQA 4: per-head groups
])
def test_fused_selection_heavy_ties(qk, oracle_c, Hq, Hkv, L, budget):
    """Keys and queries from tiny value sets: most pages share a score, the boundary bin
    holds far more than 32 keys and the fused kernel takes its multi-pass 64-bit selection
    (ties to the lower page, as criticality.cpp:64-67).  Pages bitwise, outputs 1e-5."""
    rng = np.random.default_rng(L + Hq)
    d, S = 128, 16
    vals = np.array([-0.25, 0.0, 0.25], np.float32)
    layer = Layer(qk, rng, 1, Hq, Hkv, d, S, [1], extra=L + 16)
    keys = rng.choice(vals, size=(Hkv, L - 1, d)).astype(np.float32)
    keys[:, :, 4:] = 0.0  # only 4 channels vary: few distinct page bounds
    values = half(rng.standard_normal((Hkv, L - 1, d)) * 0.1)
    layer.qc = qk.QuestCache(d, S, max_batch=1, num_q_heads=Hq, num_kv_heads=Hkv, max_tokens=L + 16)
    layer.qc.keep_step_scores(True)
    layer.qc.prefill(0, 0, torch.from_numpy(keys).half().cuda(), torch.from_numpy(values).half().cuda())
    layer.keys, layer.vals = [keys], [values]
    q = half(rng.choice(np.array([-1.0, 1.0], np.float32), size=(1, Hq, d)))
    kn = half(rng.choice(vals, size=(1, Hkv, d)))
    vn = half(rng.standard_normal((1, Hkv, d)) * 0.1)
    layer.keys[0] = np.concatenate([layer.keys[0], kn[0][:, None]], axis=1)
    layer.vals[0] = np.concatenate([layer.vals[0], vn[0][:, None]], axis=1)
    P = L // S + 1
    pages = torch.full((1, Hq, P), -1, dtype=torch.int32, device="cuda")
    counts = torch.zeros((1, Hq), dtype=torch.int32, device="cuda")
    t = lambda a: torch.from_numpy(a).half().cuda()  # noqa: E731
    out = layer.qc.decode_step(0, t(q), t(kn), t(vn), budget, pages=pages, counts=counts)
    layer.qc.check_status()
    layer.check(oracle_c, q, out.cpu().numpy(), pages.cpu().numpy(), counts.cpu().numpy(), budget)


@pytest.mark.parametrize("seed", range(32))
def test_fused_step_random_geometry(qk, oracle_c, seed):
    """Seeded random sweep over the fused step's geometry: batch, GQA group, head_dim
    (including padded ones), page size, ragged lengths, budget, forced page, score retention
    and two consecutive steps.  Pages bitwise, outputs within 1e-5 relative L2."""
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 4))
    Hkv = int(rng.choice([1, 2, 4]))
    G = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 80, 96, 128, 128, 200, 256]))  # >128: the unfused route
    S = int(rng.choice([1, 4, 8, 16, 16, 16, 32, 64]))
    max_len = 4000 if S == 1 else 24000
    lens = [int(x) for x in rng.integers(1, max_len, size=B)]
    P = max(lens) // S + 2
    budget = S * int(rng.integers(1, P + 4))
    force = bool(rng.integers(0, 4) > 0)
    keep = bool(rng.integers(0, 2))
    layer = Layer(qk, rng, B, Hkv * G, Hkv, d, S, lens, keep_scores=keep)
    for _ in range(2):
        q, out, pages, counts = layer.step(rng, budget, force)
        layer.check(oracle_c, q, out, pages, counts, budget, force)
