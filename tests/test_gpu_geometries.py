"""GPU parity of the fused decode step at the EXACT benchmark geometries (bench.py CONFIGS):
the cluster size, per-CTA page ranges, tail pass, selection tier and key-exchange path the
timed steps take.  Caches are built on the device (torch RNG, N(0, 1/d) rounded to fp16);
only sampled (sequence, query head) units are copied back and checked against the C oracle
(criticality.cpp:36-81 selection bitwise, attention rel L2 <= 1e-5, scores bitwise when kept).

Geometry notes (decode.cu):
  cfg2  32 units x C=4 -> 128 CTAs; candidates P-1 = 2047 .. 2050: 512-page passes, an 8-page
        tail pass once a CTA's range passes 512 pages (L >= 32785), 128- then 256-thread
        selection groups.  bench.py's timed steps append tokens 32767 .. 32791.
  cfg3  32 units x C=4; candidates cross 8192 (L = 131088): past the shared-memory selection
        tiers the scores go through HBM and the 512-thread selection reads them there.
  cfg4  GQA-4, 32 x 8 = 256 units -> C=1, 4095 candidates > the GQA key array: HBM scores.
  cfg5  8 x 32 = 256 units -> C=1, two waves of one-CTA clusters.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-5
D, S = 128, 16


@pytest.fixture(scope="module")
def qk():
    from paper_2406_10774_b200 import questkv

    return questkv


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.linalg.norm(got - want) / (np.linalg.norm(want) + 1e-30)


class DevLayer:
    """One layer of a QuestCache filled on the device; host mirrors of sampled units only."""

    def __init__(self, qk, seed, B, Hq, Hkv, L, sample, extra=32, keep=False):
        self.qc = qk.QuestCache(D, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                                max_tokens=L + extra)
        self.qc.keep_step_scores(keep)
        self.keep = keep
        self.B, self.Hq, self.Hkv, self.G = B, Hq, Hkv, Hq // Hkv
        self.sample = sample  # [(seq, q_head)]
        self.units = sorted({(b, h // self.G) for b, h in sample})
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(seed)
        self.sd = 1.0 / np.sqrt(D)
        self.k, self.v = {}, {}
        for b in range(B):
            k = (torch.randn((Hkv, L, D), generator=self.gen, device="cuda") * self.sd).half()
            v = (torch.randn((Hkv, L, D), generator=self.gen, device="cuda") * self.sd).half()
            self.qc.prefill(0, b, k, v)
            for (ub, uh) in self.units:
                if ub == b:
                    self.k[(b, uh)] = k[uh].float().cpu().numpy()
                    self.v[(b, uh)] = v[uh].float().cpu().numpy()
            del k, v
        torch.cuda.synchronize()

    def rand(self, shape):
        return (torch.randn(shape, generator=self.gen, device="cuda") * self.sd).half()

    def step(self, budget, force=True, enabled=True):
        B, Hq, Hkv = self.B, self.Hq, self.Hkv
        q, kn, vn = self.rand((B, Hq, D)), self.rand((B, Hkv, D)), self.rand((B, Hkv, D))
        P = max(self.qc.page_count(0, b) for b in range(B)) + 1
        pages = torch.full((B, Hq, P), -1, dtype=torch.int32, device="cuda")
        counts = torch.zeros((B, Hq), dtype=torch.int32, device="cuda")
        out = self.qc.decode_step(0, q, kn, vn, budget, force, enabled, pages=pages,
                                  counts=counts)
        self.qc.check_status()
        knh, vnh = kn.float().cpu().numpy(), vn.float().cpu().numpy()
        for (b, h) in self.units:
            self.k[(b, h)] = np.concatenate([self.k[(b, h)], knh[b, h][None]])
            self.v[(b, h)] = np.concatenate([self.v[(b, h)], vnh[b, h][None]])
        return (q.float().cpu().numpy(), out.cpu().numpy(), pages.cpu().numpy(),
                counts.cpu().numpy())

    def check(self, oracle_c, q, out, pages, counts, budget, force=True, enabled=True):
        for b, h in self.sample:
            k, v = self.k[(b, h // self.G)], self.v[(b, h // self.G)]
            s_want, p_want, o_want = oracle_c.quest_step(q[b, h], k, v, S, budget, force, enabled)
            if self.keep:
                s_got = self.qc.step_scores(b, h, len(s_want))
                assert np.array_equal(s_got.view(np.uint64), s_want.view(np.uint64)), (b, h)
            got = pages[b, h, : counts[b, h]].tolist()
            assert got == p_want.tolist(), (b, h, len(got), len(p_want))
            err = rel_l2(out[b, h], o_want)
            assert err <= TOL, (b, h, err)


SAMPLE32 = [(0, h) for h in (0, 3, 7, 8, 13, 16, 22, 27, 31)]


@pytest.mark.parametrize("L", [32767, 32783, 32784, 32785, 32791, 32800])
@pytest.mark.parametrize("keep", [False, True])
def test_cfg2_geometry(qk, oracle_c, L, keep):
    """cfg2: 32 MHA heads, budget 2048, C=4 -- every page count bench.py's timed steps see,
    the 8-page tail pass (L >= 32784) and the 256-thread selection group (> 2048 cands)."""
    layer = DevLayer(qk, L, 1, 32, 32, L, SAMPLE32, keep=keep)
    q, out, pages, counts = layer.step(2048)
    layer.check(oracle_c, q, out, pages, counts, 2048)


def test_cfg2_geometry_multi_step(qk, oracle_c):
    """cfg2 across the steps bench.py times: 26 consecutive appends from 32767 tokens."""
    layer = DevLayer(qk, 5, 1, 32, 32, 32767, [(0, 0), (0, 17), (0, 31)], extra=40)
    for _ in range(26):
        q, out, pages, counts = layer.step(2048)
        layer.check(oracle_c, q, out, pages, counts, 2048)


@pytest.mark.parametrize("L", [131071, 131087, 131088, 131104])
def test_cfg3_geometry(qk, oracle_c, L):
    """cfg3: 128K context, budget 4096, C=4; the candidate count crosses 8192 (L = 131088:
    8193 candidates) where the shared-memory selection tiers end."""
    layer = DevLayer(qk, L, 1, 32, 32, L, [(0, 0), (0, 9), (0, 20), (0, 31)], keep=(L == 131088))
    q, out, pages, counts = layer.step(4096)
    layer.check(oracle_c, q, out, pages, counts, 4096)


@pytest.mark.parametrize("B", [2, 32])
def test_cfg4_geometry(qk, oracle_c, B):
    """cfg4: GQA 32 q / 8 kv heads at 64K, budget 2048 -- B=2 (16 units, C=8) and the bench's
    B=32 (256 units, C=1); 4095 candidates take the HBM-score selection."""
    sample = [(0, 0), (0, 5), (1, 13), (B - 1, 30), (B // 2, 19)]
    layer = DevLayer(qk, 40 + B, B, 32, 8, 65535, sample)
    q, out, pages, counts = layer.step(2048)
    layer.check(oracle_c, q, out, pages, counts, 2048)


def test_cfg5_geometry(qk, oracle_c):
    """cfg5: batch 8 x 32 heads at 32K, budget 2048: 256 one-CTA clusters in two waves."""
    sample = [(0, 0), (1, 31), (3, 12), (5, 5), (7, 30), (7, 0)]
    layer = DevLayer(qk, 55, 8, 32, 32, 32767, sample)
    for _ in range(2):
        q, out, pages, counts = layer.step(2048)
        layer.check(oracle_c, q, out, pages, counts, 2048)


@pytest.mark.parametrize("keep", [False, True])
def test_gqa_append_without_force(qk, oracle_c, keep):
    """GQA with force_include_recent=false: the appended page competes on score, so its
    staged metadata is patched in shared memory after the append (the patch must follow
    every thread's cp.async of that group, decode.cu)."""
    sample = [(b, h) for b in range(2) for h in range(8)]
    layer = DevLayer(qk, 91, 2, 8, 2, 4095, sample, keep=keep)
    for _ in range(17):  # opens a page and fills it
        q, out, pages, counts = layer.step(512, force=False)
        layer.check(oracle_c, q, out, pages, counts, 512, force=False)


def test_unfused_fallback_through_decode_step(qk, oracle_c):
    """K > 512 pages per head (budget 16384) takes the unfused append -> estimate -> top-K ->
    attend sequence inside qk_decode_step; same results as the fused contract."""
    layer = DevLayer(qk, 17, 1, 4, 4, 40000, [(0, h) for h in range(4)])
    for _ in range(3):
        q, out, pages, counts = layer.step(16384)
        layer.check(oracle_c, q, out, pages, counts, 16384)


def test_unfused_graph_replay_outgrows_capture(qk, oracle_c):
    """A CUDA graph of the unfused decode step (K = 600 pages) captured at 1023 pages and
    replayed while the context grows past 1024 pages: grids and shared memory are sized for
    the cache capacity, so every replay equals the eager step and the oracle."""
    H, L, steps = 2, 1023 * 16 - 3, 24
    eager = DevLayer(qk, 3, 1, H, H, L, [(0, 0), (0, 1)], extra=steps + 8)
    graphed = DevLayer(qk, 3, 1, H, H, L, [(0, 0)], extra=steps + 8)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    rnd = lambda: (torch.randn((1, H, D), generator=gen, device="cuda") / np.sqrt(D)).half()  # noqa
    qs, ks, vs = [rnd() for _ in range(steps)], [rnd() for _ in range(steps)], [rnd() for _ in range(steps)]
    qb, kb, vb = qs[0].clone(), ks[0].clone(), vs[0].clone()
    out_g = torch.zeros((1, H, D), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    warm = qk.QuestCache(D, S, num_q_heads=H, max_tokens=64)
    warm.prefill(0, 0, ks[0].view(H, 1, D).contiguous(), vs[0].view(H, 1, D).contiguous())
    warm.decode_step(0, qb, kb, vb, 9600, stream=s)  # load the kernels before capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        graphed.qc.decode_step(0, qb, kb, vb, 9600, out=out_g, stream=s)
    for i in range(steps):
        with torch.cuda.stream(s):
            qb.copy_(qs[i])
            kb.copy_(ks[i])
            vb.copy_(vs[i])
            g.replay()
        s.synchronize()
        ref = eager.qc.decode_step(0, qs[i], ks[i], vs[i], 9600)
        assert torch.equal(out_g, ref), i
        for h in range(H):
            eager.k[(0, h)] = np.concatenate([eager.k[(0, h)], ks[i][0, h].float().cpu().numpy()[None]])
            eager.v[(0, h)] = np.concatenate([eager.v[(0, h)], vs[i][0, h].float().cpu().numpy()[None]])
    graphed.qc.sync_lengths()
    graphed.qc.check_status()
    assert graphed.qc.token_count(0, 0) == L + steps
    out = out_g.cpu().numpy()
    qh = qs[-1].float().cpu().numpy()
    for h in range(H):
        _, _, o_want = oracle_c.quest_step(qh[0, h], eager.k[(0, h)], eager.v[(0, h)], S, 9600)
        assert rel_l2(out[0, h], o_want) <= TOL, h


def test_sparse_attend_rejects_overlong_count(qk):
    """A device count past the page-list row is rejected (status), not read past the row."""
    qc = qk.QuestCache(D, S, num_q_heads=2, max_tokens=4096)
    k = (torch.randn((2, 4000, D), device="cuda") / np.sqrt(D)).half()
    qc.prefill(0, 0, k, k)
    q = (torch.randn((1, 2, D), device="cuda") / np.sqrt(D)).half()
    pages = torch.arange(8, dtype=torch.int32, device="cuda").view(1, 1, 8).repeat(1, 2, 1)
    counts = torch.tensor([[8, 9]], dtype=torch.int32, device="cuda")
    qc.sparse_attend(0, q, pages, counts)
    with pytest.raises(ValueError):
        qc.check_status()
    counts = torch.tensor([[8, 8]], dtype=torch.int32, device="cuda")
    qc.sparse_attend(0, q, pages, counts)
    qc.check_status()


@pytest.mark.parametrize("L", [65536, 65552])
def test_cfg4_geometry_bench_page_counts(qk, oracle_c, L):
    """cfg4 at the page counts bench.py's timed steps reach: 4097 pages after the append
    (4096 candidates: the row-pair top-K's half-CTA mode) and 4098 (4097 candidates: one
    512-thread row at a time); wide GQA, so the separate kernels run."""
    sample = [(0, 0), (3, 9), (17, 22), (31, 31)]
    layer = DevLayer(qk, L, 32, 32, 8, L, sample)
    q, out, pages, counts = layer.step(2048)
    layer.check(oracle_c, q, out, pages, counts, 2048)


@pytest.mark.parametrize("force", [True, False])
def test_row_pair_topk_mixed_modes(qk, oracle_c, force):
    """select_top_k rows paired across sequences (one query head per sequence): a pair whose
    rows straddle the 4096-candidate bound takes the whole-CTA mode, the others the halves."""
    rng = np.random.default_rng(4097)
    d, Sz = 8, 16
    lens = [65552, 40000, 65537, 65536, 100, 70000]
    B = len(lens)
    qc = qk.QuestCache(d, Sz, max_batch=B, num_q_heads=1, max_tokens=max(lens) + 16)
    for b, L in enumerate(lens):
        k = torch.zeros((1, L, d), dtype=torch.float16, device="cuda")
        qc.prefill(0, b, k, k)
    P = max((L + Sz - 1) // Sz for L in lens)
    scores = torch.from_numpy(rng.standard_normal((B, 1, qc.max_pages))).cuda()
    budget = 1024
    pages, counts = qc.select_topk(0, scores, budget, force)
    pages, counts, sc = pages.cpu().numpy(), counts.cpu().numpy(), scores.cpu().numpy()
    for b, L in enumerate(lens):
        Pb = (L + Sz - 1) // Sz
        want = oracle_c.select_top_k(sc[b, 0, :Pb], Sz, budget, force)
        assert pages[b, 0, :counts[b, 0]].tolist() == want.tolist(), b
