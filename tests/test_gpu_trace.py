"""GPU replay of a decode trace (paper_2406_10774_b200/trace.py replay_quest): every step's
page selection from the fused decode kernel equals the oracle's Quest step on the same
fp16 values, and the reported recall / traffic follow the reference's definitions."""

import numpy as np
import pytest

from paper_2406_10774_b200 import trace as tr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("budget,force", [(64, True), (128, False)])
def test_replay_quest_matches_oracle(oracle_c, budget, force):
    rng = np.random.default_rng(budget)
    n, d, S, top_n = 300, 128, 16, 16
    sd = 1 / np.sqrt(d)
    k, v, q = (rng.standard_normal((n, d)).astype(np.float32) * sd for _ in range(3))
    t = tr.make_trace(k, v, q)
    rep = tr.replay_quest(t, budget, top_n, S, force)
    assert len(rep.rows) == n - top_n + 1
    k16, v16, q16 = (a.astype(np.float16).astype(np.float32) for a in (k, v, q))
    for row in rep.rows:
        c = row.step + 1
        _, p_want, o_sparse = oracle_c.quest_step(q16[row.step], k16[:c], v16[:c], S, budget, force,
                                                  True)
        assert row.pages == p_want.tolist(), row.step
        tokens = [x for p in p_want for x in range(p * S, min((p + 1) * S, c))]
        assert row.recall == tr.recall_at_n(tokens, q16[row.step], k16[:c], top_n)
        assert row.traffic == ((c + S - 1) // S + len(tokens)) / c
        # the reference's output_error(sparse, dense) from the oracle's fp64 outputs; the GPU
        # computes both in fp32 (outputs within 1e-5 relative L2 each)
        want_err = tr.output_error(o_sparse, oracle_c.full_attention(q16[row.step], k16[:c], v16[:c]))
        assert abs(row.error - want_err) <= 1e-4 * (1.0 + want_err), row.step
    assert 0.0 < rep.mean_recall <= 1.0
