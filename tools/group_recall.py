#!/usr/bin/env python
"""Recall and K/V traffic of GQA group-shared selection vs the reference's per-head
selection, on the GPU path.

    python tools/group_recall.py [--ctx 8192] [--group 4] [--top-n 32] [--trials 16]

Synthetic GQA data with attention structure (random N(0, 1/d) data has none): keys are
N(0, 1/d) plus, for 10% of the tokens, a strong component along one of 64 "topic"
directions; the G query heads of a group share a topic and differ by per-head noise
(correlation `--rho`).  Per KV head and budget this reports, averaged over trials:
  * recall@n of each query head (trace.recall_at_n, the reference's metric,
    metrics.cpp:12-38) under per-head selection (qk_select_topk) and group-shared selection
    (qk_select_topk_grouped, max and sum);
  * K/V tokens read per KV head: the union of the G per-head page sets vs the one shared set.
Prints one JSON line per budget.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_10774_b200 import QuestCache  # noqa: E402
from paper_2406_10774_b200.trace import recall_at_n  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=8192)
    ap.add_argument("--group", type=int, default=4)
    ap.add_argument("--top-n", type=int, default=32)
    ap.add_argument("--trials", type=int, default=16)
    ap.add_argument("--rho", type=float, default=0.8)
    ap.add_argument("--budgets", default="256,512,1024,2048")
    a = ap.parse_args()
    d, S, G, L = 128, 16, a.group, a.ctx
    rng = np.random.default_rng(7)
    sd = 1 / np.sqrt(d)
    topics = rng.standard_normal((64, d)) / np.sqrt(d)
    keys = rng.standard_normal((L, d)) * sd
    hot = rng.random(L) < 0.1
    z = rng.integers(0, 64, L)
    keys[hot] += 3.0 * topics[z[hot]] * np.sqrt(d) * sd
    k16 = keys.astype(np.float16)
    v16 = (rng.standard_normal((L, d)) * sd).astype(np.float16)
    qc = QuestCache(d, S, num_q_heads=G, num_kv_heads=1, max_tokens=L)
    qc.prefill(0, 0, torch.from_numpy(k16).cuda().view(1, L, d),
               torch.from_numpy(v16).cuda().view(1, L, d))
    kf = k16.astype(np.float32)
    for budget in [int(x) for x in a.budgets.split(",")]:
        acc = {"per_head": [], "group_max": [], "group_sum": []}
        tok = {"per_head": [], "group_max": [], "group_sum": []}
        for _ in range(a.trials):
            base = topics[rng.integers(0, 64)] * np.sqrt(d)
            qs = np.stack([a.rho * base + np.sqrt(1 - a.rho ** 2) * rng.standard_normal(d)
                           for _ in range(G)]) * sd * 4
            q16 = qs.astype(np.float16)
            q = torch.from_numpy(q16).cuda().view(1, G, d)
            scores = qc.estimate(0, q)
            hp, hc = qc.select_topk(0, scores, budget)
            sets = {"per_head": [hp[0, g, :hc[0, g]].cpu().numpy() for g in range(G)]}
            for red in ("max", "sum"):
                gp, gc = qc.select_topk_grouped(0, scores, budget, red)
                shared = gp[0, 0, :gc[0, 0]].cpu().numpy()
                sets[f"group_{red}"] = [shared] * G
            for mode, pages in sets.items():
                rec = []
                for g in range(G):
                    t = np.concatenate([np.arange(p * S, min((p + 1) * S, L)) for p in pages[g]])
                    rec.append(recall_at_n(t, q16[g].astype(np.float32), kf, a.top_n))
                acc[mode].append(float(np.mean(rec)))
                union = set()
                for g in range(G):
                    union.update(pages[g].tolist())
                tok[mode].append(len(union) * S)
        line = {"ctx": L, "group": G, "budget": budget, "top_n": a.top_n, "rho": a.rho,
                "trials": a.trials}
        for mode in acc:
            line[f"recall_{mode}"] = round(float(np.mean(acc[mode])), 4)
            line[f"kv_tokens_{mode}"] = round(float(np.mean(tok[mode])), 1)
        print(json.dumps(line))
    qc.close()


if __name__ == "__main__":
    main()
