"""Bulk prefill throughput (qk_prefill): one layer of the cfg2 shape (32 KV heads x 32767
tokens x d=128), CUDA events around the launch; bytes = K/V in + K/V out + metadata out."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_10774_b200 import QuestCache  # noqa: E402

H, L, D, S = 32, 32767, 128, 16
qc = QuestCache(D, S, num_layers=4, num_q_heads=H, num_kv_heads=H, max_tokens=L + 8)
k = (torch.randn((H, L, D), device="cuda") / D ** 0.5).half()
v = (torch.randn((H, L, D), device="cuda") / D ** 0.5).half()
for layer in range(4):
    qc.prefill(layer, 0, k, v)
torch.cuda.synchronize()
best = 1e9
for rep in range(6):
    qc.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    qc.prefill(rep % 4, 0, k, v)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1e3)
P = (L + S - 1) // S
nbytes = 2 * (2 * H * L * D * 2) + H * 2 * D * P * 2
print(json.dumps({"prefill_us": round(best, 1), "bytes": nbytes,
                  "gbs": round(nbytes / (best * 1e-6) / 1e9, 1)}))
