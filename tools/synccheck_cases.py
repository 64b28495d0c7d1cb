"""One fused decode step per geometry (for compute-sanitizer synccheck triage):
python tools/synccheck_cases.py Hq Hkv B L"""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_10774_b200 import QuestCache  # noqa: E402

Hq, Hkv, B, L = (int(x) for x in sys.argv[1:5])
qc = QuestCache(128, 16, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv, max_tokens=L + 4)
for b in range(B):
    k = (torch.randn((Hkv, L, 128), device="cuda") / 11.3).half()
    qc.prefill(0, b, k, k)
q = (torch.randn((B, Hq, 128), device="cuda") / 11.3).half()
kn = (torch.randn((B, Hkv, 128), device="cuda") / 11.3).half()
qc.decode_step(0, q, kn, kn, 2048)
qc.check_status()
print("ok", Hq, Hkv, B, L)
