import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2406_10774_b200 import questkv as qk
H, d, S, NL, ctx = 32, 128, 16, 8, 32768
qc = qk.QuestCache(d, S, num_layers=NL, num_q_heads=H, max_tokens=ctx + 4000)
kv = torch.randn((1, H, ctx - 1, d), dtype=torch.float16, device='cuda') / d**0.5
for l in range(NL):
    qc.prefill(l, 0, kv[0], kv[0])
torch.cuda.synchronize()
def mk(pinned):
    t = [torch.randn((NL, 1, H, d), dtype=torch.float16) / d**0.5 for _ in range(3)] + [torch.zeros((NL, 1, H, d), dtype=torch.float32)]
    if pinned: t = [x.pin_memory() for x in t]
    return [x.numpy() for x in t]
for name, pinned in (("pageable", False), ("pinned", True), ("pageable", False), ("pinned", True)):
    q, k, v, o = mk(pinned)
    for _ in range(3):
        for l in range(NL): qc.decode_step_host(l, q[l], k[l], v[l], 2048, out=o[l])
    n = 40
    t0 = time.perf_counter()
    for _ in range(n):
        for l in range(NL): qc.decode_step_host(l, q[l], k[l], v[l], 2048, out=o[l])
    print(name, (time.perf_counter() - t0) * 1e6 / (n * NL), "us/layer")
