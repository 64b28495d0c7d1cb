import os, sys, numpy as np, torch
os.environ["QK_PROBE"] = "1"
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2406_10774_b200 import QuestCache, _lib
rng = np.random.default_rng(5)
for Hq, L, budget in [(4, 8000, 1024), (4, 32800, 2048), (2, 70000, 4096)]:
    d, S = 128, 16
    vals = np.array([-0.25, 0.0, 0.25], np.float32)
    keys = rng.choice(vals, size=(Hq, L - 1, d)).astype(np.float32); keys[:, :, 4:] = 0
    qc = QuestCache(d, S, num_q_heads=Hq, num_kv_heads=Hq, max_tokens=L + 16)
    qc.prefill(0, 0, torch.from_numpy(keys).half().cuda(), torch.from_numpy(keys).half().cuda())
    q = torch.from_numpy(rng.choice(np.array([-1.0, 1.0], np.float32), size=(1, Hq, d))).half().cuda()
    qc.decode_step(0, q, None, None, budget); torch.cuda.synchronize()
    n = Hq * 16 * 32
    buf = np.zeros(n, dtype=np.uint64)
    _lib.load().qk_debug_probe(qc._h, buf.ctypes.data, buf.size, None)
    t = buf.reshape(-1, 32)
    t = t[t[:, 0] > 0]
    print(Hq, L, budget, "ctas", len(t), "wide pass1 stamped:", int((t[:, 12] > 0).sum()), "pass2:", int((t[:, 13] > 0).sum()))
    qc.close()
