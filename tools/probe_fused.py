"""Phase timeline of the fused decode kernel (QK_PROBE globaltimer stamps).

    QK_PROBE=1 python tools/probe_fused.py [--ctx 32768] [--budget 2048] [--heads 32]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("QK_PROBE", "1")

from paper_2406_10774_b200 import QuestCache  # noqa: E402
from paper_2406_10774_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--budget", type=int, default=2048)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=None)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
H, D, S = args.heads, 128, 16
Hkv = args.kv_heads or H
dev = torch.device("cuda", 0)
qc = QuestCache(D, S, num_layers=args.layers, max_batch=args.batch, num_q_heads=H,
                num_kv_heads=Hkv, max_tokens=args.ctx + 64)
g = torch.Generator(device=dev)
g.manual_seed(0)
for layer in range(args.layers):
    for b in range(args.batch):
        k = (torch.randn((Hkv, args.ctx - 1, D), generator=g, device=dev) / D ** 0.5).half()
        qc.prefill(layer, b, k, k)
q = (torch.randn((args.batch, H, D), generator=g, device=dev) / D ** 0.5).half()
kn = (torch.randn((args.batch, Hkv, D), generator=g, device=dev) / D ** 0.5).half()
out = torch.empty((args.batch, H, D), dtype=torch.float32, device=dev)
torch.cuda.synchronize()
n = args.batch * Hkv * 8 * 16
buf = np.zeros(n, dtype=np.uint64)
lib = _lib.load()
names = ["wait", "qload+estimate", "barrier1", "select", "attend", "barrier2", "merge"]
res = []
for rep in range(args.reps):
    for layer in range(args.layers):
        qc.decode_step(layer, q, kn, kn, args.budget, out=out)
        torch.cuda.synchronize()
        lib.qk_debug_probe(qc._h, buf.ctypes.data, n, None)
        t16 = buf.reshape(-1, 16).astype(np.int64)
        valid = t16[:, 0] > 0
        t16 = t16[valid]
        t = t16[:, :8]
        # select internals: 3 -> 8 (load keys), 8 -> 9 (pass 1), 9 -> 12 (rest + pair),
        # 12 -> 13 (compaction), 13 -> 4 (tail)
        sel = {}
        for nm, a, b in (("sel.load", 3, 8), ("sel.pass1", 8, 9), ("sel.to_pair", 9, 12),
                         ("sel.compact", 12, 13), ("sel.tail", 13, 4)):
            ok = (t16[:, a] > 0) & (t16[:, b] > 0)
            if ok.any():
                d = (t16[ok, b] - t16[ok, a]) / 1000.0
                sel[nm] = round(float(np.median(d)), 2)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0  # us
        phases = np.diff(t, axis=1) / 1000.0
        ranks0 = t[:, 7] > 0
        row = {"total_us": float((t[ranks0, 7].max() - t0) / 1000.0),
               "start_spread_us": float(rel[:, 0].max())}
        for i, nm in enumerate(names):
            col = phases[:, i] if i < 6 else phases[ranks0, i]
            col = col[col >= 0]
            row[nm] = (round(float(np.median(col)), 2), round(float(col.max()), 2))
        row.update(sel)
        res.append(row)
for r in res[-args.layers:]:
    print(json.dumps(r))
