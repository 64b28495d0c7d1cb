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
ap.add_argument("--graph-steps", type=int, default=1, help="graph mode: replays before the measured one")
ap.add_argument("--fresh-q", action="store_true", help="graph mode: new random q/k/v per replay (as bench.py)")
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
SLOTS = 32
n = args.batch * Hkv * 16 * SLOTS      # one layer's record
buf = np.zeros(n * args.layers, dtype=np.uint64)
lib = _lib.load()
names = {0: "entry", 1: "dep_wait", 2: "prologue", 21: "pre_cwait", 22: "cluster_wait", 3: "loads_issued", 5: "w0_computed", 6: "partials_synced", 7: "pushed", 4: "est_loop_end", 8: "estimate_end", 9: "barrier1", 10: "keys_pulled",
         11: "sel_pass0", 26: "pair_gathered", 27: "pair_sync1", 28: "pair_ranked", 29: "pair_sync2", 12: "sel_pass1", 13: "sel_pass2", 14: "sel_pair", 15: "sel_compact",
         29: "x29", 30: "x30", 16: "select_end", 31: "x31", 17: "attend_end", 18: "partials", 19: "barrier2", 20: "merged"}
for _ in range(50):  # clocks up
    for layer in range(args.layers):
        qc.decode_step(layer, q, None, None, args.budget, out=out)
torch.cuda.synchronize()
lib.qk_debug_probe(qc._h, buf.ctypes.data, buf.size, None)
res = []
for rep in range(args.reps):
    for layer in range(args.layers):
        qc.decode_step(layer, q, kn, kn, args.budget, out=out)
        torch.cuda.synchronize()
        lib.qk_debug_probe(qc._h, buf.ctypes.data, buf.size, None)
        t = buf[layer * n:(layer + 1) * n].reshape(-1, SLOTS).astype(np.int64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        fb = int(t[:, 23].sum())
        t[:, 23] = 0
        cyc = (t[:, 25] - t[:, 24]).astype(np.float64)
        ns = (t[:, 19] - t[:, 0]).astype(np.float64)
        mhz = float(np.median(cyc / ns * 1000.0))
        t[:, 24] = 0
        t[:, 25] = 0
        row = {"ctas": int(len(t)), "fallback_pages": fb, "sm_mhz": round(mhz),
               "total_us": round(float((t.max() - t0) / 1000.0), 3)}
        for k, nm in names.items():
            col = t[:, k]
            ok = col > 0
            if ok.any():
                rel = (col[ok] - t0) / 1000.0
                row[nm] = (round(float(np.median(rel)), 2), round(float(rel.max()), 2))
        res.append(row)
for r in res[-args.layers:]:
    print(json.dumps(r))
if os.environ.get("QK_PROBE_RANKS"):
    # Per cluster rank (CTA index % cluster size): median stamp of the last layer's CTAs.
    t = buf[(args.layers - 1) * n:args.layers * n].reshape(-1, SLOTS).astype(np.int64)
    idx = np.nonzero(t[:, 0] > 0)[0]
    t = t[idx]
    t0 = t[:, 0].min()
    C = int(os.environ.get("QK_PROBE_RANKS"))
    for k in (3, 5, 6, 7, 8, 9, 10, 16, 17, 18):
        col = (t[:, k] - t0) / 1000.0
        print(json.dumps({"stamp": names.get(k, k), **{f"rank{r}": round(float(np.median(col[idx % C == r])), 2)
                                                        for r in range(C)},
                          "max_rank": int(np.argmax([np.max(col[idx % C == r]) for r in range(C)]))}))

# ---- graph mode: inter-kernel gaps of a CUDA graph of every layer (as bench.py runs) ----
if os.environ.get("QK_PROBE_GRAPH"):
    s = torch.cuda.Stream()
    qb, kb = q.clone(), kn.clone()
    g2 = torch.cuda.CUDAGraph()
    qc.decode_step(0, qb, kb, kb, args.budget, out=out, stream=s)  # warm
    s.synchronize()
    with torch.cuda.graph(g2, stream=s):
        for layer in range(args.layers):
            qc.decode_step(layer, qb, kb, kb, args.budget, out=out, stream=s)
    for _ in range(3):
        g2.replay()
    s.synchronize()
    qs = (torch.randn((args.graph_steps + 1, args.batch, H, D), generator=g, device=dev) / D ** 0.5).half()
    ks = (torch.randn((args.graph_steps + 1, args.batch, Hkv, D), generator=g, device=dev) / D ** 0.5).half()
    t_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        for i in range(args.graph_steps):
            if args.fresh_q:
                qb.copy_(qs[i], non_blocking=True)
                kb.copy_(ks[i], non_blocking=True)
            if i == args.graph_steps - 1:
                s.synchronize()
                lib.qk_debug_probe(qc._h, buf.ctypes.data, buf.size, None)  # clear
                t_ev[0].record(s)
            g2.replay()
        t_ev[1].record(s)
    s.synchronize()
    print(json.dumps({"last_replay_event_us_per_layer": round(t_ev[0].elapsed_time(t_ev[1]) * 1e3 / args.layers, 2)}))
    big = np.zeros(n * args.layers, dtype=np.uint64)
    lib.qk_debug_probe(qc._h, big.ctypes.data, big.size, None)
    per = big.reshape(args.layers, -1, SLOTS).astype(np.int64)
    prev_end = None
    for layer in range(args.layers):
        t = per[layer]
        t = t[t[:, 0] > 0]
        start = t[:, 0].min()
        ends = t[:, 1:23].max(axis=1)
        end = ends.max()
        gap = (start - prev_end) / 1000.0 if prev_end is not None else 0.0
        print(json.dumps({"layer": layer, "kernel_us": round((end - start) / 1000.0, 2),
                          "gap_from_prev_us": round(gap, 2),
                          "entry_spread_us": round((t[:, 0].max() - start) / 1000.0, 2)}))
        prev_end = end
    # Phase medians of the last graph layer, relative to its median dep_wait stamp (early
    # PDL-placed CTAs make the minimum entry meaningless).
    t = per[args.layers - 1]
    t = t[t[:, 0] > 0]
    ref = np.median(t[:, 1])
    row = {}
    for k, nm in names.items():
        col = t[:, k]
        ok = col > 0
        if ok.any():
            rel = (col[ok] - ref) / 1000.0
            row[nm] = (round(float(np.median(rel)), 2), round(float(rel.max()), 2))
    print(json.dumps({"graph_layer_phases": row}))
