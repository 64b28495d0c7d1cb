#!/usr/bin/env python
"""Quest decode-attention benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the headline): Llama-2-7B attention shape -- 32 heads
(MHA), head_dim 128, page size 16 -- at 32K context with a 2048-token budget, batch 1 per
GPU, fp16 K/V/q with synthetic N(0, 1/d) data.  One *step* is one decode step through
NL = 32 independent layer caches (a model's worth of layers): for every layer, append the
new token's K/V (fused metadata update) -> estimate -> top-K -> sparse attend + LSE merge,
captured once in a CUDA graph.  `value` is microseconds per layer (step time / NL).  The
32 layer caches are 17 GB, so every layer's 67 MB working set comes from HBM, not L2
(each layer is revisited only after 31 other layers have streamed ~2 GB through L2).

N > 1 (`--gpus N`; bench.py re-launches itself under torch.distributed.run when WORLD_SIZE
is unset, and refuses a WORLD_SIZE that differs from N):
  --shard requests (default, weak scaling): each rank serves its own batch of requests, no
      collective on the attention path; `value` = max_time / (NL * N), the whole job's time
      per request-layer.
  --shard heads (strong scaling): the config's (request, KV head) units are
      partitioned over the ranks (shard.partition; GQA groups stay on one GPU) and the
      per-head outputs are all-gathered over NCCL inside the e2e timed region; `value` =
      max_time / NL.  Per-GPU kernel time is reported separately (per_gpu_us_per_layer).

--impl reference: the reference's own CPU implementation (oracle/_ref, compiled from
/root/reference) of the same path on the host cores: estimate_all -> select_top_k ->
sparse_attention for all 32 heads of a layer via questkv::parallel_for.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Quest attn decode latency us/layer @32K ctx, 2048 budget; achieved HBM GB/s"
UNIT = "us/layer"
HEADS, HEAD_DIM, PAGE, CTX, BUDGET, LAYERS = 32, 128, 16, 32768, 2048, 32


CONFIGS = {
    # name: (q heads, kv heads, context, budget, batch, layers, description)
    "cfg1": (32, 32, 8192, 1024, 1, 32, "cfg1: Llama-2-7B attention (32 heads MHA, d=128, page 16), "
             "8K context, budget 1024, batch 1"),
    "cfg2": (32, 32, 32768, 2048, 1, 32, "cfg2: Llama-2-7B attention shape (32 heads MHA, d=128, "
             "page 16), 32K context, token budget 2048, batch 1 per GPU"),
    "cfg3": (32, 32, 131072, 4096, 1, 8, "cfg3: LongChat-7B attention (32 heads MHA, d=128, page 16), "
             "128K context, budget 4096, batch 1 per GPU"),
    "cfg4": (32, 8, 65536, 2048, 32, 2, "cfg4: Llama-3-8B GQA attention (32 q / 8 kv heads, d=128, "
             "page 16), 64K context, budget 2048, batch 32 per GPU"),
    "cfg5": (32, 32, 32768, 2048, 8, 32, "cfg5: Llama-2-7B decode loop, 32 layers x (append + "
             "estimate + top-K + attend), 32K context, budget 2048, batch 8 per GPU"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--shard", choices=["requests", "heads"], default="requests")
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-native-e2e", action="store_true")
    ap.add_argument("--group-select", choices=["none", "max", "sum"], default="none",
                    help="GQA group-shared selection (SURVEY §8f item 3, opt-in variant): one "
                         "page set per KV head from the max/sum of its query heads' scores")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_if_needed(args):
    """--gpus N without a torchrun environment: run N ranks of this script under
    torch.distributed.run (one process per GPU) and exit with its status."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


class Workload:
    """The benchmarked configuration (shared by both arms, so their `config` dicts match)."""

    def __init__(self, args, world):
        HQ, HKV, ctx0, budget0, B, NL0, desc = CONFIGS[args.config]
        self.name, self.HQ, self.HKV, self.B, self.desc = args.config, HQ, HKV, B, desc
        self.ctx = args.ctx if args.ctx else ctx0
        self.budget = args.budget if args.budget else budget0
        self.NL = args.layers if args.layers else NL0
        self.world, self.shard = world, args.shard
        if args.shard == "heads":
            self.global_batch = B
            par = f"(request, KV head) units partitioned over {world} GPU(s), NCCL output gather"
            scaling = "strong"
        else:
            self.global_batch = B * world
            par = f"request-sharded x{world} (no collective)"
            scaling = "weak"
        self.scaling = scaling
        self.config = {
            "workload": desc + "; one step = one decode step (append + estimate + top-K + "
                        f"sparse attend) through {self.NL} independent layer caches",
            "name": self.name, "seq_len": self.ctx, "budget": self.budget, "q_heads": HQ,
            "kv_heads": HKV, "head_dim": HEAD_DIM, "page_size": PAGE,
            "layers_per_step": self.NL, "batch_per_gpu": B if args.shard == "requests" else None,
            "global_batch": self.global_batch, "parallelism": par,
            "selection": ("per query head (the reference's semantics)"
                          if args.group_select == "none" else
                          f"GQA group-shared, group score = {args.group_select} over the query "
                          "heads (opt-in variant, SURVEY §8f item 3)"),
            "l2": f"inputs larger than L2: {self.NL} rotating layer caches, each revisited after "
                  f"{self.NL - 1} other layers' traffic",
        }


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def page_lengths_tokens(L, page, pages):
    """Tokens held by `pages` (sorted page indices) of an L-token cache."""
    P = (L + page - 1) // page
    last = L - (P - 1) * page
    return sum(last if p == P - 1 else page for p in pages)


def algorithmic_bytes(lengths, heads, head_dim, page, budget, bpe=2, kv_heads=None,
                      union_tokens=None):
    """Reference byte accounting (metrics.cpp:90-108) for one layer step.
    Per (request, KV head): metadata 2*d*bpe per page + K/V 2*d*bpe per token of the UNION
    of the pages its query heads selected.  MHA: the union is the head's own selection,
    top-(K-1) full pages + the (possibly partial) newest page.  GQA: pass the measured
    union size per (request, KV head) in `union_tokens` (tokens)."""
    kv_heads = heads if kv_heads is None else kv_heads
    total = 0
    vec = head_dim * bpe
    for L in lengths:
        P = (L + page - 1) // page
        k = budget // page
        last_len = L - (P - 1) * page
        if union_tokens is not None:
            attended = union_tokens
        elif k >= P:
            attended = L
        else:
            attended = (k - 1) * page + last_len  # top-(K-1) full pages + the newest page
        total += kv_heads * (2 * vec * P + 2 * vec * attended)
    return total


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML in-process every
    ~2 ms (the timed region lasts tens of ms), nvidia-smi as a fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return float(sm), float(mx), int(rs)
        out = subprocess.run(
            ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
             "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        sm, mx = [float(x) for x in out.stdout.strip().split(",")[:2]]
        return sm, mx, 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.samples:  # region shorter than one sample period
            try:
                self.samples.append(self._sample())
            except Exception:
                pass

    def summary(self):
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        reasons = set()
        for s in self.samples:
            for name, bit in self.REASONS.items():
                if s[2] & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profiled_traffic():
    """dram bytes per launch of the decode step from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_layer_step")
    return None


def synthetic_layer(ctx):
    rng = np.random.default_rng(1)
    sd = 1.0 / np.sqrt(HEAD_DIM)
    keys = (rng.standard_normal((HEADS, ctx, HEAD_DIM), dtype=np.float32) * sd)
    keys = keys.astype(np.float16).astype(np.float32)
    vals = (rng.standard_normal((HEADS, ctx, HEAD_DIM), dtype=np.float32) * sd)
    vals = vals.astype(np.float16).astype(np.float32)
    q = (rng.standard_normal((HEADS, HEAD_DIM)) * sd).astype(np.float16).astype(np.float32)
    return keys, vals, q


def cpu_baseline_sample(ctx, budget, threads, warmup=3, reps=10):
    """The reference (oracle/_ref) on one full layer, 32 heads at `ctx` tokens, phases as
    cmd_bench (warmup 3, reps 10, cmd_bench.cpp:32-51), on all host threads and on one."""
    from oracle import REF_SO, Oracle, Reference  # checker / baseline only

    keys, vals, q = synthetic_layer(ctx)
    sample = (f"1 layer = {HEADS} heads x {ctx} tokens, d={HEAD_DIM}, S={PAGE}, budget {budget}; "
              "estimate_all->select_top_k->sparse_attention per head via questkv::parallel_for")
    if os.path.exists(REF_SO):
        layer = Reference().layer(keys, vals, PAGE)
        mean_ns, min_ns, _ = layer.step(q, budget, threads=threads, warmup=warmup, reps=reps)
        mean1, min1, _ = layer.step(q, budget, threads=1, warmup=1, reps=3)
        layer.close()
        return {"value": round(mean_ns / 1e3, 3), "unit": UNIT, "cores": threads,
                "kind": "reference", "min": round(min_ns / 1e3, 3),
                "one_thread": {"value": round(mean1 / 1e3, 3), "min": round(min1 / 1e3, 3),
                               "reps": 3},
                "cpu": cpu_model(),
                "sample": sample + f"; mean of {reps} reps after {warmup} warmup"}
    orc = Oracle()  # the C restatement, one head at a time (single thread)
    t0 = time.perf_counter()
    for h in range(HEADS):
        orc.quest_step(q[h], keys[h], vals[h], PAGE, budget)
    us = (time.perf_counter() - t0) * 1e6
    return {"value": round(us, 3), "unit": UNIT, "cores": 1, "kind": "port", "cpu": cpu_model(),
            "sample": sample + "; one pass"}


def run_reference(args):
    """The reference's own CPU path (oracle/_ref = the unmodified reference compiled from
    /root/reference) on the host cores: every step is one full layer of the workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    w = Workload(args, world)
    keys, vals, q = synthetic_layer(w.ctx)
    layer = Reference().layer(keys, vals, PAGE)
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    mean_ns, min_ns, _ = layer.step(q, w.budget, threads=threads, warmup=warmup, reps=steps)
    layer.close()
    us = mean_ns / 1e3
    line = {
        "metric": METRIC, "value": round(us, 3), "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": round(mean_ns * w.NL / 1e6, 4), "higher_is_better": False,
        "scaling": w.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1/d) fp16-representable",
        "config": w.config,
        "cpu_baseline": {"value": round(us, 3), "unit": UNIT, "cores": threads,
                         "kind": "reference", "cpu": cpu_model(),
                         "sample": f"every step = 1 full layer ({HEADS} heads x {w.ctx} tokens, "
                                   f"budget {w.budget}) on the host; ms_per_step = "
                                   f"{w.NL} layers x the per-layer mean"},
        "e2e": {"value": round(us, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "min_us_per_layer": round(min_ns / 1e3, 3),
    }
    print(json.dumps(line))


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2406_10774_b200 import QuestCache
    from paper_2406_10774_b200.shard import gather_outputs, partition

    rank, world, local = dist_env()
    # QK_BENCH_BACKEND=gloo: a code-path check of N > 1 on a one-GPU rig (ranks share the
    # device modulo the device count; the numbers are not scaling measurements).
    backend = os.environ.get("QK_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll_dev = dev if backend == "nccl" else torch.device("cpu")  # gloo: host tensors
    w = Workload(args, world)
    HQ, HKV, B, NL, ctx, budget = w.HQ, w.HKV, w.B, w.NL, w.ctx, w.budget
    G = HQ // HKV
    shards = partition(B, HKV, world) if args.shard == "heads" else None
    if shards is not None:
        lb, lkv = shards[rank].num_requests, shards[rank].num_kv_heads
    else:
        lb, lkv = B, HKV
    lq = lkv * G
    headroom = args.warmup + args.steps + args.e2e_steps + 8
    qc = QuestCache(HEAD_DIM, PAGE, num_layers=NL, max_batch=lb, num_q_heads=lq,
                    num_kv_heads=lkv, max_tokens=ctx + headroom, device=local)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    sd = 1.0 / HEAD_DIM ** 0.5
    n0 = ctx - 1  # the first timed step appends token ctx-1 -> a full `ctx` context
    for layer in range(NL):
        for bb in range(lb):
            k = (torch.randn((lkv, n0, HEAD_DIM), generator=g, device=dev) * sd).half()
            v = (torch.randn((lkv, n0, HEAD_DIM), generator=g, device=dev) * sd).half()
            qc.prefill(layer, bb, k, v)
            del k, v
    total_steps = args.warmup + args.steps
    q = (torch.randn((total_steps, NL, lb, lq, HEAD_DIM), generator=g, device=dev) * sd).half()
    kn = (torch.randn((total_steps, NL, lb, lkv, HEAD_DIM), generator=g, device=dev) * sd).half()
    vn = (torch.randn((total_steps, NL, lb, lkv, HEAD_DIM), generator=g, device=dev) * sd).half()
    qbuf, kbuf, vbuf = q[0].clone(), kn[0].clone(), vn[0].clone()
    out = torch.empty((NL, lb, lq, HEAD_DIM), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    stream = torch.cuda.Stream(device=dev)
    # Load every kernel of the step eagerly on a throwaway cache of the same geometry
    # (lazy module loading must not happen inside the capture).
    warm = QuestCache(HEAD_DIM, PAGE, num_layers=1, max_batch=lb, num_q_heads=lq,
                      num_kv_heads=lkv, max_tokens=ctx + headroom, device=local)
    for bb in range(lb):
        warm.prefill(0, bb, kn[0, 0, bb].view(lkv, 1, HEAD_DIM).contiguous(),
                     vn[0, 0, bb].view(lkv, 1, HEAD_DIM).contiguous())
    grouped = args.group_select != "none"

    def decode(cache, layer, qq, kk, vv, o=None, pages=None, counts=None):
        if grouped:
            return cache.decode_step_grouped(layer, qq, kk, vv, budget, args.group_select, out=o,
                                             pages=pages, counts=counts, stream=stream)
        return cache.decode_step(layer, qq, kk, vv, budget, out=o, pages=pages, counts=counts,
                                 stream=stream)

    decode(warm, 0, qbuf[0], kbuf[0], vbuf[0])
    stream.synchronize()
    warm.close()
    launches0 = qc.kernel_launches
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for layer in range(NL):
            decode(qc, layer, qbuf[layer], kbuf[layer], vbuf[layer], o=out[layer])
    kernels_per_step = qc.kernel_launches - launches0

    def step(i):
        qbuf.copy_(q[i], non_blocking=True)
        kbuf.copy_(kn[i], non_blocking=True)
        vbuf.copy_(vn[i], non_blocking=True)
        graph.replay()

    # the capture itself did not execute; the first replay appends token ctx-1
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # One event after every step too: the per-step distribution (median, p10,
    # p90); the headline is the first-to-last span.
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for j, i in enumerate(range(args.warmup, total_steps)):
                step(i)
                evs[j].record(stream)
            ev1.record(stream)
        stream.synchronize()
    step_us = [ev0.elapsed_time(evs[0]) * 1e3 / NL] + [
        evs[j - 1].elapsed_time(evs[j]) * 1e3 / NL for j in range(1, args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    own_ms = ev0.elapsed_time(ev1)
    elapsed_ms = own_ms
    qc.sync_lengths(stream=stream)  # graph replays advanced only the device lengths
    qc.check_status(stream=stream)
    if world > 1:
        t = torch.tensor([elapsed_ms], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    us_per_layer = ms_per_step * 1e3 / NL
    value = us_per_layer / world if args.shard == "requests" else us_per_layer

    # Algorithmic bytes of the timed steps on this GPU (reference accounting).
    # GQA: the K/V term counts the union of the pages a KV head's query heads selected,
    # measured on the final state (one extra, untimed, non-appending step per layer).
    union = None
    if G > 1 and not grouped:  # grouped: one shared page set per KV head (the MHA formula)
        pages = torch.full((lb, lq, max(1, budget // PAGE)), -1, dtype=torch.int32, device=dev)
        counts = torch.zeros((lb, lq), dtype=torch.int32, device=dev)
        L_now = qc.token_count(0, 0)
        tot, n = 0, 0
        scratch = torch.empty((lb, lq, HEAD_DIM), dtype=torch.float32, device=dev)
        for layer in range(NL):
            qc.decode_step(layer, q[total_steps - 1, layer], None, None, budget, out=scratch,
                           pages=pages, counts=counts, stream=stream)
            stream.synchronize()
            pc, cc = pages.cpu().numpy(), counts.cpu().numpy()
            for bb in range(lb):
                for h in range(lkv):
                    sel = set()
                    for gq in range(G):
                        sel.update(pc[bb, h * G + gq, :cc[bb, h * G + gq]].tolist())
                    tot += page_lengths_tokens(L_now, PAGE, sorted(sel))
                    n += 1
        union = tot / max(n, 1)
    bytes_total = 0
    for i in range(args.warmup, total_steps):
        L = ctx + i  # tokens after this step's append (first replay -> ctx)
        bytes_total += lb * algorithmic_bytes([L], lq, HEAD_DIM, PAGE, budget, kv_heads=lkv,
                                              union_tokens=union)
    bytes_per_layer = bytes_total / args.steps
    own_us_per_layer = own_ms * 1e3 / (args.steps * NL)
    achieved_gbs = bytes_per_layer / (us_per_layer * 1e-6) / 1e9
    peak, peak_src = measured_peaks()
    traffic = profiled_traffic() if args.config == "cfg2" and world == 1 else None

    # Per-kernel breakdown (one layer, eager, CUDA events) on the current state.
    breakdown = (kernel_breakdown(qc, q[0], NL, budget, stream)
                 if rank == 0 and lb == 1 and not grouped else {})

    # End to end through the public API with host buffers: H2D of q/k/v and D2H of the
    # fp32 output inside the timed region.
    qh = torch.empty((NL, lb, lq, HEAD_DIM), dtype=torch.float16).pin_memory()
    kh = torch.empty((NL, lb, lkv, HEAD_DIM), dtype=torch.float16).pin_memory()
    vh = torch.empty_like(kh).pin_memory()
    qh.copy_(q[0].cpu())
    kh.copy_(kn[0].cpu())
    vh.copy_(vn[0].cpu())
    e2e_steps = max(1, args.e2e_steps)
    if shards is None and not grouped:
        # qk_decode_step_host: the kernel reads and writes the pinned, mapped host arrays
        # (questkv.host_empty = qk_host_alloc) in place over PCIe.
        from paper_2406_10774_b200.questkv import host_empty

        qn = host_empty(tuple(qh.shape), np.float16)
        kn_ = host_empty(tuple(kh.shape), np.float16)
        vn_ = host_empty(tuple(vh.shape), np.float16)
        on = host_empty((NL, lb, lq, HEAD_DIM), np.float32)
        qn[...], kn_[...], vn_[...] = qh.numpy(), kh.numpy(), vh.numpy()
        # Warm every layer once (each layer's host-step graph is instantiated on first use).
        for layer in range(NL):
            qc.decode_step_host(layer, qn[layer], kn_[layer], vn_[layer], budget, out=on[layer],
                                stream=stream)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            for layer in range(NL):
                qc.decode_step_host(layer, qn[layer], kn_[layer], vn_[layer], budget,
                                    out=on[layer], stream=stream)
        e2e_s = time.perf_counter() - t0
        e2e_path = "Python QuestCache.decode_step_host -> qk_decode_step_host (C ABI) per layer"
        d2h = lq * lb * HEAD_DIM * 4 * NL
    else:
        # Sharded: H2D of this rank's q/k/v, the decode step, NCCL all-gather of every
        # rank's per-head outputs, D2H of the full output -- per layer.
        oh = torch.empty((NL, B, HQ, HEAD_DIM), dtype=torch.float32).pin_memory()
        dq, dk, dv = torch.empty_like(qbuf[0]), torch.empty_like(kbuf[0]), torch.empty_like(vbuf[0])
        lout = torch.empty((lb, lq, HEAD_DIM), dtype=torch.float32, device=dev)

        def e2e_layer(layer):
            with torch.cuda.stream(stream):  # the collective is ordered on `stream` too
                dq.copy_(qh[layer], non_blocking=True)
                dk.copy_(kh[layer], non_blocking=True)
                dv.copy_(vh[layer], non_blocking=True)
                decode(qc, layer, dq, dk, dv, o=lout)
                full = (gather_outputs(lout, shards, B, HKV, G) if world > 1 and shards
                        else lout)
                oh[layer].copy_(full, non_blocking=True)
            stream.synchronize()

        torch.cuda.synchronize()
        e2e_layer(0)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            for layer in range(NL):
                e2e_layer(layer)
        e2e_s = time.perf_counter() - t0
        e2e_path = ("Python QuestCache.decode_step on this rank's units + NCCL all-gather of the "
                    "per-head outputs (shard.gather_outputs) per layer" if shards is not None else
                    "Python QuestCache.decode_step_grouped per layer: H2D of q/k/v from pinned "
                    "host memory, the step, D2H of the fp32 output")
        d2h = HQ * B * HEAD_DIM * 4 * NL
    if world > 1:
        t = torch.tensor([e2e_s], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_us = e2e_s * 1e6 / (e2e_steps * NL)
    if args.shard == "requests":
        e2e_us /= world
    # The native host API (C++ questkv_b200::DeviceCache::decode_step_host), compiled here
    # against the in-tree library; it replaces the Python number when it builds and runs.
    e2e_pageable = None
    if world == 1 and not args.no_native_e2e and args.config == "cfg2" and not grouped:
        native = native_e2e(ctx, budget)
        if native is not None:
            e2e_us, e2e_pageable = native
            e2e_path = ("C++ questkv_b200::DeviceCache::decode_step_host (include/questkv_b200.hpp) "
                        "per layer, 8 layers x 20 steps; q/k/v in and fp32 out in pinned host "
                        "memory (qk_host_alloc), read and written by the kernel over PCIe")
    h2d = (lq + 2 * lkv) * lb * HEAD_DIM * 2 * NL  # q, k, v fp16 per layer

    per_gpu = torch.tensor([own_us_per_layer], device=coll_dev)
    if world > 1:
        gathered = [torch.zeros_like(per_gpu) for _ in range(world)]
        dist.all_gather(gathered, per_gpu)
        per_gpu_list = [round(float(x.item()), 3) for x in gathered]
    else:
        per_gpu_list = [round(own_us_per_layer, 3)]
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1 and args.config == "cfg2":
        cpu = cpu_baseline_sample(ctx, budget, os.cpu_count() or 1)
    bytes_model = ("reference accounting metrics.cpp:90-108 / SURVEY §8d: per (request, KV head) "
                   "2*d*2B per page of metadata + 2*d*2B per token of the union of its query "
                   "heads' selected pages")
    if union is not None:
        bytes_model += f" (GQA union measured: {union:.1f} tokens per (request, KV head))"
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": False,
        "scaling": w.scaling,
        "vs_baseline": None,
        "dtype": "fp16 storage, fp64 estimate, fp32 attention accumulate",
        "data": "synthetic N(0,1/d) fp16 K/V/q (random-init, generated on device)",
        "config": w.config,
        "latency_us_per_layer": round(us_per_layer, 3),
        "per_gpu_us_per_layer": per_gpu_list,
        "tokens_per_s": round(w.global_batch * 1e6 / (us_per_layer * NL), 1),
        "achieved_hbm_gbs": round(achieved_gbs, 1),
        "roofline": {
            "bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved_gbs / peak, 4),
            "frac_at_8tbs": round(achieved_gbs / 8000.0, 4),  # report both fractions
            "traffic": traffic,
            "frac_physical": (round(traffic / (us_per_layer * 1e-6) / 1e9 / peak, 4)
                              if traffic else None),
            "kernel": ("decode_fused_kernel (one launch = append+estimate+top-K+attend of a layer)"
                       if not grouped else
                       "append_kernel + estimate_kernel + group_topk_kernel + "
                       "grouped_attend_kernel (mma.sync) per layer"),
            "timing": "per-layer time of the CUDA-graph replay (launch gaps included), CUDA "
                      "events on the launching stream, max over ranks",
            "bytes_per_launch": int(bytes_per_layer),
            "bytes_model": bytes_model,
            "peak_source": peak_src,
        },
        "step_distribution_us_per_layer": percentiles(step_us),
        "kernel_breakdown_us": breakdown,
        "gpu_launches": int(kernels_per_step * args.steps),
        "clocks": clocks.summary(),
        "e2e": {"value": round(e2e_us, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "path": e2e_path,
                **({"pageable_host_buffers": round(e2e_pageable, 3)} if e2e_pageable else {})},
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def percentiles(xs):
    """p10 / median / p90 of per-step µs per layer (nearest rank)."""
    ys = sorted(xs)
    pick = lambda f: round(ys[min(len(ys) - 1, int(f * (len(ys) - 1) + 0.5))], 3)  # noqa: E731
    return {"p10": pick(0.1), "median": pick(0.5), "p90": pick(0.9), "n": len(ys)}


def native_e2e(ctx, budget):
    """(pinned, pageable) e2e µs/layer through the C++ host API (tools/e2e_bench.cpp), or
    None."""
    exe = os.path.join(ROOT, "build", "e2e_bench")
    src = os.path.join(ROOT, "tools", "e2e_bench.cpp")
    lib_dir = os.path.join(ROOT, "paper_2406_10774_b200")
    try:
        os.makedirs(os.path.dirname(exe), exist_ok=True)
        if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
            subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src,
                            "-o", exe, "-L", lib_dir, "-lquestkv_b200", f"-Wl,-rpath,{lib_dir}"],
                           check=True, capture_output=True, timeout=120)
        out = subprocess.run([exe, str(ctx), str(budget), "8", "20", "3"], capture_output=True,
                             text=True, timeout=300)
        line = json.loads(out.stdout.strip().splitlines()[-1])
        return float(line["e2e_us_per_layer"]), float(line["e2e_pageable_us_per_layer"])
    except Exception:
        return None


def kernel_breakdown(qc, q0, NL, budget, stream):
    """Device time per layer of the separate (unfused) ops on the current caches: each op's
    launches over n layers captured in a CUDA graph and replayed (so host dispatch is not
    timed), CUDA events on the stream, outputs preallocated, one untimed replay first."""
    import torch

    n = min(8, NL)
    dev = qc.device
    H, P = qc.num_q_heads, qc.max_pages
    K = max(1, min(budget // qc.page_size, P))
    scores = [torch.zeros((1, H, P), dtype=torch.float64, device=dev) for _ in range(n)]
    pages = [torch.zeros((1, H, K), dtype=torch.int32, device=dev) for _ in range(n)]
    counts = [torch.zeros((1, H), dtype=torch.int32, device=dev) for _ in range(n)]

    def run(name, layer):
        if name == "estimate":
            qc.estimate(layer, q0[layer], scores=scores[layer], stream=stream)
        elif name == "select_topk":
            qc.select_topk(layer, scores[layer], budget, pages=pages[layer], counts=counts[layer],
                           stream=stream)
        elif name == "sparse_attend":
            qc.sparse_attend(layer, q0[layer], pages[layer], counts[layer], stream=stream)
        else:
            qc.dense_attend(layer, q0[layer], stream=stream)

    res = {}
    names = ("estimate", "select_topk", "sparse_attend", "dense_attend")
    with torch.cuda.stream(stream):
        for name in names:  # eager first: module load, real selections for the attend graphs
            for layer in range(n):
                run(name, layer)
        stream.synchronize()
        for name in names:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for layer in range(n):
                    run(name, layer)
            g.replay()
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(4):
                g.replay()
            e1.record(stream)
            stream.synchronize()
            res[name] = round(e0.elapsed_time(e1) * 1e3 / (4 * n), 2)
    res["note"] = ("unfused ops (the reference-style separate calls), each op over 8 layers "
                   "captured in a CUDA graph (kernel + in-graph launch gap per layer), same caches; "
                   "the bench step uses the fused kernel")
    return res


def main():
    args = parse()
    relaunch_if_needed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
