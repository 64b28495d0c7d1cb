"""ShardedDecoder (shard.py) on the GPU: world size 2, both ranks on cuda:0 over gloo (the
one-GPU rig; NCCL over NVLink runs the same code on a multi-GPU box).  Each rank owns a
rectangle of (request, KV head) units, runs the fused decode step on them, and
the gathered output must equal a single-process cache holding every unit (pages bitwise per
unit, outputs within the fp32 tolerance: the cluster split differs with the unit count) and
the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
D, S = 128, 16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(B, Hq, Hkv, L, steps):
    rng = np.random.default_rng(B * 100 + Hq + Hkv)
    sd = 1 / np.sqrt(D)
    f = lambda *sh: rng.standard_normal(sh).astype(np.float32) * sd  # noqa: E731
    keys, vals = f(B, Hkv, L, D).astype(np.float16), f(B, Hkv, L, D).astype(np.float16)
    qs = [f(B, Hq, D).astype(np.float16) for _ in range(steps)]
    ks = [f(B, Hkv, D).astype(np.float16) for _ in range(steps)]
    vs = [f(B, Hkv, D).astype(np.float16) for _ in range(steps)]
    return keys, vals, qs, ks, vs


def _worker(rank, world, port, B, Hq, Hkv, L, budget, steps, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2406_10774_b200.shard import ShardedDecoder

        torch.cuda.set_device(0)
        keys, vals, qs, ks, vs = _data(B, Hq, Hkv, L, steps)
        t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        dec = ShardedDecoder(D, S, num_layers=1, batch=B, num_q_heads=Hq, num_kv_heads=Hkv,
                             max_tokens=L + steps + 4, device=0)
        for b in range(B):
            dec.prefill(0, b, t(keys[b]), t(vals[b]))
        outs = []
        for i in range(steps):
            out = dec.decode_step(0, dec.local_q(t(qs[i])), dec.local_kv(t(ks[i])),
                                  dec.local_kv(t(vs[i])), budget)
            outs.append(out.cpu().numpy())
        if rank == 0:
            np.save(path, np.stack(outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,Hq,Hkv,L,budget", [
    (1, 8, 8, 5000, 512),    # cfg3-style: one request, heads split over the ranks
    (4, 8, 2, 3000, 256),    # cfg4-style GQA: requests split, groups kept whole
    (2, 4, 4, 40000, 16384),  # unfused path (K > 512 pages) per rank
])
def test_sharded_decoder_two_ranks(tmp_path, oracle_c, B, Hq, Hkv, L, budget):
    from paper_2406_10774_b200 import QuestCache

    steps = 3
    path = str(tmp_path / "out.npy")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, Hq, Hkv, L, budget, steps, path))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    got = np.load(path)

    keys, vals, qs, ks, vs = _data(B, Hq, Hkv, L, steps)
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    qc = QuestCache(D, S, max_batch=B, num_q_heads=Hq, num_kv_heads=Hkv, max_tokens=L + steps + 4)
    for b in range(B):
        qc.prefill(0, b, t(keys[b]), t(vals[b]))
    G = Hq // Hkv
    kf = [[keys[b, h].astype(np.float32) for h in range(Hkv)] for b in range(B)]
    vf = [[vals[b, h].astype(np.float32) for h in range(Hkv)] for b in range(B)]
    for i in range(steps):
        want = qc.decode_step(0, t(qs[i]), t(ks[i]), t(vs[i]), budget).cpu().numpy()
        rel = np.linalg.norm(got[i] - want) / np.linalg.norm(want)
        assert rel <= 1e-5, (i, rel)
        for b in range(B):
            for h in range(Hkv):
                kf[b][h] = np.concatenate([kf[b][h], ks[i][b, h].astype(np.float32)[None]])
                vf[b][h] = np.concatenate([vf[b][h], vs[i][b, h].astype(np.float32)[None]])
        for b, hq in [(0, 0), (B - 1, Hq - 1)]:
            _, _, o = oracle_c.quest_step(qs[i][b, hq].astype(np.float32), kf[b][hq // G],
                                          vf[b][hq // G], S, budget)
            err = np.linalg.norm(got[i][b, hq] - o) / np.linalg.norm(o)
            assert err <= 1e-5, (i, b, hq, err)
