"""Multi-GPU sharding logic on CPU: the (request, KV head) partition of SURVEY.md §8e and
the output all-gather, with world_size 2 over gloo (the NCCL path runs the same code)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_10774_b200.shard import gather_outputs, partition


@pytest.mark.parametrize("batch,heads,world", [
    (1, 32, 1), (1, 32, 2), (1, 32, 8),   # cfg3: heads of one request split over GPUs
    (32, 8, 8), (8, 32, 8), (8, 32, 2),   # cfg4 / cfg5: requests split first
    (2, 8, 4),                            # 2 ranks per request
])
def test_partition_covers_every_unit_once(batch, heads, world):
    shards = partition(batch, heads, world)
    assert [s.rank for s in shards] == list(range(world))
    units = [u for s in shards for u in s.units()]
    assert sorted(units) == [(b, h) for b in range(batch) for h in range(heads)]
    sizes = {len(s.units()) for s in shards}
    assert len(sizes) == 1  # balanced: equal rectangles


def test_partition_rejects_uneven_splits():
    with pytest.raises(ValueError):
        partition(3, 5, 2)
    with pytest.raises(ValueError):
        partition(0, 8, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, heads, G, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shards = partition(batch, heads, world)
        s = shards[rank]
        # Each rank's "output" for its units: a deterministic function of (b, q head, c).
        local = torch.empty((s.num_requests, s.num_kv_heads * G, d))
        for i, b in enumerate(range(s.b0, s.b1)):
            for j, hq in enumerate(range(s.h0 * G, s.h1 * G)):
                local[i, j] = torch.arange(d) + 1000.0 * b + 10.0 * hq
        full = gather_outputs(local, shards, batch, heads, G)
        want = torch.empty((batch, heads * G, d))
        for b in range(batch):
            for hq in range(heads * G):
                want[b, hq] = torch.arange(d) + 1000.0 * b + 10.0 * hq
        q.put((rank, bool(torch.equal(full, want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch,heads,G", [(2, 4, 1), (1, 8, 4), (4, 2, 2)])
def test_gather_outputs_world_size_2_gloo(batch, heads, G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, heads, G, 16, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(results) == [(0, True), (1, True)]
