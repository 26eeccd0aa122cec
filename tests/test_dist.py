"""Multi-rank host logic on CPU: world_size 2 over gloo (the GPU box uses NCCL)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08417_b200 import dist as odist
from paper_2603_08417_b200 import workloads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # uneven shards: rank r holds r + 2 blocks tagged with its rank
        blocks = torch.full((rank + 2, 5), float(rank), dtype=torch.float64)
        parts = odist.gather_blocks(blocks, world)
        mx = odist.all_max(float(rank) * 10.0, "cpu")
        sm = odist.all_sum(1.5, "cpu")
        q.put((rank, [p.shape[0] for p in parts], [float(p[0, 0]) for p in parts], mx, sm))
    finally:
        dist.destroy_process_group()


def test_gather_and_reduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sizes, tags, mx, sm in out:
        assert sizes == [2, 3]
        assert tags == [0.0, 1.0]
        assert mx == 10.0 and sm == 3.0


def test_lpt_shard_partitions_and_balances():
    cfgs = [workloads.c4(seed=s, clients=n, variant="TC") for n in (10, 300, 3000, 10000) for s in range(1, 9)]
    for world in (1, 2, 4, 8):
        parts = [odist.shard(cfgs, r, world) for r in range(world)]
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(cfgs)))
        loads = [sum(odist.scenario_cost(cfgs[i]) for i in p) for p in parts]
        assert max(loads) <= 1.35 * (sum(loads) / world) + max(odist.scenario_cost(c) for c in cfgs)
