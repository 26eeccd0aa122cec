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


def _stub_rows(cfgs, device):
    """Stand-in for the GPU runner: one deterministic row per config
    [status, clients, workers, seed, cache bytes, <8 payload words>]."""
    import numpy as np
    rows = np.zeros((len(cfgs), 13), dtype=np.int64)
    for k, c in enumerate(cfgs):
        rows[k, :5] = (0, c.clients, c.workers, c.seed, c.cache_capacity_bytes)
        rows[k, 5:] = np.arange(8) + 1000 * c.seed + c.clients
    return rows


def _sharded_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfgs = workloads.c5_sweep(seeds=range(1, 7))             # 6 seeds x 16 scenarios
        mine = odist.shard(cfgs, rank, world)
        out = odist.run_sharded(cfgs, runner=_stub_rows)
        q.put((rank, mine, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_run_sharded_gathers_every_scenario_in_order_world2():
    """Two gloo ranks: seed-grouped shards, the all-gather of the result rows, and
    the reorder into config order (the GPU runner replaced by a CPU stub)."""
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=180) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfgs = workloads.c5_sweep(seeds=range(1, 7))
    want = np.concatenate([np.arange(len(cfgs))[:, None], _stub_rows(cfgs, None)], axis=1)
    (_, mine0, out0), (_, mine1, out1) = got
    assert sorted(mine0 + mine1) == list(range(len(cfgs)))
    seeds0 = {cfgs[i].seed for i in mine0}
    assert seeds0.isdisjoint({cfgs[i].seed for i in mine1})    # whole seed groups per rank
    assert np.array_equal(out0, want) and np.array_equal(out1, want)


def test_shard_by_seed_falls_back_to_scenarios():
    cfgs = workloads.c3_sweep(seeds=range(1, 2))                 # one seed, 11 points
    parts = [odist.shard(cfgs, r, 4) for r in range(4)]
    assert all(parts) and sorted(i for p in parts for i in p) == list(range(11))
