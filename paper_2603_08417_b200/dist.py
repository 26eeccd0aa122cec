"""Multi-GPU sweeps: one process per GPU, scenarios sharded, one gather at the end.

Scenarios are independent closed simulations (orchestrator.py:327-370), so a
sweep shards across ranks with no data-path communication.  The only
collective is a gather of the fixed-size per-scenario QoE / counter blocks
after the sweep, issued through torch.distributed: NCCL over
NVLink/NVSwitch on the GPU box, gloo in the CPU tests.
"""

from __future__ import annotations

import heapq

import torch
import torch.distributed as dist

__all__ = ["scenario_cost", "shard", "gather_blocks", "all_max", "all_sum", "run_sharded"]


def scenario_cost(cfg) -> float:
    """Work estimate: client-seconds per segment (requests scale with it)."""
    segdur = min((e.get("segment_duration_s", cfg.segment_duration_s) for e in cfg.sequences),
                 default=cfg.segment_duration_s) if cfg.sequences else cfg.segment_duration_s
    return cfg.clients * cfg.horizon_s / max(segdur, 1e-3)


def shard(configs, rank: int, world: int) -> list[int]:
    """Longest-processing-time-first assignment of scenarios to ranks (deterministic)."""
    order = sorted(range(len(configs)), key=lambda i: (-scenario_cost(configs[i]), i))
    load = [(0.0, r) for r in range(world)]
    heapq.heapify(load)
    owner = [0] * len(configs)
    for i in order:
        l, r = heapq.heappop(load)
        owner[i] = r
        heapq.heappush(load, (l + scenario_cost(configs[i]), r))
    return [i for i in range(len(configs)) if owner[i] == rank]


def gather_blocks(blocks: torch.Tensor, world: int) -> list[torch.Tensor]:
    """All-gather equally shaped per-rank blocks (pad to the largest shard first)."""
    if world == 1:
        return [blocks]
    n = torch.tensor([blocks.shape[0]], dtype=torch.int64, device=blocks.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    m = int(max(int(x.item()) for x in sizes))
    pad = torch.zeros((m,) + tuple(blocks.shape[1:]), dtype=blocks.dtype, device=blocks.device)
    pad[:blocks.shape[0]] = blocks
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad)
    return [o[:int(s.item())] for o, s in zip(out, sizes)]


def all_max(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def run_sharded(configs, device=None):
    """Strong-scaling sweep: this rank runs its LPT shard in histogram mode and
    every rank receives all per-scenario QoE blocks (in config order)."""
    from . import _lib, engine, inputs
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
    mine = shard(configs, rank, world)
    inp = inputs.build_inputs([configs[i] for i in mine], engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM)
    db = engine.DeviceBatch(inp, device)
    db.launch()
    torch.cuda.synchronize(db.device)
    idx = torch.tensor(mine, dtype=torch.int64, device=db.device).unsqueeze(1)
    blocks = torch.cat([idx, db.counts, db.qoe], dim=1)
    parts = gather_blocks(blocks, world)
    allb = torch.cat(parts, dim=0).cpu()
    order = torch.argsort(allb[:, 0])
    return allb[order]
