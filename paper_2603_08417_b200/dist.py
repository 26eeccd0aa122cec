"""Multi-GPU sweeps: one process per GPU, scenarios sharded, one gather at the end.

Scenarios are independent closed simulations (orchestrator.py:327-370), so a
sweep shards across ranks with no data-path communication.  The only
collective is a gather of the fixed-size per-scenario QoE / counter blocks
after the sweep, issued through torch.distributed: NCCL over
NVLink/NVSwitch on the GPU box, gloo in the CPU tests.
"""

from __future__ import annotations

import heapq

import numpy as np
import torch
import torch.distributed as dist

RERUN_BITS = 0x2 | 0x8 | 0x20 | 0x80                   # OTF_S_EPS_OVERFLOW | TIE | UNFIT | LIST_OVERFLOW

__all__ = ["scenario_cost", "shard", "gather_blocks", "all_max", "all_sum", "run_sharded"]


def scenario_cost(cfg) -> float:
    """Work estimate: client-seconds per segment (requests scale with it)."""
    segdur = min((e.get("segment_duration_s", cfg.segment_duration_s) for e in cfg.sequences),
                 default=cfg.segment_duration_s) if cfg.sequences else cfg.segment_duration_s
    return cfg.clients * cfg.horizon_s / max(segdur, 1e-3)


def _lpt(costs, world: int) -> list[int]:
    """Longest-processing-time-first owner of each item (deterministic ties)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [(0.0, r) for r in range(world)]
    heapq.heapify(load)
    owner = [0] * len(costs)
    for i in order:
        l, r = heapq.heappop(load)
        owner[i] = r
        heapq.heappush(load, (l + costs[i], r))
    return owner


def shard(configs, rank: int, world: int, by_seed: bool = True) -> list[int]:
    """The config indices rank `rank` runs.

    Scenarios that share a seed share their input streams (traces, arrivals,
    worker noise, segment sizes: orchestrator.py:241-268, content.py:204-218),
    which the input builder generates once per batch.  So whole seed groups are
    assigned, LPT on their summed cost, as long as there
    are at least two groups per rank; with fewer groups the scenarios themselves
    are spread LPT (a rank may then rebuild a seed's streams)."""
    seeds = sorted({c.seed for c in configs})
    if by_seed and len(seeds) >= 2 * world:
        gcost = {s: 0.0 for s in seeds}
        for c in configs:
            gcost[c.seed] += scenario_cost(c)
        gowner = dict(zip(seeds, _lpt([gcost[s] for s in seeds], world)))
        return [i for i, c in enumerate(configs) if gowner[c.seed] == rank]
    owner = _lpt([scenario_cost(c) for c in configs], world)
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


def _gpu_rows(cfgs, device):
    """Run cfgs in histogram mode on this rank's GPU: rows of [status, counts(4), otf_qoe...]."""
    from . import _lib, engine, inputs
    inp = inputs.build_inputs(cfgs, engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM)
    db = engine.DeviceBatch(inp, device)
    db.launch()
    br = db.fetch()
    rows = np.concatenate([br.status.astype(np.int64)[:, None], br.counts, br.qoe], axis=1)
    redo = [k for k in range(len(cfgs)) if br.status[k] & RERUN_BITS]
    if redo:
        for k, res in zip(redo, engine.run_batch([cfgs[k] for k in redo], mode="histograms", device=db.device)):
            rows[k, 0] = res.status
            rows[k, 1:5] = res.counts
            rows[k, 5:] = res.qoe_row
    return rows


def run_sharded(configs, device=None, runner=None):
    """Strong-scaling sweep: this rank runs its LPT shard in histogram mode and
    every rank receives all per-scenario blocks, in config order.  A block row is
    [config index, status, requests, sessions, segments, jobs, otf_qoe...].

    Scenarios the windowed engine flags (a tie, outside its limits, noise table
    too short) are re-run through engine.run_batch, which routes them to the
    exact engine / a longer noise table, so every gathered block is final."""
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
    mine = shard(configs, rank, world)
    rows = (runner or _gpu_rows)([configs[i] for i in mine], device)   # runner: test hook (CPU stub)
    rows = np.concatenate([np.asarray(mine, dtype=np.int64)[:, None], rows.astype(np.int64)], axis=1)
    if device is not None:
        dev = device
    elif runner is None and torch.cuda.is_available():
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = "cpu"
    blocks = torch.from_numpy(rows).to(dev)
    parts = gather_blocks(blocks, world)
    allb = torch.cat(parts, dim=0).cpu()
    order = torch.argsort(allb[:, 0])
    return allb[order]
