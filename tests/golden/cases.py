"""Golden-fixture configurations (shared by make_golden.py and the tests).

Small enough that the reference finishes each in seconds, chosen to cover the
reference's behaviours: every variant, coalescing, speculation skip reasons,
LRU eviction and rejection, cut-off sessions, zero noise (worker timer ties),
zero latency, partial final segments, per-rank rho, Zipf popularity.
"""

from __future__ import annotations

import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_2603_08417_b200.config import ClientConfig, ExperimentConfig, NetemConfig  # noqa: E402
from paper_2603_08417_b200 import workloads as W  # noqa: E402


def golden_cases():
    out = []
    # config 1 (BASELINE configs[0]) at three seeds
    for s in (1, 2, 3):
        out.append((f"c1_seed{s}", W.c1(seed=s)))
    # paper grid points (orchestrator.py:373-390) at a shorter horizon
    base = ExperimentConfig(horizon_s=240.0)
    for clients, workers, segdur, variant in [
        (4, 4, 2.0, "T"), (24, 4, 2.0, "B"), (24, 4, 2.0, "T"), (24, 4, 2.0, "TC"),
        (24, 4, 2.0, "TCP"), (24, 4, 2.0, "TCF"), (24, 4, 2.0, "TCPF"), (40, 8, 4.0, "TCPF"),
        (40, 4, 4.0, "TCP"),
    ]:
        cfg = dataclasses.replace(base, variant=variant, clients=clients, workers=workers,
                                  segment_duration_s=segdur)
        out.append((f"grid_c{clients}_k{workers}_t{int(segdur)}_{variant}", cfg))
    # configs 2 and 3 (Zipf, 50 sequences, cache fraction), shortened horizon
    out.append(("c2_seed1_h120", W.c2(seed=1, horizon_s=120.0)))
    out.append(("c3_f0_h90", W.c3(seed=2, fraction=0.0, horizon_s=90.0)))
    out.append(("c3_f05_h90", W.c3(seed=3, fraction=0.5, horizon_s=90.0)))
    out.append(("c3_f01_h90_uniform", W.c3(seed=4, fraction=0.1, horizon_s=90.0, popularity="uniform")))
    # edge cases
    out.append(("edge_noise0_tcp", dataclasses.replace(base, variant="TCP", clients=12, noise_rel_std=0.0,
                                                       horizon_s=120.0, seed=5)))
    out.append(("edge_k1_tcpf", dataclasses.replace(base, variant="TCPF", clients=10, workers=1,
                                                    horizon_s=120.0, seed=6)))
    out.append(("edge_tiny_cache", dataclasses.replace(base, variant="TCP", clients=16, cache_capacity_bytes=600_000,
                                                       horizon_s=120.0, seed=7)))
    # the request latency lives in the netem section of the config document
    # (orchestrator.py:133: ClientConfig.latency_s = netem.latency_s)
    out.append(("edge_latency0", dataclasses.replace(base, variant="TCP", clients=8, horizon_s=100.0, seed=8,
                                                     client=ClientConfig(latency_s=0.0),
                                                     netem=NetemConfig(latency_s=0.0))))
    out.append(("edge_partial_seg", dataclasses.replace(
        base, variant="TCP", clients=10, horizon_s=150.0, seed=9,
        sequences=[{"id": "a", "duration_s": 9.5, "segment_duration_s": 2.0},
                   {"id": "b", "duration_s": 7.0, "segment_duration_s": 3.0}])))
    out.append(("edge_rho_per_rank", dataclasses.replace(
        base, variant="TC", clients=14, horizon_s=120.0, seed=10,
        per_rank_rho={1: 0.3, 2: 0.5, 3: 0.9, 4: 1.4, 5: 0.2})))
    out.append(("edge_short_horizon", dataclasses.replace(base, variant="TCP", clients=30, horizon_s=7.0,
                                                          arrival_rate_per_s=5.0, seed=11)))
    out.append(("edge_two_clients", dataclasses.replace(base, variant="TCP", clients=2, workers=2, horizon_s=60.0,
                                                        seed=12)))
    out.append(("c5_small", W.c5(seed=1, clients=60, horizon_s=60.0)))
    # bounded job queue: OverloadError -> error records, client retry/backoff, aborted sessions
    out.append(("knob_qbound_tcp", dataclasses.replace(base, variant="TCP", clients=40, workers=1, queue_bound=2,
                                                       horizon_s=150.0, arrival_rate_per_s=1.0, seed=13)))
    out.append(("knob_qbound_abort", dataclasses.replace(base, variant="TC", clients=30, workers=1, queue_bound=1,
                                                         horizon_s=150.0, arrival_rate_per_s=1.0, seed=14,
                                                         client=ClientConfig(retries=1, retry_backoff_s=0.25))))
    out.append(("knob_qbound_c2", W.c2(seed=15, horizon_s=90.0, queue_bound=3, variant="TCPF")))
    # demand-priority queues (speculative jobs only when no demand job waits)
    out.append(("knob_prio_tcp", dataclasses.replace(base, variant="TCP", clients=30, workers=2, demand_priority=True,
                                                     horizon_s=150.0, arrival_rate_per_s=1.0, seed=16)))
    out.append(("knob_prio_qbound", dataclasses.replace(base, variant="TCPF", clients=40, workers=1,
                                                        demand_priority=True, queue_bound=2, horizon_s=150.0,
                                                        arrival_rate_per_s=1.0, seed=17)))
    out.append(("knob_prio_c3", W.c3(seed=18, fraction=0.2, horizon_s=90.0, demand_priority=True)))
    # CSV bandwidth traces (netem.trace_dir): uneven steps, header/comment rows, a leading gap
    tdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traces")
    out.append(("knob_trace_dir", dataclasses.replace(base, variant="TCP", clients=9, horizon_s=200.0,
                                                      arrival_rate_per_s=0.5, seed=19,
                                                      netem=NetemConfig(trace_dir=tdir))))
    return out
