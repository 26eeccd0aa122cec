"""The five BASELINE.json configurations lowered to concrete ExperimentConfigs.

Interpretation decisions (recorded in DESIGN.md):

* "300 frames"                -> one 10 s sequence at 1 s segments (10 segments).
* "Zipf(0.8) over 50 seqs"    -> ``popularity="zipf"``: P(k) ~ k^-0.8 over the
                                 catalog order, inverse CDF on ``picks.random()``.
* "LRU cache f% of ladder"    -> capacity = max(1, floor(f * nominal ladder bytes)),
                                 nominal = bitrate * duration / 8 summed over every
                                 (sequence, rank, index); f = 0 -> 1 byte (the
                                 reference forbids 0 and has no TP variant).
* 10 .. 10,000 clients        -> arrival rate = clients / 60 s for configs 2-5 (at the
                                 default 0.1/s only ~65 clients ever start in 600 s).
* "4 transcoder slots"        -> workers = 4.
* "10-rep ladder"             -> config.LADDER_10 (geometric 1 -> 24 Mbit/s).
* "1M-request traces"         -> 2,800 clients, 1 s segments, 600 s horizon.
"""

from __future__ import annotations

import dataclasses
import math

from .config import FIXTURE_LADDER, LADDER_10, ExperimentConfig, nominal_ladder_bytes

__all__ = ["c1", "c2", "c3", "c4", "c5", "c3_sweep", "c4_sweep", "c5_sweep", "c5t_sweep", "with_cache_fraction",
           "C4_CLIENTS", "C4_VARIANTS"]

C4_CLIENTS = (10, 30, 100, 300, 1000, 3000, 10000)
C4_VARIANTS = ("B", "T", "TC", "TCP", "TCF", "TCPF")


def with_cache_fraction(cfg: ExperimentConfig, fraction: float) -> ExperimentConfig:
    cap = max(1, int(math.floor(fraction * nominal_ladder_bytes(cfg))))
    return dataclasses.replace(cfg, cache_capacity_bytes=cap)


def _seqs(n: int, duration: float = 10.0, segdur: float = 1.0) -> list[dict]:
    return [{"id": f"s{i:02d}", "duration_s": duration, "segment_duration_s": segdur} for i in range(n)]


def c1(seed: int = 1, **kw) -> ExperimentConfig:
    """Config 1: 1 sequence (10 s, 1 s segments, 5-rank ladder), 10 clients, variant T."""
    base = dict(variant="T", clients=10, workers=4, seed=seed,
                sequences=[{"id": "seq00", "duration_s": 10.0, "segment_duration_s": 1.0}],
                segment_duration_s=1.0, sequence_duration_s=10.0, ladder=list(FIXTURE_LADDER))
    base.update(kw)
    return ExperimentConfig(**base)


def c2(seed: int = 1, clients: int = 100, variant: str = "TC", fraction: float = 0.20, **kw) -> ExperimentConfig:
    """Config 2: 100 clients, Zipf(0.8) over 50 sequences, LRU 20% of ladder, K = 4."""
    base = dict(variant=variant, clients=clients, workers=4, seed=seed, sequences=_seqs(50),
                segment_duration_s=1.0, sequence_duration_s=10.0, ladder=list(FIXTURE_LADDER),
                arrival_rate_per_s=clients / 60.0, popularity="zipf", zipf_exponent=0.8)
    base.update(kw)
    return with_cache_fraction(ExperimentConfig(**base), fraction)


def c3(seed: int = 1, fraction: float = 0.2, **kw) -> ExperimentConfig:
    """Config 3: config 2 + speculation (TCP); cache fraction swept 0..1 in 0.1 steps."""
    return c2(seed=seed, variant="TCP", fraction=fraction, **kw)


def c4(seed: int = 1, clients: int = 10, variant: str = "TCP", fraction: float = 0.20, **kw) -> ExperimentConfig:
    """Config 4: client-count sweep {10..10,000} x variants x 64 seeds (one point)."""
    return c2(seed=seed, clients=clients, variant=variant, fraction=fraction, **kw)


def c5(seed: int = 1, variant: str = "TCPF", fraction: float = 0.20, clients: int = 2800, **kw) -> ExperimentConfig:
    """Config 5: ~1M answered requests per scenario, 10-rank ladder (one of 1,024 scenarios)."""
    base = dict(variant=variant, clients=clients, workers=4, seed=seed, sequences=_seqs(50),
                segment_duration_s=1.0, sequence_duration_s=10.0, ladder=list(LADDER_10),
                arrival_rate_per_s=clients / 60.0, popularity="zipf", zipf_exponent=0.8)
    base.update(kw)
    return with_cache_fraction(ExperimentConfig(**base), fraction)


C3_FRACTIONS = tuple(k / 10 for k in range(11))


def c3_sweep(seeds=range(1, 2)):
    """Config 3: TCP with the cache swept 0..100% of the ladder in 10% steps, per seed."""
    return [c3(seed=s, fraction=f) for s in seeds for f in C3_FRACTIONS]


def c4_sweep(seeds=range(1, 65)):
    return [c4(seed=s, clients=n, variant=v) for n in C4_CLIENTS for v in C4_VARIANTS for s in seeds]


C5_VARIANTS = ("TC", "TCP", "TCF", "TCPF")
C5_FRACTIONS = (0.05, 0.10, 0.20, 0.50)


def c5_sweep(seeds=range(1, 65), clients: int = 2800):
    """1,024 scenarios = 64 seeds x 4 variants x 4 cache fractions."""
    return [c5(seed=s, variant=v, fraction=f, clients=clients)
            for s in seeds for v in C5_VARIANTS for f in C5_FRACTIONS]


C5T_VARIANTS = ("T", "TC", "TCP", "TCF")
C5T_FRACTIONS = (0.0, 0.005, 0.01, 0.02)


def c5t_sweep(seeds=range(1, 65), clients: int = 2800):
    """The transcode-bound counterpart of config 5 (not a BASELINE config): the same
    2,800-client / 600 s / 10-rank scenarios with no cache (T) or caches of
    0-2% of the ladder, so most requests wait on the 4 transcoders.  T ignores the
    cache size: its four points per seed are the same simulation."""
    return [c5(seed=s, variant=v, fraction=f, clients=clients)
            for s in seeds for v in C5T_VARIANTS for f in C5T_FRACTIONS]
