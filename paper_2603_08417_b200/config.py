"""Experiment configuration: the reference's config document, re-declared.

The dataclasses below keep the reference's field names, defaults, validation
and JSON document shape so a reference config file or object loads unchanged:

* ``ExperimentConfig``  -- orchestrator.py:74-268
* ``NetemConfig``       -- orchestrator.py:61-71
* ``BufferConfig``/``ClientConfig`` -- client.py:49-71
* ``BackendPolicy``/``VARIANTS``    -- backend.py:41,52-82
* ``LatencyModel``      -- transcode.py:40-81
* ``CatalogConfig``/``SequenceConfig``/ladder validation -- content.py:46-135

Two extensions needed by the BASELINE sweep configs are added as optional
fields that are omitted from ``to_dict()`` while at their defaults, so the
config fingerprint of every reference-expressible config is unchanged:

* ``popularity`` ("uniform" | "zipf") and ``zipf_exponent``: sequence picks by
  inverse CDF over ``picks.random()`` instead of ``picks.integers(n)``
  (orchestrator.py:340-342 draws uniformly; Zipf is not in the reference).
"""

from __future__ import annotations

import dataclasses
import json
import math
from dataclasses import dataclass, field

__all__ = [
    "ConfigError", "NotFoundError", "OverloadError",
    "VARIANTS", "FIXTURE_LADDER", "FIXTURE_SEQUENCES", "LADDER_10",
    "SequenceConfig", "CatalogConfig", "BufferConfig", "ClientConfig", "NetemConfig",
    "BackendPolicy", "LatencyModel", "ExperimentConfig", "scenario_matrix",
    "DEFAULT_CAPACITY_BYTES", "DEFAULT_LATENCY_S",
]

VARIANTS = ("B", "T", "TC", "TCP", "TCF", "TCPF")
DEFAULT_CAPACITY_BYTES = 134217728  # 128 MiB (cache.py:24)
DEFAULT_LATENCY_S = 0.020           # netem.py:26

FIXTURE_LADDER = [  # content.py:251-257
    (1, 2_000_000),
    (2, 3_500_000),
    (3, 6_000_000),
    (4, 10_000_000),
    (5, 16_000_000),
]
FIXTURE_SEQUENCES = ["longdress", "loot", "redandblack", "soldier"]  # content.py:259

# 10-representation ladder for the large sweep (BASELINE config 5): geometric
# 1 -> 24 Mbit/s, rounded to kbit/s.  Not in the reference (new fixture).
LADDER_10 = [(r, int(round(1e6 * 24.0 ** ((r - 1) / 9.0) / 1000.0)) * 1000) for r in range(1, 11)]


class ConfigError(ValueError):
    """Invalid configuration (content.py:38)."""


class NotFoundError(KeyError):
    """Unknown sequence, rank, or out-of-range segment index (content.py:42)."""


class OverloadError(RuntimeError):
    """Job queue is at its bound (backend.py:48)."""


@dataclass(frozen=True)
class SequenceConfig:
    id: str
    duration_s: float
    segment_duration_s: float


@dataclass
class CatalogConfig:
    sequences: list[SequenceConfig]
    ladder: list[tuple[int, int]]
    stored_ranks: list[int]
    seed: int = 0
    size_jitter: float = 0.05

    def validate(self) -> None:
        """Catalog.__init__ + BitrateLadder.__post_init__ checks (content.py:102-118,173-183)."""
        if not self.sequences:
            raise ConfigError("catalog needs at least one sequence")
        for s in self.sequences:
            if s.duration_s <= 0 or s.segment_duration_s <= 0:
                raise ConfigError(f"sequence {s.id!r}: durations must be positive")
        if not 0 <= self.size_jitter < 1:
            raise ConfigError(f"size_jitter must be in [0, 1), got {self.size_jitter}")
        ids = [s.id for s in self.sequences]
        if len(set(ids)) != len(ids):
            raise ConfigError("duplicate sequence ids")
        bitrates = dict(self.ladder)
        ranks = sorted(bitrates)
        if len(ranks) < 2:
            raise ConfigError("ladder needs at least 2 representations")
        if ranks != list(range(1, len(ranks) + 1)):
            raise ConfigError(f"ladder ranks must be 1..L without gaps, got {ranks}")
        rates = [bitrates[r] for r in ranks]
        if any(b <= 0 for b in rates):
            raise ConfigError("bitrates must be positive")
        if any(hi <= lo for lo, hi in zip(rates, rates[1:])):
            raise ConfigError("bitrates must strictly increase with rank")
        stored = set(self.stored_ranks)
        if not stored:
            raise ConfigError("stored_ranks must not be empty")
        if not stored <= set(ranks):
            raise ConfigError(f"stored_ranks {sorted(stored)} outside ladder {ranks}")
        if len(ranks) not in stored:
            raise ConfigError("the highest rank must be stored (it is the transcoding source)")


@dataclass(frozen=True)
class BufferConfig:
    target_s: float = 12.0
    safe_s: float = 8.0
    panic_s: float = 2.0
    resume_s: float = 2.0
    startup_s: float = 3.0

    def __post_init__(self):
        if not (self.panic_s < self.startup_s <= self.safe_s < self.target_s):
            raise ValueError("thresholds must satisfy panic < startup <= safe < target")
        if self.resume_s <= 0:
            raise ValueError("resume threshold must be positive")


@dataclass(frozen=True)
class ClientConfig:
    buffer: BufferConfig = field(default_factory=BufferConfig)
    ewma_alpha: float = 0.3
    headroom: float = 1.2
    retries: int = 3
    retry_backoff_s: float = 0.5
    latency_s: float = DEFAULT_LATENCY_S


@dataclass(frozen=True)
class NetemConfig:
    median_bps: float = 17e6
    sigma: float = 0.35
    theta_per_s: float = 0.08
    floor_bps: float = 2e6
    cap_bps: float = 400e6
    step_s: float = 1.0
    trace_duration_s: float = 600.0
    latency_s: float = 0.020
    trace_dir: str | None = None


@dataclass
class BackendPolicy:
    variant: str
    cache_capacity_bytes: int = DEFAULT_CAPACITY_BYTES
    workers: int = 4
    queue_bound: int = 0
    demand_priority: bool = False

    def __post_init__(self):
        self.variant = self.variant.replace("+", "").upper()
        if self.variant not in VARIANTS:
            raise ConfigError(f"unknown variant {self.variant!r}; expected one of {VARIANTS}")
        if self.workers < 1:
            raise ConfigError("need at least one worker")
        if self.queue_bound < 0:
            raise ConfigError("queue_bound must be >= 0")

    @property
    def cache_enabled(self) -> bool:
        return "C" in self.variant

    @property
    def speculative_enabled(self) -> bool:
        return "P" in self.variant

    def stored_ranks(self, top_rank: int) -> list[int]:
        if self.variant == "B":
            return list(range(1, top_rank + 1))
        if "F" in self.variant:
            return [1, top_rank]
        return [top_rank]


@dataclass
class LatencyModel:
    per_rank_rho: dict[int, float]
    noise_rel_std: float = 0.05
    seed: int = 0

    def __post_init__(self):
        if not self.per_rank_rho:
            raise ConfigError("latency model needs at least one rank entry")
        if any(rho <= 0 for rho in self.per_rank_rho.values()):
            raise ConfigError("rho must be positive for every rank")
        if self.noise_rel_std < 0:
            raise ConfigError("noise_rel_std must be >= 0")

    def rho(self, rank: int) -> float:
        try:
            return self.per_rank_rho[rank]
        except KeyError:
            raise ConfigError(f"latency model has no rho for rank {rank}") from None


@dataclass
class ExperimentConfig:
    variant: str = "TC"
    clients: int = 4
    workers: int = 4
    horizon_s: float = 600.0
    arrival_rate_per_s: float = 0.1
    seed: int = 1
    clock: str = "virtual"

    segment_duration_s: float = 4.0
    sequence_duration_s: float = 80.0
    size_jitter: float = 0.05
    ladder: list[tuple[int, int]] = field(default_factory=lambda: list(FIXTURE_LADDER))
    sequences: list[dict] | None = None

    cache_capacity_bytes: int = DEFAULT_CAPACITY_BYTES
    queue_bound: int = 0
    demand_priority: bool = False

    rho: float = 0.5
    per_rank_rho: dict[int, float] | None = None
    noise_rel_std: float = 0.05

    netem: NetemConfig = field(default_factory=NetemConfig)
    client: ClientConfig = field(default_factory=ClientConfig)

    # -- extensions (not in the reference; omitted from to_dict at defaults) --
    popularity: str = "uniform"   # "uniform" | "zipf"
    zipf_exponent: float = 0.8

    def __post_init__(self):
        if self.clients < 1:
            raise ConfigError("need at least one client")
        if self.horizon_s <= 0:
            raise ConfigError("horizon must be positive")
        if self.arrival_rate_per_s <= 0:
            raise ConfigError("arrival rate must be positive")
        if self.clock not in ("virtual", "wall"):
            raise ConfigError(f"unknown clock mode {self.clock!r}")
        if self.popularity not in ("uniform", "zipf"):
            raise ConfigError(f"unknown popularity {self.popularity!r}")
        BackendPolicy(self.variant)

    # -- config document (orchestrator.py:117-209) ------------------------------

    @classmethod
    def from_dict(cls, d: dict) -> "ExperimentConfig":
        exp = d.get("experiment", {})
        cat = d.get("catalog", {})
        be = d.get("backend", {})
        lm = d.get("latency_model", {})
        ne = d.get("netem", {})
        cl = d.get("client", {})
        buffer_keys = {"target_s", "safe_s", "panic_s", "resume_s", "startup_s"}
        buf = BufferConfig(**{k: v for k, v in cl.items() if k in buffer_keys})
        client = ClientConfig(
            buffer=buf,
            ewma_alpha=cl.get("ewma_alpha", 0.3),
            headroom=cl.get("headroom", 1.2),
            retries=cl.get("retries", 3),
            retry_backoff_s=cl.get("retry_backoff_s", 0.5),
            latency_s=ne.get("latency_s", 0.020),
        )
        per_rank = lm.get("per_rank_rho")
        return cls(
            variant=exp.get("variant", "TC"),
            clients=int(exp.get("clients", 4)),
            workers=int(exp.get("workers", 4)),
            horizon_s=float(exp.get("horizon_s", 600.0)),
            arrival_rate_per_s=float(exp.get("arrival_rate_per_s", 0.1)),
            seed=int(exp.get("seed", 1)),
            clock=exp.get("clock", "virtual"),
            segment_duration_s=float(cat.get("segment_duration_s", 4.0)),
            sequence_duration_s=float(cat.get("duration_s", 80.0)),
            size_jitter=float(cat.get("size_jitter", 0.05)),
            ladder=[(int(e["rank"]), int(e["bitrate_bps"])) for e in cat["ladder"]]
            if "ladder" in cat else list(FIXTURE_LADDER),
            sequences=cat.get("sequences"),
            cache_capacity_bytes=int(be.get("cache_capacity_bytes", DEFAULT_CAPACITY_BYTES)),
            queue_bound=int(be.get("queue_bound", 0)),
            demand_priority=bool(be.get("demand_priority", False)),
            rho=float(lm.get("rho", 0.5)),
            per_rank_rho={int(k): float(v) for k, v in per_rank.items()} if per_rank else None,
            noise_rel_std=float(lm.get("noise_rel_std", 0.05)),
            netem=NetemConfig(**{k: v for k, v in ne.items() if k in
                                 {f.name for f in dataclasses.fields(NetemConfig)}}),
            client=client,
            popularity=exp.get("popularity", "uniform"),
            zipf_exponent=float(exp.get("zipf_exponent", 0.8)),
        )

    @classmethod
    def from_file(cls, path) -> "ExperimentConfig":
        with open(path, encoding="utf-8") as fh:
            return cls.from_dict(json.load(fh))

    @classmethod
    def from_reference(cls, ref) -> "ExperimentConfig":
        """Accept a reference ``otfstream.orchestrator.ExperimentConfig`` (duck-typed)."""
        if isinstance(ref, cls):
            return ref
        return cls.from_dict(ref.to_dict())

    def to_dict(self) -> dict:
        client = {
            "target_s": self.client.buffer.target_s,
            "safe_s": self.client.buffer.safe_s,
            "panic_s": self.client.buffer.panic_s,
            "resume_s": self.client.buffer.resume_s,
            "startup_s": self.client.buffer.startup_s,
            "ewma_alpha": self.client.ewma_alpha,
            "headroom": self.client.headroom,
            "retries": self.client.retries,
            "retry_backoff_s": self.client.retry_backoff_s,
        }
        catalog = {
            "segment_duration_s": self.segment_duration_s,
            "duration_s": self.sequence_duration_s,
            "size_jitter": self.size_jitter,
            "ladder": [{"rank": r, "bitrate_bps": b} for r, b in self.ladder],
        }
        if self.sequences is not None:
            catalog["sequences"] = self.sequences
        latency_model = {"rho": self.rho, "noise_rel_std": self.noise_rel_std}
        if self.per_rank_rho is not None:
            latency_model["per_rank_rho"] = {str(k): v for k, v in self.per_rank_rho.items()}
        experiment = {
            "variant": self.variant,
            "clients": self.clients,
            "workers": self.workers,
            "horizon_s": self.horizon_s,
            "arrival_rate_per_s": self.arrival_rate_per_s,
            "seed": self.seed,
            "clock": self.clock,
        }
        if self.popularity != "uniform":
            experiment["popularity"] = self.popularity
            experiment["zipf_exponent"] = self.zipf_exponent
        return {
            "experiment": experiment,
            "catalog": catalog,
            "backend": {
                "cache_capacity_bytes": self.cache_capacity_bytes,
                "queue_bound": self.queue_bound,
                "demand_priority": self.demand_priority,
            },
            "latency_model": latency_model,
            "netem": dataclasses.asdict(self.netem),
            "client": client,
        }

    # -- derived pieces (orchestrator.py:213-268) --------------------------------

    def policy(self) -> BackendPolicy:
        return BackendPolicy(self.variant, self.cache_capacity_bytes, self.workers,
                             self.queue_bound, self.demand_priority)

    def catalog_config(self) -> CatalogConfig:
        top = max(rank for rank, _ in self.ladder)
        entries = self.sequences or [{"id": sid} for sid in FIXTURE_SEQUENCES]
        seqs = [
            SequenceConfig(
                e["id"],
                float(e.get("duration_s", self.sequence_duration_s)),
                float(e.get("segment_duration_s", self.segment_duration_s)),
            )
            for e in entries
        ]
        return CatalogConfig(
            sequences=seqs,
            ladder=list(self.ladder),
            stored_ranks=self.policy().stored_ranks(top),
            seed=self.seed,
            size_jitter=self.size_jitter,
        )

    def latency_model(self) -> LatencyModel:
        ranks = [rank for rank, _ in self.ladder]
        rho_map = self.per_rank_rho or {r: self.rho for r in ranks}
        return LatencyModel(rho_map, self.noise_rel_std, seed=self.seed)

    def validate(self) -> None:
        """Every check the reference runs before its first event (Catalog, Backend,
        SegmentCache, LatencyModel constructors)."""
        policy = self.policy()
        self.catalog_config().validate()
        lm = self.latency_model()
        for r, _ in self.ladder:
            lm.rho(r)
        if policy.cache_enabled and policy.cache_capacity_bytes <= 0:
            raise ValueError("cache capacity must be positive")  # cache.py:29-30
        if self.clock != "virtual":
            raise ConfigError("the GPU engine runs the virtual clock only")
        if not 0 <= self.client.retries < 255:
            raise ConfigError("client.retries must be in [0, 255) for the GPU engine")
        if not 0 <= int(self.seed) < 2 ** 64:
            # numpy's SeedSequence rejects negative entropy; seeds are carried as uint64 words
            # through the C ABI (otf_scenario.seed, otf_np_draws entropy)
            raise ConfigError("seed must be in [0, 2**64) for the GPU engine")


def nominal_ladder_bytes(config: ExperimentConfig) -> float:
    """Sum over (sequence, rank, index) of bitrate * duration / 8 (no jitter).

    Used to express "cache = f % of the ladder" (BASELINE configs 2-5) as bytes:
    capacity = max(1, floor(f * nominal_ladder_bytes)).
    """
    total = 0.0
    for s in config.catalog_config().sequences:
        count = math.ceil(s.duration_s / s.segment_duration_s)
        for i in range(count):
            duration = min(s.segment_duration_s, s.duration_s - i * s.segment_duration_s)
            for _, b in config.ladder:
                total += b * duration / 8
    return total


def scenario_matrix(base: ExperimentConfig) -> list[tuple[str, ExperimentConfig]]:
    """The paper's evaluation grid (orchestrator.py:373-390): {4,24,40} clients x
    {1,2} nodes (4 workers each) x {2,4} s segments x the six variants."""
    out = []
    for clients in (4, 24, 40):
        for nodes in (1, 2):
            for segdur in (2.0, 4.0):
                for variant in VARIANTS:
                    cfg = dataclasses.replace(
                        base, variant=variant, clients=clients, workers=4 * nodes,
                        segment_duration_s=segdur)
                    out.append((f"c{clients:02d}_n{nodes}_t{int(segdur)}_{variant}", cfg))
    return out
