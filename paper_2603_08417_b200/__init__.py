"""paper_2603_08417_b200 -- B200 engine for the otfstream scalability experiment.

Drop-in for the reference's virtual-clock hot path
(otfstream.orchestrator.run_experiment, /root/reference/pkg/src/otfstream/
orchestrator.py:327-370): same ExperimentConfig document, same
ExperimentResult shape, every scenario replayed on the GPU by libotfgpu.so.

    from paper_2603_08417_b200 import ExperimentConfig, run_experiment, run_batch
    res = run_experiment(ExperimentConfig(variant="TCP", clients=24))
    res.summary()
"""

from .config import (  # noqa: F401
    VARIANTS, BackendPolicy, BufferConfig, CatalogConfig, ClientConfig, ConfigError, ExperimentConfig,
    LatencyModel, NetemConfig, NotFoundError, OverloadError, SequenceConfig, scenario_matrix,
)
from .results import (  # noqa: F401
    ExperimentResult, RequestRecord, SegmentRecord, SessionReport, TranscodeJob, fingerprint,
    quality_proportions, response_time_cdf, stalls_per_session,
)

__version__ = "0.1.0"


def run_experiment(config):
    """Run one config on the GPU (records mode); see engine.run_experiment."""
    from .engine import run_experiment as _run
    return _run(config)


def run_batch(configs, mode: str = "records", engine: str = "windowed", device=None):
    """Run many configs in one launch; see engine.run_batch."""
    from .engine import run_batch as _run
    return _run(configs, mode=mode, engine=engine, device=device)
