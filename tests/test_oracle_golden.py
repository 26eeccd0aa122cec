"""Pin the C oracle against the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by running the unmodified reference
(tests/golden/make_golden.py); every field must match bit-for-bit.
"""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle  # noqa: E402
from paper_2603_08417_b200.config import ExperimentConfig  # noqa: E402
from tests import parity  # noqa: E402


def _cfg(meta):
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta["popularity"]
    cfg.zipf_exponent = meta["zipf_exponent"]
    return cfg


@pytest.mark.parametrize("name", parity.golden_names())
def test_oracle_matches_reference(name):
    want, meta = parity.load_golden(name)
    cfg = _cfg(meta)
    got = oracle.run(cfg)
    errs = parity.compare(got, want)
    assert not errs, "\n".join(errs[:20])
    stats = oracle.backend_stats(got, "C" in cfg.variant)
    errs = parity.compare_stats(stats, meta["backend_stats"])
    assert not errs, "\n".join(errs)
    assert got["stats"][oracle.ST["status"]] == 0


def test_oracle_sizes_match_numpy():
    """Segment sizes: SeedSequence/PCG64/uniform restated in C vs numpy (content.py:208-218)."""
    import hashlib
    cfg = ExperimentConfig(seed=123456789012, size_jitter=0.07)
    prep = oracle.Prepared(cfg)
    sizes, counts = prep.sizes()
    for s, sid in enumerate(prep.seq_ids):
        key = int.from_bytes(hashlib.sha256(sid.encode()).digest()[:8], "big")
        for r, b in cfg.ladder:
            for i in range(counts[s]):
                g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, key, r, i])))
                dur = min(cfg.segment_duration_s, cfg.sequence_duration_s - i * cfg.segment_duration_s)
                u = g.uniform(-cfg.size_jitter, cfg.size_jitter)
                want = max(1, round(b * dur / 8 * (1 + u)))
                assert sizes[s, r - 1, i] == want


def test_oracle_picks_match_numpy():
    """Uniform picks: PCG64 bounded integers restated in C (orchestrator.py:340-342)."""
    for seed, n in [(1, 4), (77, 50), (2**33 + 5, 3)]:
        cfg = ExperimentConfig(seed=seed, clients=3, variant="B", horizon_s=400.0,
                               sequences=[{"id": f"q{i}", "duration_s": 4.0, "segment_duration_s": 1.0}
                                          for i in range(n)], arrival_rate_per_s=1.0)
        res = oracle.run(cfg)
        for c in range(cfg.clients):
            seqs = res["sess_seq"][res["sess_client"] == c]
            g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 3, c])))
            want = [int(g.integers(n)) for _ in range(len(seqs))]
            assert list(seqs) == want
