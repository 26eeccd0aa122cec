"""The Python-level drop-in boundary on CPU: a real reference ExperimentConfig
passed through ExperimentConfig.from_reference (config.py, orchestrator.py:117-209),
the INTEGRATION.md backend switch, and the CLI's flag handling (cli.py:29-90).

The reference is imported from /root/reference when it is present (this
container); the tests skip elsewhere (the GPU box has no reference tree).
"""

from __future__ import annotations

import dataclasses
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(os.path.join(REF_SRC, "otfstream"))
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="reference tree not present")


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import otfstream.metrics as metrics
    import otfstream.orchestrator as orch
    return orch, metrics


def _ref_configs(orch):
    base = orch.ExperimentConfig()
    yield base
    yield dataclasses.replace(base, variant="TCPF", clients=40, workers=8, seed=11, queue_bound=6,
                              demand_priority=True, per_rank_rho={1: 0.3, 2: 0.4, 3: 0.5, 4: 0.6, 5: 0.7})
    yield dataclasses.replace(base, variant="T", sequences=[{"id": "a", "duration_s": 12.0, "segment_duration_s": 2.0},
                                                            {"id": "b", "duration_s": 9.0}],
                              noise_rel_std=0.0, cache_capacity_bytes=1 << 20)
    yield dataclasses.replace(base, netem=dataclasses.replace(base.netem, sigma=0.5, step_s=0.5, latency_s=0.05),
                              client=dataclasses.replace(base.client, retries=1, retry_backoff_s=0.25,
                                                         latency_s=0.05))


@needs_ref
def test_from_reference_round_trips_every_field():
    orch, metrics = _ref()
    from paper_2603_08417_b200.config import ExperimentConfig
    for ref_cfg in _ref_configs(orch):
        ours = ExperimentConfig.from_reference(ref_cfg)
        assert ours.to_dict() == ref_cfg.to_dict()
        from paper_2603_08417_b200.results import fingerprint
        assert fingerprint(ours.to_dict()) == metrics.fingerprint(ref_cfg.to_dict())
        # and the lowered policy matches the reference's variant table (backend.py:52-82)
        p_ref, p_ours = ref_cfg.policy(), ours.policy()
        for f in ("cache_enabled", "speculative_enabled"):
            assert getattr(p_ref, f) == getattr(p_ours, f), f


@needs_ref
def test_integration_patch_routes_reference_configs(monkeypatch):
    """The three-line reference-side patch of INTEGRATION.md, applied to the real
    reference module: with OTFSTREAM_BACKEND=b200 its run_experiment hands the
    converted config to this package (captured here; the GPU run itself is
    covered by the -m gpu tests)."""
    orch, metrics = _ref()
    import paper_2603_08417_b200 as gpu

    seen = []
    monkeypatch.setattr(gpu, "run_experiment", lambda cfg: seen.append(cfg) or "gpu-result")
    original = orch.run_experiment

    def patched(config):                               # INTEGRATION.md section 1, verbatim logic
        if os.environ.get("OTFSTREAM_BACKEND") == "b200":
            return gpu.run_experiment(gpu.ExperimentConfig.from_reference(config))
        return original(config)

    monkeypatch.setenv("OTFSTREAM_BACKEND", "b200")
    cfg = dataclasses.replace(orch.ExperimentConfig(), variant="TCP", clients=24, seed=5)
    assert patched(cfg) == "gpu-result"
    assert len(seen) == 1 and isinstance(seen[0], gpu.ExperimentConfig)
    assert metrics.fingerprint(cfg.to_dict()) == gpu.results.fingerprint(seen[0].to_dict())


def test_product_path_fails_loudly_without_cuda():
    import torch

    from paper_2603_08417_b200 import _lib, engine, workloads
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_lib.OtfError):
        engine.run_experiment(workloads.c1(seed=1))


def test_cli_overrides_and_subcommands(tmp_path):
    import json

    from paper_2603_08417_b200 import cli
    cfg_file = tmp_path / "c.json"
    from paper_2603_08417_b200.config import ExperimentConfig
    cfg_file.write_text(json.dumps(ExperimentConfig(variant="TC", clients=7).to_dict()))
    p = cli.build_parser()
    a = p.parse_args(["run", "--config", str(cfg_file), "--clients", "12", "--seed", "9"])
    got = cli._configured(a)
    assert (got.variant, got.clients, got.seed) == ("TC", 12, 9)
    a = p.parse_args(["run", "--variant", "TCPF"])
    assert cli._configured(a) == dataclasses.replace(ExperimentConfig(), variant="TCPF")
    a = p.parse_args(["sweep", "c5", "--seeds", "2"])
    assert a.fn is cli.cmd_sweep and a.seeds == 2
    with pytest.raises(SystemExit):
        p.parse_args(["matrix"])                       # --out is required, as in the reference
