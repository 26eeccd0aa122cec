"""On-disk contract: ExperimentResult.write() is byte-identical to the reference's
(metrics.py:122-162, orchestrator.py:311-324), and summary() equals the
reference's summary dict.  Uses oracle arrays (CPU) through the same result
class the GPU engine returns."""

import filecmp
import json
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2603_08417_b200.config import ExperimentConfig
from paper_2603_08417_b200.results import ExperimentResult, read_csv
from tests import parity

CSV_DIR = os.path.join(parity.GOLDEN_DIR, "csv")
CASES = sorted(os.listdir(CSV_DIR)) if os.path.isdir(CSV_DIR) else []


def _result(name):
    _, meta = parity.load_golden(name)
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta["popularity"]
    res = oracle.run(cfg)
    prep = oracle.Prepared(cfg)
    sizes, _ = prep.sizes()
    arrays = {k: v for k, v in res.items() if isinstance(v, np.ndarray) and k != "stats"}
    return ExperimentResult(cfg, arrays, res["stats"], prep.seq_ids, sizes=sizes,
                            seq_dur=list(prep.seq_duration), seq_segdur=list(prep.seq_segdur)), meta


@pytest.mark.parametrize("name", CASES)
def test_write_is_byte_identical(name, tmp_path):
    res, _ = _result(name)
    res.write(tmp_path)
    for f in ("requests.csv", "sessions.csv", "segments.csv", "jobs.csv", "config.json", "summary.json"):
        assert filecmp.cmp(tmp_path / f, os.path.join(CSV_DIR, name, f), shallow=False), f


@pytest.mark.parametrize("name", CASES)
def test_summary_equals_reference(name):
    res, meta = _result(name)
    got = json.loads(json.dumps(res.summary(), default=float))
    assert got == meta["summary"]


def test_read_csv_roundtrip(tmp_path):
    res, _ = _result(CASES[0])
    res.write(tmp_path)
    fields, rows = read_csv(tmp_path / "requests.csv", "requests")
    assert fields["schema"] == "requests.v1" and fields["config"] == res.fingerprint
    assert len(rows) == len(res.requests)
    with pytest.raises(ValueError):
        read_csv(tmp_path / "requests.csv", "jobs")
