"""Known-answer tests of the per-client model functions (csrc/otf_model.cuh).

tests/golden/model_kat.json holds answers of the UNMODIFIED reference
(tests/golden/make_model_kat.py): BandwidthTrace.completion_time
(netem.py:77-118), including the reference's own netem test cases
(tests/test_netem.py:28-86), select_quality (client.py:134-146), including
its band-edge tests (tests/test_client.py:138-171), and PlayerBuffer
(client.py:74-121) step sequences.  The host build of the
same source must match them bit-for-bit (CPU tests).  The device build must
match the host build bit-for-bit (-m gpu).
"""

from __future__ import annotations

import ctypes
import json
import math
import os

import numpy as np
import pytest

from paper_2603_08417_b200 import _lib

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "model_kat.json")))
dp = ctypes.POINTER(ctypes.c_double)


def _grid(starts):
    """The engine's bisect-free lookup applies when starts[i] == i * step exactly (inputs.py)."""
    if len(starts) < 2:
        return 0.0
    g = float(starts[1] - starts[0])
    return g if g > 0 and all(x == float(i) * g for i, x in enumerate(starts)) else 0.0


def _same(a: float, b: float) -> bool:
    return (math.isinf(a) and math.isinf(b)) or a == b


def test_completion_time_matches_reference():
    L = _lib.lib()
    n_checked = 0
    for doc in KAT["completion_time"]:
        starts = np.asarray(doc["starts"], dtype=np.float64)
        values = np.asarray(doc["values"], dtype=np.float64)
        for grid in {0.0, _grid(doc["starts"])}:
            for start, nbytes, want in doc["queries"]:
                got = L.otf_model_completion_time(starts.ctypes.data_as(dp), values.ctypes.data_as(dp),
                                                  len(starts), doc["period"], doc["pbits"], grid, start, nbytes)
                assert _same(got, want), (doc["samples"], start, nbytes, got, want)
                n_checked += 1
    assert n_checked > 2000


def test_completion_time_reference_unit_cases():
    """The reference's own netem known answers (tests/test_netem.py:28-53)."""
    fixed = KAT["completion_time"][:4]
    assert fixed[0]["queries"][0][2] == pytest.approx(1.0)
    assert fixed[1]["queries"][0][2] == pytest.approx(2.0)
    assert math.isinf(fixed[2]["queries"][0][2])
    assert fixed[3]["queries"][0][2] == pytest.approx(2.25)
    mono = [q[2] for q in KAT["completion_time"][4]["queries"]]
    assert mono == sorted(mono)


def test_select_quality_matches_reference():
    L = _lib.lib()
    ladder = np.asarray(KAT["ladder"], dtype=np.int64)
    c = KAT["client"]
    for level, cur, est, want in KAT["select_quality"]:
        got = L.otf_model_select_quality(level, cur, 0 if est is None else 1, 0.0 if est is None else est,
                                         ladder.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(ladder),
                                         c["panic"], c["safe"], c["headroom"])
        assert got == want, (level, cur, est, got, want)


def test_player_buffer_matches_reference():
    """PlayerBuffer.advance / on_segment (client.py:91-121): 200 random sequences, the
    state after every step, bit-exact (stall counts are a discrete outcome)."""
    L = _lib.lib()
    B = KAT["buffer"]
    for seq in B["sequences"]:
        ops = np.asarray([int(o[0]) for o in seq["ops"]], dtype=np.int32)
        t = np.asarray([o[1] for o in seq["ops"]], dtype=np.float64)
        dur = np.asarray([o[2] for o in seq["ops"]], dtype=np.float64)
        out = np.empty((len(ops), 6))
        _lib.check(L.otf_model_buffer_run(seq["t0"], len(ops), ops.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                          t.ctypes.data_as(dp), dur.ctypes.data_as(dp), B["startup"], B["resume"],
                                          out.ctypes.data_as(dp)), "otf_model_buffer_run")
        for o, got in zip(seq["ops"], out):
            want = o[3:]
            assert got[0] == want[0] and int(got[1]) == want[1] and int(got[2]) == want[2], (seq["t0"], o, got)
            assert got[3] == want[3] and got[5] == want[5], (o, got)
            assert (math.isnan(got[4]) and math.isnan(want[4])) or got[4] == want[4], (o, got)


@pytest.mark.gpu
def test_completion_time_device_equals_host():
    """The device compilation (--fmad=false) computes exactly what the host does."""
    import torch
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    for doc in KAT["completion_time"]:
        starts = torch.tensor(doc["starts"], dtype=torch.float64, device=dev)
        values = torch.tensor(doc["values"], dtype=torch.float64, device=dev)
        qs = torch.tensor([q[0] for q in doc["queries"]], dtype=torch.float64, device=dev)
        nb = torch.tensor([q[1] for q in doc["queries"]], dtype=torch.int64, device=dev)
        for grid in {0.0, _grid(doc["starts"])}:
            out = torch.empty_like(qs)
            _lib.check(L.otf_model_completion_times(starts.data_ptr(), values.data_ptr(), len(doc["starts"]),
                                                    doc["period"], doc["pbits"], grid, qs.data_ptr(),
                                                    nb.data_ptr(), len(qs), out.data_ptr(),
                                                    torch.cuda.current_stream(dev).cuda_stream),
                       "otf_model_completion_times")
            got = out.cpu().numpy()
            for (start, nbytes, want), g in zip(doc["queries"], got):
                assert _same(float(g), want), (doc["samples"], start, nbytes, float(g), want)
