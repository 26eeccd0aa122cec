"""GPU request generation (csrc/otf_gen.cu) against the host replicas and glibc.

* otf_libm.cuh's device build == glibc exp / log1p (the oracle library calls
  the host libm) on 1e8 arguments drawn over the ranges the streams use, plus
  random bit patterns;
* the device-generated f64 prefix (traces, period bits, arrivals, worker
  noise) == the host generators' replay of the same jobs (inputs.host_generate,
  itself pinned against numpy in tests/test_host.py), bit for bit, for the
  whole config-5 sweep and the small configs.
"""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2603_08417_b200 import _lib, engine, inputs, workloads

pytestmark = pytest.mark.gpu


def _device_libm(fn, xs):
    x = torch.from_numpy(xs).cuda()
    out = torch.empty_like(x)
    _lib.check(_lib.lib().otf_model_libm_dev(fn, x.data_ptr(), x.numel(), out.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream), "otf_model_libm_dev")
    return out.cpu().numpy()


def _glibc(fn, xs):
    out = np.empty_like(xs)
    assert oracle.lib().oracle_libm(fn, xs.ctypes.data, xs.size, out.ctypes.data) == 0
    return out


def test_device_libm_matches_glibc_1e8():
    rng = np.random.default_rng(2026)
    total = 0
    for chunk in range(8):
        n = 6_250_000
        u = rng.random(n)
        exp_args = np.concatenate([13.0 + 8.0 * u,                       # trace log-bandwidths
                                   -0.5 * (3.7 * u) ** 2,                # normal wedge test
                                   -7.7 * u,                             # exponential wedge test
                                   rng.integers(0, 2 ** 63, n // 4, dtype=np.int64).view(np.float64)])
        log_args = np.concatenate([-u,                                   # ziggurat tails: log1p(-U)
                                   -np.ldexp(u, -rng.integers(0, 60, n)),
                                   np.ldexp(u[:n // 4], rng.integers(-20, 80, n // 4))])
        for fn, xs in ((0, exp_args), (1, log_args)):
            xs = np.ascontiguousarray(xs)
            got, want = _device_libm(fn, xs), _glibc(fn, xs)
            same = (got.view(np.int64) == want.view(np.int64)) | (np.isnan(got) & np.isnan(want))
            bad = np.nonzero(~same)[0]
            assert bad.size == 0, (fn, xs[bad[:4]], got[bad[:4]], want[bad[:4]])
            total += xs.size
    assert total >= 100_000_000


def _check_prefix(cfgs):
    inp = inputs.build_inputs(cfgs, engine=_lib.ENGINE_WINDOWED, mode=_lib.MODE_HISTOGRAM, pin=True)
    db = engine.DeviceBatch(inp, pin=True)
    db.generate()
    torch.cuda.synchronize()
    got = db.f64[:inp.f64_dev].cpu().numpy()
    want = inputs.host_generate(inp)
    bad = np.nonzero(got.view(np.int64) != want.view(np.int64))[0]
    assert bad.size == 0, f"{bad.size} of {want.size} generated values differ (first at {bad[:5]})"
    # the host part of the pool reached the device unchanged
    assert np.array_equal(db.f64[inp.f64_dev:].cpu().numpy().view(np.int64), inp.f64.view(np.int64))
    return inp


def test_device_tables_config5_full_sweep():
    inp = _check_prefix(workloads.c5_sweep(seeds=range(1, 65)))
    kinds = [j.kind for j in inp.gen_jobs[:inputs.n_gen_jobs(inp)]]
    assert kinds.count(_lib.GEN_TRACE) == 64 and kinds.count(_lib.GEN_ARRIVALS) == 64
    assert kinds.count(_lib.GEN_NOISE) == 64


def test_device_tables_small_configs():
    cfgs = [workloads.c1(seed=s) for s in (1, 2, 3)] + [workloads.c2(seed=1), workloads.c3(seed=2, fraction=0.3)]
    cfgs += [workloads.c4(seed=5, clients=c, variant="TCPF") for c in (10, 300, 3000)]
    _check_prefix(cfgs)
