"""Known-answer vectors for the per-client model functions, from the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_model_kat.py

Writes tests/golden/model_kat.json:
* completion_time: BandwidthTrace(samples).completion_time(start, nbytes)
  (netem.py:77-118) for the reference's own test traces (tests/test_netem.py)
  plus 400 random looping traces of 1-12 pieces, starts and sizes;
* select_quality: select_quality(level, cur, est, ladder, ClientConfig())
  (client.py:134-146) on the reference test ladder's band edges plus 400
  random points;
* PlayerBuffer.advance / on_segment (client.py:91-121): 200 random sequences
  with the state after every step.
The engine's restatement (csrc/otf_model.cuh) must reproduce every value
bit-for-bit (tests/test_model_kat.py on the host build, -m gpu on the device).
"""

from __future__ import annotations

import json
import math
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from otfstream.client import BufferConfig, ClientConfig, PlayerBuffer, select_quality  # noqa: E402
from otfstream.netem import BandwidthTrace  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
LADDER = [(1, 2_000_000), (2, 3_500_000), (3, 6_000_000), (4, 10_000_000), (5, 16_000_000)]


def trace_doc(samples):
    tr = BandwidthTrace(samples)
    return {"samples": samples, "starts": tr._starts, "values": tr._values, "period": tr.period,
            "pbits": tr._period_bits}


def main():
    rnd = random.Random(2603)
    ct = []
    fixed = [  # tests/test_netem.py:28-53,74-86
        ([(0.0, 8e6)], [(0.0, 1_000_000)]),
        ([(0.0, 8e6), (0.5, 0.0), (1.5, 8e6)], [(0.0, 1_000_000)]),
        ([(0.0, 0.0)], [(0.0, 1)]),
        ([(0.0, 8e6), (1.0, 0.0)], [(0.0, 10_000_000 // 8)]),
        ([(0.0, 5e6), (2.0, 1e6), (3.0, 20e6)], [(0.7, n) for n in range(100_000, 2_000_000, 100_000)]),
    ]
    for samples, queries in fixed:
        tr = BandwidthTrace(samples)
        doc = trace_doc(samples)
        doc["queries"] = [[s, n, tr.completion_time(s, n)] for s, n in queries]
        ct.append(doc)
    for _ in range(400):
        samples, t = [], round(rnd.uniform(0.0, 0.5), 3)
        for _ in range(rnd.randint(1, 12)):
            samples.append((t, rnd.choice([0.0, 2e6, 8e6, 17e6, 40e6, rnd.uniform(1e6, 5e7)])))
            t += round(rnd.uniform(0.05, 3.0), 3)
        if all(bw == 0 for _, bw in samples):
            samples[0] = (samples[0][0], 8e6)
        tr = BandwidthTrace(samples)
        doc = trace_doc(samples)
        doc["queries"] = []
        for _ in range(5):
            s = rnd.choice([0.0, round(rnd.uniform(0, 40), 6), rnd.uniform(0, 600)])
            n = rnd.choice([0, 1, rnd.randint(100, 5_000_000), rnd.randint(10_000_000, 80_000_000)])
            doc["queries"].append([s, n, tr.completion_time(s, n)])
        ct.append(doc)

    cfg = ClientConfig()
    sq = []
    points = [(1.5, 3, 100e6), (5.0, 3, 100e6), (5.0, 1, 100e6), (10.0, 3, 1.5 * LADDER[3][1]),
              (10.0, 3, 1.1 * LADDER[3][1]), (10.0, 5, 1e12), (10.0, 2, None), (2.0, 3, None), (8.0, 3, 0.0)]
    for _ in range(400):
        points.append((rnd.uniform(0, 14), rnd.randint(1, 5), rnd.choice([None, rnd.uniform(1e6, 2e8)])))
    for level, cur, est in points:
        sq.append([level, cur, est, select_quality(level, cur, est, dict(LADDER), cfg)])

    # PlayerBuffer (client.py:74-121): random advance / on_segment sequences
    phases = {"startup": 0, "playing": 1, "stalled": 2, "finished": 3}
    bufs = []
    bc = BufferConfig()
    for _ in range(200):
        t = rnd.uniform(0, 100)
        b = PlayerBuffer(bc, t)
        seq = {"t0": t, "ops": []}
        for _ in range(rnd.randint(1, 40)):
            t += rnd.choice([0.0, rnd.uniform(0, 0.5), rnd.uniform(0, 3), rnd.uniform(0, 12)])
            if rnd.random() < 0.5:
                dur = rnd.choice([1.0, 2.0, rnd.uniform(0.1, 4.0)])
                b.on_segment(t, dur)
                op = [1, t, dur]
            else:
                b.advance(t)
                op = [0, t, 0.0]
            seq["ops"].append(op + [b.level, phases[b.phase], b.stall_events, b.stall_time,
                                    b.started_at if b.started_at is not None else float("nan"), b.last_sync])
        bufs.append(seq)

    out = {"ladder": [b for _, b in LADDER],
           "client": {"panic": cfg.buffer.panic_s, "safe": cfg.buffer.safe_s, "headroom": cfg.headroom},
           "buffer": {"startup": bc.startup_s, "resume": bc.resume_s, "sequences": bufs},
           "completion_time": ct, "select_quality": sq}
    with open(os.path.join(HERE, "model_kat.json"), "w") as fh:
        json.dump(out, fh, allow_nan=True)
    print("wrote", sum(len(d["queries"]) for d in ct), "completion_time and", len(sq), "select_quality vectors")


if __name__ == "__main__":
    main()
