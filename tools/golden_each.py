"""Run each golden fixture alone on the windowed engine (debug helper: finds a hanging/failing case)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import parity
if len(sys.argv) > 1:
    from paper_2603_08417_b200 import engine
    from paper_2603_08417_b200.config import ExperimentConfig
    name = sys.argv[1]
    _, meta = parity.load_golden(name)
    cfg = ExperimentConfig.from_dict(meta["config"])
    cfg.popularity = meta.get("popularity", cfg.popularity)
    r = engine.run_batch([cfg], mode="records", engine="windowed", device="cuda:0")[0]
    print(name, "ok", r.engine, len(r.arrays["req_id"]), flush=True)
else:
    for name in parity.golden_names():
        rc = subprocess.run([sys.executable, __file__, name], timeout=None, capture_output=True, text=True) if False else \
            subprocess.run(["timeout", "25", sys.executable, __file__, name], capture_output=True, text=True)
        print(name, "rc", rc.returncode, rc.stdout.strip()[-80:], rc.stderr.strip()[-200:] if rc.returncode else "", flush=True)
