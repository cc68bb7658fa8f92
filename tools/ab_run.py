"""A/B of libgis builds (GIS_LIB_VARIANT) on a whole run(): min wall of 3
warm runs, per-phase times of one run, digest of the final covering.
  python tools/ab_run.py [config]     (default 5)"""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import _device as D, run
from paper_2202_06111_b200.configs import config

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
res = run(config(cid))
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run(config(cid))
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
D.enable_timing(True)
D.phase_times()
res = run(config(cid))
torch.cuda.synchronize()
ph = {k: round(v[0], 3) for k, v in D.phase_times().items()}
D.enable_timing(False)
h = hashlib.sha256(res.covering.bits.tobytes() + res.covering.depths.tobytes()).hexdigest()[:16]
print(json.dumps({"variant": os.environ.get("GIS_LIB_VARIANT", "default"), "config": cid,
                  "wall_s_min": min(ts), "phases_ms": ph, "cells": len(res.covering),
                  "covering": h}), flush=True)
