"""A/B of box reuse on a whole adaptive run: python tools/ab_memo.py CONFIG [reps]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import _device as D, run
from paper_2202_06111_b200.configs import config

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for flag in ("0", "1", "0", "1"):
    os.environ["GIS_BOX_MEMO"] = flag
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run(config(cid))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    D.enable_timing(True)
    D.phase_times()
    D.integrations()
    t0 = time.perf_counter()
    res = run(config(cid))
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
    ph = {k: round(v[0], 2) for k, v in D.phase_times().items()}
    D.enable_timing(False)
    print("memo", flag, "walls", [round(t, 4) for t in ts], "timed", round(tt, 4),
          "phases", ph, "k1", D.integrations(),
          [(m.t_subdivide_ms, m.t_build_ms, m.t_analyze_ms) for m in res.metrics], flush=True)
