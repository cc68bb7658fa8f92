"""A/B of K2 builds (GIS_LIB_VARIANT): config 2's graph build (phase times,
digest of the CSR) and the whole runs of configs 1 and 3 (2-D adaptive).
  python tools/ab_rows.py [reps]"""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, SpatialIndex, _device as D, run, sample_inputs
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import build_graph_rows

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
var = os.environ.get("GIS_LIB_VARIANT", "default")
cfg = config(2)
m = cfg.model
cov = Covering.initial(m.X)
for _ in range(cfg.initial_depth):
    cov = cov.subdivide(None)
inputs = sample_inputs(m.U, cfg.input_counts)
idx = SpatialIndex._dyadic(cov)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ip, ix = build_graph_rows(cov, idx, m, inputs, cfg.image)
D.enable_timing(True)
rows = []
for _ in range(reps):
    flush.fill_(1)
    D.phase_times()
    ip, ix = build_graph_rows(cov, idx, m, inputs, cfg.image)
    torch.cuda.synchronize()
    ph = D.phase_times()
    rows.append(ph["csr_rows"][0])
D.enable_timing(False)
h = hashlib.sha256(ip.cpu().numpy().tobytes() + ix.cpu().numpy().tobytes()).hexdigest()[:16]
out = {"variant": var, "config": 2, "E": int(ix.shape[0]), "csr": h,
       "rows_ms_median": sorted(rows)[len(rows) // 2], "rows_ms": sorted(rows)[:3]}
for cid in (1, 3):
    res = run(config(cid))
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run(config(cid))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[f"run{cid}_s"] = min(ts)
    out[f"run{cid}_cells"] = hashlib.sha256(res.covering.bits.tobytes()
                                            + res.covering.depths.tobytes()).hexdigest()[:16]
print(json.dumps(out), flush=True)
