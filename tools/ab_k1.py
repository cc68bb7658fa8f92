"""A/B of libgis builds (GIS_LIB_VARIANT): per-phase times (enclose = K1
with its corner kernels, csr_rows = K2 rows, csr_aux) of one graph build of
configs 2 and 4 and of config 5's first iteration, with a digest of the CSR.
  python tools/ab_k1.py [reps]"""
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, SpatialIndex, _device as D, sample_inputs
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import build_graph_rows

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = {"variant": os.environ.get("GIS_LIB_VARIANT", "default")}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for cid in (2, 4, 5):
    cfg = config(cid)
    m = cfg.model
    if cfg.initial_grid is not None:
        cov = Covering.grid(m.X, cfg.initial_grid)
    else:
        cov = Covering.uniform(m.X, cfg.initial_depth)
    inputs = sample_inputs(m.U, cfg.input_counts)
    idx = SpatialIndex._dyadic(cov)
    ip, ix = build_graph_rows(cov, idx, m, inputs, cfg.image)
    D.enable_timing(True)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        D.phase_times()
        ip, ix = build_graph_rows(cov, idx, m, inputs, cfg.image)
        torch.cuda.synchronize()
        ph = D.phase_times()
        ts.append((ph["enclose"][0], ph["csr_rows"][0], ph["csr_aux"][0]))
    D.enable_timing(False)
    h = hashlib.sha256(ip.cpu().numpy().tobytes() + ix.cpu().numpy().tobytes()).hexdigest()[:16]
    for i, name in enumerate(("enclose", "rows", "aux")):
        out[f"c{cid}_{name}_ms"] = sorted(t[i] for t in ts)[len(ts) // 2]
    out[f"c{cid}_csr"] = h
    del ip, ix
print(json.dumps(out), flush=True)
