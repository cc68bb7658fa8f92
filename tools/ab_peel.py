"""A/B of K3 builds: python tools/ab_peel.py CONFIG [reps]; the library is
chosen by GIS_LIB_VARIANT (build.py --variant).  Prints the variant, the
sweep count, a digest of the keep mask and the sorted gis_prune times."""
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, SpatialIndex, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = config(cid)
m = cfg.model
if cfg.initial_grid is not None:
    cov = Covering.grid(m.X, cfg.initial_grid)
else:
    cov = Covering.initial(m.X)
    for _ in range(cfg.initial_depth):
        cov = cov.subdivide(None)
inputs = sample_inputs(m.U, cfg.input_counts)
ip, ix = build_graph_rows(cov, SpatialIndex._dyadic(cov), m, inputs, cfg.image)
g = SymbolicImage._from_device(cov, ip, ix)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    keep, sweeps = non_leaving_dev(g)
ts = []
for _ in range(reps):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    keep, sweeps = non_leaving_dev(g)
    b.record()
    b.synchronize()
    ts.append(round(a.elapsed_time(b), 4))
h = hashlib.sha256(keep.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps({"variant": os.environ.get("GIS_LIB_VARIANT", "default"), "config": cid,
                  "sweeps": sweeps, "keep": h, "kept": int(keep.sum()),
                  "median_ms": sorted(ts)[len(ts) // 2], "ms": sorted(ts)}), flush=True)
