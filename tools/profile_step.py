"""One warm config-2 build + prune step (target for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, SpatialIndex, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows

cfg = config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
m = cfg.model
if cfg.initial_grid is not None:
    cov = Covering.grid(m.X, cfg.initial_grid)
else:
    cov = Covering.initial(m.X)
    for _ in range(cfg.initial_depth):
        cov = cov.subdivide(None)
inputs = sample_inputs(m.U, cfg.input_counts)
for it in range(2):
    index = SpatialIndex._dyadic(cov)
    ip, ix = build_graph_rows(cov, index, m, inputs, cfg.image)
    keep, sweeps = non_leaving_dev(SymbolicImage._from_device(cov, ip, ix))
    torch.cuda.synchronize()
    print("step", it, "E", ix.shape[0], "kept", int(keep.sum()), "sweeps", sweeps, flush=True)
