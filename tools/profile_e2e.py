"""Stage breakdown of bench.py's e2e path (config 2) and of run(config(2)).

Each stage is bracketed by torch.cuda.synchronize() so the host clock sees
it whole; prints one JSON line per repetition.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, run, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_mask
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import build_graph_serial

cfg = config(2)
m = cfg.model
inputs = sample_inputs(m.U, cfg.input_counts)
cov = Covering.initial(m.X)
for _ in range(cfg.initial_depth):
    cov = cov.subdivide(None)
pin = [torch.from_numpy(x.copy()).pin_memory() for x in (cov.depths, cov.bits, cov.lo, cov.hi)]


def stamp(t, key, acc):
    torch.cuda.synchronize()
    now = time.perf_counter()
    acc[key] = round((now - t) * 1e3, 3)
    return now


flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
c2 = g = None
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    flush.fill_(1)
    acc = {}
    torch.cuda.synchronize()
    t = t0 = time.perf_counter()
    c2 = Covering(m.X, pin[0], pin[1], pin[2], pin[3], _sorted=True)
    t = stamp(t, "covering_h2d", acc)
    idx = c2.build_index()
    t = stamp(t, "index", acc)
    g = build_graph_serial(c2, idx, m, inputs, cfg.image)
    t = stamp(t, "build", acc)
    mask = non_leaving_mask(g)
    t = stamp(t, "prune_d2h", acc)
    acc["total"] = round((t - t0) * 1e3, 3)
    print(json.dumps({"rep": rep, "e2e_ms": acc}), flush=True)

for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run(cfg)
    torch.cuda.synchronize()
    print(json.dumps({"rep": rep, "run_config2_s": round(time.perf_counter() - t0, 4),
                      "final": len(res.covering)}), flush=True)
