"""Where the config-2 e2e step's time goes beyond the device step: the
reference-facing sequence timed piece by piece (host clock, synchronised
after each piece), and the whole sequence unsynchronised.
  python tools/e2e_anatomy.py [reps]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_mask
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import build_graph_serial

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = config(2)
m = cfg.model
cov = Covering.uniform(m.X, cfg.initial_depth)
inputs = sample_inputs(m.U, cfg.input_counts)
pin = [torch.from_numpy(x.copy()).pin_memory() for x in (cov.depths, cov.bits, cov.lo, cov.hi)]


def piecewise():
    t = [time.perf_counter()]
    c2 = Covering(m.X, pin[0], pin[1], pin[2], pin[3], _sorted=True)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    idx = c2.build_index()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    g = build_graph_serial(c2, idx, m, inputs, cfg.image)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    mask = non_leaving_mask(g)
    t.append(time.perf_counter())
    return [(b - a) * 1e3 for a, b in zip(t, t[1:])]


def whole():
    t0 = time.perf_counter()
    c2 = Covering(m.X, pin[0], pin[1], pin[2], pin[3], _sorted=True)
    g = build_graph_serial(c2, c2.build_index(), m, inputs, cfg.image)
    mask = non_leaving_mask(g)
    return (time.perf_counter() - t0) * 1e3


for _ in range(3):
    piecewise(); whole()
pw = [piecewise() for _ in range(reps)]
wh = sorted(whole() for _ in range(reps))
names = ["covering_upload", "index", "graph_build", "prune_to_numpy"]
print(json.dumps({"piecewise_ms_median": {n: sorted(p[i] for p in pw)[reps // 2]
                                          for i, n in enumerate(names)},
                  "whole_ms_median": wh[reps // 2], "whole_ms_min": wh[0]}))
