"""Quick end-to-end GPU check against the oracle (development tool)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from oracle import gis_oracle as O
from paper_2202_06111_b200 import Covering, RunConfig, run, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import build_graph_serial
from paper_2202_06111_b200.image import batch_enclosures, sample_fractions
from paper_2202_06111_b200.adaptive import select_boundary_mask, select_neighborhood_mask
from paper_2202_06111_b200 import _device as D


def step(msg):
    print(f"== {msg}", flush=True)


step("smoke")
import __graft_entry__ as G
G.smoke()

step("enclosures pendulum rk4 vs oracle")
cfg = config(2)
m = cfg.model
rng = np.random.default_rng(0)
lo = rng.uniform(m.X.lo, m.X.hi - 0.01, (1000, 2))
hi = lo + rng.uniform(0.001, 0.01, (1000, 2))
frac = sample_fractions(cfg.image, 2)
ost = O.make_step(m.step.spec())
for u in ([-2.0], [0.4], [2.0]):
    a = batch_enclosures(m, lo, hi, np.array(u), cfg.image)
    b = O.enclosures(ost, lo, hi, np.array(u), frac, 0.1)
    rel = np.max(np.abs(a[0] - b[0]) / np.maximum(np.abs(b[0]), 1e-300))
    print(" u", u, "valid eq", np.array_equal(a[2], b[2]), "max rel lo", rel,
          "exact frac", np.mean(a[0] == b[0]))

step("config 1 run vs oracle")
t = time.time()
res = run(config(1))
print(" gpu run", time.time() - t, [(x.cells_before, x.cells_after, x.edges, x.boundary_cells)
                                    for x in res.metrics])
t = time.time()
c1 = config(1)
orr = O.run(c1.model.step.spec(), c1.model.X.lo, c1.model.X.hi, c1.model.U.lo, c1.model.U.hi,
            11, 4, sample_fractions(c1.image, 2), 0.1, initial_depth=12, prune="peel")
print(" oracle run", time.time() - t, [(x["cells_before"], x["cells_after"], x["edges"],
                                        x["boundary_cells"]) for x in orr["metrics"]])
print(" final equal:", np.array_equal(res.covering.bits, orr["cover"].bits)
      and np.array_equal(res.covering.depths, orr["cover"].depths),
      np.array_equal(res.covering.lo, orr["cover"].lo))

step("adaptive config 3 vs oracle")
t = time.time()
c3 = config(3)
res3 = run(c3)
print(" gpu", time.time() - t, len(res3.covering), [x.cells_after for x in res3.metrics])
t = time.time()
o3 = O.run(c3.model.step.spec(), c3.model.X.lo, c3.model.X.hi, c3.model.U.lo, c3.model.U.hi,
           21, 9, sample_fractions(c3.image, 2), 0.1, initial_depth=10, mode="adaptive",
           n_neighbors=3, prune="peel")
print(" oracle", time.time() - t, len(o3["cover"]), [x["cells_after"] for x in o3["metrics"]])
print(" final equal:", np.array_equal(res3.covering.bits, o3["cover"].bits))

step("config 2 timing")
c2 = config(2)
m2 = c2.model
cov = Covering.initial(m2.X)
for _ in range(20):
    cov = cov.subdivide(None)
inputs = sample_inputs(m2.U, 21)
idx = cov.build_index()
for it in range(3):
    torch.cuda.synchronize()
    t = time.time()
    g = build_graph_serial(cov, idx, m2, inputs, c2.image)
    torch.cuda.synchronize()
    t1 = time.time()
    keep, rounds = non_leaving_dev(g)
    torch.cuda.synchronize()
    t2 = time.time()
    print(f" build {t1 - t:.4f}s prune {t2 - t1:.4f}s E={g.edge_count} kept={int(keep.sum())} "
          f"sweeps={rounds}")
print("launches", D.launch_count())
