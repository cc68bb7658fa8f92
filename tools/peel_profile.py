"""Per-sweep anatomy of the K3 prune on a BASELINE config (diagnostic).

  python tools/peel_profile.py [config]      (default 2)

Builds the config's first graph, then runs the peel one sweep per launch
(gis_peel_init + gis_peel_sweep, wide scan state) with CUDA events around
each sweep, and reads the scan state between sweeps: per sweep the deaths,
the vertices whose current target had died (row walks), the row entries
walked (offset advance) and the longest walk.  Also times gis_prune (the
cooperative kernel) on the same graph.  Prints one JSON line per sweep."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, SpatialIndex, _device as D, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = config(cid)
m = cfg.model
if cfg.initial_grid is not None:
    cov = Covering.grid(m.X, cfg.initial_grid)
else:
    cov = Covering.initial(m.X)
    for _ in range(cfg.initial_depth):
        cov = cov.subdivide(None)
inputs = sample_inputs(m.U, cfg.input_counts)
index = SpatialIndex._dyadic(cov)
ip, ix = build_graph_rows(cov, index, m, inputs, cfg.image)
g = SymbolicImage._from_device(cov, ip, ix)
V = len(cov)
torch.cuda.synchronize()

# the cooperative prune, timed
for _ in range(3):
    keep, sweeps = non_leaving_dev(g)
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    keep, sweeps = non_leaving_dev(g)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"config": cid, "V": V, "E": int(ix.shape[0]), "kept": int(keep.sum()),
                  "coop_sweeps": sweeps, "coop_ms": sorted(ts)}), flush=True)

lib, ctx = D.load_library(), D.ctx()
words = (V + 31) // 32
alive = torch.empty(words, dtype=torch.int32, device="cuda")
state = torch.empty(V, dtype=torch.int64, device="cuda")
D.check(lib.gis_peel_init(ctx, D.ptr(ip), V, 0, V, D.ptr(alive), D.ptr(state)), "init")
deg = (ip[1:] - ip[:-1])
deaths = C.c_int64(0)
k = 0
total = 0.0
while True:
    prev = state.clone()
    bits_before = alive.clone()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    D.check(lib.gis_peel_sweep(ctx, D.ptr(ip), D.ptr(ix), 0, V, D.ptr(alive), D.ptr(state),
                               C.byref(deaths)), "sweep")
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    total += ms
    off0 = torch.where(prev == -2 * 2**32, torch.zeros_like(prev), (prev & 0xffffffff) + 1)
    dead_now = (state >> 32) == -1
    off1 = torch.where(dead_now, deg, state & 0xffffffff)
    was_alive = ((bits_before.view(torch.int32).to(torch.int64) & 0xffffffff).repeat_interleave(32)[:V]
                 >> (torch.arange(V, device="cuda") & 31)) & 1
    moved = (off1 != (prev & 0xffffffff)) & (was_alive == 1)
    walk = torch.where(moved, off1 - off0 + 1, torch.zeros_like(off1))
    print(json.dumps({"sweep": k, "ms": round(ms, 4), "deaths": int(deaths.value),
                      "walkers": int(moved.sum()), "entries_walked": int(walk.sum()),
                      "max_walk": int(walk.max())}), flush=True)
    k += 1
    if deaths.value == 0 or k > 500:
        break
print(json.dumps({"sweeps": k, "sum_ms": round(total, 3)}))
