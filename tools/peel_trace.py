"""Sweep timeline of the K3 cooperative prune (diagnostics build):
  python paper_2202_06111_b200/build.py --variant=trace -DGIS_PEEL_TRACE
  GIS_LIB_VARIANT=trace python tools/peel_trace.py [config]
Per sweep: start (previous barrier exit), the blocks' finish times
(median / p90 / max, microseconds from the sweep's start) and the barrier
exit."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
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
ip, ix = build_graph_rows(cov, SpatialIndex._dyadic(cov), m, inputs, cfg.image)
g = SymbolicImage._from_device(cov, ip, ix)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = D.load_library()
for rep in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    keep, sweeps = non_leaving_dev(g)
    torch.cuda.synchronize()
tr = np.zeros((2, 64, 1024), dtype=np.uint64)
t0 = C.c_uint64(0)
lib.gis_debug_peel_trace(tr.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(t0))
start = int(t0.value)
for r in range(sweeps):
    row = tr[0, r].astype(np.int64)
    st = tr[1, r].astype(np.int64)
    ok = row[1:] > 0
    fin = row[1:][ok] - start
    beg = st[1:][ok] - start
    dur = fin - beg
    print(json.dumps({"sweep": r,
                      "start_med_us": round(float(np.median(beg)) / 1e3, 2),
                      "start_max_us": round(float(beg.max()) / 1e3, 2),
                      "dur_med_us": round(float(np.median(dur)) / 1e3, 2),
                      "dur_p99_us": round(float(np.percentile(dur, 99)) / 1e3, 2),
                      "dur_max_us": round(float(dur.max()) / 1e3, 2),
                      "slowest_block": int(np.argmax(dur)),
                      "fin_max_us": round(float(fin.max()) / 1e3, 2),
                      "sync_exit_us": round((int(row[0]) - start) / 1e3, 2)}))
    start = int(row[0])
