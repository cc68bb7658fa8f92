"""Timings of the on-demand analysis kernels (K6 SCC, strict mode, reverse
CSR, edge-list formatting) on full-size BASELINE graphs.

  python tools/bench_analysis.py [config ids...]   (default 2 4)
Prints one JSON line per config (ms, CUDA events on the current stream)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev, non_leaving_scc_dev, scc_dev
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.graph import build_graph_serial


def timed(fn, reps=3):
    fn()
    out = None
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), out


for cid in [int(x) for x in sys.argv[1:]] or [2, 4]:
    rc = config(cid)
    m = rc.model
    if rc.initial_grid is not None:
        cov = Covering.grid(m.X, rc.initial_grid)
    else:
        cov = Covering.initial(m.X)
        for _ in range(rc.initial_depth):
            cov = cov.subdivide(None)
    g = build_graph_serial(cov, cov.build_index(), m, sample_inputs(m.U, rc.input_counts),
                           rc.image)
    t_peel, (keep, sweeps) = timed(lambda: non_leaving_dev(g))
    t_scc, (comp, sizes, nontriv, ncomp, stats) = timed(lambda: scc_dev(g))
    t_lit, _ = timed(lambda: non_leaving_scc_dev(g, strict_largest=False))
    t_strict, _ = timed(lambda: non_leaving_scc_dev(g, strict_largest=True))
    g._rev = None
    t_rev, _ = timed(lambda: (setattr(g, "_rev", None), g.reverse_csr())[1], reps=1)
    t_fmt, _ = timed(lambda: sum(len(c) for c in g._edge_list_chunks()), reps=1)
    print(json.dumps({"config": cid, "V": len(cov), "E": g.edge_count,
                      "prune_peel_ms": t_peel, "sweeps": sweeps, "scc_ms": t_scc,
                      "components": ncomp, "scc_outer_rounds": stats,
                      "non_leaving_literal_ms": t_lit, "strict_largest_ms": t_strict,
                      "reverse_csr_sorted_to_host_ms": t_rev,
                      "edge_list_format_to_host_ms": t_fmt}), flush=True)
