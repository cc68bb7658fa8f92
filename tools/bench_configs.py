"""Wall times of the BASELINE configurations through the public API.

  python tools/bench_configs.py [ids...]     (default 1 3 4 5)

Config 1/3/5: the whole run() (GIS wall time to the final covering).
Config 4: one build + prune pass of the 256^3 Lorenz grid (V = 16.7M).
Prints one JSON line per config."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import Covering, SpatialIndex, _device as D, run, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev
from paper_2202_06111_b200.configs import CONFIG_NAMES, config
from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows
from paper_2202_06111_b200.image import sample_fractions


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


def one_pass(rc):
    m = rc.model
    cov = Covering.initial(m.X)
    for _ in range(rc.initial_depth):
        cov = cov.subdivide(None)
    inputs = sample_inputs(m.U, rc.input_counts)

    def step():
        idx = SpatialIndex._dyadic(cov)
        ip, ix = build_graph_rows(cov, idx, m, inputs, rc.image)
        keep, sweeps = non_leaving_dev(SymbolicImage._from_device(cov, ip, ix))
        return int(ix.shape[0]), int(keep.sum()), sweeps
    t, (E, kept, sweeps) = timed(step, reps=2)
    S = len(sample_fractions(rc.image, m.n))
    I = len(cov) * len(inputs) * S
    return {"cells": len(cov), "edges": E, "kept": kept, "sweeps": sweeps, "seconds": t,
            "integrations": I, "integrations_per_s": I / t}


def full_run(rc):
    t, res = timed(lambda: run(rc), reps=2)
    S = len(sample_fractions(rc.image, rc.model.n))
    U = len(sample_inputs(rc.model.U, rc.input_counts))
    I = sum(mm.cells_before for mm in res.metrics) * U * S
    return {"seconds": t, "final_cells": len(res.covering), "integrations": I,
            "metrics": [(mm.cells_before, mm.cells_after, mm.edges) for mm in res.metrics],
            "containment_ok": res.containment_ok}


if __name__ == "__main__":
    ids = [int(a) for a in sys.argv[1:]] or [1, 3, 4, 5]
    for i in ids:
        rc = config(i)
        out = one_pass(rc) if i in (2, 4) else full_run(rc)
        D.enable_timing(True)
        D.phase_times()
        D.integrations()
        one_pass(rc) if i in (2, 4) else run(rc)
        phases = {k: round(v[0], 3) for k, v in D.phase_times().items()}
        images, ints = D.integrations()  # K1 work of the timed pass / run
        D.enable_timing(False)
        print(json.dumps({"config": i, "name": CONFIG_NAMES[i], **out, "phases_ms": phases,
                          "k1_images": images, "k1_integrations_run": ints}),
              flush=True)
