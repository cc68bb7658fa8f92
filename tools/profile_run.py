"""One warm engine run() of a BASELINE config (target for ncu launch lists):
python tools/profile_run.py CONFIG [runs]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2202_06111_b200 import run
from paper_2202_06111_b200.configs import config

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    res = run(config(cid))
    torch.cuda.synchronize()
    print("run", i, [(m.cells_before, m.cells_after, m.edges) for m in res.metrics], flush=True)
