"""Timing of the pruning variants on BASELINE config 2's full graph, one GPU:
gis_prune (single-GPU cooperative kernel), the fused peer-memory protocol
with R ranks emulated in one launch (gis_peel_p2p, rank = -1), and a 1-rank
NCCL group through distributed.build_and_prune_sharded's two exchanges
(fused gis_peel_p2p vs sweep kernel + NCCL all-gather per sweep)."""
import json
import os
import socket
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from paper_2202_06111_b200 import Covering, sample_inputs
from paper_2202_06111_b200.analysis import non_leaving_dev
from paper_2202_06111_b200.configs import config
from paper_2202_06111_b200.distributed import emulated_fused_peel, fused_peel, sharded_peel
from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


cfg = config(2)
m = cfg.model
cov = Covering.initial(m.X)
for _ in range(cfg.initial_depth):
    cov = cov.subdivide(None)
idx = cov.build_index()
ip, ix = build_graph_rows(cov, idx, m, sample_inputs(m.U, cfg.input_counts), cfg.image)
V = len(cov)
g = SymbolicImage._from_device(cov, ip, ix)
out = {"V": V, "E": int(ix.shape[0])}
out["gis_prune_ms"] = timed(lambda: non_leaving_dev(g))
for R in (1, 2, 4, 8):
    out[f"fused_emulated_R{R}_ms"] = timed(lambda: emulated_fused_peel(ip, ix, V, R))
with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
out["nccl1_fused_ms"] = timed(lambda: fused_peel(ip, ix, V))
out["nccl1_allgather_ms"] = timed(lambda: sharded_peel(ip, ix, V, 0, 1))
from paper_2202_06111_b200.distributed import release_peer_bitmaps  # noqa: E402

release_peer_bitmaps()
dist.destroy_process_group()
print(json.dumps(out))
