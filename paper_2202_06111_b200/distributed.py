"""Multi-GPU sharding of the build + prune (one process per GPU).

Cells are partitioned into contiguous CellId ranges aligned to 32-vertex
bitmap words -- the reference's contiguous ownership model
(cg/graph.py:306-345, merge_subgraphs ownership :237-270).  The covering is
replicated; each rank integrates and builds the CSR rows it owns (targets
are global indices, so rows need no exchange).  Pruning runs the forward
peeling sweep on owned rows; after every sweep the ranks all-gather the
vertex bitmap (each rank contributes its owned words) and all-reduce the
number of deletions; the loop ends when a sweep deletes nothing anywhere.

The per-rank sweep is pluggable so the exchange protocol can be exercised
on CPU with the gloo backend (tests/test_distributed.py); the product sweep
is libgis ``gis_peel_sweep``.
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _device as D

__all__ = ["word_partition", "owned_range", "sharded_peel", "build_and_prune_sharded",
           "sharded_boundary", "sharded_neighborhood", "sharded_containment", "world"]


def world():
    """(rank, world_size) of the default process group, (0, 1) without one."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def word_partition(V: int, size: int) -> int:
    """Bitmap words per rank (equal slices for the all-gather)."""
    nwords = (V + 31) // 32
    return max(1, -(-nwords // size))


def owned_range(V: int, rank: int, size: int):
    """[begin, end) vertices owned by rank: word-aligned contiguous ranges."""
    W = word_partition(V, size)
    b = min(V, rank * W * 32)
    e = min(V, (rank + 1) * W * 32)
    return b, e


def _allgather_words(full, W, rank, size, group=None):
    import torch
    import torch.distributed as dist

    mine = full[rank * W:(rank + 1) * W].clone()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(size)]
        dist.all_gather(parts, mine, group=group)
        full.copy_(torch.cat(parts))


def _device_sweep(indptr_local, indices, b, e, alive_words, ptr):
    deaths = C.c_int64()
    D.check(D.load_library().gis_peel_sweep(D.ctx(), D.ptr(indptr_local), D.ptr(indices), b, e,
                                            D.ptr(alive_words), D.ptr(ptr), C.byref(deaths)),
            "peel_sweep")
    return int(deaths.value)


def sharded_peel(indptr_local, indices, V: int, rank: int, size: int,
                 sweep: Optional[Callable] = None, init: Optional[Callable] = None, group=None,
                 check_every: int = 4):
    """Peeling fixed point with owned rows [b, e) on this rank.

    Every sweep is followed by the bitmap all-gather; the deletion counts of
    ``check_every`` sweeps are summed in one all-reduce, and the host reads
    that sum (the only host synchronisation) to stop.  Sweeps past the fixed
    point delete nothing, so checking in batches changes the sweep count,
    not the result.

    Returns (alive_words int32 tensor of size*W words -- the global bitmap,
    sweeps).  ``sweep(indptr_local, indices, b, e, alive_words, ptr) -> deaths``
    and ``init(indptr_local, V, b, e, alive_words, ptr)`` default to libgis."""
    import torch
    import torch.distributed as dist

    b, e = owned_range(V, rank, size)
    W = word_partition(V, size)
    dev = indptr_local.device
    full = torch.zeros(size * W, dtype=torch.int32, device=dev)
    ptr = torch.empty(max(e - b, 1), dtype=torch.int64, device=dev)
    if init is None:
        D.check(D.load_library().gis_peel_init(D.ctx(), D.ptr(indptr_local), V, b, e,
                                               D.ptr(full), D.ptr(ptr)), "peel_init")
    else:
        init(indptr_local, V, b, e, full, ptr)
    rounds = 0
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lib = D.load_library() if sweep is None else None
    while True:
        cnt.zero_()
        for _ in range(max(1, int(check_every))):
            if sweep is None:  # device sweep: deletions accumulate on the device
                D.check(lib.gis_peel_sweep_acc(D.ctx(), D.ptr(indptr_local), D.ptr(indices), b,
                                               e, D.ptr(full), D.ptr(ptr), D.ptr(cnt)),
                        "peel_sweep")
            else:
                cnt += sweep(indptr_local, indices, b, e, full, ptr)
            rounds += 1
            _allgather_words(full, W, rank, size, group)
        dist.all_reduce(cnt, group=group)
        if int(cnt.item()) == 0:
            return full, rounds


def build_and_prune_sharded(covering, index, model, inputs, cfg, group=None):
    """Build owned rows and prune cooperatively; returns (keep uint8 device
    tensor over all cells, total edges, sweeps)."""
    import torch
    import torch.distributed as dist

    from .graph import build_graph_rows

    rank, size = world()
    V = len(covering)
    b, e = owned_range(V, rank, size)
    indptr, indices = build_graph_rows(covering, index, model, inputs, cfg, b, e)
    full, rounds = sharded_peel(indptr, indices, V, rank, size, group=group)
    keep = torch.empty(V, dtype=torch.uint8, device=D.device())
    if V:
        D.check(D.load_library().gis_bitmap_to_mask(D.ctx(), D.ptr(full), V, D.ptr(keep)))
    ne = torch.tensor([indices.shape[0]], dtype=torch.int64, device=D.device())
    dist.all_reduce(ne, group=group)
    return keep, int(ne.item()), rounds


# -- adaptive selection and containment, sharded by owned cells ---------------
# The covering is replicated; each rank evaluates the probes / k-NN queries /
# containment of its owned cells and the ranks combine: boundary and
# neighbourhood masks by a MAX all-reduce (a logical OR over uint8), the
# containment defect by an all-gather of one scalar per rank.

def sharded_boundary(covering, index, delta: float, include_face_points=False, group=None):
    """select_boundary_mask (cg/adaptive.py:93-123) over all cells, each rank
    probing its owned range; uint8 device mask."""
    import torch
    import torch.distributed as dist

    rank, size = world()
    V = len(covering)
    out = torch.zeros(V, dtype=torch.uint8, device=D.device())
    if V:
        b, e = owned_range(V, rank, size)
        D.check(D.load_library().gis_select_boundary_range(
            D.ctx(), index._h, D.ptr(covering._lo), D.ptr(covering._hi), V, b, e, float(delta),
            int(bool(include_face_points)), D.ptr(out)), "select_boundary")
        dist.all_reduce(out, op=dist.ReduceOp.MAX, group=group)
    return out


def sharded_neighborhood(index, boundary, n_neighbors: int, group=None):
    """select_neighborhood_mask (cg/adaptive.py:136-150): each rank runs the
    k-NN of the boundary cells it owns, the marks are OR-reduced, then the
    boundary is removed; uint8 device mask."""
    import torch
    import torch.distributed as dist

    rank, size = world()
    V = index.size
    out = torch.zeros(V, dtype=torch.uint8, device=D.device())
    if V and n_neighbors > 0:
        b, e = owned_range(V, rank, size)
        lib = D.load_library()
        D.check(lib.gis_select_neighborhood_range(
            D.ctx(), index._h, D.ptr(index._lo), D.ptr(index._hi), V, D.ptr(boundary), b, e,
            int(n_neighbors), 0, D.ptr(out)), "select_neighborhood")
        dist.all_reduce(out, op=dist.ReduceOp.MAX, group=group)
        D.check(lib.gis_mask_andnot(D.ctx(), D.ptr(out), D.ptr(boundary), V),
                "select_neighborhood")
    return out


def sharded_containment(new_cov, prev_cov, prev_index, group=None) -> float:
    """engine._containment_defect (cg/engine.py:114-130) over the new cells,
    each rank its owned range; NaN if any rank saw a negative coverage."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    rank, size = world()
    V = len(new_cov)
    d = C.c_double(0.0)
    if V:
        b, e = owned_range(V, rank, size)
        D.check(D.load_library().gis_containment_defect_range(
            D.ctx(), prev_index._h, D.ptr(prev_cov._lo), D.ptr(prev_cov._hi), len(prev_cov),
            D.ptr(new_cov._lo), D.ptr(new_cov._hi), V, b, e, C.byref(d)), "containment")
    mine = torch.tensor([d.value], dtype=torch.float64, device=D.device())
    parts = [torch.empty_like(mine) for _ in range(size)]
    dist.all_gather(parts, mine, group=group)
    vals = torch.cat(parts).cpu().numpy()
    return float("nan") if np.isnan(vals).any() else float(vals.max())
