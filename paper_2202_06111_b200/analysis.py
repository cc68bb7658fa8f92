"""Non-leaving cells on the GPU (mirror of cg/analysis.py).

``non_leaving_mask`` returns the vertices with an infinite path.  The
reference obtains them as the reverse-reachability closure of nontrivial
SCCs (cg/analysis.py:120-161); libgis K3 computes the identical set as the
zero-out-degree peeling fixed point (tests/conftest.py:75-89) with forward
scan pointers and a vertex bitmap, in one cooperative kernel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as D
from .geometry import Covering
from .graph import SymbolicImage

__all__ = ["non_leaving", "non_leaving_mask", "non_leaving_dev", "retain"]


def non_leaving_dev(graph: SymbolicImage):
    """(keep uint8 device tensor, sweeps) for the whole graph on one GPU."""
    torch = D._torch()
    nv = graph.n_vertices
    keep = torch.zeros(nv, dtype=torch.uint8, device=D.device())
    rounds = C.c_int32(0)
    if nv == 0:
        return keep, 0
    indptr, indices = graph._dev()
    D.check(D.load_library().gis_prune(D.ctx(), D.ptr(indptr), D.ptr(indices), nv, D.ptr(keep),
                                       C.byref(rounds)), "non_leaving_mask")
    return keep, int(rounds.value)


def non_leaving_mask(graph: SymbolicImage, strict_largest: bool = False) -> np.ndarray:
    """Boolean mask of vertices that can reach a cycle (cg/analysis.py:120)."""
    if strict_largest:
        raise NotImplementedError(
            "strict_largest needs a GPU SCC decomposition (SURVEY.md section 8(f) rank 3); "
            "the default mode is the non-leaving set")
    if graph.n_vertices == 0:
        return np.zeros(0, dtype=bool)
    keep, _ = non_leaving_dev(graph)
    return keep.cpu().numpy().astype(bool)


def non_leaving(graph: SymbolicImage, strict_largest: bool = False) -> set:
    mask = non_leaving_mask(graph, strict_largest=strict_largest)
    return {graph.vertex_id(int(i)) for i in np.flatnonzero(mask)}


def retain(covering: Covering, keep) -> Covering:
    return covering.retain(keep)
