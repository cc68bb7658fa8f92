"""Graph analysis on the GPU (mirror of cg/analysis.py).

``non_leaving_mask`` returns the vertices with an infinite path.  The
reference obtains them as the reverse-reachability closure of nontrivial
SCCs (cg/analysis.py:120-161); libgis K3 computes the identical set as the
zero-out-degree peeling fixed point (tests/conftest.py:75-89) with forward
scan pointers and a vertex bitmap, in one cooperative kernel.

``strongly_connected_components`` and the ``strict_largest`` mode run libgis
K6 (csrc/gis_scc.cu: trim + colour propagation + backward marking in one
cooperative kernel) in place of the reference's pure-Python Tarjan
(cg/analysis.py:51-117).  The partition is the same; component ids are
numbered by each component's smallest vertex instead of Tarjan's DFS pop
order (the reference's tests pin the partition: tests/test_analysis.py:21-63).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as D
from .geometry import Covering
from .graph import SymbolicImage

__all__ = ["SccResult", "strongly_connected_components", "non_leaving", "non_leaving_mask",
           "non_leaving_dev", "non_leaving_scc_dev", "retain"]


@dataclass
class SccResult:
    """SCC decomposition (cg/analysis.py:30-48): per-vertex component id
    plus per-component data."""

    component_of: np.ndarray  # (V,) component id per vertex
    n_components: int
    nontrivial: np.ndarray    # (C,) True when the component contains a cycle

    def members(self) -> list:
        """Member vertex indices per component id."""
        if self.n_components == 0:
            return []
        order = np.argsort(self.component_of, kind="stable")
        comps = self.component_of[order]
        bounds = np.flatnonzero(np.diff(comps)) + 1
        return [np.sort(part) for part in np.split(order, bounds)]

    def sizes(self) -> np.ndarray:
        return np.bincount(self.component_of, minlength=self.n_components)


def scc_dev(graph: SymbolicImage):
    """(comp int64, sizes int64, nontrivial uint8 device tensors, n_comp,
    (outer iterations, grid rounds)) from libgis K6."""
    torch = D._torch()
    nv = graph.n_vertices
    dev = D.device()
    comp = torch.empty(nv, dtype=torch.int64, device=dev)
    sizes = torch.empty(max(nv, 1), dtype=torch.int64, device=dev)
    nontriv = torch.zeros(max(nv, 1), dtype=torch.uint8, device=dev)
    ncomp = C.c_int64(0)
    stats = (C.c_int32 * 2)()
    if nv:
        indptr, indices = graph._dev()
        D.check(D.load_library().gis_scc(D.ctx(), D.ptr(indptr), D.ptr(indices), nv, D.ptr(comp),
                                         D.ptr(sizes), D.ptr(nontriv), C.byref(ncomp), stats),
                "strongly_connected_components")
    k = int(ncomp.value)
    return comp, sizes[:k], nontriv[:k], k, (int(stats[0]), int(stats[1]))


def strongly_connected_components(graph: SymbolicImage) -> SccResult:
    """Exact SCC decomposition of the symbolic image (cg/analysis.py:109-117)."""
    comp, _, nontriv, k, _ = scc_dev(graph)
    return SccResult(component_of=comp.cpu().numpy(), n_components=k,
                     nontrivial=nontriv.cpu().numpy().view(bool))


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


def non_leaving_scc_dev(graph: SymbolicImage, strict_largest: bool = True):
    """(keep uint8 device tensor, closure rounds) by the reference's literal
    method (cg/analysis.py:120-161): SCCs (K6), then the reverse-reachability
    closure of the nontrivial components -- all of them, or with
    ``strict_largest`` the largest, ties toward the component holding the
    smallest vertex (cg/analysis.py:140-150)."""
    torch = D._torch()
    nv = graph.n_vertices
    keep = torch.zeros(nv, dtype=torch.uint8, device=D.device())
    rounds = C.c_int32(0)
    if nv == 0:
        return keep, 0
    indptr, indices = graph._dev()
    D.check(D.load_library().gis_non_leaving_scc(D.ctx(), D.ptr(indptr), D.ptr(indices), nv,
                                                 int(bool(strict_largest)), D.ptr(keep),
                                                 C.byref(rounds)),
            "non_leaving_mask(strict_largest=%s)" % bool(strict_largest))
    return keep, int(rounds.value)


def non_leaving_strict_dev(graph: SymbolicImage):
    return non_leaving_scc_dev(graph, strict_largest=True)


def non_leaving_mask(graph: SymbolicImage, strict_largest: bool = False) -> np.ndarray:
    """Boolean mask of vertices that can reach a cycle (cg/analysis.py:120)."""
    if graph.n_vertices == 0:
        return np.zeros(0, dtype=bool)
    keep, _ = non_leaving_strict_dev(graph) if strict_largest else non_leaving_dev(graph)
    return keep.cpu().numpy().view(bool)


def non_leaving(graph: SymbolicImage, strict_largest: bool = False) -> set:
    mask = non_leaving_mask(graph, strict_largest=strict_largest)
    return {graph.vertex_id(int(i)) for i in np.flatnonzero(mask)}


def retain(covering: Covering, keep) -> Covering:
    return covering.retain(keep)
