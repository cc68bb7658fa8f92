"""Adaptive subdivision selection on the GPU (mirror of cg/adaptive.py).

Boundary cells: some probe of the slightly enlarged box (2^n corners, plus
edge midpoints on request) lies in no cell (cg/adaptive.py:61-123) -- libgis
point location in the grid index.  Neighbourhood: union of the exact N
nearest cell centres of every boundary cell minus the boundary
(cg/adaptive.py:136-150) -- libgis windowed k-NN.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as D
from .geometry import Covering, SpatialIndex

__all__ = ["AdaptiveConfig", "select_boundary", "select_boundary_mask", "select_neighborhood",
           "select_neighborhood_mask", "select_for_subdivision", "select_for_subdivision_mask",
           "subdivide_selected", "boundary_dev", "neighborhood_dev"]

MODES = ("full", "adaptive")


@dataclass(frozen=True)
class AdaptiveConfig:
    mode: str = "full"
    n_neighbors: int = 3
    delta: float = 0.01
    include_face_points: bool = False

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.n_neighbors < 0:
            raise ValueError("n_neighbors must be nonnegative")
        if not self.delta > 0:
            raise ValueError("delta must be positive")


def _soa(covering):
    if isinstance(covering, Covering):
        return covering._lo, covering._hi, len(covering)
    lo = np.atleast_2d(np.asarray(covering.lo, dtype=np.float64))
    hi = np.atleast_2d(np.asarray(covering.hi, dtype=np.float64))
    return D.to_dev(lo.T.copy()), D.to_dev(hi.T.copy()), len(lo)


def boundary_dev(covering, index: SpatialIndex, delta: float, include_face_points=False):
    torch = D._torch()
    lo, hi, V = _soa(covering)
    out = torch.zeros(V, dtype=torch.uint8, device=D.device())
    if V:
        D.check(D.load_library().gis_select_boundary(D.ctx(), index._h, D.ptr(lo), D.ptr(hi), V,
                                                     float(delta), int(bool(include_face_points)),
                                                     D.ptr(out)), "select_boundary")
    return out


def neighborhood_dev(index: SpatialIndex, boundary, n_neighbors: int):
    torch = D._torch()
    V = index.size
    b = boundary if isinstance(boundary, torch.Tensor) else D.to_dev(
        np.asarray(boundary, dtype=np.uint8))
    b = b.to(torch.uint8)
    if b.shape != (V,):
        raise ValueError("boundary mask length does not match the index")
    out = torch.zeros(V, dtype=torch.uint8, device=D.device())
    if V:
        D.check(D.load_library().gis_select_neighborhood(
            D.ctx(), index._h, D.ptr(index._lo), D.ptr(index._hi), V, D.ptr(b),
            int(n_neighbors), D.ptr(out)), "select_neighborhood")
    return out


def select_boundary_mask(covering, index: SpatialIndex, delta: float,
                         include_face_points: bool = False) -> np.ndarray:
    if (len(covering) if isinstance(covering, Covering) else len(covering.lo)) == 0:
        return np.zeros(0, dtype=bool)
    return boundary_dev(covering, index, delta, include_face_points).cpu().numpy().view(bool)


def _mask_to_labels(index: SpatialIndex, mask) -> set:
    if index.labels is None:
        return {int(i) for i in np.flatnonzero(mask)}
    return {index.labels[int(i)] for i in np.flatnonzero(mask)}


def _labels_to_mask(covering, index: SpatialIndex, labels: set) -> np.ndarray:
    V = index.size
    mask = np.zeros(V, dtype=bool)
    if not labels:
        return mask
    if index.labels is None:
        for i in labels:
            mask[int(i)] = True
        return mask
    lookup = {index.labels[i]: i for i in range(V)}
    for lab in labels:
        mask[lookup[lab]] = True
    return mask


def select_boundary(covering, index: SpatialIndex, delta: float,
                    include_face_points: bool = False) -> set:
    return _mask_to_labels(index, select_boundary_mask(covering, index, delta,
                                                       include_face_points))


def select_neighborhood_mask(covering, index: SpatialIndex, boundary_mask,
                             n_neighbors: int) -> np.ndarray:
    bm = np.asarray(boundary_mask, dtype=bool)
    if n_neighbors == 0 or not bm.any():
        return np.zeros(len(bm), dtype=bool)
    return neighborhood_dev(index, bm, n_neighbors).cpu().numpy().view(bool)


def select_neighborhood(covering, index: SpatialIndex, boundary: set, n_neighbors: int) -> set:
    mask = _labels_to_mask(covering, index, boundary)
    return _mask_to_labels(index, select_neighborhood_mask(covering, index, mask, n_neighbors))


def select_for_subdivision_mask(covering, index: SpatialIndex, cfg: AdaptiveConfig) -> np.ndarray:
    if cfg.mode == "full":
        return np.ones(index.size, dtype=bool)
    b = select_boundary_mask(covering, index, cfg.delta, cfg.include_face_points)
    return b | select_neighborhood_mask(covering, index, b, cfg.n_neighbors)


def select_for_subdivision(covering, index: SpatialIndex, cfg: AdaptiveConfig) -> set:
    return _mask_to_labels(index, select_for_subdivision_mask(covering, index, cfg))


def subdivide_selected(covering: Covering, selection) -> Covering:
    return covering.subdivide(selection)
