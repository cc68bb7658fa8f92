"""Sampled one-step image enclosures (mirror of cg/image.py), evaluated by
the libgis integrator kernel (K1).

``ImageConfig`` keeps the reference's knobs (samples_per_dim, bloat) and adds
``fractions``: an explicit (S, n) table of sample positions in [0,1]^n for
the BASELINE sampling schemes (corners + centre, corners + seeded uniform).
Without it the reference lattice (samples_per_dim^n points,
cg/image.py:43-48) is used.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _device as D
from .geometry import Box

__all__ = ["ImageConfig", "cell_sample_points", "cell_image", "cell_images",
           "batch_enclosures", "lattice_fractions", "corner_fractions",
           "corners_plus_center", "corners_plus_seeded", "sample_fractions"]


@dataclass(frozen=True)
class ImageConfig:
    """samples_per_dim >= 2 (lattice), bloat >= 0 (cg/image.py:24-40);
    fractions: optional explicit sample table (tuple of n-tuples)."""

    samples_per_dim: int = 3
    bloat: float = 0.1
    fractions: Optional[tuple] = None

    def __post_init__(self):
        if self.samples_per_dim < 2:
            raise ValueError("samples_per_dim must be at least 2")
        if self.bloat < 0:
            raise ValueError("bloat must be nonnegative")
        if self.fractions is not None:
            f = np.asarray(self.fractions, dtype=np.float64)
            if f.ndim != 2 or len(f) == 0 or np.any(f < 0) or np.any(f > 1):
                raise ValueError("fractions must be a non-empty (S, n) table in [0, 1]")
            object.__setattr__(self, "fractions", tuple(map(tuple, f.tolist())))


def lattice_fractions(n: int, spd: int) -> np.ndarray:
    """spd^n lattice, axis 0 slowest (cg/image.py:43-48)."""
    ax = np.linspace(0.0, 1.0, spd)
    mesh = np.meshgrid(*([ax] * n), indexing="ij")
    return np.stack([g.ravel() for g in mesh], axis=-1)


def corner_fractions(n: int) -> np.ndarray:
    """2^n corners in vertices() order (cg/geometry.py:185-197)."""
    codes = np.arange(1 << n)
    return np.stack([((codes >> (n - 1 - d)) & 1).astype(np.float64) for d in range(n)], -1)


def corners_plus_center(n: int) -> np.ndarray:
    """BASELINE config 1: the 2^n corners then the centre."""
    return np.vstack([corner_fractions(n), np.full((1, n), 0.5)])


def corners_plus_seeded(n: int, k: int, seed: int) -> np.ndarray:
    """BASELINE configs 2, 4, 5: the 2^n corners then k rows of
    numpy.random.default_rng(seed).random((k, n))."""
    return np.vstack([corner_fractions(n), np.random.default_rng(seed).random((k, n))])


def sample_fractions(cfg: ImageConfig, n: int) -> np.ndarray:
    if cfg.fractions is not None:
        f = np.asarray(cfg.fractions, dtype=np.float64)
        if f.shape[1] != n:
            raise ValueError(f"sample table has {f.shape[1]} columns, model has n={n}")
        return f
    return lattice_fractions(n, cfg.samples_per_dim)


def cell_sample_points(box: Box, samples_per_dim: int) -> np.ndarray:
    """Sample lattice of one box (cg/image.py:51-56)."""
    if samples_per_dim < 2:
        raise ValueError("samples_per_dim must be at least 2")
    frac = lattice_fractions(box.n, samples_per_dim)
    return box.lo * (1.0 - frac) + box.hi * frac


def enclosures_dev(model, lo_soa, hi_soa, inputs, cfg: ImageConfig):
    """Device enclosures for all inputs: enc_lo/enc_hi [U][B][n], valid [U][B]."""
    torch = D._torch()
    step = model.step
    mstruct = D.encode_model(step)
    n, B = lo_soa.shape
    u = np.atleast_2d(np.asarray(inputs, dtype=np.float64))
    U = len(u)
    frac = sample_fractions(cfg, n)
    _, up = D.host_f64(u)
    _, fp = D.host_f64(frac)
    enc_lo = torch.empty((U, B, n), dtype=torch.float64, device=D.device())
    enc_hi = torch.empty_like(enc_lo)
    valid = torch.empty((U, B), dtype=torch.uint8, device=D.device())
    D.check(D.load_library().gis_batch_enclosures(
        D.ctx(), C.byref(mstruct), D.ptr(lo_soa), D.ptr(hi_soa), B, up, U, fp, len(frac),
        float(cfg.bloat), D.ptr(enc_lo), D.ptr(enc_hi), D.ptr(valid)), "batch_enclosures")
    return enc_lo, enc_hi, valid


def batch_enclosures(model, lo, hi, u, cfg: ImageConfig):
    """Per-cell enclosure of the sampled image for one input
    (cg/image.py:65-85): (enc_lo, enc_hi, valid) as numpy arrays."""
    lo = np.atleast_2d(np.asarray(lo, dtype=np.float64))
    hi = np.atleast_2d(np.asarray(hi, dtype=np.float64))
    if len(lo) == 0:
        n = lo.shape[1]
        return np.empty((0, n)), np.empty((0, n)), np.empty(0, dtype=bool)
    el, eh, v = enclosures_dev(model, D.to_dev(lo.T.copy()), D.to_dev(hi.T.copy()),
                               np.asarray(u, dtype=np.float64).reshape(1, -1), cfg)
    return el[0].cpu().numpy(), eh[0].cpu().numpy(), v[0].cpu().numpy().view(bool)


def cell_image(model, box: Box, u, cfg: ImageConfig):
    """Enclosure of f(box, u), or None when every sample escapes
    (cg/image.py:88-99)."""
    elo, ehi, valid = batch_enclosures(model, box.lo[None, :], box.hi[None, :],
                                       np.asarray(u, dtype=np.float64), cfg)
    if not valid[0]:
        return None
    return Box(elo[0], ehi[0])


def cell_images(model, box: Box, inputs, cfg: ImageConfig) -> list:
    """[(u, Box-or-None), ...] in input order (cg/image.py:102-106)."""
    pts = np.atleast_2d(np.asarray(getattr(inputs, "points", inputs), dtype=np.float64))
    el, eh, v = enclosures_dev(model, D.to_dev(box.lo[:, None].copy()),
                               D.to_dev(box.hi[:, None].copy()), pts, cfg)
    el, eh, v = el.cpu().numpy(), eh.cpu().numpy(), v.cpu().numpy()
    return [(u, Box(el[i, 0], eh[i, 0]) if v[i, 0] else None) for i, u in enumerate(pts)]
