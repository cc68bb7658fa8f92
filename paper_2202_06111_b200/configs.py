"""The BASELINE.json configurations as RunConfigs.

bloat = 0.1 is the reference default (cg/image.py:34); BASELINE.json does
not state one.  'Initial grid g^n' is ``initial_depth = n*log2(g)`` root
splits at iteration 1; 'R rounds' are R further iterations.
"""

from __future__ import annotations

from .adaptive import AdaptiveConfig
from .engine import RunConfig
from .image import ImageConfig, corners_plus_center, corners_plus_seeded, lattice_fractions
from .system import cartpole_model, cstr_dimless_model, lorenz_model, pendulum_model

__all__ = ["config", "CONFIG_NAMES", "BLOAT"]

BLOAT = 0.1
CONFIG_NAMES = {1: "pendulum-euler-64x64+3", 2: "pendulum-rk4-1024x1024",
                3: "cstr-dimless-32x32+8-adaptive", 4: "lorenz-256^3", 5: "cartpole-48^4+2-adaptive"}


def _img(frac):
    return ImageConfig(samples_per_dim=2, bloat=BLOAT, fractions=frac)


def config(i: int, **over) -> RunConfig:
    """RunConfig of BASELINE.json configs[i-1] (1-based)."""
    if i == 1:
        m = pendulum_model(integrator="euler", substeps=1, dt=0.05)
        kw = dict(model=m, iterations=4, initial_depth=12, input_counts=11,
                  image=_img(corners_plus_center(2)))
    elif i == 2:
        m = pendulum_model(integrator="rk4", substeps=10, dt=0.05)
        kw = dict(model=m, iterations=1, initial_depth=20, input_counts=21,
                  image=_img(corners_plus_seeded(2, 16, 0)))
    elif i == 3:
        # reference selector (Alg. 1 probe + N-NN, N=3): the SVM classifier of
        # BASELINE config 3 does not exist in the reference
        m = cstr_dimless_model(integrator="rk4", substeps=20, dt=0.1)
        kw = dict(model=m, iterations=9, initial_depth=10, input_counts=21,
                  image=_img(lattice_fractions(2, 3)),
                  adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3))
    elif i == 4:
        m = lorenz_model(integrator="rk4", substeps=5, dt=0.01)
        kw = dict(model=m, iterations=1, initial_depth=24, input_counts=9,
                  image=_img(corners_plus_seeded(3, 8, 1)))
    elif i == 5:
        # 48^4 is not a dyadic grid of X: it is the first 48 cells per axis of
        # the 64^4 dyadic grid of an extended root (geometry.extended_root)
        m = cartpole_model(integrator="rk4", substeps=4, dt=0.02)
        kw = dict(model=m, iterations=3, initial_grid=(48, 48, 48, 48), input_counts=11,
                  image=_img(corners_plus_seeded(4, 8, 2)),
                  adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3))
    else:
        raise ValueError("configs are numbered 1..5")
    kw.update(over)
    return RunConfig(**kw)
