"""Discrete-time systems as device-model descriptors (mirror of cg/system.py).

The reference's plugin contract is ``SystemModel(name, n, m, X, U, step)``
with ``step(x:(N,n), u:(m,)) -> (N,n)`` a pure, broadcasting, picklable
callable (/root/reference/pkg/src/cisgraph/system.py:52-75).  Here ``step``
is a *descriptor* of a vector field + integrator that the sm_100a integrator
(libgis ``gis_map_points`` / ``gis_build_graph``) evaluates; calling it runs
the CUDA kernel.  Arbitrary Python callables are rejected when they reach the
device path: there is no CPU fallback.

Operation order of every vector field is fixed here.  ``csrc/gis_models.cuh``
follows it with separately rounded IEEE ops for the reference models and the
CSTR fields, and with a few fused one-rounding updates for pendulum, Lorenz
and cart-pole (states within 1e-12 relative, graphs unchanged): see DESIGN.md
section 3.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .geometry import Box

__all__ = [
    "SystemModel", "InputGrid", "CstrParameters", "rk4_discretize",
    "cstr_model", "linear_test_model", "affine_test_model", "identity_model",
    "shift_model", "pendulum_model", "cstr_dimless_model", "lorenz_model",
    "cartpole_model", "sample_inputs", "make_model", "MODEL_NAMES", "MODEL_PARAMS",
    "DeviceStep", "CstrStep", "LinearStep", "AffineStep", "IdentityStep",
    "ShiftStep", "PendulumStep", "DimlessCstrStep", "LorenzStep", "CartPoleStep",
    "CudaStep",
]

# model kind ids and integrator ids shared with include/gis.h
KIND_IDS = {"identity": 0, "shift": 1, "linear": 2, "affine": 3, "cstr": 4,
            "pendulum": 5, "cstr_dimless": 6, "lorenz": 7, "cartpole": 8, "jit": 9}
INTEGRATOR_IDS = {"map": 0, "euler": 1, "rk4": 2, "rhs": 3}
MAX_PARAMS = 64


class DeviceStep:
    """A vector field (or direct map) plus its discretisation, evaluated by
    the CUDA integrator.  Subclasses define ``kind``, ``n``, ``m`` and
    ``param_vector()``; ``integrator`` is 'map', 'euler' or 'rk4' with
    ``substeps`` steps of h = dt / substeps (h computed once, in Python)."""

    kind = ""
    integrator = "map"
    substeps = 1
    dt = 1.0

    def param_vector(self) -> list:
        return []

    def param_dict(self) -> dict:
        return {}

    @property
    def h(self) -> float:
        return float(self.dt) / int(self.substeps)

    def spec(self) -> dict:
        """Plain-dict description (used by tests to drive the CPU oracle)."""
        return {"kind": self.kind, "params": self.param_dict(),
                "integrator": self.integrator, "substeps": int(self.substeps),
                "dt": float(self.dt)}

    def __call__(self, x, u):
        from ._device import map_points_numpy

        x = np.asarray(x, dtype=np.float64)
        pts = x.reshape(-1, self.n)
        out = map_points_numpy(self, pts, np.asarray(u, dtype=np.float64).reshape(-1))
        return out.reshape(x.shape)

    def rhs(self, x, u):
        """Vector field only (one evaluation, no integration) on the GPU."""
        if self.integrator == "map":
            raise TypeError(f"{type(self).__name__} is a direct map, not an ODE")
        from ._device import map_points_numpy

        x = np.asarray(x, dtype=np.float64)
        out = map_points_numpy(self, x.reshape(-1, self.n),
                               np.asarray(u, dtype=np.float64).reshape(-1), rhs_only=True)
        return out.reshape(x.shape)

    def __eq__(self, other):
        return type(self) is type(other) and self.spec_key() == other.spec_key()

    def __hash__(self):
        return hash(self.spec_key())

    def spec_key(self):
        return (self.kind, self.integrator, int(self.substeps), float(self.dt),
                tuple(self.param_vector()))

    def __repr__(self):
        return (f"{type(self).__name__}({self.param_dict()}, integrator={self.integrator!r}, "
                f"substeps={self.substeps}, dt={self.dt})")


def rk4_discretize(ode_rhs, x, u, h: float):
    """One RK4 step with u held (cg/system.py:34-49), evaluated on the GPU.

    ``ode_rhs`` must be the ``rhs`` of a device model (e.g. ``step.rhs``);
    arbitrary Python callables are refused (no CPU fallback)."""
    if h <= 0:
        raise ValueError("step size must be positive")
    owner = getattr(ode_rhs, "__self__", None)
    if not isinstance(owner, DeviceStep) or owner.integrator == "map":
        raise TypeError("rk4_discretize accepts the .rhs of a device model only")
    probe = replace_step(owner, integrator="rk4", substeps=1, dt=float(h))
    return probe(x, u)


def replace_step(step: DeviceStep, **changes) -> DeviceStep:
    import copy

    s = copy.copy(step)
    for k, v in changes.items():
        setattr(s, k, v)
    return s


@dataclass(frozen=True)
class SystemModel:
    """Discrete-time map with state box X and input box U
    (cg/system.py:52-75)."""

    name: str
    n: int
    m: int
    X: Box
    U: Box
    step: object

    def __post_init__(self):
        if self.X.n != self.n or self.U.n != self.m:
            raise ValueError("constraint box dimensions do not match n, m")

    def map_points(self, points, u) -> np.ndarray:
        pts = np.asarray(points, dtype=np.float64).reshape(-1, self.n)
        out = np.asarray(self.step(pts, np.asarray(u, dtype=np.float64)))
        return out.reshape(pts.shape)


@dataclass(frozen=True)
class InputGrid:
    """Finite input set, endpoints included (cg/system.py:78-93)."""

    points: np.ndarray
    counts: tuple

    def __post_init__(self):
        object.__setattr__(self, "points", np.asarray(self.points, dtype=np.float64))

    def __len__(self):
        return len(self.points)

    def __iter__(self):
        return iter(self.points)


def sample_inputs(U: Box, counts) -> InputGrid:
    """Cartesian linspace grid over U, duplicates dropped (cg/system.py:96-116).
    Host-side configuration (a few dozen points), not part of the hot path."""
    m = U.n
    if np.isscalar(counts):
        counts = (int(counts),) * m
    counts = tuple(int(c) for c in counts)
    if len(counts) != m:
        raise ValueError("one count per input dimension required")
    if any(c < 2 for c in counts):
        raise ValueError("counts must be at least 2 (endpoints included)")
    axes = [np.linspace(U.lo[d], U.hi[d], counts[d]) for d in range(m)]
    mesh = np.meshgrid(*axes, indexing="ij")
    pts = np.unique(np.stack([g.ravel() for g in mesh], axis=-1), axis=0)
    return InputGrid(pts, counts)


# -- CSTR (reference Table 2 model) ------------------------------------------

@dataclass(frozen=True)
class CstrParameters:
    """Exothermic CSTR parameters (cg/system.py:122-145)."""

    q: float = 100.0
    V: float = 100.0
    c_Af: float = 1.0
    T_f: float = 350.0
    E_over_R: float = 8750.0
    k0: float = 7.2e10
    minus_dH: float = 5.0e4
    UA: float = 5.0e4
    c_p: float = 0.239
    rho: float = 1000.0
    h: float = 0.1

    def __post_init__(self):
        for name, value in self.__dict__.items():
            if not value > 0:
                raise ValueError(f"CSTR parameter {name} must be positive")



class CudaStep(DeviceStep):
    """A user-defined model as CUDA C++ source: the reference's plugin API
    (``SystemModel(step=callable)``, cg/system.py:52-75) without a CPU
    fallback.  libgis compiles the source with NVRTC into the same K1
    kernels the built-in models use (``gis_jit_register``) the first time the
    model runs, and evaluates it on the GPU in the reference's operation
    order (one rounding per operation, CUDA libm).

    ``form='ode'``: ``body`` sets ``f[0..n-1]`` from ``x[0..n-1]``,
    ``u[0..m-1]`` and ``p[...]`` (= ``params``); it is integrated by
    ``integrator`` ('euler' or 'rk4', cg/system.py:34-49) with ``substeps``
    steps of h = dt / substeps.  ``form='map'``: ``body`` sets ``y[0..n-1]``,
    the next state.  Example (the damped pendulum of BASELINE config 1)::

        CudaStep("f[0] = x[1]; f[1] = (-p[0] * sin(x[0]) - p[1] * x[1]) + u[0];",
                 n=2, m=1, params=[9.81, 0.5], integrator="euler", dt=0.05)
    """

    kind = "jit"

    def __init__(self, body: str, n: int, m: int, params=(), form: str = "ode",
                 integrator: str = "rk4", substeps: int = 1, dt: float = 1.0):
        if form not in ("ode", "map"):
            raise ValueError("form must be 'ode' or 'map'")
        if form == "map":
            integrator = "map"
        elif integrator not in ("euler", "rk4"):
            raise ValueError("an ODE model integrates by 'euler' or 'rk4'")
        if not 1 <= int(n) <= 4 or not 1 <= int(m) <= 4:
            raise ValueError("n and m must be in [1, 4]")
        if int(substeps) < 1 or not float(dt) > 0:
            raise ValueError("substeps must be >= 1 and dt > 0")
        self.body = str(body)
        self.n, self.m = int(n), int(m)
        self.params = [float(v) for v in params]
        if len(self.params) > MAX_PARAMS:
            raise ValueError(f"at most {MAX_PARAMS} parameters")
        self.form = form
        self.integrator = integrator
        self.substeps = int(substeps)
        self.dt = float(dt)

    def param_vector(self) -> list:
        return list(self.params)

    def param_dict(self) -> dict:
        return {"p": list(self.params)}

    def spec_key(self):
        return (self.kind, self.form, self.body, self.n, self.m) + super().spec_key()[1:]

    def __repr__(self):
        return (f"CudaStep({self.body!r}, n={self.n}, m={self.m}, params={self.params}, "
                f"form={self.form!r}, integrator={self.integrator!r}, "
                f"substeps={self.substeps}, dt={self.dt})")

class CstrStep(DeviceStep):
    """One RK4 step of h of the CSTR (cg/system.py:148-169)."""

    kind, n, m, integrator = "cstr", 2, 1, "rk4"

    def __init__(self, params: CstrParameters):
        self.params_ = params
        self.dt = params.h
        self.substeps = 1

    @property
    def params(self):  # reference attribute name (tests read step.params.h)
        return self.params_

    def param_dict(self):
        return self._folded()

    def _folded(self):
        p = self.params_
        return {"qV": p.q / p.V, "c_Af": p.c_Af, "T_f": p.T_f, "E_over_R": p.E_over_R,
                "k0": p.k0, "c1": p.minus_dH / (p.rho * p.c_p),
                "c2": p.UA / (p.V * p.rho * p.c_p)}

    def param_vector(self):
        f = self._folded()
        return [f["qV"], f["c_Af"], f["T_f"], -f["E_over_R"], f["k0"], f["c1"], f["c2"]]

    def spec_key(self):
        return ("cstr", tuple(self.param_vector()), self.dt)


def cstr_model(params: CstrParameters | None = None) -> SystemModel:
    params = params or CstrParameters()
    return SystemModel("cstr", 2, 1, Box([0.0, 345.0], [1.0, 355.0]),
                       Box([285.0], [315.0]), CstrStep(params))


# -- analytic test maps (cg/system.py:185-261) --------------------------------

class LinearStep(DeviceStep):
    kind, n, m = "linear", 1, 1

    def __init__(self, a: float):
        self.a = float(a)

    def param_dict(self):
        return {"a": self.a}

    def param_vector(self):
        return [self.a]


class AffineStep(DeviceStep):
    """x+ = A x + B u + c, evaluated as ((sum_k x_k A_jk) + (sum_l u_l B_jl)) + c_j."""

    kind = "affine"

    def __init__(self, A, B, c):
        self.A = np.asarray(A, dtype=np.float64)
        self.B = np.asarray(B, dtype=np.float64)
        self.c = np.asarray(c, dtype=np.float64)
        self.n, self.m = self.A.shape[0], self.B.shape[1]
        if self.n > 4 or self.m > 4:
            raise ValueError("affine device model supports n, m <= 4")

    def param_dict(self):
        return {"A": self.A.tolist(), "B": self.B.tolist(), "c": self.c.tolist()}

    def param_vector(self):
        return list(self.A.ravel()) + list(self.B.ravel()) + list(self.c.ravel())


class IdentityStep(DeviceStep):
    kind, n, m = "identity", 1, 1


class ShiftStep(DeviceStep):
    kind, n, m = "shift", 1, 1

    def __init__(self, offset: float):
        self.offset = float(offset)

    def param_dict(self):
        return {"offset": self.offset}

    def param_vector(self):
        return [self.offset]


def linear_test_model(a: float, X=(-1.0, 1.0), U=(-0.5, 0.5)) -> SystemModel:
    return SystemModel("linear", 1, 1, Box([X[0]], [X[1]]), Box([U[0]], [U[1]]),
                       LinearStep(a))


def affine_test_model(A, B, c, X: Box, U: Box) -> SystemModel:
    st = AffineStep(A, B, c)
    return SystemModel("affine", st.n, st.m, X, U, st)


def identity_model(X=(0.0, 1.0)) -> SystemModel:
    return SystemModel("identity", 1, 1, Box([X[0]], [X[1]]), Box([0.0], [0.0]),
                       IdentityStep())


def shift_model(offset: float = 10.0, X=(0.0, 1.0)) -> SystemModel:
    return SystemModel("shift", 1, 1, Box([X[0]], [X[1]]), Box([0.0], [0.0]),
                       ShiftStep(offset))


# -- BASELINE.json models (not in the reference registry) ---------------------

class _OdeStep(DeviceStep):
    def __init__(self, integrator="rk4", substeps=1, dt=0.05):
        if integrator not in ("euler", "rk4"):
            raise ValueError("integrator must be 'euler' or 'rk4'")
        if int(substeps) < 1 or not float(dt) > 0:
            raise ValueError("substeps >= 1 and dt > 0 required")
        self.integrator, self.substeps, self.dt = integrator, int(substeps), float(dt)


class PendulumStep(_OdeStep):
    """Damped torque-limited pendulum: x1' = x2,
    x2' = ((-a) sin x1 - b x2) + u  (BASELINE.json configs 1-2)."""

    kind, n, m = "pendulum", 2, 1

    def __init__(self, a=9.81, b=0.5, **kw):
        super().__init__(**kw)
        self.a, self.b = float(a), float(b)

    def param_dict(self):
        return {"a": self.a, "b": self.b}

    def param_vector(self):
        return [self.a, self.b]


class DimlessCstrStep(_OdeStep):
    """Dimensionless exothermic CSTR (BASELINE.json config 3):
    t = (Da (1 - x1)) exp(x2 / (1 + x2/gamma)); x1' = (-x1) + t;
    x2' = ((-x2) + B t) - beta (x2 - u)."""

    kind, n, m = "cstr_dimless", 2, 1

    def __init__(self, Da=0.072, gamma=20.0, B=8.0, beta=0.3, **kw):
        super().__init__(**kw)
        self.Da, self.gamma, self.B, self.beta = float(Da), float(gamma), float(B), float(beta)

    def param_dict(self):
        return {"Da": self.Da, "gamma": self.gamma, "B": self.B, "beta": self.beta}

    def param_vector(self):
        return [self.Da, self.gamma, self.B, self.beta]


class LorenzStep(_OdeStep):
    """Controlled Lorenz (BASELINE.json config 4): x' = s (y - x);
    y' = (x (r - z) - y) + u; z' = x y - b z."""

    kind, n, m = "lorenz", 3, 1

    def __init__(self, sigma=10.0, rho=28.0, beta=8.0 / 3.0, **kw):
        super().__init__(**kw)
        self.sigma, self.rho, self.beta = float(sigma), float(rho), float(beta)

    def param_dict(self):
        return {"sigma": self.sigma, "rho": self.rho, "beta": self.beta}

    def param_vector(self):
        return [self.sigma, self.rho, self.beta]


class CartPoleStep(_OdeStep):
    """Frictionless cart-pole, gym form (BASELINE.json config 5), state
    (p, v, theta, omega), l = half pole length:
    temp = (F + (pml w^2) sin th) / M;
    th'' = (g sin th - cos th temp) / (l (4/3 - (mp cos^2 th) / M));
    p'' = temp - ((pml th'') cos th) / M."""

    kind, n, m = "cartpole", 4, 1

    def __init__(self, g=9.81, mc=1.0, mp=0.1, l=0.5, **kw):
        super().__init__(**kw)
        self.g, self.mc, self.mp, self.l = float(g), float(mc), float(mp), float(l)

    def param_dict(self):
        return {"g": self.g, "mp": self.mp, "l": self.l, "M": self.mc + self.mp,
                "pml": self.mp * self.l, "four_thirds": 4.0 / 3.0}

    def param_vector(self):
        p = self.param_dict()
        # then host-folded products of constants (one rounding each, inside
        # the fused-update contract): the device field multiplies by 1/M
        # instead of dividing, and forms the denominator with one fma
        inv_m = 1.0 / p["M"]
        return [p["g"], p["mp"], p["l"], p["M"], p["pml"], p["four_thirds"], inv_m,
                p["pml"] * inv_m, p["l"] * p["four_thirds"], p["l"] * (p["mp"] * inv_m)]


def pendulum_model(X=((-1.0, -2.0), (1.0, 2.0)), U=((-2.0,), (2.0,)), **kw) -> SystemModel:
    return SystemModel("pendulum", 2, 1, Box(*X), Box(*U), PendulumStep(**kw))


def cstr_dimless_model(X=((0.0, 0.0), (1.0, 8.0)), U=((-2.0,), (2.0,)), **kw) -> SystemModel:
    return SystemModel("cstr_dimless", 2, 1, Box(*X), Box(*U), DimlessCstrStep(**kw))


def lorenz_model(X=((-20.0, -20.0, 0.0), (20.0, 20.0, 50.0)), U=((-5.0,), (5.0,)),
                 **kw) -> SystemModel:
    return SystemModel("lorenz", 3, 1, Box(*X), Box(*U), LorenzStep(**kw))


def cartpole_model(X=((-2.4, -3.0, -0.21, -3.0), (2.4, 3.0, 0.21, 3.0)),
                   U=((-10.0,), (10.0,)), **kw) -> SystemModel:
    return SystemModel("cartpole", 4, 1, Box(*X), Box(*U), CartPoleStep(**kw))


# -- registry (cg/system.py:264-314) -----------------------------------------

MODEL_NAMES = ("cstr", "linear", "identity", "shift")
# accepted parameter names per registered model (cg/system.py:268-273)
MODEL_PARAMS = {
    "cstr": frozenset(CstrParameters().__dict__),
    "linear": frozenset({"a", "xlo", "xhi", "ulo", "uhi"}),
    "identity": frozenset({"xlo", "xhi"}),
    "shift": frozenset({"offset", "xlo", "xhi"}),
}


def make_model(name: str, **params) -> SystemModel:
    """Registered model by name; unknown names and parameters fail loudly."""
    if name in MODEL_PARAMS:
        unknown = set(params) - MODEL_PARAMS[name]
        if unknown:
            label = "CSTR" if name == "cstr" else name
            raise ValueError(f"unknown {label} parameter(s): {sorted(unknown)}")
    if name == "cstr":
        return cstr_model(replace(CstrParameters(),
                                  **{k: float(v) for k, v in params.items()}))
    if name == "linear":
        return linear_test_model(
            float(params.get("a", 2.0)),
            X=(float(params.get("xlo", -1.0)), float(params.get("xhi", 1.0))),
            U=(float(params.get("ulo", -0.5)), float(params.get("uhi", 0.5))))
    if name == "identity":
        return identity_model((float(params.get("xlo", 0.0)), float(params.get("xhi", 1.0))))
    if name == "shift":
        return shift_model(float(params.get("offset", 10.0)),
                           X=(float(params.get("xlo", 0.0)), float(params.get("xhi", 1.0))))
    raise ValueError(f"unknown model {name!r}; known models: {', '.join(MODEL_NAMES)}")
