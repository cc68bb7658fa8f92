"""User-defined models (CudaStep): the reference's SystemModel plugin API
(cg/system.py:52-75) reopened through NVRTC-compiled K1 kernels.  A user
field runs in the reference's operation order, so polynomial fields match
the numpy oracle bit for bit (transcendentals to CUDA libm's ulp)."""

import numpy as np
import pytest

from helpers import REL, assert_states_close

pytestmark = pytest.mark.gpu

PENDULUM = "f[0] = x[1]; f[1] = ((-p[0]) * sin(x[0]) - p[1] * x[1]) + u[0];"
VDP = "f[0] = x[1]; f[1] = (p[0] * (1.0 - x[0] * x[0])) * x[1] - x[0] + u[0];"
HENON = "y[0] = ((1.0 - p[0] * (x[0] * x[0])) + x[1]) + u[0]; y[1] = p[1] * x[0];"


def _vdp_np(mu):
    def rhs(x, u):
        u0 = np.asarray(u, dtype=np.float64).reshape(-1)[0]
        return np.stack([x[..., 1], (mu * (1.0 - x[..., 0] * x[..., 0])) * x[..., 1] - x[..., 0]
                         + u0], axis=-1)
    return rhs


def _rk4_step(rhs, dt, sub):
    from oracle import gis_oracle as O

    h = dt / sub

    def step(x, u):
        x = np.asarray(x, dtype=np.float64)
        for _ in range(sub):
            x = O.rk4(rhs, x, u, h)
        return x
    return step


def _henon_np(a, b):
    def step(x, u):
        x = np.asarray(x, dtype=np.float64)
        u0 = np.asarray(u, dtype=np.float64).reshape(-1)[0]
        return np.stack([((1.0 - a * (x[..., 0] * x[..., 0])) + x[..., 1]) + u0, b * x[..., 0]],
                        axis=-1)
    return step


def _grid(X, depth):
    from paper_2202_06111_b200 import Covering

    cov = Covering.initial(X)
    for _ in range(depth):
        cov = cov.subdivide(None)
    return cov


def _oracle_graph(cov, step, inputs, cfg):
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.image import sample_fractions

    return O.build_graph(cov.lo, cov.hi, step, np.atleast_2d(inputs.points),
                         sample_fractions(cfg, cov.n), cfg.bloat)


def test_user_pendulum_euler_equals_builtin_and_oracle():
    """BASELINE config 1's pendulum written as a CudaStep: the same graph as
    the built-in kind (both in the reference's Euler order) and the oracle."""
    from paper_2202_06111_b200 import SystemModel, sample_inputs
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.graph import build_graph_serial
    from paper_2202_06111_b200.system import CudaStep

    rc = config(1)
    m = rc.model
    user = SystemModel("pendulum-user", 2, 1, m.X, m.U,
                       CudaStep(PENDULUM, n=2, m=1, params=[9.81, 0.5], integrator="euler",
                                substeps=1, dt=0.05))
    cov = _grid(m.X, 12)
    inputs = sample_inputs(m.U, rc.input_counts)
    gb = build_graph_serial(cov, cov.build_index(), m, inputs, rc.image)
    gu = build_graph_serial(cov, cov.build_index(), user, inputs, rc.image)
    assert np.array_equal(gb.indptr, gu.indptr) and np.array_equal(gb.indices, gu.indices)
    assert gu.edge_count == 46120  # the reference's count
    from oracle import gis_oracle as O

    ip, ix = _oracle_graph(cov, O.make_step(m.step.spec()), inputs, rc.image)
    assert np.array_equal(gu.indptr, ip) and np.array_equal(gu.indices, ix)


def test_user_van_der_pol_rk4_bit_exact_vs_numpy():
    """A model the library does not ship: Van der Pol with input, RK4 x 5.
    Polynomial field, reference order: states and graph bit-exact."""
    from paper_2202_06111_b200 import Box, ImageConfig, SystemModel, sample_inputs
    from paper_2202_06111_b200.system import CudaStep

    mu, dt, sub = 0.8, 0.1, 5
    step = CudaStep(VDP, n=2, m=1, params=[mu], integrator="rk4", substeps=sub, dt=dt)
    model = SystemModel("vdp", 2, 1, Box([-3.0, -4.0], [3.0, 4.0]), Box([-1.0], [1.0]), step)
    rng = np.random.default_rng(0)
    x = rng.uniform(-3, 3, (1000, 2))
    ref = _rk4_step(_vdp_np(mu), dt, sub)
    for u in (-1.0, 0.25):
        got = model.map_points(x, np.array([u]))
        assert np.array_equal(got, ref(x, np.array([u])))
    rhs = step.rhs(x, np.array([0.5]))
    assert np.array_equal(rhs, _vdp_np(mu)(x, np.array([0.5])))
    cov = _grid(model.X, 11)
    inputs = sample_inputs(model.U, 7)
    cfg = ImageConfig(3, 0.1)
    from paper_2202_06111_b200.graph import build_graph_serial

    g = build_graph_serial(cov, cov.build_index(), model, inputs, cfg)
    ip, ix = _oracle_graph(cov, ref, inputs, cfg)
    assert np.array_equal(g.indptr, ip) and np.array_equal(g.indices, ix)


def test_user_map_henon_run_vs_oracle():
    """A direct map (form='map'): the whole engine loop, adaptive, against
    the oracle's restatement of cg/engine.py with the same numpy map."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import (AdaptiveConfig, Box, ImageConfig, RunConfig, SystemModel,
                                       run)
    from paper_2202_06111_b200.image import lattice_fractions
    from paper_2202_06111_b200.system import CudaStep

    a, b = 1.2, 0.3
    model = SystemModel("henon", 2, 1, Box([-1.5, -0.6], [1.5, 0.6]), Box([-0.05], [0.05]),
                        CudaStep(HENON, n=2, m=1, params=[a, b], form="map"))
    res = run(RunConfig(model=model, iterations=6, input_counts=3, initial_depth=10,
                        image=ImageConfig(3, 0.05),
                        adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3)))
    r = O.run(_henon_np(a, b), model.X.lo, model.X.hi, model.U.lo, model.U.hi, 3, 6,
              lattice_fractions(2, 3), 0.05, mode="adaptive", initial_depth=10, prune="peel")
    got = [(x.cells_before, x.cells_after, x.edges, x.boundary_cells) for x in res.metrics]
    want = [(x["cells_before"], x["cells_after"], x["edges"], x["boundary_cells"])
            for x in r["metrics"]]
    assert got == want
    assert np.array_equal(res.covering.bits, r["cover"].bits)


def test_user_model_compile_error_reports_log():
    from paper_2202_06111_b200 import Box, SystemModel
    from paper_2202_06111_b200.system import CudaStep

    bad = SystemModel("bad", 1, 1, Box([0.0], [1.0]), Box([0.0], [1.0]),
                      CudaStep("f[0] = x[0] +;", n=1, m=1, integrator="euler", dt=0.1))
    with pytest.raises(ValueError, match="does not compile"):
        bad.map_points(np.zeros((3, 1)), np.zeros(1))
