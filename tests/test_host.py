"""Host-side logic that needs no GPU: value types, configuration, model
descriptors, sampling tables and the sharding arithmetic."""

import numpy as np
import pytest


def test_box_and_cellid():
    from paper_2202_06111_b200 import Box, CellId
    from paper_2202_06111_b200.geometry import enlarge, subdivide_cell, vertices

    with pytest.raises(ValueError):
        Box([0.0], [np.inf])
    with pytest.raises(ValueError):
        Box([1.0], [0.0])
    b = Box([0.0, 0.0], [1.0, 1.0])
    assert b.volume == 1.0 and b == Box([0, 0], [1, 1]) and hash(b) == hash(Box([0, 0], [1, 1]))
    assert vertices(b).tolist() == [[0, 0], [0, 1], [1, 0], [1, 1]]
    assert enlarge(b, 0.1) == Box([-0.05, -0.05], [1.05, 1.05])
    (c0, b0), (c1, b1) = subdivide_cell(CellId.root(), b, 0)
    assert b0 == Box([0, 0], [0.5, 1]) and (c0.path, c1.path) == ("0", "1")
    rng = np.random.default_rng(5)
    paths = sorted({""} | {"".join(rng.choice(["0", "1"], int(rng.integers(1, 12))))
                           for _ in range(200)})
    assert [c.path for c in sorted(CellId.from_path(p) for p in paths)] == paths
    with pytest.raises(ValueError):
        CellId.root().parent()


def test_sample_inputs_reference_semantics():
    from paper_2202_06111_b200 import Box, sample_inputs

    assert sample_inputs(Box([285.0], [315.0]), 3).points[:, 0].tolist() == [285.0, 300.0, 315.0]
    assert len(sample_inputs(Box([0.0, -1.0], [1.0, 1.0]), (3, 4))) == 12
    assert len(sample_inputs(Box([0.0], [0.0]), 3)) == 1
    with pytest.raises(ValueError):
        sample_inputs(Box([0.0], [1.0]), 1)


def test_image_config_and_tables():
    from paper_2202_06111_b200.image import (ImageConfig, corners_plus_center,
                                             corners_plus_seeded, lattice_fractions,
                                             sample_fractions)

    with pytest.raises(ValueError):
        ImageConfig(samples_per_dim=1)
    with pytest.raises(ValueError):
        ImageConfig(bloat=-0.1)
    with pytest.raises(ValueError):
        ImageConfig(fractions=[[1.5, 0.0]])
    assert lattice_fractions(2, 3).shape == (9, 2)
    cc = corners_plus_center(2)
    assert cc.tolist() == [[0, 0], [0, 1], [1, 0], [1, 1], [0.5, 0.5]]
    s = corners_plus_seeded(3, 8, 1)
    assert s.shape == (16, 3)
    assert np.array_equal(s[8:], np.random.default_rng(1).random((8, 3)))
    cfg = ImageConfig(2, 0.1, fractions=cc)
    assert np.array_equal(sample_fractions(cfg, 2), cc)
    with pytest.raises(ValueError):
        sample_fractions(cfg, 3)


@pytest.mark.parametrize("i,S,n,V0", [(1, 5, 2, 4096), (2, 20, 2, 1 << 20), (3, 9, 2, 1024),
                                      (4, 16, 3, 1 << 24), (5, 24, 4, 48 ** 4)])
def test_baseline_configs(i, S, n, V0):
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.image import sample_fractions

    rc = config(i)
    assert rc.model.n == n
    assert len(sample_fractions(rc.image, n)) == S
    if rc.initial_grid is not None:
        assert int(np.prod(rc.initial_grid)) == V0
    else:
        assert 2 ** rc.initial_depth == V0
    assert rc.image.bloat == 0.1


def test_extended_root_for_non_dyadic_grids():
    from paper_2202_06111_b200 import Box
    from paper_2202_06111_b200.geometry import extended_root

    X = Box([-2.4, -3.0, -0.21, -3.0], [2.4, 3.0, 0.21, 3.0])
    root, depth = extended_root(X, (48, 48, 48, 48))
    assert depth == 24 and np.array_equal(root.lo, X.lo)
    assert np.allclose(root.hi - root.lo, (X.hi - X.lo) * 64 / 48, rtol=1e-15)
    assert extended_root(Box([0.0, 0.0], [1.0, 1.0]), (64, 64))[1] == 12
    assert extended_root(Box([0.0, 0.0], [1.0, 1.0]), (6, 3))[1] == 5   # 8 x 4
    with pytest.raises(ValueError):
        extended_root(Box([0.0, 0.0], [1.0, 1.0]), (3, 48))  # 4 x 64 not cycled


def test_model_descriptors():
    from paper_2202_06111_b200 import system as S

    m = S.cstr_model()
    assert m.step.params.h == 0.1 and m.X == S.Box([0.0, 345.0], [1.0, 355.0])
    assert S.make_model("cstr", h=0.05).step.params.h == 0.05
    with pytest.raises(ValueError, match="unknown model"):
        S.make_model("pendulum")  # registry is the reference's (tests/test_system.py:164)
    with pytest.raises(ValueError, match="unknown CSTR parameter"):
        S.make_model("cstr", mass=1.0)
    p = S.pendulum_model(integrator="rk4", substeps=10, dt=0.05).step
    assert p.h == 0.05 / 10 and p.param_vector() == [9.81, 0.5]
    assert p.spec()["kind"] == "pendulum"
    c = S.cartpole_model().step
    assert c.param_vector()[3] == 1.1 and c.n == 4
    with pytest.raises(ValueError):
        S.PendulumStep(integrator="midpoint")
    with pytest.raises(TypeError):
        S.rk4_discretize(lambda x, u: -x, np.array([1.0]), np.array([0.0]), 0.1)
    with pytest.raises(ValueError):
        S.rk4_discretize(S.pendulum_model().step.rhs, np.zeros(2), np.zeros(1), 0.0)


def test_device_encoding_refuses_callables():
    from paper_2202_06111_b200 import _device as D
    from paper_2202_06111_b200 import system as S

    with pytest.raises(TypeError, match="not a device model"):
        D.encode_model(lambda x, u: x)
    enc = D.encode_model(S.lorenz_model(integrator="rk4", substeps=5, dt=0.01).step)
    assert (enc.kind, enc.integrator, enc.substeps, enc.n) == (7, 2, 5, 3)
    assert enc.h == 0.01 / 5 and enc.params[2] == 8.0 / 3.0


def test_word_partition_covers_all_vertices():
    from paper_2202_06111_b200.distributed import owned_range, word_partition

    for V in (0, 1, 31, 32, 33, 1000, 1 << 20, 1_000_003):
        for size in (1, 2, 3, 4, 8):
            ranges = [owned_range(V, r, size) for r in range(size)]
            assert ranges[0][0] == 0 and ranges[-1][1] == V
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            for b, e in ranges:
                assert (b % 32 == 0 or b == e == V) and b <= e
            assert word_partition(V, size) * size * 32 >= V


def test_reference_input_grid_and_registry_behaviours():
    """The reference's tests/test_system.py:129-180 (input grids, model
    registry) restated on the host side of the package."""
    import pytest

    from paper_2202_06111_b200 import Box, sample_inputs
    from paper_2202_06111_b200.system import MODEL_NAMES, make_model

    assert sample_inputs(Box([285.0], [315.0]), 3).points[:, 0].tolist() == [285.0, 300.0, 315.0]
    g = sample_inputs(Box([-0.5, -0.5], [0.5, 0.5]), (2, 2))
    assert len(g) == 4 and sorted(map(tuple, g.points.tolist())) == [
        (-0.5, -0.5), (-0.5, 0.5), (0.5, -0.5), (0.5, 0.5)]
    assert sample_inputs(Box([1.0], [3.0]), 2).points[:, 0].tolist() == [1.0, 3.0]
    g = sample_inputs(Box([0.0, -1.0], [1.0, 1.0]), (3, 4))
    assert len(g) == 12 and (g.points[:, 0] >= 0).all() and (g.points[:, 1] <= 1).all()
    assert len(sample_inputs(Box([0.0], [0.0]), 3)) == 1
    with pytest.raises(ValueError):
        sample_inputs(Box([0.0], [1.0]), 1)
    for name in MODEL_NAMES:
        assert make_model(name).name == name
    with pytest.raises(ValueError, match="unknown model"):
        make_model("no-such-model")
    assert make_model("cstr", h=0.05).step.params.h == 0.05
    with pytest.raises(ValueError, match="unknown CSTR parameter"):
        make_model("cstr", mass=1.0)
    m = make_model("linear", a=3.0, ulo=-1.0, uhi=1.0)
    assert m.step.a == 3.0 and m.U == Box([-1.0], [1.0])
