"""The sparse dyadic index and K2-general: coverings too
deep for a dense slot table (the reference allows MAX_DEPTH = 62,
cg/geometry.py:34) and input grids with more than 128 points
(cg/system.py:78-116).

* sparse == dense on every index query, for random mixed-depth coverings
  where both fit (graph, query_boxes, boundary probes, k-NN neighbourhoods,
  containment);
* 2-D adaptive coverings of depth >= 40 against the oracle (whose box tree
  has no depth limit), and a 1-D adaptive run to depth ~50 against the
  reference itself (tests/golden/runs.npz);
* m = 2 inputs on a 21 x 21 grid (441 points) and 200 scalar inputs against
  the oracle."""

import numpy as np
import pytest

from helpers import explain_edge_diffs

pytestmark = pytest.mark.gpu


def _mixed_covering(rng, m, splits, cap=4000):
    from paper_2202_06111_b200 import Covering

    cov = Covering.initial(m.X)
    for _ in range(splits):
        cov = cov.subdivide(rng.random(len(cov)) < rng.uniform(0.6, 1.0))
    if len(cov) > cap:
        cov = cov.retain(np.sort(rng.choice(len(cov), cap, replace=False)))
    return cov.retain(rng.random(len(cov)) < rng.uniform(0.7, 1.0))


def _graph_vs_oracle(cov, m, inputs, cfg, index=None):
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.graph import build_graph_serial
    from paper_2202_06111_b200.image import sample_fractions

    g = build_graph_serial(cov, index or cov.build_index(), m, inputs, cfg)
    frac = sample_fractions(cfg, m.n)
    step = O.make_step(m.step.spec())
    pts = np.atleast_2d(inputs.points)
    ip, ix = O.build_graph(cov.lo, cov.hi, step, pts, frac, cfg.bloat)
    if not (np.array_equal(g.indptr, ip) and np.array_equal(g.indices, ix)):
        near, unex = explain_edge_diffs(cov.lo, cov.hi, step, pts, frac, cfg.bloat,
                                        (g.indptr, g.indices), (ip, ix))
        assert not unex, unex[:10]
        assert not near, f"{len(near)} near-face edge differences: {near[:5]}"
    return g


@pytest.mark.parametrize("seed", range(8))
def test_sparse_index_equals_dense(seed):
    from paper_2202_06111_b200 import ImageConfig, SpatialIndex, sample_inputs
    from paper_2202_06111_b200.adaptive import boundary_dev, neighborhood_dev
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.engine import containment_defect
    from paper_2202_06111_b200.graph import build_graph_serial

    rng = np.random.default_rng(700 + seed)
    m = config([1, 2, 3, 4, 5][seed % 5]).model
    cov = _mixed_covering(rng, m, {2: 13, 3: 14, 4: 14}[m.n])
    dense = SpatialIndex._dyadic(cov, "dense")
    sparse = SpatialIndex._dyadic(cov, "sparse")
    assert sparse.sparse and not dense.sparse
    inputs = sample_inputs(m.U, int(rng.integers(2, 7)))
    cfg = ImageConfig(2, float(rng.choice([0.0, 0.1, 0.5])))
    gd = build_graph_serial(cov, dense, m, inputs, cfg)
    gs = build_graph_serial(cov, sparse, m, inputs, cfg)
    assert np.array_equal(gd.indptr, gs.indptr) and np.array_equal(gd.indices, gs.indices)
    # query_boxes: random boxes, some degenerate, some outside, some NaN
    span = m.X.hi - m.X.lo
    q0 = rng.uniform(m.X.lo - 0.2 * span, m.X.hi, (300, m.n))
    q1 = q0 + span * rng.uniform(0, 0.3, (300, m.n)) * (rng.random((300, 1)) < 0.8)
    q0[::37, 0] = np.nan
    da, db = dense.query_boxes(q0, q1)
    sa, sb = sparse.query_boxes(q0, q1)
    assert np.array_equal(da, sa) and np.array_equal(db, sb)
    for fp in (False, True):
        bd = boundary_dev(cov, dense, 0.01, fp)
        bs = boundary_dev(cov, sparse, 0.01, fp)
        assert bool((bd == bs).all())
    for N in (1, 3, 40):
        nd = neighborhood_dev(dense, bd, N)
        ns = neighborhood_dev(sparse, bd, N)
        assert bool((nd == ns).all()), N
    new = cov.retain(rng.random(len(cov)) < 0.5).subdivide(None)
    assert containment_defect(new, cov, dense) == containment_defect(new, cov, sparse)


def _deep_covering(m, point, depth, rng):
    """2-D adaptive covering: every level splits the cells near `point`
    (a shrinking neighbourhood) plus a random few elsewhere."""
    from paper_2202_06111_b200 import Covering

    cov = Covering.initial(m.X)
    p = np.asarray(point)
    for lev in range(depth):
        lo, hi = cov.lo, cov.hi
        w = (m.X.hi - m.X.lo) * 2.0 ** (-(lev // 2)) * 3.0
        near = np.all((lo <= p + w) & (hi >= p - w), axis=1)
        sel = near | (rng.random(len(cov)) < 0.02)
        cov = cov.subdivide(sel)
    return cov


@pytest.mark.parametrize("depth,cfg_id,point", [(40, 1, (0.0, 0.0)), (46, 2, (0.0, 0.0)),
                                                (41, 3, (0.1, 0.6))])
def test_deep_2d_covering_graph_and_queries_vs_oracle(depth, cfg_id, point):
    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import ImageConfig, sample_inputs
    from paper_2202_06111_b200.adaptive import select_boundary_mask
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.configs import config

    rng = np.random.default_rng(depth)
    m = config(cfg_id).model
    cov = _deep_covering(m, point, depth, rng)
    assert int(cov.depths.max()) >= depth
    idx = cov.build_index()
    assert idx.sparse  # too deep for a dense table: chosen automatically
    inputs = sample_inputs(m.U, 5)
    cfg = ImageConfig(2, 0.1)
    g = _graph_vs_oracle(cov, m, inputs, cfg, idx)
    assert g.edge_count > 0
    keep = non_leaving_mask(g)
    assert np.array_equal(keep, O.non_leaving_mask(g.indptr, g.indices, len(cov)))
    tree = O.BoxTree(cov.lo, cov.hi)
    for fp in (False, True):
        want = O.select_boundary_mask(cov.lo, cov.hi, tree, 0.01, fp)
        assert np.array_equal(select_boundary_mask(cov, idx, 0.01, fp), want)
    c = cov.centers()[rng.integers(0, len(cov), 50)]
    span = m.X.hi - m.X.lo
    q0, q1 = c - span * 1e-9, c + span * rng.uniform(0, 1e-3, (50, 2))
    qi, ci = idx.query_boxes(q0, q1)
    oq, oc = tree.query(q0, q1)
    assert np.array_equal(qi, oq) and np.array_equal(ci, oc)


def test_deep_adaptive_run_vs_reference_golden():
    """The reference's own adaptive loop on the 1-D linear model (x+ = 2x +
    u, CIS [-0.5, 0.5]) for 48 iterations: the two boundary points refine to
    depth ~50, far past a dense slot table; metrics and final covering equal
    the reference's (tests/golden/runs.npz linear_n3_48)."""
    from pathlib import Path

    from paper_2202_06111_b200 import AdaptiveConfig, ImageConfig, RunConfig, run
    from paper_2202_06111_b200.system import linear_test_model

    z = np.load(Path(__file__).parent / "golden" / "runs.npz")
    res = run(RunConfig(model=linear_test_model(2.0), iterations=48, input_counts=3,
                        image=ImageConfig(3, 0.05),
                        adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3)))
    want = z["linear_n3_48__metrics"]
    got = np.array([(x.iteration, x.cells_before, x.cells_after, x.edges, x.boundary_cells,
                     x.diameter) for x in res.metrics], dtype=np.float64)
    assert int(res.covering.depths.max()) >= 45
    assert np.array_equal(got, want)
    assert np.array_equal(res.covering.bits, z["linear_n3_48__bits"])
    assert np.array_equal(res.covering.depths, z["linear_n3_48__depths"])
    assert bool(res.containment_ok) == bool(z["linear_n3_48__containment_ok"])


def test_input_grid_441_points_m2_vs_oracle():
    """m = 2 inputs, 21 x 21 grid = 441 points (> 128: K2-general)."""
    from paper_2202_06111_b200 import Box, Covering, ImageConfig, sample_inputs
    from paper_2202_06111_b200.system import affine_test_model

    rng = np.random.default_rng(3)
    A = 0.9 * np.array([[np.cos(0.3), -np.sin(0.3)], [np.sin(0.3), np.cos(0.3)]])
    B = rng.normal(size=(2, 2)) * 0.05
    m = affine_test_model(A, B, [0.01, -0.02], X=Box([-1.0, -1.0], [1.0, 1.0]),
                          U=Box([-1.0, -1.0], [1.0, 1.0]))
    inputs = sample_inputs(m.U, (21, 21))
    assert len(inputs.points) == 441
    cov = Covering.initial(m.X)
    for _ in range(10):
        cov = cov.subdivide(None)
    _graph_vs_oracle(cov, m, inputs, ImageConfig(2, 0.1))
    _graph_vs_oracle(_mixed_covering(rng, m, 11), m, inputs, ImageConfig(3, 0.0))


def test_200_scalar_inputs_vs_oracle():
    from paper_2202_06111_b200 import ImageConfig, sample_inputs
    from paper_2202_06111_b200.configs import config

    m = config(2).model
    rng = np.random.default_rng(4)
    cov = _mixed_covering(rng, m, 12)
    _graph_vs_oracle(cov, m, sample_inputs(m.U, 200), ImageConfig(2, 0.1))
