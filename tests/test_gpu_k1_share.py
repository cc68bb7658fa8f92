"""Shared grid corners in K1 (EncArgs::S1, csrc/gis_k1.cuh): a cell corner
that is, bit for bit, the lower corner of the cell above it is integrated
once.  The graph must be identical with and without sharing (GIS_K1_SHARE=0)
on uniform and mixed-depth coverings, row ranges, retained coverings with
holes, escaping / non-finite samples and the speculative-trig replay; and
the work counters must say what ran."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _build(cov, model, inputs, cfg, share, rows=None):
    from paper_2202_06111_b200 import _device as D
    from paper_2202_06111_b200.graph import build_graph_rows, build_graph_serial

    old = os.environ.get("GIS_K1_SHARE")
    os.environ["GIS_K1_SHARE"] = "1" if share else "0"
    try:
        D.integrations()  # reset the counters
        index = cov.build_index()
        if rows is None:
            g = build_graph_serial(cov, index, model, inputs, cfg)
            out = (np.asarray(g.indptr).copy(), np.asarray(g.indices).copy())
        else:
            ip, ix = build_graph_rows(cov, index, model, inputs, cfg, *rows)
            out = (ip.cpu().numpy(), ix.cpu().numpy())
        return out, D.integrations()
    finally:
        if old is None:
            del os.environ["GIS_K1_SHARE"]
        else:
            os.environ["GIS_K1_SHARE"] = old


def _same(cov, model, inputs, cfg, rows=None):
    (a, (img0, int0)) = _build(cov, model, inputs, cfg, False, rows)
    (b, (img1, int1)) = _build(cov, model, inputs, cfg, True, rows)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert img0 == img1 == int0  # without sharing every image is one integration
    return img1, int1


def _grid(model, depth):
    from paper_2202_06111_b200 import Covering

    cov = Covering.initial(model.X)
    for _ in range(depth):
        cov = cov.subdivide(None)
    return cov


def _inputs(model, k):
    from paper_2202_06111_b200 import sample_inputs

    return sample_inputs(model.U, k)


def test_pendulum_uniform_counts():
    """config 2's sampling (16 seeded + 4 corners) on a 128^2 grid: 17 + a
    few boundary corners per pair instead of 20."""
    from paper_2202_06111_b200.configs import config

    rc = config(2)
    m = rc.model
    cov = _grid(m, 14)
    V, U = len(cov), 5
    img, ints = _same(cov, m, _inputs(m, U), rc.image)
    assert img == V * U * 20
    side = 128
    # no owner on the root's upper faces: corner (1,0) for the last column,
    # (0,1) for the last row, (1,1) for both
    assert ints == V * U * 17 + (4 * side - 1) * U


@pytest.mark.parametrize("cid,depth,U", [(4, 12, 3), (5, 12, 3), (3, 10, 5), (1, 10, 3)])
def test_models_uniform(cid, depth, U):
    from paper_2202_06111_b200.configs import config

    rc = config(cid)
    m = rc.model
    cov = _grid(m, depth)
    img, ints = _same(cov, m, _inputs(m, U), rc.image)
    assert ints < img


def test_mixed_depth_and_holes():
    """random adaptive coverings (coarse / fine neighbours: T-junction
    corners have no owner) with retained holes (slot -> -1)."""
    from paper_2202_06111_b200 import Covering
    from paper_2202_06111_b200.configs import config

    rng = np.random.default_rng(7)
    for cid in (2, 5):
        rc = config(cid)
        m = rc.model
        cov = Covering.initial(m.X)
        for _ in range(4 * m.n):
            mask = rng.random(len(cov)) < 0.6
            mask[0] = True
            cov = cov.subdivide(mask)
        keep = rng.random(len(cov)) < 0.8
        keep[0] = True
        cov = cov.retain(keep)
        img, ints = _same(cov, m, _inputs(m, 3), rc.image)
        assert ints < img


def test_row_ranges():
    """a row range: owners outside it are integrated by the cell itself."""
    from paper_2202_06111_b200.configs import config

    rc = config(2)
    m = rc.model
    cov = _grid(m, 12)
    V = len(cov)
    for rows in [(0, V), (37, 1000), (V // 2, V), (100, 101)]:
        _same(cov, m, _inputs(m, 3), rc.image, rows)


def test_speculative_replay_and_escaping():
    """pendulum angles beyond the polynomial sin's range flag lower corners
    (kCornerBad) and whole pairs go to the exact replay; CSTR cells near
    T = 0 give non-finite corner images."""
    from paper_2202_06111_b200 import Box, ImageConfig, SystemModel
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.system import CstrParameters, CstrStep

    rc = config(2)
    m = rc.model
    wide = SystemModel(m.name, m.n, m.m, Box([-3.0, -4.0], [3.0, 4.0]), m.U, m.step)
    cov = _grid(wide, 10)
    _same(cov, wide, _inputs(wide, 3), rc.image)
    cstr = SystemModel("cstr", 2, 1, Box([0.0, -0.05], [1.0, 0.05]), Box([285.0], [315.0]),
                       CstrStep(CstrParameters()))
    _same(_grid(cstr, 8), cstr, _inputs(cstr, 3), ImageConfig(3, 0.1))


def test_oracle_parity_with_sharing():
    """the shared build against the CPU oracle (config 5's sampling, 4-D)."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.image import sample_fractions

    rc = config(5)
    m = rc.model
    cov = _grid(m, 8)
    inputs = _inputs(m, 3)
    (ip, ix), (img, ints) = _build(cov, m, inputs, rc.image, True)
    assert ints < img
    frac = sample_fractions(rc.image, m.n)
    oip, oix = O.build_graph(cov.lo, cov.hi, O.make_step(m.step.spec()),
                             np.atleast_2d(inputs.points), frac, rc.image.bloat)
    assert np.array_equal(ip, oip) and np.array_equal(ix, oix)


@pytest.mark.parametrize("mixed", [False, True])
def test_nonuniform_faces_boxes_index(mixed):
    """a monotone warp of the grid (faces far from uniform) through the
    boxes index: the K1 epilogue's slot guesses miss and fall back to
    walking / binary search; graph equal to the oracle, shared or not."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import Covering, SpatialIndex
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.image import sample_fractions

    rc = config(2)
    m = rc.model
    cov = _grid(m, 12)
    if mixed:
        rng = np.random.default_rng(3)
        for _ in range(3):
            cov = cov.subdivide(rng.random(len(cov)) < 0.3)

    def warp(x):
        return np.sign(x) * np.abs(x) ** 2.5

    lo, hi = warp(cov.lo), warp(cov.hi)
    wc = Covering(cov.root, cov.depths, cov.bits, lo, hi)
    inputs = _inputs(m, 3)
    frac = sample_fractions(rc.image, m.n)
    oip, oix = O.build_graph(lo, hi, O.make_step(m.step.spec()), np.atleast_2d(inputs.points),
                             frac, rc.image.bloat)
    for share in (False, True):
        old = os.environ.get("GIS_K1_SHARE")
        os.environ["GIS_K1_SHARE"] = "1" if share else "0"
        try:
            from paper_2202_06111_b200.graph import build_graph_rows

            ip, ix = build_graph_rows(wc, SpatialIndex(lo, hi), m, inputs, rc.image)
        finally:
            if old is None:
                del os.environ["GIS_K1_SHARE"]
            else:
                os.environ["GIS_K1_SHARE"] = old
        assert np.array_equal(ip.cpu().numpy(), oip)
        assert np.array_equal(ix.cpu().numpy(), oix)
