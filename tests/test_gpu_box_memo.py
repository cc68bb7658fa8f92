"""Box reuse across the coverings of an adaptive run
(gis_build_graph_memo_begin, gis_covering_origin): a cell carried over
unchanged keeps the padded enclosure boxes of the previous build.  The graph
must equal a from-scratch build's, and whole adaptive runs must match with
the reuse on and off (GIS_BOX_MEMO)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _grid(model, depth):
    from paper_2202_06111_b200 import Covering

    cov = Covering.initial(model.X)
    for _ in range(depth):
        cov = cov.subdivide(None)
    return cov


def _step_and_compare(cov0, model, inputs, cfg, rng, keep_frac=0.8, sel_frac=0.3):
    from paper_2202_06111_b200.graph import build_graph_rows, build_graph_rows_memo

    torch = pytest.importorskip("torch")
    ip0, ix0, memo = build_graph_rows_memo(cov0, cov0.build_index(), model, inputs, cfg,
                                           keep_memo=True)
    ref0 = build_graph_rows(cov0, cov0.build_index(), model, inputs, cfg)
    assert torch.equal(ip0, ref0[0]) and torch.equal(ix0, ref0[1])
    keep = rng.random(len(cov0)) < keep_frac
    mid = cov0.retain(keep)
    sel = rng.random(len(mid)) < sel_frac
    cov1 = mid.subdivide(sel)
    origin = cov0.origin_after(keep, sel, cov1).cpu().numpy()
    # origin: unchanged cells point at themselves in cov0
    o = origin >= 0
    assert (~o).sum() == 2 * sel.sum()
    assert np.array_equal(cov1.depths[o], cov0.depths[origin[o]])
    assert np.array_equal(cov1.bits[o], cov0.bits[origin[o]])
    assert np.array_equal(cov1.lo[o], cov0.lo[origin[o]])
    fwd = cov0.forward_after(keep, sel).cpu().numpy()
    # fwd: the inverse of origin on unchanged cells, children of selected ones
    assert np.array_equal(fwd[origin[o]], np.flatnonzero(o))
    assert (fwd == -1).sum() == (~keep).sum()
    split = fwd <= -2
    assert np.array_equal(cov1.depths[-2 - fwd[split]], cov0.depths[split] + 1)
    D = pytest.importorskip("paper_2202_06111_b200._device")
    ref1 = build_graph_rows(cov1, cov1.build_index(), model, inputs, cfg)
    for with_rows in (False, True):
        D.integrations()
        ip1, ix1, _ = build_graph_rows_memo(
            cov1, cov1.build_index(), model, inputs, cfg,
            origin=torch.as_tensor(origin, device="cuda"), memo=memo,
            fwd=torch.as_tensor(fwd, device="cuda") if with_rows else None)
        images, ints = D.integrations()
        assert torch.equal(ip1, ref1[0]) and torch.equal(ix1, ref1[1]), with_rows
    return images, ints


@pytest.mark.parametrize("cid,depth", [(2, 10), (5, 8), (4, 9), (3, 8)])
def test_memo_step_equals_fresh_build(cid, depth):
    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.configs import config

    rc = config(cid)
    m = rc.model
    rng = np.random.default_rng(cid)
    images, ints = _step_and_compare(_grid(m, depth), m, sample_inputs(m.U, 3), rc.image, rng)
    assert ints < images


@pytest.mark.parametrize("share", ["0", "1"])
def test_memo_with_replays_and_sharing(share):
    """pendulum angles outside the polynomial range: pairs replayed by the
    exact kernel keep their boxes too; corner sharing on and off."""
    from paper_2202_06111_b200 import Box, SystemModel, sample_inputs
    from paper_2202_06111_b200.configs import config

    rc = config(2)
    m = rc.model
    wide = SystemModel(m.name, m.n, m.m, Box([-3.0, -4.0], [3.0, 4.0]), m.U, m.step)
    old = os.environ.get("GIS_K1_SHARE")
    os.environ["GIS_K1_SHARE"] = share
    try:
        _step_and_compare(_grid(wide, 9), wide, sample_inputs(wide.U, 3), rc.image,
                          np.random.default_rng(5))
    finally:
        if old is None:
            del os.environ["GIS_K1_SHARE"]
        else:
            os.environ["GIS_K1_SHARE"] = old


def test_memo_nothing_kept_and_everything_selected():
    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.configs import config

    rc = config(2)
    m = rc.model
    cov = _grid(m, 8)
    for kf, sf in [(1.0, 0.0), (1.0, 1.0), (0.05, 0.5)]:
        _step_and_compare(cov, m, sample_inputs(m.U, 3), rc.image, np.random.default_rng(1),
                          keep_frac=kf, sel_frac=sf)


@pytest.mark.parametrize("cid,over", [
    (3, {"iterations": 4}),
    (5, {"initial_grid": (16, 16, 16, 16), "iterations": 3}),
])
def test_adaptive_run_with_and_without_reuse(cid, over):
    from paper_2202_06111_b200 import _device as D, run
    from paper_2202_06111_b200.configs import config

    results = {}
    for flag in ("0", "1"):
        old = os.environ.get("GIS_BOX_MEMO")
        os.environ["GIS_BOX_MEMO"] = flag
        try:
            D.integrations()
            res = run(config(cid, **over))
            results[flag] = (res, D.integrations())
        finally:
            if old is None:
                del os.environ["GIS_BOX_MEMO"]
            else:
                os.environ["GIS_BOX_MEMO"] = old
    (a, (ia, na)), (b, (ib, nb)) = results["0"], results["1"]
    assert np.array_equal(a.covering.depths, b.covering.depths)
    assert np.array_equal(a.covering.bits, b.covering.bits)
    assert [(x.cells_before, x.cells_after, x.edges) for x in a.metrics] == \
        [(x.cells_before, x.cells_after, x.edges) for x in b.metrics]
    assert np.array_equal(a.boundary_mask, b.boundary_mask)
    assert ia == ib and nb < na


@pytest.mark.parametrize("size", [2, 3])
def test_memo_per_rank_row_ranges(size):
    """the multi-GPU engine's reuse (distributed.build_and_prune_sharded,
    memo_io), emulated rank by rank: each rank keeps the boxes of its owned
    rows; in the next covering its rows' origins may point into another
    rank's rows (integrated again).  Row blocks equal the full build's."""
    import torch

    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.distributed import owned_range
    from paper_2202_06111_b200.graph import build_graph_rows, build_graph_rows_memo

    rc = config(5)
    m = rc.model
    inputs = sample_inputs(m.U, 3)
    rng = np.random.default_rng(size)
    cov0 = _grid(m, 8)
    V0 = len(cov0)
    memos = []
    for r in range(size):
        b, e = owned_range(V0, r, size)
        memos.append(build_graph_rows_memo(cov0, cov0.build_index(), m, inputs, rc.image, b, e,
                                           keep_memo=True)[2])
    keep = rng.random(V0) < 0.85
    mid = cov0.retain(keep)
    sel = rng.random(len(mid)) < 0.2
    cov1 = mid.subdivide(sel)
    origin = cov0.origin_after(keep, sel, cov1)
    fwd = cov0.forward_after(keep, sel)
    idx1 = cov1.build_index()
    full_ip, full_ix = build_graph_rows(cov1, idx1, m, inputs, rc.image)
    full_ip, full_ix = full_ip.cpu().numpy(), full_ix.cpu().numpy()
    V1 = len(cov1)
    for r in range(size):
        b, e = owned_range(V1, r, size)
        for f in (None, fwd):
            ip, ix, _ = build_graph_rows_memo(cov1, idx1, m, inputs, rc.image, b, e,
                                              origin=origin, memo=memos[r], fwd=f)
            ip, ix = ip.cpu().numpy(), ix.cpu().numpy()
            assert np.array_equal(ip, full_ip[b:e + 1] - full_ip[b])
            assert np.array_equal(ix, full_ix[full_ip[b]:full_ip[e]])
