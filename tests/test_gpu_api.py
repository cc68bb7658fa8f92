"""Reference behaviours through the drop-in API on the GPU (ports of the
reference tests that pin this path: tests/test_graph.py, test_geometry.py,
test_adaptive.py, test_engine.py, test_image.py of cisgraph 0.1.0)."""

import math

import numpy as np
import pytest

from conftest import grid_boxes

pytestmark = pytest.mark.gpu


def grid_index(nx, ny, drop=()):
    from types import SimpleNamespace

    from paper_2202_06111_b200 import SpatialIndex

    lo, hi = grid_boxes(nx, ny)
    keep = np.array([i for i in range(nx * ny) if (i + 1) not in set(drop)])
    lo, hi = lo[keep], hi[keep]
    return SimpleNamespace(lo=lo, hi=hi), SpatialIndex(lo, hi, labels=[int(i) + 1 for i in keep])


RING_5X5 = {1, 2, 3, 4, 5, 6, 10, 11, 15, 16, 20, 21, 22, 23, 24, 25}


def test_boundary_worked_grid_and_knn_figures():
    from paper_2202_06111_b200.adaptive import select_boundary, select_neighborhood
    from paper_2202_06111_b200.geometry import knn_centers

    bs, idx = grid_index(5, 5, drop=(25,))
    assert select_boundary(bs, idx, 0.01) == (RING_5X5 - {25}) | {19}
    assert set(knn_centers(idx, [0.5, 0.5], 3).cells) == {2, 6, 7}
    assert set(knn_centers(idx, [0.5, 0.5], 7).cells) == {2, 6, 7, 3, 8, 11, 12}
    bs, idx = grid_index(5, 5, drop=(4,))
    b = select_boundary(bs, idx, 0.01)
    assert 9 not in b and {3, 5, 8, 10} <= b
    assert 9 in select_boundary(bs, idx, 0.01, include_face_points=True)
    assert 9 in select_neighborhood(bs, idx, b, 2)
    bs, idx = grid_index(3, 3)
    assert select_neighborhood(bs, idx, select_boundary(bs, idx, 0.01), 100) == {5}


def test_knn_matches_exhaustive_sort():
    from paper_2202_06111_b200.geometry import knn_centers

    for nx, ny, k in [(10, 10, 7), (100, 100, 12), (57, 31, 5)]:
        _, idx = grid_index(nx, ny)
        rng = np.random.default_rng(nx * ny + k)
        centers = 0.5 * (idx.lo + idx.hi)
        for _ in range(20):
            p = centers[rng.integers(len(centers))] if rng.random() < 0.5 else \
                rng.uniform(-1, nx + 1, 2)
            got = knn_centers(idx, p, k).cells
            d = np.sqrt(((centers - p) ** 2).sum(axis=1))
            cand = np.flatnonzero(~np.all(centers == p, axis=1))
            want = [int(c) + 1 for c in cand[np.lexsort((cand, d[cand]))][:k]]
            assert got == want


def test_knn_clamped_and_zero():
    from paper_2202_06111_b200.geometry import knn_centers

    _, idx = grid_index(2, 1)
    r = knn_centers(idx, [0.5, 0.5], 5)
    assert r.cells == [2] and r.clamped
    _, idx = grid_index(5, 5)
    r = knn_centers(idx, [0.5, 0.5], 0)
    assert r.cells == [] and not r.clamped
    _, idx = grid_index(3, 1)
    assert knn_centers(idx, [0.51, 0.5], 3).cells == [1, 2, 3]


def test_query_boxes_vs_linear_scan_and_touching():
    from paper_2202_06111_b200 import Box, Covering
    from paper_2202_06111_b200.geometry import query_intersecting

    rng = np.random.default_rng(13)
    cov = Covering.initial(Box([-1.0, -1.0], [2.0, 1.0]))
    for _ in range(7):
        cov = cov.subdivide(rng.random(len(cov)) < 0.7)
    cov = cov.retain(rng.random(len(cov)) < 0.8)
    idx = cov.build_index()
    qlo = rng.uniform(-1.5, 2.0, (1000, 2))
    qhi = qlo + rng.uniform(0.0, 0.8, (1000, 2))
    qi, ci = idx.query_boxes(qlo, qhi)
    got = set(zip(qi.tolist(), ci.tolist()))
    want = set()
    for q in range(1000):
        m = np.all(qlo[q] <= cov.hi, axis=1) & np.all(cov.lo <= qhi[q], axis=1)
        want |= {(q, int(c)) for c in np.flatnonzero(m)}
    assert got == want
    c2 = Covering.initial(Box([0.0, 0.0], [1.0, 1.0])).subdivide(None)
    assert len(query_intersecting(c2.build_index(), Box([0.5, 0.2], [0.5, 0.3]))) == 2


@pytest.mark.parametrize("k", range(1, 7))
def test_subdivision_closed_form(k):
    from paper_2202_06111_b200 import Box, Covering

    cov = Covering.initial(Box([0.0, 0.0], [1.0, 1.0]))
    for _ in range(k):
        cov = cov.subdivide(None)
    assert len(cov) == 2 ** k
    w = cov.hi - cov.lo
    assert np.all(w[:, 0] == 2.0 ** -math.ceil(k / 2))
    assert np.all(w[:, 1] == 2.0 ** -math.floor(k / 2))
    assert cov.diameter() == pytest.approx(math.hypot(w[0, 0], w[0, 1]), rel=1e-15)
    assert cov.verify_reconstruction()


def test_covering_canonical_order_and_duplicates():
    from paper_2202_06111_b200 import Box, CellId, Covering

    root = Box([0.0], [1.0])
    with pytest.raises(ValueError):
        Covering(root, [1, 1], [0, 0], [[0.0], [0.0]], [[0.5], [0.5]])
    rng = np.random.default_rng(7)
    cov = Covering.initial(Box([-1.0, 345.0], [1.0, 355.0]))
    for _ in range(8):
        cov = cov.subdivide(rng.random(len(cov)) < 0.7)
    perm = rng.permutation(len(cov))
    shuffled = Covering(cov.root, cov.depths[perm], cov.bits[perm], cov.lo[perm], cov.hi[perm])
    assert np.array_equal(shuffled.bits, cov.bits) and np.array_equal(shuffled.lo, cov.lo)
    ids = cov.cell_ids()
    assert ids == sorted(ids)
    assert CellId.from_path("01").child(1).path == "011"


def test_graph_api_behaviours():
    from paper_2202_06111_b200 import ImageConfig, sample_inputs
    from paper_2202_06111_b200.graph import (BuildPlan, OwnershipError, SymbolicImage,
                                             build_graph_parallel, build_graph_serial,
                                             merge_subgraphs)
    from paper_2202_06111_b200.system import cstr_model, linear_test_model

    m = cstr_model()
    from paper_2202_06111_b200 import Covering
    cov = Covering.initial(m.X)
    for _ in range(6):
        cov = cov.subdivide(None)
    idx = cov.build_index()
    inp = sample_inputs(m.U, 3)
    serial = build_graph_serial(cov, idx, m, inp, ImageConfig())
    exports = {build_graph_parallel(cov, idx, m, inp, ImageConfig(), p).edge_list_bytes()
               for p in [BuildPlan(1024, 1), BuildPlan(64, 2), BuildPlan(5, 2)]}
    assert exports == {serial.edge_list_bytes()}
    src, dst = serial.edge_pairs()
    half = len(cov) // 2
    from oracle import gis_oracle as O
    parts = []
    for owned in (np.arange(half), np.arange(half, len(cov))):
        mk = np.isin(src, owned)
        ip, ix = O.csr_from_pairs(src[mk], dst[mk], len(cov))
        parts.append(SymbolicImage(cov.depths, cov.bits, ip, ix, owned=owned))
    assert merge_subgraphs(parts).same_edges(serial)
    assert merge_subgraphs(parts[::-1]).same_edges(serial)
    bad = SymbolicImage(cov.depths, cov.bits, parts[1].indptr, parts[1].indices,
                        owned=np.concatenate([parts[1].owned, parts[0].owned[:1]]))
    with pytest.raises(OwnershipError):
        merge_subgraphs([parts[0], bad])
    with pytest.raises(KeyError):
        serial.out_degree(len(cov) + 5)


def test_engine_behaviours():
    from paper_2202_06111_b200 import AdaptiveConfig, ImageConfig, RunConfig, run
    from paper_2202_06111_b200.system import cstr_model, identity_model, shift_model

    res = run(RunConfig(model=identity_model(), iterations=5, image=ImageConfig(2, 0.0)))
    assert res.termination == "iterations"
    assert all(m.cells_before == m.cells_after for m in res.metrics)
    res = run(RunConfig(model=shift_model(), iterations=5))
    assert res.termination == "empty" and len(res.metrics) == 1 and res.empty
    res = run(RunConfig(model=cstr_model(), iterations=1))
    assert res.metrics[0].cells_before == 4 and (res.covering.depths == 2).all()
    full = run(RunConfig(model=cstr_model(), iterations=9))
    adap = run(RunConfig(model=cstr_model(), iterations=9,
                         adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3)))
    assert len(adap.covering) < len(full.covering) and adap.containment_ok
    res = run(RunConfig(model=identity_model(), iterations=50, min_diameter=0.1,
                        image=ImageConfig(2, 0.0)))
    assert res.termination == "min_diameter" and res.covering.diameter() <= 0.1


def test_no_cpu_fallback_for_python_callables():
    from paper_2202_06111_b200 import Box, ImageConfig, SystemModel, sample_inputs, Covering
    from paper_2202_06111_b200.graph import build_graph_serial

    class Boom:
        def __call__(self, x, u):
            raise RuntimeError("vector field blew up")

    m = SystemModel("boom", 1, 1, Box([0.0], [1.0]), Box([0.0], [0.0]), step=Boom())
    cov = Covering.initial(m.X).subdivide(None)
    with pytest.raises(TypeError, match="not a device model"):
        build_graph_serial(cov, cov.build_index(), m, sample_inputs(m.U, 2), ImageConfig(2, 0))


def test_native_library_is_loaded_and_launches():
    from paper_2202_06111_b200 import _device as D

    import paper_2202_06111_b200.system as S
    before = D.launch_count()
    S.cstr_model().step(np.array([[0.5, 350.0]]), np.array([300.0]))
    assert D.launch_count() > before


def test_csr_from_pairs_matches_oracle():
    """gis_csr_from_pairs (merge_subgraphs' union) equals _csr_from_pairs
    (cg/graph.py:181-193) on random pairs with duplicates; out-of-range
    endpoints raise."""
    import ctypes as C

    import torch

    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import _device as D

    lib = D.load_library()
    rng = np.random.default_rng(19)
    for V, n in [(1, 5), (7, 60), (1000, 5000), (100_000, 1_000_000)]:
        src = rng.integers(0, V, n)
        dst = rng.integers(0, V, n)
        ip_w, ix_w = O.csr_from_pairs(src, dst, V)
        s_t, d_t = D.to_dev(src.astype(np.int64)), D.to_dev(dst.astype(np.int64))
        ip = torch.empty(V + 1, dtype=torch.int64, device="cuda")
        ix = torch.empty(n, dtype=torch.int32, device="cuda")
        E = C.c_int64()
        D.check(lib.gis_csr_from_pairs(D.ctx(), D.ptr(s_t), D.ptr(d_t), n, V, D.ptr(ip),
                                       D.ptr(ix), C.byref(E)))
        assert np.array_equal(ip.cpu().numpy(), ip_w)
        assert np.array_equal(ix[:E.value].cpu().numpy(), ix_w)
    bad = D.to_dev(np.array([0, 5], dtype=np.int64))
    ip = torch.empty(3, dtype=torch.int64, device="cuda")
    ix = torch.empty(2, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        D.check(lib.gis_csr_from_pairs(D.ctx(), D.ptr(bad), D.ptr(bad), 2, 2, D.ptr(ip),
                                       D.ptr(ix), C.byref(C.c_int64())))


def test_covering_from_pinned_host_tensors_uploads_async():
    """Pinned host tensors upload without blocking (stream-ordered); the graph
    built right after equals the one from numpy arrays."""
    import torch

    from paper_2202_06111_b200 import Covering, sample_inputs
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.graph import build_graph_serial

    rc = config(1)
    m = rc.model
    cov = Covering.initial(m.X)
    for _ in range(12):
        cov = cov.subdivide(None)
    inputs = sample_inputs(m.U, rc.input_counts)
    want = build_graph_serial(cov, cov.build_index(), m, inputs, rc.image)
    for _ in range(3):
        pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
               for x in (cov.depths, cov.bits, cov.lo, cov.hi)]
        c2 = Covering(m.X, *pin, _sorted=True)
        del pin  # the pinned blocks must outlive the copies: torch keeps them
        g = build_graph_serial(c2, c2.build_index(), m, inputs, rc.image)
        assert g.same_edges(want)


@pytest.mark.parametrize("n,depth,limits", [(1, 0, None), (1, 7, None), (2, 9, None),
                                            (2, 8, (11, 16)), (3, 10, (3, 4, 2)),
                                            (4, 12, (6, 5, 8, 7)), (4, 24, (48, 48, 48, 48))])
def test_uniform_grid_equals_repeated_subdivision(n, depth, limits):
    """Covering.uniform (gis_uniform_grid) == `depth` rounds of subdivide on
    the one-cell covering (+ the grid mask): same cells, bounds, order."""
    from paper_2202_06111_b200 import Box, Covering

    rng = np.random.default_rng(depth)
    lo = rng.uniform(-3, 0, n)
    root = Box(lo, lo + rng.uniform(0.1, 5, n))
    got = Covering.uniform(root, depth, limits)
    want = Covering._uniform_by_splits(root, depth, None if limits is None
                                       else np.asarray(limits, dtype=np.int64))
    assert len(got) == len(want)
    for a, b in ((got.depths, want.depths), (got.bits, want.bits), (got.lo, want.lo),
                 (got.hi, want.hi)):
        assert np.array_equal(a, b)


def test_engine_outputs_and_stop_rules(tmp_path):
    """The reference's tests/test_engine.py output and stop-rule behaviours
    (:50-163) restated: full mode doubles before retention, snapshots and the
    kept final graph, plan independence, check_stop, reproducible output
    files, the cells file's status column, metrics / timings headers, the
    summary of an emptied run, and edges requiring a kept graph."""
    import filecmp
    from pathlib import Path

    from paper_2202_06111_b200 import Covering, ImageConfig, RunConfig, run
    from paper_2202_06111_b200.engine import check_stop, write_run_outputs
    from paper_2202_06111_b200.geometry import read_cells_file
    from paper_2202_06111_b200.graph import BuildPlan
    from paper_2202_06111_b200.system import cstr_model, identity_model, shift_model

    res = run(RunConfig(model=cstr_model(), iterations=6))
    for prev, cur in zip(res.metrics, res.metrics[1:]):
        assert cur.cells_before == 2 * prev.cells_after
    assert res.containment_ok
    res = run(RunConfig(model=cstr_model(), iterations=4, snapshot_iterations=(2, 3),
                        keep_final_graph=True))
    assert set(res.snapshots) == {2, 3}
    assert res.final_graph is not None
    assert res.final_graph.n_vertices == res.metrics[-1].cells_before
    serial = run(RunConfig(model=cstr_model(), iterations=5))
    par = run(RunConfig(model=cstr_model(), iterations=5, plan=BuildPlan(batch_size=16, workers=2)))
    assert np.array_equal(serial.covering.bits, par.covering.bits)
    assert [m.edges for m in serial.metrics] == [m.edges for m in par.metrics]

    cfg = RunConfig(model=identity_model(), iterations=20)
    cov = Covering.initial(identity_model().X)
    assert check_stop(20, cov, cfg) == "iterations" and check_stop(19, cov, cfg) is None
    cfg = RunConfig(model=identity_model(), iterations=50, min_diameter=0.3)
    assert check_stop(1, cov, cfg) is None
    assert check_stop(2, cov.subdivide(None).subdivide(None), cfg) == "min_diameter"

    kw = dict(model=cstr_model(), iterations=5, keep_final_graph=True)
    a = write_run_outputs(run(RunConfig(**kw)), tmp_path / "a", export_edges=True)
    b = write_run_outputs(run(RunConfig(**kw)), tmp_path / "b", export_edges=True)
    for key in ("cells", "metrics", "summary", "edges"):
        assert filecmp.cmp(a[key], b[key], shallow=False), key
    res = run(RunConfig(model=cstr_model(), iterations=4))
    paths = write_run_outputs(res, tmp_path / "c")
    with open(paths["cells"]) as fp:
        cov2, status = read_cells_file(fp)
    assert len(cov2) == len(res.covering)
    assert set(status) <= {"boundary", "interior"}
    assert status.count("boundary") == int(res.boundary_mask.sum())
    res = run(RunConfig(model=identity_model(), iterations=3, image=ImageConfig(2, 0.0)))
    paths = write_run_outputs(res, tmp_path / "d")
    assert Path(paths["metrics"]).read_text().splitlines()[0].split("\t") == [
        "iteration", "cells_before", "cells_after", "edges", "boundary_cells", "diameter"]
    assert Path(paths["timings"]).read_text().splitlines()[0].split("\t") == [
        "iteration", "t_subdivide_ms", "t_build_ms", "t_analyze_ms"]
    with pytest.raises(ValueError):
        write_run_outputs(res, tmp_path / "e", export_edges=True)
    text = Path(write_run_outputs(run(RunConfig(model=shift_model(), iterations=2)),
                                  tmp_path / "f")["summary"]).read_text()
    assert "final_cells = 0" in text and "termination = empty" in text


def test_cell_image_behaviours():
    """The reference's tests/test_image.py:47-177 restated on K1
    (cell_image / cell_images through gis_batch_enclosures): identity
    equality and bloat superset, the linear endpoint image, random-point
    containment for the CSTR cell, input order, nesting under cell growth,
    soundness at the sample points, bloat monotonicity, and the exact
    vertex bounding box of affine maps."""
    from paper_2202_06111_b200 import Box, ImageConfig, sample_inputs
    from paper_2202_06111_b200.image import cell_image, cell_images, cell_sample_points
    from paper_2202_06111_b200.system import (affine_test_model, cstr_model, identity_model,
                                              linear_test_model)

    box = Box([0.25], [0.5])
    assert cell_image(identity_model(), box, np.array([0.0]), ImageConfig(3, 0.0)) == box
    enc = cell_image(identity_model(), box, np.array([0.0]), ImageConfig(3, 0.2))
    assert enc.lo[0] < box.lo[0] and enc.hi[0] > box.hi[0]
    assert cell_image(linear_test_model(2.0), Box([0.0], [0.1]), np.array([0.0]),
                      ImageConfig(3, 0.0)) == Box([0.0], [0.2])

    m = cstr_model()
    box = Box([0.475, 349.75], [0.525, 350.25])
    pts = np.random.default_rng(7).uniform(box.lo, box.hi, (200, 2))
    for u in sample_inputs(m.U, 3):
        imgs = np.asarray(m.map_points(pts, u))
        enc = cell_image(m, box, u, ImageConfig(3, 0.05))
        assert np.all(imgs >= enc.lo) and np.all(imgs <= enc.hi)

    out = cell_images(linear_test_model(2.0), Box([0.0], [0.1]),
                      sample_inputs(linear_test_model(2.0).U, 3), ImageConfig(2, 0.0))
    assert [u[0] for u, _ in out] == [-0.5, 0.0, 0.5]
    for _, enc in cell_images(identity_model(), Box([0.125], [0.375]),
                              sample_inputs(identity_model().U, 2), ImageConfig(2, 0.0)):
        assert enc.lo[0] <= 0.125 and enc.hi[0] >= 0.375

    rng = np.random.default_rng(17)
    m = affine_test_model(rng.normal(size=(2, 2)), rng.normal(size=(2, 1)), rng.normal(size=2),
                          X=Box([-5.0, -5.0], [5.0, 5.0]), U=Box([-1.0], [1.0]))
    grid = sample_inputs(m.U, 3)
    for _ in range(20):
        lo = rng.uniform(-2, 1, 2)
        w = rng.uniform(0.1, 1, 2)
        small = Box(lo, lo + w)
        big = Box(lo - rng.uniform(0, 0.5, 2), lo + w + rng.uniform(0, 0.5, 2))
        for (_, s), (_, b) in zip(cell_images(m, small, grid, ImageConfig(3, 0.07)),
                                  cell_images(m, big, grid, ImageConfig(3, 0.07))):
            assert np.all(b.lo <= s.lo) and np.all(b.hi >= s.hi)

    rng = np.random.default_rng(23)
    for m in (cstr_model(),
              affine_test_model(rng.normal(size=(2, 2)), rng.normal(size=(2, 1)),
                                rng.normal(size=2), X=Box([-5.0, -5.0], [5.0, 5.0]),
                                U=Box([-1.0], [1.0]))):
        grid = sample_inputs(m.U, 3)
        for _ in range(10):
            lo = rng.uniform(m.X.lo, m.X.center)
            hi = rng.uniform(lo, m.X.hi)
            box = Box(lo, np.maximum(hi, lo + 1e-6))
            for spd in (2, 3, 4):
                pts = cell_sample_points(box, spd)
                for u, enc in cell_images(m, box, grid, ImageConfig(spd, 0.0)):
                    mapped = np.asarray(m.map_points(pts, u))
                    assert np.all(mapped >= enc.lo) and np.all(mapped <= enc.hi)

    rng = np.random.default_rng(29)
    m = cstr_model()
    for _ in range(10):
        lo = rng.uniform([0.0, 345.0], [0.8, 353.0])
        box = Box(lo, lo + rng.uniform([0.01, 0.1], [0.2, 2.0]))
        bloats = sorted(rng.uniform(0, 0.5, 3))
        for u in sample_inputs(m.U, 3):
            encs = [cell_image(m, box, u, ImageConfig(3, b)) for b in bloats]
            for s, b in zip(encs, encs[1:]):
                assert np.all(b.lo <= s.lo) and np.all(b.hi >= s.hi)

    rng = np.random.default_rng(31)
    for _ in range(25):
        A, B, c = rng.normal(size=(2, 2)), rng.normal(size=(2, 1)), rng.normal(size=2)
        m = affine_test_model(A, B, c, X=Box([-9.0, -9.0], [9.0, 9.0]), U=Box([-1.0], [1.0]))
        lo = rng.uniform(-2, 2, 2)
        box = Box(lo, lo + rng.uniform(0.1, 2, 2))
        u = rng.uniform(-1, 1, 1)
        enc = cell_image(m, box, u, ImageConfig(2, 0.0))
        center = A @ box.center + B @ u + c
        hw = np.abs(A) @ box.half_widths
        assert enc.lo == pytest.approx(center - hw, rel=1e-12, abs=1e-12)
        assert enc.hi == pytest.approx(center + hw, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("model_dim", [1, 2])
def test_graph_refinement_and_soundness(model_dim):
    """The reference's tests/test_graph.py:59-89 and :211-242 restated:
    every recorded edge has a per-input enclosure meeting its target, the
    8-cell linear graph equals a brute-force double loop, and with the
    coarse sample points kept every coarse edge i -> j has a child edge
    i' -> j' one subdivision finer."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import Box, Covering, ImageConfig, sample_inputs
    from paper_2202_06111_b200.graph import build_graph_serial
    from paper_2202_06111_b200.image import cell_images, sample_fractions
    from paper_2202_06111_b200.system import affine_test_model, linear_test_model

    if model_dim == 1:
        m = linear_test_model(2.0)
    else:
        m = affine_test_model([[0.9, 0.3], [-0.2, 0.8]], [[0.5], [0.2]], [0.05, -0.02],
                              X=Box([-1.0, -1.0], [1.0, 1.0]), U=Box([-0.5], [0.5]))
    inputs = sample_inputs(m.U, 3)

    rng = np.random.default_rng(5)
    cov = Covering.initial(m.X)
    for _ in range(4):
        cov = cov.subdivide(rng.random(len(cov)) < 0.8)
    cov = cov.retain(rng.random(len(cov)) < 0.7)
    cfg = ImageConfig(3, 0.1)
    g = build_graph_serial(cov, cov.build_index(), m, inputs, cfg)
    src, dst = g.edge_pairs()
    for s, d in zip(src.tolist(), dst.tolist()):
        encs = [e for _, e in cell_images(m, cov.box_at(s), inputs, cfg) if e]
        assert any(e.intersects(cov.box_at(d)) for e in encs)

    cov = Covering.initial(m.X)
    for _ in range(3 * m.n):
        cov = cov.subdivide(None)
    cfg0 = ImageConfig(3, 0.0)
    g = build_graph_serial(cov, cov.build_index(), m, inputs, cfg0)
    step = O.make_step(m.step.spec())
    pairs = set()
    for u in inputs.points:
        elo, ehi, valid = O.enclosures(step, cov.lo, cov.hi, u, sample_fractions(cfg0, m.n), 0.0)
        for i in np.flatnonzero(valid):
            hit = np.all(elo[i] <= cov.hi, axis=1) & np.all(cov.lo <= ehi[i], axis=1)
            pairs.update((int(i), int(j)) for j in np.flatnonzero(hit))
    src, dst = g.edge_pairs()
    got = set(zip(src.tolist(), dst.tolist()))
    if got != pairs:  # only near-face ties may differ (bloat 0: bounds can sit on faces)
        from helpers import explain_edge_diffs

        ip, ix = O.csr_from_pairs(np.array([p[0] for p in sorted(pairs)], dtype=np.int64),
                                  np.array([p[1] for p in sorted(pairs)], dtype=np.int64),
                                  len(cov))
        ex, unex = explain_edge_diffs(cov.lo, cov.hi, step, np.atleast_2d(inputs.points),
                                      sample_fractions(cfg0, m.n), 0.0,
                                      (g.indptr, g.indices), (ip, ix))
        assert not unex, unex[:10]
        assert len(ex) <= 2

    coarse = Covering.initial(m.X)
    for _ in range(2 * m.n):
        coarse = coarse.subdivide(None)
    fine = coarse.subdivide(None)
    g_coarse = build_graph_serial(coarse, coarse.build_index(), m, inputs, cfg)
    g_fine = build_graph_serial(fine, fine.build_index(), m, inputs, cfg)
    fs, fd = g_fine.edge_pairs()
    fine_pairs = {(fine.cell_id_at(s).parent(), fine.cell_id_at(d).parent())
                  for s, d in zip(fs.tolist(), fd.tolist())}
    cs, cd = g_coarse.edge_pairs()
    for s, d in zip(cs.tolist(), cd.tolist()):
        assert (coarse.cell_id_at(s), coarse.cell_id_at(d)) in fine_pairs


def test_adaptive_selection_behaviours():
    """The reference's tests/test_adaptive.py:33-200 restated on the K4
    selector kernels: single cell, uniform and dyadic rings, full mode,
    N = 0, huge N behaves like full, subdivide_selected growth and volume,
    and boundary-band refinement of a disk."""
    from paper_2202_06111_b200 import AdaptiveConfig, Box, Covering
    from paper_2202_06111_b200.adaptive import (select_boundary, select_boundary_mask,
                                                select_for_subdivision,
                                                select_for_subdivision_mask,
                                                subdivide_selected)

    bs, idx = grid_index(1, 1)
    assert select_boundary(bs, idx, 0.01) == {1}
    bs, idx = grid_index(6, 6)
    ring = {r * 6 + c + 1 for r in range(6) for c in range(6) if r in (0, 5) or c in (0, 5)}
    assert select_boundary(bs, idx, 0.01) == ring and len(ring) == 20
    cov = Covering.initial(Box([0.0, 0.0], [1.0, 1.0]))
    for _ in range(6):
        cov = cov.subdivide(None)
    c = cov.centers()
    on_ring = (c[:, 0] < 0.125) | (c[:, 0] > 0.875) | (c[:, 1] < 0.125) | (c[:, 1] > 0.875)
    assert np.array_equal(select_boundary_mask(cov, cov.build_index(), 0.01), on_ring)

    bs, idx = grid_index(4, 6)
    assert select_for_subdivision(bs, idx, AdaptiveConfig(mode="full")) == set(range(1, 25))
    bs, idx = grid_index(5, 5, drop=(25,))
    assert select_for_subdivision(bs, idx, AdaptiveConfig(mode="adaptive", n_neighbors=0)) == \
        (RING_5X5 - {25}) | {19}
    cov = Covering.initial(Box([0.0, 0.0], [1.0, 1.0]))
    for _ in range(5):
        cov = cov.subdivide(None)
    sel = select_for_subdivision_mask(cov, cov.build_index(),
                                      AdaptiveConfig(mode="adaptive", n_neighbors=1000))
    assert sel.all()
    a, b = subdivide_selected(cov, sel), subdivide_selected(cov, None)
    assert np.array_equal(a.bits, b.bits) and np.array_equal(a.depths, b.depths)

    cov = Covering.initial(Box([0.0, 0.0], [1.0, 1.0]))
    for _ in range(4):
        cov = cov.subdivide(None)
    assert len(subdivide_selected(cov, None)) == 2 * len(cov)
    assert np.array_equal(subdivide_selected(cov, np.zeros(len(cov), dtype=bool)).bits, cov.bits)
    mask = np.random.default_rng(3).random(len(cov)) < 0.4
    assert len(subdivide_selected(cov, mask)) == len(cov) + int(mask.sum())
    mask = np.random.default_rng(5).random(len(cov)) < 0.5
    assert subdivide_selected(cov, mask).volume() == pytest.approx(cov.volume(), rel=1e-12)

    center, radius = np.array([0.5, 0.5]), 0.35

    def disk(cv):
        nearest = np.clip(center, cv.lo, cv.hi)
        return ((nearest - center) ** 2).sum(axis=1) <= radius ** 2

    cov = Covering.initial(Box([0.0, 0.0], [1.0, 1.0])).subdivide(None).subdivide(None)
    cov = cov.retain(disk(cov))
    for _ in range(6):
        sel = select_for_subdivision_mask(cov, cov.build_index(),
                                          AdaptiveConfig(mode="adaptive", n_neighbors=1))
        cov = subdivide_selected(cov, sel)
        cov = cov.retain(disk(cov))
    far = np.where(cov.lo < center, cov.lo, cov.hi)
    max_d = np.sqrt(((far - center) ** 2).sum(axis=1))
    min_d = np.sqrt(((np.clip(center, cov.lo, cov.hi) - center) ** 2).sum(axis=1))
    straddle = (min_d <= radius) & (max_d >= radius)
    deep = max_d <= 0.6 * radius
    assert straddle.any() and deep.any()
    assert cov.depths[straddle].min() > cov.depths[deep].max()


def test_system_model_behaviours():
    """The reference's tests/test_system.py:40-125 restated on the device
    integrator: fourth-order convergence of RK4 against a tight solve_ivp,
    the CSTR equilibrium as a fixed point, vectorised = scalar steps, the
    test models' steps, constraint boxes / defaults / rejection, pickling."""
    import pickle

    from scipy.integrate import solve_ivp
    from scipy.optimize import fsolve

    from paper_2202_06111_b200 import Box, CstrParameters
    from paper_2202_06111_b200.system import (CstrStep, cstr_model, identity_model,
                                              linear_test_model, rk4_discretize, shift_model)

    step = CstrStep(CstrParameters())
    rng = np.random.default_rng(42)
    p = CstrParameters()

    def rhs_np(y, u):  # cg/system.py:148-166 in numpy, for the reference solution
        ca, t = y
        rate = p.k0 * np.exp(-p.E_over_R / t) * ca
        return [p.q / p.V * (p.c_Af - ca) - rate,
                p.q / p.V * (p.T_f - t) + p.minus_dH / (p.rho * p.c_p) * rate
                + p.UA / (p.V * p.rho * p.c_p) * (u[0] - t)]

    ratios = []
    for _ in range(100):
        x = np.array([rng.uniform(0, 1), rng.uniform(345, 355)])
        u = np.array([rng.uniform(285, 315)])
        ref = solve_ivp(lambda t, y: rhs_np(y, u), (0.0, 0.1), x, rtol=1e-12, atol=1e-12).y[:, -1]
        err_h = np.linalg.norm(np.asarray(step(x, u)) - ref)
        half = rk4_discretize(step.rhs, rk4_discretize(step.rhs, x, u, 0.05), u, 0.05)
        err_h2 = np.linalg.norm(np.asarray(half) - ref)
        if err_h2 > 1e-14:
            ratios.append(err_h / err_h2)
    assert 10 < np.median(ratios) < 30

    u = np.array([300.0])
    eq = fsolve(lambda x: np.asarray(step.rhs(np.asarray(x), u)), [0.5, 350.0], xtol=1e-13)
    assert np.linalg.norm(np.asarray(step.rhs(np.asarray(eq), u))) < 1e-9
    assert np.asarray(step(np.asarray(eq), u)) == pytest.approx(eq, abs=1e-9)

    m = cstr_model()
    assert m.X == Box([0.0, 345.0], [1.0, 355.0]) and m.U == Box([285.0], [315.0])
    assert (m.n, m.m) == (2, 1)
    assert (p.q, p.V, p.c_Af, p.T_f, p.E_over_R, p.k0) == (100.0, 100.0, 1.0, 350.0, 8750.0, 7.2e10)
    with pytest.raises(ValueError):
        CstrParameters(q=0.0)
    pts = np.column_stack([rng.uniform(0, 1, 50), rng.uniform(345, 355, 50)])
    batch = np.asarray(m.map_points(pts, np.array([290.0])))
    for i in range(0, 50, 7):
        assert np.array_equal(batch[i], np.asarray(m.step(pts[i], np.array([290.0]))).reshape(-1))

    lin = linear_test_model(2.0)
    assert np.asarray(lin.step(np.array([0.25]), np.array([-0.5]))).reshape(-1)[0] == 0.0
    assert np.asarray(identity_model().step(np.array([0.3]), np.array([0.0]))).reshape(-1)[0] == 0.3
    assert np.asarray(shift_model(10.0).step(np.array([0.3]), np.array([0.0]))).reshape(-1)[0] == 10.3
    for mm in (cstr_model(), linear_test_model(2.0), identity_model(), shift_model()):
        clone = pickle.loads(pickle.dumps(mm))
        x = np.full(mm.n, float(np.mean(mm.X.lo)))
        assert np.array_equal(np.asarray(clone.step(x, mm.U.lo.copy())),
                              np.asarray(mm.step(x, mm.U.lo.copy())))


def test_retain_behaviours():
    """The reference's tests/test_analysis.py:98-138 restated: retain by
    mask (all / none) and by cell ids, and the 8-cell linear retention equal
    to the peeling fixed point of its symbolic image."""
    from conftest import peeling_fixed_point

    from paper_2202_06111_b200 import Box, Covering, ImageConfig, sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_mask, retain
    from paper_2202_06111_b200.graph import build_graph_serial
    from paper_2202_06111_b200.system import linear_test_model

    cov = Covering.initial(Box([0.0], [1.0]))
    for _ in range(3):
        cov = cov.subdivide(None)
    assert np.array_equal(retain(cov, np.ones(len(cov), dtype=bool)).lo, cov.lo)
    assert len(retain(cov, np.zeros(len(cov), dtype=bool))) == 0
    assert len(retain(cov, {cov.cell_id_at(0), cov.cell_id_at(3)})) == 2

    m = linear_test_model(2.0)
    cov = Covering.initial(m.X)
    for _ in range(3):
        cov = cov.subdivide(None)
    g = build_graph_serial(cov, cov.build_index(), m, sample_inputs(m.U, 3), ImageConfig(3, 0.05))
    src, dst = g.edge_pairs()
    want = peeling_fixed_point(len(cov), list(zip(src.tolist(), dst.tolist())))
    got = non_leaving_mask(g)
    assert np.array_equal(got, want)
    assert len(retain(cov, got)) == int(want.sum())


def test_covering_index_and_cells_file_behaviours():
    """The reference's tests/test_geometry.py:141-300 restated: volume
    partition of random coverings, reconstruction from paths, retain /
    growth, empty covering diameter, single-cell and root queries, empty
    index, off-centre k-NN without exclusion, and the cells-file round trip
    (exact bounds, status column, '-' root, missing header rejected)."""
    import io

    from paper_2202_06111_b200 import Box, Covering, SpatialIndex
    from paper_2202_06111_b200.geometry import (knn_centers, query_intersecting, read_cells_file,
                                                write_cells_file)

    def random_covering(rng, root, rounds, keep_fraction=1.0):
        cov = Covering.initial(root)
        for _ in range(rounds):
            mask = rng.random(len(cov)) < 0.7
            if not mask.any():
                mask[rng.integers(len(cov))] = True
            cov = cov.subdivide(mask)
        if keep_fraction < 1.0:
            keep = rng.random(len(cov)) < keep_fraction
            if not keep.any():
                keep[rng.integers(len(cov))] = True
            cov = cov.retain(keep)
        return cov

    rng = np.random.default_rng(11)
    root = Box([-2.0, 1.0], [3.0, 4.0])
    for _ in range(10):
        cov = random_covering(rng, root, int(rng.integers(3, 9)))
        assert cov.volume() == pytest.approx(root.volume, rel=1e-12)
    root = Box([-1.0, 345.0], [1.0, 355.0])
    cov = random_covering(np.random.default_rng(7), root, 8, 0.6)
    assert cov.verify_reconstruction()
    rebuilt = Covering.from_paths(root, cov.paths())
    assert np.array_equal(rebuilt.lo, cov.lo) and np.array_equal(rebuilt.hi, cov.hi)

    unit = Box([0.0, 0.0], [1.0, 1.0])
    cov = Covering.initial(unit)
    for _ in range(4):
        cov = cov.subdivide(None)
    kept = cov.retain(np.arange(5))
    assert len(kept) == 5 and len(kept.subdivide(np.array([0, 1]))) == 7
    empty = Covering.initial(unit).retain(np.array([], dtype=np.int64))
    assert len(empty) == 0 and empty.diameter() == 0.0
    index = cov.build_index()
    t = cov.box_at(7)
    assert query_intersecting(index, Box(t.center - 1e-3, t.center + 1e-3)) == [cov.cell_id_at(7)]
    c3 = Covering.initial(unit)
    for _ in range(3):
        c3 = c3.subdivide(None)
    assert len(query_intersecting(c3.build_index(), unit)) == len(c3)
    qi, ci = SpatialIndex(np.empty((0, 2)), np.empty((0, 2))).query_boxes(np.zeros((3, 2)),
                                                                          np.ones((3, 2)))
    assert len(qi) == 0 and len(ci) == 0
    _, idx = grid_index(5, 5)
    r = knn_centers(idx, [0.5, 0.5], 3)
    assert set(r.cells) == {2, 6, 7} and not r.clamped

    rng = np.random.default_rng(23)
    root = Box([0.1234567890123456, -7.0], [9.87654321e3, 355.0])
    cov = random_covering(rng, root, 6, 0.5)
    status = ["boundary" if i % 3 == 0 else "interior" for i in range(len(cov))]
    buf = io.StringIO()
    write_cells_file(cov, buf, status)
    buf.seek(0)
    cov2, status2 = read_cells_file(buf)
    assert np.array_equal(cov2.lo, cov.lo) and np.array_equal(cov2.hi, cov.hi)
    assert np.array_equal(cov2.depths, cov.depths) and status2 == status
    buf = io.StringIO()
    write_cells_file(Covering.initial(unit), buf)
    assert "\n- 0 " in "\n" + "\n".join(buf.getvalue().splitlines()[2:])
    with pytest.raises(ValueError):
        read_cells_file(io.StringIO("0 1 0.0 0.5 retained\n"))


def test_engine_loop_behaviours():
    """The rest of the reference's tests/test_engine.py:27-118: identity keeps
    all volume, shift empties after one iteration, the linear map recovers
    [-0.5, 0.5] within 4 cell widths, full mode through the adaptive path
    equals the standard sequence, and check_stop on an empty covering."""
    from paper_2202_06111_b200 import AdaptiveConfig, Covering, ImageConfig, RunConfig, run
    from paper_2202_06111_b200.engine import check_stop
    from paper_2202_06111_b200.system import (cstr_model, identity_model, linear_test_model,
                                              shift_model)

    res = run(RunConfig(model=identity_model(), iterations=5, image=ImageConfig(2, 0.0)))
    assert res.termination == "iterations" and res.covering.volume() == pytest.approx(1.0, rel=0)
    res = run(RunConfig(model=shift_model(), iterations=5))
    assert res.termination == "empty" and len(res.metrics) == 1
    assert res.metrics[0].cells_after == 0 and res.empty
    res = run(RunConfig(model=linear_test_model(2.0), iterations=10, image=ImageConfig(3, 0.05)))
    lo, hi = float(res.covering.lo.min()), float(res.covering.hi.max())
    width = 2.0 / 2 ** 10
    assert lo <= -0.5 and hi >= 0.5
    assert lo >= -0.5 - 4 * width and hi <= 0.5 + 4 * width
    a = run(RunConfig(model=cstr_model(), iterations=5, adaptive=AdaptiveConfig(mode="full")))
    b = run(RunConfig(model=cstr_model(), iterations=5))
    assert np.array_equal(a.covering.bits, b.covering.bits)
    assert np.array_equal(a.covering.depths, b.covering.depths)
    cfg = RunConfig(model=identity_model(), iterations=50)
    empty = Covering.initial(identity_model().X).retain(np.array([], dtype=np.int64))
    assert check_stop(1, empty, cfg) == "empty"
