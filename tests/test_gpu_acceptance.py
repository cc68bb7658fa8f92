"""The reference's acceptance criteria for this path, on the GPU
(/root/reference/pkg/tests/test_acceptance.py, criteria 1-9; the CLI exit
code of criterion 3, the shapely hull comparison of criterion 8 and the
CPU-parallel speed-up of criterion 10 are outside this path).  The
independent oracles the reference uses (cg/bench.py brute_force_cis_1d /
brute_force_graph) are restated here in numpy."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LINEAR_ITERATIONS = 12  # test_acceptance.py:41-46


def _linear_config(**kw):
    from paper_2202_06111_b200 import ImageConfig, RunConfig
    from paper_2202_06111_b200.system import linear_test_model

    return RunConfig(model=linear_test_model(2.0), image=ImageConfig(samples_per_dim=3, bloat=0.05),
                     input_counts=3, **kw)


@pytest.fixture(scope="module")
def linear_run():
    from paper_2202_06111_b200 import run

    return run(_linear_config(iterations=LINEAR_ITERATIONS))


@pytest.fixture(scope="module")
def cstr_runs():
    from paper_2202_06111_b200 import AdaptiveConfig, RunConfig, run
    from paper_2202_06111_b200.system import cstr_model

    full = run(RunConfig(model=cstr_model(), iterations=20, snapshot_iterations=(5, 10, 15)))
    n3 = run(RunConfig(model=cstr_model(), iterations=20,
                       adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3)))
    n5 = run(RunConfig(model=cstr_model(), iterations=20,
                       adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=5)))
    return full, n3, n5


def union_intervals(covering):
    """Merged (lo, hi) intervals of a 1-D covering (test_acceptance.py:83-95)."""
    if len(covering) == 0:
        return []
    lo, hi = covering.lo[:, 0], covering.hi[:, 0]
    order = np.argsort(lo)
    merged = [[lo[order[0]], hi[order[0]]]]
    for i in order[1:]:
        if lo[i] <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], hi[i])
        else:
            merged.append([lo[i], hi[i]])
    return [(float(a), float(b)) for a, b in merged]


def union_contains(covering, lo, hi):
    return any(a <= lo and hi <= b for a, b in union_intervals(covering))


def brute_force_cis_1d(a, xlo, xhi, ulo, uhi, resolution, input_points=201):
    """Grid fixed point of x+ = a x + u (cg/bench.py:62-108 restated): grid
    points die when no input maps them onto a surviving grid point."""
    npts = int(round((xhi - xlo) / resolution)) + 1
    xs = np.linspace(xlo, xhi, npts)
    h = xs[1] - xs[0]
    us = np.linspace(ulo, uhi, input_points)
    images = a * xs[:, None] + us[None, :]
    idx = np.round((images - xlo) / h).astype(np.int64)
    in_range = (idx >= 0) & (idx < npts)
    idx = np.where(in_range, idx, 0)
    alive = np.ones(npts, dtype=bool)
    while True:
        new = alive & (in_range & alive[idx]).any(axis=1)
        if np.array_equal(new, alive):
            break
        alive = new
    pts = xs[alive]
    return float(pts.min()), float(pts.max())


def test_criterion_01_analytic_cis_recovery(linear_run):
    """test_acceptance.py:102-147: x+ = 2x + u, |u| <= 0.5 has the largest
    CIS [-0.5, 0.5]; the retained union is one interval around it."""
    olo, ohi = brute_force_cis_1d(2.0, -1.0, 1.0, -0.5, 0.5, 1e-4)
    assert olo == pytest.approx(-0.5, abs=2e-4) and ohi == pytest.approx(0.5, abs=2e-4)
    d = 2.0 / 2 ** LINEAR_ITERATIONS
    cov = linear_run.covering
    assert union_contains(cov, olo, ohi)
    intervals = union_intervals(cov)
    assert len(intervals) == 1
    a, b = intervals[0]
    margin = 4 * d + 2e-4
    assert -0.5 - margin <= a and b <= 0.5 + margin


def test_criterion_02_outer_approximation_every_iteration():
    """test_acceptance.py:150-165: [-0.5, 0.5] stays inside the retained
    union at every iteration."""
    from paper_2202_06111_b200 import run

    for k in range(1, LINEAR_ITERATIONS + 1):
        assert union_contains(run(_linear_config(iterations=k)).covering, -0.5, 0.5), k


def test_criterion_03_identity_and_escape_extremes():
    """test_acceptance.py:168-185 (without the CLI exit code)."""
    from paper_2202_06111_b200 import ImageConfig, RunConfig, run
    from paper_2202_06111_b200.system import identity_model, shift_model

    ident = run(RunConfig(model=identity_model(), iterations=6, image=ImageConfig(2, 0.0)))
    assert ident.covering.volume() == 1.0
    assert all(m.cells_before == m.cells_after for m in ident.metrics)
    assert float(ident.covering.lo.min()) == 0.0 and float(ident.covering.hi.max()) == 1.0
    shift = run(RunConfig(model=shift_model(), iterations=5))
    assert shift.termination == "empty" and len(shift.metrics) == 1


def test_criterion_04_parallel_equals_serial_bytewise(cstr_runs):
    """test_acceptance.py:188-214: every BuildPlan exports the serial
    graph's edge list byte for byte, on the full-mode CSTR snapshots."""
    from paper_2202_06111_b200 import ImageConfig, sample_inputs
    from paper_2202_06111_b200.graph import BuildPlan, build_graph_parallel, build_graph_serial
    from paper_2202_06111_b200.system import cstr_model

    full = cstr_runs[0]
    model = cstr_model()
    inputs = sample_inputs(model.U, 3)
    cfg = ImageConfig()
    for it in (5, 10, 15):
        cov = full.snapshots[it]
        index = cov.build_index()
        exports = {build_graph_serial(cov, index, model, inputs, cfg).edge_list_bytes()}
        for workers in (1, 2, 4):
            for batch_size in (64, 1024):
                plan = BuildPlan(batch_size, workers)
                exports.add(build_graph_parallel(cov, index, model, inputs, cfg,
                                                 plan).edge_list_bytes())
                # and the plan's own work split, as the reference's workers
                # do it (cg/graph.py:306-345): contiguous chunks of batches
                # built separately (the row-range build that multi-GPU ranks
                # use) and merged by merge_subgraphs with disjoint ownership
                exports.add(_chunked_build(cov, index, model, inputs, cfg, plan)
                            .edge_list_bytes())
        assert len(exports) == 1, it


def _chunked_build(cov, index, model, inputs, cfg, plan):
    import math

    import torch

    from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows, merge_subgraphs

    V = len(cov)
    starts = list(range(0, V, plan.batch_size))
    per = max(1, math.ceil(len(starts) / plan.workers))
    parts = []
    for c in range(0, len(starts), per):
        b = starts[c]
        e = min(starts[min(c + per, len(starts)) - 1] + plan.batch_size, V)
        ip, ix = build_graph_rows(cov, index, model, inputs, cfg, b, e)
        full = torch.zeros(V + 1, dtype=torch.int64, device=ip.device)
        full[b + 1:e + 1] = ip[1:]
        full[e + 1:] = ip[-1]
        parts.append(SymbolicImage(cov.depths, cov.bits, full.cpu().numpy(),
                                   ix.cpu().numpy().astype(np.int64),
                                   owned=np.arange(b, e, dtype=np.int64)))
    return merge_subgraphs(parts)


def _random_covering(rng, root, rounds, keep_fraction):
    """tests/conftest.py:36-51 of the reference."""
    from paper_2202_06111_b200 import Covering

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


def _brute_force_edges(cov, model, inputs, cfg):
    """cg/bench.py:111-135 restated: per cell and input the oracle's
    enclosure, tested against every cell box by a linear scan."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.image import sample_fractions

    step = O.make_step(model.step.spec())
    frac = sample_fractions(cfg, model.n)
    lo, hi = cov.lo, cov.hi
    pairs = set()
    for u in np.atleast_2d(inputs.points):
        elo, ehi, valid = O.enclosures(step, lo, hi, u, frac, cfg.bloat)
        for i in np.flatnonzero(valid):
            hit = np.all(elo[i] <= hi, axis=1) & np.all(lo <= ehi[i], axis=1)
            pairs.update((int(i), int(j)) for j in np.flatnonzero(hit))
    return pairs


def test_criterion_05_serial_builder_matches_brute_force():
    """test_acceptance.py:217-249: 50 random instances (linear and rotated
    affine maps on random mixed-resolution coverings)."""
    from paper_2202_06111_b200 import Box, ImageConfig, sample_inputs
    from paper_2202_06111_b200.graph import build_graph_serial
    from paper_2202_06111_b200.system import affine_test_model, linear_test_model

    rng = np.random.default_rng(20260809)
    for trial in range(50):
        if trial % 2 == 0:
            model = linear_test_model(float(rng.uniform(1.2, 3.0)))
            rounds = int(rng.integers(2, 8))
        else:
            angle = rng.uniform(0, 2 * np.pi)
            scale = rng.uniform(0.6, 1.2)
            rot = scale * np.array([[np.cos(angle), -np.sin(angle)],
                                    [np.sin(angle), np.cos(angle)]])
            model = affine_test_model(rot, [[0.3], [0.1]], rng.uniform(-0.1, 0.1, 2),
                                      X=Box([-1.0, -1.0], [1.0, 1.0]), U=Box([-0.5], [0.5]))
            rounds = int(rng.integers(2, 9))
        cov = _random_covering(rng, model.X, rounds, float(rng.uniform(0.6, 1.0)))
        if len(cov) > 500:
            cov = cov.retain(np.arange(500))
        inputs = sample_inputs(model.U, int(rng.integers(2, 4)))
        cfg = ImageConfig(int(rng.integers(2, 4)), float(rng.uniform(0, 0.15)))
        g = build_graph_serial(cov, cov.build_index(), model, inputs, cfg)
        src, dst = g.edge_pairs()
        assert set(zip(src.tolist(), dst.tolist())) == \
            _brute_force_edges(cov, model, inputs, cfg), trial


def test_criterion_08_adaptive_efficiency(cstr_runs):
    """test_acceptance.py:295-314, cell-count part: the N=3 adaptive run
    keeps at most half the cells of the full-mode run (the reference's
    wall-time and shapely hull parts are not reproduced here)."""
    full, n3, _ = cstr_runs
    assert 2 * len(n3.covering) <= len(full.covering)


def test_criterion_09_monotone_shrinkage(linear_run, cstr_runs):
    """test_acceptance.py:317-328: the containment check holds on every run."""
    full, n3, n5 = cstr_runs
    assert linear_run.containment_ok and full.containment_ok
    assert n3.containment_ok and n5.containment_ok
