"""GPU parity: libgis (through the package API) against the reference's
golden outputs and the CPU oracle on the same seeded inputs."""

import numpy as np
import pytest

from conftest import oracle_cover, peeling_fixed_point
from helpers import assert_states_close, explain_edge_diffs, model_for, model_from_spec

pytestmark = pytest.mark.gpu


def _cov(case):
    from paper_2202_06111_b200 import Box, Covering

    return Covering.from_paths(Box(case["root_lo"], case["root_hi"]),
                               ["-" if d == 0 else format(int(b), f"0{int(d)}b")
                                for d, b in zip(case["depths"], case["bits"])])


# ------------------------------------------------------------------ K1 ----

def test_steps_match_reference(golden):
    """States from X agree to 1e-12 relative (north star); the 56 probe
    points far outside X (up to one box width beyond it) are held to 1e-10,
    since an ulp-level difference in sin/exp is amplified there."""
    g = golden("steps")
    for name in g.keys("out"):
        c = g.case(name)
        m = model_for(name, c["spec"])
        scale = np.max(np.abs(c["x"]))
        for i, u in enumerate(c["u"]):
            got = m.map_points(c["x"], u)
            try:
                assert_states_close(got[:200], c["out"][i][:200], scale=scale)
                assert_states_close(got[200:], c["out"][i][200:], scale=scale, rel=1e-10)
            except AssertionError as e:
                raise AssertionError(f"{name} u={u}: {e}") from None


def test_cstr_golden_step():
    from paper_2202_06111_b200.system import cstr_model

    got = cstr_model().step(np.array([0.5, 350.0]), np.array([300.0]))
    assert got == pytest.approx((0.50000441966181541, 349.99915616861051), rel=0, abs=1e-12)


def test_enclosures_match_reference(golden):
    from paper_2202_06111_b200.image import ImageConfig, batch_enclosures

    g = golden("enclosures")
    keys = g.keys("enc_lo")
    assert len(keys) >= 40
    for k in keys:
        c = g.case(k)
        m = model_for(k.split("__")[0], c["spec"])
        cfg = ImageConfig(2, float(c["bloat"]), fractions=c["frac"])
        for i, u in enumerate(c["u"]):
            el, eh, va = batch_enclosures(m, c["lo"], c["hi"], u, cfg)
            assert np.array_equal(va, c["valid"][i]), k
            scale = max(np.max(np.abs(c["lo"])), 1.0)
            assert_states_close(el[va], c["enc_lo"][i][va], scale=scale)
            assert_states_close(eh[va], c["enc_hi"][i][va], scale=scale)


# ------------------------------------------------------------- K2 + K3 ----

def test_graphs_and_keep_match_reference(golden):
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.graph import build_graph_serial
    from paper_2202_06111_b200.image import ImageConfig

    g = golden("graphs")
    total_explained = 0
    for k in g.keys("indptr"):
        c = g.case(k)
        cov = _cov(c)
        ins = c["inputs"]
        m = model_from_spec(c["spec"], (c["root_lo"], c["root_hi"]), (ins.min(0), ins.max(0)))
        cfg = ImageConfig(2, float(c["bloat"]), fractions=c["frac"])
        gg = build_graph_serial(cov, cov.build_index(), m, ins, cfg)
        if not (np.array_equal(gg.indptr, c["indptr"])
                and np.array_equal(gg.indices, c["indices"])):
            oc = oracle_cover(c)
            ex, unex = explain_edge_diffs(oc.lo, oc.hi, O.make_step(c["spec"]), ins, c["frac"],
                                          float(c["bloat"]), (gg.indptr, gg.indices),
                                          (c["indptr"], c["indices"]))
            assert not unex, f"{k}: unexplained edge differences {unex[:10]}"
            total_explained += len(ex)
            continue
        assert np.array_equal(non_leaving_mask(gg), c["keep"]), k
    assert total_explained == 0, f"{total_explained} near-face edge differences"


def test_prune_matches_reference_digraphs(golden):
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.graph import SymbolicImage

    g = golden("prune")
    for k in g.keys("keep"):
        c = g.case(k)
        V = len(c["indptr"]) - 1
        gr = SymbolicImage(np.zeros(V), np.arange(V), c["indptr"], c["indices"])
        assert np.array_equal(non_leaving_mask(gr), c["keep"]), k


def test_prune_equals_peeling_200_digraphs():
    """tests/test_acceptance.py:252-272 (criterion 6) on the GPU kernel."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.graph import SymbolicImage

    rng = np.random.default_rng(97)
    for trial in range(200):
        n = int(rng.integers(2, 2001))
        m = int(rng.uniform(0.5, 3.0) * n)
        src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
        ip, ix = O.csr_from_pairs(src, dst, n)
        got = non_leaving_mask(SymbolicImage(np.zeros(n), np.arange(n), ip, ix))
        want = peeling_fixed_point(n, list(zip(src.tolist(), dst.tolist())))
        assert np.array_equal(got, want), trial


@pytest.mark.parametrize("n", [10_000_037, 10_485_760])
def test_prune_large_graph_sparse_tail(n):
    """Graphs large enough for K3's four-word sweeps (>= 16 four-word groups
    per resident warp: V >= 9.7M at 592 blocks) whose deaths thin out over
    many sweeps, so the late sweeps take sweep_loop4; one size ends inside a
    bitmap word.  Against the oracle's peeling fixed point."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.analysis import non_leaving_dev
    from paper_2202_06111_b200.graph import SymbolicImage

    rng = np.random.default_rng(n)
    deg = rng.choice(np.array([0, 1, 2, 3]), size=n, p=[0.01, 0.45, 0.34, 0.20])
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    # targets near the source (the dynamics' locality), some far
    off = rng.integers(-300, 301, len(src))
    far = rng.random(len(src)) < 0.1
    dst = np.where(far, rng.integers(0, n, len(src)), np.clip(src + off, 0, n - 1))
    ip, ix = O.csr_from_pairs(src, dst, n)
    g = SymbolicImage(np.zeros(n), np.arange(n), ip, ix)
    keep, sweeps = non_leaving_dev(g)
    want = O.peel_fixed_point(ip, ix, n)
    got = keep.cpu().numpy().astype(bool)
    assert 0 < want.sum() < n and sweeps >= 3
    assert np.array_equal(got, want)


def test_prune_edge_cases():
    from paper_2202_06111_b200.analysis import non_leaving, non_leaving_mask
    from paper_2202_06111_b200.graph import SymbolicImage

    def G(n, edges):
        from oracle import gis_oracle as O
        s = np.array([e[0] for e in edges], dtype=np.int64)
        d = np.array([e[1] for e in edges], dtype=np.int64)
        ip, ix = O.csr_from_pairs(s, d, n)
        return SymbolicImage(np.full(n, 12), np.arange(n), ip, ix)

    assert non_leaving_mask(G(0, [])).shape == (0,)
    assert {v.bits for v in non_leaving(G(4, [(1, 2), (2, 1), (2, 3)]))} == {1, 2}
    assert {v.bits for v in non_leaving(G(4, [(1, 2), (2, 1), (2, 3), (3, 1)]))} == {1, 2, 3}
    assert len(non_leaving(G(5, [(i, i) for i in range(5)]))) == 5
    assert not non_leaving_mask(G(7, [])).any()
    # a 50k-vertex chain: every vertex eventually loses its only successor
    n = 50_000
    assert not non_leaving_mask(G(n, [(i, i + 1) for i in range(n - 1)])).any()
    # the same chain feeding a cycle survives entirely
    assert non_leaving_mask(G(n, [(i, i + 1) for i in range(n - 1)] + [(n - 1, n - 2)])).all()


# ---------------------------------------------------------------- K4 ----

def test_selection_on_grids_matches_reference(golden):
    from paper_2202_06111_b200 import SpatialIndex
    from paper_2202_06111_b200.adaptive import select_boundary_mask, select_neighborhood_mask
    from types import SimpleNamespace

    g = golden("select")
    for k in ("g5_drop25", "g6", "g5_drop4", "g5_drop4_fp"):
        c = g.case(k)
        idx = SpatialIndex(c["lo"], c["hi"])
        bs = SimpleNamespace(lo=c["lo"], hi=c["hi"])
        b = select_boundary_mask(bs, idx, 0.01, bool(c["fp"]))
        assert np.array_equal(b, c["boundary"]), k
        for N in (1, 2, 3):
            assert np.array_equal(select_neighborhood_mask(bs, idx, b, N), c[f"nbr{N}"]), (k, N)


def test_selection_mixed_coverings_match_reference(golden):
    from paper_2202_06111_b200.adaptive import select_boundary_mask, select_neighborhood_mask

    g = golden("select")
    for t in range(4):
        c = g.case(f"mixed{t}")
        cov = _cov(c)
        idx = cov.build_index()
        b = select_boundary_mask(cov, idx, 0.01)
        assert np.array_equal(b, c["boundary"]), t
        assert np.array_equal(select_boundary_mask(cov, idx, 0.01, True), c["boundary_fp"]), t
        for N in (1, 3, 5):
            assert np.array_equal(select_neighborhood_mask(cov, idx, b, N), c[f"nbr{N}"]), (t, N)
        res = idx.knn_indices_many(c["knn_q"], 7)
        got = np.stack([np.pad(r[0], (0, 7 - len(r[0])), constant_values=-1) for r in res])
        assert np.array_equal(got, c["knn7"]), t


def test_subdivide_retain_query_match_reference(golden):
    g = golden("select")
    for t in range(4):
        c = g.case(f"mixed{t}")
        cov = _cov(c)
        c3 = cov.subdivide(c["sub_mask"]).retain(c["ret_mask"])
        assert np.array_equal(c3.depths, c["c3_depths"])
        assert np.array_equal(c3.bits, c["c3_bits"])
        assert np.array_equal(c3.lo, c["c3_lo"]) and np.array_equal(c3.hi, c["c3_hi"])
        assert c3.diameter() == float(c["c3_diameter"])
        q = c["knn_q"]
        qi, ci = c3.build_index().query_boxes(q - 0.05, q + 0.05)
        assert np.array_equal(qi, c["qb_qi"]) and np.array_equal(ci, c["qb_ci"])


# --------------------------------------------------------------- engine ----

@pytest.mark.parametrize("key,cfg_id,over", [
    ("config1", 1, {}), ("config3", 3, {}),
    ("pendulum_grid48", 1, dict(initial_depth=None, initial_grid=(48, 48), iterations=3)),
    ("cartpole_grid6", 5, dict(initial_grid=(6, 6, 6, 6), iterations=3)),
])
def test_runs_match_reference_baseline_configs(golden, key, cfg_id, over):
    from paper_2202_06111_b200 import run
    from paper_2202_06111_b200.configs import config

    c = golden("runs").case(key)
    res = run(config(cfg_id, **over))
    got = np.array([[m.iteration, m.cells_before, m.cells_after, m.edges, m.boundary_cells,
                     m.diameter] for m in res.metrics])
    assert np.array_equal(got, c["metrics"])
    assert np.array_equal(res.covering.bits, c["bits"])
    assert np.array_equal(res.covering.depths, c["depths"])
    assert res.containment_ok == bool(c["containment_ok"])


def test_runs_match_reference_models(golden):
    from paper_2202_06111_b200 import AdaptiveConfig, ImageConfig, RunConfig, run
    from paper_2202_06111_b200.system import cstr_model, linear_test_model

    g = golden("runs")
    cases = [("cstr_full6", RunConfig(model=cstr_model(), iterations=6)),
             ("cstr_n3_9", RunConfig(model=cstr_model(), iterations=9,
                                     adaptive=AdaptiveConfig(mode="adaptive", n_neighbors=3))),
             ("linear12", RunConfig(model=linear_test_model(2.0), iterations=12,
                                    image=ImageConfig(3, 0.05)))]
    for key, rc in cases:
        c = g.case(key)
        res = run(rc)
        got = np.array([[m.iteration, m.cells_before, m.cells_after, m.edges, m.boundary_cells,
                         m.diameter] for m in res.metrics])
        assert np.array_equal(got, c["metrics"]), key
        assert np.array_equal(res.covering.bits, c["bits"]), key


def test_large_k_knn_and_neighborhoods_match_reference(golden):
    """k beyond one lane per entry (warp top-k up to 256, radix-sort path
    beyond) and N-NN neighbourhoods of 40 / 300 (cg/geometry.py:529-555,
    cg/adaptive.py:136-150)."""
    from paper_2202_06111_b200.adaptive import select_neighborhood_mask

    g = golden("knn")
    for key in ("cov0", "cov1", "cov2"):
        c = g.case(key)
        cov = _cov(c)
        idx = cov.build_index()
        for k in c["ks"]:
            k = int(k)
            res = idx.knn_indices_many(c["q"], k)
            width = c[f"knn{k}"].shape[1]
            got = np.stack([np.pad(r[0], (0, width - len(r[0])), constant_values=-1) for r in res])
            assert np.array_equal(got, c[f"knn{k}"]), (key, k)
            assert np.array_equal([r[1] for r in res], c[f"clamped{k}"]), (key, k)
        for N in (40, 300):
            got = select_neighborhood_mask(cov, idx, c["boundary"], N)
            assert np.array_equal(got, c[f"nbr{N}"]), (key, N)
