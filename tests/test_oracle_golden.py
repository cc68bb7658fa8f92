"""Pin the CPU oracle (oracle/gis_oracle.py) to the reference's own outputs
(tests/golden/*.npz, produced by tests/golden/make_golden.py importing
cisgraph 0.1.0).  Integers and masks bit for bit; floats exactly (same numpy
operations in the same order)."""

import numpy as np
import pytest

from conftest import oracle_cover

from oracle import gis_oracle as O


def test_steps_exact(golden):
    g = golden("steps")
    keys = g.keys("out")
    assert len(keys) == 10
    for k in keys:
        c = g.case(k)
        step = O.make_step(c["spec"])
        got = np.stack([step(c["x"], u) for u in c["u"]])
        assert np.array_equal(got, c["out"], equal_nan=True), k


def test_cstr_golden_step(golden):
    # tests/test_system.py:22-24,42-51 of the reference
    g = golden("steps")
    want = (0.50000441966181541, 349.99915616861051)
    step = O.make_step(g.case("cstr")["spec"])
    got = step(np.array([0.5, 350.0]), np.array([300.0]))
    assert got == pytest.approx(want, rel=0, abs=1e-12)
    assert np.array_equal(got, g.z["cstr_golden_step"])


def test_enclosures_exact(golden):
    g = golden("enclosures")
    keys = g.keys("enc_lo")
    assert len(keys) >= 40
    for k in keys:
        c = g.case(k)
        step = O.make_step(c["spec"])
        for i, u in enumerate(c["u"]):
            el, eh, va = O.enclosures(step, c["lo"], c["hi"], u, c["frac"], float(c["bloat"]))
            assert np.array_equal(va, c["valid"][i]), k
            assert np.array_equal(el[va], c["enc_lo"][i][va]), k
            assert np.array_equal(eh[va], c["enc_hi"][i][va]), k


def test_graphs_and_keep_exact(golden):
    g = golden("graphs")
    for k in g.keys("indptr"):
        c = g.case(k)
        cov = oracle_cover(c)
        step = O.make_step(c["spec"])
        ip, ix = O.build_graph(cov.lo, cov.hi, step, c["inputs"], c["frac"], float(c["bloat"]))
        assert np.array_equal(ip, c["indptr"]), k
        assert np.array_equal(ix, c["indices"]), k
        V = len(cov)
        assert np.array_equal(O.non_leaving_mask(ip, ix, V), c["keep"]), k
        assert np.array_equal(O.peel_fixed_point(ip, ix, V), c["keep"]), k


def test_prune_random_digraphs(golden):
    g = golden("prune")
    for k in g.keys("keep"):
        c = g.case(k)
        V = len(c["indptr"]) - 1
        assert np.array_equal(O.non_leaving_mask(c["indptr"], c["indices"], V), c["keep"]), k
        assert np.array_equal(O.peel_fixed_point(c["indptr"], c["indices"], V), c["keep"]), k


def test_selection_grids(golden):
    g = golden("select")
    for k in ("g5_drop25", "g6", "g5_drop4", "g5_drop4_fp"):
        c = g.case(k)
        tree = O.BoxTree(c["lo"], c["hi"])
        b = O.select_boundary_mask(c["lo"], c["hi"], tree, 0.01, bool(c["fp"]))
        assert np.array_equal(b, c["boundary"]), k
        for N in (1, 2, 3):
            got = O.select_neighborhood_mask(c["lo"], c["hi"], b, N)
            assert np.array_equal(got, c[f"nbr{N}"]), (k, N)


def test_selection_mixed_and_cover_ops(golden):
    g = golden("select")
    for t in range(4):
        c = g.case(f"mixed{t}")
        cov = oracle_cover(c)
        tree = O.BoxTree(cov.lo, cov.hi)
        b = O.select_boundary_mask(cov.lo, cov.hi, tree, 0.01)
        assert np.array_equal(b, c["boundary"])
        assert np.array_equal(O.select_boundary_mask(cov.lo, cov.hi, tree, 0.01, True),
                              c["boundary_fp"])
        for N in (1, 3, 5):
            assert np.array_equal(O.select_neighborhood_mask(cov.lo, cov.hi, b, N), c[f"nbr{N}"])
        res = O.knn(cov.centers(), c["knn_q"], 7)
        got = np.stack([np.pad(r[0], (0, 7 - len(r[0])), constant_values=-1) for r in res])
        assert np.array_equal(got, c["knn7"])
        c3 = cov.subdivide(c["sub_mask"]).retain(c["ret_mask"])
        assert np.array_equal(c3.depths, c["c3_depths"])
        assert np.array_equal(c3.bits, c["c3_bits"])
        assert np.array_equal(c3.lo, c["c3_lo"]) and np.array_equal(c3.hi, c["c3_hi"])
        assert c3.diameter() == float(c["c3_diameter"])
        q = c["knn_q"]
        qi, ci = O.BoxTree(c3.lo, c3.hi).query(q - 0.05, q + 0.05)
        assert np.array_equal(qi, c["qb_qi"]) and np.array_equal(ci, c["qb_ci"])


@pytest.mark.parametrize("key,kw", [
    ("config1", dict(cfg=1, iterations=4, counts=11, initial_depth=12)),
    ("config3", dict(cfg=3, iterations=9, counts=21, initial_depth=10, mode="adaptive")),
    ("pendulum_grid48", dict(cfg=1, iterations=3, counts=11, initial_grid=(48, 48))),
    ("cartpole_grid6", dict(cfg=5, iterations=3, counts=11, initial_grid=(6, 6, 6, 6),
                            mode="adaptive")),
])
def test_engine_runs_baseline(golden, key, kw):
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.image import sample_fractions

    c = golden("runs").case(key)
    rc = config(kw["cfg"])
    m = rc.model
    r = O.run(m.step.spec(), m.X.lo, m.X.hi, m.U.lo, m.U.hi, kw["counts"], kw["iterations"],
              sample_fractions(rc.image, m.n), 0.1, mode=kw.get("mode", "full"),
              initial_depth=kw.get("initial_depth"), initial_grid=kw.get("initial_grid"),
              prune="peel")
    got = np.array([[x["iteration"], x["cells_before"], x["cells_after"], x["edges"],
                     x["boundary_cells"], x["diameter"]] for x in r["metrics"]])
    assert np.array_equal(got, c["metrics"])
    assert np.array_equal(r["cover"].bits, c["bits"])
    assert np.array_equal(r["cover"].depths, c["depths"])
    assert r["containment_ok"] == bool(c["containment_ok"])


def test_engine_runs_reference_models(golden):
    from paper_2202_06111_b200.image import lattice_fractions
    from paper_2202_06111_b200.system import cstr_model, linear_test_model

    g = golden("runs")
    cases = [("cstr_full6", cstr_model(), 6, "full", 0.1, 3),
             ("cstr_n3_9", cstr_model(), 9, "adaptive", 0.1, 3),
             ("linear12", linear_test_model(2.0), 12, "full", 0.05, 3),
             ("linear_n3_48", linear_test_model(2.0), 48, "adaptive", 0.05, 3)]
    for key, m, it, mode, bloat, spd in cases:
        c = g.case(key)
        r = O.run(m.step.spec(), m.X.lo, m.X.hi, m.U.lo, m.U.hi, 3, it,
                  lattice_fractions(m.n, spd), bloat, mode=mode, prune="tarjan")
        got = np.array([[x["iteration"], x["cells_before"], x["cells_after"], x["edges"],
                         x["boundary_cells"], x["diameter"]] for x in r["metrics"]])
        assert np.array_equal(got, c["metrics"]), key
        assert np.array_equal(r["cover"].bits, c["bits"]), key
    # the reference's own engine.run agrees with the composed driver
    assert np.array_equal(g.z["cstr_full6_engine__bits"], g.case("cstr_full6")["bits"])
    assert np.array_equal(g.z["cstr_full6_engine__edges"], g.case("cstr_full6")["metrics"][:, 3])


def test_oracle_large_k_knn_matches_reference(golden):
    from conftest import oracle_cover

    g = golden("knn")
    for key in ("cov0", "cov1", "cov2"):
        c = g.case(key)
        cov = oracle_cover(c)
        for k in c["ks"]:
            k = int(k)
            res = O.knn(cov.centers(), c["q"], k)
            width = c[f"knn{k}"].shape[1]
            got = np.stack([np.pad(r[0], (0, width - len(r[0])), constant_values=-1) for r in res])
            assert np.array_equal(got, c[f"knn{k}"]), (key, k)
            assert np.array_equal([r[1] for r in res], c[f"clamped{k}"]), (key, k)
