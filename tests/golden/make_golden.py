"""Generate the golden fixtures by running the REFERENCE implementation.

Imports ``cisgraph`` 0.1.0 from /root/reference/pkg/src (read-only) with a
test-only ``shapely`` stub (shapely is not installed; only hull post-
processing needs it) and records the reference's own outputs for the hot
path on seeded inputs.  The BASELINE models the reference registry lacks
enter through its public plugin API, SystemModel(step=callable), with the
numpy steps of oracle/gis_oracle.py; BASELINE sampling tables are injected
by replacing cisgraph.image._unit_grid.

Run in the build container (not on the GPU box):
    python tests/golden/make_golden.py
Outputs tests/golden/*.npz (committed).
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))


def _import_reference():
    stub = Path(tempfile.mkdtemp(prefix="shapely_stub_"))
    (stub / "shapely").mkdir()
    (stub / "shapely" / "__init__.py").write_text("")
    (stub / "shapely" / "geometry.py").write_text(
        "class Polygon:\n    def __init__(self, *a, **k):\n"
        "        raise RuntimeError('shapely stub')\n")
    sys.path[:0] = [str(stub), str(REF), str(REF.parent / "tests")]
    import cisgraph  # noqa: F401
    return cisgraph


cg = _import_reference()
import cisgraph.image as cg_image  # noqa: E402
from cisgraph import adaptive as cg_ad  # noqa: E402
from cisgraph import analysis as cg_an  # noqa: E402
from cisgraph import engine as cg_en  # noqa: E402
from cisgraph import geometry as cg_geo  # noqa: E402
from cisgraph import graph as cg_gr  # noqa: E402
from cisgraph import system as cg_sys  # noqa: E402

from oracle import gis_oracle as O  # noqa: E402
from paper_2202_06111_b200 import system as S  # noqa: E402
from paper_2202_06111_b200.configs import config  # noqa: E402
from paper_2202_06111_b200.image import (corners_plus_center, corners_plus_seeded,  # noqa: E402
                                         lattice_fractions)

_ORIG_UNIT_GRID = cg_image._unit_grid


def set_fractions(frac):
    """Inject an explicit sample table into the reference (or restore)."""
    if frac is None:
        cg_image._unit_grid = _ORIG_UNIT_GRID
    else:
        f = np.asarray(frac, dtype=np.float64)
        cg_image._unit_grid = lambda n, spd, f=f: f


# -- model specs -----------------------------------------------------------

def model_cases():
    """(name, reference SystemModel, spec) for every device model kind."""
    rng = np.random.default_rng(99)
    A = rng.normal(size=(2, 2))
    B = rng.normal(size=(2, 1))
    c = rng.normal(size=2)
    out = [
        ("cstr", cg_sys.cstr_model(), S.cstr_model().step.spec()),
        ("linear", cg_sys.linear_test_model(2.0), S.linear_test_model(2.0).step.spec()),
        ("affine", cg_sys.affine_test_model(A, B, c, X=cg_geo.Box([-5, -5], [5, 5]),
                                            U=cg_geo.Box([-1.0], [1.0])),
         S.affine_test_model(A, B, c, X=S.Box([-5, -5], [5, 5]), U=S.Box([-1.0], [1.0]))
         .step.spec()),
        ("identity", cg_sys.identity_model(), S.identity_model().step.spec()),
        ("shift", cg_sys.shift_model(), S.shift_model().step.spec()),
    ]
    for key in (1, 2, 3, 4, 5):
        m = config(key).model
        ref = cg_sys.SystemModel(m.name, m.n, m.m, cg_geo.Box(m.X.lo, m.X.hi),
                                 cg_geo.Box(m.U.lo, m.U.hi), O.make_step(m.step.spec()))
        out.append((f"config{key}_{m.name}", ref, m.step.spec()))
    return out


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({(HERE / f'{name}.npz').stat().st_size} bytes)")


def spec_arrays(prefix, spec):
    import json
    return {f"{prefix}spec": np.frombuffer(json.dumps(spec).encode(), dtype=np.uint8)}


# -- 1. steps ----------------------------------------------------------------

def gen_steps():
    rng = np.random.default_rng(1)
    arrays = {}
    for name, ref, spec in model_cases():
        X, U = ref.X, ref.U
        inside = rng.uniform(X.lo, X.hi, (200, ref.n))
        outside = X.lo + (X.hi - X.lo) * rng.uniform(-1.0, 2.0, (56, ref.n))
        x = np.vstack([inside, outside])
        u = rng.uniform(U.lo, U.hi, (4, ref.m))
        out = np.stack([ref.map_points(x, uu) for uu in u])
        arrays.update({f"{name}__x": x, f"{name}__u": u, f"{name}__out": out,
                       **spec_arrays(f"{name}__", spec)})
    step = cg_sys.CstrStep(cg_sys.CstrParameters())
    arrays["cstr_golden_step"] = step(np.array([0.5, 350.0]), np.array([300.0]))
    save("steps", **arrays)


# -- 2. enclosures -------------------------------------------------------------

def gen_enclosures():
    rng = np.random.default_rng(2)
    arrays = {}
    for name, ref, spec in model_cases():
        n = ref.n
        X = ref.X
        w = (X.hi - X.lo) / 16.0
        lo = rng.uniform(X.lo, X.hi - w, (48, n))
        hi = lo + w * rng.uniform(0.05, 1.0, (48, n))
        tables = [lattice_fractions(n, 2), lattice_fractions(n, 3)]
        if name.startswith("config"):
            tables = [corners_plus_center(n), corners_plus_seeded(n, 6, 3)]
        for ti, frac in enumerate(tables):
            for bloat in (0.0, 0.1):
                set_fractions(frac)
                cfg = cg_image.ImageConfig(2, bloat)
                us = rng.uniform(ref.U.lo, ref.U.hi, (3, ref.m))
                el, eh, va = zip(*[cg_image.batch_enclosures(ref, lo, hi, uu, cfg) for uu in us])
                set_fractions(None)
                k = f"{name}__t{ti}_b{int(bloat * 10)}"
                arrays.update({f"{k}__lo": lo, f"{k}__hi": hi, f"{k}__u": us, f"{k}__frac": frac,
                               f"{k}__bloat": np.float64(bloat), f"{k}__enc_lo": np.stack(el),
                               f"{k}__enc_hi": np.stack(eh), f"{k}__valid": np.stack(va),
                               **spec_arrays(f"{k}__", spec)})
    save("enclosures", **arrays)


# -- 3. graphs + prune on coverings ----------------------------------------------

def split_all(cov, times):
    for _ in range(times):
        cov = cov.subdivide(None)
    return cov


def graph_case(arrays, key, cov, ref_model, spec, inputs_pts, frac, bloat):
    set_fractions(frac)
    g = cg_gr.build_graph_serial(cov, cov.build_index(), ref_model,
                                 cg_sys.InputGrid(inputs_pts, (len(inputs_pts),)),
                                 cg_image.ImageConfig(2, bloat))
    keep = cg_an.non_leaving_mask(g) if len(cov) else np.zeros(0, bool)
    set_fractions(None)
    arrays.update({f"{key}__root_lo": cov.root.lo, f"{key}__root_hi": cov.root.hi,
                   f"{key}__depths": cov.depths.astype(np.int16), f"{key}__bits": cov.bits,
                   f"{key}__inputs": inputs_pts, f"{key}__frac": frac,
                   f"{key}__bloat": np.float64(bloat), f"{key}__indptr": g.indptr,
                   f"{key}__indices": g.indices.astype(np.int32), f"{key}__keep": keep,
                   **spec_arrays(f"{key}__", spec)})
    print(f"  graph {key}: V={len(cov)} E={g.edge_count} kept={int(keep.sum())}")


def gen_graphs():
    from conftest import random_covering

    arrays = {}
    models = {name: (ref, spec) for name, ref, spec in model_cases()}

    def setting(ref, rounds, keep=1.0, seed=0):
        cov = split_all(cg_geo.Covering.initial(ref.X), ref.n + rounds)
        if keep < 1.0:
            mask = np.random.default_rng(seed).random(len(cov)) < keep
            mask[0] |= not mask.any()
            cov = cov.retain(mask)
        return cov

    ref, spec = models["identity"]
    graph_case(arrays, "identity4", setting(ref, 4), ref, spec, np.array([[0.0]]),
               lattice_fractions(1, 2), 0.0)
    ref, spec = models["shift"]
    graph_case(arrays, "shift3", setting(ref, 3), ref, spec, np.array([[0.0]]),
               lattice_fractions(1, 2), 0.0)
    ref, spec = models["linear"]
    pts = cg_sys.sample_inputs(ref.U, 3).points
    graph_case(arrays, "linear8", split_all(cg_geo.Covering.initial(ref.X), 3), ref, spec, pts,
               lattice_fractions(1, 3), 0.0)
    graph_case(arrays, "linear_keep07", setting(ref, 4, 0.7, 5), ref, spec, pts,
               lattice_fractions(1, 3), 0.1)
    ref, spec = models["cstr"]
    graph_case(arrays, "cstr_keep08", setting(ref, 5, 0.8, 2), ref, spec,
               cg_sys.sample_inputs(ref.U, 3).points, lattice_fractions(2, 3), 0.1)
    # BASELINE models
    ref, spec = models["config1_pendulum"]
    c = config(1)
    graph_case(arrays, "pendulum_cfg1_it1", split_all(cg_geo.Covering.initial(ref.X), 12), ref,
               spec, cg_sys.sample_inputs(ref.U, 11).points, corners_plus_center(2), 0.1)
    ref, spec = models["config2_pendulum"]
    graph_case(arrays, "pendulum_cfg2_64", split_all(cg_geo.Covering.initial(ref.X), 12), ref,
               spec, cg_sys.sample_inputs(ref.U, 21).points, corners_plus_seeded(2, 16, 0), 0.1)
    ref, spec = models["config3_cstr_dimless"]
    graph_case(arrays, "cstr_dimless_32", split_all(cg_geo.Covering.initial(ref.X), 10), ref,
               spec, cg_sys.sample_inputs(ref.U, 21).points, lattice_fractions(2, 3), 0.1)
    ref, spec = models["config4_lorenz"]
    graph_case(arrays, "lorenz_16", split_all(cg_geo.Covering.initial(ref.X), 12), ref, spec,
               cg_sys.sample_inputs(ref.U, 9).points, corners_plus_seeded(3, 8, 1), 0.1)
    ref, spec = models["config5_cartpole"]
    graph_case(arrays, "cartpole_8", split_all(cg_geo.Covering.initial(ref.X), 12), ref, spec,
               cg_sys.sample_inputs(ref.U, 11).points, corners_plus_seeded(4, 8, 2), 0.1)
    # mixed-resolution coverings (criterion 5 style, tests/test_acceptance.py:216-249)
    rng = np.random.default_rng(20260809)
    for t in range(6):
        if t % 2 == 0:
            ref, spec = models["linear"]
            a = float(rng.uniform(1.2, 3.0))
            ref = cg_sys.linear_test_model(a)
            spec = S.linear_test_model(a).step.spec()
            rounds = int(rng.integers(2, 8))
            nb = 1
        else:
            ang, sc = rng.uniform(0, 2 * np.pi), rng.uniform(0.6, 1.2)
            rot = sc * np.array([[np.cos(ang), -np.sin(ang)], [np.sin(ang), np.cos(ang)]])
            off = rng.uniform(-0.1, 0.1, 2)
            ref = cg_sys.affine_test_model(rot, [[0.3], [0.1]], off,
                                           X=cg_geo.Box([-1.0, -1.0], [1.0, 1.0]),
                                           U=cg_geo.Box([-0.5], [0.5]))
            spec = S.affine_test_model(rot, [[0.3], [0.1]], off, X=S.Box([-1.0, -1.0], [1.0, 1.0]),
                                       U=S.Box([-0.5], [0.5])).step.spec()
            rounds = int(rng.integers(2, 9))
            nb = 2
        cov = random_covering(rng, ref.X, rounds, keep_fraction=float(rng.uniform(0.6, 1.0)))
        if len(cov) > 500:
            cov = cov.retain(np.arange(500))
        pts = cg_sys.sample_inputs(ref.U, int(rng.integers(2, 4))).points
        spd = int(rng.integers(2, 4))
        graph_case(arrays, f"mixed{t}", cov, ref, spec, pts, lattice_fractions(nb, spd),
                   float(rng.uniform(0, 0.15)))
    save("graphs", **arrays)


# -- 4. prune on random digraphs -----------------------------------------------------

def gen_prune():
    from conftest import graph_from_edges

    rng = np.random.default_rng(97)
    arrays = {}
    for t in range(40):
        n = int(rng.integers(2, 2001))
        m = int(rng.uniform(0.5, 3.0) * n)
        src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
        g = graph_from_edges(n, list(zip(src.tolist(), dst.tolist())))
        arrays.update({f"g{t}__indptr": g.indptr, f"g{t}__indices": g.indices.astype(np.int32),
                       f"g{t}__keep": cg_an.non_leaving_mask(g)})
    save("prune", **arrays)


# -- 4b. SCC / strict mode / reverse CSR on digraphs and symbolic images ---------------

def gen_scc():
    """The reference's strongly_connected_components (Tarjan ids),
    non_leaving_mask in both modes, reverse_csr and self_loop_mask."""
    from conftest import graph_from_edges

    rng = np.random.default_rng(131)
    graphs = {}
    for t in range(30):  # random digraphs from sparse (many SCCs) to dense
        n = int(rng.integers(2, 1500))
        m = int(rng.uniform(0.3, 3.0) * n)
        src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
        graphs[f"rand{t}"] = graph_from_edges(n, list(zip(src.tolist(), dst.tolist())))
    # reference test shapes (tests/test_analysis.py:27-91)
    graphs["two_cycle_tail"] = graph_from_edges(4, [(1, 2), (2, 1), (2, 3)])
    graphs["self_loop"] = graph_from_edges(2, [(1, 1)])
    graphs["strict_two_regions"] = graph_from_edges(
        6, [(0, 1), (1, 2), (2, 0), (3, 4), (4, 3), (5, 3)])
    graphs["strict_tie"] = graph_from_edges(7, [(4, 5), (5, 4), (1, 2), (2, 1), (6, 1), (0, 4)])
    graphs["chain50k"] = graph_from_edges(50_000, [(i, i + 1) for i in range(49_999)])
    # a chain of 2-cycles (many colour rounds) with ascending and descending ids
    k = 400
    up = [(2 * i, 2 * i + 1) for i in range(k)] + [(2 * i + 1, 2 * i) for i in range(k)]
    up += [(2 * i + 1, 2 * i + 2) for i in range(k - 1)]
    graphs["cycle_chain_up"] = graph_from_edges(2 * k, up)
    graphs["cycle_chain_down"] = graph_from_edges(2 * k, [(2 * k - 1 - a, 2 * k - 1 - b)
                                                          for a, b in up])
    graphs["empty_edges"] = graph_from_edges(5, [])
    # symbolic images recorded from the reference (graphs.npz)
    gz = np.load(HERE / "graphs.npz")
    for key in ("pendulum_cfg1_it1", "cstr_dimless_32", "lorenz_16", "cartpole_8", "identity4"):
        ip, ix = gz[f"{key}__indptr"], gz[f"{key}__indices"]
        nv = len(ip) - 1
        graphs[f"img_{key}"] = cg_gr.SymbolicImage(np.zeros(nv, np.int64), np.arange(nv),
                                                   ip, ix.astype(np.int64))
    arrays = {}
    for name, g in graphs.items():
        scc = cg_an.strongly_connected_components(g)
        rptr, rind = g.reverse_csr()
        arrays.update({
            f"{name}__indptr": g.indptr, f"{name}__indices": g.indices.astype(np.int32),
            f"{name}__component_of": scc.component_of,
            f"{name}__nontrivial": scc.nontrivial,
            f"{name}__keep": cg_an.non_leaving_mask(g),
            f"{name}__keep_strict": cg_an.non_leaving_mask(g, strict_largest=True),
            f"{name}__rptr": rptr, f"{name}__rind": rind.astype(np.int32),
            f"{name}__loops": g.self_loop_mask()})
    save("scc", **arrays)


# -- 4c. text formats: edge lists and cells files ---------------------------------------

def gen_formats():
    """Bytes of the reference's SymbolicImage.edge_list_bytes and
    write_cells_file on recorded graphs / coverings (with random statuses)."""
    import io

    rng = np.random.default_rng(211)
    gz = np.load(HERE / "graphs.npz")
    arrays = {}
    for key in ("pendulum_cfg1_it1", "cstr_dimless_32", "lorenz_16", "cartpole_8", "identity4",
                "linear_keep07", "mixed3", "mixed0", "shift3"):
        dep, bits = gz[f"{key}__depths"], gz[f"{key}__bits"]
        g = cg_gr.SymbolicImage(dep, bits, gz[f"{key}__indptr"],
                                gz[f"{key}__indices"].astype(np.int64))
        root = cg_geo.Box(gz[f"{key}__root_lo"], gz[f"{key}__root_hi"])
        cov = cg_geo.Covering.from_paths(
            root, ["-" if d == 0 else format(int(b), f"0{int(d)}b") for d, b in zip(dep, bits)])
        status = [cg_geo.CELL_STATUSES[i] for i in rng.integers(0, 3, len(cov))]
        buf = io.StringIO()
        cg_geo.write_cells_file(cov, buf, status)
        buf2 = io.StringIO()
        cg_geo.write_cells_file(cov, buf2)
        arrays.update({
            f"{key}__depths": dep, f"{key}__bits": bits,
            f"{key}__indptr": gz[f"{key}__indptr"], f"{key}__indices": gz[f"{key}__indices"],
            f"{key}__root_lo": root.lo, f"{key}__root_hi": root.hi,
            f"{key}__status": np.array([cg_geo.CELL_STATUSES.index(x) for x in status],
                                       dtype=np.uint8),
            f"{key}__edges_txt": np.frombuffer(g.edge_list_bytes(), dtype=np.uint8),
            f"{key}__cells_txt": np.frombuffer(buf.getvalue().encode(), dtype=np.uint8),
            f"{key}__cells_plain_txt": np.frombuffer(buf2.getvalue().encode(), dtype=np.uint8)})
    save("formats", **arrays)


# -- 5. selection / kNN / covering ops ----------------------------------------------

def gen_select():
    from conftest import grid_boxes, random_covering

    arrays = {}
    for key, (nx, ny, drop, fp) in {"g5_drop25": (5, 5, (25,), False),
                                    "g6": (6, 6, (), False),
                                    "g5_drop4": (5, 5, (4,), False),
                                    "g5_drop4_fp": (5, 5, (4,), True)}.items():
        lo, hi = grid_boxes(nx, ny)
        keep = np.array([i for i in range(nx * ny) if (i + 1) not in set(drop)])
        lo, hi = lo[keep], hi[keep]
        index = cg_geo.SpatialIndex(lo, hi)
        from types import SimpleNamespace
        b = cg_ad.select_boundary_mask(SimpleNamespace(lo=lo, hi=hi), index, 0.01, fp)
        arrays.update({f"{key}__lo": lo, f"{key}__hi": hi, f"{key}__fp": np.int8(fp),
                       f"{key}__boundary": b})
        for N in (1, 2, 3):
            arrays[f"{key}__nbr{N}"] = cg_ad.select_neighborhood_mask(
                SimpleNamespace(lo=lo, hi=hi), index, b, N)
    rng = np.random.default_rng(5)
    for t in range(4):
        root = cg_geo.Box([-2.0, 1.0], [3.0, 4.0]) if t % 2 else cg_geo.Box([0.0, 0.0], [1.0, 1.0])
        cov = random_covering(rng, root, rounds=8 + 2 * t, keep_fraction=0.75)
        idx = cov.build_index()
        b = cg_ad.select_boundary_mask(cov, idx, 0.01)
        k = f"mixed{t}"
        arrays.update({f"{k}__root_lo": root.lo, f"{k}__root_hi": root.hi,
                       f"{k}__depths": cov.depths.astype(np.int16), f"{k}__bits": cov.bits,
                       f"{k}__boundary": b,
                       f"{k}__boundary_fp": cg_ad.select_boundary_mask(cov, idx, 0.01, True)})
        for N in (1, 3, 5):
            arrays[f"{k}__nbr{N}"] = cg_ad.select_neighborhood_mask(cov, idx, b, N)
        q = np.vstack([cov.centers()[:40], rng.uniform(root.lo - 0.3, root.hi + 0.3, (40, 2))])
        res = idx.knn_indices_many(q, 7)
        arrays[f"{k}__knn_q"] = q
        arrays[f"{k}__knn7"] = np.stack([np.pad(r[0], (0, 7 - len(r[0])), constant_values=-1)
                                         for r in res])
        # subdivision / retention chain with recorded masks
        m1 = rng.random(len(cov)) < 0.4
        c2 = cov.subdivide(m1)
        m2 = rng.random(len(c2)) < 0.7
        c3 = c2.retain(m2)
        arrays.update({f"{k}__sub_mask": m1, f"{k}__ret_mask": m2,
                       f"{k}__c3_depths": c3.depths.astype(np.int16), f"{k}__c3_bits": c3.bits,
                       f"{k}__c3_lo": c3.lo, f"{k}__c3_hi": c3.hi,
                       f"{k}__c3_diameter": np.float64(c3.diameter())})
        qi, ci = c3.build_index().query_boxes(q - 0.05, q + 0.05)
        arrays[f"{k}__qb_qi"], arrays[f"{k}__qb_ci"] = qi.astype(np.int32), ci.astype(np.int32)
    save("select", **arrays)


def gen_knn():
    """Large-k nearest neighbours and neighbourhood selection (warp top-k up to
    256 entries, radix-sort path beyond) from the reference."""
    from conftest import random_covering

    rng = np.random.default_rng(307)
    arrays = {}
    for t in range(3):
        root = cg_geo.Box([-2.0, 1.0], [3.0, 4.0]) if t % 2 else cg_geo.Box([0.0, 0.0], [1.0, 1.0])
        cov = random_covering(rng, root, rounds=10 + t, keep_fraction=0.8)
        idx = cov.build_index()
        key = f"cov{t}"
        arrays.update({f"{key}__root_lo": root.lo, f"{key}__root_hi": root.hi,
                       f"{key}__depths": cov.depths.astype(np.int16), f"{key}__bits": cov.bits})
        q = np.vstack([cov.centers()[rng.integers(0, len(cov), 12)],
                       rng.uniform(root.lo - 0.3, root.hi + 0.3, (12, 2))])
        arrays[f"{key}__q"] = q
        for k in (33, 64, 100, 129, 256, 257, 400, len(cov) + 5):
            res = idx.knn_indices_many(q, k)
            width = min(k, len(cov))
            arrays[f"{key}__knn{k}"] = np.stack(
                [np.pad(r[0], (0, width - len(r[0])), constant_values=-1) for r in res])
            arrays[f"{key}__clamped{k}"] = np.array([r[1] for r in res])
        b = cg_ad.select_boundary_mask(cov, idx, 0.01)
        arrays[f"{key}__boundary"] = b
        for N in (40, 300):
            arrays[f"{key}__nbr{N}"] = cg_ad.select_neighborhood_mask(cov, idx, b, N)
        arrays[f"{key}__ks"] = np.array([33, 64, 100, 129, 256, 257, 400, len(cov) + 5])
    save("knn", **arrays)


# -- 6. engine runs ------------------------------------------------------------------

def ref_run(ref_model, iterations, inputs_counts, frac, bloat, mode="full", N=3,
            initial_depth=None, initial_grid=None):
    """cg/engine.py:133-215 with the BASELINE 'initial grid' (iteration 1
    splits the root initial_depth times, or builds a non-dyadic grid in an
    extended root); reference functions throughout."""
    set_fractions(frac)
    inputs = cg_sys.sample_inputs(ref_model.U, inputs_counts)
    cfg = cg_image.ImageConfig(2 if frac is not None else 3, bloat)
    if initial_grid is not None:
        r_lo, r_hi, initial_depth = O.extended_root(ref_model.X.lo, ref_model.X.hi, initial_grid)
        cov = cg_geo.Covering.initial(cg_geo.Box(r_lo, r_hi))
    else:
        cov = cg_geo.Covering.initial(ref_model.X)
    metrics = []
    ok = True
    for k in range(1, iterations + 1):
        pre = cov.build_index()
        bnd = cg_ad.select_boundary_mask(cov, pre, 0.01)
        if k == 1:
            cov = split_all(cov, ref_model.n if initial_depth is None else initial_depth)
            if initial_grid is not None:
                cov = cov.retain(O.grid_mask(cov.depths, cov.bits, cov.n, initial_grid))
        elif mode == "full":
            cov = cov.subdivide(None)
        else:
            cov = cov.subdivide(bnd | cg_ad.select_neighborhood_mask(cov, pre, bnd, N))
        before = len(cov)
        g = cg_gr.build_graph_serial(cov, cov.build_index(), ref_model, inputs, cfg)
        keep = cg_an.non_leaving_mask(g)
        new = cov.retain(keep)
        ok &= cg_en._containment_defect(new, pre) <= 1e-12
        metrics.append((k, before, len(new), g.edge_count, int(bnd.sum()), new.diameter()))
        cov = new
        if len(cov) == 0:
            break
    set_fractions(None)
    return cov, np.array(metrics, dtype=np.float64), ok


def gen_runs():
    arrays = {}

    def rec(key, cov, metrics, ok):
        arrays.update({f"{key}__depths": cov.depths.astype(np.int16), f"{key}__bits": cov.bits,
                       f"{key}__metrics": metrics, f"{key}__containment_ok": np.int8(ok)})
        print(f"  run {key}: final {len(cov)} cells, metrics rows {len(metrics)}")

    c1 = config(1)
    ref1 = cg_sys.SystemModel("pendulum", 2, 1, cg_geo.Box(c1.model.X.lo, c1.model.X.hi),
                              cg_geo.Box(c1.model.U.lo, c1.model.U.hi),
                              O.make_step(c1.model.step.spec()))
    rec("config1", *ref_run(ref1, 4, 11, corners_plus_center(2), 0.1, initial_depth=12))
    c3 = config(3)
    ref3 = cg_sys.SystemModel("cstr_dimless", 2, 1, cg_geo.Box(c3.model.X.lo, c3.model.X.hi),
                              cg_geo.Box(c3.model.U.lo, c3.model.U.hi),
                              O.make_step(c3.model.step.spec()))
    rec("config3", *ref_run(ref3, 9, 21, lattice_fractions(2, 3), 0.1, mode="adaptive", N=3,
                            initial_depth=10))
    rec("pendulum_grid48", *ref_run(ref1, 3, 11, corners_plus_center(2), 0.1,
                                    initial_grid=(48, 48)))
    c5 = config(5)
    ref5 = cg_sys.SystemModel("cartpole", 4, 1, cg_geo.Box(c5.model.X.lo, c5.model.X.hi),
                              cg_geo.Box(c5.model.U.lo, c5.model.U.hi),
                              O.make_step(c5.model.step.spec()))
    rec("cartpole_grid6", *ref_run(ref5, 3, 11, corners_plus_seeded(4, 8, 2), 0.1,
                                   mode="adaptive", N=3, initial_grid=(6, 6, 6, 6)))
    cstr = cg_sys.cstr_model()
    rec("cstr_full6", *ref_run(cstr, 6, 3, None, 0.1))
    rec("cstr_n3_9", *ref_run(cstr, 9, 3, None, 0.1, mode="adaptive", N=3))
    rec("linear12", *ref_run(cg_sys.linear_test_model(2.0), 12, 3, None, 0.05))
    # adaptive to depth ~50: past any dense slot table (the sparse index)
    rec("linear_n3_48", *ref_run(cg_sys.linear_test_model(2.0), 48, 3, None, 0.05,
                                 mode="adaptive", N=3))
    # the reference's own engine.run on its default configuration (cross-check of ref_run)
    res = cg_en.run(cg_en.RunConfig(model=cstr, iterations=6))
    arrays["cstr_full6_engine__bits"] = res.covering.bits
    arrays["cstr_full6_engine__edges"] = np.array([m.edges for m in res.metrics])
    save("runs", **arrays)


# -- 7. config front end (cg/config.py) ---------------------------------------------

CONFIG_CASES = [  # (file_values, overrides, CISGRAPH_WORKERS or None)
    ({}, {}, None),
    ({"iterations": "5"}, {"iterations": "7"}, None),
    ({"model": "linear", "linear.a": "2.0", "mode": "adaptive", "N": "5", "delta": "0.02",
      "include_face_points": "yes", "input_grid": "5"}, {}, None),
    ({"model": "cstr", "cstr.q": "120", "cstr.UA": "6e4", "input_grid": "4,3"},
     {"samples_per_dim": "4"}, None),
    ({"model": "shift", "shift.offset": "0.25", "min_diameter": "0.01", "bloat": "0.2",
      "batch_size": "64", "workers": "2", "strict_largest_scc": "on"}, {"mode": None}, None),
    ({"model": "identity", "identity.xlo": "-2", "identity.xhi": "3"},
     {"workers": "1", "N": "0"}, "3"),
    ({"cell_count": "4"}, {}, None),
    ({"iterations": "many"}, {}, None),
    ({"iterations": "0"}, {}, None),
    ({"model": "cstr", "linear.a": "2"}, {}, None),
    ({"model": "linear", "linear.zz": "2"}, {}, None),
    ({"model": "linear", "linear.a": "two"}, {}, None),
    ({"model": "foo"}, {}, None),
    ({"mode": "bar"}, {}, None),
    ({"delta": "0"}, {}, None),
    ({"bloat": "-1"}, {}, None),
    ({"min_diameter": "-1"}, {}, None),
    ({"N": "-1"}, {}, None),
    ({"include_face_points": "maybe"}, {}, None),
    ({"input_grid": "1"}, {}, None),
    ({"input_grid": "a,b"}, {}, None),
    ({"samples_per_dim": "1"}, {}, None),
    ({"batch_size": "0"}, {}, None),
    ({"workers": "0"}, {}, None),
    ({}, {}, "0"),
    ({"model": "linear", "linear.xlo": "3", "linear.xhi": "1"}, {}, None),
    ({"strict_largest_scc": "nope"}, {}, None),
]

CONFIG_TEXTS = [
    "iterations = 12\nmodel = linear\nlinear.a = 2.0\n",
    "# a comment\n\nmode = adaptive  # trailing\n",
    "  a = b = c  \n\tbloat=0.3\n#x = 1\n",
    "iterations 12\n",
    "ok = 1\n\n  # only comment\nbroken line here\n",
]


def _summarize_run_config(rc):
    m = rc.model
    return {"model": m.name, "n": m.n, "m": m.m,
            "X": [list(map(float, m.X.lo)), list(map(float, m.X.hi))],
            "U": [list(map(float, m.U.lo)), list(map(float, m.U.hi))],
            "iterations": rc.iterations, "min_diameter": rc.min_diameter,
            "mode": rc.adaptive.mode, "N": rc.adaptive.n_neighbors, "delta": rc.adaptive.delta,
            "include_face_points": rc.adaptive.include_face_points,
            "samples_per_dim": rc.image.samples_per_dim, "bloat": rc.image.bloat,
            "batch_size": rc.plan.batch_size, "workers": rc.plan.workers,
            "input_counts": rc.input_counts if isinstance(rc.input_counts, int)
            else list(rc.input_counts),
            "strict_largest_scc": rc.strict_largest_scc}


def gen_config():
    """The reference's resolve_config / parse_config_text / render_config on
    valid and invalid inputs: effective dicts, RunConfig fields, the model's
    step on fixed points, or the ConfigError key and message."""
    import json
    import os
    from cisgraph import config as cg_cfg

    cases = []
    rng = np.random.default_rng(77)
    for fv, ov, env in CONFIG_CASES:
        saved = os.environ.pop(cg_cfg.WORKERS_ENV_VAR, None)
        if env is not None:
            os.environ[cg_cfg.WORKERS_ENV_VAR] = env
        try:
            r = cg_cfg.resolve_config(fv, ov)
            rc = r.run_config
            x = rng.uniform(rc.model.X.lo, rc.model.X.hi, size=(6, rc.model.n))
            u = np.asarray(rc.model.U.lo, dtype=np.float64)
            out = {"effective": r.effective, "rendered": cg_cfg.render_config(r.effective),
                   "run_config": _summarize_run_config(rc),
                   "x": x.tolist(), "u": u.tolist(),
                   "step": np.asarray(rc.model.map_points(x, u)).tolist()}
        except cg_cfg.ConfigError as exc:
            out = {"error_key": exc.key, "error": str(exc)}
        finally:
            os.environ.pop(cg_cfg.WORKERS_ENV_VAR, None)
            if saved is not None:
                os.environ[cg_cfg.WORKERS_ENV_VAR] = saved
        cases.append({"file": fv, "overrides": ov, "env_workers": env, **out})
    texts = []
    for t in CONFIG_TEXTS:
        try:
            texts.append({"text": t, "values": cg_cfg.parse_config_text(t)})
        except cg_cfg.ConfigError as exc:
            texts.append({"text": t, "error_key": exc.key, "error": str(exc)})
    (HERE / "config.json").write_text(json.dumps({"cases": cases, "texts": texts}, indent=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["steps", "enclosures", "graphs", "prune", "scc", "formats", "select",
                             "knn", "runs", "config"]
    for w in which:
        globals()[f"gen_{w}"]()
