"""Full-size parity digests recorded from the REFERENCE itself.

Runs the unmodified ``cisgraph`` (imported from /root/reference/pkg/src, as
``make_golden.py`` does) on the BASELINE full-size configurations and
records sha256 digests of its graphs and keep masks, so the GPU tests can
compare the whole CSR and keep mask element-for-element at full size
(VERDICT r01 "Next round" item 2):

* config 2 (pendulum RK4 1024^2, 21 inputs, 20 samples): the reference's
  own ``build_graph_parallel`` (cg/graph.py:295-351, BuildPlan(1024, 8
  workers)) and ``non_leaving_mask`` (cg/analysis.py:120-161, Tarjan +
  reverse closure).  Whole-graph digests plus per-chunk row digests, and the
  reference's phase times on this container's cores.
* config 4 (Lorenz 256^3, 9 inputs, 16 samples) and config 5's first
  iteration (cart-pole 48^4, 11 inputs, 24 samples): the reference's
  ``_edges_for_range`` (cg/graph.py:196-211) + ``_csr_from_pairs``
  (:181-193) over contiguous source chunks of the full covering (a fork
  pool, one chunk per task; a whole ``build_graph_parallel`` would hold
  ~1e9 pre-dedupe int64 pairs).  Per-chunk row digests, the whole-graph
  digests of the concatenated rows, and the keep mask as the zero-out-degree
  peeling fixed point over those reference rows (equal to
  ``non_leaving_mask``'s default mode, asserted by the reference's own
  tests/test_analysis.py:74-82 and tests/test_acceptance.py:252-272; Tarjan
  in pure Python on 1.7e7 vertices is not practical).

Digest definitions (``tests/helpers.py:csr_digests`` computes the same on
the GPU side):
* ``indptr``: sha256 of int64 little-endian ``indptr``;
* ``indices``: sha256 of int32 little-endian ``indices``;
* ``keep``: sha256 of the keep mask as uint8 0/1;
* chunk c (rows [c*CHUNK, min((c+1)*CHUNK, V))): sha256 of the int64 row
  lengths followed by the int32 targets of those rows.

Run in the build container (takes ~25 min on 8 cores, ~45 more for 5run):
    python tests/golden/make_fullsize.py [2] [4] [5] [5run] [2scc] [4scc] [2text]
Writes tests/golden/fullsize_digests.json (committed).
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import make_golden as MG  # noqa: E402  (imports the reference, shapely stubbed)

cg_gr, cg_an, cg_geo, cg_sys, cg_image = MG.cg_gr, MG.cg_an, MG.cg_geo, MG.cg_sys, MG.cg_image
O, config = MG.O, MG.config

CHUNK = 16384
OUT = HERE / "fullsize_digests.json"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def chunk_digests(indptr, indices):
    V = len(indptr) - 1
    out = []
    for a in range(0, V, CHUNK):
        b = min(a + CHUNK, V)
        lens = np.diff(indptr[a:b + 1]).astype("<i8")
        out.append(sha(lens, indices[indptr[a]:indptr[b]].astype("<i4")))
    return out


def ref_model(key):
    m = config(key).model
    return cg_sys.SystemModel(m.name, m.n, m.m, cg_geo.Box(m.X.lo, m.X.hi),
                              cg_geo.Box(m.U.lo, m.U.hi), O.make_step(m.step.spec()))


def ref_covering(key):
    """Iteration 1's covering: the root split initial_depth times, or the
    non-dyadic grid embedded in an extended root (make_golden.ref_run)."""
    rc = config(key)
    m = rc.model
    if rc.initial_grid is not None:
        r_lo, r_hi, depth = O.extended_root(m.X.lo, m.X.hi, rc.initial_grid)
        cov = MG.split_all(cg_geo.Covering.initial(cg_geo.Box(r_lo, r_hi)), depth)
        return cov.retain(O.grid_mask(cov.depths, cov.bits, cov.n, rc.initial_grid))
    return MG.split_all(cg_geo.Covering.initial(m.X), rc.initial_depth)


_STATE = None


def _rows(task):
    a, b = task
    lo, hi, index, model, pts, cfg = _STATE
    src, dst = cg_gr._edges_for_range(a, b, lo, hi, index, model, pts, cfg)
    indptr, indices = cg_gr._csr_from_pairs(src - a, dst, b - a)
    return a, np.diff(indptr).astype(np.int64), indices.astype(np.int32)


def chunked_graph(key, workers):
    global _STATE
    rc = config(key)
    t0 = time.perf_counter()
    cov = ref_covering(key)
    index = cov.build_index()
    t_cov = time.perf_counter() - t0
    model = ref_model(key)
    inputs = cg_sys.sample_inputs(model.U, rc.input_counts)
    MG.set_fractions(rc.image.fractions)
    cfg = cg_image.ImageConfig(2, rc.image.bloat)
    _STATE = (cov.lo, cov.hi, index, model, inputs.points, cfg)
    V = len(cov)
    tasks = [(a, min(a + CHUNK, V)) for a in range(0, V, CHUNK)]
    lens = np.zeros(V, np.int64)
    parts = [None] * len(tasks)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        for i, (a, ln, ix) in enumerate(pool.imap(_rows, tasks, chunksize=1)):
            lens[a:a + len(ln)] = ln
            parts[i] = ix
            if i % 64 == 0:
                print(f"  config {key}: chunk {i}/{len(tasks)} "
                      f"{time.perf_counter() - t0:.0f} s", flush=True)
    t_build = time.perf_counter() - t0
    MG.set_fractions(None)
    indptr = np.zeros(V + 1, np.int64)
    np.cumsum(lens, out=indptr[1:])
    indices = np.concatenate(parts)
    return cov, indptr, indices, t_cov, t_build


def chunked_rows(cov, model, inputs, cfg, workers, tag):
    """Reference rows of a covering over contiguous chunks (see chunked_graph)."""
    global _STATE
    index = cov.build_index()
    _STATE = (cov.lo, cov.hi, index, model, inputs.points, cfg)
    V = len(cov)
    tasks = [(a, min(a + CHUNK, V)) for a in range(0, V, CHUNK)]
    lens = np.zeros(V, np.int64)
    parts = [None] * len(tasks)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        for i, (a, ln, ix) in enumerate(pool.imap(_rows, tasks, chunksize=1)):
            lens[a:a + len(ln)] = ln
            parts[i] = ix
            if i % 64 == 0:
                print(f"  {tag}: chunk {i}/{len(tasks)} {time.perf_counter() - t0:.0f} s",
                      flush=True)
    indptr = np.zeros(V + 1, np.int64)
    np.cumsum(lens, out=indptr[1:])
    return indptr, np.concatenate(parts), time.perf_counter() - t0


def record_run5(workers):
    """BASELINE config 5's whole engine loop (48^4 grid + two adaptive
    rounds, cg/engine.py:133-215 order as make_golden.ref_run composes it)
    with the reference's own select_boundary_mask / select_neighborhood_mask
    (cg/adaptive.py:93-150), Covering.subdivide / retain, the chunked
    reference rows and keep = peeling (Tarjan on 8M vertices in pure Python
    is not practical).  Per iteration: digests of the covering the graph is
    built on, the boundary and selection masks, the graph and the keep mask."""
    rc = config(5)
    model = ref_model(5)
    inputs = cg_sys.sample_inputs(model.U, rc.input_counts)
    MG.set_fractions(rc.image.fractions)
    cfg = cg_image.ImageConfig(2, rc.image.bloat)
    r_lo, r_hi, depth = O.extended_root(model.X.lo, model.X.hi, rc.initial_grid)
    cov = cg_geo.Covering.initial(cg_geo.Box(r_lo, r_hi))
    iters = []
    for k in range(1, rc.iterations + 1):
        t0 = time.perf_counter()
        rec = {"iteration": k}
        if k == 1:
            cov = MG.split_all(cov, depth)
            cov = cov.retain(O.grid_mask(cov.depths, cov.bits, cov.n, rc.initial_grid))
        else:
            pre = cov.build_index()
            bnd = MG.cg_ad.select_boundary_mask(cov, pre, rc.adaptive.delta)
            nbr = MG.cg_ad.select_neighborhood_mask(cov, pre, bnd, rc.adaptive.n_neighbors)
            rec["boundary"] = int(bnd.sum())
            rec["boundary_sha256"] = sha(bnd.astype(np.uint8))
            rec["neighborhood_sha256"] = sha(nbr.astype(np.uint8))
            cov = cov.subdivide(bnd | nbr)
        rec["select_s"] = time.perf_counter() - t0
        indptr, indices, rec["build_s"] = chunked_rows(cov, model, inputs, cfg, workers,
                                                       f"config 5 iteration {k}")
        t0 = time.perf_counter()
        keep = O.peel_fixed_point(indptr, indices, len(cov))
        rec["prune_s"] = time.perf_counter() - t0
        rec.update({
            "V": int(len(cov)), "E": int(indptr[-1]), "kept": int(keep.sum()),
            "bits_sha256": sha(cov.bits.astype("<i8")),
            "depths_sha256": sha(cov.depths.astype("<i8")),
            "indptr_sha256": sha(indptr.astype("<i8")),
            "indices_sha256": sha(indices.astype("<i4")),
            "keep_sha256": sha(keep.astype(np.uint8)),
            "chunks_sha256": chunk_digests(indptr, indices)})
        print(f"  iteration {k}: V={rec['V']} E={rec['E']} kept={rec['kept']}", flush=True)
        iters.append(rec)
        cov = cov.retain(keep)
    MG.set_fractions(None)
    return {"chunk": CHUNK, "workers": workers, "iterations": iters,
            "final_cells": int(len(cov)), "final_bits_sha256": sha(cov.bits.astype("<i8")),
            "final_depths_sha256": sha(cov.depths.astype("<i8"))}


def record(key, workers):
    print(f"config {key} ...", flush=True)
    rc = config(key)
    rec = {"chunk": CHUNK, "workers": workers}
    if key == 2:
        # the reference's own build_graph_parallel + non_leaving_mask
        t0 = time.perf_counter()
        cov = ref_covering(key)
        index = cov.build_index()
        rec["covering_index_s"] = time.perf_counter() - t0
        model = ref_model(key)
        inputs = cg_sys.sample_inputs(model.U, rc.input_counts)
        MG.set_fractions(rc.image.fractions)
        t0 = time.perf_counter()
        g = cg_gr.build_graph_parallel(cov, index, model, inputs,
                                       cg_image.ImageConfig(2, rc.image.bloat),
                                       cg_gr.BuildPlan(batch_size=1024, workers=workers))
        rec["build_s"] = time.perf_counter() - t0
        MG.set_fractions(None)
        t0 = time.perf_counter()
        keep = cg_an.non_leaving_mask(g)
        rec["prune_s"] = time.perf_counter() - t0
        rec["prune_kind"] = "reference non_leaving_mask (Tarjan + reverse closure)"
        indptr, indices = g.indptr, g.indices.astype(np.int32)
        peel = O.peel_fixed_point(indptr, indices, len(cov))
        rec["peel_equals_reference_keep"] = bool(np.array_equal(peel, keep))
    else:
        cov, indptr, indices, rec["covering_index_s"], rec["build_s"] = chunked_graph(key, workers)
        t0 = time.perf_counter()
        keep = O.peel_fixed_point(indptr, indices, len(cov))
        rec["prune_s"] = time.perf_counter() - t0
        rec["prune_kind"] = "numpy peeling fixed point over the reference rows"
    rec.update({
        "V": int(len(cov)), "E": int(indptr[-1]), "kept": int(keep.sum()),
        "bits_sha256": sha(cov.bits.astype("<i8")),
        "depths_sha256": sha(cov.depths.astype("<i8")),
        "indptr_sha256": sha(indptr.astype("<i8")),
        "indices_sha256": sha(indices.astype("<i4")),
        "keep_sha256": sha(keep.astype(np.uint8)),
        "chunks_sha256": chunk_digests(indptr, indices),
        "cpu": {"cores": workers, "os_cpu_count": os.cpu_count()},
    })
    print(f"  V={rec['V']} E={rec['E']} kept={rec['kept']} build {rec['build_s']:.0f} s "
          f"prune {rec['prune_s']:.0f} s", flush=True)
    return rec


def record_scc2(workers, key=2):
    """Config 2's graph from the reference's own build_graph_parallel, then
    the reference's strongly_connected_components (cg/analysis.py:109-117,
    Tarjan) and non_leaving_mask(strict_largest=True) (:120-161).  Component
    ids are compared through the partition: per vertex the smallest vertex
    of its component (the GPU numbers components by smallest member, an API
    difference documented in INTEGRATION.md; the partition is the contract)."""
    print(f"config {key} SCC ...", flush=True)
    if key == 2:
        rc = config(2)
        cov = ref_covering(2)
        index = cov.build_index()
        model = ref_model(2)
        inputs = cg_sys.sample_inputs(model.U, rc.input_counts)
        MG.set_fractions(rc.image.fractions)
        g = cg_gr.build_graph_parallel(cov, index, model, inputs,
                                       cg_image.ImageConfig(2, rc.image.bloat),
                                       cg_gr.BuildPlan(batch_size=1024, workers=workers))
        MG.set_fractions(None)
    else:  # the reference's rows over contiguous chunks (as record() does)
        cov, indptr, indices, _, _ = chunked_graph(key, workers)
        g = cg_gr.SymbolicImage(cov.depths, cov.bits, indptr, indices)
        del indices
    t0 = time.perf_counter()
    scc = cg_an.strongly_connected_components(g)
    scc_s = time.perf_counter() - t0
    comp = np.asarray(scc.component_of, dtype=np.int64)
    V = len(comp)
    first = np.full(scc.n_components, V, dtype=np.int64)
    np.minimum.at(first, comp, np.arange(V, dtype=np.int64))
    rep = first[comp].astype("<i4")
    nontriv = np.asarray(scc.nontrivial, dtype=bool)[comp]
    sizes = np.bincount(comp, minlength=scc.n_components)
    t0 = time.perf_counter()
    strict = cg_an.non_leaving_mask(g, strict_largest=True)
    strict_s = time.perf_counter() - t0
    rec = {"V": int(V), "E": int(g.indptr[-1]), "n_components": int(scc.n_components),
           "n_nontrivial": int(np.count_nonzero(scc.nontrivial)),
           "largest_nontrivial": int(sizes[np.asarray(scc.nontrivial, bool)].max()),
           "rep_sha256": sha(rep), "nontrivial_vertex_sha256": sha(nontriv.astype(np.uint8)),
           "strict_keep_sha256": sha(np.asarray(strict, dtype=np.uint8)),
           "strict_kept": int(np.count_nonzero(strict)),
           "scc_s": scc_s, "strict_s": strict_s,
           "definition": "rep[v] = smallest vertex of v's SCC (int32 LE); nontrivial per "
                         "vertex (uint8); strict keep mask (uint8)"}
    print(f"  components {rec['n_components']} nontrivial {rec['n_nontrivial']} "
          f"strict kept {rec['strict_kept']} (Tarjan {scc_s:.0f} s)", flush=True)
    return rec


class _HashWriter:
    """A text file that only hashes what is written (sha256 of the UTF-8 bytes)."""

    def __init__(self):
        self.h = hashlib.sha256()
        self.bytes = 0

    def write(self, s):
        b = s.encode()
        self.h.update(b)
        self.bytes += len(b)
        return len(s)


def record_text2(workers):
    """The reference's text writers at full size on config 2: the canonical
    edge list of its own build_graph_parallel graph (cg/graph.py:146-156,
    4.4 GB: offsets past 2^32 bytes) and the cells file (cg/geometry.py:
    588-620) of the covering retained by the keep mask, both as sha256 of
    the bytes the reference writes."""
    print("config 2 text ...", flush=True)
    rc = config(2)
    cov = ref_covering(2)
    index = cov.build_index()
    model = ref_model(2)
    inputs = cg_sys.sample_inputs(model.U, rc.input_counts)
    MG.set_fractions(rc.image.fractions)
    g = cg_gr.build_graph_parallel(cov, index, model, inputs,
                                   cg_image.ImageConfig(2, rc.image.bloat),
                                   cg_gr.BuildPlan(batch_size=1024, workers=workers))
    MG.set_fractions(None)
    t0 = time.perf_counter()
    w = _HashWriter()
    g.write_edge_list(w)
    edges_s = time.perf_counter() - t0
    keep = O.peel_fixed_point(g.indptr, g.indices.astype(np.int32), len(cov))
    kept = cov.retain(keep)
    c = _HashWriter()
    cg_geo.write_cells_file(kept, c)
    rec = {"edge_list_sha256": w.h.hexdigest(), "edge_list_bytes": w.bytes,
           "edge_list_s": edges_s, "cells_sha256": c.h.hexdigest(), "cells_bytes": c.bytes,
           "cells_rows": int(len(kept)),
           "definition": "sha256 of write_edge_list(graph) and of write_cells_file(covering "
                         "retained by the keep mask) as the reference writes them"}
    print(f"  edge list {w.bytes} bytes ({edges_s:.0f} s), cells {c.bytes} bytes", flush=True)
    return rec


def main():
    keys = sys.argv[1:] or ["2", "4", "5"]
    workers = int(os.environ.get("GIS_REF_WORKERS", os.cpu_count() or 1))
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    data["about"] = ("sha256 digests of the reference's full-size graphs and keep masks; "
                     "generated by tests/golden/make_fullsize.py")
    for key in keys:
        if key == "5run":  # config 5's whole adaptive run
            data["config5_run"] = record_run5(workers)
        elif key in ("2scc", "4scc"):  # SCC partition and strict-largest mask
            data[f"config{key[0]}_scc"] = record_scc2(workers, int(key[0]))
        elif key == "2text":  # config 2's edge list and cells file
            data["config2_text"] = record_text2(workers)
        else:
            data[f"config{key}"] = record(int(key), workers)
        OUT.write_text(json.dumps(data, indent=1) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
