"""GPU parity of K6 (csrc/gis_scc.cu): strongly_connected_components,
non_leaving_mask(strict_largest=True), reverse_csr and self_loop_mask against
the reference's own outputs (tests/golden/scc.npz), the reference's
tests/test_analysis.py shapes, and -- at BASELINE config 2's full size --
scipy's strong-components partition and the K3 peel mask."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _graph(c):
    from paper_2202_06111_b200.graph import SymbolicImage

    nv = len(c["indptr"]) - 1
    return SymbolicImage(np.zeros(nv, np.int64), np.arange(nv), c["indptr"],
                         c["indices"].astype(np.int64))


def test_scc_matches_reference_golden(golden):
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.analysis import strongly_connected_components

    g = golden("scc")
    keys = g.keys("component_of")
    assert len(keys) >= 40
    for k in keys:
        c = g.case(k)
        got = strongly_connected_components(_graph(c))
        want, order = O.canonical_components(c["component_of"])
        assert np.array_equal(got.component_of, want), k
        assert got.n_components == len(order), k
        assert np.array_equal(got.nontrivial, c["nontrivial"][order]), k
        # members() partitions the vertices (tests/test_analysis.py:42-48)
        assert sorted(int(v) for p in got.members() for v in p) == list(range(len(want))), k


def test_modes_match_reference_golden(golden):
    from paper_2202_06111_b200.analysis import non_leaving_mask

    g = golden("scc")
    for k in g.keys("component_of"):
        c = g.case(k)
        gr = _graph(c)
        assert np.array_equal(non_leaving_mask(gr), c["keep"]), k
        assert np.array_equal(non_leaving_mask(gr, strict_largest=True), c["keep_strict"]), k


def test_reverse_csr_and_self_loops_match_reference(golden):
    g = golden("scc")
    for k in g.keys("component_of"):
        c = g.case(k)
        gr = _graph(c)
        rptr, rind = gr.reverse_csr()
        assert np.array_equal(rptr, c["rptr"]), k
        assert np.array_equal(rind, c["rind"]), k
        assert np.array_equal(gr.self_loop_mask(), c["loops"]), k


def test_reference_analysis_shapes():
    """tests/test_analysis.py:27-91 of the reference, through the package API."""
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.analysis import non_leaving, strongly_connected_components
    from paper_2202_06111_b200.graph import SymbolicImage

    def graph_from_edges(n, edges):
        src = np.array([e[0] for e in edges], dtype=np.int64)
        dst = np.array([e[1] for e in edges], dtype=np.int64)
        ip, ix = O.csr_from_pairs(src, dst, n)
        depth = max(1, int(np.ceil(np.log2(max(n, 2)))))
        return SymbolicImage(np.full(n, depth), np.arange(n), ip, ix)

    g = graph_from_edges(4, [(1, 2), (2, 1), (2, 3)])
    scc = strongly_connected_components(g)
    comps = {frozenset(int(v) for v in p): bool(scc.nontrivial[scc.component_of[p[0]]])
             for p in scc.members()}
    assert comps[frozenset({1, 2})] is True and comps[frozenset({3})] is False
    g = graph_from_edges(2, [(1, 1)])
    scc = strongly_connected_components(g)
    assert scc.nontrivial[scc.component_of[1]] and not scc.nontrivial[scc.component_of[0]]
    g = graph_from_edges(50_000, [(i, i + 1) for i in range(49_999)])
    assert strongly_connected_components(g).n_components == 50_000
    g = graph_from_edges(6, [(0, 1), (1, 2), (2, 0), (3, 4), (4, 3), (5, 3)])
    assert {v.bits for v in non_leaving(g)} == {0, 1, 2, 3, 4, 5}
    assert {v.bits for v in non_leaving(g, strict_largest=True)} == {0, 1, 2}
    g = graph_from_edges(0, [])
    assert strongly_connected_components(g).n_components == 0
    assert non_leaving(g, strict_largest=True) == set()


@pytest.mark.parametrize("n", [50, 300, 1000, 5000])
def test_random_digraphs_against_oracle(n):
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.analysis import non_leaving_mask, strongly_connected_components
    from paper_2202_06111_b200.graph import SymbolicImage

    rng = np.random.default_rng(n)
    for deg in (0.7, 1.0, 2.0, 4.0):
        m = int(deg * n)
        ip, ix = O.csr_from_pairs(rng.integers(0, n, m), rng.integers(0, n, m), n)
        g = SymbolicImage(np.zeros(n, np.int64), np.arange(n), ip, ix)
        labels, ncomp, nontriv = O.scc(ip, ix, n)
        got = strongly_connected_components(g)
        assert np.array_equal(got.component_of, labels)
        assert got.n_components == ncomp and np.array_equal(got.nontrivial, nontriv)
        assert np.array_equal(non_leaving_mask(g, strict_largest=True),
                              O.non_leaving_mask(ip, ix, n, strict_largest=True))


def test_config2_full_size_scc():
    """V = 1,048,576, E = 103,838,696: the K6 partition equals scipy's strong
    components (canonicalised); the union of nontrivial components lies in
    the K3 keep mask and the strict mask lies inside it."""
    import torch
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import Covering, SpatialIndex, sample_inputs
    from paper_2202_06111_b200.analysis import (non_leaving_dev, non_leaving_strict_dev,
                                                scc_dev)
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.graph import SymbolicImage, build_graph_rows

    cfg = config(2)
    m = cfg.model
    cov = Covering.initial(m.X)
    for _ in range(cfg.initial_depth):
        cov = cov.subdivide(None)
    ip, ix = build_graph_rows(cov, SpatialIndex._dyadic(cov), m,
                              sample_inputs(m.U, cfg.input_counts), cfg.image)
    g = SymbolicImage._from_device(cov, ip, ix)
    assert g.edge_count == 103_838_696
    comp, sizes, nontriv, ncomp, stats = scc_dev(g)
    keep, _ = non_leaving_dev(g)
    strict, _ = non_leaving_strict_dev(g)
    torch.cuda.synchronize()
    V = g.n_vertices
    A = csr_matrix((np.ones(g.edge_count, dtype=np.int8), ix.cpu().numpy(), ip.cpu().numpy()),
                   shape=(V, V))
    n_ref, lab = connected_components(A, directed=True, connection="strong")
    want, _ = O.canonical_components(lab)
    got = comp.cpu().numpy()
    assert ncomp == n_ref
    assert np.array_equal(got, want)
    keep = keep.cpu().numpy().astype(bool)
    strict = strict.cpu().numpy().astype(bool)
    in_nontriv = nontriv.cpu().numpy().astype(bool)[got]
    assert not (in_nontriv & ~keep).any()
    assert not (strict & ~keep).any()
    assert int(strict.sum()) > 0
    print(f"config 2: {ncomp} components, nontrivial {int(nontriv.sum())}, "
          f"strict kept {int(strict.sum())} of {int(keep.sum())}; K6 outer/rounds {stats}")
