"""CPU: the oracle's SCC / strict-mode / reverse-CSR restatement against the
reference's own outputs (tests/golden/scc.npz, made by make_golden.py)."""

import numpy as np

from oracle import gis_oracle as O


def test_scc_partition_matches_reference(golden):
    g = golden("scc")
    keys = g.keys("component_of")
    assert len(keys) >= 40
    for k in keys:
        c = g.case(k)
        nv = len(c["indptr"]) - 1
        labels, ncomp, nontriv = O.scc(c["indptr"], c["indices"], nv)
        want, order = O.canonical_components(c["component_of"])
        assert np.array_equal(labels, want), k
        assert ncomp == (int(c["component_of"].max()) + 1 if nv else 0), k
        assert np.array_equal(nontriv, c["nontrivial"][order]), k


def test_tarjan_ids_match_reference_exactly(golden):
    """The oracle's Tarjan reproduces the reference's pop-order ids bit for bit."""
    g = golden("scc")
    for k in g.keys("component_of"):
        c = g.case(k)
        comp, _ = O.tarjan(np.asarray(c["indptr"]), np.asarray(c["indices"], dtype=np.int64),
                           len(c["indptr"]) - 1)
        assert np.array_equal(comp, c["component_of"]), k


def test_modes_and_reverse_csr_match_reference(golden):
    g = golden("scc")
    for k in g.keys("component_of"):
        c = g.case(k)
        nv = len(c["indptr"]) - 1
        ip, ix = c["indptr"], c["indices"].astype(np.int64)
        assert np.array_equal(O.non_leaving_mask(ip, ix, nv), c["keep"]), k
        assert np.array_equal(O.non_leaving_mask(ip, ix, nv, strict_largest=True),
                              c["keep_strict"]), k
        rptr, rind = O.reverse_csr(ip, ix, nv)
        assert np.array_equal(rptr, c["rptr"]) and np.array_equal(rind, c["rind"]), k


def test_canonical_components_small():
    labels, order = O.canonical_components(np.array([2, 0, 2, 1, 0]))
    assert labels.tolist() == [0, 1, 0, 2, 1]
    assert order.tolist() == [2, 0, 1]
