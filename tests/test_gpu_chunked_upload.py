"""Coverings built from pinned host tensors upload their cell bounds in
chunks on a side stream (geometry._upload_chunked); a graph build's K1
starts on each chunk as it lands (gis_ctx_input_chunks).  The graph must
equal the one built from device arrays, and every other use of the bounds
must wait for the copies."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pinned_twin(cov):
    from paper_2202_06111_b200 import Covering

    pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
           for x in (cov.depths, cov.bits, cov.lo, cov.hi)]
    c2 = Covering(cov.root, pin[0], pin[1], pin[2], pin[3], _sorted=True)
    return c2, pin


def _uniform(cid, depth=None):
    from paper_2202_06111_b200 import Covering
    from paper_2202_06111_b200.configs import config

    cfg = config(cid)
    m = cfg.model
    d = cfg.initial_depth if depth is None else depth
    return cfg, Covering.uniform(m.X, d)


@pytest.mark.parametrize("cid,depth", [(2, 18), (2, 20), (4, 18)])
def test_chunked_upload_graph_equals_device_build(cid, depth):
    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.graph import build_graph_serial

    cfg, cov = _uniform(cid, depth)
    m = cfg.model
    inputs = sample_inputs(m.U, cfg.input_counts)
    g0 = build_graph_serial(cov, cov.build_index(), m, inputs, cfg.image)
    c2, _pin = _pinned_twin(cov)
    assert c2._pend is not None, "pinned bounds should take the chunked upload"
    g1 = build_graph_serial(c2, c2.build_index(), m, inputs, cfg.image)
    assert c2._pend is None
    assert np.array_equal(g0.indptr, g1.indptr)
    assert np.array_equal(g0.indices, g1.indices)
    assert np.array_equal(non_leaving_mask(g0), non_leaving_mask(g1))


def test_chunked_upload_other_uses_wait():
    """Bounds read before any graph build (host views, retain, k-NN through
    the index, boundary selection) see the whole upload."""
    from paper_2202_06111_b200.adaptive import boundary_dev

    cfg, cov = _uniform(2, 18)
    keep = np.zeros(len(cov), dtype=bool)
    keep[::3] = True
    c2, _pin = _pinned_twin(cov)
    assert np.array_equal(c2.lo, cov.lo) and np.array_equal(c2.hi, cov.hi)
    c3, _pin3 = _pinned_twin(cov)
    r = c3.retain(keep)
    assert np.array_equal(r.lo, cov.retain(keep).lo)
    c4, _pin4 = _pinned_twin(cov)
    idx = c4.build_index()
    b4 = boundary_dev(c4, idx, 0.01, True).cpu().numpy()
    b0 = boundary_dev(cov, cov.build_index(), 0.01, True).cpu().numpy()
    assert np.array_equal(b4, b0)
    c5, _pin5 = _pinned_twin(cov)
    idx5 = c5.build_index()
    assert np.array_equal(idx5.lo, cov.lo)


def test_chunked_upload_row_range_and_repeat():
    """A row-range build (multi-GPU ranks) and a second build of the same
    covering after the chunks were consumed."""
    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.graph import build_graph_rows

    cfg, cov = _uniform(2, 18)
    m = cfg.model
    inputs = sample_inputs(m.U, cfg.input_counts)
    V = len(cov)
    a, b = V // 3, 2 * V // 3
    ip0, ix0 = build_graph_rows(cov, cov.build_index(), m, inputs, cfg.image, a, b)
    c2, _pin = _pinned_twin(cov)
    ip1, ix1 = build_graph_rows(c2, c2.build_index(), m, inputs, cfg.image, a, b)
    assert torch.equal(ip0, ip1) and torch.equal(ix0, ix1)
    ip2, ix2 = build_graph_rows(c2, c2.build_index(), m, inputs, cfg.image)
    ip3, ix3 = build_graph_rows(cov, cov.build_index(), m, inputs, cfg.image)
    assert torch.equal(ip2, ip3) and torch.equal(ix2, ix3)
