"""GPU: edge lists formatted by libgis (gis_format_edges) and cells files
written through the package API, byte-for-byte against the reference's
outputs (tests/golden/formats.npz), plus config 2's full 103,838,696-edge
list checked by size and sampled rows."""

import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _graph_and_cov(c):
    from paper_2202_06111_b200 import Box, Covering
    from paper_2202_06111_b200.graph import SymbolicImage

    paths = ["-" if d == 0 else format(int(b), f"0{int(d)}b")
             for d, b in zip(c["depths"], c["bits"])]
    cov = Covering.from_paths(Box(c["root_lo"], c["root_hi"]), paths)
    g = SymbolicImage(c["depths"], c["bits"], c["indptr"], c["indices"].astype(np.int64))
    return g, cov


def test_edge_lists_match_reference(golden):
    g = golden("formats")
    for k in g.keys("edges_txt"):
        c = g.case(k)
        gr, cov = _graph_and_cov(c)
        want = c["edges_txt"].tobytes()
        assert gr.edge_list_bytes() == want, k
        buf = io.StringIO()
        gr.write_edge_list(buf)
        assert buf.getvalue().encode() == want, k


def test_cells_files_match_reference(golden):
    from paper_2202_06111_b200.geometry import CELL_STATUSES, write_cells_file

    g = golden("formats")
    for k in g.keys("cells_txt"):
        c = g.case(k)
        _, cov = _graph_and_cov(c)
        buf = io.StringIO()
        write_cells_file(cov, buf, [CELL_STATUSES[i] for i in c["status"]])
        assert buf.getvalue().encode() == c["cells_txt"].tobytes(), k
        buf = io.StringIO()
        write_cells_file(cov, buf)
        assert buf.getvalue().encode() == c["cells_plain_txt"].tobytes(), k


def test_config2_edge_list_full_size(tmp_path):
    from paper_2202_06111_b200 import Covering, SpatialIndex, sample_inputs
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
    E = g.edge_count
    path = tmp_path / "edges.tsv"
    with open(path, "w") as fp:
        g.write_edge_list(fp)
    assert path.stat().st_size == E * (20 + 1 + 20 + 1)  # every path has depth 20
    indptr, indices = g.indptr, g.indices
    paths = lambda v: format(int(cov.bits[v]), "020b")  # noqa: E731
    rng = np.random.default_rng(5)
    with open(path, "rb") as fp:
        for r in rng.integers(0, len(cov), 50):
            a, b = int(indptr[r]), int(indptr[r + 1])
            fp.seek(a * 42)
            got = fp.read((b - a) * 42).decode()
            want = "".join(f"{paths(r)} {paths(int(t))}\n" for t in indices[a:b])
            assert got == want, r
