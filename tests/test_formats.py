"""CPU: libgis's cells-file row formatter (host C++, no GPU needed) against
the reference's write_cells_file bytes (tests/golden/formats.npz)."""

import ctypes as C

import numpy as np
import pytest

from oracle import gis_oracle as O


@pytest.fixture(scope="module")
def lib():
    from paper_2202_06111_b200 import _device as D
    from paper_2202_06111_b200.build import build

    build()
    return D.load_library()


def _rows(lib, dep, bits, lo, hi, status, threads):
    n = lo.shape[1]
    dep = np.ascontiguousarray(dep, dtype=np.int32)
    bits = np.ascontiguousarray(bits, dtype=np.int64)
    lo_s, hi_s = np.ascontiguousarray(lo.T), np.ascontiguousarray(hi.T)
    out, nb = C.c_void_p(), C.c_int64()
    st = None if status is None else np.ascontiguousarray(status, dtype=np.uint8)
    rc = lib.gis_format_cells(dep.ctypes.data, bits.ctypes.data, lo_s.ctypes.data,
                              hi_s.ctypes.data, n, len(dep),
                              None if st is None else st.ctypes.data, threads,
                              C.byref(out), C.byref(nb))
    assert rc == 0
    try:
        return C.string_at(out, nb.value)
    finally:
        lib.gis_free_host(out)


def _body(txt):
    return b"".join(txt.splitlines(keepends=True)[2:])


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_cells_rows_match_reference(golden, lib, threads):
    g = golden("formats")
    keys = g.keys("cells_txt")
    assert len(keys) >= 8
    for k in keys:
        c = g.case(k)
        lo, hi = O.boxes_from_paths(c["root_lo"], c["root_hi"], c["depths"], c["bits"])
        got = _rows(lib, c["depths"], c["bits"], lo, hi, c["status"], threads)
        assert got == _body(c["cells_txt"].tobytes()), k
        got = _rows(lib, c["depths"], c["bits"], lo, hi, None, threads)
        assert got == _body(c["cells_plain_txt"].tobytes()), k


def test_g17_edge_values(lib):
    """'%.17g' from libgis equals CPython's format(x, '.17g') on awkward values."""
    vals = np.array([0.0, -0.0, 1e16, 1e17, 1.5e-5, 0.1, -2.4, 1 / 3, 5e-324, 1.7976931348623157e308,
                     np.inf, -np.inf, 123456789012345678.0, 2.0 ** -30, 0.21, -0.20999999999999999])
    lo = vals[:, None]
    hi = vals[:, None]
    got = _rows(lib, np.ones(len(vals)), np.zeros(len(vals)), lo, hi, None, 1).decode()
    want = "".join(f"0 1 {format(v, '.17g')} {format(v, '.17g')} retained\n" for v in vals)
    assert got == want
