"""The drop-in boundary at the C ABI, exercised with the REFERENCE package:
the unmodified cisgraph (baseline/_ref, installed by __graft_entry__.build)
runs its own engine.run once natively and once with integration/
cisgraph_gis.py installed (build_graph_parallel and non_leaving_mask through
libgis over ctypes); coverings, metrics and termination must be identical.
Skipped when the reference is not installed next to the repo."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def cg():
    if not (REF / "cisgraph" / "__init__.py").exists():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT / "integration"))
    import cisgraph

    yield cisgraph
    import cisgraph_gis

    cisgraph_gis.uninstall()


def _summary(res):
    return ([(m.cells_before, m.cells_after, m.edges, m.boundary_cells, m.diameter)
             for m in res.metrics], res.covering.depths.tolist(), res.covering.bits.tolist(),
            res.termination, res.containment_ok)


@pytest.mark.parametrize("case", ["cstr_full5", "cstr_adaptive8", "linear12", "identity4",
                                  "shift"])
def test_reference_engine_with_libgis_binding_equals_native(cg, case):
    import cisgraph_gis
    from cisgraph import system as S
    from cisgraph.adaptive import AdaptiveConfig
    from cisgraph.engine import RunConfig, run

    rc = {"cstr_full5": lambda: RunConfig(model=S.cstr_model(), iterations=5),
          "cstr_adaptive8": lambda: RunConfig(model=S.cstr_model(), iterations=8,
                                              adaptive=AdaptiveConfig(mode="adaptive",
                                                                      n_neighbors=3)),
          "linear12": lambda: RunConfig(model=S.linear_test_model(2.0), iterations=12),
          "identity4": lambda: RunConfig(model=S.identity_model(), iterations=4),
          "shift": lambda: RunConfig(model=S.shift_model(), iterations=3)}[case]()
    cisgraph_gis.uninstall()
    native = _summary(run(rc))
    cisgraph_gis.install()
    try:
        gpu = _summary(run(rc))
    finally:
        cisgraph_gis.uninstall()
    assert gpu == native


def test_unsupported_step_is_refused(cg):
    import cisgraph_gis
    from cisgraph import geometry as G, system as S

    model = S.SystemModel("custom", 1, 1, G.Box([0.0], [1.0]), G.Box([0.0], [1.0]),
                          lambda x, u: x)
    with pytest.raises(TypeError, match="no device form"):
        cisgraph_gis.device_model(model.step, 1, 1)
