"""The binding a `cisgraph` maintainer would add to route the reference's
own hot path through libgis.  Plain ctypes over the C ABI
of include/gis.h -- none of paper_2202_06111_b200's Python -- with the
reference's numpy arrays at the boundary and torch only for device memory.

    import cisgraph, cisgraph_gis
    cisgraph_gis.install()          # cisgraph.engine now builds and prunes on the GPU
    cisgraph.run(cisgraph.RunConfig(model=cisgraph.system.cstr_model(), iterations=20))

Replaces `build_graph_parallel` (cg/graph.py:295-351, the engine's call at
cg/engine.py:169) and `non_leaving_mask` (cg/analysis.py:120-161, called at
cg/engine.py:171).  The reference's registry models (cstr, linear, identity,
shift; cg/system.py:148-261) have device forms; any other step raises
TypeError (there is no CPU fallback).  tests/test_gpu_integration.py runs the
reference's engine with and without this binding and requires identical
coverings and metrics.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB = Path(os.environ.get("GIS_LIBRARY", Path(__file__).resolve().parents[1] /
                          "paper_2202_06111_b200" / "libgis.so"))
vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
pf64, pi64 = C.POINTER(C.c_double), C.POINTER(C.c_int64)
GIS_CSTR, GIS_LINEAR, GIS_IDENTITY, GIS_SHIFT = 4, 2, 0, 1
GIS_MAP, GIS_RK4 = 0, 2


class GisModel(C.Structure):  # include/gis.h: gis_model
    _fields_ = [("kind", C.c_int32), ("integrator", C.c_int32), ("substeps", C.c_int32),
                ("n", C.c_int32), ("m", C.c_int32), ("jit", C.c_int32),
                ("h", C.c_double), ("params", C.c_double * 64)]


_lib = None
_ctx = vp()


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(str(LIB))
        lib.gis_last_error.restype = C.c_char_p
        lib.gis_ctx_create.argtypes = [C.POINTER(vp), C.c_int]
        lib.gis_ctx_set_stream.argtypes = [vp, vp]
        lib.gis_index_build_dyadic.argtypes = [vp, i32, pf64, pf64, vp, vp, i64, C.POINTER(vp)]
        lib.gis_build_graph_begin.argtypes = [vp, vp, C.POINTER(GisModel), vp, vp, i64, i64,
                                              i64, pf64, i32, pf64, i32, f64, vp, pi64]
        lib.gis_csr_finish.argtypes = [vp, vp]
        lib.gis_prune.argtypes = [vp, vp, vp, i64, vp, C.POINTER(C.c_int32)]
        lib.gis_non_leaving_scc.argtypes = [vp, vp, vp, i64, C.c_int32, vp,
                                            C.POINTER(C.c_int32)]
        lib.gis_index_free.argtypes = [vp]
        _ok(lib.gis_ctx_create(C.byref(_ctx), 0), lib)
        _lib = lib
    return _lib


def _ok(rc, lib=None):
    if rc:
        raise RuntimeError((lib or _lib).gis_last_error().decode())


def _stream():
    import torch

    _ok(_load().gis_ctx_set_stream(_ctx, vp(torch.cuda.current_stream().cuda_stream)))


def device_model(step, n: int, m: int) -> GisModel:
    """gis_model for the reference's registry steps (cg/system.py:148-261)."""
    from cisgraph import system as S

    mm = GisModel()
    mm.n, mm.m, mm.substeps, mm.integrator = n, m, 1, GIS_MAP
    if isinstance(step, S.CstrStep):  # one RK4 step of h, parameters as its rhs folds them
        p = step.params
        mm.kind, mm.integrator, mm.h = GIS_CSTR, GIS_RK4, p.h
        vals = [p.q / p.V, p.c_Af, p.T_f, -p.E_over_R, p.k0, p.minus_dH / (p.rho * p.c_p),
                p.UA / (p.V * p.rho * p.c_p)]
    elif isinstance(step, S.LinearStep):
        mm.kind, mm.h, vals = GIS_LINEAR, 1.0, [step.a]
    elif isinstance(step, S.IdentityStep):
        mm.kind, mm.h, vals = GIS_IDENTITY, 1.0, []
    elif isinstance(step, S.ShiftStep):
        mm.kind, mm.h, vals = GIS_SHIFT, 1.0, [step.offset]
    else:
        raise TypeError(f"{type(step).__name__} has no device form in libgis")
    for i, v in enumerate(vals):
        mm.params[i] = float(v)
    return mm


def build_graph_parallel(covering, index, model, inputs, cfg, plan):
    """Drop-in for cisgraph.graph.build_graph_parallel (cg/graph.py:295):
    the same edge set for every plan, built in one K1 + K2 launch."""
    import torch

    from cisgraph.graph import SymbolicImage
    from cisgraph.image import _unit_grid

    lib = _load()
    _stream()
    dev = torch.device("cuda")
    V, n = covering.lo.shape
    if V == 0:
        return SymbolicImage(covering.depths, covering.bits, np.zeros(1, np.int64),
                             np.zeros(0, np.int64))
    depths = torch.as_tensor(covering.depths.astype(np.int32), device=dev)
    bits = torch.as_tensor(covering.bits, device=dev)
    lo = torch.as_tensor(np.ascontiguousarray(covering.lo.T), device=dev)  # SoA [n][V]
    hi = torch.as_tensor(np.ascontiguousarray(covering.hi.T), device=dev)
    rlo = np.ascontiguousarray(covering.root.lo, dtype=np.float64)
    rhi = np.ascontiguousarray(covering.root.hi, dtype=np.float64)
    idx = vp()
    _ok(lib.gis_index_build_dyadic(_ctx, n, rlo.ctypes.data_as(pf64), rhi.ctypes.data_as(pf64),
                                   vp(depths.data_ptr()), vp(bits.data_ptr()), V, C.byref(idx)))
    try:
        u = np.ascontiguousarray(np.atleast_2d(inputs.points), dtype=np.float64)
        frac = np.ascontiguousarray(_unit_grid(n, cfg.samples_per_dim), dtype=np.float64)
        mstruct = device_model(model.step, model.n, model.m)
        indptr = torch.empty(V + 1, dtype=torch.int64, device=dev)
        E = C.c_int64()
        _ok(lib.gis_build_graph_begin(_ctx, idx, C.byref(mstruct), vp(lo.data_ptr()),
                                      vp(hi.data_ptr()), V, 0, V, u.ctypes.data_as(pf64),
                                      len(u), frac.ctypes.data_as(pf64), len(frac),
                                      float(cfg.bloat), vp(indptr.data_ptr()), C.byref(E)))
        indices = torch.empty(max(E.value, 1), dtype=torch.int32, device=dev)
        _ok(lib.gis_csr_finish(_ctx, vp(indices.data_ptr())))
    finally:
        lib.gis_index_free(idx)
    return SymbolicImage(covering.depths, covering.bits, indptr.cpu().numpy(),
                         indices[:E.value].cpu().numpy().astype(np.int64))


def non_leaving_mask(graph, strict_largest: bool = False):
    """Drop-in for cisgraph.analysis.non_leaving_mask (cg/analysis.py:120)."""
    import torch

    lib = _load()
    _stream()
    V = len(graph.indptr) - 1
    if V == 0:
        return np.zeros(0, dtype=bool)
    ip = torch.as_tensor(np.asarray(graph.indptr, dtype=np.int64), device="cuda")
    ix = torch.as_tensor(np.asarray(graph.indices, dtype=np.int32), device="cuda")
    keep = torch.zeros(V, dtype=torch.uint8, device="cuda")
    if strict_largest:  # SCCs + closure of the largest nontrivial component
        _ok(lib.gis_non_leaving_scc(_ctx, vp(ip.data_ptr()), vp(ix.data_ptr()), V, 1,
                                    vp(keep.data_ptr()), None))
    else:  # the default mode's set, as the peeling fixed point
        _ok(lib.gis_prune(_ctx, vp(ip.data_ptr()), vp(ix.data_ptr()), V, vp(keep.data_ptr()),
                          None))
    return keep.cpu().numpy().astype(bool)


def install():
    """Rebind the reference engine's two hot calls (cg/engine.py:24-26 import
    them at module level, so the engine module is where they are rebound)."""
    import cisgraph.engine as E

    E.build_graph_parallel = build_graph_parallel
    E.non_leaving_mask = non_leaving_mask


def uninstall():
    import cisgraph.analysis as A
    import cisgraph.engine as E
    import cisgraph.graph as G

    E.build_graph_parallel = G.build_graph_parallel
    E.non_leaving_mask = A.non_leaving_mask
