"""ctypes binding of libgis.so (include/gis.h) and device-buffer plumbing.

Device buffers are torch tensors (PyTorch is used for device memory and the
current stream only); every computation is a libgis kernel.  There is no
CPU fallback: if the library or a CUDA device is missing, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libgis.so"
if os.environ.get("GIS_LIB_VARIANT"):  # tools: an experimental build (build.py --variant)
    LIB_PATH = _HERE / "build_obj" / f"var_{os.environ['GIS_LIB_VARIANT']}" / "libgis.so"

GIS_OK, GIS_E_INVALID, GIS_E_CUDA, GIS_E_OVERLAP, GIS_E_CAPACITY, GIS_E_STATE = range(6)
MAX_PARAMS = 64

p_i8 = C.POINTER(C.c_uint8)
p_i32 = C.POINTER(C.c_int32)
p_i64 = C.POINTER(C.c_int64)
p_f64 = C.POINTER(C.c_double)
vp = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


class GisModel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("integrator", C.c_int32), ("substeps", C.c_int32),
                ("n", C.c_int32), ("m", C.c_int32), ("jit", C.c_int32), ("h", C.c_double),
                ("params", C.c_double * MAX_PARAMS)]


# name -> (restype, argtypes); mirrors include/gis.h
SIGNATURES = {
    "gis_abi_version": (C.c_int, []),
    "gis_last_error": (C.c_char_p, []),
    "gis_ctx_create": (C.c_int, [C.POINTER(vp), C.c_int]),
    "gis_ctx_destroy": (C.c_int, [vp]),
    "gis_ctx_set_stream": (C.c_int, [vp, vp]),
    "gis_ctx_launch_count": (C.c_int64, [vp]),
    "gis_jit_register": (C.c_int, [vp, C.c_char_p, i32, i32, i32, i32, C.POINTER(C.c_int32)]),
    "gis_jit_compile_check": (C.c_int, [C.c_char_p, i32, i32, i32, i32, p_i64]),
    "gis_ctx_trim": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "gis_ctx_input_chunks": (C.c_int, [vp, C.c_int32, p_i64, C.POINTER(vp)]),
    "gis_ctx_pool_reserved": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "gis_ctx_enable_timing": (C.c_int, [vp, C.c_int]),
    "gis_ctx_phase_times": (C.c_int, [vp, p_f64, p_i64]),
    "gis_ctx_integrations": (C.c_int, [vp, p_i64, p_i64]),
    "gis_fp64_peak": (C.c_int, [vp, p_f64]),
    "gis_map_points": (C.c_int, [vp, C.POINTER(GisModel), vp, i64, p_f64, vp]),
    "gis_batch_enclosures": (C.c_int, [vp, C.POINTER(GisModel), vp, vp, i64, p_f64, i32, p_f64,
                                       i32, f64, vp, vp, vp]),
    "gis_index_build_dyadic": (C.c_int, [vp, i32, p_f64, p_f64, vp, vp, i64, C.POINTER(vp)]),
    "gis_index_build_boxes": (C.c_int, [vp, i32, vp, vp, i64, C.POINTER(vp)]),
    "gis_index_build_dyadic_mode": (C.c_int, [vp, i32, p_f64, p_f64, vp, vp, i64, i32,
                                              C.POINTER(vp)]),
    "gis_index_is_sparse": (C.c_int, [vp]),
    "gis_index_free": (C.c_int, [vp]),
    "gis_index_shape": (C.c_int, [vp, p_i64, p_i64]),
    "gis_query_boxes_begin": (C.c_int, [vp, vp, vp, vp, i64, vp, p_i64]),
    "gis_csr_finish": (C.c_int, [vp, vp]),
    "gis_build_graph_begin": (C.c_int, [vp, vp, C.POINTER(GisModel), vp, vp, i64, i64, i64,
                                        p_f64, i32, p_f64, i32, f64, vp, p_i64]),
    "gis_build_graph_memo_begin": (C.c_int, [vp, vp, C.POINTER(GisModel), vp, vp, i64, i64,
                                             i64, p_f64, i32, p_f64, i32, f64, vp, vp, i64,
                                             i64, vp, vp, vp, vp, vp, p_i64]),
    "gis_covering_origin": (C.c_int, [vp, i64, vp, i64, vp, i64, vp]),
    "gis_covering_forward": (C.c_int, [vp, i64, vp, i64, vp, vp]),
    "gis_csr_from_pairs": (C.c_int, [vp, vp, vp, i64, i64, vp, vp, p_i64]),
    "gis_csr_sources": (C.c_int, [vp, vp, i64, vp]),
    "gis_prune": (C.c_int, [vp, vp, vp, i64, vp, p_i32]),
    "gis_peel_init": (C.c_int, [vp, vp, i64, i64, i64, vp, vp]),
    "gis_peel_sweep": (C.c_int, [vp, vp, vp, i64, i64, vp, vp, p_i64]),
    "gis_peel_sweep_acc": (C.c_int, [vp, vp, vp, i64, i64, vp, vp, vp]),
    "gis_peel_local": (C.c_int, [vp, vp, vp, i64, i64, vp, vp, vp]),
    "gis_peel_p2p": (C.c_int, [vp, vp, vp, i64, i64, i64, vp, vp, i32, i32, C.c_uint32,
                               C.POINTER(C.c_int32)]),
    "gis_ipc_alloc": (C.c_int, [vp, i64, C.POINTER(vp), vp]),
    "gis_ipc_open": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "gis_ipc_close": (C.c_int, [vp]),
    "gis_ipc_free": (C.c_int, [vp]),
    "gis_bitmap_to_mask": (C.c_int, [vp, vp, i64, vp]),
    "gis_mask_to_bitmap": (C.c_int, [vp, vp, i64, vp]),
    "gis_scc": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, p_i64, p_i32]),
    "gis_non_leaving_scc": (C.c_int, [vp, vp, vp, i64, i32, vp, p_i32]),
    "gis_reverse_csr": (C.c_int, [vp, vp, vp, i64, vp, vp, i32]),
    "gis_self_loops": (C.c_int, [vp, vp, vp, i64, vp]),
    "gis_edge_list_offsets": (C.c_int, [vp, vp, vp, vp, i64, vp]),
    "gis_format_edges": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, i64, i64, vp]),
    "gis_format_cells": (C.c_int, [vp, vp, vp, vp, i32, i64, vp, i32, C.POINTER(vp), p_i64]),
    "gis_free_host": (None, [vp]),
    "gis_uniform_grid": (C.c_int, [vp, i32, i32, p_f64, p_f64, p_i64, p_i64, vp, vp, vp, vp]),
    "gis_count_mask": (C.c_int, [vp, vp, i64, p_i64]),
    "gis_grid_mask": (C.c_int, [vp, i32, i64, vp, vp, p_i64, vp]),
    "gis_subdivide": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "gis_retain": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "gis_select_boundary": (C.c_int, [vp, vp, vp, vp, i64, f64, i32, vp]),
    "gis_knn": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, i32, i32, vp, vp]),
    "gis_select_neighborhood": (C.c_int, [vp, vp, vp, vp, i64, vp, i32, vp]),
    "gis_containment_defect": (C.c_int, [vp, vp, vp, vp, i64, vp, vp, i64, p_f64]),
    "gis_select_boundary_range": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, f64, i32, vp]),
    "gis_select_neighborhood_range": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, i64, i32, i32,
                                                vp]),
    "gis_mask_andnot": (C.c_int, [vp, vp, vp, i64]),
    "gis_containment_defect_range": (C.c_int, [vp, vp, vp, vp, i64, vp, vp, i64, i64, i64,
                                               p_f64]),
    "gis_diameter": (C.c_int, [vp, i32, vp, vp, i64, p_f64]),
}

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load libgis.so (built in-tree by paper_2202_06111_b200.build)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2202_06111_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class GraphBuildError(RuntimeError):
    """The device graph build failed for a range of source cells
    (cg/graph.py:41-42)."""


def last_error() -> str:
    return load_library().gis_last_error().decode(errors="replace")


def check(status: int, what: str = ""):
    if status == GIS_OK:
        return
    msg = load_library().gis_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (GIS_E_INVALID, GIS_E_OVERLAP):
        raise ValueError(text)
    if status == GIS_E_CAPACITY:
        raise MemoryError(text)
    raise RuntimeError(text)


# ---------------------------------------------------------------- context --

_ctxs: dict = {}


def _torch():
    import torch

    return torch


def device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2202_06111_b200 needs a CUDA device (B200); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def ctx():
    """The libgis context of the current CUDA device, bound to torch's
    current stream."""
    torch = _torch()
    dev = device()
    lib = load_library()
    c = _ctxs.get(dev.index)
    if c is None:
        h = vp()
        check(lib.gis_ctx_create(C.byref(h), dev.index), "gis_ctx_create")
        c = _ctxs[dev.index] = h
    check(lib.gis_ctx_set_stream(c, vp(torch.cuda.current_stream(dev).cuda_stream)))
    return c


def launch_count() -> int:
    lib = load_library()
    return sum(int(lib.gis_ctx_launch_count(c)) for c in _ctxs.values())


def trim() -> int:
    """Give libgis's cached device memory back (gis_ctx_trim on every
    context) and empty torch's cache; returns the bytes libgis released."""
    torch = _torch()
    lib = load_library()
    total = 0
    for c in _ctxs.values():
        out = C.c_uint64()
        check(lib.gis_ctx_trim(c, C.byref(out)), "gis_ctx_trim")
        total += int(out.value)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return total


def pool_reserved() -> int:
    """Bytes reserved by the libgis context pools."""
    lib = load_library()
    total = 0
    for c in _ctxs.values():
        out = C.c_uint64()
        check(lib.gis_ctx_pool_reserved(c, C.byref(out)), "gis_ctx_pool_reserved")
        total += int(out.value)
    return total


PHASES = ("enclose", "csr_rows", "csr_aux", "prune", "index", "cover")


def enable_timing(on: bool = True):
    check(load_library().gis_ctx_enable_timing(ctx(), int(on)))


def phase_times():
    """{phase: (ms, launches)} accumulated since the last call."""
    ms = (C.c_double * len(PHASES))()
    cnt = (C.c_int64 * len(PHASES))()
    check(load_library().gis_ctx_phase_times(ctx(), ms, cnt))
    return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(PHASES)}


def integrations():
    """(images, integrations) of K1 since the last call: (cell, input, sample)
    images produced, and one-step integrations actually run (shared grid
    corners are integrated once)."""
    a, b = C.c_int64(), C.c_int64()
    check(load_library().gis_ctx_integrations(ctx(), C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def fp64_peak_tflops() -> float:
    out = C.c_double()
    check(load_library().gis_fp64_peak(ctx(), C.byref(out)))
    return float(out.value)


def ptr(t):
    """Raw device address of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return vp(t.data_ptr())


def host_f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(p_f64)


def to_host_i64(t):
    """Device integer tensor -> numpy int64, widened on the device and copied
    through pinned memory (the numpy array keeps the pinned buffer alive): a
    pageable copy of a 1e8-edge CSR costs several times more."""
    torch = _torch()
    if t.numel() == 0:
        return np.zeros(tuple(t.shape), dtype=np.int64)
    t64 = t.to(torch.int64)
    h = torch.empty(tuple(t64.shape), dtype=torch.int64, pin_memory=True)
    h.copy_(t64, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def empty(shape, dtype):
    torch = _torch()
    return torch.empty(shape, dtype=dtype, device=device())


def to_dev(a, dtype=None):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        # pinned host tensors copy asynchronously (stream-ordered; torch keeps
        # the pinned block alive until the copy has run)
        t = a.to(device(), non_blocking=a.device.type == "cpu" and a.is_pinned())
        return t if dtype is None else t.to(dtype)
    return torch.as_tensor(np.ascontiguousarray(a), device=device(), dtype=dtype)


# ----------------------------------------------------------------- models --

def encode_model(step, integrator=None) -> GisModel:
    """gis_model for a DeviceStep (system.py); refuses arbitrary callables."""
    from .system import INTEGRATOR_IDS, KIND_IDS, DeviceStep

    if not isinstance(step, DeviceStep):
        raise TypeError(
            f"step {step!r} is not a device model: the GPU path evaluates only the model "
            "descriptors in paper_2202_06111_b200.system (no CPU fallback for Python callables)")
    m = GisModel()
    m.kind = KIND_IDS[step.kind]
    if step.kind == "jit":
        m.jit = jit_id(step)
    m.integrator = INTEGRATOR_IDS[integrator or step.integrator]
    m.substeps = int(step.substeps)
    m.n = int(step.n)
    m.m = int(step.m)
    m.h = float(step.h)
    pv = [float(v) for v in step.param_vector()]
    if len(pv) > MAX_PARAMS:
        raise ValueError("too many model parameters")
    for i, v in enumerate(pv):
        m.params[i] = v
    return m


_jit_ids: dict = {}


def jit_id(step) -> int:
    """libgis id of a CudaStep's compiled kernels (NVRTC, once per model)."""
    key = (step.body, step.form, step.n, step.m, step.integrator)
    if key not in _jit_ids:
        from .system import INTEGRATOR_IDS

        out = C.c_int32()
        check(load_library().gis_jit_register(
            ctx(), step.body.encode(), 0 if step.form == "ode" else 1, step.n, step.m,
            INTEGRATOR_IDS[step.integrator], C.byref(out)), "user model")
        _jit_ids[key] = int(out.value)
    return _jit_ids[key]


def map_points_numpy(step, pts, u, rhs_only=False):
    """Evaluate step (or its vector field) on (N, n) host points."""
    torch = _torch()
    lib = load_library()
    pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64))
    model = encode_model(step, "rhs" if rhs_only else None)
    uu, up = host_f64(np.asarray(u, dtype=np.float64).reshape(-1))
    if len(uu) != step.m:
        raise ValueError(f"input has {len(uu)} components, model expects {step.m}")
    x = to_dev(pts)
    out = torch.empty_like(x)
    c = ctx()
    check(lib.gis_map_points(c, C.byref(model), ptr(x), len(pts), up, ptr(out)), "map_points")
    return out.cpu().numpy()
