"""The C-ABI library: builds for sm_100a, loads without a GPU, and exports
every entry point include/gis.h declares (no compute calls here)."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2202_06111_b200 import _device as D
    from paper_2202_06111_b200.build import build

    build()  # no-op when libgis.so is up to date
    return D.load_library()


def declared_functions():
    text = (ROOT / "include" / "gis.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gis_\w+)\s*\(", text)))


def test_header_declares_the_path(lib):
    names = declared_functions()
    for must in ("gis_batch_enclosures", "gis_build_graph_begin", "gis_csr_finish", "gis_prune",
                 "gis_peel_sweep", "gis_subdivide", "gis_retain", "gis_select_boundary",
                 "gis_select_neighborhood", "gis_knn", "gis_index_build_dyadic",
                 "gis_query_boxes_begin", "gis_containment_defect"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2202_06111_b200 import _device as D

    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in D.SIGNATURES, name


def test_abi_version_and_no_device_error(lib):
    assert lib.gis_abi_version() == 1
    import torch

    if not torch.cuda.is_available():
        h = C.c_void_p()
        rc = lib.gis_ctx_create(C.byref(h), 0)
        assert rc != 0 and lib.gis_last_error()


def test_library_is_sm100a(lib):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(ROOT / "paper_2202_06111_b200" / "libgis.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_enum_values_match_python(lib):
    from paper_2202_06111_b200.system import INTEGRATOR_IDS, KIND_IDS

    text = (ROOT / "include" / "gis.h").read_text()
    for name, v in KIND_IDS.items():
        assert re.search(rf"GIS_{name.upper()}\s*=\s*{v}\b", text), name
    for name, v in INTEGRATOR_IDS.items():
        assert re.search(rf"GIS_{name.upper()}\s*=\s*{v}\b", text), name


def test_null_context_is_rejected_without_touching_the_device(lib):
    """Every entry point taking a gis_ctx* answers GIS_E_INVALID ("null
    context") for a null context before any CUDA call, so this runs on CPU."""
    from paper_2202_06111_b200 import _device as D

    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "gis.h").read_text(), flags=re.S)
    takes_ctx = sorted(set(re.findall(r"\b(gis_\w+)\s*\(\s*gis_ctx\s*\*\s*ctx\b", text)))
    skip = {"gis_ctx_destroy",   # null is a documented no-op
            "gis_ctx_launch_count"}  # returns a count, 0 for null
    checked = 0
    for name in takes_ctx:
        if name in skip:
            continue
        _, argtypes = D.SIGNATURES[name]
        args = [0 if t in (C.c_int, C.c_int32, C.c_int64, C.c_uint32, C.c_double) else None
                for t in argtypes]
        rc = getattr(lib, name)(*args)
        assert rc == 1, f"{name} returned {rc}"
        assert b"null context" in lib.gis_last_error(), name
        checked += 1
    assert checked >= 35


def test_user_model_compiles_without_a_gpu():
    """gis_jit_compile_check: NVRTC compiles a user field into the K1 kernels
    for sm_100a on the CPU host; a broken field returns the compiler log."""
    import ctypes as C

    from paper_2202_06111_b200 import _device as D

    lib = D.load_library()
    n = C.c_int64()
    ok = lib.gis_jit_compile_check(
        b"f[0] = x[1]; f[1] = ((-p[0]) * sin(x[0]) - p[1] * x[1]) + u[0];", 0, 2, 1, 2,
        C.byref(n))
    assert ok == 0 and n.value > 10000
    assert lib.gis_jit_compile_check(b"y[0] = 2.0 * x[0] + u[0];", 1, 1, 1, 0, C.byref(n)) == 0
    bad = lib.gis_jit_compile_check(b"f[0] = x[0] +;", 0, 1, 1, 1, C.byref(n))
    assert bad == 1
    assert "user_field(1): error" in lib.gis_last_error().decode()
    assert lib.gis_jit_compile_check(b"f[0] = 1;", 0, 1, 1, 0, C.byref(n)) == 1  # ODE + MAP
