"""Build libgis.so (sm_100a) in-tree with nvcc.

Usage: python -m paper_2202_06111_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
INCLUDE = HERE.parent / "include"
OBJ = HERE / "build_obj"
LIB = HERE / "libgis.so"
SOURCES = ["gis_common.cu", "gis_image.cu", "gis_index.cu", "gis_graph.cu",
           "gis_prune.cu", "gis_cover.cu", "gis_scc.cu",
           "gis_format.cu", "gis_cand.cu"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# -fmad=false: every fp64 + - * / is a separately rounded IEEE operation, in
# source order, so the integrator reproduces the reference's numpy
# arithmetic.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", f"-I{INCLUDE}"]


def _deps():
    return [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [INCLUDE / "gis.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def _compile(src: str, obj_dir: Path = OBJ, defines=()) -> tuple[str, str]:
    obj = obj_dir / (Path(src).stem + ".o")
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", str(CSRC / src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return str(obj), r.stderr


def build(force: bool = False, verbose: bool = False, variant: str = "",
          defines=()) -> Path:
    """Build libgis.so; with ``variant``, an experimental build (extra -D
    ``defines``) into build_obj/var_<variant>/ for GIS_LIB_VARIANT=<variant>."""
    lib = LIB
    obj_dir = OBJ
    if variant:
        obj_dir = OBJ / f"var_{variant}"
        lib = obj_dir / "libgis.so"
    elif not force and up_to_date():
        return LIB
    obj_dir.mkdir(parents=True, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, obj_dir, defines), SOURCES))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *objs,
           "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var,
                defines=defs))
