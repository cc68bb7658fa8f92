"""Symbolic image on the GPU (mirror of cg/graph.py).

``build_graph_serial`` / ``build_graph_parallel`` run libgis K1 (integrate +
enclose + slot rectangle) and K2 (per-row gather, warp sort, dedupe, CSR)
over the covering's rows; the CSR stays on the device (indptr int64,
indices int32) and is exposed as numpy int64 arrays on demand, matching the
reference's ``SymbolicImage`` (cg/graph.py:65-169).  ``BuildPlan.workers``
counts GPUs (one process each, see ``distributed``); ``batch_size`` is kept
for API compatibility -- the device build is plan-independent by
construction, as the reference's is (cg/graph.py:1-10).
"""

from __future__ import annotations

import ctypes as C
import io
from dataclasses import dataclass
from typing import IO

import numpy as np

from . import _device as D
from ._device import GraphBuildError
from .geometry import CellId, Covering, SpatialIndex
from .image import ImageConfig, sample_fractions

__all__ = ["SymbolicImage", "BuildPlan", "GraphBuildError", "OwnershipError",
           "build_graph_serial", "build_graph_parallel", "build_graph_rows", "merge_subgraphs",
           "out_degree", "write_edge_list"]


class OwnershipError(ValueError):
    """Subgraphs passed to merge claim overlapping source vertices
    (cg/graph.py:45-46)."""


@dataclass(frozen=True)
class BuildPlan:
    batch_size: int = 1024
    workers: int = 1

    def __post_init__(self):
        if self.batch_size < 1 or self.workers < 1:
            raise ValueError("batch_size and workers must be at least 1")


class SymbolicImage:
    """CSR digraph over covering cells in canonical order; ascending unique
    targets per row.  Device-resident (``indptr_dev`` int64, ``indices_dev``
    int32); ``indptr``/``indices`` are numpy int64 views."""

    def __init__(self, vertex_depths, vertex_bits, indptr, indices, owned=None):
        torch = D._torch()
        self._cov = None
        self._vd = np.asarray(vertex_depths, dtype=np.int64)
        self._vb = np.asarray(vertex_bits, dtype=np.int64)
        if isinstance(indptr, torch.Tensor):
            self.indptr_dev = indptr.to(torch.int64)
            self.indices_dev = indices.to(torch.int32)
            self._np = {}
        else:
            self._np = {"indptr": np.asarray(indptr, dtype=np.int64),
                        "indices": np.asarray(indices, dtype=np.int64)}
            self.indptr_dev = None
            self.indices_dev = None
        self.owned = None if owned is None else np.asarray(owned, dtype=np.int64)
        self._id_map = None
        self._rev = None

    @classmethod
    def _from_device(cls, covering: Covering, indptr_dev, indices_dev) -> "SymbolicImage":
        g = cls.__new__(cls)
        g._cov = covering
        g._vd = g._vb = None
        g.indptr_dev, g.indices_dev = indptr_dev, indices_dev
        g._np = {}
        g.owned = None
        g._id_map = None
        g._rev = None
        return g

    def _dev(self):
        if self.indptr_dev is None:
            torch = D._torch()
            self.indptr_dev = D.to_dev(self._np["indptr"])
            self.indices_dev = D.to_dev(self._np["indices"].astype(np.int32))
        return self.indptr_dev, self.indices_dev

    def _host(self, key):
        if key not in self._np:
            t = self.indptr_dev if key == "indptr" else self.indices_dev
            self._np[key] = D.to_host_i64(t)
        return self._np[key]

    @property
    def indptr(self) -> np.ndarray:
        return self._host("indptr")

    @property
    def indices(self) -> np.ndarray:
        return self._host("indices")

    @property
    def vertex_depths(self) -> np.ndarray:
        return self._cov.depths if self._vd is None else self._vd

    @property
    def vertex_bits(self) -> np.ndarray:
        return self._cov.bits if self._vb is None else self._vb

    @property
    def n_vertices(self) -> int:
        if self.indptr_dev is not None:
            return int(self.indptr_dev.shape[0]) - 1
        return len(self._np["indptr"]) - 1

    @property
    def edge_count(self) -> int:
        if self.indices_dev is not None:
            return int(self.indices_dev.shape[0])
        return len(self._np["indices"])

    def vertex_id(self, i: int) -> CellId:
        return CellId(int(self.vertex_depths[i]), int(self.vertex_bits[i]))

    def vertex_ids(self) -> list:
        return [self.vertex_id(i) for i in range(self.n_vertices)]

    def _vertex_index(self, v) -> int:
        if isinstance(v, (int, np.integer)):
            if not 0 <= v < self.n_vertices:
                raise KeyError(f"vertex index {v} out of range")
            return int(v)
        if self._id_map is None:
            self._id_map = {(int(d), int(b)): i
                            for i, (d, b) in enumerate(zip(self.vertex_depths, self.vertex_bits))}
        try:
            return self._id_map[(v.depth, v.bits)]
        except (KeyError, AttributeError):
            raise KeyError(f"unknown vertex {v!r}") from None

    def out_degree(self, v) -> int:
        i = self._vertex_index(v)
        return int(self.indptr[i + 1] - self.indptr[i])

    def successors(self, v) -> list:
        i = self._vertex_index(v)
        return [self.vertex_id(j) for j in self.indices[self.indptr[i]:self.indptr[i + 1]]]

    def edge_pairs(self):
        """(src, dst) numpy int64 arrays in CSR order (cg/graph.py:119-123);
        sources expanded on the GPU (libgis gis_csr_sources)."""
        torch = D._torch()
        nv = self.n_vertices
        src = torch.empty(self.edge_count, dtype=torch.int64, device=D.device())
        if nv and self.edge_count:
            ip, _ = self._dev()
            D.check(D.load_library().gis_csr_sources(D.ctx(), D.ptr(ip), nv, D.ptr(src)),
                    "edge_pairs")
        return D.to_host_i64(src), self.indices

    def reverse_csr(self):
        """Transposed CSR (rptr, rind) with ascending rows, as the reference's
        lexsort leaves them (cg/graph.py:125-133); libgis gis_reverse_csr."""
        if self._rev is None:
            torch = D._torch()
            nv = self.n_vertices
            indptr, indices = self._dev()
            rptr = torch.zeros(nv + 1, dtype=torch.int64, device=D.device())
            rind = torch.empty(self.edge_count, dtype=torch.int32, device=D.device())
            if nv:
                D.check(D.load_library().gis_reverse_csr(D.ctx(), D.ptr(indptr), D.ptr(indices),
                                                         nv, D.ptr(rptr), D.ptr(rind), 1),
                        "reverse_csr")
            self._rev = (D.to_host_i64(rptr), D.to_host_i64(rind))
        return self._rev

    def self_loop_mask(self) -> np.ndarray:
        """Vertices with an edge to themselves (cg/graph.py:135-139)."""
        torch = D._torch()
        nv = self.n_vertices
        out = torch.zeros(nv, dtype=torch.uint8, device=D.device())
        if nv:
            indptr, indices = self._dev()
            D.check(D.load_library().gis_self_loops(D.ctx(), D.ptr(indptr), D.ptr(indices), nv,
                                                    D.ptr(out)), "self_loop_mask")
        return out.cpu().numpy().view(bool)

    def _paths(self) -> list:
        return [format(int(b), f"0{int(d)}b") if d else "-"
                for d, b in zip(self.vertex_depths, self.vertex_bits)]

    def _dev_ids(self):
        """(depths int32, bits int64) device arrays of the vertices."""
        if self._cov is not None:
            return self._cov._d, self._cov._b
        torch = D._torch()
        return (D.to_dev(self._vd.astype(np.int32)), D.to_dev(self._vb.astype(np.int64)))

    def _edge_list_chunks(self, chunk_bytes: int = 256 << 20):
        """The edge list as successive byte chunks (memoryviews), formatted on
        the GPU (libgis gis_format_edges) and copied out through pinned memory."""
        torch = D._torch()
        nv = self.n_vertices
        if nv == 0 or self.edge_count == 0:
            return
        lib = D.load_library()
        dep, bits = self._dev_ids()
        indptr, indices = self._dev()
        off = torch.empty(nv + 1, dtype=torch.int64, device=D.device())
        D.check(lib.gis_edge_list_offsets(D.ctx(), D.ptr(dep), D.ptr(indptr), D.ptr(indices), nv,
                                          D.ptr(off)), "edge_list")
        off_h = off.cpu().numpy()
        cap = int(min(off_h[-1], chunk_bytes))
        buf = torch.empty(max(cap, 1), dtype=torch.uint8, device=D.device())
        host = torch.empty(max(cap, 1), dtype=torch.uint8, pin_memory=True)
        r = 0
        while r < nv:
            r2 = int(np.searchsorted(off_h, off_h[r] + cap, side="right")) - 1
            r2 = min(max(r2, r + 1), nv)
            nb = int(off_h[r2] - off_h[r])
            if nb > buf.numel():  # a single row larger than the chunk
                buf = torch.empty(nb, dtype=torch.uint8, device=D.device())
                host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
            if nb:
                D.check(lib.gis_format_edges(D.ctx(), D.ptr(dep), D.ptr(bits), D.ptr(indptr),
                                             D.ptr(indices), nv, D.ptr(off), r, r2, D.ptr(buf)),
                        "edge_list")
                host[:nb].copy_(buf[:nb])
                yield memoryview(host.numpy())[:nb]
            r = r2

    def write_edge_list(self, fp: IO[str]) -> None:
        """'src_path dst_path' lines in CSR (canonical) order
        (cg/graph.py:147-156), formatted on the GPU."""
        raw = getattr(fp, "buffer", None)
        if raw is not None:
            fp.flush()
        for chunk in self._edge_list_chunks():
            if raw is not None:
                raw.write(chunk)
            else:
                fp.write(bytes(chunk).decode("ascii"))

    def edge_list_bytes(self) -> bytes:
        return b"".join(bytes(c) for c in self._edge_list_chunks())

    def same_edges(self, other: "SymbolicImage") -> bool:
        return (np.array_equal(self.vertex_depths, other.vertex_depths)
                and np.array_equal(self.vertex_bits, other.vertex_bits)
                and np.array_equal(self.indptr, other.indptr)
                and np.array_equal(self.indices, other.indices))


def out_degree(graph: SymbolicImage, v) -> int:
    return graph.out_degree(v)


def write_edge_list(graph: SymbolicImage, fp: IO[str]) -> None:
    graph.write_edge_list(fp)


def _inputs_array(inputs):
    return np.atleast_2d(np.asarray(getattr(inputs, "points", inputs), dtype=np.float64))


def build_graph_rows(covering: Covering, index: SpatialIndex, model, inputs,
                     cfg: ImageConfig, row_begin: int = 0, row_end=None):
    """Device CSR of rows [row_begin, row_end): (indptr int64[rows+1],
    indices int32[E]) with global target indices."""
    indptr, indices, _ = build_graph_rows_memo(covering, index, model, inputs, cfg,
                                               row_begin, row_end)
    return indptr, indices


class BoxMemo:
    """What a graph build keeps for the next covering of an adaptive run
    (gis_build_graph_memo_begin): the padded enclosure boxes [rows][U][2n]
    of the covering's cells [begin, begin + rows) and their CSR rows
    (indptr relative to begin, global targets)."""

    def __init__(self, boxes, begin: int, rows: int, indptr=None, indices=None):
        self.boxes, self.begin, self.rows = boxes, int(begin), int(rows)
        self.indptr, self.indices = indptr, indices


def build_graph_rows_memo(covering: Covering, index: SpatialIndex, model, inputs,
                          cfg: ImageConfig, row_begin: int = 0, row_end=None, origin=None,
                          memo: "BoxMemo | None" = None, keep_memo: bool = False, fwd=None):
    """build_graph_rows, optionally keeping every pair's padded box and the
    rows (keep_memo) and reusing those of an earlier build for the cells
    that `origin` (device int64 [V], Covering.origin_after) maps into it --
    the same graph, with the unchanged cells of an adaptive step not
    integrated again; with `fwd` (Covering.forward_after) their rows are
    the earlier rows mapped forward instead of enumerated again.  Returns
    (indptr, indices, BoxMemo or None)."""
    torch = D._torch()
    V = len(covering)
    row_end = V if row_end is None else int(row_end)
    rows = row_end - row_begin
    if model.n != covering.n:
        raise ValueError("model dimension does not match the covering")
    mstruct = D.encode_model(model.step)
    u = _inputs_array(inputs)
    frac = sample_fractions(cfg, covering.n)
    _, up = D.host_f64(u)
    _, fp = D.host_f64(frac)
    indptr = torch.empty(rows + 1, dtype=torch.int64, device=D.device())
    E = C.c_int64()
    lib = D.load_library()
    c = D.ctx()
    use_memo = (keep_memo or origin is not None) and not index.sparse
    out = None
    if use_memo and keep_memo:
        out = torch.empty((max(rows, 1), len(u), 2 * covering.n), dtype=torch.float64,
                          device=D.device())
    lo_t, hi_t = covering._k1_bounds()  # cell-bound copies in flight go to K1
    try:
        if use_memo:
            if origin is not None and memo is None:
                raise ValueError("origin given without the previous build's boxes")
            reuse = origin is not None
            rows_fwd = reuse and fwd is not None and memo.indptr is not None
            D.check(lib.gis_build_graph_memo_begin(
                c, index._h, C.byref(mstruct), D.ptr(lo_t), D.ptr(hi_t), V,
                int(row_begin), int(row_end), up, len(u), fp, len(frac), float(cfg.bloat),
                D.ptr(origin), D.ptr(memo.boxes) if reuse else None,
                memo.begin if reuse else 0, memo.rows if reuse else 0,
                D.ptr(memo.indptr) if rows_fwd else None,
                D.ptr(memo.indices) if rows_fwd else None, D.ptr(fwd) if rows_fwd else None,
                D.ptr(out), D.ptr(indptr), C.byref(E)), "build_graph")
        else:
            D.check(lib.gis_build_graph_begin(
                c, index._h, C.byref(mstruct), D.ptr(lo_t), D.ptr(hi_t), V,
                int(row_begin), int(row_end), up, len(u), fp, len(frac), float(cfg.bloat),
                D.ptr(indptr), C.byref(E)), "build_graph")
        indices = torch.empty(int(E.value), dtype=torch.int32, device=D.device())
        D.check(lib.gis_csr_finish(c, D.ptr(indices)), "build_graph")
    except (RuntimeError, MemoryError) as exc:
        raise GraphBuildError(
            f"graph build failed in batch 0 (cells {row_begin}:{row_end}): {exc}") from exc
    finally:
        covering._k1_done()
    return indptr, indices, (BoxMemo(out, row_begin, rows, indptr, indices)
                             if out is not None else None)


def build_graph_serial(covering: Covering, index: SpatialIndex, model, inputs,
                       cfg: ImageConfig) -> SymbolicImage:
    """Symbolic image of the whole covering (cg/graph.py:214-234)."""
    if len(covering) == 0:
        torch = D._torch()
        z = torch.zeros(1, dtype=torch.int64, device=D.device())
        e = torch.zeros(0, dtype=torch.int32, device=D.device())
        return SymbolicImage._from_device(covering, z, e)
    indptr, indices = build_graph_rows(covering, index, model, inputs, cfg)
    return SymbolicImage._from_device(covering, indptr, indices)


def build_graph_parallel(covering: Covering, index: SpatialIndex, model, inputs,
                         cfg: ImageConfig, plan: BuildPlan) -> SymbolicImage:
    """Same edge set as the serial build for every plan
    (cg/graph.py:295-351).  Inside a multi-GPU job use
    ``distributed.build_graph_sharded``."""
    return build_graph_serial(covering, index, model, inputs, cfg)


def merge_subgraphs(parts: list) -> SymbolicImage:
    """Union of subgraphs with disjoint source ownership (cg/graph.py:237-270).
    Ownership is validated on the host (it is per-vertex metadata); the edge
    union -- every part's (src, dst) pairs, sorted and deduplicated into one
    CSR -- runs on the GPU (libgis gis_csr_sources + gis_csr_from_pairs)."""
    if not parts:
        raise ValueError("merge requires at least one subgraph")
    torch = D._torch()
    first = parts[0]
    owned_sets = []
    for p in parts:
        if not (np.array_equal(p.vertex_depths, first.vertex_depths)
                and np.array_equal(p.vertex_bits, first.vertex_bits)):
            raise ValueError("subgraphs are over different coverings")
        if p.owned is not None:
            owned_sets.append(np.asarray(p.owned, dtype=np.int64))
        else:  # sources that have edges
            owned_sets.append(np.flatnonzero(np.diff(p.indptr) > 0))
    cat = np.concatenate(owned_sets) if owned_sets else np.empty(0, dtype=np.int64)
    if len(np.unique(cat)) != len(cat):
        raise OwnershipError("overlapping source ownership between subgraphs")
    nv = first.n_vertices
    lib = D.load_library()
    srcs, dsts = [], []
    for p in parts:
        ip, ix = p._dev()
        src = torch.empty(p.edge_count, dtype=torch.int64, device=D.device())
        if nv and p.edge_count:
            D.check(lib.gis_csr_sources(D.ctx(), D.ptr(ip), nv, D.ptr(src)), "merge_subgraphs")
        srcs.append(src)
        dsts.append(ix.to(torch.int64))
    src = torch.cat(srcs) if srcs else torch.empty(0, dtype=torch.int64, device=D.device())
    dst = torch.cat(dsts) if dsts else torch.empty(0, dtype=torch.int64, device=D.device())
    indptr = torch.empty(nv + 1, dtype=torch.int64, device=D.device())
    indices = torch.empty(max(int(src.shape[0]), 1), dtype=torch.int32, device=D.device())
    E = C.c_int64()
    D.check(lib.gis_csr_from_pairs(D.ctx(), D.ptr(src), D.ptr(dst), int(src.shape[0]), nv,
                                   D.ptr(indptr), D.ptr(indices), C.byref(E)), "merge_subgraphs")
    return SymbolicImage(first.vertex_depths, first.vertex_bits, indptr, indices[:E.value])