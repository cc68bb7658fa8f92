"""Test helpers: golden-case model lookup, state tolerance, and the
near-face explanation of edge differences (BASELINE north star: the graph
must be bit-exact except edges whose image bound lies within 1e-12 relative
of a grid face; those are listed and counted)."""

from __future__ import annotations

import numpy as np

REL = 1e-12  # north-star tolerance for integrated states and face ties


def model_for(name, spec):
    """Package SystemModel for a golden case name (see make_golden.model_cases)."""
    from paper_2202_06111_b200 import system as S
    from paper_2202_06111_b200.configs import config

    if name == "cstr":
        return S.cstr_model()
    if name == "linear":
        return S.linear_test_model(float(spec["params"]["a"]))
    if name == "affine":
        p = spec["params"]
        return S.affine_test_model(p["A"], p["B"], p["c"], X=S.Box([-5, -5], [5, 5]),
                                   U=S.Box([-1.0], [1.0]))
    if name == "identity":
        return S.identity_model()
    if name == "shift":
        return S.shift_model()
    if name.startswith("config"):
        return config(int(name[6])).model
    raise KeyError(name)


def model_from_spec(spec, X, U):
    """Package model for a golden graph case (by kind + params)."""
    from paper_2202_06111_b200 import system as S

    k, p = spec["kind"], spec["params"]
    Xb, Ub = S.Box(*X), S.Box(*U)
    if k == "cstr":
        return S.cstr_model()
    if k == "linear":
        return S.SystemModel("linear", 1, 1, Xb, Ub, S.LinearStep(p["a"]))
    if k == "affine":
        return S.affine_test_model(p["A"], p["B"], p["c"], X=Xb, U=Ub)
    if k == "identity":
        return S.SystemModel("identity", 1, 1, Xb, Ub, S.IdentityStep())
    if k == "shift":
        return S.SystemModel("shift", 1, 1, Xb, Ub, S.ShiftStep(p["offset"]))
    kw = dict(integrator=spec["integrator"], substeps=spec["substeps"], dt=spec["dt"])
    cls = {"pendulum": S.PendulumStep, "cstr_dimless": S.DimlessCstrStep,
           "lorenz": S.LorenzStep, "cartpole": S.CartPoleStep}[k]
    if k == "cartpole":
        st = cls(g=p["g"], mc=p["M"] - p["mp"], mp=p["mp"], l=p["l"], **kw)
    else:
        st = cls(**p, **kw)
    return S.SystemModel(k, st.n, st.m, Xb, Ub, st)


def assert_states_close(got, want, scale=None, rel=REL):
    """Same non-finite pattern; finite entries within rel * state scale."""
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    fg, fw = np.isfinite(got), np.isfinite(want)
    assert np.array_equal(fg, fw), "non-finite pattern differs"
    if scale is None:
        scale = np.max(np.abs(want[fw]), initial=1.0)
    err = np.abs(got[fg] - want[fw])
    tol = rel * np.maximum(np.abs(want[fw]), scale)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} entries beyond {rel}: max err {err.max()}"


def rows_as_sets(indptr, indices, rows):
    return {int(r): set(indices[indptr[r]:indptr[r + 1]].tolist()) for r in rows}


def explain_edge_diffs(lo, hi, step, inputs, frac, bloat, got, want, rel=REL):
    """Differing edges between two CSRs (indptr, indices) over the same cells.
    Returns (explained, unexplained) lists of (src, dst): an edge is
    explained when, for some input, the closed-box intersection decision of
    the oracle enclosure of src with cell dst hinges on a bound within rel
    of a face."""
    from oracle import gis_oracle as O

    gi, gx = got
    wi, wx = want
    V = len(gi) - 1
    diff_rows = [r for r in range(V)
                 if not np.array_equal(gx[gi[r]:gi[r + 1]], wx[wi[r]:wi[r + 1]])]
    explained, unexplained = [], []
    for r in diff_rows:
        a = set(gx[gi[r]:gi[r + 1]].tolist())
        b = set(wx[wi[r]:wi[r + 1]].tolist())
        for t in sorted(a ^ b):
            ok = False
            for u in inputs:
                el, eh, va = O.enclosures(step, lo[r:r + 1], hi[r:r + 1], u, frac, bloat)
                if not va[0]:
                    continue
                el, eh = el[0], eh[0]
                tl, th = lo[t], hi[t]
                tol = rel * np.maximum.reduce([np.abs(el), np.abs(eh), np.abs(tl), np.abs(th),
                                               np.ones_like(el)])
                loose = np.all(el - tol <= th) and np.all(tl <= eh + tol)
                tight = np.all(el + tol <= th) and np.all(tl <= eh - tol)
                if loose and not tight:
                    ok = True
                    break
            (explained if ok else unexplained).append((r, t))
    return explained, unexplained


# -- full-size digests (tests/golden/make_fullsize.py defines them) -----------

def sha256(*arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_digests(indptr, indices, keep, chunk):
    """Whole-graph and per-chunk digests in make_fullsize.py's definitions."""
    indptr = np.asarray(indptr, dtype="<i8")
    indices = np.asarray(indices, dtype="<i4")
    V = len(indptr) - 1
    chunks = []
    for a in range(0, V, chunk):
        b = min(a + chunk, V)
        chunks.append(sha256(np.diff(indptr[a:b + 1]).astype("<i8"),
                             indices[indptr[a]:indptr[b]]))
    return {"indptr_sha256": sha256(indptr), "indices_sha256": sha256(indices),
            "keep_sha256": sha256(np.asarray(keep).astype(np.uint8)), "chunks_sha256": chunks}


def load_fullsize_digests():
    import json
    from pathlib import Path

    p = Path(__file__).resolve().parent / "golden" / "fullsize_digests.json"
    return json.loads(p.read_text())
