"""CPU ORACLE for the GIS graph-construction / graph-pruning hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2202_06111_b200`` imports this
module; it is imported by ``tests/``, by ``__graft_entry__.smoke()`` (as the
checker) and by ``bench.py``'s ``cpu_baseline`` leg / ``--impl reference`` arm
(as the timed CPU reference).  It is never the thing measured as the product
and never a fallback for it.

It restates, in plain numpy, the algorithm of the reference package
``cisgraph`` 0.1.0 (``/root/reference/pkg/src/cisgraph``, abbreviated ``cg/``
below) for the path named by BASELINE.json's north star: sampled one-step
image enclosures, closed-box intersection enumeration through a blocked box
tree, CSR construction with dedupe, non-leaving pruning (Tarjan SCC +
reverse reachability), canonical-order subdivision / retention, the vertex
probe boundary selector, exact k-NN widening, the containment check and the
engine loop.  Each function cites the reference lines it follows.

Parity pinning: ``tests/golden/make_golden.py`` imports the reference itself
in the build container and records its outputs on the cases in
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against those fixtures bit for bit (integers, masks) and exactly for floats
(the same numpy operations in the same order).  The BASELINE models that the
reference registry lacks (pendulum, dimensionless CSTR, Lorenz, cart-pole)
enter the reference through its public ``SystemModel(step=callable)`` plugin
API with the step functions defined here (``make_step``).  Their operation
order is the reference contract: the CUDA integrator follows it exactly for
the CSTR fields, and with fused one-rounding updates (inside the 1e-12 state
tolerance, graphs unchanged) for pendulum, Lorenz and cart-pole (DESIGN.md
section 3).
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os

import numpy as np

MAX_DEPTH = 62  # cg/geometry.py:34


# ---------------------------------------------------------------------------
# dynamics (cg/system.py)
# ---------------------------------------------------------------------------

def rk4(rhs, x, u, h):
    """Classical RK4 with u held (cg/system.py:34-49): stages k1..k4, then
    x + (h/6)*(((k1 + 2k2) + 2k3) + k4)."""
    if h <= 0:
        raise ValueError("step size must be positive")
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        half = 0.5 * h
        k1 = rhs(x, u)
        k2 = rhs(x + half * k1, u)
        k3 = rhs(x + half * k2, u)
        k4 = rhs(x + h * k3, u)
        return x + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def _u0(u):
    return np.asarray(u, dtype=np.float64).reshape(-1)[0]


def _rhs_pendulum(p):
    a, b = float(p["a"]), float(p["b"])

    def rhs(x, u):
        x1, x2 = x[..., 0], x[..., 1]
        d2 = ((-a) * np.sin(x1) - b * x2) + _u0(u)
        return np.stack([x2, d2], axis=-1)
    return rhs


def _rhs_cstr(p):
    # cg/system.py:148-166 with the host-folded constants of CstrParameters
    qV, c_af, t_f = float(p["qV"]), float(p["c_Af"]), float(p["T_f"])
    neg_e, k0 = -float(p["E_over_R"]), float(p["k0"])
    c1, c2 = float(p["c1"]), float(p["c2"])

    def rhs(x, u):
        ca, temp = x[..., 0], x[..., 1]
        tc = _u0(u)
        rate = k0 * np.exp(neg_e / temp) * ca
        dca = qV * (c_af - ca) - rate
        dtemp = qV * (t_f - temp) + c1 * rate + c2 * (tc - temp)
        return np.stack([dca, dtemp], axis=-1)
    return rhs


def _rhs_cstr_dimless(p):
    da, gam, bb, beta = (float(p[k]) for k in ("Da", "gamma", "B", "beta"))

    def rhs(x, u):
        x1, x2 = x[..., 0], x[..., 1]
        t = (da * (1.0 - x1)) * np.exp(x2 / (1.0 + x2 / gam))
        d1 = (-x1) + t
        d2 = ((-x2) + bb * t) - beta * (x2 - _u0(u))
        return np.stack([d1, d2], axis=-1)
    return rhs


def _rhs_lorenz(p):
    sig, rho, beta = float(p["sigma"]), float(p["rho"]), float(p["beta"])

    def rhs(x, u):
        a, b, c = x[..., 0], x[..., 1], x[..., 2]
        da = sig * (b - a)
        db = (a * (rho - c) - b) + _u0(u)
        dc = a * b - beta * c
        return np.stack([da, db, dc], axis=-1)
    return rhs


def _rhs_cartpole(p):
    g, mp_, ell = float(p["g"]), float(p["mp"]), float(p["l"])
    mt, pml, four3 = float(p["M"]), float(p["pml"]), float(p["four_thirds"])

    def rhs(x, u):
        v, th, om = x[..., 1], x[..., 2], x[..., 3]
        s, c = np.sin(th), np.cos(th)
        temp = (_u0(u) + pml * (om * om) * s) / mt
        thacc = (g * s - c * temp) / (ell * (four3 - mp_ * (c * c) / mt))
        xacc = temp - pml * thacc * c / mt
        return np.stack([v, xacc, om, thacc], axis=-1)
    return rhs


def _map_linear(p):
    a = float(p["a"])  # cg/system.py:188-196
    return lambda x, u: a * np.asarray(x, dtype=np.float64) + _u0(u)


def _map_affine(p):
    A = np.asarray(p["A"], dtype=np.float64)  # cg/system.py:211-222
    B = np.asarray(p["B"], dtype=np.float64)
    c = np.asarray(p["c"], dtype=np.float64)
    return lambda x, u: (np.asarray(x, dtype=np.float64) @ A.T
                         + np.asarray(u, dtype=np.float64) @ B.T + c)


def _map_identity(p):
    return lambda x, u: np.asarray(x, dtype=np.float64)  # cg/system.py:233-235


def _map_shift(p):
    off = float(p["offset"])  # cg/system.py:247-252
    return lambda x, u: np.asarray(x, dtype=np.float64) + off


_RHS = {"pendulum": _rhs_pendulum, "cstr": _rhs_cstr,
        "cstr_dimless": _rhs_cstr_dimless, "lorenz": _rhs_lorenz,
        "cartpole": _rhs_cartpole}
_MAPS = {"linear": _map_linear, "affine": _map_affine,
         "identity": _map_identity, "shift": _map_shift}


def make_step(spec):
    """numpy ``step(x, u)`` for a model spec dict (kind, params, integrator,
    substeps, dt).  ``integrator`` is 'map' for direct maps, else 'euler'
    (x + h f) or 'rk4' (rk4 above), repeated ``substeps`` times with
    h = dt / substeps computed once in Python."""
    if callable(spec):  # a user step(x, u) (the reference's plugin API) as is
        return spec
    kind, params = spec["kind"], spec.get("params", {})
    if kind in _MAPS:
        return _MAPS[kind](params)
    rhs = _RHS[kind](params)
    sub = int(spec.get("substeps", 1))
    h = float(spec["dt"]) / sub
    integ = spec.get("integrator", "rk4")

    def step(x, u):
        x = np.asarray(x, dtype=np.float64)
        with np.errstate(over="ignore", invalid="ignore", under="ignore"):
            for _ in range(sub):
                if integ == "euler":
                    x = x + h * rhs(x, u)
                else:
                    x = rk4(rhs, x, u, h)
        return x
    return step


def input_grid(U_lo, U_hi, counts):
    """Cartesian input grid, endpoints included, duplicates dropped
    (cg/system.py:96-116)."""
    U_lo = np.atleast_1d(np.asarray(U_lo, dtype=np.float64))
    U_hi = np.atleast_1d(np.asarray(U_hi, dtype=np.float64))
    m = len(U_lo)
    counts = (int(counts),) * m if np.isscalar(counts) else tuple(int(c) for c in counts)
    if len(counts) != m or any(c < 2 for c in counts):
        raise ValueError("one count >= 2 per input dimension required")
    axes = [np.linspace(U_lo[d], U_hi[d], counts[d]) for d in range(m)]
    grids = np.meshgrid(*axes, indexing="ij")
    return np.unique(np.stack([g.ravel() for g in grids], axis=-1), axis=0)


# ---------------------------------------------------------------------------
# image enclosures (cg/image.py)
# ---------------------------------------------------------------------------

def lattice_fractions(n, spd):
    """spd^n lattice in [0,1]^n, axis 0 slowest (cg/image.py:43-48)."""
    ax = np.linspace(0.0, 1.0, spd)
    grids = np.meshgrid(*([ax] * n), indexing="ij")
    return np.stack([g.ravel() for g in grids], axis=-1)


def corner_fractions(n):
    """The 2^n vertices in ``vertices()`` order (cg/geometry.py:185-197)."""
    codes = np.arange(1 << n)
    return np.stack([((codes >> (n - 1 - d)) & 1).astype(np.float64)
                     for d in range(n)], axis=-1)


def enclosures(step, lo, hi, u, frac, bloat):
    """Per-cell enclosure of the sampled image for one input
    (cg/image.py:59-85): samples lo*(1-f)+hi*f, map, finite = all coords
    finite, valid = any finite, masked min/max, pad (0.5*bloat)*(hi-lo)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    nb, n = lo.shape
    frac = np.asarray(frac, dtype=np.float64)
    pts = lo[:, None, :] * (1.0 - frac[None]) + hi[:, None, :] * frac[None]
    with np.errstate(over="ignore", invalid="ignore", under="ignore"):
        img = np.asarray(step(pts.reshape(-1, n), np.asarray(u, dtype=np.float64)))
        img = img.reshape(pts.shape)
        ok = np.isfinite(img).all(axis=2)
        valid = ok.any(axis=1)
        elo = np.where(ok[:, :, None], img, np.inf).min(axis=1)
        ehi = np.where(ok[:, :, None], img, -np.inf).max(axis=1)
        pad = (0.5 * bloat) * (ehi - elo)
        return elo - pad, ehi + pad, valid


# ---------------------------------------------------------------------------
# blocked box tree (cg/geometry.py:416-505)
# ---------------------------------------------------------------------------

class BoxTree:
    """Fanout-F bulk-loaded box tree over boxes in the given order; each tier
    is (blocks, F, n) padded with never-matching (+inf, -inf) sentinels and
    queried by level-synchronous gather + compare (cg/geometry.py:425-505)."""

    def __init__(self, lo, hi, fanout=16):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.f = fanout
        self.tiers = []
        lo_t, hi_t = self.lo, self.hi
        while len(lo_t):
            nb = -(-len(lo_t) // fanout)
            blo = np.full((nb * fanout, lo_t.shape[1]), np.inf)
            bhi = np.full((nb * fanout, lo_t.shape[1]), -np.inf)
            blo[:len(lo_t)] = lo_t
            bhi[:len(hi_t)] = hi_t
            blo = blo.reshape(nb, fanout, -1)
            bhi = bhi.reshape(nb, fanout, -1)
            self.tiers.append((blo, bhi))
            if nb == 1:
                break
            lo_t, hi_t = blo.min(axis=1), bhi.max(axis=1)

    def query(self, qlo, qhi, chunk=1 << 18):
        """(query, box) index pairs of intersecting closed boxes, sorted by
        query then box."""
        qlo = np.atleast_2d(np.asarray(qlo, dtype=np.float64))
        qhi = np.atleast_2d(np.asarray(qhi, dtype=np.float64))
        if not self.tiers or len(qlo) == 0:
            return np.empty(0, np.int64), np.empty(0, np.int64)
        outs_q, outs_c = [], []
        for s in range(0, len(qlo), chunk):
            a, b = qlo[s:s + chunk], qhi[s:s + chunk]
            qi = np.arange(len(a), dtype=np.int64)
            node = np.zeros(len(a), dtype=np.int64)
            for blo, bhi in self.tiers[::-1]:
                glo, ghi = blo[node], bhi[node]
                hit = np.ones(glo.shape[:2], dtype=bool)
                for d in range(a.shape[1]):
                    hit &= (a[qi, d, None] <= ghi[:, :, d]) & (glo[:, :, d] <= b[qi, d, None])
                r, c = np.nonzero(hit)
                qi = qi[r]
                node = node[r] * self.f + c
            outs_q.append(qi + s)
            outs_c.append(node)
        return np.concatenate(outs_q), np.concatenate(outs_c)


# ---------------------------------------------------------------------------
# symbolic image CSR (cg/graph.py)
# ---------------------------------------------------------------------------

def csr_from_pairs(src, dst, nv):
    """Sort by (src, dst), drop duplicates, CSR (cg/graph.py:181-193)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if len(src):
        o = np.lexsort((dst, src))
        src, dst = src[o], dst[o]
        new = np.ones(len(src), dtype=bool)
        new[1:] = (src[1:] != src[:-1]) | (dst[1:] != dst[:-1])
        src, dst = src[new], dst[new]
    indptr = np.zeros(nv + 1, dtype=np.int64)
    if len(src):
        np.cumsum(np.bincount(src, minlength=nv), out=indptr[1:])
    return indptr, dst


def edges_for_range(start, end, lo, hi, tree, step, inputs, frac, bloat):
    """(src, dst) pairs for sources start:end, looping over inputs
    (cg/graph.py:196-211)."""
    srcs, dsts = [], []
    base = np.arange(start, end, dtype=np.int64)
    for u in inputs:
        elo, ehi, valid = enclosures(step, lo[start:end], hi[start:end], u, frac, bloat)
        if not valid.any():
            continue
        qi, ci = tree.query(elo[valid], ehi[valid])
        srcs.append(base[np.flatnonzero(valid)][qi])
        dsts.append(ci)
    if not srcs:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    return np.concatenate(srcs), np.concatenate(dsts)


def build_graph(lo, hi, step, inputs, frac, bloat, tree=None, batch=8192,
                sources=None):
    """Serial build in 8192-cell batches (cg/graph.py:38,214-234).  With
    ``sources=(a, b)`` only rows a:b are built (the other rows stay empty),
    which is how sampled checks and the bounded CPU baseline use it."""
    nv = len(lo)
    tree = tree if tree is not None else BoxTree(lo, hi)
    a, b = sources if sources is not None else (0, nv)
    srcs, dsts = [], []
    for s in range(a, b, batch):
        x, y = edges_for_range(s, min(s + batch, b), lo, hi, tree, step, inputs, frac, bloat)
        srcs.append(x)
        dsts.append(y)
    src = np.concatenate(srcs) if srcs else np.empty(0, np.int64)
    dst = np.concatenate(dsts) if dsts else np.empty(0, np.int64)
    return csr_from_pairs(src, dst, nv)


_POOL_STATE = None


def _pool_init(state):
    global _POOL_STATE
    _POOL_STATE = state


def _pool_task(task):
    s, e = task
    lo, hi, tree, step, inputs, frac, bloat = _POOL_STATE
    return edges_for_range(s, e, lo, hi, tree, step, inputs, frac, bloat)


def build_graph_pool(lo, hi, step, inputs, frac, bloat, workers, batch=1024,
                     tree=None):
    """Fork-pool build over contiguous batch chunks + deterministic merge
    (cg/graph.py:295-351, merge :237-270).  Must run in a process that has not
    initialised CUDA (fork)."""
    nv = len(lo)
    tree = tree if tree is not None else BoxTree(lo, hi)
    tasks = [(s, min(s + batch, nv)) for s in range(0, nv, batch)]
    state = (lo, hi, tree, step, inputs, frac, bloat)
    if workers <= 1 or len(tasks) <= 1:
        _pool_init(state)
        parts = [_pool_task(t) for t in tasks]
    else:
        chunks = max(1, math.ceil(len(tasks) / workers))
        with mp.get_context("fork").Pool(workers, initializer=_pool_init,
                                          initargs=(state,)) as pool:
            parts = pool.map(_pool_task, tasks, chunksize=chunks)
    if not parts:
        return np.zeros(nv + 1, np.int64), np.empty(0, np.int64)
    return csr_from_pairs(np.concatenate([p[0] for p in parts]),
                          np.concatenate([p[1] for p in parts]), nv)


# ---------------------------------------------------------------------------
# pruning (cg/analysis.py)
# ---------------------------------------------------------------------------

def tarjan(indptr, indices, nv):
    """Iterative Tarjan SCC (cg/analysis.py:51-106).  Returns (comp, ncomp)
    with component ids in pop order."""
    NONE = -1
    index = np.full(nv, NONE, dtype=np.int64)
    low = np.zeros(nv, dtype=np.int64)
    comp = np.full(nv, NONE, dtype=np.int64)
    onstk = np.zeros(nv, dtype=bool)
    ip = indptr.tolist() if nv < (1 << 22) else indptr
    nb = indices
    stk = []
    nxt = 0
    ncomp = 0
    for r in range(nv):
        if index[r] != NONE:
            continue
        index[r] = low[r] = nxt
        nxt += 1
        stk.append(r)
        onstk[r] = True
        work = [[r, int(ip[r])]]
        while work:
            top = work[-1]
            v, p = top
            e = ip[v + 1]
            pushed = False
            while p < e:
                w = int(nb[p])
                p += 1
                if index[w] == NONE:
                    top[1] = p
                    index[w] = low[w] = nxt
                    nxt += 1
                    stk.append(w)
                    onstk[w] = True
                    work.append([w, int(ip[w])])
                    pushed = True
                    break
                if onstk[w] and index[w] < low[v]:
                    low[v] = index[w]
            if pushed:
                continue
            work.pop()
            if low[v] == index[v]:
                while True:
                    w = stk.pop()
                    onstk[w] = False
                    comp[w] = ncomp
                    if w == v:
                        break
                ncomp += 1
            elif work:
                p0 = work[-1][0]
                if low[v] < low[p0]:
                    low[p0] = low[v]
    return comp, ncomp


def canonical_components(comp):
    """Relabel a component array so ids follow each component's smallest
    vertex (the numbering libgis K6 emits; Tarjan's ids are DFS pop order,
    cg/analysis.py:51-106).  Returns (labels int64, order) where
    order[new_id] = old_id."""
    comp = np.asarray(comp, dtype=np.int64)
    if len(comp) == 0:
        return comp.copy(), np.zeros(0, dtype=np.int64)
    ncomp = int(comp.max()) + 1
    first = np.full(ncomp, len(comp), dtype=np.int64)
    np.minimum.at(first, comp, np.arange(len(comp), dtype=np.int64))
    order = np.argsort(first, kind="stable")
    rank = np.empty(ncomp, dtype=np.int64)
    rank[order] = np.arange(ncomp, dtype=np.int64)
    return rank[comp], order


def scc(indptr, indices, nv):
    """strongly_connected_components (cg/analysis.py:109-117) in canonical
    numbering: (component_of, n_components, nontrivial)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    comp, ncomp = tarjan(indptr, indices, nv)
    labels, order = canonical_components(comp)
    sizes = np.bincount(labels, minlength=ncomp)
    src = np.repeat(np.arange(nv, dtype=np.int64), np.diff(indptr))
    loops = np.zeros(nv, dtype=bool)
    loops[src[src == indices]] = True
    nontriv = (sizes >= 2) | np.bincount(labels[loops], minlength=ncomp).astype(bool)
    return labels, ncomp, nontriv


def reverse_csr(indptr, indices, nv):
    """Transpose by lexsort on (dst, src) (cg/graph.py:125-133)."""
    src = np.repeat(np.arange(nv, dtype=np.int64), np.diff(indptr))
    dst = np.asarray(indices, dtype=np.int64)
    o = np.lexsort((src, dst))
    rptr = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(dst, minlength=nv), out=rptr[1:])
    return rptr, src[o]


def non_leaving_mask(indptr, indices, nv, strict_largest=False):
    """Vertices that can reach a cycle: seeds = nontrivial SCCs (size >= 2 or
    a self-loop), then reverse BFS (cg/analysis.py:109-161)."""
    if nv == 0:
        return np.zeros(0, dtype=bool)
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    comp, ncomp = tarjan(indptr, indices, nv)
    sizes = np.bincount(comp, minlength=ncomp)
    nontriv = sizes >= 2
    src = np.repeat(np.arange(nv, dtype=np.int64), np.diff(indptr))
    loops = np.zeros(nv, dtype=bool)
    loops[src[src == indices]] = True
    nontriv |= np.bincount(comp[loops], minlength=ncomp).astype(bool)
    if strict_largest and nontriv.any():
        sz = np.where(nontriv, sizes, 0)
        best = np.flatnonzero(sz == sz.max())
        if len(best) > 1:
            first = [int(np.flatnonzero(comp == c)[0]) for c in best]
            best = [best[int(np.argmin(first))]]
        nontriv = np.zeros_like(nontriv)
        nontriv[best[0]] = True
    seen = nontriv[comp]
    front = np.flatnonzero(seen)
    rptr, rind = reverse_csr(indptr, indices, nv)
    while len(front):
        st = rptr[front]
        cnt = rptr[front + 1] - st
        tot = int(cnt.sum())
        if tot == 0:
            break
        offs = np.repeat(np.cumsum(cnt) - cnt, cnt)
        preds = rind[np.repeat(st, cnt) + (np.arange(tot, dtype=np.int64) - offs)]
        fresh = preds[~seen[preds]]
        if len(fresh) == 0:
            break
        front = np.unique(fresh)
        seen[front] = True
    return seen


def peel_fixed_point(indptr, indices, nv):
    """Zero-out-degree peeling fixed point (tests/conftest.py:75-89), the
    semantics kernel K3 implements; equal to non_leaving_mask's default mode
    (tests/test_analysis.py:74-82, tests/test_acceptance.py:252-272)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    dst = np.asarray(indices, dtype=np.int64)
    src = np.repeat(np.arange(nv, dtype=np.int64), np.diff(indptr))
    alive = np.ones(nv, dtype=bool)
    if len(dst) == 0:
        return alive & False
    rounds = 0
    while True:
        live = alive[src] & alive[dst]
        dead = alive & (np.bincount(src[live], minlength=nv) == 0)
        if not dead.any():
            return alive
        alive &= ~dead
        rounds += 1


# ---------------------------------------------------------------------------
# coverings (cg/geometry.py:200-385)
# ---------------------------------------------------------------------------

def order_keys(depths, bits):
    """(primary, secondary) keys realising CellId path order
    (cg/geometry.py:200-203)."""
    d = np.asarray(depths).astype(np.uint64)
    return np.asarray(bits).astype(np.uint64) << (np.uint64(MAX_DEPTH + 1) - d), d


def canonical_order(depths, bits):
    p, s = order_keys(depths, bits)
    return np.lexsort((s, p))


def boxes_from_paths(root_lo, root_hi, depths, bits):
    """Replay the midpoint splits from the root (cg/geometry.py:206-224)."""
    depths = np.asarray(depths, dtype=np.int64)
    bits = np.asarray(bits, dtype=np.int64)
    n = len(root_lo)
    lo = np.tile(np.asarray(root_lo, dtype=np.float64), (len(depths), 1))
    hi = np.tile(np.asarray(root_hi, dtype=np.float64), (len(depths), 1))
    for lev in range(int(depths.max(initial=0))):
        act = np.flatnonzero(depths > lev)
        if len(act) == 0:
            break
        ax = lev % n
        mid = 0.5 * (lo[act, ax] + hi[act, ax])
        up = (bits[act] >> (depths[act] - lev - 1)) & 1
        hi[act, ax] = np.where(up == 0, mid, hi[act, ax])
        lo[act, ax] = np.where(up == 1, mid, lo[act, ax])
    return lo, hi


class Cover:
    """Canonically ordered SoA covering: depths, bits (int64), lo, hi."""

    def __init__(self, root_lo, root_hi, depths, bits, lo, hi, presorted=False):
        self.root_lo = np.asarray(root_lo, dtype=np.float64)
        self.root_hi = np.asarray(root_hi, dtype=np.float64)
        n = len(self.root_lo)
        depths = np.asarray(depths, dtype=np.int64)
        bits = np.asarray(bits, dtype=np.int64)
        lo = np.asarray(lo, dtype=np.float64).reshape(len(depths), n)
        hi = np.asarray(hi, dtype=np.float64).reshape(len(depths), n)
        if not presorted and len(depths) > 1:
            o = canonical_order(depths, bits)
            depths, bits, lo, hi = depths[o], bits[o], lo[o], hi[o]
            p, s = order_keys(depths, bits)
            if np.any((p[1:] == p[:-1]) & (s[1:] == s[:-1])):
                raise ValueError("duplicate cells in covering")
        self.depths, self.bits, self.lo, self.hi = depths, bits, lo, hi

    @classmethod
    def root(cls, lo, hi):
        return cls(lo, hi, [0], [0], [lo], [hi], presorted=True)

    def __len__(self):
        return len(self.depths)

    @property
    def n(self):
        return len(self.root_lo)

    def subdivide(self, sel=None):
        """Split selected cells at the midpoint of axis depth mod n
        (cg/geometry.py:343-372)."""
        m = np.ones(len(self), dtype=bool) if sel is None else np.asarray(sel, dtype=bool)
        if int(self.depths.max(initial=0)) + 1 > MAX_DEPTH:
            raise ValueError("maximum subdivision depth exceeded")
        s, k = np.flatnonzero(m), np.flatnonzero(~m)
        ax = self.depths[s] % self.n
        r = np.arange(len(s))
        mid = 0.5 * (self.lo[s, ax] + self.hi[s, ax])
        lo0, hi0 = self.lo[s].copy(), self.hi[s].copy()
        lo1, hi1 = self.lo[s].copy(), self.hi[s].copy()
        hi0[r, ax] = mid
        lo1[r, ax] = mid
        dc = self.depths[s] + 1
        b0 = self.bits[s] << 1
        return Cover(self.root_lo, self.root_hi,
                     np.concatenate([self.depths[k], dc, dc]),
                     np.concatenate([self.bits[k], b0, b0 | 1]),
                     np.concatenate([self.lo[k], lo0, lo1]),
                     np.concatenate([self.hi[k], hi0, hi1]))

    def retain(self, keep):
        """Stable restriction (cg/geometry.py:374-385)."""
        i = np.flatnonzero(np.asarray(keep, dtype=bool))
        return Cover(self.root_lo, self.root_hi, self.depths[i], self.bits[i],
                     self.lo[i], self.hi[i], presorted=True)

    def centers(self):
        return 0.5 * (self.lo + self.hi)

    def volumes(self):
        return np.prod(self.hi - self.lo, axis=1)

    def diameter(self):
        if len(self) == 0:
            return 0.0
        return float(np.sqrt(((self.hi - self.lo) ** 2).sum(axis=1)).max())


# ---------------------------------------------------------------------------
# adaptive selection (cg/adaptive.py) and k-NN (cg/geometry.py:519-555)
# ---------------------------------------------------------------------------

def probe_choices(n, face_points):
    """Per probe, per axis: 0 = enlarged lo, 1 = enlarged hi, 2 = centre
    (cg/adaptive.py:61-90)."""
    ch = [[(c >> (n - 1 - d)) & 1 for d in range(n)] for c in range(1 << n)]
    if face_points:
        for free in range(n):
            for c in range(1 << (n - 1)):
                row, k = [], 0
                for d in range(n):
                    if d == free:
                        row.append(2)
                    else:
                        row.append((c >> (n - 2 - k)) & 1)
                        k += 1
                ch.append(row)
    return np.asarray(ch, dtype=np.int64)


def probe_points(lo, hi, delta, face_points):
    hw = 0.5 * (hi - lo)
    srcs = (lo - delta * hw, hi + delta * hw, 0.5 * (lo + hi))
    ch = probe_choices(lo.shape[1], face_points)
    out = np.empty((lo.shape[0], len(ch), lo.shape[1]))
    for j, row in enumerate(ch):
        for d, which in enumerate(row):
            out[:, j, d] = srcs[which][:, d]
    return out


def select_boundary_mask(lo, hi, tree, delta, face_points=False):
    """Boundary iff some enlarged-box probe lies in no closed cell
    (cg/adaptive.py:93-123)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    nc, n = lo.shape
    if nc == 0:
        return np.zeros(0, dtype=bool)
    pr = probe_points(lo, hi, delta, face_points)
    npb = pr.shape[1]
    hw = 0.5 * (hi - lo)
    qi, ci = tree.query(lo - delta * hw, hi + delta * hw)
    cov = np.zeros(nc * npb, dtype=bool)
    for s in range(0, len(qi), 1 << 18):
        q, c = qi[s:s + (1 << 18)], ci[s:s + (1 << 18)]
        pb = pr[q]
        ins = np.ones(pb.shape[:2], dtype=bool)
        for d in range(n):
            ins &= (pb[:, :, d] >= tree.lo[c, d, None]) & (pb[:, :, d] <= tree.hi[c, d, None])
        r, cc = np.nonzero(ins)
        cov[q[r] * npb + cc] = True
    return ~cov.reshape(nc, npb).all(axis=1)


def knn(centers, points, k, exclude_point=True):
    """Exact k nearest centres by (distance, index), excluding a centre equal
    to the query (cg/geometry.py:529-555); candidates from a cKDTree ball as
    in the reference, then the exact lexsort."""
    from scipy.spatial import cKDTree

    centers = np.asarray(centers, dtype=np.float64)
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    nc = len(centers)
    if nc == 0 or k == 0:
        return [(np.empty(0, np.int64), k > 0 and nc == 0) for _ in pts]
    tree = cKDTree(centers)
    kq = min(nc, k + 2)
    dq, _ = tree.query(pts, k=kq)
    dq = np.asarray(dq, dtype=np.float64).reshape(len(pts), kq)
    balls = tree.query_ball_point(pts, dq[:, -1] * (1.0 + 1e-9) + 1e-300)
    out = []
    for p, cand in zip(pts, balls):
        cand = np.arange(nc, dtype=np.int64) if kq == nc else np.sort(np.asarray(cand, dtype=np.int64))
        diff = centers[cand] - p
        d = np.sqrt((diff ** 2).sum(axis=1))
        if exclude_point:
            keep = ~np.all(centers[cand] == p, axis=1)
            cand, d = cand[keep], d[keep]
        o = np.lexsort((cand, d))
        out.append((cand[o][:min(k, len(cand))], k > len(cand)))
    return out


def select_neighborhood_mask(lo, hi, boundary, k):
    """Union of k-NN of boundary centres minus the boundary
    (cg/adaptive.py:136-150)."""
    boundary = np.asarray(boundary, dtype=bool)
    out = np.zeros(len(boundary), dtype=bool)
    if k == 0 or not boundary.any():
        return out
    c = 0.5 * (np.asarray(lo) + np.asarray(hi))
    for idx, _ in knn(c, c[boundary], k):
        out[idx] = True
    return out & ~boundary


# ---------------------------------------------------------------------------
# engine (cg/engine.py)
# ---------------------------------------------------------------------------

def extended_root(X_lo, X_hi, shape):
    """Root box whose 2^k_d dyadic grid has its first G_d cells per axis
    tiling X (hi' = lo + ((hi - lo) * 2^k) / G); the non-dyadic initial grid
    definition of paper_2202_06111_b200.geometry.extended_root."""
    n = len(X_lo)
    k = [max(0, (int(g) - 1).bit_length()) for g in shape]
    depth = sum(k)
    if any((depth + n - 1 - d) // n != k[d] for d in range(n)):
        raise ValueError("grid not reachable by cycled bisection")
    hi = np.array([X_lo[d] + ((X_hi[d] - X_lo[d]) * float(1 << k[d])) / int(shape[d])
                   for d in range(n)])
    return np.asarray(X_lo, dtype=np.float64), hi, depth


def grid_mask(depths, bits, n, shape):
    """Cells of a uniform dyadic grid whose per-axis index is < shape[d]."""
    depths = np.asarray(depths, dtype=np.int64)
    bits = np.asarray(bits, dtype=np.int64)
    idx = np.zeros((len(depths), n), dtype=np.int64)
    for lev in range(int(depths.max(initial=0))):
        act = depths > lev
        ax = lev % n
        bit = (bits >> np.maximum(depths - lev - 1, 0)) & 1
        idx[act, ax] = (idx[act, ax] << 1) | bit[act]
    return np.all(idx < np.asarray(shape, dtype=np.int64)[None, :], axis=1)


def containment_defect(new, prev_tree):
    """Max uncovered relative volume of new cells w.r.t. the previous
    covering (cg/engine.py:114-130)."""
    if len(new) == 0:
        return 0.0
    qi, ci = prev_tree.query(new.lo, new.hi)
    inter = np.prod(np.maximum(0.0, np.minimum(new.hi[qi], prev_tree.hi[ci])
                               - np.maximum(new.lo[qi], prev_tree.lo[ci])), axis=1)
    got = np.bincount(qi, weights=inter, minlength=len(new))
    return float(np.max(1.0 - got / new.volumes()))


def run(spec, X_lo, X_hi, U_lo, U_hi, input_counts, iterations, frac, bloat,
        mode="full", n_neighbors=3, delta=0.01, face_points=False,
        initial_depth=None, workers=1, batch=1024, check_containment=True,
        keep_graphs=False, prune="tarjan", min_diameter=None, initial_grid=None):
    """The subdivide -> build -> prune -> retain loop (cg/engine.py:133-215).
    ``initial_depth`` (BASELINE 'initial grid') replaces iteration 1's
    n root splits; None keeps the reference behaviour (n splits).
    ``initial_grid`` = (G_0, ..): a non-dyadic initial grid embedded in an
    extended root (``extended_root``)."""
    step = make_step(spec)
    inputs = input_grid(U_lo, U_hi, input_counts)
    if initial_grid is not None:
        r_lo, r_hi, initial_depth = extended_root(np.asarray(X_lo, float),
                                                  np.asarray(X_hi, float), initial_grid)
        cov = Cover.root(r_lo, r_hi)
    else:
        cov = Cover.root(np.asarray(X_lo, float), np.asarray(X_hi, float))
    metrics, graphs = [], []
    ok = True
    term = "iterations"
    for k in range(1, iterations + 1):
        pre = BoxTree(cov.lo, cov.hi)
        bnd = select_boundary_mask(cov.lo, cov.hi, pre, delta, face_points)
        if k == 1:
            for _ in range(cov.n if initial_depth is None else initial_depth):
                cov = cov.subdivide(None)
            if initial_grid is not None:
                cov = cov.retain(grid_mask(cov.depths, cov.bits, cov.n, initial_grid))
        elif mode == "full":
            cov = cov.subdivide(None)
        else:
            sel = bnd | select_neighborhood_mask(cov.lo, cov.hi, bnd, n_neighbors)
            cov = cov.subdivide(sel)
        before = len(cov)
        if workers > 1:
            indptr, indices = build_graph_pool(cov.lo, cov.hi, step, inputs, frac,
                                               bloat, workers, batch)
        else:
            indptr, indices = build_graph(cov.lo, cov.hi, step, inputs, frac, bloat)
        if prune == "tarjan":
            keep = non_leaving_mask(indptr, indices, before)
        else:
            keep = peel_fixed_point(indptr, indices, before)
        new = cov.retain(keep)
        if check_containment and containment_defect(new, pre) > 1e-12:
            ok = False
        if keep_graphs:
            graphs.append((cov, indptr, indices, keep))
        metrics.append(dict(iteration=k, cells_before=before, cells_after=len(new),
                            edges=len(indices), boundary_cells=int(bnd.sum()),
                            diameter=new.diameter()))
        cov = new
        if len(cov) == 0:
            term = "empty"
            break
        if min_diameter is not None and cov.diameter() <= min_diameter:
            term = "min_diameter"
            break
    return dict(cover=cov, metrics=metrics, termination=term,
                containment_ok=ok, graphs=graphs, inputs=inputs)


def worker_count():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
