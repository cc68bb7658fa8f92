"""Multi-GPU sharding of the build + prune (one process per GPU).

Cells are partitioned into contiguous CellId ranges aligned to 32-vertex
bitmap words -- the reference's contiguous ownership model
(cg/graph.py:306-345, merge_subgraphs ownership :237-270).  The covering is
replicated; each rank integrates and builds the CSR rows it owns (targets
are global indices, so rows need no exchange).  Pruning runs the forward
peeling sweep on owned rows, the ranks exchange the vertex bitmap (each
rank contributes its owned words) and sum the deletions after every sweep;
the loop ends when a sweep deletes nothing anywhere.

The default exchange is the north star's NCCL all-gather of the owned
bitmap words (``sharded_peel``; the same protocol the CPU tests run with
gloo, tests/test_distributed.py), once per round of local sweeps: each rank
first runs its owned rows to their local fixed point in one cooperative
kernel, so a round costs one all-gather where the per-sweep form paid one per
sweep.  The
fused form -- one cooperative kernel per rank (libgis ``gis_peel_p2p``) that
stores its owned words into every peer's bitmap replica over NVLink (CUDA IPC
mappings, ``PeerBitmaps``) and meets the other ranks at a flag barrier in
peer memory every sweep -- is opt-in (GIS_PEEL_EXCHANGE=p2p) until it has
run across real GPUs (tests/test_gpu_multirank.py has the 2-GPU check,
skipped on one GPU).  It is used only when every rank is on one node and
every pair of GPUs has peer access; if mapping the peers' buffers fails on
any rank, all ranks fall back to the NCCL form together.
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _device as D

__all__ = ["word_partition", "owned_range", "sharded_peel", "fused_peel", "PeerBitmaps",
           "PeerMappingError", "exchange_mode", "gather_rows",
           "emulated_fused_peel", "release_peer_bitmaps", "build_and_prune_sharded",
           "sharded_boundary", "sharded_neighborhood", "sharded_containment", "world"]


def world():
    """(rank, world_size) of the default process group, (0, 1) without one."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def _staged(group) -> bool:
    """Collectives of a non-NCCL group (gloo) run on host copies of device
    tensors: the CPU tests, and several ranks sharing one GPU in the tests
    of the multi-rank engine (no kernel of one rank waits on another's)."""
    import torch.distributed as dist

    return dist.get_backend(group) != "nccl"


def all_reduce_(t, op=None, group=None):
    """In-place all-reduce of a tensor on any device."""
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if not _staged(group) or t.device.type == "cpu":
        dist.all_reduce(t, op=op, group=group)
        return
    h = t.cpu()
    dist.all_reduce(h, op=op, group=group)
    t.copy_(h)


def all_gather_(t, group=None) -> list:
    """Every rank's copy of a same-shaped tensor, on t's device."""
    import torch
    import torch.distributed as dist

    _, size = world()
    if not _staged(group) or t.device.type == "cpu":
        parts = [torch.empty_like(t) for _ in range(size)]
        dist.all_gather(parts, t, group=group)
        return parts
    h = t.cpu()
    parts = [torch.empty_like(h) for _ in range(size)]
    dist.all_gather(parts, h, group=group)
    return [p.to(t.device) for p in parts]


def word_partition(V: int, size: int) -> int:
    """Bitmap words per rank (equal slices for the all-gather)."""
    nwords = (V + 31) // 32
    return max(1, -(-nwords // size))


def owned_range(V: int, rank: int, size: int):
    """[begin, end) vertices owned by rank: word-aligned contiguous ranges."""
    W = word_partition(V, size)
    b = min(V, rank * W * 32)
    e = min(V, (rank + 1) * W * 32)
    return b, e


def _allgather_words(full, W, rank, size, group=None):
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        # in place: NCCL accepts the input as the rank's slice of the output
        dist.all_gather_into_tensor(full, full[rank * W:(rank + 1) * W], group=group)
    else:
        parts = all_gather_(full[rank * W:(rank + 1) * W].clone(), group)
        full.copy_(torch.cat(parts))


def _device_sweep(indptr_local, indices, b, e, alive_words, ptr):
    deaths = C.c_int64()
    D.check(D.load_library().gis_peel_sweep(D.ctx(), D.ptr(indptr_local), D.ptr(indices), b, e,
                                            D.ptr(alive_words), D.ptr(ptr), C.byref(deaths)),
            "peel_sweep")
    return int(deaths.value)


def sharded_peel(indptr_local, indices, V: int, rank: int, size: int,
                 sweep: Optional[Callable] = None, init: Optional[Callable] = None, group=None):
    """Peeling fixed point with owned rows [b, e) on this rank.

    A round is: the owned rows' LOCAL fixed point against the bitmap as it
    stands (libgis gis_peel_local: one cooperative launch of block-local
    sweeps; remote words read, never written), then the in-place all-gather
    of every rank's owned words and an all-reduce of the round's deletions,
    which the host reads to stop.  A round in which no rank deleted anything
    started every rank's first sweep from the complete bitmap: the global
    fixed point.  Rounds are exchange steps, far fewer than sweeps (most
    deletion chains run inside one rank's CellId range).

    Returns (alive_words int32 tensor of size*W words -- the global bitmap,
    rounds).  ``sweep(indptr_local, indices, b, e, alive_words, ptr) -> deaths``
    (one sweep; repeated until it deletes nothing) and
    ``init(indptr_local, V, b, e, alive_words, ptr)`` default to libgis."""
    import torch

    b, e = owned_range(V, rank, size)
    W = word_partition(V, size)
    dev = indptr_local.device
    full = torch.zeros(size * W, dtype=torch.int32, device=dev)
    ptr = torch.empty(max(e - b, 1), dtype=torch.int64, device=dev)
    if init is None:
        D.check(D.load_library().gis_peel_init(D.ctx(), D.ptr(indptr_local), V, b, e,
                                               D.ptr(full), D.ptr(ptr)), "peel_init")
    else:
        init(indptr_local, V, b, e, full, ptr)
    rounds = 0
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lib = D.load_library() if sweep is None else None
    while True:
        cnt.zero_()
        if sweep is None:  # deletions accumulate on the device
            D.check(lib.gis_peel_local(D.ctx(), D.ptr(indptr_local), D.ptr(indices), b, e,
                                       D.ptr(full), D.ptr(ptr), D.ptr(cnt)), "peel_local")
        else:
            while True:
                d = int(sweep(indptr_local, indices, b, e, full, ptr))
                cnt += d
                if d == 0:
                    break
        rounds += 1
        _allgather_words(full, W, rank, size, group)
        all_reduce_(cnt, group=group)
        if int(cnt.item()) == 0:
            return full, rounds


class PeerMappingError(RuntimeError):
    """CUDA IPC mapping of a peer's exchange buffers failed on some rank."""


class PeerBitmaps:
    """Per-rank bitmap replica and flag area in CUDA IPC memory, mapped into
    every rank of the group (the fused prune's exchange buffers).  Grown on
    demand (a collective: every rank sees the same V); ``seq`` is the flag
    sequence the next ``gis_peel_p2p`` call starts from."""

    def __init__(self, group=None):
        self.group = group
        self.rank, self.size = world()
        self.cap = 0
        self.own = []      # our allocations (freed)
        self.opened = []   # peer mappings (closed)
        self.rep_addrs = self.flag_addrs = None
        self.seq = 1

    def ensure(self, words: int):
        import torch.distributed as dist

        need = max(4 * int(words), 4)
        if need <= self.cap:
            return
        self.release()
        lib, c = D.load_library(), D.ctx()
        cap = 1 << max(12, (need - 1).bit_length())
        mine = []
        for nbytes in (cap, 2 * self.size * 8):
            p, h = C.c_void_p(), (C.c_char * 64)()
            D.check(lib.gis_ipc_alloc(c, nbytes, C.byref(p), h), "ipc_alloc")
            self.own.append(p)
            mine.append(bytes(h))
        handles = [None] * self.size
        dist.all_gather_object(handles, mine, group=self.group)
        reps, flags, err = [], [], None
        for q, (hr, hf) in enumerate(handles):
            if q == self.rank:
                reps.append(self.own[0].value)
                flags.append(self.own[1].value)
                continue
            for h, out in ((hr, reps), (hf, flags)):
                p = C.c_void_p()
                st = lib.gis_ipc_open(c, C.create_string_buffer(h, 64), C.byref(p))
                if st != 0:
                    err = err or D.last_error()
                    continue
                self.opened.append(p)
                out.append(p.value)
        self.cap = cap
        # every rank must agree: one failed mapping sends all ranks to NCCL
        bad = [err is not None]
        votes = [None] * self.size
        dist.all_gather_object(votes, bad, group=self.group)
        if any(v[0] for v in votes):
            self.release()
            raise PeerMappingError(err or "a peer rank could not map the IPC buffers")
        self.rep_addrs = (C.c_uint64 * self.size)(*reps)
        self.flag_addrs = (C.c_uint64 * self.size)(*flags)

    def release(self):
        import torch
        import torch.distributed as dist

        if not self.cap:
            return
        lib = D.load_library()
        torch.cuda.synchronize()
        live = dist.is_initialized()
        if live:
            dist.barrier(group=self.group)  # nobody still writes into our buffers
        for p in self.opened:
            lib.gis_ipc_close(p)
        if live:
            dist.barrier(group=self.group)  # nobody still maps them
        for p in self.own:
            lib.gis_ipc_free(p)
        self.own, self.opened, self.cap = [], [], 0

    def local_words(self):
        """Address of this rank's replica (the global bitmap after a prune)."""
        return C.c_void_p(self.rep_addrs[self.rank])


_PEERS = {}


def _peer_key(group):
    return (id(group), world())


def _peer_bitmaps(group=None) -> PeerBitmaps:
    key = _peer_key(group)
    if key not in _PEERS:
        _PEERS[key] = PeerBitmaps(group)
    return _PEERS[key]


def release_peer_bitmaps():
    """Free every PeerBitmaps (collective: call on all ranks, before the
    process group is destroyed)."""
    for ex in _PEERS.values():
        ex.release()
    _PEERS.clear()


def fused_peel(indptr_local, indices, V: int, group=None):
    """Multi-GPU peeling fixed point, exchange fused into the sweep kernel
    (libgis gis_peel_p2p over CUDA IPC replicas).  Returns (PeerBitmaps whose
    local replica holds the surviving vertices, sweeps).

    A host barrier precedes the launch, so the kernel's peer waits (bounded
    by its %globaltimer deadline) only cover the sweeps, never a peer's
    graph build.  A failed launch (e.g. a peer timeout) releases the
    exchange buffers: flag areas with partial posts are never reused."""
    import torch
    import torch.distributed as dist

    rank, size = world()
    b, e = owned_range(V, rank, size)
    ex = _peer_bitmaps(group)
    ex.ensure((V + 31) // 32)
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)
    rounds = C.c_int32(0)
    st = D.load_library().gis_peel_p2p(
        D.ctx(), D.ptr(indptr_local), D.ptr(indices), V, b, e - b, ex.rep_addrs, ex.flag_addrs,
        rank, size, ex.seq, C.byref(rounds))
    if st != 0:
        msg = D.last_error()
        _PEERS.pop(_peer_key(group), None)
        try:
            ex.release()
        finally:
            raise RuntimeError(f"peel_p2p: {msg}")
    ex.seq = (ex.seq + rounds.value + 1) & 0xFFFFFFFF or 1
    return ex, int(rounds.value)


def emulated_fused_peel(indptr, indices, V: int, size: int):
    """The fused protocol with `size` ranks emulated in one cooperative
    launch on this GPU (replicas and flag areas local): the test of the
    exchange logic without `size` GPUs.  Returns (list of the ranks' replica
    tensors, sweeps); every replica must end equal to the single-GPU bitmap."""
    import torch

    dev = indptr.device
    words = (V + 31) // 32
    reps = [torch.zeros(max(words, 1), dtype=torch.int32, device=dev) for _ in range(size)]
    flags = [torch.zeros(2 * size, dtype=torch.int64, device=dev) for _ in range(size)]
    ra = (C.c_uint64 * size)(*[t.data_ptr() for t in reps])
    fa = (C.c_uint64 * size)(*[t.data_ptr() for t in flags])
    rounds = C.c_int32(0)
    D.check(D.load_library().gis_peel_p2p(D.ctx(), D.ptr(indptr), D.ptr(indices), V, 0, V, ra,
                                          fa, -1, size, 1, C.byref(rounds)), "peel_p2p")
    return reps, int(rounds.value)


_FUSED_OK = {}


def exchange_mode(group=None) -> str:
    """'p2p' (fused peer-memory prune) or 'nccl' (sweep + all-gather).

    p2p needs GIS_PEEL_EXCHANGE=p2p, an NCCL group whose ranks all live on
    this node (LOCAL_WORLD_SIZE == WORLD_SIZE: CUDA IPC handles do not cross
    nodes) and peer access between every pair of this job's GPUs; every rank
    evaluates the same inputs, and the answer is agreed by an all-reduce."""
    import os

    import torch
    import torch.distributed as dist

    key = _peer_key(group)
    if key in _FUSED_OK:
        return _FUSED_OK[key]
    want = (dist.get_backend(group) == "nccl"
            and os.environ.get("GIS_PEEL_EXCHANGE", "nccl").lower() == "p2p")
    _, size = world()
    if want:
        local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", "-1"))
        want = local_ws == size
    if want:
        me = torch.cuda.current_device()
        devs = [None] * size
        dist.all_gather_object(devs, me, group=group)
        want = all(a == b or torch.cuda.can_device_access_peer(a, b)
                   for a in devs for b in devs)
    if dist.get_backend(group) == "nccl":
        flag = torch.tensor([0 if want else 1], dtype=torch.int32, device=D.device())
        dist.all_reduce(flag, group=group)
        want = int(flag.item()) == 0
    _FUSED_OK[key] = "p2p" if want else "nccl"
    return _FUSED_OK[key]


def gather_rows(indptr_local, indices, V: int, group=None):
    """All ranks' owned rows assembled into the whole device CSR on every
    rank (indptr int64[V+1], indices int32[E]): the graph a single-process
    build returns, for ``RunConfig.keep_final_graph`` in a sharded run."""
    import torch

    _, size = world()
    dev = indptr_local.device
    counts = torch.tensor([indices.shape[0]], dtype=torch.int64, device=dev)
    allc = all_gather_(counts, group)
    ec = [int(t.item()) for t in allc]
    pad = max(max(ec), 1)
    buf = torch.zeros(pad, dtype=torch.int32, device=dev)
    buf[:indices.shape[0]] = indices
    parts = all_gather_(buf, group)
    W = word_partition(V, size) * 32
    rl = torch.zeros(W + 1, dtype=torch.int64, device=dev)
    rl[:indptr_local.shape[0]] = indptr_local
    rl[indptr_local.shape[0]:] = indptr_local[-1]
    rls = all_gather_(rl, group)
    indptr = torch.zeros(V + 1, dtype=torch.int64, device=dev)
    off = 0
    for r in range(size):
        b, e = owned_range(V, r, size)
        if e > b:
            indptr[b + 1:e + 1] = rls[r][1:e - b + 1] + off
        off += ec[r]
    out = torch.cat([parts[r][:ec[r]] for r in range(size)])
    return indptr, out


def build_and_prune_sharded(covering, index, model, inputs, cfg, group=None,
                            return_graph: bool = False, memo_io=None):
    """Build owned rows and prune cooperatively; returns (keep uint8 device
    tensor over all cells, total edges, sweeps), plus the whole gathered CSR
    (indptr, indices) when ``return_graph``.  memo_io (dict, adaptive runs):
    "origin" / "memo" in -- this rank's boxes of the previous covering, see
    graph.build_graph_rows_memo -- and "keep" (bool); the owned rows' boxes
    come back in memo_io["out"]."""
    import torch

    from .graph import build_graph_rows_memo

    rank, size = world()
    V = len(covering)
    b, e = owned_range(V, rank, size)
    if memo_io is None:
        indptr, indices, _ = build_graph_rows_memo(covering, index, model, inputs, cfg, b, e)
    else:
        indptr, indices, memo_io["out"] = build_graph_rows_memo(
            covering, index, model, inputs, cfg, b, e, origin=memo_io.get("origin"),
            memo=memo_io.get("memo"), keep_memo=bool(memo_io.get("keep")),
            fwd=memo_io.get("fwd"))
    keep = torch.empty(V, dtype=torch.uint8, device=D.device())
    full = None
    if exchange_mode(group) == "p2p":
        try:
            ex, rounds = fused_peel(indptr, indices, V, group=group)
            words = ex.local_words()
        except PeerMappingError:
            _FUSED_OK[_peer_key(group)] = "nccl"
            _PEERS.pop(_peer_key(group), None)
            full = True
    else:
        full = True
    if full is not None:
        full, rounds = sharded_peel(indptr, indices, V, rank, size, group=group)
        words = D.ptr(full)
    if V:
        D.check(D.load_library().gis_bitmap_to_mask(D.ctx(), words, V, D.ptr(keep)))
    ne = torch.tensor([indices.shape[0]], dtype=torch.int64, device=D.device())
    all_reduce_(ne, group=group)
    if return_graph:
        return keep, int(ne.item()), rounds, gather_rows(indptr, indices, V, group)
    return keep, int(ne.item()), rounds


# -- adaptive selection and containment, sharded by owned cells ---------------
# The covering is replicated; each rank evaluates the probes / k-NN queries /
# containment of its owned cells and the ranks combine: boundary and
# neighbourhood masks by a MAX all-reduce (a logical OR over uint8), the
# containment defect by an all-gather of one scalar per rank.

def sharded_boundary(covering, index, delta: float, include_face_points=False, group=None):
    """select_boundary_mask (cg/adaptive.py:93-123) over all cells, each rank
    probing its owned range; uint8 device mask."""
    import torch
    import torch.distributed as dist

    rank, size = world()
    V = len(covering)
    out = torch.zeros(V, dtype=torch.uint8, device=D.device())
    if V:
        b, e = owned_range(V, rank, size)
        D.check(D.load_library().gis_select_boundary_range(
            D.ctx(), index._h, D.ptr(covering._lo), D.ptr(covering._hi), V, b, e, float(delta),
            int(bool(include_face_points)), D.ptr(out)), "select_boundary")
        all_reduce_(out, op=dist.ReduceOp.MAX, group=group)
    return out


def sharded_neighborhood(index, boundary, n_neighbors: int, group=None):
    """select_neighborhood_mask (cg/adaptive.py:136-150): each rank runs the
    k-NN of the boundary cells it owns, the marks are OR-reduced, then the
    boundary is removed; uint8 device mask."""
    import torch
    import torch.distributed as dist

    rank, size = world()
    V = index.size
    out = torch.zeros(V, dtype=torch.uint8, device=D.device())
    if V and n_neighbors > 0:
        b, e = owned_range(V, rank, size)
        lib = D.load_library()
        D.check(lib.gis_select_neighborhood_range(
            D.ctx(), index._h, D.ptr(index._lo), D.ptr(index._hi), V, D.ptr(boundary), b, e,
            int(n_neighbors), 0, D.ptr(out)), "select_neighborhood")
        all_reduce_(out, op=dist.ReduceOp.MAX, group=group)
        D.check(lib.gis_mask_andnot(D.ctx(), D.ptr(out), D.ptr(boundary), V),
                "select_neighborhood")
    return out


def sharded_containment(new_cov, prev_cov, prev_index, group=None) -> float:
    """engine._containment_defect (cg/engine.py:114-130) over the new cells,
    each rank its owned range; NaN if any rank saw a negative coverage."""
    import ctypes as C

    import torch

    rank, size = world()
    V = len(new_cov)
    d = C.c_double(0.0)
    if V:
        b, e = owned_range(V, rank, size)
        D.check(D.load_library().gis_containment_defect_range(
            D.ctx(), prev_index._h, D.ptr(prev_cov._lo), D.ptr(prev_cov._hi), len(prev_cov),
            D.ptr(new_cov._lo), D.ptr(new_cov._hi), V, b, e, C.byref(d)), "containment")
    mine = torch.tensor([d.value], dtype=torch.float64, device=D.device())
    vals = torch.cat(all_gather_(mine, group)).cpu().numpy()
    return float("nan") if np.isnan(vals).any() else float(vals.max())
