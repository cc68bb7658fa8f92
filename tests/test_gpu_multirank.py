"""Sharded build + prune kernels on one GPU.

Ranks are emulated *sequentially* in one process (no kernel ever waits on
another): each emulated rank builds its owned rows with gis_build_graph_begin
and sweeps them with gis_peel_sweep on its own bitmap copy; between sweeps
the owned words are merged exactly as the NCCL all-gather would.  A real
1-rank NCCL group exercises distributed.build_and_prune_sharded end to end."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _grid(model, depth):
    from paper_2202_06111_b200 import Covering

    cov = Covering.initial(model.X)
    for _ in range(depth):
        cov = cov.subdivide(None)
    return cov


def _emulated(cov, idx, model, inputs, cfg, size):
    import torch

    from paper_2202_06111_b200.distributed import _device_sweep, owned_range, word_partition
    from paper_2202_06111_b200 import _device as D
    from paper_2202_06111_b200.graph import build_graph_rows

    V = len(cov)
    W = word_partition(V, size)
    shards, fulls, ptrs = [], [], []
    for r in range(size):
        b, e = owned_range(V, r, size)
        ip, ix = build_graph_rows(cov, idx, model, inputs, cfg, b, e)
        full = torch.zeros(size * W, dtype=torch.int32, device="cuda")
        ptr = torch.empty(max(e - b, 1), dtype=torch.int64, device="cuda")
        D.check(D.load_library().gis_peel_init(D.ctx(), D.ptr(ip), V, b, e, D.ptr(full),
                                               D.ptr(ptr)))
        shards.append((b, e, ip, ix))
        fulls.append(full)
        ptrs.append(ptr)
    sweeps = 0
    while True:
        deaths = sum(_device_sweep(ip, ix, b, e, fulls[r], ptrs[r])
                     for r, (b, e, ip, ix) in enumerate(shards))
        sweeps += 1
        merged = torch.cat([fulls[r][r * W:(r + 1) * W] for r in range(size)])
        for f in fulls:
            f.copy_(merged)
        if deaths == 0:
            break
    keep = torch.empty(V, dtype=torch.uint8, device="cuda")
    D.check(D.load_library().gis_bitmap_to_mask(D.ctx(), D.ptr(merged), V, D.ptr(keep)))
    return shards, keep.cpu().numpy().astype(bool), sweeps


@pytest.mark.parametrize("size", [2, 3, 8])
def test_emulated_ranks_match_single_gpu(size):
    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.graph import build_graph_serial

    rc = config(2)
    m = rc.model
    cov = _grid(m, 16)  # 256 x 256 cells
    idx = cov.build_index()
    inputs = sample_inputs(m.U, rc.input_counts)
    g = build_graph_serial(cov, idx, m, inputs, rc.image)
    want = non_leaving_mask(g)
    shards, keep, sweeps = _emulated(cov, idx, m, inputs, rc.image, size)
    assert np.array_equal(keep, want)
    ip_full, ix_full = g.indptr, g.indices
    for b, e, ip, ix in shards:  # owned rows are exactly the global rows
        ip, ix = ip.cpu().numpy(), ix.cpu().numpy()
        assert np.array_equal(ip, ip_full[b:e + 1] - ip_full[b])
        assert np.array_equal(ix, ix_full[ip_full[b]:ip_full[e]])


@pytest.mark.parametrize("mode", ["nccl", "p2p"])
def test_nccl_one_rank_sharded_path(mode, monkeypatch):
    """build_and_prune_sharded in a real 1-rank NCCL group, with the default
    exchange (sweep + in-place all-gather) and the opt-in fused one."""
    import torch
    import torch.distributed as dist

    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200 import distributed as DI
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.graph import build_graph_serial

    monkeypatch.setenv("GIS_PEEL_EXCHANGE", mode)
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    DI._FUSED_OK.clear()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        assert DI.exchange_mode() == mode
        rc = config(1)
        m = rc.model
        cov = _grid(m, 12)
        idx = cov.build_index()
        inputs = sample_inputs(m.U, rc.input_counts)
        keep, edges, sweeps, (gip, gix) = DI.build_and_prune_sharded(
            cov, idx, m, inputs, rc.image, return_graph=True)
        g = build_graph_serial(cov, idx, m, inputs, rc.image)
        assert edges == g.edge_count == 46120
        assert np.array_equal(gip.cpu().numpy(), g.indptr)
        assert np.array_equal(gix.cpu().numpy(), g.indices)
        assert np.array_equal(keep.cpu().numpy().astype(bool), non_leaving_mask(g))
        assert any(ex.cap for ex in DI._PEERS.values()) == (mode == "p2p")
        keep2, _, _ = DI.build_and_prune_sharded(cov, idx, m, inputs, rc.image)  # seq advanced
        assert torch.equal(keep, keep2)
        DI.release_peer_bitmaps()
    finally:
        DI._FUSED_OK.clear()
        dist.destroy_process_group()


def _two_gpu_worker(rank, port, mode, q):
    try:
        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE="2", LOCAL_WORLD_SIZE="2", GIS_PEEL_EXCHANGE=mode)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=2,
                                device_id=torch.device("cuda", rank))
        from paper_2202_06111_b200 import sample_inputs
        from paper_2202_06111_b200 import distributed as DI
        from paper_2202_06111_b200.configs import config

        rc = config(2)
        m = rc.model
        cov = _grid(m, 16)
        idx = cov.build_index()
        inputs = sample_inputs(m.U, rc.input_counts)
        got_mode = DI.exchange_mode()
        keep, edges, sweeps = DI.build_and_prune_sharded(cov, idx, m, inputs, rc.image)
        DI.release_peer_bitmaps()
        dist.destroy_process_group()
        q.put((rank, got_mode, keep.cpu().numpy().astype(bool), edges, None))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, None, repr(exc)))


@pytest.mark.parametrize("mode", ["nccl", "p2p"])
def test_two_gpus_sharded_prune_matches_single_gpu(mode):
    """the multi-GPU prune on two real GPUs (NCCL all-gather
    default, and the fused peer-memory kernel) must give the single-GPU keep
    mask.  Skipped with fewer than two GPUs (this round's boxes have one)."""
    import torch
    import torch.multiprocessing as tmp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.graph import build_graph_serial

    rc = config(2)
    m = rc.model
    cov = _grid(m, 16)
    idx = cov.build_index()
    g = build_graph_serial(cov, idx, m, sample_inputs(m.U, rc.input_counts), rc.image)
    want = non_leaving_mask(g)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_gpu_worker, args=(r, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for rank, got_mode, keep, edges, err in res:
        assert err is None, err
        assert got_mode == mode
        assert edges == g.edge_count
        assert np.array_equal(keep, want)


@pytest.mark.parametrize("size", [2, 3, 8])
@pytest.mark.parametrize("cfg_id", [3, 5])
def test_emulated_sharded_selection_and_containment(size, cfg_id):
    """The multi-GPU engine's range kernels (distributed.sharded_boundary /
    sharded_neighborhood / sharded_containment), emulated rank by rank on one
    GPU: OR-combined range masks and the max of range defects equal the
    single-GPU results."""
    import ctypes as C

    import torch

    from paper_2202_06111_b200 import _device as D, run
    from paper_2202_06111_b200.adaptive import boundary_dev, neighborhood_dev
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.distributed import owned_range
    from paper_2202_06111_b200.engine import containment_defect

    rc = config(cfg_id, iterations=2) if cfg_id == 3 else \
        config(5, initial_grid=None, initial_depth=8, iterations=2)
    cov = run(rc).covering  # an adaptive (mixed-depth) covering
    idx = cov.build_index()
    ad = rc.adaptive
    lib = D.load_library()
    V = len(cov)
    want_b = boundary_dev(cov, idx, ad.delta, ad.include_face_points)
    want_n = neighborhood_dev(idx, want_b, ad.n_neighbors)
    got_b = torch.zeros(V, dtype=torch.uint8, device="cuda")
    got_n = torch.zeros(V, dtype=torch.uint8, device="cuda")
    child = cov.subdivide(want_b | want_n)
    defects = []
    for r in range(size):
        b, e = owned_range(V, r, size)
        part = torch.zeros(V, dtype=torch.uint8, device="cuda")
        D.check(lib.gis_select_boundary_range(D.ctx(), idx._h, D.ptr(cov._lo), D.ptr(cov._hi), V,
                                              b, e, float(ad.delta),
                                              int(bool(ad.include_face_points)), D.ptr(part)))
        got_b = torch.maximum(got_b, part)
        D.check(lib.gis_select_neighborhood_range(D.ctx(), idx._h, D.ptr(idx._lo),
                                                  D.ptr(idx._hi), V, D.ptr(want_b), b, e,
                                                  ad.n_neighbors, 0, D.ptr(part)))
        got_n = torch.maximum(got_n, part)
        cb, ce = owned_range(len(child), r, size)
        d = C.c_double()
        D.check(lib.gis_containment_defect_range(D.ctx(), idx._h, D.ptr(cov._lo), D.ptr(cov._hi),
                                                 V, D.ptr(child._lo), D.ptr(child._hi),
                                                 len(child), cb, ce, C.byref(d)))
        defects.append(d.value)
    D.check(lib.gis_mask_andnot(D.ctx(), D.ptr(got_n), D.ptr(want_b), V))
    assert torch.equal(got_b, want_b)
    assert torch.equal(got_n, want_n)
    assert max(defects) == containment_defect(child, cov, idx)


@pytest.mark.parametrize("size", [1, 2, 3, 8])
def test_emulated_fused_peer_prune_matches_single_gpu(size):
    """gis_peel_p2p with `size` ranks emulated in ONE cooperative launch
    (block groups as ranks, replicas + flag areas on this GPU): the fused
    sweep / push / flag-barrier protocol leaves every rank's replica equal to
    the single-GPU keep mask (config 2 at 256^2 and random digraphs)."""
    import torch

    from oracle import gis_oracle as O
    from paper_2202_06111_b200 import _device as D, sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.distributed import emulated_fused_peel
    from paper_2202_06111_b200.graph import build_graph_serial

    rc = config(2)
    m = rc.model
    cov = _grid(m, 16)
    g = build_graph_serial(cov, cov.build_index(), m, sample_inputs(m.U, rc.input_counts),
                           rc.image)
    cases = [(g.indptr, g.indices, g.n_vertices, non_leaving_mask(g))]
    rng = np.random.default_rng(size)
    for nv in (1, 31, 33, 1000, 5000):
        deg = np.minimum(rng.integers(0, 3, nv), nv)
        ip = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        ix = np.concatenate([np.sort(rng.choice(nv, d, replace=False)) if d else
                             np.zeros(0, np.int64) for d in deg]).astype(np.int64)
        cases.append((ip, ix, nv, O.peel_fixed_point(ip, ix, nv)))
    for ip, ix, nv, want in cases:
        ipd = torch.as_tensor(ip, device="cuda")
        ixd = torch.as_tensor(ix.astype(np.int32), device="cuda")
        reps, rounds = emulated_fused_peel(ipd, ixd, nv, size)
        assert rounds >= 1
        for rep in reps:
            keep = torch.empty(nv, dtype=torch.uint8, device="cuda")
            D.check(D.load_library().gis_bitmap_to_mask(D.ctx(), D.ptr(rep), nv, D.ptr(keep)))
            assert np.array_equal(keep.cpu().numpy().astype(bool), want)


def _ipc_worker(rank, port, V, q):
    import torch
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        from paper_2202_06111_b200 import _device as D
        from paper_2202_06111_b200.distributed import PeerBitmaps

        ex = PeerBitmaps()
        ex.ensure((V + 31) // 32)
        lib, c = D.load_library(), D.ctx()
        # write a rank-specific mask into the PEER's replica through the
        # IPC mapping, then read our own replica (written by the peer)
        mask = torch.zeros(V, dtype=torch.uint8, device="cuda")
        mask[rank::3] = 1
        peer = 1 - rank
        D.check(lib.gis_mask_to_bitmap(c, D.ptr(mask), V, C_void(ex.rep_addrs[peer])))
        torch.cuda.synchronize()
        dist.barrier()
        got = torch.empty(V, dtype=torch.uint8, device="cuda")
        D.check(lib.gis_bitmap_to_mask(c, ex.local_words(), V, D.ptr(got)))
        want = torch.zeros(V, dtype=torch.uint8, device="cuda")
        want[peer::3] = 1
        ok = bool(torch.equal(got, want))
        ex.release()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(exc)))


def C_void(addr):
    import ctypes

    return ctypes.c_void_p(addr)


def test_peer_bitmaps_ipc_mapping_two_processes():
    """PeerBitmaps' handle exchange and gis_ipc_open across two processes on
    one GPU: each writes into the other's replica through its mapping (plain
    kernels, nothing waits on another process's kernel)."""
    import torch.multiprocessing as tmp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, 1000, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def test_bench_multirank_path_two_ranks_on_one_gpu():
    """bench.py's multi-rank path end to end on a one-GPU box: the launcher
    starts two ranks that share cuda:0 in the gloo test mode
    (GIS_DIST_BACKEND=gloo: collectives on host copies, no kernel of one rank
    waits on the other's).  The sharded config-2 step, its e2e twin and the
    sharded engine runs of configs 2 and 5 must reproduce the single-GPU
    results (edges, kept cells, final coverings)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, GIS_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "1", "--no-cpu-baseline"], capture_output=True, text=True,
                       timeout=900, env=env, cwd=str(root))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    ln = lines[0]
    assert ln["n_gpus"] == 2 and ln["config"]["dist_backend"] == "gloo"
    assert ln["config"]["edges"] == 103_838_696 and ln["config"]["kept"] == 932_972
    assert ln["gis_wall_s_config2"]["final_cells"] == 932_972
    assert ln["gis_wall_s_config5"]["final_cells"] == 7_898_713
    assert ln["e2e"]["value"] > 0
