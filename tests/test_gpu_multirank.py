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


def test_nccl_one_rank_sharded_path():
    import torch
    import torch.distributed as dist

    from paper_2202_06111_b200 import sample_inputs
    from paper_2202_06111_b200.analysis import non_leaving_mask
    from paper_2202_06111_b200.configs import config
    from paper_2202_06111_b200.distributed import build_and_prune_sharded
    from paper_2202_06111_b200.graph import build_graph_serial

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rc = config(1)
        m = rc.model
        cov = _grid(m, 12)
        idx = cov.build_index()
        inputs = sample_inputs(m.U, rc.input_counts)
        keep, edges, sweeps = build_and_prune_sharded(cov, idx, m, inputs, rc.image)
        g = build_graph_serial(cov, idx, m, inputs, rc.image)
        assert edges == g.edge_count == 46120
        assert np.array_equal(keep.cpu().numpy().astype(bool), non_leaving_mask(g))
    finally:
        dist.destroy_process_group()


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
