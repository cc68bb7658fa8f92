"""Multi-rank pruning protocol (row shards + per-sweep bitmap all-gather +
deletion-count all-reduce) at world_size 2 on CPU with gloo.  The per-rank
sweep is a numpy restatement of gis_peel_sweep's semantics; the exchange
logic under test is paper_2202_06111_b200.distributed.sharded_peel."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _np_init(indptr_local, V, b, e, full, ptr):
    nw = (V + 31) // 32
    words = np.zeros(len(full), dtype=np.uint32)
    words[:nw] = 0xFFFFFFFF
    if V % 32:
        words[nw - 1] = (1 << (V % 32)) - 1
    full.copy_(torch.from_numpy(words.view(np.int32)))
    ptr[:e - b] = indptr_local[:-1]


def _np_sweep(indptr_local, indices, b, e, full, ptr):
    words = full.numpy().view(np.uint32)
    alive = lambda t: (words[t >> 5] >> np.uint32(t & 31)) & np.uint32(1)  # noqa: E731
    deaths = 0
    ip, ix = indptr_local.numpy(), indices.numpy()
    p_arr = ptr.numpy()
    for v in range(b, e):
        if not alive(v):
            continue
        r = v - b
        p, end = p_arr[r], ip[r + 1]
        while p < end and not alive(int(ix[p])):
            p += 1
        p_arr[r] = p
        if p == end:
            words[v >> 5] &= np.uint32(~(1 << (v & 31)) & 0xFFFFFFFF)
            deaths += 1
    return deaths


def _worker(rank, size, port, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.distributed import owned_range, sharded_peel

    rng = np.random.default_rng(seed)
    n = int(rng.integers(40, 700))
    m = int(rng.uniform(0.5, 3.0) * n)
    ip, ix = O.csr_from_pairs(rng.integers(0, n, m), rng.integers(0, n, m), n)
    b, e = owned_range(n, rank, size)
    local_ip = torch.from_numpy(ip[b:e + 1] - ip[b])
    local_ix = torch.from_numpy(ix[ip[b]:ip[e]].astype(np.int32))
    full, rounds = sharded_peel(local_ip, local_ix, n, rank, size, sweep=_np_sweep,
                                init=_np_init)
    words = full.numpy().view(np.uint32)
    keep = ((words[np.arange(n) >> 5] >> (np.arange(n) & 31).astype(np.uint32)) & 1).astype(bool)
    out[rank] = (keep.tolist(), O.peel_fixed_point(ip, ix, n).tolist(), rounds)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_sharded_peel_world2_matches_oracle(seed):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), seed, out), nprocs=2, join=True)
    k0, want, r0 = out[0]
    k1, _, r1 = out[1]
    assert k0 == k1 == want
    assert r0 == r1 >= 1


def _gather_worker(rank, size, port, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from oracle import gis_oracle as O
    from paper_2202_06111_b200.distributed import gather_rows, owned_range

    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    m = int(rng.uniform(0.0, 3.0) * n)
    ip, ix = O.csr_from_pairs(rng.integers(0, n, m), rng.integers(0, n, m), n)
    b, e = owned_range(n, rank, size)
    local_ip = torch.from_numpy(ip[b:e + 1] - ip[b])
    local_ix = torch.from_numpy(ix[ip[b]:ip[e]].astype(np.int32))
    gip, gix = gather_rows(local_ip, local_ix, n)
    out[rank] = (gip.tolist(), gix.tolist(), ip.tolist(), ix.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("size,seed", [(2, 4), (3, 5), (2, 6)])
def test_gather_rows_reassembles_the_graph(size, seed):
    """engine.run(keep_final_graph=True) in a sharded job: every rank's owned
    rows gathered into the whole CSR (final_graph was None)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(size, _free_port(), seed, out), nprocs=size, join=True)
    for r in range(size):
        gip, gix, ip, ix = out[r]
        assert gip == ip and gix == ix
