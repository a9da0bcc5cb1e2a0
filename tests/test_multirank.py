"""Host logic of the row-sharded path on CPU (no GPU): balanced row splits and the
halo plan, checked across a world_size-2 gloo process group.

Each rank computes, with the library's host code, the reader-rank bitmask of its
own rows (sketchycgal_halo_plan).  By symmetry of L, rank p must mark row r for rank
q exactly when one of q's rows has column r: the ranks exchange what they computed
and each checks the other's plan against the columns of its own rows.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1912_02949_b200 as scg
import scg_inputs as si


def test_row_splits_balanced_and_cover():
    scg.build()
    for cfg, P in [("c0", 2), ("c1", 4), ("c0", 8)]:
        L = si.laplacian(cfg)
        sp = scg.row_splits(L.row_ptr, P)
        assert sp[0] == 0 and sp[-1] == L.n and np.all(np.diff(sp) > 0)
        cost = np.diff(sp) + np.diff(L.row_ptr[sp])
        tot = L.n + L.row_ptr[-1]
        # optimal bottleneck is at least tot/P and at most tot/P + the heaviest row
        heaviest = int(np.max(1 + np.diff(L.row_ptr)))
        assert cost.max() <= tot / P + heaviest


def test_row_splits_skewed_degrees():
    """A star: the heavy row must not drag every other row onto one rank."""
    n = 1000
    L = si.laplacian_from_edges(n, np.zeros(n - 1, dtype=np.int64), np.arange(1, n), np.ones(n - 1))
    sp = scg.row_splits(L.row_ptr, 4)
    cost = np.diff(sp) + np.diff(L.row_ptr[sp])
    assert cost.max() <= (n + L.row_ptr[-1]) / 4 + n


def _worker(rank, world, port, cfg, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = si.laplacian(cfg)
        sp = scg.row_splits(L.row_ptr, world)
        a, b = int(sp[rank]), int(sp[rank + 1])
        rp = L.row_ptr[a:b + 1]
        col = L.col[L.row_ptr[a]:L.row_ptr[b]]
        mask, halo = scg.halo_plan(rp, col, a, b, sp)
        # exchange every rank's mask (padded to n) and check the pair (p -> me)
        full = torch.zeros(L.n, dtype=torch.int32)
        full[a:b] = torch.from_numpy(mask.astype(np.int32))
        got = [torch.zeros(L.n, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(got, full)
        ok = True
        rows = np.repeat(np.arange(a, b), np.diff(rp))
        my_cols = set(int(c) for c, r in zip(col, rows) if not (a <= c < b))
        for p in range(world):
            if p == rank:
                continue
            pa, pb = int(sp[p]), int(sp[p + 1])
            marked = set(np.nonzero(got[p][pa:pb].numpy() & (1 << rank))[0] + pa)
            needed = set(c for c in my_cols if pa <= c < pb)
            ok &= marked == needed
        ok &= halo == int(np.count_nonzero(mask))
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        result[rank] = int(flag.item())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["c0", "c1"])
def test_halo_plan_consistent_across_ranks(cfg):
    scg.build()
    si.laplacian(cfg)  # build the generator library before forking
    world = 2
    port = 29500 + (os.getpid() % 2000)
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, port, cfg, result), nprocs=world, join=True)
    assert all(result[r] == 1 for r in range(world))


def _comm_worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes
        hc = scg.TorchHostComm()
        st = hc.struct
        ok = True
        # allgather: every rank contributes 24 bytes, receives world x 24 in rank order
        mine = bytes([rank * 10 + i for i in range(24)])
        out = ctypes.create_string_buffer(24 * world)
        ok &= st.allgather(None, mine, out, 24) == 0
        ok &= out.raw == b"".join(bytes([p * 10 + i for i in range(24)]) for p in range(world))
        # allreduce_sum in place over doubles
        buf = (ctypes.c_double * 5)(*[rank + 0.25 * i for i in range(5)])
        ok &= st.allreduce_sum(None, buf, 5) == 0
        ok &= list(buf) == [sum(p + 0.25 * i for p in range(world)) for i in range(5)]
        ok &= st.barrier(None) == 0
        ok &= st.sync_collectives == 1
        result[rank] = int(ok)
    finally:
        dist.destroy_process_group()


def test_torch_host_comm_callbacks_gloo():
    """The scg_host_comm transport the library calls for a multi-process run without NCCL
    (include/sketchycgal.h): allgather in rank order, in-place double sum, barrier -- over gloo."""
    world = 2
    port = 31500 + (os.getpid() % 2000)
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_comm_worker, args=(world, port, result), nprocs=world, join=True)
    assert all(result[r] == 1 for r in range(world))
