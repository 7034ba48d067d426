"""N > 1 path on CPU: world_size-2 gloo groups run the partition + single
all_gather combine of paper_1510_01041_b200.distributed, with the CPU oracle
standing in for the per-rank GPU solve.  The combined record must equal the
single-process result bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1510_01041_b200 import distributed


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, a, b, q, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def solve_range(r0, r1):
            rec = oracle.min_bracelet(a, b, q, r0, r1, threads=1)
            if rec is None:
                return None
            from paper_1510_01041_b200.backend import CandidateRecord

            return CandidateRecord(rec.height, rec.i, rec.j, rec.u, rec.v_low, rec.v_high)

        rec = distributed.solve_distributed(a, b, q, solve_range=solve_range)
        np.save(f"{out_path}.{rank}.npy", distributed.pack(rec))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_partitioned_solve_matches_single(tmp_path, world):
    oracle.build()
    rng = np.random.default_rng(77)
    pts = rng.normal(0, 10, (70, 2))
    pts[:20, 0] = pts[0, 0]
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = 36
    out = str(tmp_path / "rec")
    mp.start_processes(_worker, args=(world, _free_port(), a, b, q, out), nprocs=world,
                       start_method="spawn")
    ref = oracle.min_bracelet(a, b, q)
    for r in range(world):
        got = distributed.unpack(np.load(f"{out}.{r}.npy"))
        assert (got.height, got.i, got.j, got.u, got.v_low, got.v_high) == \
            (ref.height, ref.i, ref.j, ref.u, ref.v_low, ref.v_high)


def test_partition_matches_batch_plan():
    from paper_1510_01041_b200.backend import BatchPlan

    for n in (5, 9, 64, 1000):
        total = n * (n - 1) // 2
        for w in (1, 2, 3, 4, 8):
            plan = BatchPlan.create(np.arange(n, dtype=float), w).partitions()
            ours = [distributed.partition(total, w, r) for r in range(w)]
            ours = [p for p in ours if p[1] > p[0]]
            assert ours == plan


def test_pack_roundtrip_and_combine_order():
    from paper_1510_01041_b200.backend import CandidateRecord

    r1 = CandidateRecord(1.5, 3, 7, 0.25, -1.0, 0.5)
    r2 = CandidateRecord(1.5, 2, 9, 0.5, -2.0, -0.5)
    rows = np.stack([distributed.pack(r1), distributed.pack(None), distributed.pack(r2)])
    assert distributed.unpack(rows[0]) == r1 and distributed.unpack(rows[1]) is None
    assert distributed.combine(rows) == r2  # equal height: smaller (i, j) wins


def _table_worker(rank, world, port, nbands, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_01041_b200.backend import CandidateRecord

        full = np.arange(nbands * 7, dtype=np.float64).reshape(nbands, 7) * 0.5 - 3.0
        mine = full[list(distributed.band_slice(nbands, world, rank))]
        seed = None if rank == 0 else CandidateRecord(2.0, 10 - rank, 20, 0.5, -1.0, 1.0)
        got, best = distributed.exchange_band_table(mine, nbands, seed)
        np.save(f"{out_path}.{rank}.npy", got)
        np.save(f"{out_path}.{rank}.seed.npy", distributed.pack(best))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nbands", [(2, 1024), (3, 1024), (3, 2), (2, 5)])
def test_gloo_band_table_exchange(tmp_path, world, nbands):
    """The sharded plan's all_gather reassembles every rank's band slice into
    the full table in band order, including short and empty last slices."""
    out = str(tmp_path / "tab")
    mp.start_processes(_table_worker, args=(world, _free_port(), nbands, out), nprocs=world,
                       start_method="spawn")
    full = np.arange(nbands * 7, dtype=np.float64).reshape(nbands, 7) * 0.5 - 3.0
    for r in range(world):
        assert np.array_equal(np.load(f"{out}.{r}.npy"), full)
        best = distributed.unpack(np.load(f"{out}.{r}.seed.npy"))
        assert (best.i, best.j) == (10 - (world - 1), 20)  # equal heights: smallest (i, j)


def test_band_table_pack_roundtrip():
    from paper_1510_01041_b200 import _native

    rng = np.random.default_rng(3)
    lb = rng.normal(size=9)
    wq = rng.normal(size=9)
    edge = rng.normal(size=(9, _native.BAND_EDGE_KEYS)).astype(np.float32)
    t = _native.pack_band_table(lb, wq, edge)
    assert t.shape == (9, _native.BAND_TABLE_COLS)
    l2, w2, e2 = _native.unpack_band_table(t)
    assert np.array_equal(l2, lb) and np.array_equal(w2, wq) and np.array_equal(e2, edge)
