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


class _OracleShardCtx:
    """CPU stand-in for one rank's engine context in the sharded search: the
    plan's seed is the oracle minimum over a few vertices of the rank's own
    share, the own-band search the oracle minimum over the whole share merged
    with the exchanged seed (as the device installs it)."""

    def __init__(self, a, b):
        self.a, self.b = a, b

    def _rec(self, q, r0, r1):
        from paper_1510_01041_b200._native import Candidate
        from paper_1510_01041_b200.backend import CandidateRecord

        rec = oracle.min_bracelet(self.a, self.b, q, r0, r1, threads=1)
        return Candidate.of(None if rec is None else
                            CandidateRecord(rec.height, rec.i, rec.j, rec.u, rec.v_low, rec.v_high))

    def shard_plan(self, q, world, rank):
        n = self.a.size
        r0, r1 = distributed.partition(n * (n - 1) // 2, world, rank)
        self.share = (r0, r1)
        return 3 * world, None, self._rec(q, r0, min(r1, r0 + 7))

    def shard_search_owned(self, q, world, rank, seed):
        from paper_1510_01041_b200._native import Candidate
        from paper_1510_01041_b200.backend import merge, record_from_native

        own = record_from_native(self._rec(q, *self.share))
        return Candidate.of(merge(record_from_native(seed), own))


def _owned_worker(rank, world, port, a, b, q, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = distributed.solve_sharded(_OracleShardCtx(a, b), q)
        np.save(f"{out_path}.{rank}.npy", distributed.pack(rec))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seed", [(2, 40, 0), (3, 33, 1), (2, 25, 2)])
def test_gloo_sharded_search_flow(tmp_path, world, n, seed):
    """The sharded search's host flow over gloo: plan seeds all-gathered and
    merged, each rank's own search started from the best seed, records
    all-gathered and merged -- every rank ends with the single-process
    record (duplicate x and exact ties included)."""
    rng = np.random.default_rng(seed)
    pts = rng.integers(0, 12, (n, 2)).astype(float)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    out = str(tmp_path / "own")
    mp.start_processes(_owned_worker, args=(world, _free_port(), a, b, q, out), nprocs=world,
                       start_method="spawn")
    want = oracle.min_bracelet(a, b, q, threads=1)
    for r in range(world):
        got = distributed.unpack(np.load(f"{out}.{r}.npy"))
        assert (got.height, got.i, got.j, got.u, got.v_low, got.v_high) == \
            (want.height, want.i, want.j, want.u, want.v_low, want.v_high)


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
