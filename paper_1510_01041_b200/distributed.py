"""Multi-GPU exact LMS: one process per GPU, rank-space partitions, one collective.

The vertex index space (row-major pair ranks, backend.py:111-122) is split
into contiguous partitions exactly as ``BatchPlan.partitions`` does
(backend.py:84-92).  Each process solves its partition on its own GPU; the
per-rank best records are combined with a single ``all_gather`` (NCCL over
NVLink on the GPU box) and every rank takes the same lexicographic
(height, i, j) minimum (backend.py:182-187), so the result is bit-identical
for any world size.

``solve_sharded`` is the band-search form of the same split: the slope-band
table (one lower bound, window and edge keys per band) is computed in slices,
one per rank, and exchanged with one more ``all_gather`` before each rank
searches its partition, so the per-band work is divided as well instead of
being repeated on every rank.

The combine is expressed over ``torch.distributed`` so the same code runs on
``nccl`` (GPU tensors) and ``gloo`` (CPU tensors, used by the CPU tests).
"""

from __future__ import annotations

import threading
from typing import Callable

import numpy as np

from .backend import CandidateRecord, merge, record_from_native

RECORD_FIELDS = 7  # found, height, i, j, u, v_low, v_high (int64 i/j exact in fp64 below 2**53)


def partition(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous rank range of partition ``rank`` (ceil split, backend.py:81,84-92)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    size = max(1, -(-total // world))
    lo = min(total, rank * size)
    return lo, min(total, lo + size)


def pack(rec: CandidateRecord | None) -> np.ndarray:
    out = np.zeros(RECORD_FIELDS, dtype=np.float64)
    if rec is not None:
        out[:] = (1.0, rec.height, float(rec.i), float(rec.j), rec.u, rec.v_low, rec.v_high)
    return out


def unpack(row: np.ndarray) -> CandidateRecord | None:
    if row[0] == 0.0:
        return None
    return CandidateRecord(height=float(row[1]), i=int(row[2]), j=int(row[3]), u=float(row[4]),
                           v_low=float(row[5]), v_high=float(row[6]))


def combine(rows: np.ndarray) -> CandidateRecord | None:
    """Lexicographic minimum of gathered records, in rank order."""
    best = None
    for row in rows:
        best = merge(best, unpack(row))
    return best


def all_gather_records(rec: CandidateRecord | None, group=None, device=None) -> np.ndarray:
    """One all_gather of the packed 7-double record across the process group."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = torch.from_numpy(pack(rec))
    if device is not None:
        mine = mine.to(device)
    out = torch.empty(world * RECORD_FIELDS, dtype=torch.float64, device=mine.device)
    dist.all_gather_into_tensor(out, mine, group=group)
    return out.view(world, RECORD_FIELDS).cpu().numpy()


def solve_distributed(a: np.ndarray, b: np.ndarray, q: int, *, group=None,
                      solve_range: Callable[[int, int], CandidateRecord | None] | None = None,
                      device=None) -> CandidateRecord | None:
    """Solve this rank's partition and return the global exact minimum.

    By default the CUDA engine on this process's GPU
    (``torch.cuda.current_device()``) runs the sharded band search
    (``solve_sharded``).  ``solve_range(r0, r1)`` substitutes a per-partition
    exact solver: tests use the CPU oracle to exercise the partition/combine
    logic on CPU-only ``gloo`` groups.
    """
    import torch.distributed as dist

    if solve_range is None:
        import torch

        dev = torch.cuda.current_device()
        if device is None and dist.get_backend(group) == "nccl":
            device = torch.device("cuda", dev)  # NCCL collectives take device tensors
        ctx = _context(dev)
        with _solve_lock:  # upload, plan and search bind the lines to one shared context
            ctx.upload(a, b)
            return solve_sharded(ctx, q, group=group, device=device)
    n = int(np.asarray(a).size)
    total = n * (n - 1) // 2
    r0, r1 = partition(total, dist.get_world_size(group), dist.get_rank(group))
    rec = solve_range(r0, r1) if r1 > r0 else None
    return combine(all_gather_records(rec, group=group, device=device))


_contexts: dict = {}
_contexts_lock = threading.Lock()
_solve_lock = threading.Lock()


def _context(device: int):
    """This process's engine context on `device` (created on first use)."""
    with _contexts_lock:
        if device not in _contexts:
            from . import _native

            _contexts[device] = _native.Context(device)
        return _contexts[device]


def band_slice(nbands: int, world: int, rank: int) -> range:
    """Bands a rank bounds in a sharded plan: rank, rank + world, ... (interleaved)."""
    return range(rank, nbands, world)


def interleave_band_table(slices: list, nbands: int) -> np.ndarray:
    """Full (nbands, cols) table from the ranks' slices (band k = row k // world of
    rank k % world's slice)."""
    world = len(slices)
    cols = slices[0].shape[1] if slices and slices[0].ndim == 2 else 0
    full = np.empty((nbands, cols), dtype=np.float64)
    for r, t in enumerate(slices):
        full[r::world] = t[: len(range(r, nbands, world))]
    return full


def exchange_band_table(table: np.ndarray, nbands: int, seed: CandidateRecord | None = None,
                        group=None, device=None) -> tuple[np.ndarray, CandidateRecord | None]:
    """All-gather every rank's band-table slice and plan seed in one collective.

    Returns the full (nbands, cols) table and the minimum of the seeds.  Each
    rank sends one header row (its packed seed record, RECORD_FIELDS wide)
    followed by its slice (bands rank, rank + world, ...; band_slice), padded
    to ceil(nbands / world) rows.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cols = table.shape[1]
    assert cols == RECORD_FIELDS, "band table rows and records share one row width"
    per = max(1, -(-nbands // world))
    mine = torch.zeros((1 + per, cols), dtype=torch.float64)
    mine[0] = torch.from_numpy(pack(seed))
    if len(table):
        mine[1: 1 + len(table)] = torch.from_numpy(np.ascontiguousarray(table))
    if device is not None:
        mine = mine.to(device)
    out = torch.empty((world, 1 + per, cols), dtype=torch.float64, device=mine.device)
    dist.all_gather_into_tensor(out.view(world * (1 + per), cols), mine, group=group)
    out = out.cpu().numpy()
    full = interleave_band_table([out[r, 1:] for r in range(world)], nbands)
    return full, combine(out[:, 0])


def solve_sharded(ctx, q: int, *, group=None, device=None) -> CandidateRecord | None:
    """Sharded band search of the lines bound to ``ctx`` (this rank's GPU).

    plan (this rank's band slice and seed) -> one all_gather of the band table
    and seeds -> search of this rank's partition against the full table ->
    all_gather of the records -> lexicographic minimum.  Same record as one
    ``ctx.solve`` over the whole pair space.
    """
    import torch.distributed as dist

    from ._native import Candidate

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nbands, table, seed = ctx.shard_plan(q, world, rank)
    full, best_seed = table[:0], None
    if nbands:
        full, best_seed = exchange_band_table(table, nbands, record_from_native(seed), group=group,
                                              device=device)
    rec = record_from_native(ctx.shard_search(q, world, rank, full, Candidate.of(best_seed)))
    return combine(all_gather_records(rec, group=group, device=device))
