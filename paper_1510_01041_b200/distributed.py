"""Multi-GPU exact LMS: one process per GPU, one fit's vertices shared out.

``solve_sharded`` is the sharded band search with band ownership (SURVEY
section 8e; the C ABI's lms_ctx_solve_distributed): every rank samples the
whole pair space (the same slope bands everywhere), bounds and seeds its own
interleaved slice of the bands, the 56-byte seed records are all-gathered,
each rank searches the vertices of its own bands that the best seed cannot
dismiss, and the records are all-gathered and merged with the lexicographic
(height, i, j) minimum (backend.py:182-187) -- the one-GPU record for any
world size.  With the ``nccl`` backend both collectives run inside the
library (ncclAllGather on device buffers over NVLink, the communicator
bootstrapped from a unique id that rank 0 broadcasts); with ``gloo`` (CPU
tests, functional runs on one GPU) the same flow runs over
``torch.distributed`` on host records.

``solve_distributed(..., solve_range=f)`` keeps the plain contiguous-partition
form (``BatchPlan.partitions``, backend.py:84-92) for CPU tests: each rank
solves its rank range and one all-gather of records combines them.
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
    """Bands a rank owns in a sharded search: rank, rank + world, ... (interleaved)."""
    return range(rank, nbands, world)


def interleave_band_table(slices: list, nbands: int) -> np.ndarray:
    """Full (nbands, cols) band table from the ranks' interleaved slices (band
    k = row k // world of rank k % world's slice), the input of the
    rank-range shard search (lms_ctx_shard_search)."""
    world = len(slices)
    cols = slices[0].shape[1] if slices and slices[0].ndim == 2 else 0
    full = np.empty((nbands, cols), dtype=np.float64)
    for r, t in enumerate(slices):
        full[r::world] = t[: len(range(r, nbands, world))]
    return full


_comms: dict = {}


def _native_comm(ctx, group) -> bool:
    """Bind an NCCL communicator over ``group`` to ``ctx`` inside the library
    (rank 0 makes the unique id, one broadcast); False when the library
    cannot load NCCL."""
    import torch.distributed as dist

    from . import _native

    key = (id(ctx), id(group) if group is not None else 0)
    if key in _comms:
        return True
    ok, _ = _native.nccl_available()
    flags = [ok]
    dist.broadcast_object_list(flags, src=0, group=group)  # every rank takes the same road
    if not flags[0]:
        return False
    obj = [_native.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(dist.get_world_size(group), dist.get_rank(group), obj[0])
    _comms[key] = True
    return True


def solve_sharded(ctx, q: int, *, group=None, device=None) -> CandidateRecord | None:
    """Sharded band search of the lines bound to ``ctx`` (this rank's GPU).

    plan (this rank's own bands and seed) -> all-gather of the seed records ->
    search of this rank's own bands (or, for fits too small for bands, its
    pair-rank partition) -> all-gather of the records -> lexicographic
    minimum.  Same record as one ``ctx.solve`` over the whole pair space.
    """
    import torch.distributed as dist

    from ._native import Candidate

    if dist.get_backend(group) == "nccl" and _native_comm(ctx, group):
        return record_from_native(ctx.solve_distributed(q))
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    _, _, seed = ctx.shard_plan(q, world, rank)
    seeds = all_gather_records(record_from_native(seed), group=group, device=device)
    rec = record_from_native(ctx.shard_search_owned(q, world, rank, Candidate.of(combine(seeds))))
    return combine(all_gather_records(rec, group=group, device=device))
