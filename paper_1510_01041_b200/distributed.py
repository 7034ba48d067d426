"""Multi-GPU exact LMS: one process per GPU, rank-space partitions, one collective.

The vertex index space (row-major pair ranks, backend.py:111-122) is split
into contiguous partitions exactly as ``BatchPlan.partitions`` does
(backend.py:84-92).  Each process solves its partition on its own GPU; the
per-rank best records are combined with a single ``all_gather`` (NCCL over
NVLink on the GPU box) and every rank takes the same lexicographic
(height, i, j) minimum (backend.py:182-187), so the result is bit-identical
for any world size.

The combine is expressed over ``torch.distributed`` so the same code runs on
``nccl`` (GPU tensors) and ``gloo`` (CPU tensors, used by the CPU tests).
"""

from __future__ import annotations

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

    ``solve_range(r0, r1)`` defaults to the CUDA engine on this process's GPU
    (``torch.cuda.current_device()``); tests substitute another exact solver
    to exercise the partition/combine logic on CPU-only ``gloo`` groups.
    """
    import torch.distributed as dist

    n = int(np.asarray(a).size)
    total = n * (n - 1) // 2
    r0, r1 = partition(total, dist.get_world_size(group), dist.get_rank(group))
    if solve_range is None:
        import torch

        from . import _native

        dev = torch.cuda.current_device()
        device = device if device is not None else torch.device("cuda", dev)

        def solve_range(lo, hi):  # noqa: E306
            return record_from_native(_native.min_bracelet(a, b, q, lo, hi, dev))

    rec = solve_range(r0, r1) if r1 > r0 else None
    return combine(all_gather_records(rec, group=group, device=device))
