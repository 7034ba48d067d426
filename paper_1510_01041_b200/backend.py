"""Execution backends (drop-in for lmsline.backend), both running the CUDA engine.

The reference's backend protocol (backend.py:234-303) is kept: ``get_backend``
returns an object with ``.name`` and ``.minimum_bracelet(a, b, q, *,
materialize=False) -> CandidateRecord | None`` over the row-major upper
triangle of pair ranks.  Both registered names run the same sm_100a engine
(``_native``); there is no CPU path and no other backend name -- in
particular ``"gpu"`` is not a backend, exactly as in the reference
(test_backend.py:168-172).

* ``seq`` solves the whole rank range on device 0.
* ``par`` splits the rank range into contiguous partitions
  (``BatchPlan.partitions``, backend.py:84-92), one per visible GPU (capped by
  the worker count), solves them concurrently and merges the partition
  minima with the exact lexicographic key (backend.py:182-187), so the result
  is bit-identical to ``seq`` for any worker or device count.
* ``materialize=True`` runs the materialised two-kernel flow of the
  reference (``_materialized_inputs`` + ``_scan_materialized``,
  backend.py:210-231; the paper's K1 -> K2): every non-parallel pair becomes
  an explicit (i, j, u) triple on the device and each one is evaluated
  exactly, without the pruning stages.  The record is the same as the
  streaming engine's (the reference states the same equivalence).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Iterable, Iterator, Sequence

import numpy as np

from . import _native
from .geometry import DualIntersection, DualLine, InvalidInputError, pair_intersection

WORKERS_ENV_VAR = "LMSLINE_WORKERS"


@dataclass(frozen=True)
class CandidateRecord:
    """Best bracelet over some set of pairs (backend.py:37-54)."""

    height: float
    i: int
    j: int
    u: float
    v_low: float
    v_high: float

    @property
    def sort_key(self) -> tuple[float, int, int]:
        return (self.height, self.i, self.j)


def record_from_native(c) -> CandidateRecord | None:
    if not c.found:
        return None
    return CandidateRecord(height=c.height, i=int(c.i), j=int(c.j), u=c.u, v_low=c.v_low, v_high=c.v_high)


@dataclass(frozen=True)
class BatchPlan:
    """Pair count and contiguous rank partitions (backend.py:57-92)."""

    n: int
    pair_count: int
    partition_size: int
    worker_count: int

    @classmethod
    def create(cls, a: np.ndarray, worker_count: int) -> "BatchPlan":
        n = int(np.asarray(a).size)
        if n < 2:
            raise InvalidInputError(f"a batch needs at least 2 lines, got {n}")
        if worker_count < 1:
            raise InvalidInputError(f"worker count must be positive, got {worker_count}")
        total = n * (n - 1) // 2
        _, mult = np.unique(np.asarray(a, dtype=float), return_counts=True)
        parallel_pairs = int((mult * (mult - 1) // 2).sum())
        return cls(n=n, pair_count=total - parallel_pairs,
                   partition_size=max(1, math.ceil(total / worker_count)), worker_count=worker_count)

    def partitions(self) -> list[tuple[int, int]]:
        total = self.n * (self.n - 1) // 2
        return [(s, min(s + self.partition_size, total)) for s in range(0, total, self.partition_size)]


def resolve_workers(workers: int | None) -> int:
    """Explicit argument, else ``LMSLINE_WORKERS``, else the CPU count (backend.py:95-108)."""
    if workers is None:
        env = os.environ.get(WORKERS_ENV_VAR)
        if env is not None:
            try:
                workers = int(env)
            except ValueError as exc:
                raise InvalidInputError(f"{WORKERS_ENV_VAR} must be an integer, got {env!r}") from exc
        else:
            workers = os.cpu_count() or 1
    if workers < 1:
        raise InvalidInputError(f"worker count must be positive, got {workers}")
    return workers


def merge(best: CandidateRecord | None, cand: CandidateRecord | None) -> CandidateRecord | None:
    """Strict lexicographic (height, i, j) minimum (backend.py:182-187)."""
    if cand is None:
        return best
    if best is None or cand.sort_key < best.sort_key:
        return cand
    return best


def solve_range(a: np.ndarray, b: np.ndarray, q: int, rank_begin: int, rank_end: int,
                device: int = 0, materialize: bool = False) -> CandidateRecord | None:
    """Exact minimum over one contiguous rank range on one GPU."""
    if materialize:
        return record_from_native(_native.min_bracelet_materialized(a, b, q, rank_begin, rank_end,
                                                                    device))
    return record_from_native(_native.min_bracelet(a, b, q, rank_begin, rank_end, device))


class SequentialBackend:
    """Whole rank range on one GPU."""

    name = "seq"

    def minimum_bracelet(self, a: np.ndarray, b: np.ndarray, q: int, *,
                         materialize: bool = False) -> CandidateRecord | None:
        n = int(a.size)
        return solve_range(a, b, q, 0, n * (n - 1) // 2, 0, materialize)


class ParallelBackend:
    """Contiguous rank partitions over the visible GPUs, merged exactly."""

    name = "par"

    def __init__(self, workers: int | None = None):
        self.workers = resolve_workers(workers)

    def minimum_bracelet(self, a: np.ndarray, b: np.ndarray, q: int, *,
                         materialize: bool = False) -> CandidateRecord | None:
        devices = max(1, min(self.workers, _native.device_count()))
        # LMSB_PAR_SHARDS: shard count of the sharded band search (tests run
        # several shards on one GPU); by default one per visible device
        shards = _env_shards(devices)
        plan = BatchPlan.create(a, devices)
        parts = plan.partitions()
        if shards > 1 and not materialize:
            return _sharded_search(a, b, q, shards, devices)
        if len(parts) <= 1:
            return solve_range(a, b, q, *parts[0], 0, materialize) if parts else None
        with ThreadPoolExecutor(max_workers=len(parts)) as pool:
            results = list(pool.map(lambda kp: solve_range(a, b, q, kp[1][0], kp[1][1], kp[0] % devices,
                                                           materialize),
                                    enumerate(parts)))
        best: CandidateRecord | None = None
        for rec in results:
            best = merge(best, rec)
        return best


def _env_shards(devices: int) -> int:
    raw = os.environ.get("LMSB_PAR_SHARDS")
    if raw is None:
        return devices
    try:
        shards = int(raw)
    except ValueError:
        raise InvalidInputError(f"LMSB_PAR_SHARDS must be an integer, got {raw!r}") from None
    if shards < 1:
        raise InvalidInputError(f"LMSB_PAR_SHARDS must be positive, got {shards}")
    return shards


def _sharded_search(a: np.ndarray, b: np.ndarray, q: int, shards: int,
                    devices: int) -> CandidateRecord | None:
    """The sharded band search over the visible GPUs of this process
    (lms_min_bracelet_multi): shard r on GPU r % devices, one host thread per
    shard inside the library, NCCL between distinct GPUs; each shard bounds
    and seeds its own slice of the slope bands, the seed records are
    all-gathered, each shard searches its own bands, and the records are
    all-gathered and merged (backend.py:182-187).  Same record as one solve."""
    return record_from_native(_native.min_bracelet_multi(a, b, q, [r % devices for r in range(shards)]))


_BACKENDS = {"seq": SequentialBackend, "par": ParallelBackend}


def get_backend(name: str, workers: int | None = None) -> SequentialBackend | ParallelBackend:
    """Backend by name, ``seq`` or ``par`` (backend.py:295-303)."""
    try:
        cls = _BACKENDS[name]
    except KeyError:
        raise InvalidInputError(f"unknown backend {name!r}; expected one of {sorted(_BACKENDS)}") from None
    if cls is ParallelBackend:
        return ParallelBackend(workers)
    return SequentialBackend()


def run_phase1(lines: Sequence[DualLine]) -> Iterator[DualIntersection]:
    """All non-parallel dual crossings in row-major pair order (backend.py:306-318)."""
    n = len(lines)
    for i in range(n - 1):
        for j in range(i + 1, n):
            ip = pair_intersection(lines[i], lines[j])
            if ip is not None:
                yield ip


def run_phase2(intersections: Iterable[DualIntersection], lines: Sequence[DualLine], q: int,
               worker_count: int = 1) -> CandidateRecord:
    """Exact (height, i, j) minimum over the given crossings on the GPU (backend.py:321-354)."""
    ips = list(intersections)
    if not ips:
        raise InvalidInputError("phase 2 needs at least one intersection")
    if not 2 <= q <= len(lines):
        raise InvalidInputError(f"coverage must satisfy 2 <= q <= {len(lines)}, got {q}")
    if worker_count < 1:
        raise InvalidInputError(f"worker count must be positive, got {worker_count}")
    a = np.fromiter((ln.a for ln in lines), dtype=float, count=len(lines))
    b = np.fromiter((ln.b for ln in lines), dtype=float, count=len(lines))
    ii = np.fromiter((ip.i for ip in ips), dtype=np.int64, count=len(ips))
    jj = np.fromiter((ip.j for ip in ips), dtype=np.int64, count=len(ips))
    uu = np.fromiter((ip.u for ip in ips), dtype=float, count=len(ips))
    best = record_from_native(_native.min_over_vertices(a, b, q, ii, jj, uu))
    if best is None:
        raise InvalidInputError(f"no window of coverage {q} fits {len(lines)} lines")
    return best
