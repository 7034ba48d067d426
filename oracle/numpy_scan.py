"""The reference's own scan, restated in numpy -- TEST INFRASTRUCTURE ONLY.

Timed as the CPU baseline of bench.py (``cpu_baseline`` and ``--impl
reference``); never imported by the product package.  The reference package
(pure Python + numpy) cannot be imported on the GPU box, so this module
reproduces its cost model operation for operation, not just its result:

* ``scan_rank_range`` follows ``_scan_rank_range`` (backend.py:190-207):
  chunks of ``4_000_000 // n`` pair ranks, ranks decoded through the row
  offsets with ``searchsorted`` (backend.py:111-122), parallel duals dropped,
  slopes ``(b_i - b_j) / (a_i - a_j)``;
* ``_chunk_best`` follows ``_evaluate_pairs`` (backend.py:125-179): the full
  (m, n) cut matrix, both anchors snapped, the two rank counts, a full row
  sort (``ndarray.sort``, numpy's introsort -- the reference's dominant
  cost), the two order statistics, the (height, i*n + j) chunk minimum;
* ``merge`` is ``_merge`` (backend.py:182-187);
* ``par_scan`` is ParallelBackend's fan-out (backend.py:264-289): the rank
  range in contiguous partitions on a thread pool (numpy releases the GIL in
  the sort and the elementwise kernels), merged in partition order.

``tests/test_cpu_port.py`` checks the records against the reference goldens;
profiles/r02_cpu_port_calibration.json compares its time with the reference
package's own ``_scan_rank_range`` on the same slices (measured in the build
container, where the reference is importable).
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK_ELEMENTS = 4_000_000  # backend.py:_CHUNK_ELEMENTS


def row_offsets(n: int) -> np.ndarray:
    """Rank of pair (i, i+1) for every row i of the upper triangle."""
    lengths = np.arange(n - 1, 0, -1, dtype=np.int64)
    out = np.zeros(n - 1, dtype=np.int64)
    if n > 2:
        out[1:] = np.cumsum(lengths[:-1])
    return out


def _chunk_best(a, b, ii, jj, u, q):
    """(height, i, j, u, v_low, v_high) of the best anchored window among the
    given vertices, or None."""
    m, n = ii.size, a.size
    if m == 0:
        return None
    anchor = a[ii] * u - b[ii]
    cut = u[:, None] * a[None, :] - b[None, :]
    r = np.arange(m)
    cut[r, ii] = anchor
    cut[r, jj] = anchor
    below = np.count_nonzero(cut < anchor[:, None], axis=1)
    upto = np.count_nonzero(cut <= anchor[:, None], axis=1) - 1
    cut.sort(axis=1)
    lo_rank = upto - (q - 1)
    hi_rank = below + (q - 1)
    lo_val = np.take_along_axis(cut, np.clip(lo_rank, 0, None)[:, None], axis=1)[:, 0]
    hi_val = np.take_along_axis(cut, np.clip(hi_rank, None, n - 1)[:, None], axis=1)[:, 0]
    h_lo = np.where(lo_rank >= 0, anchor - lo_val, np.inf)
    h_hi = np.where(hi_rank <= n - 1, hi_val - anchor, np.inf)
    upward = h_hi <= h_lo
    h = np.where(upward, h_hi, h_lo)
    ok = np.isfinite(h)
    if not ok.any():
        return None
    hmin = h[ok].min()
    cand = np.flatnonzero(h == hmin)
    w = cand[np.argmin(ii[cand] * np.int64(n) + jj[cand])]
    if upward[w]:
        lo, hi = float(anchor[w]), float(hi_val[w])
    else:
        lo, hi = float(lo_val[w]), float(anchor[w])
    return (float(h[w]), int(ii[w]), int(jj[w]), float(u[w]), lo, hi)


def merge(best, cand):
    """Lexicographic (height, i, j) minimum; the earlier one wins ties."""
    if cand is None:
        return best
    if best is None or cand[:3] < best[:3]:
        return cand
    return best


def scan_rank_range(a: np.ndarray, b: np.ndarray, q: int, start: int, stop: int):
    """The reference's streamed scan of pair ranks [start, stop)."""
    n = a.size
    offs = row_offsets(n)
    step = max(1, CHUNK_ELEMENTS // n)
    best = None
    for pos in range(start, stop, step):
        ranks = np.arange(pos, min(pos + step, stop), dtype=np.int64)
        ii = np.searchsorted(offs, ranks, side="right") - 1
        jj = ranks - offs[ii] + ii + 1
        keep = (a[ii] - a[jj]) != 0.0
        if keep.any():
            ik, jk = ii[keep], jj[keep]
            u = (b[ik] - b[jk]) / (a[ik] - a[jk])
            best = merge(best, _chunk_best(a, b, ik, jk, u, q))
    return best


def par_scan(a: np.ndarray, b: np.ndarray, q: int, ranges, workers: int):
    """Several rank ranges on a thread pool, merged in order."""
    with ThreadPoolExecutor(max_workers=max(1, workers)) as pool:
        recs = list(pool.map(lambda r: scan_rank_range(a, b, q, r[0], r[1]), ranges))
    best = None
    for rec in recs:
        best = merge(best, rec)
    return best
