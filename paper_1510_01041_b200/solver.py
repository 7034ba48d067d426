"""Exact least-median-of-squares line fit (drop-in for lmsline.solver).

``solve_lms`` keeps the reference's signature, validation, errors and result
type (solver.py:45-140).  The pair search -- every arrangement vertex of the
dual lines, each vertex's anchored q-window, the lexicographic argmin -- runs
in the sm_100a engine; the host only validates, maps the winning record back
to the primal line and classifies the O(n) contact set exactly as
solver.py:122-133 does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import backend as _backend
from .geometry import GEOM_EPS, DegenerateInputError, InvalidInputError, LineEq, as_xy_arrays


@dataclass(frozen=True)
class LmsFit:
    """Result of an exact LMS fit (solver.py:45-59)."""

    line: LineEq
    lms_value: float
    slab_height: float
    coverage: int
    contact_indices: tuple[int, ...]


def default_coverage(n: int) -> int:
    """``n // 2 + 1``, a strict majority (solver.py:62-64)."""
    return n // 2 + 1


def validated(points, q: int | None) -> tuple[np.ndarray, np.ndarray, int]:
    """solver.py:67-80: >= 3 points, >= 2 distinct x, 2 <= q <= n."""
    x, y = as_xy_arrays(points)
    n = x.size
    if n < 3:
        raise DegenerateInputError(f"LMS needs at least 3 points, got {n}")
    if not x.min() < x.max():  # fewer than two distinct x (x is finite here)
        raise DegenerateInputError("all points share one x-coordinate; no non-vertical line fits")
    if q is None:
        q = default_coverage(n)
    if not 2 <= q <= n:
        raise InvalidInputError(f"coverage must satisfy 2 <= q <= {n}, got {q}")
    return x, y, q


def fit_from_record(x: np.ndarray, y: np.ndarray, q: int, rec: "_backend.CandidateRecord") -> LmsFit:
    """Primal line and contact set of the winning window (solver.py:122-140)."""
    half = (rec.v_high - rec.v_low) * 0.5
    cut = x * rec.u - y
    # the anchor pair sits exactly on the anchor ordinate, as in the search
    cut[[rec.i, rec.j]] = x[rec.i] * rec.u - y[rec.i]
    tol = GEOM_EPS * max(1.0, float(np.max(np.abs(cut))))
    touching = (np.abs(cut - rec.v_low) <= tol) | (np.abs(cut - rec.v_high) <= tol)
    return LmsFit(
        line=LineEq(slope=rec.u, intercept=-(rec.v_low + rec.v_high) * 0.5),
        lms_value=half * half,
        slab_height=rec.v_high - rec.v_low,
        coverage=q,
        contact_indices=tuple(int(k) for k in np.flatnonzero(touching)),
    )


def solve_lms(points, q: int | None = None, *, backend: str = "seq", workers: int | None = None,
              materialize: bool = False) -> LmsFit:
    """Exact LMS line fit (solver.py:83-140) on the GPU.

    Raises :class:`DegenerateInputError` for fewer than 3 points or a single
    x value, :class:`InvalidInputError` for non-finite input, a bad ``q``, an
    unknown backend or a bad worker count.
    """
    x, y, q = validated(points, q)
    engine = _backend.get_backend(backend, workers)
    if backend == "seq" and not materialize:
        # one device call: the search and the contact set (solver.py:115-140)
        from . import _native

        cand, contacts = _native.solve_fit(x, y, q)
        rec = _backend.record_from_native(cand)
        if rec is None:
            raise DegenerateInputError("no candidate slab found")
        half = (rec.v_high - rec.v_low) * 0.5
        return LmsFit(
            line=LineEq(slope=rec.u, intercept=-(rec.v_low + rec.v_high) * 0.5),
            lms_value=half * half,
            slab_height=rec.v_high - rec.v_low,
            coverage=q,
            contact_indices=tuple(contacts.tolist()),
        )
    rec = engine.minimum_bracelet(x, y, q, materialize=materialize)
    if rec is None:
        raise DegenerateInputError("no candidate slab found")
    return fit_from_record(x, y, q, rec)


def oracle_lms(points, q: int | None = None) -> LmsFit:
    """The reference's independent primal brute force (solver.py:143-196),
    evaluated on the GPU: every pair's slope, all its sorted intercepts, the
    narrowest q-window (first on ties); lexicographic (span, i, j) winner;
    the line through the window's midpoint.  Limited to n <= 16,384.
    """
    from . import _native

    x, y, q = validated(points, q)
    c = _native.primal_brute(x, y, q)
    if not c.found:
        raise DegenerateInputError("no candidate slope found")
    slope, c_low, c_high = c.u, c.v_low, c.v_high
    half = (c_high - c_low) * 0.5
    c_all = y - slope * x
    tol = GEOM_EPS * max(1.0, float(np.max(np.abs(c_all))))
    on_edge = (np.abs(c_all - c_low) <= tol) | (np.abs(c_all - c_high) <= tol)
    return LmsFit(
        line=LineEq(slope=slope, intercept=(c_low + c_high) * 0.5),
        lms_value=half * half,
        slab_height=c_high - c_low,
        coverage=q,
        contact_indices=tuple(int(k) for k in np.flatnonzero(on_edge)),
    )


def solve_lms_batch(point_sets, q=None) -> list[LmsFit]:
    """Exact LMS fits of many independent point sets in one GPU batch.

    The batched form of calling :func:`solve_lms` once per set (the
    reference's per-peak loop, detect.py:184-213): every set is validated as
    solve_lms validates it (solver.py:67-80) and its result is identical to
    ``solve_lms(points, q)``.  ``q`` is None (each set's default), an int
    (the same coverage for every set) or a sequence with one entry per set.
    """
    from . import _native
    from .backend import record_from_native

    sets = list(point_sets)
    if q is None or isinstance(q, (int, np.integer)):
        qs = [q] * len(sets)
    else:
        qs = list(q)
        if len(qs) != len(sets):
            raise InvalidInputError(f"got {len(qs)} coverages for {len(sets)} point sets")
    if not sets:
        return []
    if all(type(p) is np.ndarray and p.dtype == np.float64 and p.ndim == 2 and p.shape[1] == 2
           and p.flags.c_contiguous for p in sets):
        # the sets stay where they are: the library gathers them into pinned
        # staging and checks them on the device
        return _solve_sets(sets, qs, q)
    if all(isinstance(p, np.ndarray) and p.ndim == 2 and p.shape[1] == 2 and p.shape[0] > 0
           for p in sets):
        # fast path: (n, 2) arrays, validated all at once (same checks, same
        # order of the first failure)
        counts = np.array([p.shape[0] for p in sets], dtype=np.int64)
        offsets = np.zeros(len(sets) + 1, dtype=np.int64)
        offsets[1:] = np.cumsum(counts)
        X = np.concatenate([p[:, 0] for p in sets]).astype(float, copy=False)
        Y = np.concatenate([p[:, 1] for p in sets]).astype(float, copy=False)
        if not (np.isfinite(X).all() and np.isfinite(Y).all()):
            for pts, qq in zip(sets, qs):  # raises the first set's error, as the loop below
                validated(pts, qq)
        if q is None:
            qv = counts // 2 + 1
        elif isinstance(q, (int, np.integer)):
            qv = np.full(len(sets), int(q), dtype=np.int64)
        else:
            qv = np.array([default_coverage(int(c)) if qq is None else int(qq)
                           for c, qq in zip(counts, qs)], dtype=np.int64)
        return _solve_concat(X, Y, offsets, qv)
    xs, ys, qv = [], [], []
    for pts, qq in zip(sets, qs):
        x, y, qq = validated(pts, qq)
        xs.append(x)
        ys.append(y)
        qv.append(qq)
    offsets = np.zeros(len(sets) + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([x.size for x in xs])
    return _solve_concat(np.concatenate(xs), np.concatenate(ys), offsets,
                         np.asarray(qv, dtype=np.int64), checked=True)


def _solve_concat(X: np.ndarray, Y: np.ndarray, offsets: np.ndarray, q, *,
                  checked: bool = False) -> list[LmsFit]:
    """Batched solve of the sets X[offsets[k]:offsets[k+1]] (fp64, finite)
    with the solve_lms tail vectorised over all sets: the checks of
    validated() in set order unless already `checked`, one batched device
    call, then the contact sets of fit_from_record computed for every set at
    once with the same elementwise arithmetic (solver.py:122-140)."""
    from . import _native
    from .backend import record_from_native

    F = offsets.size - 1
    counts = np.diff(offsets)
    if q is None or isinstance(q, (int, np.integer)):
        qv = counts // 2 + 1 if q is None else np.full(F, int(q), dtype=np.int64)
    else:
        qv = np.asarray(q, dtype=np.int64)
    if not checked:
        # validated()'s checks per set, the first failing set reported
        small = counts < 3
        starts = np.minimum(offsets[:-1], max(X.size - 1, 0))
        lo = np.minimum.reduceat(X, starts) if X.size else np.zeros(F)
        hi = np.maximum.reduceat(X, starts) if X.size else np.zeros(F)
        bad_x = ~small & ~(lo < hi)
        bad_q = ~small & ~bad_x & ((qv < 2) | (qv > counts))
        if small.any() or bad_x.any() or bad_q.any():
            k = int(np.flatnonzero(small | bad_x | bad_q)[0])
            if counts[k] == 0:
                raise InvalidInputError("point set must be nonempty")
            if small[k]:
                raise DegenerateInputError(f"LMS needs at least 3 points, got {int(counts[k])}")
            if bad_x[k]:
                raise DegenerateInputError(
                    "all points share one x-coordinate; no non-vertical line fits")
            raise InvalidInputError(f"coverage must satisfy 2 <= q <= {int(counts[k])}, got {int(qv[k])}")
    # the records and, computed on the device with fit_from_record's
    # arithmetic, one contact flag per point; several visible GPUs share the
    # fits (contiguous groups, no collective: SURVEY section 8e row 2)
    cands, flags = _batched_fit_devices(X, Y, offsets, qv)
    if not bool(cands["found"].all()):
        raise DegenerateInputError("no candidate slab found")
    return _fits_from_arrays(cands, flags, offsets, qv)


def _solve_sets(sets, qs, q) -> list[LmsFit]:
    """solve_lms_batch over C-contiguous (n, 2) float64 arrays through
    lms_batched_fit_sets_f64 (split over the visible GPUs by contiguous
    groups of sets); errors as the per-set loop raises them."""
    from concurrent.futures import ThreadPoolExecutor

    from . import _native

    F = len(sets)
    counts = np.fromiter((p.shape[0] for p in sets), dtype=np.int64, count=F)
    if q is None:
        qv = counts // 2 + 1
    elif isinstance(q, (int, np.integer)):
        qv = np.full(F, int(q), dtype=np.int64)
    else:
        qv = np.array([default_coverage(int(c)) if qq is None else int(qq) for c, qq in zip(counts, qs)],
                      dtype=np.int64)
    visible = _native.device_count()
    if visible == 0:
        # no GPU: the same errors, checked on the host, before the library
        # reports that it cannot run
        for p, qq in zip(sets, qs):
            validated(p, qq)
    ndev = max(1, min(visible, F))
    bounds = np.linspace(0, F, ndev + 1).astype(int)

    def run(d):
        f0, f1 = int(bounds[d]), int(bounds[d + 1])
        return _native.batched_fit_sets(sets[f0:f1], qv[f0:f1], device=d)

    if ndev == 1:
        parts = [run(0)]
    else:
        with ThreadPoolExecutor(max_workers=ndev) as pool:
            parts = list(pool.map(run, range(ndev)))
    status = np.concatenate([p[0] for p in parts])
    bad = np.flatnonzero(status)
    if bad.size:
        k = int(bad[0])
        validated(sets[k], qs[k])  # raises the per-set loop's error for the first failing set
        raise DegenerateInputError("no candidate slab found")
    cands = np.concatenate([p[1] for p in parts])
    if not bool(cands["found"].all()):
        raise DegenerateInputError("no candidate slab found")
    coff = [parts[0][2]]
    for p in parts[1:]:
        coff.append(p[2][1:] + coff[-1][-1])
    coff = np.concatenate(coff)
    contacts = np.concatenate([p[3] for p in parts])
    return _fits_from_contacts(cands, coff, contacts, qv)


def _batched_fit_devices(X, Y, offsets, qv):
    """lms_batched_fit_f64 over the visible GPUs: fit groups with about equal
    point counts, one thread per device (the library releases the GIL), the
    records as a structured array and the per-point contact flags."""
    from concurrent.futures import ThreadPoolExecutor

    from . import _native

    F = offsets.size - 1
    ndev = max(1, min(_native.device_count(), F))
    if ndev == 1:
        out, flags = _native.batched_fit(X, Y, offsets, qv)
        return _native.candidates_array(out, F), flags
    # split points at fit boundaries near k / ndev of the total
    cuts = np.searchsorted(offsets, np.linspace(0, offsets[-1], ndev + 1)[1:-1])
    fb = np.unique(np.concatenate([[0], cuts, [F]]))

    def run(d):
        f0, f1 = int(fb[d]), int(fb[d + 1])
        p0, p1 = int(offsets[f0]), int(offsets[f1])
        out, fl = _native.batched_fit(X[p0:p1], Y[p0:p1], offsets[f0:f1 + 1] - p0, qv[f0:f1], device=d)
        return _native.candidates_array(out, f1 - f0), fl

    with ThreadPoolExecutor(max_workers=len(fb) - 1) as pool:
        parts = list(pool.map(run, range(len(fb) - 1)))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def _fits_from_contacts(cands, coff, contacts, qv) -> list[LmsFit]:
    """_fits_from_arrays with the contact sets already compacted (set-local
    ascending indices, contacts[coff[k] .. coff[k+1]))."""
    import gc

    F = coff.size - 1
    u, vl, vh = cands["u"], cands["v_low"], cands["v_high"]
    slope = u.tolist()
    intercept = (-(vl + vh) * 0.5).tolist()
    half = (vh - vl) * 0.5
    lms_value = (half * half).tolist()
    slab = (vh - vl).tolist()
    local = contacts.tolist()
    bounds = coff.tolist()
    cov = np.asarray(qv, dtype=np.int64).tolist()
    new = object.__new__
    fits = []
    was = gc.isenabled()
    gc.disable()
    try:
        for k in range(F):
            line = new(LineEq)
            d = line.__dict__
            d["slope"] = slope[k]
            d["intercept"] = intercept[k]
            fit = new(LmsFit)
            d = fit.__dict__
            d["line"] = line
            d["lms_value"] = lms_value[k]
            d["slab_height"] = slab[k]
            d["coverage"] = cov[k]
            d["contact_indices"] = tuple(local[bounds[k]:bounds[k + 1]])
            fits.append(fit)
    finally:
        if was:
            gc.enable()
    return fits


def _fits_from_arrays(cands, flags, offsets, qv) -> list[LmsFit]:
    """LmsFit objects of a batch from the record arrays: the solve_lms tail's
    arithmetic (solver.py:122-140) elementwise over all fits (same IEEE
    operations as the scalar form), contact sets from the device's flags;
    the objects are filled directly (the dataclasses stay frozen to users)
    with the cyclic GC paused while thousands are created."""
    import gc

    F = offsets.size - 1
    u, vl, vh = cands["u"], cands["v_low"], cands["v_high"]
    slope = u.tolist()
    intercept = (-(vl + vh) * 0.5).tolist()
    half = (vh - vl) * 0.5
    lms_value = (half * half).tolist()
    slab = (vh - vl).tolist()
    idx = np.flatnonzero(flags)
    owner = np.searchsorted(offsets, idx, side="right") - 1
    local = (idx - offsets[owner]).tolist()
    bounds = np.searchsorted(owner, np.arange(F + 1)).tolist()
    cov = np.asarray(qv, dtype=np.int64).tolist()
    new = object.__new__
    fits = []
    was = gc.isenabled()
    gc.disable()
    try:
        for k in range(F):
            line = new(LineEq)
            d = line.__dict__
            d["slope"] = slope[k]
            d["intercept"] = intercept[k]
            fit = new(LmsFit)
            d = fit.__dict__
            d["line"] = line
            d["lms_value"] = lms_value[k]
            d["slab_height"] = slab[k]
            d["coverage"] = cov[k]
            d["contact_indices"] = tuple(local[bounds[k]:bounds[k + 1]])
            fits.append(fit)
    finally:
        if was:
            gc.enable()
    return fits
