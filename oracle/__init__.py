"""CPU oracle for the exact-LMS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and only
as the checker or the timed CPU baseline.  The product package
(``paper_1510_01041_b200``) never imports it.

It wraps ``lms_oracle.cpp`` (a C restatement of the reference's
``_scan_rank_range`` / ``_evaluate_pairs`` / ``_merge``, see the file header
for the file:line map) and restates the solver's primal mapping and contact
set (``solver.py:115-140``) in numpy, so that an oracle ``LmsFit`` can be
compared field by field with the product's.

Parity pinning: ``tests/test_oracle.py`` checks every function here against
the golden vectors that ``tests/golden/make_golden.py`` produced by running
the reference package itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liblmsoracle.so")
_lib = None

GEOM_EPS = 1e-9  # geometry.py:20


class OracleCandidate(ctypes.Structure):
    _fields_ = [
        ("height", ctypes.c_double),
        ("u", ctypes.c_double),
        ("v_low", ctypes.c_double),
        ("v_high", ctypes.c_double),
        ("i", ctypes.c_int64),
        ("j", ctypes.c_int64),
        ("found", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


def build() -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        cp = ctypes.POINTER(OracleCandidate)
        lib.oracle_min_bracelet.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int, cp]
        lib.oracle_eval_vertices.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int64, ip, ip, dp, dp,
                                             ctypes.c_int64, cp]
        lib.oracle_all_heights.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, dp]
        _lib = lib
    return _lib


def _dptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _iptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


@dataclass(frozen=True)
class Record:
    """Same fields as the reference's CandidateRecord (backend.py:37-54)."""

    height: float
    i: int
    j: int
    u: float
    v_low: float
    v_high: float


def _record(c: OracleCandidate) -> Record | None:
    if not c.found:
        return None
    return Record(c.height, int(c.i), int(c.j), c.u, c.v_low, c.v_high)


def min_bracelet(a, b, q: int, r0: int = 0, r1: int | None = None, threads: int = 1) -> Record | None:
    """minimum_bracelet over pair ranks [r0, r1) (backend.py:190-207, 264-289)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = a.size
    if r1 is None:
        r1 = n * (n - 1) // 2
    out = OracleCandidate()
    rc = _load().oracle_min_bracelet(_dptr(a), _dptr(b), n, q, r0, r1, threads, ctypes.byref(out))
    if rc != 0:
        raise ValueError("oracle_min_bracelet: invalid arguments")
    return _record(out)


def eval_vertices(a, b, q: int, i, j, u, v=None) -> list[Record | None]:
    """Per-vertex anchored windows (bracelet_at semantics when v is given)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    i = np.ascontiguousarray(i, dtype=np.int64)
    j = np.ascontiguousarray(j, dtype=np.int64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    m = i.size
    out = (OracleCandidate * max(m, 1))()
    vp = None
    if v is not None:
        v = np.ascontiguousarray(v, dtype=np.float64)
        vp = _dptr(v)
    rc = _load().oracle_eval_vertices(_dptr(a), _dptr(b), a.size, q, _iptr(i), _iptr(j), _dptr(u), vp, m, out)
    if rc != 0:
        raise ValueError("oracle_eval_vertices: invalid arguments")
    return [_record(out[k]) for k in range(m)]


def all_heights(a, b, q: int, r0: int = 0, r1: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = a.size
    if r1 is None:
        r1 = n * (n - 1) // 2
    h = np.empty(r1 - r0, dtype=np.float64)
    _load().oracle_all_heights(_dptr(a), _dptr(b), n, q, r0, r1, _dptr(h))
    return h


def fit_from_record(x: np.ndarray, y: np.ndarray, q: int, rec: Record) -> dict:
    """solve_lms' primal mapping and contact set (solver.py:122-140)."""
    slope = rec.u
    intercept = -(rec.v_low + rec.v_high) * 0.5
    half = (rec.v_high - rec.v_low) * 0.5
    vals = x * rec.u - y
    vals[[rec.i, rec.j]] = x[rec.i] * rec.u - y[rec.i]
    scale = max(1.0, float(np.max(np.abs(vals))))
    tol = GEOM_EPS * scale
    on_low = np.abs(vals - rec.v_low) <= tol
    on_high = np.abs(vals - rec.v_high) <= tol
    contacts = tuple(int(k) for k in np.flatnonzero(on_low | on_high))
    return {
        "slope": slope,
        "intercept": intercept,
        "lms_value": half * half,
        "slab_height": rec.v_high - rec.v_low,
        "coverage": q,
        "contact_indices": contacts,
    }


def solve(points, q: int | None = None, threads: int = 1) -> dict:
    """Oracle LMS fit of an (n, 2) array (validation per solver.py:67-80)."""
    pts = np.asarray(points, dtype=np.float64)
    x = np.ascontiguousarray(pts[:, 0])
    y = np.ascontiguousarray(pts[:, 1])
    n = x.size
    if q is None:
        q = n // 2 + 1
    rec = min_bracelet(x, y, q, threads=threads)
    if rec is None:
        raise ValueError("no candidate slab found")
    out = fit_from_record(x, y, q, rec)
    out["record"] = rec
    return out
