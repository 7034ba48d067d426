"""ctypes binding of the sm_100a C-ABI library (``_lib/liblmsb200.so``).

This is the only path from Python to the engine: there is no CPU fallback.
If the library is missing, or no CUDA device is visible, every call raises
``NativeUnavailableError`` (a ``RuntimeError``) instead of computing
anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from ._build import LIB_PATH

LMS_OK = 0
LMS_ERR_INVALID = -1
LMS_ERR_CUDA = -2
LMS_ERR_NODEVICE = -3
LMS_ERR_NOMEM = -4


class NativeUnavailableError(RuntimeError):
    """The CUDA engine cannot run here (library not built or no GPU)."""


class EngineError(RuntimeError):
    """A CUDA runtime failure inside the engine."""


class Candidate(ctypes.Structure):
    """lms_candidate (include/lms_b200.h)."""

    @classmethod
    def of(cls, rec) -> "Candidate":
        """From a CandidateRecord (None: not found)."""
        if rec is None:
            return cls()
        return cls(height=rec.height, u=rec.u, v_low=rec.v_low, v_high=rec.v_high, i=rec.i, j=rec.j,
                   found=1)

    _fields_ = [
        ("height", ctypes.c_double),
        ("u", ctypes.c_double),
        ("v_low", ctypes.c_double),
        ("v_high", ctypes.c_double),
        ("i", ctypes.c_int64),
        ("j", ctypes.c_int64),
        ("found", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    """lms_stats (include/lms_b200.h)."""

    _fields_ = [
        ("n", ctypes.c_int64),
        ("pairs", ctypes.c_int64),
        ("seed_vertices", ctypes.c_int64),
        ("filtered_vertices", ctypes.c_int64),
        ("survivors", ctypes.c_int64),
        ("line_evals", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("chunks", ctypes.c_int64),
        ("ms_total", ctypes.c_float),
        ("ms_filter", ctypes.c_float),
        ("ms_exact", ctypes.c_float),
        ("ms_bound_kernel", ctypes.c_float),
        ("bands", ctypes.c_int64),
        ("bands_searched", ctypes.c_int64),
        ("ms_partition", ctypes.c_float),
        ("ms_bound", ctypes.c_float),
        ("ms_band_filter", ctypes.c_float),
        ("ms_collect", ctypes.c_float),
        ("seed_height", ctypes.c_double),
        ("band_survivors", ctypes.c_int64),
        ("small_fits", ctypes.c_int64),
        ("direct_groups", ctypes.c_int64),
        ("bands_refined", ctypes.c_int64),
        ("sweep_runs", ctypes.c_int64),
        ("ms_filter_kernel", ctypes.c_float),
        ("ms_sweep_enum", ctypes.c_float),
        ("ms_hough_vote", ctypes.c_float),
        ("ms_hough_support", ctypes.c_float),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_ if not name.startswith("reserved")}


MAX_BANDS = 16384       # kBandMaxK (lms_band.cuh)
BAND_EDGE_KEYS = 10     # LMS_BAND_EDGE_KEYS
BAND_TABLE_COLS = 2 + BAND_EDGE_KEYS // 2


def pack_band_table(lb, wq, edge) -> np.ndarray:
    """(m, BAND_TABLE_COLS) float64 rows: lb, wq, then the fp32 edge keys' bytes."""
    m = len(lb)
    t = np.empty((m, BAND_TABLE_COLS), dtype=np.float64)
    t[:, 0] = lb
    t[:, 1] = wq
    t[:, 2:] = np.ascontiguousarray(edge, dtype=np.float32).reshape(m, BAND_EDGE_KEYS).view(np.float64)
    return t


def unpack_band_table(table):
    t = np.ascontiguousarray(table, dtype=np.float64).reshape(-1, BAND_TABLE_COLS)
    lb = np.ascontiguousarray(t[:, 0])
    wq = np.ascontiguousarray(t[:, 1])
    edge = np.ascontiguousarray(t[:, 2:]).view(np.float32).reshape(len(t), BAND_EDGE_KEYS)
    return lb, wq, np.ascontiguousarray(edge)


_lib = None
_lock = threading.Lock()

# The Hough entry points keep the points of the last vote on the device and
# lms_hough_support reads them, so a vote and the support gather that follows
# it must not interleave with another thread's vote on the same device: every
# Hough call holds the device's re-entrant lock, and callers that chain a
# vote and a gather (detect_lines, supporting_points) hold it across both.
_hough_locks: dict = {}


def hough_lock(device: int = 0) -> threading.RLock:
    with _lock:
        lk = _hough_locks.get(int(device))
        if lk is None:
            lk = _hough_locks[int(device)] = threading.RLock()
        return lk

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)
_C = ctypes.POINTER(Candidate)

# name -> (restype, argtypes); every symbol include/lms_b200.h declares.
SIGNATURES = {
    "lms_version": (ctypes.c_int, []),
    "lms_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "lms_last_error": (ctypes.c_char_p, []),
    "lms_min_bracelet_f64": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int, _C]),
    "lms_min_bracelet_materialized_f64": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64,
                                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                                         _C]),
    "lms_solve_fit_f64": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _C, _I,
                                         ctypes.c_int64, _I]),
    "lms_batched_f64": (ctypes.c_int, [_D, _D, _I, _I, ctypes.c_int64, ctypes.c_int, _C]),
    "lms_batched_fit_f64": (ctypes.c_int, [_D, _D, _I, _I, ctypes.c_int64, ctypes.c_int, _C,
                                           ctypes.POINTER(ctypes.c_uint8)]),
    "lms_primal_brute_f64": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _C]),
    "lms_hough_vote_u8": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                         _D, _D, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int64, ctypes.c_int, _I, _I]),
    "lms_hough_vote_points": (ctypes.c_int, [_D, _D, ctypes.c_int64, _D, _D, ctypes.c_int64,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_int64,
                                             ctypes.c_int, _I]),
    "lms_hough_support": (ctypes.c_int, [_D, _D, _I, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int64, ctypes.c_int, _I, _I, ctypes.c_int64]),
    "lms_hough_support_i32": (ctypes.c_int, [_D, _D, _I, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_int64, ctypes.c_int, _I,
                                             ctypes.POINTER(ctypes.c_int32), ctypes.c_int64]),
    "lms_eval_vertices_f64": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64, _I, _I, _D, _D,
                                             ctypes.c_int64, ctypes.c_int, _C]),
    "lms_min_over_vertices_f64": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64, _I, _I, _D,
                                                 ctypes.c_int64, ctypes.c_int, _C]),
    "lms_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "lms_ctx_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "lms_ctx_upload": (ctypes.c_int, [ctypes.c_void_p, _D, _D, ctypes.c_int64]),
    "lms_ctx_bind_dev": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64]),
    "lms_ctx_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     _C]),
    "lms_ctx_solve_materialized": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                                  ctypes.c_int64, _C]),
    "lms_ctx_solve_batch": (ctypes.c_int, [ctypes.c_void_p, _I, _I, ctypes.c_int64, _C]),
    "lms_ctx_shard_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int64, _I, _I, _D, _D,
                                          ctypes.POINTER(ctypes.c_float), _C]),
    "lms_ctx_shard_search": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_int64, _D, _D,
                                            ctypes.POINTER(ctypes.c_float), _C, _C]),
    "lms_ctx_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Stats)]),
    "lms_ctx_event_record": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "lms_ctx_event_elapsed_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(ctypes.c_float)]),
    "lms_ctx_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "lms_min_bracelet_multi": (ctypes.c_int, [_D, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                              ctypes.POINTER(ctypes.c_int32), _C]),
    "lms_nccl_available": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "lms_nccl_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8)]),
    "lms_ctx_comm_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_uint8)]),
    "lms_ctx_solve_distributed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _C]),
    "lms_ctx_shard_search_owned": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                                  ctypes.c_int32, _C, _C]),
    "lms_detect_peaks_u8": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                           _D, _D, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                           _I, _I, _I, _I]),
    "lms_detect_supports_u8": (ctypes.c_int, [_D, _D, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int64, _I,
                                              ctypes.c_int, ctypes.c_int, _I,
                                              ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, _I, _D, _C,
                                              ctypes.POINTER(ctypes.c_uint8)]),
    "lms_device_stats": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(Stats)]),
    "lms_batched_fit_sets_f64": (ctypes.c_int, [ctypes.c_void_p, _I, _I, ctypes.c_int64, ctypes.c_int,
                                                ctypes.POINTER(ctypes.c_int32), _C, _I,
                                                ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, _I]),
    "lms_ndarray_rows_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, _I]),
    "lms_probe_fp64_rate": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "lms_probe_fp32_rate": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "lms_debug_seg_sort": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "lms_debug_sample_sort": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]),
}


def load_library():
    """Load and bind the library (no device needed for loading)."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("LMSB_LIB_PATH", LIB_PATH)  # dev override for A/B builds
            if not os.path.exists(path):
                raise NativeUnavailableError(
                    f"CUDA engine library not built: {path} is missing "
                    "(run __graft_entry__.build() or python -m paper_1510_01041_b200._build)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def device_count() -> int:
    n = ctypes.c_int(0)
    load_library().lms_device_count(ctypes.byref(n))
    return n.value


def _lib_ready():
    lib = load_library()
    if device_count() == 0:
        raise NativeUnavailableError("no CUDA device visible; the exact-LMS engine runs only on the GPU")
    return lib


def check(rc: int) -> None:
    if rc == LMS_OK:
        return
    msg = load_library().lms_last_error().decode(errors="replace")
    if rc == LMS_ERR_INVALID:
        from .geometry import InvalidInputError

        raise InvalidInputError(msg)
    if rc == LMS_ERR_NODEVICE:
        raise NativeUnavailableError(msg)
    raise EngineError(f"engine error {rc}: {msg}")


def _dp(x: np.ndarray):
    return x.ctypes.data_as(_D)


def _ip(x: np.ndarray):
    return x.ctypes.data_as(_I)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int64)


def min_bracelet(a, b, q: int, rank_begin: int, rank_end: int, device: int = 0) -> Candidate:
    lib = _lib_ready()
    a = _f64(a)
    b = _f64(b)
    out = Candidate()
    check(lib.lms_min_bracelet_f64(_dp(a), _dp(b), a.size, int(q), int(rank_begin), int(rank_end),
                                   int(device), ctypes.byref(out)))
    return out


def device_stats(device: int = 0) -> dict:
    """lms_device_stats: counters of the last call on the device's shared context."""
    s = Stats()
    check(_lib_ready().lms_device_stats(int(device), ctypes.byref(s)))
    return s.as_dict()


def min_bracelet_multi(a, b, q: int, devices) -> Candidate:
    """lms_min_bracelet_multi: one fit sharded over len(devices) shards, shard r
    on GPU devices[r] (NCCL between distinct GPUs, host exchange otherwise)."""
    lib = _lib_ready()
    a = _f64(a)
    b = _f64(b)
    dv = np.ascontiguousarray(devices, dtype=np.int32)
    out = Candidate()
    check(lib.lms_min_bracelet_multi(_dp(a), _dp(b), a.size, int(q), dv.size,
                                     dv.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(out)))
    return out


def nccl_available() -> tuple[bool, int]:
    """(libnccl.so.2 loadable, its version code)."""
    v = ctypes.c_int(0)
    ok = load_library().lms_nccl_available(ctypes.byref(v))
    return bool(ok), v.value


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0 of a torchrun job makes it)."""
    buf = (ctypes.c_uint8 * 128)()
    check(load_library().lms_nccl_unique_id(buf))
    return bytes(buf)


def solve_fit(a, b, q: int, device: int = 0):
    """lms_solve_fit_f64: the record over all pairs and its contact indices
    (ascending int64 array), or (not-found record, empty array)."""
    lib = _lib_ready()
    a = _f64(a)
    b = _f64(b)
    out = Candidate()
    cap = 64
    while True:
        idx = np.empty(cap, dtype=np.int64)
        cnt = ctypes.c_int64()
        check(lib.lms_solve_fit_f64(_dp(a), _dp(b), a.size, int(q), int(device), ctypes.byref(out),
                                    idx.ctypes.data_as(_I), cap, ctypes.byref(cnt)))
        if cnt.value <= cap:
            return out, idx[: cnt.value]
        cap = int(cnt.value)


def min_bracelet_materialized(a, b, q: int, rank_begin: int, rank_end: int,
                              device: int = 0) -> Candidate:
    """lms_min_bracelet_materialized_f64: the two-kernel K1/K2 flow."""
    lib = _lib_ready()
    a = _f64(a)
    b = _f64(b)
    out = Candidate()
    check(lib.lms_min_bracelet_materialized_f64(_dp(a), _dp(b), a.size, int(q), int(rank_begin),
                                                int(rank_end), int(device), ctypes.byref(out)))
    return out


def batched_fit(x, y, offsets, q, device: int = 0):
    """lms_batched_fit_f64: the records and one contact flag per point."""
    lib = _lib_ready()
    x, y = _f64(x), _f64(y)
    offsets, q = _i64(offsets), _i64(q)
    nfits = offsets.size - 1
    out = (Candidate * max(nfits, 1))()
    flags = np.zeros(max(int(offsets[-1]), 1), dtype=np.uint8)
    check(lib.lms_batched_fit_f64(_dp(x), _dp(y), _ip(offsets), _ip(q), nfits, int(device), out,
                                  flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
    return out, flags[: int(offsets[-1])]


CANDIDATE_DTYPE = np.dtype([("height", "<f8"), ("u", "<f8"), ("v_low", "<f8"), ("v_high", "<f8"),
                            ("i", "<i8"), ("j", "<i8"), ("found", "<i4"), ("reserved", "<i4")])


def candidates_array(out, count: int) -> np.ndarray:
    """A ctypes lms_candidate array as a numpy structured array (copied)."""
    assert ctypes.sizeof(Candidate) == CANDIDATE_DTYPE.itemsize
    return np.frombuffer(out, dtype=CANDIDATE_DTYPE, count=count).copy()


def batched_fit_sets(sets, q, device: int = 0):
    """lms_batched_fit_sets_f64 over a list of C-contiguous (n, 2) float64
    arrays -> (status int32[F], records structured[F] or None, contact
    offsets int64[F + 1], contacts int32).  status all zero: fitted."""
    lib = _lib_ready()
    F = len(sets)
    objs = np.fromiter(map(id, sets), dtype=np.uintp, count=F)
    ptrs = np.empty(F, dtype=np.uintp)
    rows = np.empty(F, dtype=np.int64)
    check(lib.lms_ndarray_rows_f64(objs.ctypes.data, F, ptrs.ctypes.data, _ip(rows)))
    qv = np.ascontiguousarray(q, dtype=np.int64)
    status = np.zeros(F, dtype=np.int32)
    out = (Candidate * max(F, 1))()
    coff = np.zeros(F + 1, dtype=np.int64)
    total = int(rows.sum())
    contacts = np.empty(max(total, 1), dtype=np.int32)
    ncon = ctypes.c_int64(0)
    rc = lib.lms_batched_fit_sets_f64(ptrs.ctypes.data, _ip(rows), _ip(qv), F, int(device),
                                      status.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), out, _ip(coff),
                                      contacts.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), total,
                                      ctypes.byref(ncon))
    if rc == LMS_NOT_FITTED:
        return status, None, coff, contacts[:0]
    check(rc)
    return status, candidates_array(out, F), coff, contacts[: ncon.value]


def batched(x, y, offsets, q, device: int = 0) -> list:
    """lms_batched_f64: one exact LMS record per fit [offsets[f], offsets[f+1])."""
    lib = _lib_ready()
    x, y = _f64(x), _f64(y)
    offsets, q = _i64(offsets), _i64(q)
    nf = q.size
    out = (Candidate * max(nf, 1))()
    check(lib.lms_batched_f64(_dp(x), _dp(y), _ip(offsets), _ip(q), nf, int(device), out))
    return [out[k] for k in range(nf)]


def primal_brute(x, y, q: int, device: int = 0) -> Candidate:
    """lms_primal_brute_f64 (oracle_lms, solver.py:143-196)."""
    lib = _lib_ready()
    x, y = _f64(x), _f64(y)
    out = Candidate()
    check(lib.lms_primal_brute_f64(_dp(x), _dp(y), x.size, int(q), int(device), ctypes.byref(out)))
    return out


def _hough_vote_image_locked(img, threshold: int, cos_t, sin_t, rho_max: float, delta_rho: float,
                     n_rho: int, device: int = 0):
    """lms_hough_vote_u8 -> (acc int64[n_rho, n_theta], number of lit pixels)."""
    lib = _lib_ready()
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    cos_t, sin_t = _f64(cos_t), _f64(sin_t)
    n_theta = cos_t.size
    acc = np.zeros((n_rho, n_theta), dtype=np.int64)
    npts = ctypes.c_int64(0)
    check(lib.lms_hough_vote_u8(img.ctypes.data_as(ctypes.c_void_p), h, w, int(threshold), _dp(cos_t),
                                _dp(sin_t), n_theta, float(rho_max), float(delta_rho), int(n_rho),
                                int(device), _ip(acc), ctypes.byref(npts)))
    return acc, npts.value


def _hough_vote_points_locked(x, y, cos_t, sin_t, rho_max: float, delta_rho: float, n_rho: int,
                      device: int = 0) -> np.ndarray:
    """lms_hough_vote_points -> acc int64[n_rho, n_theta]."""
    lib = _lib_ready()
    x, y, cos_t, sin_t = _f64(x), _f64(y), _f64(cos_t), _f64(sin_t)
    n_theta = cos_t.size
    acc = np.zeros((n_rho, n_theta), dtype=np.int64)
    check(lib.lms_hough_vote_points(_dp(x), _dp(y), x.size, _dp(cos_t), _dp(sin_t), n_theta,
                                    float(rho_max), float(delta_rho), int(n_rho), int(device), _ip(acc)))
    return acc


def _hough_support_locked(cos_p, sin_p, rbin_p, rho_max: float, delta_rho: float, n_rho: int,
                  capacity: int, device: int = 0, narrow: bool = False):
    """lms_hough_support on the last vote's points -> (offsets[P+1], ids);
    narrow=True: int32 ids through lms_hough_support_i32 (half the download)."""
    lib = _lib_ready()
    cos_p, sin_p, rbin_p = _f64(cos_p), _f64(sin_p), _i64(rbin_p)
    npk = cos_p.size
    offsets = np.zeros(npk + 1, dtype=np.int64)
    if narrow:
        out = np.empty(max(int(capacity), 1), dtype=np.int32)
        rc = lib.lms_hough_support_i32(_dp(cos_p), _dp(sin_p), _ip(rbin_p), npk, float(rho_max),
                                       float(delta_rho), int(n_rho), int(device), _ip(offsets),
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       int(capacity))
    else:
        out = np.empty(max(int(capacity), 1), dtype=np.int64)
        rc = lib.lms_hough_support(_dp(cos_p), _dp(sin_p), _ip(rbin_p), npk, float(rho_max),
                                   float(delta_rho), int(n_rho), int(device), _ip(offsets), _ip(out),
                                   int(capacity))
    if rc == LMS_ERR_INVALID and offsets[-1] > capacity:
        return _hough_support_locked(cos_p, sin_p, rbin_p, rho_max, delta_rho, n_rho,
                                     int(offsets[-1]), device, narrow)
    check(rc)
    return offsets, out[: offsets[-1]]


LMS_NOT_FITTED = 1
DETECT_MAX_BINS = 16384
DETECT_MAX_PEAKS = 64


def detect_peaks(img, threshold: int, cos_t, sin_t, rho_max: float, delta_rho: float, n_rho: int,
                 max_peaks: int, min_votes: int, device: int = 0, want_acc: bool = False):
    """lms_detect_peaks_u8 -> (npoints, peaks int64[P, 3] (rho_bin, theta_bin, votes), acc or None).
    Hold hough_lock(device) from here through detect_supports."""
    lib = _lib_ready()
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    cos_t, sin_t = _f64(cos_t), _f64(sin_t)
    n_theta = cos_t.size
    acc = np.zeros((n_rho, n_theta), dtype=np.int64) if want_acc else None
    npts, npk = ctypes.c_int64(0), ctypes.c_int64(0)
    peaks = np.zeros((DETECT_MAX_PEAKS, 3), dtype=np.int64)
    check(lib.lms_detect_peaks_u8(img.ctypes.data_as(ctypes.c_void_p), h, w, int(threshold), _dp(cos_t),
                                  _dp(sin_t), n_theta, float(rho_max), float(delta_rho), int(n_rho),
                                  int(max_peaks), int(min_votes), int(device),
                                  _ip(acc) if acc is not None else None, ctypes.byref(npts), _ip(peaks),
                                  ctypes.byref(npk)))
    return npts.value, peaks[: npk.value].copy(), acc


def detect_supports(cos_s, sin_s, swap_t, support_cap: int, q, fit: bool, npeaks: int, votes,
                    device: int = 0):
    """lms_detect_supports_u8 on the last detect_peaks -> dict with the support
    offsets and int32 pixel ids, the design offsets and abscissa ranges, and
    (fit and fitted) the records (structured array) and contact flags."""
    lib = _lib_ready()
    cos_s, sin_s = _f64(cos_s), _f64(sin_s)
    swap = np.ascontiguousarray(swap_t, dtype=np.uint8)
    votes = np.asarray(votes, dtype=np.int64)
    total = int(votes.sum())
    cap = int(support_cap or 0)
    keep = np.minimum(votes, cap) if cap > 0 else votes
    soffs = np.zeros(npeaks + 1, dtype=np.int64)
    doffs = np.zeros(npeaks + 1, dtype=np.int64)
    ids = np.empty(max(total, 1), dtype=np.int32)
    lim = np.zeros(2 * max(npeaks, 1), dtype=np.float64)
    recs = (Candidate * max(npeaks, 1))()
    flags = np.zeros(max(int(keep.sum()), 1), dtype=np.uint8)
    qv = np.ascontiguousarray(q if q is not None else np.zeros(npeaks), dtype=np.int64)
    rc = lib.lms_detect_supports_u8(_dp(cos_s), _dp(sin_s), swap.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                    cap, _ip(qv), 1 if fit else 0, int(device), _ip(soffs),
                                    ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), total, _ip(doffs),
                                    _dp(lim), recs, flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    if rc != LMS_NOT_FITTED:
        check(rc)
    fitted = bool(fit) and rc == 0
    return {"support_offsets": soffs, "ids": ids[:total], "design_offsets": doffs,
            "abscissa_range": lim[: 2 * npeaks].reshape(npeaks, 2), "fitted": fitted,
            "records": candidates_array(recs, npeaks) if fitted else None,
            "contact_flags": flags[: int(doffs[-1])] if fitted else None}


def hough_vote_image(img, threshold: int, cos_t, sin_t, rho_max: float, delta_rho: float,
                     n_rho: int, device: int = 0):
    """lms_hough_vote_u8 -> (acc int64[n_rho, n_theta], number of lit pixels)."""
    with hough_lock(device):
        return _hough_vote_image_locked(img, threshold, cos_t, sin_t, rho_max, delta_rho, n_rho, device)


def hough_vote_points(x, y, cos_t, sin_t, rho_max: float, delta_rho: float, n_rho: int,
                      device: int = 0) -> np.ndarray:
    """lms_hough_vote_points -> acc int64[n_rho, n_theta]."""
    with hough_lock(device):
        return _hough_vote_points_locked(x, y, cos_t, sin_t, rho_max, delta_rho, n_rho, device)


def hough_support(cos_p, sin_p, rbin_p, rho_max: float, delta_rho: float, n_rho: int,
                  capacity: int, device: int = 0, narrow: bool = False):
    """lms_hough_support on the last vote's points -> (offsets[P+1], ids)."""
    with hough_lock(device):
        return _hough_support_locked(cos_p, sin_p, rbin_p, rho_max, delta_rho, n_rho, capacity,
                                     device, narrow)


def eval_vertices(a, b, q: int, i, j, u, v=None, device: int = 0):
    lib = _lib_ready()
    a, b = _f64(a), _f64(b)
    i, j, u = _i64(i), _i64(j), _f64(u)
    m = i.size
    out = (Candidate * max(m, 1))()
    vp = None
    if v is not None:
        v = _f64(v)
        vp = _dp(v)
    check(lib.lms_eval_vertices_f64(_dp(a), _dp(b), a.size, int(q), _ip(i), _ip(j), _dp(u), vp, m,
                                    int(device), out))
    return [out[k] for k in range(m)]


def min_over_vertices(a, b, q: int, i, j, u, device: int = 0) -> Candidate:
    lib = _lib_ready()
    a, b = _f64(a), _f64(b)
    i, j, u = _i64(i), _i64(j), _f64(u)
    out = Candidate()
    check(lib.lms_min_over_vertices_f64(_dp(a), _dp(b), a.size, int(q), _ip(i), _ip(j), _dp(u), i.size,
                                        int(device), ctypes.byref(out)))
    return out


def probe_fp64_rate(device: int = 0) -> float:
    """Measured DFMA issue rate (per second) of the FP64 pipe on `device`."""
    lib = _lib_ready()
    r = ctypes.c_double(0.0)
    check(lib.lms_probe_fp64_rate(int(device), ctypes.byref(r)))
    return r.value


def probe_fp32_rate(device: int = 0) -> float:
    """Measured FP32 FMA lanes per second (FFMA2 chains) on `device`."""
    lib = _lib_ready()
    r = ctypes.c_double(0.0)
    check(lib.lms_probe_fp32_rate(int(device), ctypes.byref(r)))
    return r.value


def debug_seg_sort(keys: np.ndarray, seg_begin, seg_end, device: int = 0) -> np.ndarray:
    """The band stage's cluster segmented sort on host arrays (diagnostic)."""
    lib = _lib_ready()
    k = np.ascontiguousarray(keys, dtype=np.float32)
    out = np.empty_like(k)
    sb = _i64(seg_begin)
    se = _i64(seg_end)
    check(lib.lms_debug_seg_sort(int(device), k.ctypes.data, out.ctypes.data, k.size, sb.size,
                                 sb.ctypes.data, se.ctypes.data))
    return out


def debug_sample_sort(keys: np.ndarray, device: int = 0) -> np.ndarray:
    """The band stage's slope-sample bucket sort on a host array (diagnostic)."""
    lib = _lib_ready()
    k = np.ascontiguousarray(keys, dtype=np.float32)
    out = np.empty_like(k)
    check(lib.lms_debug_sample_sort(int(device), k.ctypes.data, out.ctypes.data, k.size))
    return out


class Context:
    """Device-resident solver context (lms_ctx): lines, scratch and a stream."""

    def __init__(self, device: int = 0):
        self._lib = _lib_ready()
        h = ctypes.c_void_p()
        check(self._lib.lms_ctx_create(int(device), ctypes.byref(h)))
        self._h = h
        self._keep = None

    def close(self):
        if self._h:
            self._lib.lms_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def upload(self, a, b):
        a, b = _f64(a), _f64(b)
        self._keep = (a, b)
        check(self._lib.lms_ctx_upload(self._h, _dp(a), _dp(b), a.size))

    def bind_device(self, d_a: int, d_b: int, n: int):
        check(self._lib.lms_ctx_bind_dev(self._h, ctypes.c_void_p(d_a), ctypes.c_void_p(d_b), int(n)))

    def solve(self, q: int, rank_begin: int, rank_end: int) -> Candidate:
        out = Candidate()
        check(self._lib.lms_ctx_solve(self._h, int(q), int(rank_begin), int(rank_end), ctypes.byref(out)))
        return out

    def shard_plan(self, q: int, nshards: int, shard: int):
        """Bounds of this shard's slice of the slope bands (lms_ctx_shard_plan).

        Returns ``(K, table, seed)``: ``table`` is a float64 array of shape
        ``(len(range(shard, K, nshards)), BAND_TABLE_COLS)``, one row per band
        shard, shard + nshards, ... (lower bound, narrowest q-window, then the
        window-edge keys, fp32 packed two per column); ``seed`` is the best
        vertex at the ends of the slice's narrowest windows (a Candidate).
        ``K == 0``: the fit is not searched by bands (no exchange needed).
        """
        cap = -(-MAX_BANDS // max(1, int(nshards)))
        lb = np.empty(cap, dtype=np.float64)
        wq = np.empty(cap, dtype=np.float64)
        edge = np.empty((cap, BAND_EDGE_KEYS), dtype=np.float32)
        K, m = ctypes.c_int64(), ctypes.c_int64()
        seed = Candidate()
        check(self._lib.lms_ctx_shard_plan(
            self._h, int(q), int(nshards), int(shard), cap, ctypes.byref(K), ctypes.byref(m),
            lb.ctypes.data_as(_D), wq.ctypes.data_as(_D),
            edge.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), ctypes.byref(seed)))
        m = m.value
        return K.value, pack_band_table(lb[:m], wq[:m], edge[:m]), seed

    def shard_search(self, q: int, nshards: int, shard: int, table, seed=None) -> Candidate:
        """Search this shard's rank range against the full band table (all K
        bands), starting from ``seed`` (the minimum of all shards' plan seeds)."""
        lb, wq, edge = unpack_band_table(table)
        out = Candidate()
        check(self._lib.lms_ctx_shard_search(
            self._h, int(q), int(nshards), int(shard), len(lb), lb.ctypes.data_as(_D),
            wq.ctypes.data_as(_D), edge.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
            ctypes.byref(seed) if seed is not None else None, ctypes.byref(out)))
        return out

    def shard_search_owned(self, q: int, nshards: int, shard: int, seed=None) -> Candidate:
        """Own-band search of this shard after its shard_plan on this context,
        with the best seed over all shards (lms_ctx_shard_search_owned)."""
        out = Candidate()
        check(self._lib.lms_ctx_shard_search_owned(self._h, int(q), int(nshards), int(shard),
                                                   ctypes.byref(seed) if seed is not None else None,
                                                   ctypes.byref(out)))
        return out

    def comm_init(self, nranks: int, rank: int, unique_id: bytes):
        """Bind an NCCL communicator (rank of nranks) to this context."""
        if len(unique_id) != 128:
            raise ValueError("an NCCL unique id has 128 bytes")
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        check(self._lib.lms_ctx_comm_init(self._h, int(nranks), int(rank), buf))

    def solve_distributed(self, q: int) -> Candidate:
        """The sharded band search of the bound lines over the communicator:
        plan, all-gather of seed records, own-band search, all-gather of the
        records; the same record on every rank."""
        out = Candidate()
        check(self._lib.lms_ctx_solve_distributed(self._h, int(q), ctypes.byref(out)))
        return out

    def solve_materialized(self, q: int, rank_begin: int, rank_end: int) -> Candidate:
        """The two-kernel K1/K2 flow (materialize=True) over the bound lines."""
        out = Candidate()
        check(self._lib.lms_ctx_solve_materialized(self._h, int(q), int(rank_begin), int(rank_end),
                                                   ctypes.byref(out)))
        return out

    def solve_batch(self, offsets, q) -> list:
        offsets, q = _i64(offsets), _i64(q)
        nf = q.size
        out = (Candidate * max(nf, 1))()
        check(self._lib.lms_ctx_solve_batch(self._h, _ip(offsets), _ip(q), nf, out))
        return [out[k] for k in range(nf)]

    def stats(self) -> dict:
        s = Stats()
        check(self._lib.lms_ctx_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def record(self, slot: int):
        check(self._lib.lms_ctx_event_record(self._h, int(slot)))

    def elapsed_ms(self, slot0: int, slot1: int) -> float:
        ms = ctypes.c_float(0.0)
        check(self._lib.lms_ctx_event_elapsed_ms(self._h, int(slot0), int(slot1), ctypes.byref(ms)))
        return float(ms.value)

    def synchronize(self):
        check(self._lib.lms_ctx_synchronize(self._h))
