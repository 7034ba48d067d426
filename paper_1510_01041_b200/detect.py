"""Line detection: Hough peaks refined by LMS (drop-in for lmsline.detect).

``detect_lines`` keeps the reference's signature, methods and result type
(detect.py:156-214) but runs as one device pipeline: the image is uploaded
once, lit pixels are compacted and vote on the GPU, the (small) accumulator
comes back for ``find_peaks``, every peak's support is gathered on the GPU
in scan order, and all peaks' LMS refits run as ONE batched exact solve
(``solve_lms_batch``) instead of the reference's per-peak Python loop.
Supports are returned as :class:`SupportPoints`, a lazy, tuple-comparable
sequence of ``Point2`` backed by the pixel indices (the reference's
``tuple[Point2, ...]`` of ~30k objects per peak costs seconds to build).
"""

from __future__ import annotations

import math
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from .geometry import DegenerateInputError, InvalidInputError, LineEq, Point2
from .hough import (
    HoughAccumulator,
    HoughParams,
    Peak,
    find_peaks,
    line_to_polar,
    lit_mask_u8,
    needs_axis_swap,
    polar_to_frame_fit,
)
from .solver import _solve_concat, LmsFit, solve_lms, solve_lms_batch

METHOD_SHT = "sht"
METHOD_OLS = "ols"
METHOD_LMS = "lms"
METHODS = (METHOD_SHT, METHOD_OLS, METHOD_LMS)

DEFAULT_THRESHOLD = 128
DEFAULT_MIN_VOTES = 2

LMS_SUPPORT_CAP = 256
"""Support subsample size for the LMS refit (detect.py:43)."""


class SupportPoints(Sequence):
    """Lazy ``Point2`` sequence of one peak's support, in scan order.

    Compares equal to any sequence with the same points (so to the
    reference's tuples) and hashes like the equivalent tuple.
    """

    __slots__ = ("_xy", "_ids", "_width")

    def __init__(self, x: np.ndarray, y: np.ndarray):
        self._xy = (np.asarray(x, dtype=float), np.asarray(y, dtype=float))
        self._ids = None
        self._width = 0

    @classmethod
    def from_pixels(cls, ids: np.ndarray, width: int) -> "SupportPoints":
        """Backed by pixel indices (row-major, ``width`` columns); the float
        coordinates are formed on first use."""
        sp = cls.__new__(cls)
        sp._xy = None
        ids = np.asarray(ids)
        sp._ids = ids if ids.dtype in (np.int32, np.int64) else ids.astype(np.int64)
        sp._width = int(width)
        return sp

    @staticmethod
    def _pixel_xy(ids: np.ndarray, width: int) -> tuple[np.ndarray, np.ndarray]:
        row, col = np.divmod(ids, width)
        return col.astype(float), row.astype(float)

    @property
    def xy(self) -> tuple[np.ndarray, np.ndarray]:
        if self._xy is None:
            self._xy = self._pixel_xy(self._ids, self._width)
        return self._xy

    def thinned_xy(self, cap: int) -> tuple[np.ndarray, np.ndarray]:
        """Coordinates of the even-stride subsample (detect.py:118-131)
        without materialising the whole support."""
        m = len(self)
        if m <= cap:
            return self.xy
        idx = _subsample_index(m, cap)
        if self._xy is None:
            return self._pixel_xy(self._ids[idx], self._width)
        return self._xy[0][idx], self._xy[1][idx]

    def __len__(self) -> int:
        return int(self._ids.size if self._xy is None else self._xy[0].size)

    def __getitem__(self, k):
        x, y = self.xy
        if isinstance(k, slice):
            return SupportPoints(x[k], y[k])
        return Point2(float(x[k]), float(y[k]))

    def __iter__(self):
        x, y = self.xy
        for xv, yv in zip(x.tolist(), y.tolist()):
            yield Point2(xv, yv)

    def __eq__(self, other) -> bool:
        if isinstance(other, SupportPoints):
            (ax, ay), (bx, by) = self.xy, other.xy
            return np.array_equal(ax, bx) and np.array_equal(ay, by)
        if isinstance(other, Sequence) and not isinstance(other, (str, bytes)):
            return len(other) == len(self) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __hash__(self) -> int:
        return hash(tuple(self))

    def __repr__(self) -> str:
        return f"SupportPoints({len(self)} points)"


@dataclass(frozen=True)
class LineDetection:
    """One detected line (detect.py:52-88)."""

    method: str
    rho: float
    theta: float
    slope: float
    intercept: float
    axis_swapped: bool
    support: Sequence
    lms_value: float | None = None

    @property
    def image_slope(self) -> float:
        if not self.axis_swapped:
            return self.slope
        if self.slope == 0.0:
            return math.inf
        return 1.0 / self.slope

    @property
    def image_intercept(self) -> float:
        if not self.axis_swapped:
            return self.intercept
        if self.slope == 0.0:
            return math.nan
        return -self.intercept / self.slope


def _support_xy(support) -> tuple[np.ndarray, np.ndarray]:
    if isinstance(support, SupportPoints):
        return support.xy
    pts = list(support)
    x = np.fromiter((p.x for p in pts), dtype=float, count=len(pts))
    y = np.fromiter((p.y for p in pts), dtype=float, count=len(pts))
    return x, y


def _design_xy(x: np.ndarray, y: np.ndarray, axis_swapped: bool) -> tuple[np.ndarray, np.ndarray]:
    return (y, x) if axis_swapped else (x, y)


def refine_ols(support, axis_swapped: bool = False) -> LineEq:
    """Closed-form least squares in the given frame (detect.py:98-115)."""
    t, z = _design_xy(*_support_xy(support), axis_swapped)
    if t.size < 2:
        raise DegenerateInputError(f"least squares needs at least 2 points, got {t.size}")
    if not (np.isfinite(t).all() and np.isfinite(z).all()):
        raise InvalidInputError("support coordinates must be finite")
    t_mean = t.mean()
    z_mean = z.mean()
    dt = t - t_mean
    denom = float(dt @ dt)
    if denom == 0.0:
        raise DegenerateInputError("support is constant along the regression axis")
    slope = float(dt @ (z - z_mean)) / denom
    return LineEq(slope=slope, intercept=float(z_mean - slope * t_mean))


def _subsample_index(m: int, cap: int) -> np.ndarray:
    return (np.arange(cap, dtype=np.int64) * m) // cap


def subsample_support(support, cap: int):
    """Even-stride thinning to at most ``cap`` points, scan order kept
    (detect.py:118-131)."""
    pts = list(support)
    if cap < 3:
        raise InvalidInputError(f"support cap must be at least 3, got {cap}")
    m = len(pts)
    if m <= cap:
        return pts
    return [pts[int(k)] for k in _subsample_index(m, cap)]


def _thinned_xy(support, cap: int | None) -> tuple[np.ndarray, np.ndarray]:
    if cap is not None and cap < 3:
        raise InvalidInputError(f"support cap must be at least 3, got {cap}")
    if cap is not None and isinstance(support, SupportPoints):
        return support.thinned_xy(cap)
    x, y = _support_xy(support)
    if cap is not None:
        if x.size > cap:
            idx = _subsample_index(x.size, cap)
            x, y = x[idx], y[idx]
    return x, y


def refine_lms(support, q: int | None = None, axis_swapped: bool = False, *, backend: str = "seq",
               workers: int | None = None, support_cap: int | None = None) -> LmsFit:
    """Exact LMS line through the (optionally thinned) support in the given
    frame (detect.py:134-153)."""
    t, z = _design_xy(*_thinned_xy(support, support_cap), axis_swapped)
    return solve_lms(np.column_stack([t, z]), q, backend=backend, workers=workers)


def detect_lines(image: np.ndarray, params: HoughParams, method: str = METHOD_LMS, max_peaks: int = 1,
                 *, threshold: int = DEFAULT_THRESHOLD, min_votes: int = DEFAULT_MIN_VOTES,
                 q: int | None = None, backend: str = "seq", workers: int | None = None,
                 support_cap: int | None = LMS_SUPPORT_CAP) -> list[LineDetection]:
    """Detect up to ``max_peaks`` lines (detect.py:156-214) on the GPU."""
    from . import _native
    from .backend import get_backend

    if method not in METHODS:
        raise InvalidInputError(f"unknown method {method!r}; expected one of {METHODS}")
    img, thr = lit_mask_u8(image, threshold)
    if (params.n_rho * params.n_theta <= _native.DETECT_MAX_BINS and params.n_theta <= 512
            and params.n_rho <= 4095 and img.shape[1] <= 4096 * 32
            and 1 <= max_peaks <= _native.DETECT_MAX_PEAKS and min_votes >= 1 and img.size < 2**31):
        return _detect_on_device(img, thr, params, method, max_peaks, min_votes, q, backend, workers,
                                 support_cap)
    c, s = params.vote_trig()
    # the support gather reads the points the vote leaves on the device: one
    # lock across both, so another thread's vote cannot land in between
    with _native.hough_lock(0):
        bins, npoints = _native.hough_vote_image(img, thr, c, s, params.rho_max, params.delta_rho,
                                                 params.n_rho)
        if npoints == 0:
            return []
        peaks = find_peaks(HoughAccumulator(bins=bins, params=params), max_peaks, min_votes)
        if not peaks:
            return []
        trig = [params.support_trig(p.theta_bin) for p in peaks]
        # int32 pixel ids (half the download) whenever the image has < 2^31 pixels
        offsets, ids = _native.hough_support([t[0] for t in trig], [t[1] for t in trig],
                                             [p.rho_bin for p in peaks], params.rho_max,
                                             params.delta_rho, params.n_rho,
                                             capacity=sum(p.votes for p in peaks),
                                             narrow=img.size < 2**31)
    width = img.shape[1]
    supports = [SupportPoints.from_pixels(ids[offsets[k]: offsets[k + 1]], width)
                for k in range(len(peaks))]
    swapped = [needs_axis_swap(p.theta) for p in peaks]

    lms_fits: list[LmsFit] = []
    if method == METHOD_LMS:
        get_backend(backend, workers)  # same name / worker validation as solve_lms
        if support_cap is not None and support_cap < 3:
            raise InvalidInputError(f"support cap must be at least 3, got {support_cap}")
        # every peak's thinned design in one pair of arrays: the subsample
        # picks (detect.py:118-131) gathered from the pixel ids, decoded once
        picks = []
        for sup in supports:
            m = sup._ids.size
            picks.append(sup._ids if support_cap is None or m <= support_cap
                         else sup._ids[_subsample_index(m, support_cap)])
        counts = np.array([p.size for p in picks], dtype=np.int64)
        offsets = np.zeros(len(picks) + 1, dtype=np.int64)
        offsets[1:] = np.cumsum(counts)
        row, col = np.divmod(np.concatenate(picks), width)
        col = col.astype(float)
        row = row.astype(float)
        swap = np.repeat(np.array(swapped, dtype=bool), counts)
        T = np.where(swap, row, col)  # design frame: (y, x) when axis-swapped
        Z = np.where(swap, col, row)
        lms_fits = _solve_concat(T, Z, offsets, q)

    out: list[LineDetection] = []
    for k, (peak, sup, sw) in enumerate(zip(peaks, supports, swapped)):
        lms_value = None
        if method == METHOD_SHT:
            rho, theta = peak.rho, peak.theta
            slope, intercept, sw = polar_to_frame_fit(rho, theta)
        elif method == METHOD_OLS:
            fit = refine_ols(sup, sw)
            slope, intercept = fit.slope, fit.intercept
            rho, theta = line_to_polar(slope, intercept, sw)
        else:
            fit = lms_fits[k]
            slope, intercept = fit.line.slope, fit.line.intercept
            lms_value = fit.lms_value
            rho, theta = line_to_polar(slope, intercept, sw)
        out.append(LineDetection(method=method, rho=rho, theta=theta, slope=slope, intercept=intercept,
                                 axis_swapped=sw, support=sup, lms_value=lms_value))
    return out


def _detect_on_device(img, thr, params: HoughParams, method: str, max_peaks: int, min_votes: int,
                      q, backend, workers, support_cap) -> list[LineDetection]:
    """detect_lines with vote, find_peaks, support gather, stride thinning,
    axis-swapped designs and the batched LMS refits all on the device, from
    the image (lms_detect_peaks_u8 / lms_detect_supports_u8); the host keeps
    the polar maps and the result objects.  Errors as the reference's
    per-peak loop (detect.py:184-213): the first peak whose refit fails."""
    from . import _native
    from .backend import get_backend
    from .solver import _fits_from_arrays

    do_lms = method == METHOD_LMS
    if do_lms:
        get_backend(backend, workers)  # same name / worker validation as solve_lms
        if support_cap is not None and support_cap < 3:
            raise InvalidInputError(f"support cap must be at least 3, got {support_cap}")
    c, s = params.vote_trig()
    nt = params.n_theta
    with _native.hough_lock(0):
        npts, pk, _ = _native.detect_peaks(img, thr, c, s, params.rho_max, params.delta_rho, params.n_rho,
                                           max_peaks, min_votes)
        if npts == 0 or pk.shape[0] == 0:
            return []
        P = pk.shape[0]
        peaks = [Peak(rho_bin=int(r), theta_bin=int(t), votes=int(v), rho=params.rho_center(int(r)),
                      theta=params.theta_center(int(t))) for r, t, v in pk.tolist()]
        strig = [params.support_trig(t) for t in range(nt)]
        swap_t = [needs_axis_swap(params.theta_center(t)) for t in range(nt)]
        votes = pk[:, 2]
        cap = support_cap if (do_lms and support_cap is not None) else 0
        n_fit = np.minimum(votes, cap) if cap else votes
        qv = n_fit // 2 + 1 if q is None else np.full(P, int(q), dtype=np.int64)
        res = _native.detect_supports([a for a, _ in strig], [b for _, b in strig], swap_t, cap, qv,
                                      do_lms, P, votes)
    width = img.shape[1]
    soff, ids = res["support_offsets"], res["ids"]
    supports = [SupportPoints.from_pixels(ids[soff[k]: soff[k + 1]], width) for k in range(P)]
    swapped = [bool(swap_t[p.theta_bin]) for p in peaks]
    lms_fits = []
    if do_lms:
        if not res["fitted"]:
            doff, lim = res["design_offsets"], res["abscissa_range"]
            for k in range(P):  # the reference's loop stops at the first failing peak
                n = int(doff[k + 1] - doff[k])
                if n < 3:
                    raise DegenerateInputError(f"LMS needs at least 3 points, got {n}")
                if not lim[k, 0] < lim[k, 1]:
                    raise DegenerateInputError("all points share one x-coordinate; no non-vertical line fits")
                if not 2 <= int(qv[k]) <= n:
                    raise InvalidInputError(f"coverage must satisfy 2 <= q <= {n}, got {int(qv[k])}")
            raise DegenerateInputError("no candidate slab found")
        if not bool(res["records"]["found"].all()):
            raise DegenerateInputError("no candidate slab found")
        lms_fits = _fits_from_arrays(res["records"], res["contact_flags"], res["design_offsets"], qv)
    out: list[LineDetection] = []
    for k, (peak, sup, sw) in enumerate(zip(peaks, supports, swapped)):
        lms_value = None
        if method == METHOD_SHT:
            rho, theta = peak.rho, peak.theta
            slope, intercept, sw = polar_to_frame_fit(rho, theta)
        elif method == METHOD_OLS:
            fit = refine_ols(sup, sw)
            slope, intercept = fit.slope, fit.intercept
            rho, theta = line_to_polar(slope, intercept, sw)
        else:
            fit = lms_fits[k]
            slope, intercept = fit.line.slope, fit.line.intercept
            lms_value = fit.lms_value
            rho, theta = line_to_polar(slope, intercept, sw)
        out.append(LineDetection(method=method, rho=rho, theta=theta, slope=slope, intercept=intercept,
                                 axis_swapped=sw, support=sup, lms_value=lms_value))
    return out
