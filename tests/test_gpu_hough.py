"""GPU Hough vote / support / detect_lines against the reference's golden
vectors and, at config-5 scale, against the numpy oracle."""

import math

import numpy as np
import pytest

from oracle import hough_oracle
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import _native, workloads
from test_oracle_hough import f, image_of, load, params_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cases():
    assert _native.device_count() > 0
    return load()


def test_vote_points_and_support_match_reference(cases):
    for c in cases:
        p = params_of(c)
        pts = lms.extract_points(image_of(c))
        acc = lms.hough_vote(pts, p)
        want = np.zeros((p.n_rho, p.n_theta), dtype=np.int64)
        for r, t, v in c["bins"]:
            want[r, t] = v
        assert np.array_equal(acc.bins, want), c["name"]
        peaks = lms.find_peaks(acc, c["max_peaks"], c["min_votes"])
        for pk, sup in zip(peaks, c["supports"]):
            got = lms.supporting_points(pts, pk, p)
            assert got == [pts[k] for k in sup], c["name"]


def test_detect_lines_matches_reference(cases):
    for c in cases:
        p = params_of(c)
        img = image_of(c)
        for method in ("lms", "ols", "sht"):
            want = c["detect"][method]
            if isinstance(want, dict):
                with pytest.raises(ValueError):
                    lms.detect_lines(img, p, method, c["max_peaks"], min_votes=c["min_votes"], q=c["q"],
                                     support_cap=c["support_cap"])
                continue
            got = lms.detect_lines(img, p, method, c["max_peaks"], min_votes=c["min_votes"], q=c["q"],
                                   support_cap=c["support_cap"])
            assert len(got) == len(want), (c["name"], method)
            pts = lms.extract_points(img)
            for d, w, sup in zip(got, want, c["supports"]):
                assert (d.rho, d.theta, d.slope, d.intercept) == (f(w["rho"]), f(w["theta"]), f(w["slope"]),
                                                                  f(w["intercept"])), (c["name"], method)
                assert d.axis_swapped == w["axis_swapped"]
                assert d.lms_value == f(w["lms_value"])
                assert len(d.support) == w["support_len"]
                assert d.support == tuple(pts[k] for k in sup)


def test_refine_lms_with_cap_matches_reference(cases):
    for c in cases:
        p = params_of(c)
        pts = lms.extract_points(image_of(c))
        for pk, sup, want in zip(c["peaks"], c["supports"], c["refits"]):
            if want is None or "error" in want:
                continue
            fit = lms.refine_lms([pts[k] for k in sup], None, lms.needs_axis_swap(f(pk[4])), support_cap=64)
            assert (fit.line.slope, fit.line.intercept, fit.lms_value) == \
                (f(want["slope"]), f(want["intercept"]), f(want["lms_value"]))


def test_config5_scale_vote_and_support_vs_oracle():
    img = workloads.line_image(2048, 2048, lines=24, salt=0.10, seed=5)
    p = lms.HoughParams.for_image(2048, 2048, 20.0, 20.0)
    c, s = p.vote_trig()
    bins, npts = _native.hough_vote_image(img, 128, c, s, p.rho_max, p.delta_rho, p.n_rho)
    lit = np.flatnonzero(img >= 128)
    assert npts == lit.size
    x = (lit % 2048).astype(float)
    y = (lit // 2048).astype(float)
    want = hough_oracle.vote(x, y, p.delta_rho, p.delta_theta, p.rho_max)
    assert np.array_equal(bins, want)
    peaks = lms.find_peaks(lms.HoughAccumulator(bins=bins, params=p), 70, 2)
    trig = [p.support_trig(k.theta_bin) for k in peaks]
    offsets, ids = _native.hough_support([t[0] for t in trig], [t[1] for t in trig],
                                         [k.rho_bin for k in peaks], p.rho_max, p.delta_rho, p.n_rho,
                                         capacity=10)  # forces the grow-and-retry path
    for q, k in enumerate(peaks[:12]):
        ords = hough_oracle.support(x, y, k.theta_bin, k.rho_bin, p.delta_rho, p.delta_theta, p.rho_max)
        assert np.array_equal(ids[offsets[q]:offsets[q + 1]], lit[ords])
    assert all(offsets[q + 1] - offsets[q] == k.votes for q, k in enumerate(peaks))
    # the int32 download (lms_hough_support_i32, used by detect_lines) carries
    # the same ids, including through the grow-and-retry path
    off32, ids32 = _native.hough_support([t[0] for t in trig], [t[1] for t in trig],
                                         [k.rho_bin for k in peaks], p.rho_max, p.delta_rho,
                                         p.n_rho, capacity=10, narrow=True)
    assert ids32.dtype == np.int32
    assert np.array_equal(off32, offsets) and np.array_equal(ids32.astype(np.int64), ids)


def test_detect_lines_deterministic_and_batched_equals_single():
    img = workloads.line_image(1024, 1024, lines=6, salt=0.02, seed=9)
    p = lms.HoughParams.for_image(1024, 1024, 20.0, 10.0)
    a = lms.detect_lines(img, p, "lms", 6)
    b = lms.detect_lines(img, p, "lms", 6, backend="par", workers=3)
    assert a == b
    for d in a:
        fit = lms.refine_lms(d.support, None, d.axis_swapped, support_cap=256)
        assert (fit.line.slope, fit.line.intercept, fit.lms_value) == (d.slope, d.intercept, d.lms_value)


def test_config5_staged_transfers_integrity():
    """The 4096^2 image upload and the multi-MB support downloads go through
    the pinned double-buffered staging (chunks of 4 MB): vote totals, lit
    count, per-peak support sizes, scan order, lit pixels, and the int32 and
    int64 downloads agreeing."""
    img = workloads.line_image(4096, 4096, 64, 0.30, seed=0)
    p = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
    c, s = p.vote_trig()
    bins, npts = _native.hough_vote_image(img, 128, c, s, p.rho_max, p.delta_rho, p.n_rho)
    flat = img.ravel()
    assert npts == int((flat >= 128).sum())
    assert int(bins.sum()) == npts * len(c)
    peaks = lms.find_peaks(lms.HoughAccumulator(bins=bins, params=p), 64, 2)
    trig = [p.support_trig(k.theta_bin) for k in peaks]
    args = ([t[0] for t in trig], [t[1] for t in trig], [k.rho_bin for k in peaks], p.rho_max,
            p.delta_rho, p.n_rho)
    cap = sum(k.votes for k in peaks)
    off64, ids64 = _native.hough_support(*args, capacity=cap)
    off32, ids32 = _native.hough_support(*args, capacity=cap, narrow=True)
    assert ids64.nbytes > 8 * (1 << 20)  # large enough for the staged path
    assert np.array_equal(off32, off64) and np.array_equal(ids32.astype(np.int64), ids64)
    assert all(off64[q + 1] - off64[q] == k.votes for q, k in enumerate(peaks))
    for q in range(len(peaks)):
        seg = ids64[off64[q]:off64[q + 1]]
        assert np.all(np.diff(seg) > 0) and np.all(flat[seg] >= 128)


def _config5_golden():
    import gzip
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "config5_golden.json.gz")
    with gzip.open(path, "rt") as fh:
        return json.load(fh)


def test_config5_full_size_matches_reference_golden():
    """BASELINE config 5 at full size: the 4096^2 image of 64 gen_synthetic lines
    + 30 % salt (workloads.config5_image, the reference's own generator
    recipe), detect_lines(..., "lms", 64) with support caps 256 and 512
    against the reference's own run (tests/golden/make_golden_config5.py):
    accumulator, peaks, every LineDetection field, and each peak's full
    support (length and sha256 of its (x, y) pairs in order)."""
    import hashlib

    doc = _config5_golden()
    img = workloads.config5_image(0)
    assert hashlib.sha256(img.tobytes()).hexdigest() == doc["image_sha256"]
    p = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
    assert [p.delta_rho.hex(), p.delta_theta.hex(), p.rho_max.hex()] == doc["params"]
    c, s = p.vote_trig()
    bins, npts = _native.hough_vote_image(img, 128, c, s, p.rho_max, p.delta_rho, p.n_rho)
    assert npts == doc["lit"]
    want = np.zeros_like(bins)
    for r, t, v in doc["bins"]:
        want[r, t] = v
    assert np.array_equal(bins, want)
    peaks = lms.find_peaks(lms.HoughAccumulator(bins=bins, params=p), 64, 2)
    assert [[k.rho_bin, k.theta_bin, k.votes, k.rho.hex(), k.theta.hex()] for k in peaks] == doc["peaks"]
    for cap in (256, 512):
        dets = lms.detect_lines(img, p, "lms", 64, support_cap=cap)
        gold = doc["detect"][str(cap)]
        assert len(dets) == len(gold)
        for d, g in zip(dets, gold):
            assert (d.rho, d.theta, d.slope, d.intercept, d.lms_value) == \
                tuple(f(g[k]) for k in ("rho", "theta", "slope", "intercept", "lms_value")), cap
            assert d.axis_swapped == g["axis_swapped"] and d.method == g["method"]
            assert len(d.support) == g["support_len"]
            xy = np.array([(q.x, q.y) for q in d.support], dtype=np.int32)
            assert hashlib.sha256(xy.tobytes()).hexdigest() == g["support_sha256"]
