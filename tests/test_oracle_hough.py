"""Hough oracle and the host-side Hough helpers against the reference's
golden vectors (tests/golden/make_golden_hough.py)."""

import gzip
import json
import os

import numpy as np
import pytest

from oracle import hough_oracle
import paper_1510_01041_b200 as lms

GOLD = os.path.join(os.path.dirname(__file__), "golden", "hough_golden.json.gz")


def load():
    with gzip.open(GOLD, "rt") as fh:
        return json.load(fh)["cases"]


def f(h):
    return None if h is None else float.fromhex(h)


def image_of(c):
    img = np.zeros(c["height"] * c["width"], dtype=np.uint8)
    img[np.asarray(c["lit"], dtype=np.int64)] = 255
    return img.reshape(c["height"], c["width"])


def params_of(c):
    dr, dt, rm = (f(v) for v in c["params"])
    return lms.HoughParams(delta_rho=dr, delta_theta=dt, rho_max=rm)


@pytest.fixture(scope="module")
def cases():
    return load()


def test_oracle_vote_and_support_match_reference(cases):
    for c in cases:
        p = params_of(c)
        lit = np.asarray(c["lit"], dtype=np.int64)
        x = (lit % c["width"]).astype(float)
        y = (lit // c["width"]).astype(float)
        bins = hough_oracle.vote(x, y, p.delta_rho, p.delta_theta, p.rho_max)
        want = np.zeros_like(bins)
        for r, t, v in c["bins"]:
            want[r, t] = v
        assert np.array_equal(bins, want), c["name"]
        for pk, sup in zip(c["peaks"], c["supports"]):
            got = hough_oracle.support(x, y, pk[1], pk[0], p.delta_rho, p.delta_theta, p.rho_max)
            assert got.tolist() == sup, c["name"]


def test_find_peaks_host_matches_reference(cases):
    for c in cases:
        p = params_of(c)
        bins = np.zeros((p.n_rho, p.n_theta), dtype=np.int64)
        for r, t, v in c["bins"]:
            bins[r, t] = v
        peaks = lms.find_peaks(lms.HoughAccumulator(bins=bins, params=p), c["max_peaks"], c["min_votes"])
        got = [[k.rho_bin, k.theta_bin, k.votes, k.rho, k.theta] for k in peaks]
        want = [[a, b, v, f(r), f(t)] for a, b, v, r, t in c["peaks"]]
        assert got == want, c["name"]


def test_extract_points_scan_order(cases):
    c = cases[0]
    pts = lms.extract_points(image_of(c))
    lit = np.asarray(c["lit"])
    assert [(p.x, p.y) for p in pts] == [(float(k % c["width"]), float(k // c["width"])) for k in lit]


def test_params_and_polar_helpers():
    p = lms.HoughParams(delta_rho=20.0, delta_theta=20.0, rho_max=1448.0)
    assert (p.n_theta, p.n_rho, p.theta_center(0), p.theta_center(8)) == (9, 145, 10.0, 170.0)
    q = lms.HoughParams(delta_rho=2.0, delta_theta=20.0, rho_max=10.0)
    assert [int(q.rho_bin(v)) for v in (0.0, -10.0, 9.999, 10.0)] == [5, 0, 9, 9]
    for bad in (dict(delta_rho=0.0, delta_theta=1.0, rho_max=1.0),
                dict(delta_rho=1.0, delta_theta=200.0, rho_max=1.0)):
        with pytest.raises(lms.InvalidInputError):
            lms.HoughParams(**bad)
    assert lms.needs_axis_swap(10.0) and not lms.needs_axis_swap(90.0)
    for slope, c in ((0.5, 3.0), (-2.0, 7.0), (0.0, 4.0)):
        for sw in (False, True):
            rho, th = lms.line_to_polar(slope, c, sw)
            s2, c2, sw2 = lms.polar_to_frame_fit(rho, th)
            if sw2 == sw:
                assert s2 == pytest.approx(slope, abs=1e-9) and c2 == pytest.approx(c, abs=1e-9)


def test_subsample_and_support_points_helpers():
    pts = [lms.Point2(float(k), 0.0) for k in range(10)]
    assert [p.x for p in lms.subsample_support(pts, 4)] == [0.0, 2.0, 5.0, 7.0]
    assert lms.subsample_support(pts, 10) == pts
    with pytest.raises(lms.InvalidInputError):
        lms.subsample_support(pts, 2)
    sp = lms.SupportPoints.from_pixels(np.array([5, 17, 40]), 16)
    assert sp == (lms.Point2(5.0, 0.0), lms.Point2(1.0, 1.0), lms.Point2(8.0, 2.0))
    assert len(sp) == 3 and sp[1] == lms.Point2(1.0, 1.0) and hash(sp) == hash(tuple(sp))
    fit = lms.refine_ols([lms.Point2(0, 1), lms.Point2(1, 3), lms.Point2(2, 5)])
    assert fit.slope == pytest.approx(2.0) and fit.intercept == pytest.approx(1.0)
