"""Compatibility with the reference's own test suite (/root/reference/pkg/tests),
restated against this package's public API: the same properties, on the
same kinds of inputs, run on the GPU.  Each test names the reference test it
mirrors (file::function).  The reference's CLI, PGM, synth and experiments
suites are out of scope here (synth/PGM: tests/test_synth_pgm.py)."""

import math

import numpy as np
import pytest

import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import synth

pytestmark = pytest.mark.gpu

P = lms.Point2


def _brute_value(pts, q):
    """Every non-vertical pair slope, every q-window of the sorted
    intercepts (pure Python): the optimal LMS value."""
    xs = [p.x for p in pts]
    ys = [p.y for p in pts]
    best = math.inf
    for i in range(len(pts)):
        for j in range(i + 1, len(pts)):
            if xs[i] != xs[j]:
                s = (ys[j] - ys[i]) / (xs[j] - xs[i])
                cs = sorted(y - s * x for x, y in zip(xs, ys))
                for w in range(len(pts) - q + 1):
                    best = min(best, ((cs[w + q - 1] - cs[w]) / 2) ** 2)
    return best


# ------------------------------------------------------------- test_solver.py
def test_solver_known_answers():  # test_collinear_points_fit_exactly .. test_square_splits_the_difference
    f = lms.solve_lms([P(0, 1), P(1, 3), P(2, 5), P(3, 7)], 3)
    assert (f.line.slope, f.line.intercept, f.lms_value, f.slab_height, f.coverage) == (2.0, 1.0, 0.0, 0.0, 3)
    maj = [P(x, float(x)) for x in range(5)] + [P(0.5, 50), P(1.5, -40), P(2.5, 90), P(3.5, 60)]
    f = lms.solve_lms(maj, 5)
    assert (f.line.slope, f.line.intercept, f.lms_value) == (1.0, 0.0, 0.0)
    f = lms.solve_lms([P(0, 0), P(1, 0), P(0, 1), P(1, 1)], 3)
    assert (f.line.slope, f.line.intercept, f.lms_value, f.slab_height) == (0.0, 0.5, 0.25, 1.0)
    assert set(f.contact_indices) == {0, 1, 2, 3}
    assert lms.default_coverage(4) == 3 and lms.default_coverage(5) == 3 and lms.default_coverage(100) == 51


def test_solver_value_is_median_square_of_its_line():  # test_lms_value_is_median_of_squares_of_own_line
    rng = np.random.default_rng(5)
    for _ in range(40):
        pts = rng.normal(0, 10, (int(rng.integers(4, 40)), 2))
        f = lms.solve_lms(pts)
        assert lms.median_sq_residual(pts, f.line, f.coverage) == pytest.approx(f.lms_value, rel=1e-9, abs=1e-12)
        assert f.lms_value == pytest.approx((f.slab_height / 2) ** 2, rel=1e-12)


def test_solver_agrees_with_primal_oracle():  # test_oracle_and_solver_agree_on_random_sets, _fixed_16_point_set
    rng = np.random.default_rng(17)
    for trial in range(60):
        n = int(rng.integers(4, 24))
        pts = rng.normal(0, 30, (n, 2))
        if trial % 4 == 0:
            pts[1, 0] = pts[0, 0]
        q = None if trial % 3 else int(rng.integers(3, n + 1))
        a, b = lms.solve_lms(pts, q), lms.oracle_lms(pts, q)
        assert a.lms_value == pytest.approx(b.lms_value, rel=1e-9, abs=1e-15)
        assert a.line.slope == pytest.approx(b.line.slope, rel=1e-9, abs=1e-12)
        assert a.line.intercept == pytest.approx(b.line.intercept, rel=1e-9, abs=1e-12)
        assert a.coverage == b.coverage
    pts = np.random.default_rng(53).normal(0, 12, (16, 2))
    a, b = lms.solve_lms(pts), lms.oracle_lms(pts)
    assert (a.lms_value, a.line.slope) == pytest.approx((b.lms_value, b.line.slope), rel=1e-12)


def test_solver_q2_interpolates_a_pair():  # test_coverage_two_interpolates_the_first_valid_pair
    rng = np.random.default_rng(59)
    for _ in range(10):
        pts = rng.normal(0, 10, (8, 2))
        f = lms.solve_lms(pts, 2)
        assert f.lms_value == 0.0
        for k in (0, 1):
            assert pts[k, 1] == pytest.approx(f.line.slope * pts[k, 0] + f.line.intercept, rel=1e-9, abs=1e-9)


def test_solver_tiny_sets_match_enumeration():  # test_tiny_sets_match_pure_python_enumeration
    rng = np.random.default_rng(23)
    for _ in range(30):
        n = int(rng.integers(4, 8))
        pts = [P(float(x), float(y)) for x, y in rng.normal(0, 5, (n, 2))]
        q = int(rng.integers(2, n + 1))
        assert lms.solve_lms(pts, q).lms_value == pytest.approx(_brute_value(pts, q), rel=1e-12, abs=1e-18)


def test_solver_local_optimality_and_equioscillation():  # test_solution_is_locally_optimal, test_equioscillation_contacts
    rng = np.random.default_rng(31)
    for _ in range(20):
        pts = rng.normal(0, 8, (int(rng.integers(6, 25)), 2))
        f = lms.solve_lms(pts)
        for ds in (-1e-3, 0.0, 1e-3):
            for dc in (-1e-3, 0.0, 1e-3):
                probe = lms.LineEq(f.line.slope + ds, f.line.intercept + dc)
                assert lms.median_sq_residual(pts, probe, f.coverage) >= f.lms_value - 1e-12 * max(1.0, f.lms_value)
    rng = np.random.default_rng(37)
    for _ in range(30):
        pts = rng.normal(0, 6, (int(rng.integers(6, 30)), 2))
        f = lms.solve_lms(pts)
        r = pts[:, 1] - (f.line.slope * pts[:, 0] + f.line.intercept)
        half, tol = f.slab_height / 2, 1e-9 * max(1.0, float(np.abs(r).max()))
        up = [k for k in f.contact_indices if abs(r[k] - half) <= tol]
        dn = [k for k in f.contact_indices if abs(r[k] + half) <= tol]
        assert len(f.contact_indices) >= 3 and up and dn and len(up) + len(dn) >= 3


def test_solver_exact_fits_and_equivariance():  # test_exact_fit_whenever_q_points_are_collinear, test_affine_equivariance
    rng = np.random.default_rng(41)
    for _ in range(25):
        q = int(rng.integers(3, 10))
        xs = rng.permutation(64)[:q].astype(float)
        slope, icp = float(rng.integers(-16, 17)) / 8, float(rng.integers(-64, 65)) / 8
        pts = np.vstack([np.column_stack([xs, slope * xs + icp]), rng.uniform(-50, 50, (q - 1, 2))])
        f = lms.solve_lms(pts, q)
        assert (f.lms_value, f.line.slope, f.line.intercept) == (0.0, slope, icp)
    pts = np.random.default_rng(43).normal(0, 5, (20, 2))
    f = lms.solve_lms(pts)
    g = lms.solve_lms(pts + np.array([2.5, -1.25]))
    assert g.line.slope == pytest.approx(f.line.slope, rel=1e-9)
    assert g.line.intercept == pytest.approx(f.line.intercept - 1.25 - f.line.slope * 2.5, rel=1e-9, abs=1e-12)
    h = lms.solve_lms(pts * np.array([1.0, 3.0]))
    assert (h.line.slope, h.lms_value) == pytest.approx((3 * f.line.slope, 9 * f.lms_value), rel=1e-9)


def test_solver_determinism_duplicates_and_errors():  # test_repeat_runs_are_bit_identical .. test_vertical_majority_still_solvable
    pts = np.random.default_rng(47).normal(0, 10, (32, 2))
    assert lms.solve_lms(pts) == lms.solve_lms(pts)
    f = lms.solve_lms([P(0, 0), P(0, 0), P(1, 1), P(2, 2), P(1, 5)], 4)
    assert (f.lms_value, f.line.slope) == (0.0, 1.0)
    for solver in (lms.solve_lms, lms.oracle_lms):
        with pytest.raises(lms.DegenerateInputError):
            solver([P(0, 0), P(1, 1)])
        with pytest.raises(lms.DegenerateInputError):
            solver([P(2, 0), P(2, 1), P(2, 5)])
        for q in (1, 4):
            with pytest.raises(lms.InvalidInputError):
                solver([P(0, 0), P(1, 1), P(2, 3)], q)
    with pytest.raises(lms.InvalidInputError):
        lms.solve_lms([P(0, 0), P(1, math.inf), P(2, 1)])
    assert math.isfinite(lms.solve_lms([P(1, v) for v in (0.0, 1.0, 2.0, 3.0)] + [P(2, 1.0)], 2).line.slope)


# ------------------------------------------------------------ test_backend.py
def test_backend_phases():  # test_phase2_single_intersection_identity, _worker_count_does_not_change_result
    lines = lms.dualize(np.random.default_rng(11).normal(0, 10, (64, 2)))
    ips = list(lms.run_phase1(lines))
    assert len(ips) == 64 * 63 // 2
    ref = lms.run_phase2(ips, lines, 33)
    for w in (1, 2, 5):
        assert lms.run_phase2(ips, lines, 33, worker_count=w) == ref
    one = lms.run_phase2(ips[:1], lines, 33)
    br = lms.bracelet_at(ips[0], lines, 33)
    assert (one.v_low, one.v_high) == (br.v_low, br.v_high)


def test_backend_kernel_agrees_with_scalar_bracelet():  # test_kernel_agrees_with_scalar_bracelet
    rng = np.random.default_rng(13)
    for _ in range(5):
        n = int(rng.integers(5, 14))
        pts = rng.normal(0, 5, (n, 2))
        q = int(rng.integers(2, n + 1))
        lines = lms.dualize(pts)
        best = None
        for ip in lms.run_phase1(lines):
            br = lms.bracelet_at(ip, lines, q)
            if br is not None and (best is None or (br.height, ip.i, ip.j) < best[:3]):
                best = (br.height, ip.i, ip.j)
        rec = lms.get_backend("seq").minimum_bracelet(pts[:, 0].copy(), pts[:, 1].copy(), q)
        assert (rec.height, rec.i, rec.j) == best


def test_backend_seq_par_materialize_identical(monkeypatch):  # test_seq_and_par_backends_bit_identical, test_materialized_mode_matches_streaming
    rng = np.random.default_rng(19)
    for _ in range(8):
        pts = rng.normal(0, 20, (int(rng.integers(5, 80)), 2))
        a = lms.solve_lms(pts)
        assert lms.solve_lms(pts, backend="par", workers=3) == a
        assert lms.solve_lms(pts, materialize=True) == a
        assert lms.solve_lms(pts, backend="par", workers=2, materialize=True) == a
    monkeypatch.setenv("LMSLINE_WORKERS", "2")
    assert lms.solve_lms(pts, backend="par") == lms.solve_lms(pts)


def test_backend_names():  # test_get_backend_names
    assert lms.get_backend("seq").name == "seq" and lms.get_backend("par", 2).name == "par"
    for bad in ("gpu", "cuda", ""):
        with pytest.raises(lms.InvalidInputError):
            lms.get_backend(bad)


# ------------------------------------------------------------- test_hough.py
def test_hough_vote_and_support_invariants():  # test_vote_total_is_points_times_theta_bins, test_support_matches_votes_and_revotes
    img, _ = synth.gen_synthetic(synth.SyntheticSpec(width=300, height=200, slope=0.6, intercept=20.0,
                                                     noise_prob=0.01, seed=4))
    p = lms.HoughParams.for_image(300, 200, 4.0, 6.0)
    pts = lms.extract_points(img)
    acc = lms.hough_vote(pts, p)
    assert int(acc.bins.sum()) == len(pts) * p.n_theta
    for pk in lms.find_peaks(acc, 5, 2):
        sup = lms.supporting_points(pts, pk, p)
        assert len(sup) == pk.votes
        assert int(lms.hough_vote(sup, p).bins[pk.rho_bin, pk.theta_bin]) == pk.votes


def test_hough_vertical_line_peaks_near_theta_zero():  # test_vote_vertical_line_peaks_near_theta_zero
    pts = [P(40.0, float(y)) for y in range(100)]
    p = lms.HoughParams.for_image(100, 100, 2.0, 5.0)
    pk = lms.find_peaks(lms.hough_vote(pts, p), 1, 1)[0]
    assert pk.theta < 5.0 or pk.theta > 175.0
    assert abs(abs(pk.rho) - 40.0) <= 4.5


# ------------------------------------------------------------ test_detect.py
def test_detect_lms_ignores_outliers_and_honors_cap():  # test_lms_ignores_minority_outliers, test_refine_lms_honors_support_cap
    line = [P(float(x), 2.0 * x + 1.0) for x in range(20)]
    junk = [P(3.0, 90.0), P(7.0, -50.0), P(11.0, 70.0)]
    f = lms.refine_lms(line + junk)
    assert (f.line.slope, f.line.intercept, f.lms_value) == (2.0, 1.0, 0.0)
    sup = [P(float(x), float(x % 7)) for x in range(1000)]
    f = lms.refine_lms(sup, support_cap=50)
    g = lms.solve_lms(np.array([[p.x, p.y] for p in lms.subsample_support(sup, 50)]))
    assert f == g
    swapped = lms.refine_lms([P(5.0, float(y)) for y in range(10)], axis_swapped=True)
    assert (swapped.line.slope, swapped.line.intercept) == (0.0, 5.0)


def test_detect_recovers_synthetic_lines():  # test_detect_lms_recovers_synthetic_line, _steep_line, _two_crossing_lines
    img, t = synth.gen_synthetic(synth.SyntheticSpec(slope=0.35, intercept=220.0, sampling_prob=0.5,
                                                     noise_prob=0.002, seed=3))
    p = lms.HoughParams.for_image(1024, 1024, 20.0, 20.0)
    d = lms.detect_lines(img, p, "lms")[0]
    assert d.image_slope == pytest.approx(t.slope, abs=0.02)
    assert d.image_intercept == pytest.approx(t.intercept, abs=6.0)
    assert len(d.support) > 256
    a, _ = synth.gen_synthetic(synth.SyntheticSpec(endpoints=((100, 100), (900, 900)), sampling_prob=1.0, seed=1))
    b, _ = synth.gen_synthetic(synth.SyntheticSpec(endpoints=((100, 900), (900, 100)), sampling_prob=1.0, seed=2))
    dets = lms.detect_lines(np.maximum(a, b), lms.HoughParams.for_image(1024, 1024, 20.0, 2.0), "lms", 2)
    assert sorted(d.image_slope for d in dets) == pytest.approx([-1.0, 1.0], abs=0.03)


def test_detect_blank_unknown_method_and_determinism():  # test_detect_blank_image_returns_nothing .. test_detect_deterministic
    p = lms.HoughParams.for_image(64, 64, 2.0, 10.0)
    assert lms.detect_lines(np.zeros((64, 64), dtype=np.uint8), p) == []
    with pytest.raises(lms.InvalidInputError):
        lms.detect_lines(np.zeros((8, 8), dtype=np.uint8), lms.HoughParams.for_image(8, 8, 1.0, 10.0), "ransac")
    img, _ = synth.gen_synthetic(synth.SyntheticSpec(slope=0.3, intercept=150.0, noise_prob=0.002, seed=19))
    p = lms.HoughParams.for_image(1024, 1024, 20.0, 20.0)
    assert lms.detect_lines(img, p, "lms") == lms.detect_lines(img, p, "lms")


# -------------------------------------------------------- test_acceptance.py
def test_acceptance_criterion_8_parallel_determinism():  # test_criterion_8_parallel_determinism
    rng = np.random.default_rng([88, 0])
    for _ in range(6):
        n = int(rng.integers(8, 200))
        pts = rng.uniform(-100, 100, (n, 2))
        if rng.random() < 0.3:
            pts[: int(rng.integers(2, n // 2)), 0] = pts[0, 0]
        q = int(rng.integers(2, n + 1))
        a = lms.solve_lms(pts, q)
        for w in (1, 2, 4):
            assert lms.solve_lms(pts, q, backend="par", workers=w) == a
    img, _ = synth.gen_synthetic(synth.SyntheticSpec(slope=0.35, intercept=220.0, noise_prob=0.002, seed=88))
    p = lms.HoughParams.for_image(1024, 1024, 20.0, 20.0)
    assert lms.detect_lines(img, p, "lms", 1) == lms.detect_lines(img, p, "lms", 1, backend="par", workers=4)
