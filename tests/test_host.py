"""Host-side API behaviour that needs no GPU: validation, plans, names,
phase-1 enumeration, geometry helpers (mirrors the reference's own tests)."""

import math

import numpy as np
import pytest

import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import workloads
from paper_1510_01041_b200.backend import WORKERS_ENV_VAR, BatchPlan, resolve_workers


def test_batch_plan_counts_pairs():
    plan = BatchPlan.create(np.array([0.0, 1.0, 2.0, 3.0]), 2)
    assert (plan.n, plan.pair_count, plan.partition_size, plan.worker_count) == (4, 6, 3, 2)
    assert BatchPlan.create(np.array([0.0, 1.0, 1.0, 3.0]), 1).pair_count == 5


def test_batch_plan_partitions_cover_all_ranks():
    parts = BatchPlan.create(np.arange(9, dtype=float), 4).partitions()
    assert parts[0][0] == 0 and parts[-1][1] == 36
    for (_, e1), (s2, _) in zip(parts, parts[1:]):
        assert e1 == s2


def test_batch_plan_validation():
    with pytest.raises(lms.InvalidInputError):
        BatchPlan.create(np.array([1.0]), 2)
    with pytest.raises(lms.InvalidInputError):
        BatchPlan.create(np.arange(4, dtype=float), 0)


def test_get_backend_names():
    assert lms.get_backend("seq").name == "seq"
    assert lms.get_backend("par", 2).name == "par"
    with pytest.raises(lms.InvalidInputError):
        lms.get_backend("gpu")


def test_resolve_workers_precedence(monkeypatch):
    monkeypatch.delenv(WORKERS_ENV_VAR, raising=False)
    assert resolve_workers(5) == 5
    assert resolve_workers(None) >= 1
    monkeypatch.setenv(WORKERS_ENV_VAR, "3")
    assert resolve_workers(None) == 3
    assert resolve_workers(2) == 2
    monkeypatch.setenv(WORKERS_ENV_VAR, "zero")
    with pytest.raises(lms.InvalidInputError):
        resolve_workers(None)
    monkeypatch.setenv(WORKERS_ENV_VAR, "-1")
    with pytest.raises(lms.InvalidInputError):
        resolve_workers(None)


def test_phase1_row_major_and_parallel_skip():
    ips = list(lms.run_phase1(lms.dualize([lms.Point2(0, 0), lms.Point2(1, 2), lms.Point2(3, 1)])))
    assert [(ip.i, ip.j) for ip in ips] == [(0, 1), (0, 2), (1, 2)]
    ips = list(lms.run_phase1(lms.dualize([lms.Point2(2, 0), lms.Point2(2, 5), lms.Point2(0, 1)])))
    assert [(ip.i, ip.j) for ip in ips] == [(0, 2), (1, 2)]


def test_phase2_validation_before_device():
    lines = lms.dualize([lms.Point2(0, 0), lms.Point2(1, 0), lms.Point2(0, 1), lms.Point2(1, 1)])
    ips = list(lms.run_phase1(lines))
    with pytest.raises(lms.InvalidInputError):
        lms.run_phase2([], lines, 3)
    with pytest.raises(lms.InvalidInputError):
        lms.run_phase2(ips, lines, 1)
    with pytest.raises(lms.InvalidInputError):
        lms.run_phase2(ips, lines, 3, worker_count=0)


@pytest.mark.parametrize("bad", [[lms.Point2(0, 0), lms.Point2(1, 1)],
                                 [lms.Point2(2, 0), lms.Point2(2, 1), lms.Point2(2, 5)]])
def test_degenerate_inputs_rejected(bad):
    with pytest.raises(lms.DegenerateInputError):
        lms.solve_lms(bad)


def test_coverage_and_finiteness_validation():
    pts = [lms.Point2(0, 0), lms.Point2(1, 1), lms.Point2(2, 3)]
    for q in (1, 4):
        with pytest.raises(lms.InvalidInputError):
            lms.solve_lms(pts, q)
    with pytest.raises(lms.InvalidInputError):
        lms.solve_lms([lms.Point2(0, 0), lms.Point2(1, math.inf), lms.Point2(2, 1)])
    with pytest.raises(lms.InvalidInputError):
        lms.solve_lms(np.zeros((4, 3)))
    with pytest.raises(lms.InvalidInputError):
        lms.solve_lms(np.array([[0, 0], [1, 1], [2, 5.0]]), backend="gpu")


def test_geometry_helpers():
    ip = lms.pair_intersection(lms.DualLine(1.0, 2.0, 0), lms.DualLine(3.0, 1.0, 1))
    assert (ip.u, ip.v, ip.i, ip.j) == (-0.5, -2.5, 0, 1)
    assert lms.pair_intersection(lms.DualLine(1.0, 2.0, 0), lms.DualLine(1.0, 1.0, 1)) is None
    with pytest.raises(lms.InvalidInputError):
        lms.pair_intersection(lms.DualLine(1.0, 2.0, 0), lms.DualLine(3.0, 1.0, 0))
    cut = lms.vertical_cut(lms.dualize([[0, 0], [1, 0], [0, 1], [1, 1]]), 0.5)
    assert cut == [(-1.0, 2), (-0.5, 3), (0.0, 0), (0.5, 1)]
    pts = np.array([[0, 0], [1, 1], [2, 2], [3, 10.0]])
    assert lms.median_sq_residual(pts, lms.LineEq(1.0, 0.0), 3) == 0.0
    assert lms.median_sq_residual(pts, lms.LineEq(1.0, 0.0), 4) == 49.0
    assert lms.default_coverage(4) == 3 and lms.default_coverage(100) == 51


def test_bracelet_q_validation_before_device():
    lines = lms.dualize([[0, 0], [1, 0], [0, 1], [1, 1]])
    ip = lms.pair_intersection(lines[0], lines[1])
    with pytest.raises(lms.InvalidInputError):
        lms.bracelet_at(ip, lines, 1)
    assert lms.bracelet_at(ip, lines, 5) is None


def test_workload_generators_match_golden_inputs(golden):
    cases, _ = golden
    by_name = {c.name: c for c in cases}
    for f in range(2):
        c = by_name[f"bench_points_512_s{f}"]
        assert np.array_equal(workloads.bench_points(512, seed=f), c.points)
    for s in (0, 1):
        assert np.array_equal(workloads.config1_points(s), by_name[f"config1_s{s}"].points)
    assert np.array_equal(workloads.contaminated_line_points(2000, 0), by_name["config2_gen_n2000_s0"].points)


def test_batch_validation_fast_path_matches_per_set_order():
    """solve_lms_batch's vectorised validation raises what the per-set
    validated() loop raises first (before any device work)."""
    import numpy as np

    from paper_1510_01041_b200 import solver

    good = np.array([[1.0, 2.0], [2.0, 3.0], [3.0, 5.0], [4.0, 1.0]])
    cases = [
        [np.zeros((5, 2)), np.array([[1.0, 2.0], [2.0, 3.0]])],
        [good, np.array([[1.0, 2.0], [2.0, 3.0]])],
        [good, np.array([[1.0, 2.0], [np.nan, 1.0], [3.0, 4.0]])],
        [good, np.array([[1.0, 2.0], [1.0, 1.0], [1.0, 4.0]]), np.zeros((2, 2))],
    ]
    for sets in cases:
        for q in (None, 3, 7):
            want = None
            for p in sets:
                try:
                    solver.validated(p, q)
                except ValueError as e:
                    want = e
                    break
            assert want is not None
            try:
                solver.solve_lms_batch(sets, q)
            except ValueError as got:
                assert (type(got), str(got)) == (type(want), str(want)), (sets, q)
            else:
                raise AssertionError("no error raised")


def test_lit_mask_non_finite_threshold_follows_numpy():
    """hough.py:102: img >= threshold; a NaN / inf threshold must not reach int()."""
    from paper_1510_01041_b200.hough import lit_mask_u8

    img = np.array([[0, 127, 128, 255]], dtype=np.uint8)
    for thr, want in ((math.nan, [0, 0, 0, 0]), (math.inf, [0, 0, 0, 0]), (-math.inf, [1, 1, 1, 1])):
        m, t = lit_mask_u8(img, thr)
        assert list((m >= t).ravel().astype(int)) == want
    m, t = lit_mask_u8(img, 128)
    assert t == 128 and m is not None


def test_par_shards_env_validated(monkeypatch):
    from paper_1510_01041_b200.backend import _env_shards

    monkeypatch.delenv("LMSB_PAR_SHARDS", raising=False)
    assert _env_shards(3) == 3
    monkeypatch.setenv("LMSB_PAR_SHARDS", "2")
    assert _env_shards(3) == 2
    for bad in ("x", "0", "-1", "1.5"):
        monkeypatch.setenv("LMSB_PAR_SHARDS", bad)
        with pytest.raises(lms.InvalidInputError):
            _env_shards(1)
