"""Generate golden vectors for the exact-LMS path by running the REFERENCE.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/lms_golden.json.gz``.  Every float is stored as
``float.hex`` so the fixtures are bit-exact.  Nothing at test time reads the
reference; the tests only read this committed file.

Cases (each cites the reference test it mirrors):
  * known answers: COLLINEAR4 / majority / SQUARE (test_solver.py:18-74),
    duplicates (:212-216), vertical majority (:241-245)
  * criterion-1 generic + degenerate sets, the reference's full sets: 1,000
    generic (n in 4..64 x 200 seeds) + 100 degenerate (test_acceptance.py:50-90)
  * criterion-2 breakdown sets, all 100 seeds (test_acceptance.py:95-121)
  * criterion-8 determinism sets with collapsed x (test_acceptance.py:248-266)
  * normal(0, s) sets of test_solver.py / test_backend.py
  * dyadic exact fits (test_solver.py:162-175)
  * config 1, config-2 generator at n = 2000,
    bench_points(512) (experiments.py:247-254, config 4)
  * per-vertex bracelets over every pair of small sets (test_backend.py:114-132)
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from lmsline import Point2, bracelet_at, dualize, run_phase1, solve_lms  # noqa: E402
from lmsline.backend import get_backend  # noqa: E402
from lmsline.experiments import bench_points as ref_bench_points  # noqa: E402

from paper_1510_01041_b200 import workloads  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "lms_golden.json.gz")


def hx(v: float) -> str:
    return float(v).hex()


def random_points(rng, n, collapse_x=False):
    """test_acceptance.py:38-45."""
    x = rng.uniform(-100.0, 100.0, n)
    y = rng.uniform(-100.0, 100.0, n)
    if collapse_x and n >= 8 and rng.random() < 0.3:
        k = int(rng.integers(2, n // 2))
        x[:k] = x[0]
    return np.column_stack([x, y])


def case(name, pts, q=None):
    pts = np.asarray(pts, dtype=float)
    x = np.ascontiguousarray(pts[:, 0])
    y = np.ascontiguousarray(pts[:, 1])
    n = x.size
    qq = n // 2 + 1 if q is None else q
    t0 = time.perf_counter()
    fit = solve_lms(pts, q)
    rec = get_backend("seq").minimum_bracelet(x, y, qq)
    dt = time.perf_counter() - t0
    return {
        "name": name,
        "n": n,
        "q": qq,
        "q_arg": q,
        "x": [hx(v) for v in x],
        "y": [hx(v) for v in y],
        "record": None if rec is None else {
            "height": hx(rec.height), "i": rec.i, "j": rec.j, "u": hx(rec.u),
            "v_low": hx(rec.v_low), "v_high": hx(rec.v_high),
        },
        "fit": {
            "slope": hx(fit.line.slope), "intercept": hx(fit.line.intercept),
            "lms_value": hx(fit.lms_value), "slab_height": hx(fit.slab_height),
            "coverage": fit.coverage, "contact_indices": list(fit.contact_indices),
        },
        "ref_seconds": dt,
    }


def bracelet_case(name, pts, q):
    lines = dualize(pts)
    rows = []
    for ip in run_phase1(lines):
        br = bracelet_at(ip, lines, q)
        rows.append({
            "i": ip.i, "j": ip.j, "u": hx(ip.u), "v": hx(ip.v),
            "bracelet": None if br is None else {
                "v_low": hx(br.v_low), "v_high": hx(br.v_high), "height": hx(br.height)},
        })
    pts = np.asarray(pts, dtype=float)
    return {"name": name, "q": q, "x": [hx(v) for v in pts[:, 0]], "y": [hx(v) for v in pts[:, 1]],
            "vertices": rows}


def main():
    cases = []
    # --- known answers (test_solver.py) ---
    collinear4 = [Point2(0, 1), Point2(1, 3), Point2(2, 5), Point2(3, 7)]
    square = [Point2(0, 0), Point2(1, 0), Point2(0, 1), Point2(1, 1)]
    as_arr = lambda P: [[p.x, p.y] for p in P]  # noqa: E731
    cases.append(case("kat_collinear4", as_arr(collinear4), 3))
    maj = [Point2(x, float(x)) for x in range(5)]
    maj += [Point2(0.5, 50.0), Point2(1.5, -40.0), Point2(2.5, 90.0), Point2(3.5, 60.0)]
    cases.append(case("kat_majority", as_arr(maj), 5))
    cases.append(case("kat_square", as_arr(square), 3))
    dup = [Point2(0, 0), Point2(0, 0), Point2(1, 1), Point2(2, 2), Point2(1, 5)]
    cases.append(case("kat_duplicates", as_arr(dup), 4))
    vert = [Point2(1, v) for v in (0.0, 1.0, 2.0, 3.0)] + [Point2(2, 1.0)]
    cases.append(case("kat_vertical_majority", as_arr(vert), 2))
    cases.append(case("kat_cli_bench", [[0, -2], [1, -1.5], [2, -1], [3, -0.5], [0.5, 7], [2.5, -9]], None))

    # --- criterion 1: generic and degenerate sets ---
    # the reference's full sets: 5 sizes x 200 seeds generic, 100 degenerate
    for n in (4, 8, 16, 32, 64):
        for seed in range(200):
            rng = np.random.default_rng([11, n, seed])
            pts = random_points(rng, n)
            q = int(rng.integers(3, n + 1))
            cases.append(case(f"crit1_n{n}_s{seed}", pts, q))
    for seed in range(100):
        rng = np.random.default_rng([12, seed])
        pts = random_points(rng, 16, collapse_x=True)
        q = int(rng.integers(2, 17))
        cases.append(case(f"crit1_degenerate_s{seed}", pts, q))

    # --- criterion 2: breakdown with outliers at 1e6 ---
    for seed in range(100):
        rng = np.random.default_rng([22, seed])
        n = 15
        q = n // 2 + 1
        slope = float(rng.integers(-16, 17)) / 8.0
        intercept = float(rng.integers(-64, 65)) / 8.0
        x_in = rng.choice(np.arange(-40, 41), size=q, replace=False).astype(float)
        y_in = slope * x_in + intercept
        x_out = rng.uniform(-40.0, 40.0, n - q)
        y_out = slope * x_out + intercept + 1e6 * rng.choice([-1.0, 1.0], n - q)
        pts = np.column_stack([np.concatenate([x_in, x_out]), np.concatenate([y_in, y_out])])
        pts = pts[rng.permutation(n)]
        cases.append(case(f"crit2_s{seed}", pts, q))

    # --- criterion 8: collapsed-x determinism sets ---
    for seed in range(12):
        rng = np.random.default_rng([88, seed])
        n = int(rng.integers(8, 200))
        pts = random_points(rng, n, collapse_x=True)
        q = int(rng.integers(2, n + 1))
        cases.append(case(f"crit8_n{n}_s{seed}", pts, q))

    # --- normal sets (test_solver.py / test_backend.py seeds) ---
    rng = np.random.default_rng(19)
    for trial in range(12):
        n = int(rng.integers(5, 80))
        pts = rng.normal(0, 20, (n, 2))
        if trial % 3 == 0:
            pts[: n // 3, 0] = pts[0, 0]
        cases.append(case(f"seqpar_t{trial}", pts, None))
    cases.append(case("phase2_n64_q33", np.random.default_rng(11).normal(0, 10, (64, 2)), 33))
    rng = np.random.default_rng(59)
    for k in range(5):
        cases.append(case(f"q2_s{k}", rng.normal(0, 10, (8, 2)), 2))

    # --- dyadic exact fits (test_solver.py:162-175) ---
    rng = np.random.default_rng(41)
    for k in range(10):
        q = int(rng.integers(3, 10))
        xs = rng.permutation(64)[:q].astype(float)
        slope = float(rng.integers(-16, 17)) / 8.0
        intercept = float(rng.integers(-64, 65)) / 8.0
        ys = slope * xs + intercept
        extra = rng.uniform(-50, 50, (q - 1, 2))
        cases.append(case(f"dyadic_{k}", np.vstack([np.column_stack([xs, ys]), extra]), q))

    # --- integer-grid / pixel-like data (ties, duplicate x) ---
    rng = np.random.default_rng(71)
    for k in range(6):
        n = int(rng.integers(20, 120))
        pts = rng.integers(0, 32, (n, 2)).astype(float)
        cases.append(case(f"grid_{k}", pts, None))

    # --- workload configs ---
    for seed in (0, 1):
        cases.append(case(f"config1_s{seed}", workloads.config1_points(seed), 501))
    cases.append(case("config1_noise_s0", workloads.config1_points(0, noise=True), 501))
    cases.append(case("config2_gen_n2000_s0", workloads.contaminated_line_points(2000, 0), None))
    for f in range(2):
        pts = workloads.bench_points(512, seed=f)
        assert np.array_equal(pts, ref_bench_points(512, seed=f))
        cases.append(case(f"bench_points_512_s{f}", pts, 257))

    # --- per-vertex bracelets ---
    brs = []
    rng = np.random.default_rng(13)
    for k in range(15):
        n = int(rng.integers(4, 12))
        pts = rng.normal(0, 5, (n, 2))
        q = int(rng.integers(2, n + 1))
        brs.append(bracelet_case(f"bracelet_{k}", pts, q))
    brs.append(bracelet_case("bracelet_square", [[0, 0], [1, 0], [0, 1], [1, 1]], 3))
    rng = np.random.default_rng(101)
    pts = rng.integers(0, 6, (14, 2)).astype(float)
    brs.append(bracelet_case("bracelet_grid", pts, 6))

    doc = {"generator": "tests/golden/make_golden.py", "reference": "lmsline 0.1.0",
           "numpy": np.__version__, "cases": cases, "bracelets": brs}
    with gzip.open(OUT, "wt") as fh:
        json.dump(doc, fh)
    print(f"wrote {OUT}: {len(cases)} solve cases, {len(brs)} bracelet sets")
    slow = sorted(cases, key=lambda c: -c["ref_seconds"])[:5]
    for c in slow:
        print(f"  {c['name']}: {c['ref_seconds']:.2f}s")


if __name__ == "__main__":
    main()
