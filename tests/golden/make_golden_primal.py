"""Golden vectors for oracle_lms (the reference's primal brute force,
solver.py:143-196), produced by the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_primal.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lmsline import Point2, oracle_lms  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "primal_golden.json.gz")


def hx(v):
    return float(v).hex()


def case(name, pts, q):
    pts = np.asarray(pts, dtype=float)
    fit = oracle_lms(pts, q)
    return {"name": name, "x": [hx(v) for v in pts[:, 0]], "y": [hx(v) for v in pts[:, 1]], "q": q,
            "fit": {"slope": hx(fit.line.slope), "intercept": hx(fit.line.intercept),
                    "lms_value": hx(fit.lms_value), "slab_height": hx(fit.slab_height),
                    "coverage": fit.coverage, "contact_indices": list(fit.contact_indices)}}


def random_points(rng, n, collapse_x=False):
    x = rng.uniform(-100.0, 100.0, n)
    y = rng.uniform(-100.0, 100.0, n)
    if collapse_x and n >= 8 and rng.random() < 0.3:
        k = int(rng.integers(2, n // 2))
        x[:k] = x[0]
    return np.column_stack([x, y])


def main():
    cases = []
    cases.append(case("collinear4", [[0, 1], [1, 3], [2, 5], [3, 7]], 3))
    cases.append(case("square", [[0, 0], [1, 0], [0, 1], [1, 1]], 3))
    maj = [[x, float(x)] for x in range(5)] + [[0.5, 50.0], [1.5, -40.0], [2.5, 90.0], [3.5, 60.0]]
    cases.append(case("majority", maj, 5))
    for n in (4, 8, 16, 32, 64):
        for seed in range(8):
            rng = np.random.default_rng([11, n, seed])
            pts = random_points(rng, n)
            q = int(rng.integers(3, n + 1))
            cases.append(case(f"crit1_n{n}_s{seed}", pts, q))
    for seed in range(16):
        rng = np.random.default_rng([12, seed])
        pts = random_points(rng, 16, collapse_x=True)
        q = int(rng.integers(2, 17))
        cases.append(case(f"degenerate_s{seed}", pts, q))
    rng = np.random.default_rng(53)
    cases.append(case("fixed16", rng.normal(0, 12, (16, 2)), 9))
    rng = np.random.default_rng(71)
    for k in range(4):
        n = int(rng.integers(20, 100))
        cases.append(case(f"grid_{k}", rng.integers(0, 32, (n, 2)).astype(float), n // 2 + 1))
    with gzip.open(OUT, "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden_primal.py", "cases": cases}, fh)
    print(f"wrote {OUT}: {len(cases)} cases")


if __name__ == "__main__":
    main()
