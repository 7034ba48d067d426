"""The CPU oracle (oracle/) is pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

import oracle
from conftest import record_matches


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def test_oracle_matches_reference_records(golden):
    cases, _ = golden
    threads = min(8, os.cpu_count() or 1)
    checked = 0
    for c in cases:
        rec = oracle.min_bracelet(c.x, c.y, c.q, threads=threads)
        assert record_matches(rec, c.record), c.name
        checked += 1
    assert checked == len(cases) > 150


def test_oracle_fit_mapping_matches_reference(golden):
    cases, _ = golden
    for c in cases:
        if c.record is None:
            continue
        rec = oracle.Record(**c.record)
        fit = oracle.fit_from_record(c.x.copy(), c.y.copy(), c.q, rec)
        for key in ("slope", "intercept", "lms_value", "slab_height", "coverage"):
            assert fit[key] == c.fit[key], (c.name, key)
        assert fit["contact_indices"] == c.fit["contact_indices"], c.name


def test_oracle_bracelets_match_reference(golden):
    _, brs = golden
    total = 0
    for g in brs:
        i = np.array([v["i"] for v in g.vertices])
        j = np.array([v["j"] for v in g.vertices])
        u = np.array([v["u"] for v in g.vertices])
        vv = np.array([v["v"] for v in g.vertices])
        recs = oracle.eval_vertices(g.x, g.y, g.q, i, j, u, vv)
        for rec, v in zip(recs, g.vertices):
            br = v["bracelet"]
            if br is None:
                assert rec is None
                continue
            assert rec is not None
            assert (rec.v_low, rec.v_high) == (br["v_low"], br["v_high"]), g.name
            assert rec.height == br["height"], g.name
            total += 1
    assert total > 200


def test_oracle_partition_invariance():
    rng = np.random.default_rng(5)
    pts = rng.normal(0, 10, (60, 2))
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    ref = oracle.min_bracelet(a, b, 31, threads=1)
    for t in (2, 3, 7):
        assert oracle.min_bracelet(a, b, 31, threads=t) == ref
