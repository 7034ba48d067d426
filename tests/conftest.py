"""Shared fixtures.  Tests needing a B200 are marked ``gpu``; everything else
runs on the CPU build container."""

import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "lms_golden.json.gz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def _f(h):
    return float.fromhex(h)


class GoldenCase:
    def __init__(self, d):
        self.name = d["name"]
        self.n = d["n"]
        self.q = d["q"]
        self.q_arg = d["q_arg"]
        self.x = np.array([_f(v) for v in d["x"]])
        self.y = np.array([_f(v) for v in d["y"]])
        r = d["record"]
        self.record = None if r is None else {
            "height": _f(r["height"]), "i": r["i"], "j": r["j"], "u": _f(r["u"]),
            "v_low": _f(r["v_low"]), "v_high": _f(r["v_high"])}
        f = d["fit"]
        self.fit = {"slope": _f(f["slope"]), "intercept": _f(f["intercept"]),
                    "lms_value": _f(f["lms_value"]), "slab_height": _f(f["slab_height"]),
                    "coverage": f["coverage"], "contact_indices": tuple(f["contact_indices"])}

    @property
    def points(self):
        return np.column_stack([self.x, self.y])


class GoldenBracelets:
    def __init__(self, d):
        self.name = d["name"]
        self.q = d["q"]
        self.x = np.array([_f(v) for v in d["x"]])
        self.y = np.array([_f(v) for v in d["y"]])
        self.vertices = []
        for v in d["vertices"]:
            br = v["bracelet"]
            self.vertices.append({
                "i": v["i"], "j": v["j"], "u": _f(v["u"]), "v": _f(v["v"]),
                "bracelet": None if br is None else {k: _f(br[k]) for k in ("v_low", "v_high", "height")}})


_cache = {}


def load_golden():
    if "doc" not in _cache:
        with gzip.open(GOLDEN, "rt") as fh:
            doc = json.load(fh)
        _cache["doc"] = ([GoldenCase(c) for c in doc["cases"]],
                         [GoldenBracelets(b) for b in doc["bracelets"]])
    return _cache["doc"]


@pytest.fixture(scope="session")
def golden():
    return load_golden()


def fit_matches(fit, gold: dict) -> bool:
    """Field-by-field equality with ``==`` (so -0.0 == 0.0)."""
    return (fit.line.slope == gold["slope"] and fit.line.intercept == gold["intercept"]
            and fit.lms_value == gold["lms_value"] and fit.slab_height == gold["slab_height"]
            and fit.coverage == gold["coverage"] and tuple(fit.contact_indices) == gold["contact_indices"])


def record_matches(rec, gold: dict | None) -> bool:
    if gold is None:
        return rec is None
    if rec is None:
        return False
    return (rec.i == gold["i"] and rec.j == gold["j"] and rec.height == gold["height"]
            and rec.u == gold["u"] and rec.v_low == gold["v_low"] and rec.v_high == gold["v_high"])
