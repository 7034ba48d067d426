"""Engine knobs change speed, never records.

Each knob variant solves the same fits as the defaults; the records must be
identical in every field.  Covers the two-phase band bounds (LMSB_DEFER),
the segmented-sort choice (LMSB_SEG_SORT), the cluster exact select
(LMSB_EXACT_CLUSTER / _MAX), the filter slice size (LMSB_BIG_SLICE) and the
graph / device-plan switches, on the config-2 generator (n = 16,384, whose
record is pinned to the reference's own run) and a large-n fit."""

import os

import pytest

from paper_1510_01041_b200 import _native, workloads
from paper_1510_01041_b200.backend import record_from_native

pytestmark = pytest.mark.gpu

VARIANTS = [
    {"LMSB_DEFER": "0"},
    {"LMSB_SEG_SORT": "0"},
    {"LMSB_SEG_SORT": "1"},
    {"LMSB_EXACT_CLUSTER": "0"},
    {"LMSB_EXACT_CLUSTER_MAX": "0"},
    {"LMSB_EXACT_CLUSTER_MAX": "100000"},
    {"LMSB_BIG_SLICE": "65536"},
    {"LMSB_GRAPH": "0", "LMSB_DEVICE_PLAN": "0"},
]


def _record(a, b, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ctx = _native.Context(0)
        ctx.upload(a, b)
        n = a.size
        rec = None
        for _ in range(3):  # the second identical fit is captured, the third replays
            rec = record_from_native(ctx.solve(n // 2 + 1, 0, n * (n - 1) // 2))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return (rec.height, rec.i, rec.j, rec.u, rec.v_low, rec.v_high)


@pytest.mark.parametrize("n,seed", [(16384, 0), (24000, 6)])
def test_knobs_keep_records(n, seed):
    pts = workloads.contaminated_line_points(n, seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    want = _record(a, b, {})
    for env in VARIANTS:
        assert _record(a, b, env) == want, env
