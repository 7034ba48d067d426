"""The band stage's hand-written sorts and the cluster exact select: the
8-CTA cluster segmented sort (lms_segsort.cu) and the whole-GPU slope-sample
bucket sort (lms_samplesort.cu) against numpy, and the cluster exact select
(lms_exact.cu) against the streaming one-CTA-per-vertex select.

The sort can replace the CUB device sorts of the slope samples and of the
large-n band / slice keys (LMSB_SEG_SORT=1; measured slower, so opt-in); its output must be the ascending order of the
unsigned ordered keys (the order a radix sort produces; -0.0 before +0.0),
bit for bit.  The fits that run through it are covered by the golden and
full-size parity tests; here the sort itself meets the cases a regular-
sampling sort can get wrong: ties everywhere, runs shorter than the 8 CTAs
of a cluster, already sorted / reversed input, infinities and signed zeros,
segments with gaps and empty segments."""

import os

import numpy as np
import pytest

from paper_1510_01041_b200 import _native, workloads
from paper_1510_01041_b200.backend import record_from_native

pytestmark = pytest.mark.gpu


def _radix_order(x: np.ndarray) -> np.ndarray:
    u = x.view(np.uint32)
    k = np.where(u >> 31, ~u, u | np.uint32(0x80000000))
    return x[np.argsort(k, kind="stable")]


@pytest.fixture(params=["1", "0"], ids=["bucket", "cluster"], autouse=True)
def seg_impl(request):
    """Every segmented-sort case runs through the segmented bucket sort
    (LMSB_SEG_BUCKET=1) and the cluster sort (the default)."""
    old = os.environ.get("LMSB_SEG_BUCKET")
    os.environ["LMSB_SEG_BUCKET"] = request.param
    yield request.param
    if old is None:
        os.environ.pop("LMSB_SEG_BUCKET", None)
    else:
        os.environ["LMSB_SEG_BUCKET"] = old


def _check(keys, segs):
    keys = np.asarray(keys, dtype=np.float32)
    sb = np.array([s[0] for s in segs], dtype=np.int64)
    se = np.array([s[1] for s in segs], dtype=np.int64)
    got = _native.debug_seg_sort(keys, sb, se)
    want = keys.copy()
    for b, e in segs:
        if e > b:
            want[b:e] = _radix_order(keys[b:e])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 63, 100, 1000, 8191, 8192, 8193, 40000, 65535, 65536])
def test_random_lengths(n):
    rng = np.random.default_rng(n)
    _check(rng.standard_normal(n).astype(np.float32) * 1e3, [(0, n)])


@pytest.mark.parametrize("kind", ["equal", "two", "few", "sorted", "reversed", "special", "heavy"])
def test_adversarial(kind):
    n = 65536
    rng = np.random.default_rng(7)
    if kind == "equal":
        x = np.full(n, 2.5, np.float32)
    elif kind == "two":
        x = np.where(rng.random(n) < 0.999, 1.0, -1.0).astype(np.float32)
    elif kind == "few":
        x = rng.integers(0, 5, n).astype(np.float32)
    elif kind == "sorted":
        x = np.sort(rng.standard_normal(n)).astype(np.float32)
    elif kind == "reversed":
        x = np.sort(rng.standard_normal(n))[::-1].astype(np.float32).copy()
    elif kind == "special":
        x = rng.standard_normal(n).astype(np.float32)
        idx = rng.integers(0, n, 4000)
        x[idx[:1000]] = np.inf
        x[idx[1000:2000]] = -np.inf
        x[idx[2000:3000]] = 0.0
        x[idx[3000:]] = -0.0
        x[:10] = np.float32(1e-45)
    else:  # half the keys in one tight cluster (the inlier lines at the fit slope)
        x = np.concatenate([rng.standard_normal(n // 2) * 1e-6 + 3.0,
                            rng.standard_cauchy(n - n // 2) * 1e4]).astype(np.float32)
        rng.shuffle(x)
    _check(x, [(0, n)])


def test_many_segments_with_gaps_and_empties():
    rng = np.random.default_rng(3)
    lens = [65536, 0, 17, 30000, 0, 8, 65536, 1, 12345, 0, 4096]
    segs, pos = [], 5
    for L in lens:
        segs.append((pos, pos + L))
        pos += L + int(rng.integers(0, 9))
    keys = rng.standard_normal(pos + 3).astype(np.float32)
    keys[segs[3][0]:segs[3][1]] = rng.integers(0, 3, lens[3])
    _check(keys, segs)


def test_big_band_fit_same_as_cub_sorts():
    """A large-n band fit (n > 16,384: sample, per-band and per-slice sorts
    all run through the cluster sort) gives the same record and the same
    band count as with the CUB device sorts (the default; LMSB_SEG_SORT=1
    selects the cluster sort).  (Survivor
    counts depend on when the persistent filter CTAs see the falling best
    height, so they are not compared.)"""
    pts = workloads.contaminated_line_points(20000, 5)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    n = a.size
    out = []
    for seg in ("1", "0"):
        os.environ["LMSB_SEG_SORT"] = seg
        try:
            ctx = _native.Context(0)
            ctx.upload(a, b)
            rec = record_from_native(ctx.solve(n // 2 + 1, 0, n * (n - 1) // 2))
            st = ctx.stats()
        finally:
            os.environ.pop("LMSB_SEG_SORT", None)
        out.append(((rec.height, rec.i, rec.j, rec.u, rec.v_low, rec.v_high), st["bands"]))
    assert out[0] == out[1]


@pytest.mark.parametrize("n,seed", [(20000, 1), (40000, 4), (65536, 0)])
def test_exact_cluster_select_same_as_streaming(n, seed):
    """Seeds and survivors of fits above 16,384 lines are evaluated by one
    8-CTA cluster per vertex (LMSB_EXACT_CLUSTER, default on); the record
    (and every field of it) equals the streaming select's."""
    pts = workloads.contaminated_line_points(n, seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    out = []
    for flag in ("1", "0"):
        os.environ["LMSB_EXACT_CLUSTER"] = flag
        try:
            ctx = _native.Context(0)
            ctx.upload(a, b)
            rec = record_from_native(ctx.solve(n // 2 + 1, 0, n * (n - 1) // 2))
        finally:
            os.environ.pop("LMSB_EXACT_CLUSTER", None)
        out.append((rec.height, rec.i, rec.j, rec.u, rec.v_low, rec.v_high))
    assert out[0] == out[1]


@pytest.mark.parametrize("n", [1, 2, 5, 1000, 1023, 1024, 1025, 65536, 100003, 1 << 20])
def test_sample_sort_random(n):
    rng = np.random.default_rng(n)
    x = (rng.standard_cauchy(n) * 10).astype(np.float32)
    got = _native.debug_sample_sort(x)
    assert np.array_equal(got.view(np.uint32), _radix_order(x).view(np.uint32))


@pytest.mark.parametrize("kind", ["equal", "infs", "few", "periodic", "sorted", "reversed", "special"])
def test_sample_sort_adversarial(kind):
    """Ties everywhere, invalid samples (+inf), and a periodic input whose
    every 64th key (the splitter sample) differs from all the others: one
    bucket then holds almost every key (the chunked merge fallback)."""
    n = 65536
    rng = np.random.default_rng(11)
    if kind == "equal":
        x = np.full(n, -3.25, np.float32)
    elif kind == "infs":
        x = rng.standard_normal(n).astype(np.float32)
        x[rng.random(n) < 0.6] = np.inf
    elif kind == "few":
        x = rng.integers(-2, 3, n).astype(np.float32)
    elif kind == "periodic":
        x = np.full(n, 7.0, np.float32)
        x[64::128] = rng.standard_normal(n // 128).astype(np.float32) * 100
        x[:5000] = rng.standard_normal(5000).astype(np.float32)
    elif kind == "sorted":
        x = np.sort(rng.standard_normal(n)).astype(np.float32)
    elif kind == "reversed":
        x = np.sort(rng.standard_normal(n))[::-1].astype(np.float32).copy()
    else:
        x = rng.standard_normal(n).astype(np.float32)
        x[::7] = 0.0
        x[::11] = -0.0
        x[::13] = -np.inf
    got = _native.debug_sample_sort(x)
    want = _radix_order(x)
    if kind == "special":  # -0.0 / +0.0 order is free (no caller tells them apart)
        assert np.array_equal(got, want)
    else:
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("case", ["grid", "collinear_majority", "dup_x", "huge_outliers"])
def test_exact_cluster_select_adversarial(case):
    """The cluster select on inputs full of ties (integer grids: many equal
    cut values, exact-zero heights), a collinear majority (height 0), shared
    x values (parallel duals) and 1e6 outliers, above the 16,384-line cache
    limit: the same record as the streaming select."""
    rng = np.random.default_rng(21)
    n = 20000
    if case == "grid":
        pts = rng.integers(0, 300, (n, 2)).astype(float)
    elif case == "collinear_majority":
        x = rng.uniform(-50, 50, n)
        y = 0.5 * x - 3.0
        k = rng.random(n) < 0.45
        y[k] = rng.uniform(-500, 500, k.sum())
        pts = np.column_stack([x, y])
    elif case == "dup_x":
        x = np.round(rng.uniform(0, 40, n), 1)
        pts = np.column_stack([x, -1.5 * x + rng.normal(0, 0.05, n)])
    else:
        pts = workloads.contaminated_line_points(n, 9)
        pts[: n // 10, 1] += 1e6
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    out = []
    for flag in ("1", "0"):
        os.environ["LMSB_EXACT_CLUSTER"] = flag
        try:
            ctx = _native.Context(0)
            ctx.upload(a, b)
            rec = record_from_native(ctx.solve(n // 2 + 1, 0, n * (n - 1) // 2))
        finally:
            os.environ.pop("LMSB_EXACT_CLUSTER", None)
        out.append((rec.height, rec.i, rec.j, rec.u, rec.v_low, rec.v_high))
    assert out[0] == out[1]
