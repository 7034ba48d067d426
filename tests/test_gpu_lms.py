"""GPU parity: the sm_100a engine against the reference's golden vectors and
the CPU oracle (bit-exact on the winning record), plus size-independent
properties at BASELINE.json's full sizes."""

import os

import numpy as np
import pytest

import oracle
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import _native, workloads
from paper_1510_01041_b200.backend import record_from_native
from conftest import fit_matches, record_matches

pytestmark = pytest.mark.gpu
THREADS = min(16, os.cpu_count() or 1)


@pytest.fixture(scope="module", autouse=True)
def _ready():
    oracle.build()
    assert _native.device_count() > 0, "no CUDA device"


def oracle_rec(a, b, q, r0=0, r1=None):
    rec = oracle.min_bracelet(a, b, q, r0, r1, threads=THREADS)
    if rec is None:
        return None
    return {"height": rec.height, "i": rec.i, "j": rec.j, "u": rec.u, "v_low": rec.v_low,
            "v_high": rec.v_high}


def gpu_range(a, b, q, r0, r1):
    return record_from_native(_native.min_bracelet(a, b, q, r0, r1))


def test_golden_records_and_fits(golden):
    cases, _ = golden
    for c in cases:
        rec = lms.get_backend("seq").minimum_bracelet(c.x.copy(), c.y.copy(), c.q)
        assert record_matches(rec, c.record), c.name
        fit = lms.solve_lms(c.points, c.q_arg)
        assert fit_matches(fit, c.fit), c.name


def test_golden_bracelets(golden):
    _, brs = golden
    for g in brs:
        lines = lms.dualize(np.column_stack([g.x, g.y]))
        for v in g.vertices:
            ip = lms.DualIntersection(u=v["u"], v=v["v"], i=v["i"], j=v["j"])
            br = lms.bracelet_at(ip, lines, g.q)
            want = v["bracelet"]
            if want is None:
                assert br is None
            else:
                assert (br.v_low, br.v_high, br.height) == (want["v_low"], want["v_high"], want["height"])


def test_bracelet_duplicate_and_absent_anchor_ids():
    """bracelet_at snaps every line whose source index is i or j and does not
    raise for absent anchors (geometry.py:199-203), as the reference does
    (tests/golden/make_golden_bracelet_edges.py)."""
    import json
    import os

    rows = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bracelet_edges_golden.json")))
    for r in rows:
        lines = [lms.DualLine(a=a, b=b, source_index=s) for a, b, s in zip(r["a"], r["b"], r["src"])]
        ip = lms.DualIntersection(u=float.fromhex(r["u"]), v=float.fromhex(r["v"]), i=r["i"], j=r["j"])
        br = lms.bracelet_at(ip, lines, r["q"])
        if r["bracelet"] is None:
            assert br is None
        else:
            assert (br.v_low, br.v_high, br.height) == tuple(float.fromhex(h) for h in r["bracelet"])


def test_phase2_matches_oracle_and_bracelets(golden):
    _, brs = golden
    for g in brs:
        lines = lms.dualize(np.column_stack([g.x, g.y]))
        ips = list(lms.run_phase1(lines))
        rec = lms.run_phase2(ips, lines, g.q, worker_count=3)
        want = oracle_rec(g.x, g.y, g.q)
        assert record_matches(rec, want), g.name


def random_points(rng, n, collapse_x=False):
    x = rng.uniform(-100.0, 100.0, n)
    y = rng.uniform(-100.0, 100.0, n)
    if collapse_x and n >= 8 and rng.random() < 0.3:
        k = int(rng.integers(2, n // 2))
        x[:k] = x[0]
    return x, y


def test_random_instances_bit_exact_vs_oracle():
    rng = np.random.default_rng(2024)
    for trial in range(120):
        n = int(rng.integers(3, 300))
        kind = trial % 4
        if kind == 0:
            x, y = random_points(rng, n, collapse_x=True)
        elif kind == 1:
            x, y = rng.integers(0, 24, n).astype(float), rng.integers(0, 24, n).astype(float)
        elif kind == 2:
            pts = workloads.config1_points(trial, n=max(n, 8))
            x, y = pts[:, 0].copy(), pts[:, 1].copy()
            n = x.size
        else:
            x, y = rng.normal(0, 1e3, n), rng.normal(0, 1e-3, n)
        if np.unique(x).size < 2:
            continue
        q = int(rng.integers(2, n + 1)) if trial % 3 else n // 2 + 1
        rec = lms.get_backend("seq").minimum_bracelet(x, y, q)
        assert record_matches(rec, oracle_rec(x, y, q)), (trial, n, q)


def test_filter_path_subranges_bit_exact_at_n16k():
    """n = 16,384 (config 2): rank sub-ranges large enough to take the
    filter path, at the start, middle and end of the triangle."""
    pts = workloads.contaminated_line_points(16384, 0)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = 16384 // 2 + 1
    total = 16384 * 16383 // 2
    for r0 in (0, total // 3 + 12345, total - 9000):
        r1 = min(total, r0 + 9000)
        got = gpu_range(a, b, q, r0, r1)
        assert record_matches(got, oracle_rec(a, b, q, r0, r1)), r0


def test_config1_full_bit_exact(golden):
    cases, _ = golden
    c = {g.name: g for g in cases}["config1_s0"]
    ctx = _native.Context()
    ctx.upload(c.x, c.y)
    rec = record_from_native(ctx.solve(c.q, 0, c.n * (c.n - 1) // 2))
    assert record_matches(rec, c.record)
    st = ctx.stats()
    assert st["survivors"] < st["pairs"]


def test_config2_full_n16k_properties():
    """Full n = 16,384 fit: the winner re-evaluates identically on the CPU,
    partitions merge to the same record, and the fit satisfies the LMS
    equioscillation / median properties."""
    pts = workloads.contaminated_line_points(16384, 0)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = 16384 // 2 + 1
    total = 16384 * 16383 // 2
    ctx = _native.Context()
    ctx.upload(a, b)
    rec = record_from_native(ctx.solve(q, 0, total))
    assert rec is not None
    (chk,) = oracle.eval_vertices(a, b, q, [rec.i], [rec.j], [rec.u])
    assert (chk.height, chk.v_low, chk.v_high) == (rec.height, rec.v_low, rec.v_high)
    parts = lms.BatchPlan.create(a, 4).partitions()
    merged = None
    for r0, r1 in parts:
        merged = lms.backend.merge(merged, record_from_native(ctx.solve(q, r0, r1)))
    assert merged == rec
    fit = lms.solver.fit_from_record(a, b, q, rec)
    med = lms.median_sq_residual(pts, fit.line, q)
    assert med == pytest.approx(fit.lms_value, rel=1e-9)
    assert abs(fit.line.slope - 2.0) < 0.01
    assert len(fit.contact_indices) >= 3


def test_planted_exact_fit_n16k():
    rng = np.random.default_rng(7)
    n = 16384
    q = n // 2 + 1
    x = rng.permutation(1 << 20)[:n].astype(float)
    y = rng.uniform(-1e6, 1e6, n)
    inl = rng.permutation(n)[:q]
    y[inl] = 0.75 * x[inl] - 3.5  # dyadic: exact in binary
    fit = lms.solve_lms(np.column_stack([x, y]))
    assert fit.lms_value == 0.0
    assert fit.line.slope == 0.75 and fit.line.intercept == -3.5


def test_edge_cases_vs_oracle():
    cases = []
    cases.append(([0, 1, 2], [0, 1, 5], 2))
    cases.append(([0, 1, 2], [0, 1, 5], 3))
    cases.append(([1, 1, 1, 1, 2], [0, 1, 2, 3, 1], 2))
    cases.append(([0, 0, 1, 2, 1], [0, 0, 1, 2, 5], 4))
    cases.append(([-0.0, 0.0, 1, -1, 2], [0.0, -0.0, 0.0, -0.0, 1e-300], 3))
    big = np.random.default_rng(3).normal(0, 1e150, (40, 2))
    cases.append((big[:, 0], big[:, 1], 21))
    tiny = np.random.default_rng(4).normal(0, 1e-150, (40, 2))
    cases.append((tiny[:, 0], tiny[:, 1], 21))
    mixed = np.random.default_rng(5).normal(0, 1, (50, 2)) * np.logspace(-100, 100, 50)[:, None]
    cases.append((mixed[:, 0], mixed[:, 1], 26))
    for x, y, q in cases:
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        for qq in (q, x.size):
            rec = lms.get_backend("seq").minimum_bracelet(x, y, qq)
            assert record_matches(rec, oracle_rec(x, y, qq)), (x.size, qq)


def test_seq_par_identical():
    rng = np.random.default_rng(19)
    for _ in range(6):
        n = int(rng.integers(5, 400))
        pts = rng.normal(0, 20, (n, 2))
        ref = lms.solve_lms(pts, backend="seq")
        for w in (1, 3, 7):
            assert lms.solve_lms(pts, backend="par", workers=w) == ref
        assert lms.solve_lms(pts, materialize=True) == ref


def test_batched_matches_golden_and_single(golden):
    cases, _ = golden
    sel = [c for c in cases if c.n <= 600]
    fits = lms.solve_lms_batch([c.points for c in sel], [c.q_arg if c.q_arg is not None else c.q for c in sel])
    for c, fit in zip(sel, fits):
        assert fit_matches(fit, c.fit), c.name


def test_batched_config4_slice_vs_oracle():
    sets = [workloads.bench_points(512, seed=f) for f in range(24)]
    fits = lms.solve_lms_batch(sets, 257)
    for f, (pts, fit) in enumerate(zip(sets, fits)):
        want = oracle.solve(pts, 257, threads=THREADS)
        assert fit.line.slope == want["slope"] and fit.line.intercept == want["intercept"], f
        assert fit.lms_value == want["lms_value"] and tuple(fit.contact_indices) == want["contact_indices"]


def test_batched_mixed_sizes_vs_oracle():
    rng = np.random.default_rng(404)
    sets, qs = [], []
    for k in range(40):
        n = int(rng.choice([3, 5, 17, 90, 91, 200, 700, 1500]))
        x = rng.uniform(-50, 50, n)
        if k % 5 == 0:
            x[: n // 3] = x[0]
        y = 0.5 * x + rng.normal(0, 1, n)
        bad = rng.random(n) < 0.4
        y[bad] = rng.uniform(-500, 500, int(bad.sum()))
        pts = np.column_stack([x, y])
        if np.unique(x).size < 2:
            continue
        sets.append(pts)
        qs.append(int(rng.integers(2, n + 1)))
    fits = lms.solve_lms_batch(sets, qs)
    for pts, q, fit in zip(sets, qs, fits):
        want = oracle.solve(pts, q, threads=THREADS)
        assert (fit.line.slope, fit.line.intercept, fit.lms_value) == (want["slope"], want["intercept"], want["lms_value"])


def test_oracle_lms_matches_reference_primal_brute_force():
    import gzip
    import json

    path = os.path.join(os.path.dirname(__file__), "golden", "primal_golden.json.gz")
    with gzip.open(path, "rt") as fh:
        cases = json.load(fh)["cases"]
    for c in cases:
        pts = np.column_stack([[float.fromhex(v) for v in c["x"]], [float.fromhex(v) for v in c["y"]]])
        fit = lms.oracle_lms(pts, c["q"])
        want = {k: (float.fromhex(v) if isinstance(v, str) else v) for k, v in c["fit"].items()}
        want["contact_indices"] = tuple(want["contact_indices"])
        assert fit_matches(fit, want), c["name"]


def test_solver_and_primal_agree_at_moderate_n():
    rng = np.random.default_rng(909)
    for n in (100, 300):
        pts = workloads.contaminated_line_points(n, int(rng.integers(1000)))
        a, b = lms.solve_lms(pts), lms.oracle_lms(pts)
        assert a.lms_value == pytest.approx(b.lms_value, rel=1e-9)
        assert a.line.slope == pytest.approx(b.line.slope, rel=1e-9, abs=1e-12)


def _ctx_with(env: dict):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return _native.Context()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_band_path_matches_count_filter_path_config2():
    """The slope-band stage (default) and the count-filter path give the
    identical record on the full n = 16,384 fit, and on partitions."""
    pts = workloads.contaminated_line_points(16384, 0)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = 16384 // 2 + 1
    total = 16384 * 16383 // 2
    band = _ctx_with({"LMSB_BAND": "1"})
    filt = _ctx_with({"LMSB_BAND": "0"})
    for c in (band, filt):
        c.upload(a, b)
    for r0, r1 in ((0, total), (0, total // 3), (total // 3, total)):
        got = band.solve(q, r0, r1)
        st = band.stats()
        assert st["bands"] > 0, "band stage did not run"
        want = filt.solve(q, r0, r1)
        assert filt.stats()["bands"] == 0
        assert record_from_native(got) == record_from_native(want), (r0, r1)


def test_band_path_bit_exact_vs_oracle_mid_n():
    """Band stage at n in the thousands (many bands, small ones) against
    the CPU oracle, including noisy, exact-inlier and integer-grid inputs."""
    rng = np.random.default_rng(99)
    for trial in range(6):
        n = int(rng.integers(600, 1500))
        if trial % 3 == 0:
            pts = workloads.contaminated_line_points(n, trial)
        elif trial % 3 == 1:
            pts = workloads.config1_points(trial, n=n)
        else:
            pts = np.column_stack([rng.integers(0, 60, n), rng.integers(0, 60, n)]).astype(float)
        x, y = pts[:, 0].copy(), pts[:, 1].copy()
        q = n // 2 + 1 if trial % 2 == 0 else int(rng.integers(2, n + 1))
        ctx = _ctx_with({"LMSB_BAND": "2", "LMSB_BAND_VERTICES": "2048"})
        ctx.upload(x, y)
        total = n * (n - 1) // 2
        got = record_from_native(ctx.solve(q, 0, total))
        assert ctx.stats()["bands"] > 1
        want = oracle_rec(x, y, q)
        assert record_matches(got, want), (trial, n, q)


def test_band_path_matches_count_filter_varied_inputs():
    """Forced band stage vs the count-filter path (itself pinned to the
    oracle) on n = 2,000-6,000 inputs with ties, duplicate x, exact inliers,
    huge outliers, vertical and horizontal structure."""
    rng = np.random.default_rng(5)
    cases = []
    n = 3000
    cases.append(workloads.config1_points(3, n=n))                      # exact inliers: h = 0 ties
    x = rng.integers(0, 200, n).astype(float)                            # duplicate x, integer grid
    cases.append(np.column_stack([x, rng.integers(0, 200, n).astype(float)]))
    x = rng.uniform(0, 1, n)
    y = np.where(rng.random(n) < 0.6, 3.0 - 0.5 * x, rng.uniform(-1e6, 1e6, n))
    cases.append(np.column_stack([x, y]))                                # breakdown: 1e6 outliers
    x = rng.normal(0, 1e3, 4000)
    cases.append(np.column_stack([x, rng.normal(0, 1e-3, 4000)]))        # near-horizontal
    x = np.concatenate([np.full(1500, 7.0), rng.uniform(0, 10, 1500)])   # vertical majority
    cases.append(np.column_stack([x, rng.uniform(0, 10, 3000)]))
    cases.append(workloads.contaminated_line_points(6000, 4))
    band = _ctx_with({"LMSB_BAND": "2"})
    filt = _ctx_with({"LMSB_BAND": "0"})
    for k, pts in enumerate(cases):
        a, b = pts[:, 0].copy(), pts[:, 1].copy()
        m = a.size
        for q in (m // 2 + 1, max(2, m // 4), m - 3):
            total = m * (m - 1) // 2
            band.upload(a, b)
            filt.upload(a, b)
            got = record_from_native(band.solve(q, 0, total))
            assert band.stats()["bands"] > 0
            want = record_from_native(filt.solve(q, 0, total))
            assert got == want, (k, q)


def test_small_fit_kernel_matches_count_filter_batch():
    """Fused per-fit band kernel (batches of fits with n <= 1,024) vs the
    count-filter batch path on 600 varied fits: config-4 sets, exact
    inliers, integer grids with duplicate x, huge outliers, random q."""
    rng = np.random.default_rng(77)
    sets, qs = [], []
    for k in range(600):
        kind = k % 5
        n = int(rng.choice([92, 150, 256, 333, 512, 700, 1024]))
        if kind == 0:
            pts = workloads.bench_points(n, seed=k)
        elif kind == 1:
            pts = workloads.config1_points(k, n=n)
        elif kind == 2:
            pts = np.column_stack([rng.integers(0, 40, n), rng.integers(0, 40, n)]).astype(float)
        elif kind == 3:
            x = rng.uniform(0, 1, n)
            y = np.where(rng.random(n) < 0.6, 3.0 - 0.5 * x, rng.uniform(-1e6, 1e6, n))
            pts = np.column_stack([x, y])
        else:
            pts = np.column_stack([rng.normal(0, 100, n), rng.normal(0, 1, n)])
        if np.unique(pts[:, 0]).size < 2:
            continue
        sets.append(pts)
        qs.append(n // 2 + 1 if k % 3 else int(rng.integers(2, n + 1)))
    X = np.concatenate([s[:, 0] for s in sets])
    Y = np.concatenate([s[:, 1] for s in sets])
    offs = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int64)
    q = np.asarray(qs, dtype=np.int64)
    fused = _ctx_with({"LMSB_SMALL": "1"})
    legacy = _ctx_with({"LMSB_SMALL": "0"})
    fused.upload(X, Y)
    legacy.upload(X, Y)
    got = fused.solve_batch(offs, q)
    assert fused.stats()["small_fits"] == len(sets)
    want = legacy.solve_batch(offs, q)
    assert legacy.stats()["small_fits"] == 0
    for f, (g, w) in enumerate(zip(got, want)):
        assert record_from_native(g) == record_from_native(w), f


def test_band_path_large_n_matches_count_filter():
    """n > 16,384 takes the large-n band path (global segmented sorts, 16-bit
    quantised keys): same record as the count-filter path."""
    for n, seed in ((20000, 1), (24000, 2)):
        pts = workloads.contaminated_line_points(n, seed)
        a, b = pts[:, 0].copy(), pts[:, 1].copy()
        q = n // 2 + 1
        total = n * (n - 1) // 2
        band = _ctx_with({"LMSB_BAND": "1"})
        filt = _ctx_with({"LMSB_BAND": "0"})
        band.upload(a, b)
        filt.upload(a, b)
        got = record_from_native(band.solve(q, 0, total))
        assert band.stats()["bands"] > 0
        want = record_from_native(filt.solve(q, 0, total))
        assert got == want, n


def test_config3_n65536_band_path_properties():
    """Config 3 (n = 65,536) on one GPU: the winner re-evaluates identically
    on the CPU oracle and two rank partitions merge to the same record."""
    n = 65536
    pts = workloads.contaminated_line_points(n, 0)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(a, b)
    rec = record_from_native(ctx.solve(q, 0, total))
    assert ctx.stats()["bands"] > 0
    (chk,) = oracle.eval_vertices(a, b, q, [rec.i], [rec.j], [rec.u])
    assert (chk.height, chk.v_low, chk.v_high) == (rec.height, rec.v_low, rec.v_high)
    half = total // 2
    merged = lms.backend.merge(record_from_native(ctx.solve(q, 0, half)),
                               record_from_native(ctx.solve(q, half, total)))
    assert merged == rec
    assert abs(rec.u - 2.0) < 0.01


@pytest.mark.parametrize("block", range(4))
def test_band_path_random_sweep_vs_count_filter(block):
    """Forced band stage vs the count-filter path on 40 random instances per
    block: mixtures of lines, clusters, heavy-tailed noise, rounded
    coordinates (ties) and random q."""
    rng = np.random.default_rng(1000 + block)
    band = _ctx_with({"LMSB_BAND": "2", "LMSB_BAND_VERTICES": str(int(rng.choice([4096, 16384, 65536])))})
    filt = _ctx_with({"LMSB_BAND": "0"})
    for t in range(40):
        n = int(rng.integers(2100, 3600))
        kind = t % 5
        x = rng.uniform(-1, 1, n) * 10 ** rng.uniform(0, 4)
        if kind == 0:
            y = rng.normal(0, 1, n) + rng.uniform(-3, 3) * x
        elif kind == 1:
            y = np.where(rng.random(n) < 0.5, 0.3 * x + 5, -2.0 * x + rng.standard_cauchy(n))
        elif kind == 2:
            x = np.round(x)
            y = np.round(rng.normal(0, 50, n))
        elif kind == 3:
            c = rng.integers(0, 5, n)
            y = c * 100.0 + rng.normal(0, 1, n) + 0.1 * x
        else:
            y = np.where(rng.random(n) < 0.3, 7.0, rng.normal(0, 1e4, n))
        if np.unique(x).size < 2:
            continue
        q = int(rng.integers(2, n + 1)) if t % 2 else n // 2 + 1
        total = n * (n - 1) // 2
        band.upload(x, y)
        filt.upload(x, y)
        got = record_from_native(band.solve(q, 0, total))
        assert band.stats()["bands"] > 0
        want = record_from_native(filt.solve(q, 0, total))
        assert got == want, (block, t, n, q)


def test_band_path_degenerate_q_many_ties():
    """q = 2: every vertex has height 0, the band stage admits everything and
    the exact stage sees a huge tied list; the winner is the smallest pair."""
    n = 3000
    pts = workloads.contaminated_line_points(n, 9)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    total = n * (n - 1) // 2
    band = _ctx_with({"LMSB_BAND": "2"})
    filt = _ctx_with({"LMSB_BAND": "0"})
    band.upload(a, b)
    filt.upload(a, b)
    for q in (2, 3):
        got = record_from_native(band.solve(q, 0, total))
        want = record_from_native(filt.solve(q, 0, total))
        assert got == want, q


def test_materialized_two_kernel_flow_matches():
    """materialize=True (K1 materialises every (i, j, u), K2 evaluates each
    exactly, no pruning) gives the streaming engine's record: vs the oracle
    at small n, vs the band stage on a full n = 8,192 fit."""
    rng = np.random.default_rng(31)
    for t in range(6):
        n = int(rng.integers(20, 400))
        pts = workloads.config1_points(t, n=n) if t % 2 else workloads.contaminated_line_points(n, t)
        x, y = pts[:, 0].copy(), pts[:, 1].copy()
        q = n // 2 + 1
        got = lms.get_backend("seq").minimum_bracelet(x, y, q, materialize=True)
        assert record_matches(got, oracle_rec(x, y, q)), t
    n = 8192
    pts = workloads.contaminated_line_points(n, 5)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(a, b)
    full = record_from_native(ctx.solve_materialized(q, 0, total))
    band = record_from_native(ctx.solve(q, 0, total))
    assert ctx.stats()["bands"] > 0
    assert full == band
    fit = lms.solve_lms(pts, materialize=True)
    assert fit.line.slope == full.u


def test_config2_full_fit_matches_unpruned_materialized_flow():
    """BASELINE config 2 at full size (n = 16,384): the pruned slope-band
    search returns exactly the record of the unpruned K1/K2 flow, which
    evaluates all 134,209,536 vertices with the reference's arithmetic."""
    n = 16384
    pts = workloads.contaminated_line_points(n, 0)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(a, b)
    band = record_from_native(ctx.solve(q, 0, total))
    assert ctx.stats()["bands"] > 0
    full = record_from_native(ctx.solve_materialized(q, 0, total))
    assert full == band


def test_config2_full_fit_matches_reference_golden():
    """BASELINE config 2 (n = 16,384, 49 % outliers) against the reference's
    own run: lmsline.solve_lms(pts, backend="par", workers=8) took 70 min on
    8 cores (tests/golden/make_golden_config2.py).  Record, fit and contact
    set bit-equal, through seq, par (4 shards on this GPU) and the raw
    record API."""
    import hashlib
    import json

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config2_golden.json")))
    n = gold["n"]
    pts = workloads.contaminated_line_points(n, 0)
    assert hashlib.sha256(pts.tobytes()).hexdigest() == gold["points_sha256"]
    r = gold["record"]
    want_rec = lms.CandidateRecord(height=float.fromhex(r["height"]), i=r["i"], j=r["j"],
                                   u=float.fromhex(r["u"]), v_low=float.fromhex(r["v_low"]),
                                   v_high=float.fromhex(r["v_high"]))
    f = gold["fit"]
    want_fit = {"slope": float.fromhex(f["slope"]), "intercept": float.fromhex(f["intercept"]),
                "lms_value": float.fromhex(f["lms_value"]), "slab_height": float.fromhex(f["slab_height"]),
                "coverage": f["coverage"], "contact_indices": tuple(f["contact_indices"])}
    rec = lms.get_backend("seq").minimum_bracelet(pts[:, 0].copy(), pts[:, 1].copy(), gold["q"])
    assert rec == want_rec
    assert fit_matches(lms.solve_lms(pts), want_fit)
    old = os.environ.get("LMSB_PAR_SHARDS")
    os.environ["LMSB_PAR_SHARDS"] = "4"
    try:
        assert fit_matches(lms.solve_lms(pts, backend="par", workers=4), want_fit)
    finally:
        if old is None:
            os.environ.pop("LMSB_PAR_SHARDS", None)
        else:
            os.environ["LMSB_PAR_SHARDS"] = old


def test_config3_full_fit_matches_unpruned_materialized_flow():
    """BASELINE config 3 at full size (n = 65,536): the pruned large-n band
    search returns exactly the record of the unpruned K1/K2 flow over all
    2,147,450,880 vertices (the reference's arithmetic on every vertex, no
    filter; minutes on one B200)."""
    n = 65536
    pts = workloads.contaminated_line_points(n, 0)
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(pts[:, 0].copy(), pts[:, 1].copy())
    band = record_from_native(ctx.solve(q, 0, total))
    assert ctx.stats()["bands"] > 0
    full = record_from_native(ctx.solve_materialized(q, 0, total))
    assert full == band


def _ctx_env(**env):
    import os

    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return _native.Context()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", ["config2", "grid", "outliers", "dupx", "near_parallel", "shards"])
def test_sweep_collect_matches_pretest_collect(case):
    """The output-sensitive sweep collect (lms_sweep.cu) hands the filter the
    same member set as the pre-test pass over every vertex: identical
    records and collected counts, on inputs with duplicate x, integer grids,
    1e6 outliers, nearly parallel lines, and per-shard rank ranges."""
    rng = np.random.default_rng(7)
    if case == "config2":
        pts = workloads.contaminated_line_points(16384, 0)
    elif case == "grid":
        pts = rng.integers(0, 300, (5000, 2)).astype(float)
    elif case == "outliers":
        pts = workloads.contaminated_line_points(4000, 2)
        pts[:200, 1] += 1e6
    elif case == "dupx":
        x = rng.uniform(0, 1, 4096)
        x[::7] = x[0]
        pts = np.column_stack([x, 3 * x + rng.normal(0, 0.01, 4096)])
    elif case == "near_parallel":
        x = 1.0 + np.arange(3000) * 1e-12
        pts = np.column_stack([x, rng.normal(0, 1, 3000)])
    else:
        pts = workloads.contaminated_line_points(6000, 4)
    n = len(pts)
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ranges = [(0, total)] if case != "shards" else [(0, total // 3), (total // 3, total - 5), (total - 5, total)]
    c0, c1 = _ctx_env(LMSB_SWEEP=0, LMSB_BAND=2), _ctx_env(LMSB_SWEEP=1, LMSB_BAND=2)
    for c in (c0, c1):
        c.upload(pts[:, 0].copy(), pts[:, 1].copy())
    for r0, r1 in ranges:
        a = record_from_native(c0.solve(q, r0, r1))
        sa = c0.stats()
        b = record_from_native(c1.solve(q, r0, r1))
        sb = c1.stats()
        assert a == b, (case, r0, r1)
        if sa["bands"] > 0 and sb["sweep_runs"] > 0:
            assert sa["filtered_vertices"] == sb["filtered_vertices"], (case, r0, r1)


@pytest.mark.parametrize("scale", [(1e-8, 1e8), (1e12, 1.0), (1.0, 1e-12), (3e5, 3e5)])
def test_band_and_filter_paths_vs_unpruned_at_extreme_scales(scale):
    """The fp32 pre-tests of both pruned searches carry magnitude-scaled
    margins: at extreme coordinate scales they still return the record of
    the unpruned K1/K2 flow (exact arithmetic only)."""
    sx, sy = scale
    rng = np.random.default_rng(int(np.log10(sx * sy + 1e-300) + 400))
    n = 2500
    pts = workloads.contaminated_line_points(n, 3)
    x = (pts[:, 0] + rng.uniform(0, 1e-3, n)) * sx
    y = pts[:, 1] * sy
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ref = _native.Context()
    ref.upload(x, y)
    want = record_from_native(ref.solve_materialized(q, 0, total))
    for env in ({"LMSB_BAND": "2", "LMSB_SWEEP": "0"}, {"LMSB_BAND": "2", "LMSB_SWEEP": "1"},
                {"LMSB_BAND": "0"}):
        ctx = _ctx_with(env)
        ctx.upload(x, y)
        got = record_from_native(ctx.solve(q, 0, total))
        assert got == want, (scale, env)


def test_small_fit_kernel_vs_unpruned_at_extreme_scales():
    """Fused small-fit kernel at extreme coordinate scales (and odd n, which
    takes the element-load path instead of the bulk copy) against the
    unpruned K1/K2 flow of every fit."""
    rng = np.random.default_rng(8)
    sets = []
    for k, (sx, sy) in enumerate([(1e-8, 1e8), (1e12, 1.0), (1.0, 1e-12), (3e5, 3e5)] * 6):
        n = int(rng.choice([257, 300, 511, 512, 999]))
        pts = workloads.bench_points(n, seed=100 + k)
        sets.append(np.column_stack([(pts[:, 0] + rng.uniform(0, 1e-3, n)) * sx, pts[:, 1] * sy]))
    X = np.concatenate([s[:, 0] for s in sets])
    Y = np.concatenate([s[:, 1] for s in sets])
    offs = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int64)
    q = np.asarray([len(s) // 2 + 1 for s in sets], dtype=np.int64)
    ctx = _ctx_with({"LMSB_SMALL": "1"})
    ctx.upload(X, Y)
    got = ctx.solve_batch(offs, q)
    assert ctx.stats()["small_fits"] == len(sets)
    ref = _native.Context()
    for f, s in enumerate(sets):
        ref.upload(s[:, 0], s[:, 1])
        m = len(s)
        want = record_from_native(ref.solve_materialized(int(q[f]), 0, m * (m - 1) // 2))
        assert record_from_native(got[f]) == want, f


def test_band_direct_grouping_matches():
    """The direct sub-band grouping variant of the collect pass
    (LMSB_BAND_DIRECT=1) returns the same records as the default."""
    for n, seed in ((16384, 0), (3000, 2)):
        pts = workloads.contaminated_line_points(n, seed)
        a, b = pts[:, 0].copy(), pts[:, 1].copy()
        q = n // 2 + 1
        total = n * (n - 1) // 2
        d = _ctx_with({"LMSB_BAND": "2", "LMSB_BAND_DIRECT": "1"})
        s = _ctx_with({"LMSB_BAND": "2"})
        d.upload(a, b)
        s.upload(a, b)
        got = record_from_native(d.solve(q, 0, total))
        assert d.stats()["direct_groups"] > 0
        assert got == record_from_native(s.solve(q, 0, total))


def _sharded_sequential(ctx, q, world):
    """Every shard of a world-size `world` sharded search, run one after the
    other on this GPU, with the band-table exchange done by concatenation
    (what exchange_band_table's all_gather yields)."""
    from paper_1510_01041_b200 import distributed

    plans = [ctx.shard_plan(q, world, r) for r in range(world)]
    K = plans[0][0]
    assert all(p[0] == K for p in plans)
    for r, p in enumerate(plans):
        assert len(p[1]) == (len(distributed.band_slice(K, world, r)) if K else 0)
    table = distributed.interleave_band_table([p[1] for p in plans], K) if K else plans[0][1]
    assert len(table) == K
    seed = distributed.combine(np.stack([distributed.pack(record_from_native(p[2])) for p in plans]))
    recs = [record_from_native(ctx.shard_search(q, world, r, table, _native.Candidate.of(seed)))
            for r in range(world)]
    return K, table, distributed.combine(np.stack([distributed.pack(x) for x in recs]))


@pytest.mark.parametrize("n,seed", [(16384, 0), (4096, 3), (20000, 1), (1000, 2)])
def test_sharded_band_search_matches_single_solve(n, seed):
    """Sharded search (plan slices -> exchanged band table -> per-shard range
    search -> combine) gives the single-GPU record for 1, 2, 3, 4 and 8
    shards.
    n = 1,000 is below the band threshold (no table, plain range solves);
    n = 20,000 takes the large-n path (admitted bands' keys rebuilt per shard)."""
    pts = workloads.contaminated_line_points(n, seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(a, b)
    want = record_from_native(ctx.solve(q, 0, total))
    K1, table1, got1 = _sharded_sequential(ctx, q, 1)
    assert got1 == want
    assert (K1 > 0) == (n >= 4096)
    for world in (2, 3, 4, 8):
        K, table, got = _sharded_sequential(ctx, q, world)
        assert K == K1
        assert got == want, (n, world)
    # a search on a context that did not run the plan (no reusable samples),
    # and one after an unrelated solve invalidated it: same shard records
    if K1:
        from paper_1510_01041_b200 import distributed

        plans = [ctx.shard_plan(q, 4, r) for r in range(4)]
        table = distributed.interleave_band_table([p[1] for p in plans], K1)
        seed = distributed.combine(np.stack([distributed.pack(record_from_native(p[2]))
                                             for p in plans]))
        seed = _native.Candidate.of(seed)
        warm = [record_from_native(ctx.shard_search(q, 4, r, table, seed)) for r in range(4)]
        fresh = _native.Context()
        fresh.upload(a, b)
        assert [record_from_native(fresh.shard_search(q, 4, r, table, seed))
                for r in range(4)] == warm
        ctx.solve(q, 0, total // 2)
        assert record_from_native(ctx.shard_search(q, 4, 1, table, seed)) == warm[1]


@pytest.mark.parametrize("n,seed", [(16384, 0), (4096, 3), (20000, 1), (1000, 2), (65536, 0)])
def test_owned_band_search_matches_single_solve(n, seed):
    """Band-ownership sharded search (each shard bounds, seeds and searches
    its own interleaved bands over the whole pair space; seeds and records
    exchanged) gives the single-GPU record for 1-8 shards, through the
    context API (plan + shard_search_owned) and through
    lms_min_bracelet_multi with every shard on this GPU (host exchange).
    n = 1,000 is below the band threshold: contiguous rank partitions."""
    from paper_1510_01041_b200 import distributed

    pts = workloads.contaminated_line_points(n, seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(a, b)
    want = record_from_native(ctx.solve(q, 0, total))
    worlds = (1, 2, 3, 8) if n < 65536 else (1, 4)
    for world in worlds:
        plans = [ctx.shard_plan(q, world, r) for r in range(world)]
        seed_c = _native.Candidate.of(distributed.combine(
            np.stack([distributed.pack(record_from_native(p[2])) for p in plans])))
        recs = []
        for r in range(world):
            ctx.shard_plan(q, world, r)
            recs.append(distributed.pack(record_from_native(ctx.shard_search_owned(q, world, r, seed_c))))
        assert distributed.combine(np.stack(recs)) == want, (n, world)
        got = record_from_native(_native.min_bracelet_multi(a, b, q, [0] * world))
        assert got == want, (n, world)


def test_owned_search_needs_its_plan():
    pts = workloads.contaminated_line_points(4096, 1)
    ctx = _native.Context()
    ctx.upload(pts[:, 0].copy(), pts[:, 1].copy())
    ctx.shard_plan(2049, 4, 1)
    with pytest.raises(lms.InvalidInputError):
        ctx.shard_search_owned(2049, 4, 2)  # the context holds shard 1's plan


def test_nccl_paths_one_rank():
    """The NCCL code paths with the one GPU this box has: a one-rank clique
    through lms_min_bracelet_multi (LMSB_NCCL=1) and a one-rank
    communicator bound to a context (lms_ctx_comm_init +
    lms_ctx_solve_distributed), both on device buffers; same record as the
    single solve."""
    ok, ver = _native.nccl_available()
    assert ok and ver >= 22000, ver
    n = 16384
    pts = workloads.contaminated_line_points(n, 0)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    ctx = _native.Context()
    ctx.upload(a, b)
    want = record_from_native(ctx.solve(q, 0, n * (n - 1) // 2))
    old = os.environ.get("LMSB_NCCL")
    os.environ["LMSB_NCCL"] = "1"
    try:
        assert record_from_native(_native.min_bracelet_multi(a, b, q, [0])) == want
    finally:
        if old is None:
            os.environ.pop("LMSB_NCCL", None)
        else:
            os.environ["LMSB_NCCL"] = old
    ctx.comm_init(1, 0, _native.nccl_unique_id())
    assert record_from_native(ctx.solve_distributed(q)) == want
    assert record_from_native(ctx.solve_distributed(q)) == want  # communicator reused


def test_sharded_band_search_degenerate_q_and_ties():
    """q = n (whole-set windows) and a duplicated-x, many-ties input under
    4 shards: same record as the single solve."""
    rng = np.random.default_rng(5)
    n = 6000
    x = rng.integers(0, 300, n).astype(float)
    y = np.round(2 * x + rng.integers(-3, 4, n)).astype(float)
    total = n * (n - 1) // 2
    ctx = _native.Context()
    ctx.upload(x, y)
    for q in (n // 2 + 1, n, 3):
        want = record_from_native(ctx.solve(q, 0, total))
        _, _, got = _sharded_sequential(ctx, q, 4)
        assert got == want, q


def test_shard_search_rejects_a_wrong_table():
    pts = workloads.contaminated_line_points(4096, 0)
    ctx = _native.Context()
    ctx.upload(pts[:, 0].copy(), pts[:, 1].copy())
    K, table, _ = ctx.shard_plan(2049, 1, 0)
    assert K > 1
    with pytest.raises(Exception):
        ctx.shard_search(2049, 1, 0, table[:-1])


def test_device_contacts_match_host_tail():
    """solve_lms's one-call device path (search + contact set on the GPU,
    lms_solve_fit_f64) equals the record through the backend followed by the
    numpy tail (fit_from_record, solver.py:122-140): exact fits with hundreds
    of contacts (the contact buffer regrows), noisy fits, duplicates."""
    from paper_1510_01041_b200.solver import fit_from_record, validated

    cases = [workloads.config1_points(0), workloads.config1_points(3),
             workloads.contaminated_line_points(3000, 1)]
    rng = np.random.default_rng(8)
    x = rng.integers(0, 40, 500).astype(float)
    cases.append(np.column_stack([x, 3 * x - 7]))  # every point on one line, duplicates
    cases.append(np.column_stack([rng.normal(0, 1e6, 400), rng.normal(0, 1e-3, 400)]))
    for pts in cases:
        xx, yy, q = validated(pts, None)
        got = lms.solve_lms(pts)
        rec = lms.get_backend("seq").minimum_bracelet(xx, yy, q)
        want = fit_from_record(xx, yy, q, rec)
        assert got == want
    assert len(lms.solve_lms(cases[3]).contact_indices) == 500


@pytest.mark.parametrize("n", [4096, 16384])
def test_coarse_bounds_on_small_n_and_shards_match(n):
    """The sort-free coarse bounds (LMSB_BAND_COARSE=1, the large-n default)
    forced on the shared-memory band path, single and sharded over 4: the
    same record as the default path."""
    from paper_1510_01041_b200 import distributed

    pts = workloads.contaminated_line_points(n, 6)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ref = _native.Context()
    ref.upload(a, b)
    want = record_from_native(ref.solve(q, 0, total))
    ctx = _ctx_with({"LMSB_BAND_COARSE": "1"})
    ctx.upload(a, b)
    assert record_from_native(ctx.solve(q, 0, total)) == want
    assert ctx.stats()["bands_refined"] > 0
    _, _, got = _sharded_sequential(ctx, q, 4)
    assert got == want


@pytest.mark.parametrize("n,shards", [(16384, 3), (20000, 2)])
def test_par_backend_sharded_search_matches_seq(n, shards):
    """The `par` backend's in-process sharded band search (one thread and
    context per shard; LMSB_PAR_SHARDS puts several shards on this one GPU)
    returns the seq backend's fit."""
    pts = workloads.contaminated_line_points(n, 2)
    want = lms.solve_lms(pts)
    old = os.environ.get("LMSB_PAR_SHARDS")
    os.environ["LMSB_PAR_SHARDS"] = str(shards)
    try:
        got = lms.solve_lms(pts, backend="par", workers=shards)
    finally:
        if old is None:
            os.environ.pop("LMSB_PAR_SHARDS", None)
        else:
            os.environ["LMSB_PAR_SHARDS"] = old
    assert got == want


def test_batched_device_contacts_match_host_tail():
    """solve_lms_batch's contact sets, flagged on the device
    (lms_batched_fit_f64), equal fit_from_record's numpy tail for every set:
    noisy, exact (hundreds of contacts), duplicated and pixel-grid sets."""
    from paper_1510_01041_b200.solver import fit_from_record, validated

    rng = np.random.default_rng(12)
    sets = [workloads.bench_points(512, seed=s) for s in range(5)]
    sets.append(workloads.config1_points(1, n=300))
    x = rng.integers(0, 60, 400).astype(float)
    sets.append(np.column_stack([x, 2 * x + 3]))
    sets.append(np.column_stack([rng.integers(0, 64, 256), rng.integers(0, 64, 256)]).astype(float))
    got = lms.solve_lms_batch(sets)
    for pts, g in zip(sets, got):
        xx, yy, q = validated(pts, None)
        rec = lms.get_backend("seq").minimum_bracelet(xx, yy, q)
        assert g == fit_from_record(xx, yy, q, rec)


@pytest.mark.parametrize("n,seed,qf", [(2000, 11, 0.5), (16384, 3, 0.5), (6000, 5, 0.25),
                                       (3000, 9, 0.0)])
def test_split_prepass_matches_single_cta_prepass(n, seed, qf):
    """The split pass-0 screen (LMSB_PREPASS_SPLIT=1, default: line slices over
    several CTAs, partial counts in global counters that it leaves zero) and
    the one-CTA-per-tile screen give the same record, on repeated solves
    through the same context (the counters must be clean each time) and on
    q = 2 (huge tied survivor lists)."""
    pts = workloads.contaminated_line_points(n, seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    q = max(2, int(n * qf) + 1)
    total = n * (n - 1) // 2
    one = _ctx_with({"LMSB_PREPASS_SPLIT": "0", "LMSB_BAND": "2"})
    split = _ctx_with({"LMSB_PREPASS_SPLIT": "1", "LMSB_BAND": "2"})
    one.upload(a, b)
    split.upload(a, b)
    want = record_from_native(one.solve(q, 0, total))
    for _ in range(3):
        assert record_from_native(split.solve(q, 0, total)) == want
    half = total // 2
    assert record_from_native(split.solve(q, half, total)) == record_from_native(
        one.solve(q, half, total))


def test_batch_sets_device_validation_matches_per_set_order():
    """solve_lms_batch over (n, 2) float64 arrays checks the sets on the
    device (lms_batched_fit_sets_f64): the error raised is the one the
    per-set validated() loop raises first."""
    from paper_1510_01041_b200 import solver

    good = np.array([[1.0, 2.0], [2.0, 3.0], [3.0, 5.0], [4.0, 1.0]])
    cases = [
        [np.zeros((5, 2)), np.array([[1.0, 2.0], [2.0, 3.0]])],
        [good, np.array([[1.0, 2.0], [2.0, 3.0]])],
        [good, np.array([[1.0, 2.0], [np.nan, 1.0], [3.0, 4.0]])],
        [good, np.array([[1.0, 2.0], [1.0, 1.0], [1.0, 4.0]]), np.zeros((2, 2))],
        [good, np.array([[1.0, np.inf], [2.0, 1.0], [3.0, 4.0]])],
        [good, np.zeros((0, 2))],
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
            with pytest.raises(ValueError) as ei:
                solver.solve_lms_batch(sets, q)
            assert (type(ei.value), str(ei.value)) == (type(want), str(want)), (sets, q)


def test_batch_sets_path_equals_single_fits():
    """The sets path (staged gather upload, device checks, device contact
    compaction) gives solve_lms's fit for every set, mixed sizes included."""
    rng = np.random.default_rng(3)
    sets = [workloads.bench_points(int(n), seed=k) for k, n in enumerate(rng.integers(3, 700, 40))]
    sets.append(np.ascontiguousarray(rng.integers(0, 9, (300, 2)).astype(float)))
    fits = lms.solve_lms_batch(sets)
    for p, f in zip(sets, fits):
        assert f == lms.solve_lms(p)


@pytest.mark.parametrize("case", ["config2", "grid", "outliers", "dupx", "near_parallel", "shards",
                                  "wide_q"])
def test_hybrid_grouping_matches_radix_grouping(case):
    """The hybrid grouping of the swept members (narrow bands: one group read
    with the keys the bound kernel stored; wide bands: sample sub-bands,
    device counting sort, fixed-size chunks) against the radix-sorted
    (slot, slope position) grouping with per-chunk key sorts: identical
    records and member counts, sweep forced on so n < 12,288 runs it too."""
    rng = np.random.default_rng(11)
    if case == "config2":
        pts = workloads.contaminated_line_points(16384, 0)
    elif case == "grid":
        pts = rng.integers(0, 300, (5000, 2)).astype(float)
    elif case == "outliers":
        pts = workloads.contaminated_line_points(4000, 2)
        pts[:200, 1] += 1e6
    elif case == "dupx":
        x = rng.uniform(0, 1, 4096)
        x[::7] = x[0]
        pts = np.column_stack([x, 3 * x + rng.normal(0, 0.01, 4096)])
    elif case == "near_parallel":
        x = 1.0 + np.arange(3000) * 1e-12
        pts = np.column_stack([x, rng.normal(0, 1, 3000)])
    elif case == "wide_q":
        pts = workloads.contaminated_line_points(7000, 9)
    else:
        pts = workloads.contaminated_line_points(6000, 4)
    n = len(pts)
    q = n // 2 + 1 if case != "wide_q" else (3 * n) // 4
    total = n * (n - 1) // 2
    ranges = [(0, total)] if case != "shards" else [(0, total // 3), (total // 3, total - 5), (total - 5, total)]
    c0 = _ctx_env(LMSB_SWEEP=1, LMSB_BAND=2, LMSB_GROUP_MODE=1)
    c1 = _ctx_env(LMSB_SWEEP=1, LMSB_BAND=2, LMSB_GROUP_MODE=3)
    for c in (c0, c1):
        c.upload(pts[:, 0].copy(), pts[:, 1].copy())
    for r0, r1 in ranges:
        a = record_from_native(c0.solve(q, r0, r1))
        sa = c0.stats()
        b = record_from_native(c1.solve(q, r0, r1))
        sb = c1.stats()
        assert a == b, (case, r0, r1)
        assert sa["filtered_vertices"] == sb["filtered_vertices"], (case, r0, r1)
        want = oracle_rec(pts[:, 0].copy(), pts[:, 1].copy(), q, r0, r1) if n <= 5000 else None
        if want is not None:
            assert record_matches(b, want), (case, r0, r1)


def test_deferred_member_count_overflow_resolves():
    """The hybrid grouping never reads the member count back mid-fit; a
    collect capacity that is too small (forced: 4,096 members) is caught by
    the final readback and the fit solved again with room for every member:
    the config-2 record stays the reference's, the member count the full one."""
    import json

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config2_golden.json")))
    pts = workloads.contaminated_line_points(gold["n"], 0)
    q = gold["q"]
    total = gold["n"] * (gold["n"] - 1) // 2
    ref = _ctx_env(LMSB_GROUP_MODE=3)
    tiny = _ctx_env(LMSB_GROUP_MODE=3, LMSB_CAP_TEST=1)
    for c in (ref, tiny):
        c.upload(pts[:, 0].copy(), pts[:, 1].copy())
    a = record_from_native(ref.solve(q, 0, total))
    b = record_from_native(tiny.solve(q, 0, total))
    assert a == b
    assert (b.i, b.j, b.height) == (gold["record"]["i"], gold["record"]["j"],
                                    float.fromhex(gold["record"]["height"]))
    assert tiny.stats()["filtered_vertices"] == ref.stats()["filtered_vertices"] > 4096


@pytest.mark.parametrize("case", ["config2", "outliers", "dupx", "grid", "range"])
def test_device_plan_matches_host_plan(case):
    """The device-side plan of the band search (band_plan_kernel: admitted
    bands, sweep runs and ends, sub-band groups -- no readback after the
    seeds) against the host plan: identical records, member counts, admitted
    bands and sweep runs.  The device plan runs from a context's second fit
    of a given n (the first sizes the member buffers)."""
    rng = np.random.default_rng(21)
    if case == "config2":
        pts = workloads.contaminated_line_points(16384, 0)
    elif case == "outliers":
        pts = workloads.contaminated_line_points(6000, 2)
        pts[:300, 1] += 1e6
    elif case == "dupx":
        x = rng.uniform(0, 1, 4096)
        x[::5] = x[1]
        pts = np.column_stack([x, -2 * x + rng.normal(0, 0.01, 4096)])
    elif case == "grid":
        pts = rng.integers(0, 200, (6000, 2)).astype(float)
    else:
        pts = workloads.contaminated_line_points(9000, 7)
    n = len(pts)
    q = n // 2 + 1
    total = n * (n - 1) // 2
    r0, r1 = (0, total) if case != "range" else (total // 5, total - total // 7)
    host = _ctx_env(LMSB_DEVICE_PLAN=0)
    dev = _ctx_env(LMSB_DEVICE_PLAN=1)
    for c in (host, dev):
        c.upload(pts[:, 0].copy(), pts[:, 1].copy())
        c.solve(q, r0, r1)  # sizes the member buffers (host plan on both)
    a = record_from_native(host.solve(q, r0, r1))
    sa = host.stats()
    b = record_from_native(dev.solve(q, r0, r1))
    sb = dev.stats()
    assert a == b, case
    for k in ("filtered_vertices", "bands_searched", "sweep_runs", "band_survivors"):
        if k == "band_survivors":
            continue  # (chunk order differs: the running bound tightens at other points)
        assert sa[k] == sb[k], (case, k, sa[k], sb[k])


@pytest.mark.parametrize("case", ["config2", "steep", "narrow_x", "dupx_majority", "huge_y", "small"])
def test_slope_bound_matches_plain_bounds(case):
    """Band bounds raised to the slope bound |u|min W_q(a) - 2 bmax (every
    vertex at slope u is at least the narrowest q-window of the line values
    there): identical records with and without it -- on config 2, a steep
    line (large optimal |u|), x spread over a tiny range, a majority of
    duplicate x (W_q(a) = 0: no bound), 1e12 outliers -- and against the
    oracle at small n."""
    rng = np.random.default_rng(33)
    if case == "config2":
        pts = workloads.contaminated_line_points(16384, 0)
    elif case == "steep":
        x = rng.uniform(0, 1, 6000)
        y = 5000.0 * x + rng.normal(0, 1, 6000)
        y[:2900] = rng.uniform(-1e4, 1e4, 2900)
        pts = np.column_stack([x, y])
    elif case == "narrow_x":
        x = 1e3 + rng.uniform(0, 1e-6, 5000)
        pts = np.column_stack([x, rng.normal(0, 1, 5000)])
    elif case == "dupx_majority":
        x = rng.uniform(0, 10, 5000)
        x[:2600] = 3.0
        pts = np.column_stack([x, x + rng.normal(0, 0.1, 5000)])
    elif case == "huge_y":
        pts = workloads.contaminated_line_points(5000, 5)
        pts[:1000, 1] *= 1e8
    else:
        pts = workloads.contaminated_line_points(2600, 6)
    n = len(pts)
    q = n // 2 + 1
    total = n * (n - 1) // 2
    c0 = _ctx_env(LMSB_SLOPE_BOUND=0, LMSB_BAND=2)
    c1 = _ctx_env(LMSB_SLOPE_BOUND=1, LMSB_BAND=2)
    recs = []
    for c in (c0, c1):
        c.upload(pts[:, 0].copy(), pts[:, 1].copy())
        recs.append(record_from_native(c.solve(q, 0, total)))
    assert recs[0] == recs[1], case
    if case == "small":
        assert record_matches(recs[1], oracle_rec(pts[:, 0].copy(), pts[:, 1].copy(), q))
