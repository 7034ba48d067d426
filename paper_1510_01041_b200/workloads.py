"""Synthetic inputs for the BASELINE.json configs (host-side, not the hot path).

* ``config1_points`` / ``contaminated_line_points`` -- configs 1-3
  (BASELINE.md section 3): x ~ U[0, 1000), inliers on y = 2x + 1 (optionally
  + N(0, 1)), a permutation-chosen outlier fraction with uniform y.
* ``bench_points`` -- restates the reference's fixed benchmark instance
  (experiments.py:247-254) used for config 4 (8,192 fits of n = 512).

All streams are numpy PCG64 seeded as BASELINE.md specifies, so the same
seed gives the same points here, in the golden-fixture script and on the
GPU box.
"""

from __future__ import annotations

import math

import numpy as np


def _rng(seed: int, n: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, n])))


def config1_points(seed: int = 0, n: int = 1000, noise: bool = False) -> np.ndarray:
    """Config 1: n points, 55% exactly on y = 2x + 1 (variant B adds N(0,1)),
    45% outliers with y ~ U[min y - 500, max y + 500]."""
    rng = _rng(seed, n)
    x = rng.uniform(0.0, 1000.0, n)
    y = 2.0 * x + 1.0
    if noise:
        y = y + rng.normal(0.0, 1.0, n)
    n_out = (45 * n) // 100
    out = rng.permutation(n)[:n_out]
    lo, hi = float(y.min()) - 500.0, float(y.max()) + 500.0
    y[out] = rng.uniform(lo, hi, n_out)
    return np.column_stack([x, y])


def contaminated_line_points(n: int, seed: int = 0, outlier_frac: float = 0.49) -> np.ndarray:
    """Configs 2-3: inliers y = 2x + 1 + N(0, 1), a fraction of gross
    outliers with y ~ U[-1e4, 1e4]."""
    rng = _rng(seed, n)
    x = rng.uniform(0.0, 1000.0, n)
    y = 2.0 * x + 1.0 + rng.normal(0.0, 1.0, n)
    n_out = int(outlier_frac * n)
    out = rng.permutation(n)[:n_out]
    y[out] = rng.uniform(-1e4, 1e4, n_out)
    return np.column_stack([x, y])


def bench_points(n: int, seed: int = 7) -> np.ndarray:
    """experiments.py:247-254: y = 0.75x + 40 + N(0, 5), 30% uniform outliers."""
    rng = _rng(seed, n)
    x = rng.uniform(0.0, 1000.0, n)
    y = 0.75 * x + 40.0 + rng.normal(0.0, 5.0, n)
    bad = rng.random(n) < 0.3
    y[bad] = rng.uniform(0.0, 1000.0, int(bad.sum()))
    return np.column_stack([x, y])


def line_image(width: int = 4096, height: int = 4096, lines: int = 64, salt: float = 0.30,
               sampling: float = 0.5, seed: int = 0) -> np.ndarray:
    """Config 5 input: a uint8 image (0 / 255) with ``lines`` random lines
    (normal angle in [20, 160) degrees, passing within width/4 of the
    centre, pixels kept with probability ``sampling``) plus salt noise.

    A quick generic generator for tests; the BASELINE config-5 input is
    ``config5_image`` (the reference's own ``gen_synthetic`` recipe).
    """
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0])))
    img = np.zeros((height, width), dtype=np.uint8)
    cx, cy = width / 2.0, height / 2.0
    for _ in range(lines):
        th = np.radians(rng.uniform(20.0, 160.0))
        off = rng.uniform(-width / 4.0, width / 4.0)
        # normal form x cos th + y sin th = rho through a point near the centre
        px, py = cx + off * np.cos(th), cy + off * np.sin(th)
        dx, dy = -np.sin(th), np.cos(th)  # direction along the line
        t = np.arange(-2.0 * max(width, height), 2.0 * max(width, height), 0.5)
        xs = np.rint(px + t * dx).astype(np.int64)
        ys = np.rint(py + t * dy).astype(np.int64)
        ok = (xs >= 0) & (xs < width) & (ys >= 0) & (ys < height)
        xs, ys = xs[ok], ys[ok]
        keep = rng.random(xs.size) < sampling
        img[ys[keep], xs[keep]] = 255
    noise = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 1])))
    img[noise.random((height, width)) < salt] = 255
    return img


def config5_specs(seed: int = 0, width: int = 4096, height: int = 4096, lines: int = 64,
                  sampling: float = 0.5):
    """The ``lines`` SyntheticSpecs of the config-5 image: normal
    angle θ ~ U[20°, 160°), the line passing at a signed distance ~ U[−W/4, W/4)
    from the frame centre, each rendered by ``gen_synthetic(SyntheticSpec(W, H,
    slope, intercept, sampling_prob=0.5, noise_prob=0, seed=1000·seed + k))``.
    The (θ, offset) draws come from ``PCG64(SeedSequence([seed, 2]))``."""
    from .synth import SyntheticSpec

    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 2])))
    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0
    specs = []
    for k in range(lines):
        th = math.radians(float(rng.uniform(20.0, 160.0)))
        off = float(rng.uniform(-width / 4.0, width / 4.0))
        rho = cx * math.cos(th) + cy * math.sin(th) + off
        slope = -math.cos(th) / math.sin(th)
        intercept = rho / math.sin(th)
        specs.append(SyntheticSpec(width=width, height=height, slope=slope, intercept=intercept,
                                   sampling_prob=sampling, noise_prob=0.0, seed=1000 * seed + k))
    return specs


def config5_image(seed: int = 0, width: int = 4096, height: int = 4096, lines: int = 64,
                  salt: float = 0.30, render=None) -> np.ndarray:
    """BASELINE config 5: the ``config5_specs`` lines combined with
    ``np.maximum`` (as test_detect.py:246-257 combines images), then salt
    ``PCG64(SeedSequence([seed, 1])).random((H, W)) < salt`` set to 255.

    ``render(spec) -> uint8 image`` defaults to this package's
    ``synth.render``; the golden script passes the reference's
    ``gen_synthetic`` to pin the two against each other."""
    from . import synth

    if render is None:
        render = lambda sp: synth.render(sp)[0]  # noqa: E731
    img = np.zeros((height, width), dtype=np.uint8)
    for sp in config5_specs(seed, width, height, lines):
        np.maximum(img, render(sp), out=img)
    if salt > 0.0:
        noise = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 1])))
        img[noise.random((height, width)) < salt] = 255
    return img
