"""numpy restatement of the reference's Hough vote / peaks / support
(hough.py:112-184) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pinned by tests/test_oracle_hough.py against tests/golden/hough_golden.json.gz
(produced by the reference itself).
"""

from __future__ import annotations

import math

import numpy as np


def rho_bin(rho, rho_max: float, delta_rho: float, n_rho: int) -> np.ndarray:
    """HoughParams.rho_bin (hough.py:60-63)."""
    r = np.floor((np.asarray(rho, dtype=float) + rho_max) / delta_rho).astype(np.int64)
    return np.clip(r, 0, n_rho - 1)


def vote(x: np.ndarray, y: np.ndarray, delta_rho: float, delta_theta: float, rho_max: float) -> np.ndarray:
    """hough_vote (hough.py:112-129): int64 bins [n_rho, n_theta]."""
    n_theta = math.ceil(180.0 / delta_theta)
    n_rho = math.ceil(2.0 * rho_max / delta_rho)
    bins = np.zeros((n_rho, n_theta), dtype=np.int64)
    if x.size == 0:
        return bins
    theta = np.radians((np.arange(n_theta) + 0.5) * delta_theta)
    rho = x[:, None] * np.cos(theta)[None, :] + y[:, None] * np.sin(theta)[None, :]
    rb = rho_bin(rho, rho_max, delta_rho, n_rho)
    tb = np.broadcast_to(np.arange(n_theta, dtype=np.int64), rb.shape)
    flat = np.bincount((rb * n_theta + tb).ravel(), minlength=n_rho * n_theta)
    return flat.reshape(n_rho, n_theta)


def support(x: np.ndarray, y: np.ndarray, theta_bin: int, rbin: int, delta_rho: float,
            delta_theta: float, rho_max: float) -> np.ndarray:
    """supporting_points (hough.py:171-184) as ordinals, scan order kept."""
    n_rho = math.ceil(2.0 * rho_max / delta_rho)
    theta = math.radians((theta_bin + 0.5) * delta_theta)
    rho = x * math.cos(theta) + y * math.sin(theta)
    return np.flatnonzero(rho_bin(rho, rho_max, delta_rho, n_rho) == rbin)
