"""B200-calibrated iteration-latency model for the elastic scheduler.

The reference prices a decode iteration with a three-regime piecewise-affine model
of the computed-token count x (pkg/src/dllmsim/costmodel.py:34-67, called at
sim.py:293 and scheduler.py:107-112), fitted from a GPU profile
(costmodel.py:118-176, `dllmsim calibrate`, cli.py:377-389).  Its defaults are
A100-like (costmodel.py:98-115).  This module produces that model from *measured*
B200 step latencies of this path:

* :func:`profile_csv` writes the reference's profile format ``x,latency_ms``
  (costmodel.py:179-186), so ``dllmsim calibrate`` can consume it unchanged;
* :func:`fit` fits the same model family — latency = i0 + s·x + d1·(x−b1)+ +
  d2·(x−b2)+ with nonnegative slopes/increments (continuous, nondecreasing,
  convex), breakpoints searched over the interior sample x values with ≥ 3 distinct
  x per regime, coefficients by nonnegative least squares — and returns the
  reference's JSON (``segments``: x_start, slope_us_per_token, intercept_ms;
  costmodel.py:69-96), loadable by ``CostModel.from_json``.

tools/calibrate_b200.py measures the samples on a B200 (device step of this path at
SDAR-8B shape over a grid of batch sizes and chunk sizes).
"""

from __future__ import annotations

import json
from typing import Sequence

import numpy as np

from .errors import ConfigError

CSV_HEADER = "x,latency_ms"


def profile_csv(samples: Sequence[tuple]) -> str:
    """(computed tokens, latency seconds) samples -> the reference's profile CSV."""
    rows = [CSV_HEADER] + [f"{float(x)!r},{float(t) * 1e3!r}" for x, t in samples]
    return "\n".join(rows) + "\n"


def _nnls(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    from scipy.optimize import nnls

    return nnls(a, b)[0]


def fit(samples: Sequence[tuple]) -> dict:
    """Fit the three-regime convex piecewise-affine latency model; returns the
    reference's cost-model JSON object (``{"segments": [...]}``)."""
    x = np.asarray([float(s[0]) for s in samples])
    y = np.asarray([float(s[1]) for s in samples])
    if x.size < 9:
        raise ConfigError(f"cost model fit needs >= 9 samples, got {x.size}")
    ux = np.unique(x)
    if ux.size < 9:
        raise ConfigError("cost model fit needs >= 3 distinct x values per regime")
    best = None
    cand = ux[1:-1]
    for i in range(cand.size):
        b1 = cand[i]
        lo = int(np.count_nonzero(ux <= b1))
        if lo < 3:
            continue
        for b2 in cand[i + 1:]:
            mid = int(np.count_nonzero((ux > b1) & (ux <= b2)))
            hi = int(np.count_nonzero(ux > b2))
            if mid < 3 or hi < 3:
                continue
            basis = np.stack([np.ones_like(x), x, np.clip(x - b1, 0, None), np.clip(x - b2, 0, None)], axis=1)
            th = _nnls(basis, y)
            err = float(np.square(basis @ th - y).sum())
            if best is None or err < best[0] - 1e-15:
                best = (err, float(b1), float(b2), th)
    if best is None:
        raise ConfigError("no breakpoint pair leaves 3 distinct x per regime")
    _, b1, b2, th = best
    i0, s0, d1, d2 = (float(v) for v in th)
    s1, s2, s3 = s0, s0 + d1, s0 + d1 + d2
    i1 = i0
    i2 = i1 + s1 * b1
    i3 = i2 + s2 * (b2 - b1)
    return {"segments": [
        {"x_start": 0.0, "slope_us_per_token": s1 * 1e6, "intercept_ms": i1 * 1e3},
        {"x_start": b1, "slope_us_per_token": s2 * 1e6, "intercept_ms": i2 * 1e3},
        {"x_start": b2, "slope_us_per_token": s3 * 1e6, "intercept_ms": i3 * 1e3},
    ]}


def latency(model: dict, x: float) -> float:
    """Seconds for x computed tokens under a fitted model (costmodel.py:57-67)."""
    if x < 0:
        raise ConfigError("computed tokens must be >= 0")
    seg = model["segments"][0]
    for s in model["segments"][1:]:
        if x >= s["x_start"]:
            seg = s
    return (seg["intercept_ms"] * 1e-3) + (seg["slope_us_per_token"] * 1e-6) * (x - seg["x_start"])


def to_json(model: dict) -> str:
    return json.dumps(model, indent=2)
