"""Measurement protocol of the paper (§V "Experimental Environment"),
applied to GPU timings.

The paper runs "30 preliminary tests", sizes the repetition count by a
power analysis

    n = 2 · ((Z_{1-α/2} + Z_{1-β}) / 0.5)² · σ²

with α = 0.05, power 1-β = 0.8, effect 0.5, reports the mean of the
repetitions ("Avg Time (sec)", Tables 1-2) and reads the growth of time with size as
O(n³).  Reading R14: σ² is the pilot's variance of the time
expressed in percent of its mean, so the effect 0.5 means "detect a 0.5 % change of the
mean time"; the paper's own 15 repetitions are kept as the minimum.
Pure host arithmetic; pinned by tests/test_protocol.py against SPEC.md's worked values.
"""
from __future__ import annotations

import math
import statistics
from dataclasses import dataclass


def normal_quantile(p: float) -> float:
    """Inverse standard-normal CDF ("critical values from the normal distribution")."""
    if not 0.0 < p < 1.0:
        raise ValueError("p must lie in (0, 1)")
    return statistics.NormalDist().inv_cdf(p)


def required_sample_size(alpha: float = 0.05, power: float = 0.8, effect: float = 0.5, variance: float = 1.0) -> int:
    """⌈2·((Z_{1-α/2} + Z_{power}) / effect)²·σ²⌉, floor 2."""
    z = normal_quantile(1.0 - alpha / 2.0) + normal_quantile(power)
    n = 2.0 * (z / effect) ** 2 * variance
    return max(2, math.ceil(n - 1e-12))


@dataclass
class Summary:
    n: int
    mean: float
    variance: float
    std_dev: float
    min: float
    max: float
    ci95_half_width: float


def summarize(samples) -> Summary:
    """Mean, unbiased variance, extremes and the 95 % CI half-width of repeated timings."""
    xs = [float(x) for x in samples]
    if len(xs) < 2:
        raise ValueError("need at least 2 samples")
    mean = math.fsum(xs) / len(xs)
    var = math.fsum((x - mean) ** 2 for x in xs) / (len(xs) - 1)
    sd = math.sqrt(var)
    return Summary(len(xs), mean, var, sd, min(xs), max(xs), normal_quantile(0.975) * sd / math.sqrt(len(xs)))


def fit_complexity(sizes, times) -> tuple[float, float]:
    """OLS slope and r² of log2(time) on log2(size) ("expected O(n^3) complexity")."""
    if len(sizes) < 3:
        raise ValueError("need at least 3 sizes")
    x = [math.log2(s) for s in sizes]
    y = [math.log2(t) for t in times]
    mx, my = sum(x) / len(x), sum(y) / len(y)
    sxx = sum((a - mx) ** 2 for a in x)
    sxy = sum((a - mx) * (b - my) for a, b in zip(x, y))
    slope = sxy / sxx
    ss_tot = sum((b - my) ** 2 for b in y)
    ss_res = sum((b - (my + slope * (a - mx))) ** 2 for a, b in zip(x, y))
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    return slope, r2


def speedup_efficiency(t_base: float, t: float, workers: int) -> tuple[float, float]:
    """Speedup t_base/t and parallel efficiency speedup/workers."""
    s = t_base / t
    return s, s / workers


def repetitions_from_pilot(pilot, alpha=0.05, power=0.8, effect=0.5, minimum=15) -> int:
    """Repetition count for timings whose pilot runs are `pilot` (reading R14)."""
    s = summarize(pilot)
    rel_var_pct = (100.0 * s.std_dev / s.mean) ** 2 if s.mean > 0 else 0.0
    return max(minimum, required_sample_size(alpha, power, effect, rel_var_pct))
