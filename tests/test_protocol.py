"""Pins for the paper's measurement protocol (§V) — values worked in
SPEC.md [MODULE] stats/report and the paper's own numbers.  CPU only."""
import math

import pytest

from paper_2408_15384_b200 import protocol as pr


def test_normal_quantiles():
    # SPEC.md:266-268
    assert pr.normal_quantile(0.5) == pytest.approx(0.0, abs=1e-12)
    assert pr.normal_quantile(0.975) == pytest.approx(1.95996398, abs=1e-8)
    assert pr.normal_quantile(0.8) == pytest.approx(0.84162123, abs=1e-8)
    assert pr.normal_quantile(0.3) == pytest.approx(-pr.normal_quantile(0.7), abs=1e-12)
    with pytest.raises(ValueError):
        pr.normal_quantile(1.0)


def test_required_sample_size_paper_formula():
    # PAPER.md:211-213 with α=0.05, power 0.8, effect 0.5
    assert pr.required_sample_size(variance=1.0) == 63
    assert pr.required_sample_size(variance=0.0) == 2
    n1 = 2 * ((1.959963984540054 + 0.8416212335729143) / 0.5) ** 2
    assert pr.required_sample_size(variance=4.0) == math.ceil(4 * n1)
    # monotone in variance, effect, alpha
    assert pr.required_sample_size(variance=2) >= pr.required_sample_size(variance=1)
    assert pr.required_sample_size(effect=1.0) <= pr.required_sample_size(effect=0.5)
    assert pr.required_sample_size(alpha=0.1) <= pr.required_sample_size(alpha=0.05)


def test_summarize():
    # SPEC.md:286-288
    s = pr.summarize([1, 2, 3, 4, 5])
    assert s.mean == 3 and s.variance == 2.5 and s.std_dev == pytest.approx(1.5811, abs=1e-4)
    assert pr.summarize([2, 4]).variance == 2
    c = pr.summarize([1, 1, 1, 1])
    assert c.variance == 0 and c.ci95_half_width == 0
    a = pr.summarize([0.3, 0.1, 0.2])
    b = pr.summarize([0.1, 0.2, 0.3])
    assert a == b  # permutation-invariant
    sh = pr.summarize([x + 10 for x in [0.3, 0.1, 0.2]])
    assert sh.mean == pytest.approx(a.mean + 10) and sh.variance == pytest.approx(a.variance, rel=1e-9)
    with pytest.raises(ValueError):
        pr.summarize([1.0])


def test_complexity_fit():
    sizes = [128, 256, 512, 1024]
    s3, r3 = pr.fit_complexity(sizes, [n ** 3 * 1e-9 for n in sizes])
    assert s3 == pytest.approx(3.0, abs=1e-9) and r3 == pytest.approx(1.0, abs=1e-12)
    s2, _ = pr.fit_complexity(sizes, [n ** 2 for n in sizes])
    assert s2 == pytest.approx(2.0, abs=1e-9)
    # Table 1 (GCC -O3) means at 256, 512, 1024: ~3.19
    s, _ = pr.fit_complexity([256, 512, 1024], [0.02028, 0.17037, 1.69891])
    assert s == pytest.approx(math.log2(1.69891 / 0.02028) / 2, abs=0.02)
    assert 3.1 < s < 3.3


def test_speedup_efficiency_paper_thread_sweep():
    # 9.67 s with one thread -> 0.88 s with 16 threads
    s, e = pr.speedup_efficiency(9.67, 0.88, 16)
    assert s == pytest.approx(10.99, abs=0.01) and e == pytest.approx(0.687, abs=0.001)
    s, e = pr.speedup_efficiency(1.59, 0.12, 16)  # Intel
    assert s == pytest.approx(13.25, abs=0.01)
    assert pr.speedup_efficiency(2.0, 2.0, 1) == (1.0, 1.0)


def test_repetitions_from_pilot():
    # a 1 % coefficient of variation -> σ² = 1 (percent units) -> 63 repetitions
    pilot = [100.0 + d for d in (-1, 1) * 15]
    s = pr.summarize(pilot)
    n = pr.required_sample_size(variance=(100 * s.std_dev / s.mean) ** 2)
    assert pr.repetitions_from_pilot(pilot) == max(15, n)
    assert pr.repetitions_from_pilot([1.0] * 30) == 15  # the paper's 15 runs are the floor
