"""Sanity of the NEXT-3/NEXT-4 microbenchmarks (numbers are reported, not asserted
against the paper's A40 values)."""
import pytest

from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu


def test_launch_latency_positive():
    us = J.jac_mb_launch_latency(0, 200)
    assert 0.5 < us < 1000


def test_overlap_monotone_in_work():
    h1, d1 = J.jac_mb_overlap(262144, 8, work=2000)
    h2, d2 = J.jac_mb_overlap(262144, 8, work=20000)
    assert d2 > d1 > 0 and h2 > 0


def test_launch_rate_and_pipeline():
    assert J.jac_mb_launch_rate(2, 1, 0.1) > 1000
    us = J.jac_mb_pipeline(0, 0, 1 << 22, 4, True)
    assert us > 0
    assert J.jac_mb_pipeline_batched(0, 0, 1 << 22, 16, True) > 0
    with pytest.raises(J.JacError):
        J.jac_mb_pipeline(0, 0, 16, 4, False)
