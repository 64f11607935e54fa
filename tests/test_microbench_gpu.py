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


def _ngpu():
    import torch
    return torch.cuda.device_count()


def test_launch_rate_and_pipeline():
    assert J.jac_mb_launch_rate(2, 1, 0.1) > 1000
    with pytest.raises(J.JacError):
        J.jac_mb_pipeline(0, 0, 16, 4, False)


@pytest.mark.parametrize("odf", [1, 3, 16, 64])
@pytest.mark.parametrize("compute", [False, True])
def test_pipeline_delivers_every_byte_one_device(odf, compute):
    """NEXT-3 content check (SPEC.md:398 byte conservation): every delivered byte equals
    the source pattern, for both transports, ragged message sizes included."""
    total = (1 << 22) + 8 * 37
    assert J.jac_mb_pipeline(0, 0, total, odf, compute) > 0
    assert J.jac_mb_last_verified_bytes() == (total // odf) // 8 * 8 * odf
    assert J.jac_mb_pipeline_batched(0, 0, total, odf, compute) > 0
    assert J.jac_mb_last_verified_bytes() == (total // odf) // 16 * 16 * odf


@pytest.mark.parametrize("odf", [1, 8, 64])
def test_pipeline_delivers_every_byte_over_nvlink(odf):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    total = 64 << 20
    for src, dst in ((0, 1), (1, 0)):
        assert J.jac_mb_pipeline(src, dst, total, odf, True) > 0
        assert J.jac_mb_last_verified_bytes() == (total // odf) // 8 * 8 * odf
        assert J.jac_mb_pipeline_batched(src, dst, total, odf, True) > 0
        assert J.jac_mb_last_verified_bytes() == (total // odf) // 16 * 16 * odf
