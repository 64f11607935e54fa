"""Error behaviour of the C ABI as include/jacobi3d.h documents it, called through
the raw ctypes library (no Python-side checks in between): every bad argument
returns the documented negative jac_status, leaves a message in jac_last_error(),
and leaves the context usable (the next valid call still gives oracle results)."""
import ctypes

import numpy as np
import pytest

import jac_inputs as JI
import oracle
from paper_2605_12734_b200 import jacobi3d as J

pytestmark = pytest.mark.gpu

i64, i32, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_double


def _arr(t, vals):
    return (t * len(vals))(*vals)


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@pytest.fixture
def lib():
    return J.load()


@pytest.fixture
def ctx(lib):
    c = ctypes.c_void_p()
    assert lib.jac_create(48, 40, 32, 2, 2, 2, 1, None, 0, ctypes.byref(c)) == J.JAC_OK
    yield c
    assert lib.jac_destroy(c) == J.JAC_OK


def _expect(lib, rc, status, word=None):
    assert rc == status, (rc, status)
    msg = (lib.jac_last_error() or b"").decode()
    assert msg, "jac_last_error() is empty after a failed call"
    if word:
        assert word in msg, msg


def test_create_errors(lib):
    c = ctypes.c_void_p()
    _expect(lib, lib.jac_create(48, 40, 32, 2, 2, 2, 1, None, 0, None), J.JAC_EINVAL, "out")
    import torch
    if torch.cuda.device_count() < 2:  # single-process multi-GPU needs the devices
        _expect(lib, lib.jac_create(48, 40, 32, 2, 2, 2, 2, None, 0, ctypes.byref(c)), J.JAC_EDEVICE, "devices")
    _expect(lib, lib.jac_create(48, 40, 32, 2, 2, 2, 2, None, J.JAC_F_PER_BLOCK, ctypes.byref(c)), J.JAC_EINVAL)
    _expect(lib, lib.jac_create(48, 40, 32, 5, 2, 2, 1, None, 0, ctypes.byref(c)), J.JAC_EDECOMP)
    _expect(lib, lib.jac_create(0, 40, 32, 1, 1, 1, 1, None, 0, ctypes.byref(c)), J.JAC_EINVAL)
    _expect(lib, lib.jac_create(48, 40, 32, 1, 1, 1, 1, None, J.JAC_F_2D, ctypes.byref(c)), J.JAC_EINVAL, "2D")
    _expect(lib, lib.jac_create(48, 40, 32, 2, 2, 2, 1, None, J.JAC_F_NCCL, ctypes.byref(c)), J.JAC_EINVAL, "NCCL")
    assert lib.jac_destroy(None) == J.JAC_OK  # NULL-safe


def test_call_order_and_arguments(lib, ctx):
    _expect(lib, lib.jac_step(ctx, 1), J.JAC_ESTATE, "jac_set_init")
    d = dbl()
    _expect(lib, lib.jac_profile_sweep(ctx, 1, ctypes.byref(d)), J.JAC_ESTATE)
    _expect(lib, lib.jac_set_init(ctx, None), J.JAC_EINVAL, "padded")
    u0 = JI.hash_field(48, 40, 32, seed=2)
    assert lib.jac_set_init(ctx, _dp(u0)) == J.JAC_OK
    _expect(lib, lib.jac_step(ctx, -1), J.JAC_EINVAL, "n_iters")
    _expect(lib, lib.jac_profile_sweep(ctx, 0, ctypes.byref(d)), J.JAC_EINVAL)
    out = np.empty(24 * 20 * 16)
    _expect(lib, lib.jac_get_block(ctx, 2, 0, 0, _dp(out)), J.JAC_EINVAL, "outside")
    _expect(lib, lib.jac_get_block(ctx, 0, 0, -1, _dp(out)), J.JAC_EINVAL)
    _expect(lib, lib.jac_get_block(ctx, 0, 0, 0, None), J.JAC_EINVAL)
    _expect(lib, lib.jac_get_region(ctx, _arr(i64, [40, 0, 0]), _arr(i64, [9, 1, 1]), _dp(out)), J.JAC_EINVAL)
    box = np.empty((10, 10, 10))
    _expect(lib, lib.jac_set_init_box(ctx, _dp(box), _arr(i64, [0, 0, 0]), _arr(i64, [10, 10, 10])),
            J.JAC_EINVAL, "cover")
    _expect(lib, lib.jac_set_option(ctx, 999, 1), J.JAC_EINVAL)
    _expect(lib, lib.jac_get_stats(ctx, None), J.JAC_EINVAL)
    _expect(lib, lib.jac_import_ipc(ctx, None), J.JAC_EINVAL)
    rec = (ctypes.c_char * lib.jac_ipc_handle_bytes())()
    _expect(lib, lib.jac_export_ipc(ctx, rec), J.JAC_ESTATE, "rank context")
    # the context is still good: every failed call above left the state untouched
    assert lib.jac_step(ctx, 5) == J.JAC_OK
    got = np.zeros_like(u0)
    assert lib.jac_get_field(ctx, _dp(got)) == J.JAC_OK
    want = oracle.jacobi3d(u0, 5)
    inner = (slice(1, -1),) * 3
    assert np.array_equal(got[inner].view(np.uint64), want[inner].view(np.uint64))


def test_rank_context_needs_ipc_before_init(lib):
    c = ctypes.c_void_p()
    assert lib.jac_create_rank(48, 40, 32, 2, 2, 2, 2, None, 0, 0, 0, ctypes.byref(c)) == J.JAC_OK
    try:
        u0 = JI.hash_field(48, 40, 32, seed=1)
        _expect(lib, lib.jac_set_init(c, _dp(u0)), J.JAC_ESTATE, "jac_import_ipc")
        _expect(lib, lib.jac_nccl_init(c, None), J.JAC_EINVAL)
    finally:
        assert lib.jac_destroy(c) == J.JAC_OK


def test_profile_gap(lib, ctx):
    """jac_last_profile_gap_ms: JAC_ESTATE before a profile; afterwards the median
    end-of-sweep -> next-sweep gap of the graph, a few microseconds (one kernel per
    iteration, no host round trip)."""
    g = dbl()
    _expect(lib, lib.jac_last_profile_gap_ms(ctx, ctypes.byref(g)), J.JAC_ESTATE)
    _expect(lib, lib.jac_last_profile_gap_ms(ctx, None), J.JAC_EINVAL)
    assert lib.jac_set_init_hash(ctx, 1) == J.JAC_OK
    d = dbl()
    assert lib.jac_profile_sweep(ctx, 12, ctypes.byref(d)) == J.JAC_OK
    assert lib.jac_last_profile_gap_ms(ctx, ctypes.byref(g)) == J.JAC_OK
    assert 0.0 <= g.value < 0.05, g.value


def test_options_grid_and_stats(lib, ctx):
    """jac_set_option validates the watchdog limit; jac_get_grid returns the creation
    arguments; a single-GPU context reports one partition, no remote work and no
    experiment knobs (the production state)."""
    _expect(lib, lib.jac_set_option(ctx, J.JAC_OPT_WATCHDOG_MS, -5), J.JAC_EINVAL, "WATCHDOG")
    assert lib.jac_set_option(ctx, J.JAC_OPT_WATCHDOG_MS, 0) == J.JAC_OK
    _expect(lib, lib.jac_set_option(ctx, J.JAC_OPT_LAUNCH_THREADS, 0), J.JAC_EINVAL)
    n = (i64 * 3)()
    b = (i32 * 3)()
    f = ctypes.c_uint32()
    assert lib.jac_get_grid(ctx, n, b, ctypes.byref(f)) == J.JAC_OK
    assert tuple(n) == (48, 40, 32) and tuple(b) == (2, 2, 2) and f.value == 0
    assert lib.jac_get_grid(ctx, None, None, None) == J.JAC_OK
    _expect(lib, lib.jac_get_grid(None, n, b, None), J.JAC_EINVAL)
    st = J.jac_get_stats(ctx.value)
    assert st["partitions"] == 1 and st["remote_faces"] == 0 and st["fused_sync"] == 0
    assert st["experiment"] == 0 and st["epoch_min"] == st["epoch_max"] == 0
    assert lib.jac_set_init_hash(ctx, 2) == J.JAC_OK
    assert lib.jac_step(ctx, 3) == J.JAC_OK  # with the watchdog off (0 = wait forever)
