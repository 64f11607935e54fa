"""Thin ctypes binding of libjacobi3d.so (include/jacobi3d.h) -- argument
marshalling only.  Every step of the hot path runs in the library's sm_100a kernels;
there is no Python or CPU fallback: if the shared library cannot be built or loaded
the import of this module's functions raises.

Function names mirror the C ABI (``jac_create``, ``jac_set_init``, ``jac_step``,
``jac_get_block``, ``jac_destroy``, ...).  ``Jacobi3D`` is a small convenience
wrapper around one context.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

from . import build as _build

JAC_OK, JAC_EINVAL, JAC_EDECOMP, JAC_EDEVICE, JAC_ENOMEM, JAC_ECUDA, JAC_ENCCL, JAC_ESTATE = (
    0, -1, -2, -3, -4, -5, -6, -7)
JAC_F_DEFAULT = 0
JAC_F_FMA = 1 << 0
JAC_F_NO_GRAPH = 1 << 1
JAC_F_NCCL = 1 << 2
JAC_F_UNFUSED_PACK = 1 << 4
JAC_F_NO_TMA = 1 << 5
JAC_F_VIRTUAL_GPUS = 1 << 6
JAC_F_SKIP_EXCHANGE = 1 << 7
JAC_F_PER_BLOCK = 1 << 8
JAC_F_2D = 1 << 9
JAC_OPT_LAUNCH_THREADS = 1
JAC_OPT_WATCHDOG_MS = 2
JAC_FACE_BOUNDARY, JAC_FACE_LOCAL, JAC_FACE_REMOTE = 0, 1, 2
STAT_NAMES = ["kernel_launches", "graph_launches", "kernels_per_iter", "local_blocks",
              "local_faces", "remote_faces", "remote_bytes", "arena_bytes", "sweep_variant",
              "partitions", "remote_items", "fused_sync", "epoch_min", "epoch_max", "experiment",
              "peer_wait_ns", "peer_wait_max_ns"]
EXPORTED = ["jac_plan", "jac_plan_face", "jac_create", "jac_create_rank", "jac_ipc_handle_bytes",
            "jac_export_ipc", "jac_import_ipc", "jac_set_init", "jac_set_init_hash", "jac_step",
            "jac_get_block", "jac_get_block_padded", "jac_get_field", "jac_get_layout",
            "jac_block_owner", "jac_last_step_ms", "jac_set_init_box", "jac_get_field_box", "jac_local_box",
            "jac_profile_sweep", "jac_last_profile_gap_ms", "jac_get_stats",
            "jac_destroy", "jac_last_error", "jac_version", "jac_set_option", "jac_nccl_id_bytes",
            "jac_nccl_get_unique_id", "jac_nccl_init", "jac_get_region", "jac_get_grid"]
MICROBENCH_EXPORTED = ["jac_mb_launch_latency", "jac_mb_overlap", "jac_mb_launch_rate", "jac_mb_pipeline",
                       "jac_mb_pipeline_batched", "jac_mb_last_verified_bytes"]

_ERRNAMES = {-1: "JAC_EINVAL", -2: "JAC_EDECOMP", -3: "JAC_EDEVICE", -4: "JAC_ENOMEM",
             -5: "JAC_ECUDA", -6: "JAC_ENCCL", -7: "JAC_ESTATE"}


class JacError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: {_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


_lib: Optional[ctypes.CDLL] = None


def lib_path() -> str:
    # JAC_LIB: load another build of the same ABI (same-box A/B comparisons only)
    return os.environ.get("JAC_LIB") or _build.LIB


def load() -> ctypes.CDLL:
    """Loads (building first if missing or stale) the in-tree libjacobi3d.so."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("JAC_LIB") or _build.build()
    if not os.path.exists(path):
        raise ImportError(f"libjacobi3d.so missing at {path}; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    i64, i32, u32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
    P = ctypes.POINTER
    vp, dp = ctypes.c_void_p, P(ctypes.c_double)
    sig = {
        "jac_plan": [i64, i64, i64, i32, i32, i32, i32, P(i32), P(i32), P(i64)],
        "jac_plan_face": [i64, i64, i64, i32, i32, i32, i32, P(i32), i32, i32, i32, i32, P(i32), P(i32)],
        "jac_create": [i64, i64, i64, i32, i32, i32, i32, P(i32), u32, P(vp)],
        "jac_create_rank": [i64, i64, i64, i32, i32, i32, i32, P(i32), i32, i32, u32, P(vp)],
        "jac_export_ipc": [vp, vp],
        "jac_import_ipc": [vp, vp],
        "jac_set_init": [vp, dp],
        "jac_set_init_hash": [vp, u64],
        "jac_step": [vp, i32],
        "jac_get_block": [vp, i32, i32, i32, dp],
        "jac_get_block_padded": [vp, i32, i32, i32, dp],
        "jac_get_field": [vp, dp],
        "jac_set_init_box": [vp, dp, P(i64), P(i64)],
        "jac_get_field_box": [vp, dp, P(i64), P(i64)],
        "jac_local_box": [vp, P(i64), P(i64)],
        "jac_get_layout": [vp, P(i32), P(i64), P(i64)],
        "jac_block_owner": [vp, i32, i32, i32, P(i32)],
        "jac_last_step_ms": [vp, P(ctypes.c_double)],
        "jac_profile_sweep": [vp, i32, P(ctypes.c_double)],
        "jac_last_profile_gap_ms": [vp, P(ctypes.c_double)],
        "jac_get_stats": [vp, P(i64)],
        "jac_destroy": [vp],
        "jac_set_option": [vp, i32, i64],
        "jac_nccl_get_unique_id": [vp],
        "jac_nccl_init": [vp, vp],
        "jac_get_region": [vp, P(i64), P(i64), dp],
        "jac_get_grid": [vp, P(i64), P(i32), P(u32)],
        "jac_mb_launch_latency": [i32, i32, P(ctypes.c_double)],
        "jac_mb_overlap": [i32, i64, i32, i32, P(ctypes.c_double), P(ctypes.c_double)],
        "jac_mb_launch_rate": [i32, i32, i32, ctypes.c_double, P(ctypes.c_double)],
        "jac_mb_pipeline": [i32, i32, i64, i32, i32, P(ctypes.c_double)],
        "jac_mb_pipeline_batched": [i32, i32, i64, i32, i32, P(ctypes.c_double)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.jac_nccl_id_bytes.argtypes = []
    L.jac_nccl_id_bytes.restype = ctypes.c_size_t
    L.jac_ipc_handle_bytes.argtypes = []
    L.jac_ipc_handle_bytes.restype = ctypes.c_size_t
    L.jac_last_error.argtypes = []
    L.jac_last_error.restype = ctypes.c_char_p
    L.jac_version.argtypes = []
    L.jac_version.restype = ctypes.c_int
    L.jac_mb_last_verified_bytes.argtypes = []
    L.jac_mb_last_verified_bytes.restype = ctypes.c_int64
    _lib = L
    return L


def _check(rc: int, fn: str) -> None:
    if rc != JAC_OK:
        raise JacError(rc, fn, (load().jac_last_error() or b"").decode())


def _grid(g: Optional[Sequence[int]]):
    if g is None:
        return None
    return (ctypes.c_int32 * 3)(*[int(v) for v in g])


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _checked(a: np.ndarray, shape, what: str):
    """The C side reads / writes exactly prod(shape) doubles at the pointer: refuse any
    array that is not C-contiguous float64 of exactly that shape (a wrong dtype, a
    strided view or a short buffer would otherwise be silent heap corruption)."""
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{what} must be a numpy array")
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError(f"{what} must be a C-contiguous float64 array (got {a.dtype}, "
                         f"contiguous={a.flags.c_contiguous})")
    if tuple(int(v) for v in a.shape) != tuple(int(v) for v in shape):
        raise ValueError(f"{what} has shape {a.shape}, expected {tuple(shape)}")
    if what.endswith("(writable)") and not a.flags.writeable:
        raise ValueError(f"{what} is read-only")
    return _dptr(a)


def _grid_info(ctx):
    """(n = interior dims (x, y, z), b = global blocks, flags) of a context."""
    n = (ctypes.c_int64 * 3)()
    b = (ctypes.c_int32 * 3)()
    f = ctypes.c_uint32()
    _check(load().jac_get_grid(ctx, n, b, ctypes.byref(f)), "jac_get_grid")
    return tuple(n), tuple(b), f.value


def _padded_shape(ctx):
    n, _, flags = _grid_info(ctx)
    zg = 0 if flags & JAC_F_2D else 1
    return (n[2] + 2 * zg, n[1] + 2, n[0] + 2)


def _block_shape(ctx, padded=False):
    _, e, _ = jac_get_layout(ctx)
    _, _, flags = _grid_info(ctx)
    if not padded:
        return (e[2], e[1], e[0])
    return (e[2] + (0 if flags & JAC_F_2D else 2), e[1] + 2, e[0] + 2)


# ------------------------------------------------------------------ C-ABI mirrors
def jac_plan(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid=None):
    g = (ctypes.c_int32 * 3)()
    e = (ctypes.c_int64 * 3)()
    _check(load().jac_plan(nx, ny, nz, bx, by, bz, n_gpus, _grid(gpu_grid), g, e), "jac_plan")
    return tuple(g), tuple(e)


def jac_plan_face(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, ix, iy, iz, f):
    kind, owner = ctypes.c_int32(), ctypes.c_int32()
    _check(load().jac_plan_face(nx, ny, nz, bx, by, bz, n_gpus, _grid(gpu_grid), ix, iy, iz, f,
                                ctypes.byref(kind), ctypes.byref(owner)), "jac_plan_face")
    return kind.value, owner.value


def jac_create(nx, ny, nz, bx, by, bz, n_gpus=1, gpu_grid=None, flags=0) -> int:
    out = ctypes.c_void_p()
    _check(load().jac_create(nx, ny, nz, bx, by, bz, n_gpus, _grid(gpu_grid), flags,
                             ctypes.byref(out)), "jac_create")
    return out.value


def jac_create_rank(nx, ny, nz, bx, by, bz, n_gpus, gpu_grid, rank, device, flags=0) -> int:
    out = ctypes.c_void_p()
    _check(load().jac_create_rank(nx, ny, nz, bx, by, bz, n_gpus, _grid(gpu_grid), rank, device,
                                  flags, ctypes.byref(out)), "jac_create_rank")
    return out.value


def jac_ipc_handle_bytes() -> int:
    return int(load().jac_ipc_handle_bytes())


def jac_export_ipc(ctx) -> bytes:
    buf = ctypes.create_string_buffer(jac_ipc_handle_bytes())
    _check(load().jac_export_ipc(ctx, buf), "jac_export_ipc")
    return buf.raw


def jac_import_ipc(ctx, records: Sequence[bytes]) -> None:
    blob = b"".join(records)
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(load().jac_import_ipc(ctx, buf), "jac_import_ipc")


def jac_nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(int(load().jac_nccl_id_bytes()))
    _check(load().jac_nccl_get_unique_id(buf), "jac_nccl_get_unique_id")
    return buf.raw


def jac_nccl_init(ctx, uid: bytes) -> None:
    buf = ctypes.create_string_buffer(uid, len(uid))
    _check(load().jac_nccl_init(ctx, buf), "jac_nccl_init")


def jac_set_init(ctx, padded: np.ndarray) -> None:
    _check(load().jac_set_init(ctx, _checked(padded, _padded_shape(ctx), "padded")), "jac_set_init")


def jac_set_init_hash(ctx, seed: int) -> None:
    _check(load().jac_set_init_hash(ctx, seed), "jac_set_init_hash")


def jac_step(ctx, n_iters: int) -> None:
    _check(load().jac_step(ctx, n_iters), "jac_step")


def jac_get_block(ctx, ix, iy, iz, out: np.ndarray) -> np.ndarray:
    p = _checked(out, _block_shape(ctx), "out (writable)")
    _check(load().jac_get_block(ctx, ix, iy, iz, p), "jac_get_block")
    return out


def jac_get_block_padded(ctx, ix, iy, iz, out: np.ndarray) -> np.ndarray:
    p = _checked(out, _block_shape(ctx, padded=True), "out (writable)")
    _check(load().jac_get_block_padded(ctx, ix, iy, iz, p), "jac_get_block_padded")
    return out


def jac_get_field(ctx, padded: np.ndarray) -> np.ndarray:
    p = _checked(padded, _padded_shape(ctx), "padded (writable)")
    _check(load().jac_get_field(ctx, p), "jac_get_field")
    return padded


def _i64x3(v):
    return (ctypes.c_int64 * 3)(*[int(x) for x in v])


def jac_set_init_box(ctx, box: np.ndarray, origin) -> None:
    """``box`` is a [sz, sy, sx] float64 sub-array of the padded grid starting at
    padded cell ``origin`` = (ox, oy, oz)."""
    if not isinstance(box, np.ndarray) or box.ndim != 3:
        raise ValueError("box must be a 3-D numpy array [sz, sy, sx]")
    p = _checked(box, box.shape, "box")
    ext = (box.shape[2], box.shape[1], box.shape[0])
    _check(load().jac_set_init_box(ctx, p, _i64x3(origin), _i64x3(ext)), "jac_set_init_box")


def jac_get_field_box(ctx, box: np.ndarray, origin) -> np.ndarray:
    if not isinstance(box, np.ndarray) or box.ndim != 3:
        raise ValueError("box must be a 3-D numpy array [sz, sy, sx]")
    p = _checked(box, box.shape, "box (writable)")
    ext = (box.shape[2], box.shape[1], box.shape[0])
    _check(load().jac_get_field_box(ctx, p, _i64x3(origin), _i64x3(ext)), "jac_get_field_box")
    return box


def jac_local_box(ctx):
    o = (ctypes.c_int64 * 3)()
    e = (ctypes.c_int64 * 3)()
    _check(load().jac_local_box(ctx, o, e), "jac_local_box")
    return tuple(o), tuple(e)


def jac_get_region(ctx, lo, ext) -> np.ndarray:
    """Interior sub-box [lo, lo+ext) (x, y, z order), returned as [ez][ey][ex]."""
    out = np.empty((int(ext[2]), int(ext[1]), int(ext[0])), dtype=np.float64)
    _check(load().jac_get_region(ctx, _i64x3(lo), _i64x3(ext), _dptr(out)), "jac_get_region")
    return out


def jac_get_layout(ctx):
    g = (ctypes.c_int32 * 3)()
    e = (ctypes.c_int64 * 3)()
    it = ctypes.c_int64()
    _check(load().jac_get_layout(ctx, g, e, ctypes.byref(it)), "jac_get_layout")
    return tuple(g), tuple(e), it.value


def jac_block_owner(ctx, ix, iy, iz) -> int:
    g = ctypes.c_int32()
    _check(load().jac_block_owner(ctx, ix, iy, iz, ctypes.byref(g)), "jac_block_owner")
    return g.value


def jac_last_step_ms(ctx) -> float:
    v = ctypes.c_double()
    _check(load().jac_last_step_ms(ctx, ctypes.byref(v)), "jac_last_step_ms")
    return v.value


def jac_profile_sweep(ctx, n_iters: int) -> float:
    v = ctypes.c_double()
    _check(load().jac_profile_sweep(ctx, n_iters, ctypes.byref(v)), "jac_profile_sweep")
    return v.value


def jac_last_profile_gap_ms(ctx) -> float:
    v = ctypes.c_double()
    _check(load().jac_last_profile_gap_ms(ctx, ctypes.byref(v)), "jac_last_profile_gap_ms")
    return v.value


def jac_get_stats(ctx) -> dict:
    st = (ctypes.c_int64 * len(STAT_NAMES))()
    _check(load().jac_get_stats(ctx, st), "jac_get_stats")
    return dict(zip(STAT_NAMES, list(st)))


def jac_set_option(ctx, option: int, value: int) -> None:
    _check(load().jac_set_option(ctx, option, value), "jac_set_option")


# ------------------------------------------------------------------ microbenchmarks (NEXT-3/4)
def jac_mb_launch_latency(device=0, iters=2000) -> float:
    v = ctypes.c_double()
    _check(load().jac_mb_launch_latency(device, iters, ctypes.byref(v)), "jac_mb_launch_latency")
    return v.value


def jac_mb_overlap(total_threads, odf, work=1000, device=0):
    h, d = ctypes.c_double(), ctypes.c_double()
    _check(load().jac_mb_overlap(device, total_threads, odf, work, ctypes.byref(h), ctypes.byref(d)), "jac_mb_overlap")
    return h.value, d.value


def jac_mb_launch_rate(chares, threads, seconds=0.5, device=0) -> float:
    v = ctypes.c_double()
    _check(load().jac_mb_launch_rate(device, chares, threads, seconds, ctypes.byref(v)), "jac_mb_launch_rate")
    return v.value


def jac_mb_pipeline(src, dst, total_bytes, odf, with_compute=False) -> float:
    v = ctypes.c_double()
    _check(load().jac_mb_pipeline(src, dst, total_bytes, odf, int(bool(with_compute)), ctypes.byref(v)), "jac_mb_pipeline")
    return v.value


def jac_mb_pipeline_batched(src, dst, total_bytes, odf, with_compute=False) -> float:
    v = ctypes.c_double()
    _check(load().jac_mb_pipeline_batched(src, dst, total_bytes, odf, int(bool(with_compute)), ctypes.byref(v)),
           "jac_mb_pipeline_batched")
    return v.value


def jac_mb_last_verified_bytes() -> int:
    return int(load().jac_mb_last_verified_bytes())


def jac_destroy(ctx) -> None:
    _check(load().jac_destroy(ctx), "jac_destroy")


def jac_last_error() -> str:
    return (load().jac_last_error() or b"").decode()


def jac_version() -> int:
    return int(load().jac_version())


# ------------------------------------------------------------------ convenience
class Jacobi3D:
    """One context.  ``dims`` = (nx, ny, nz) interior points, ``blocks`` = (bx, by, bz)
    global blocks per dim.  ``rank``/``device`` select a rank context (one process
    per GPU; see ``paper_2605_12734_b200.dist``)."""

    def __init__(self, dims, blocks, n_gpus=1, gpu_grid=None, flags=0, rank=None, device=0):
        self.dims = tuple(int(v) for v in dims)
        self.blocks = tuple(int(v) for v in blocks)
        self.n_gpus = int(n_gpus)
        if rank is None:
            self.ctx = jac_create(*self.dims, *self.blocks, self.n_gpus, gpu_grid, flags)
        else:
            self.ctx = jac_create_rank(*self.dims, *self.blocks, self.n_gpus, gpu_grid, rank, device, flags)
        self.rank = rank
        self.gpu_grid, self.block_extent, _ = jac_get_layout(self.ctx)

    @property
    def odf(self) -> int:
        return self.blocks[0] * self.blocks[1] * self.blocks[2] // self.n_gpus

    def set_init(self, padded: np.ndarray) -> None:
        jac_set_init(self.ctx, padded)

    def set_init_hash(self, seed: int) -> None:
        jac_set_init_hash(self.ctx, seed)

    def step(self, n: int) -> None:
        jac_step(self.ctx, n)

    def block(self, ix, iy, iz) -> np.ndarray:
        ex, ey, ez = self.block_extent
        return jac_get_block(self.ctx, ix, iy, iz, np.empty((ez, ey, ex), dtype=np.float64))

    def block_padded(self, ix, iy, iz) -> np.ndarray:
        shape = _block_shape(self.ctx, padded=True)  # (ez+2, ey+2, ex+2); one plane in 2-D
        return jac_get_block_padded(self.ctx, ix, iy, iz, np.empty(shape, dtype=np.float64))

    def field(self, like: np.ndarray) -> np.ndarray:
        """Padded array: shell/non-local cells copied from ``like`` (which must have the
        padded shape), local interiors from the device."""
        out = np.array(like, dtype=np.float64, copy=True, order="C")
        return jac_get_field(self.ctx, out)

    def region(self, lo, ext) -> np.ndarray:
        """Interior sub-box [lo, lo+ext) (x, y, z), as [ez][ey][ex]."""
        return jac_get_region(self.ctx, lo, ext)

    def local_box(self):
        """(origin, extent) of this context's ghosted bounding box, padded coords (x, y, z)."""
        return jac_local_box(self.ctx)

    def set_init_box(self, box: np.ndarray, origin) -> None:
        jac_set_init_box(self.ctx, box, origin)

    def field_box(self, box: np.ndarray, origin) -> np.ndarray:
        return jac_get_field_box(self.ctx, box, origin)

    @property
    def iterations(self) -> int:
        return jac_get_layout(self.ctx)[2]

    def last_step_ms(self) -> float:
        return jac_last_step_ms(self.ctx)

    def profile_sweep(self, n: int) -> float:
        return jac_profile_sweep(self.ctx, n)

    def profile_gap_ms(self) -> float:
        """Median gap between consecutive sweeps of the last profile_sweep (n >= 2)."""
        return jac_last_profile_gap_ms(self.ctx)

    def set_option(self, option: int, value: int) -> None:
        jac_set_option(self.ctx, option, value)

    def stats(self) -> dict:
        return jac_get_stats(self.ctx)

    def owner(self, ix, iy, iz) -> int:
        return jac_block_owner(self.ctx, ix, iy, iz)

    def close(self) -> None:
        if self.ctx:
            jac_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Jacobi2D(Jacobi3D):
    """Jacobi2D (NEXT-1) through the same library: dims (nx, ny), blocks (bx, by);
    padded arrays are [ny+2, nx+2]."""

    def __init__(self, dims, blocks, n_gpus=1, gpu_grid=None, flags=0, rank=None, device=0):
        g = None if gpu_grid is None else (int(gpu_grid[0]), int(gpu_grid[1]), 1)
        super().__init__((dims[0], dims[1], 1), (blocks[0], blocks[1], 1), n_gpus=n_gpus, gpu_grid=g,
                         flags=flags | JAC_F_2D, rank=rank, device=device)

    def set_init(self, padded: np.ndarray) -> None:
        jac_set_init(self.ctx, np.ascontiguousarray(padded).reshape(1, *padded.shape))

    def set_init_box(self, box: np.ndarray, origin) -> None:
        b = box if box.ndim == 3 else np.ascontiguousarray(box).reshape(1, *box.shape)
        o = tuple(origin) + (0,) * (3 - len(tuple(origin)))
        jac_set_init_box(self.ctx, b, o)

    def field(self, like: np.ndarray) -> np.ndarray:
        out = np.array(like, dtype=np.float64, copy=True).reshape(1, *like.shape)
        return jac_get_field(self.ctx, out).reshape(like.shape)

    def field_box(self, box: np.ndarray, origin) -> np.ndarray:
        b = box if box.ndim == 3 else box.reshape(1, *box.shape)
        o = tuple(origin) + (0,) * (3 - len(tuple(origin)))
        return jac_get_field_box(self.ctx, b, o).reshape(box.shape)

    def block(self, ix, iy) -> np.ndarray:
        return super().block(ix, iy, 0)[0]

    def block_padded(self, ix, iy) -> np.ndarray:
        return super().block_padded(ix, iy, 0)[0]
