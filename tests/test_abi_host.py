"""Host-side checks of the C ABI (-m "not gpu"): the library loads, exports every
function include/jacobi3d.h declares, and the planner (pure host code) enforces the
decomposition rules and reading R10."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

import paper_2605_12734_b200 as jb
from paper_2605_12734_b200 import jacobi3d as J

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions(name="jacobi3d.h"):
    src = open(os.path.join(ROOT, "include", name)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jac_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = jb.load()
    names = _header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(J.EXPORTED)
    assert jb.jac_version() == 100
    mb = _header_functions("jacobi3d_microbench.h")
    assert set(mb) == set(J.MICROBENCH_EXPORTED)
    for n in mb:
        assert hasattr(L, n), n


def test_library_is_in_tree_and_built_for_sm100a():
    path = J.lib_path()
    assert path.startswith(os.path.join(ROOT, "paper_2605_12734_b200"))
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tma_kernels_have_no_large_stack_frame():
    """No TMA sweep instantiation of the production build carries more than a spilled
    register or two of stack (performance hygiene: the z-march keeps its state in
    registers).  History: a build whose peer-wait call copied the 240-byte kernel
    parameters to a stack frame showed stale 32-point row segments at 512^3.  The cause
    was not the frame but a write-after-read race it exposed -- plane 0's stage was
    refilled while the loads feeding the first plane's z- neighbour could still be in
    flight; the same frame-carrying build is bit-exact once refills overwrite the
    previous plane's stage (profiles/r02_ring_war_race.txt)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-res-usage", J.lib_path()], capture_output=True, text=True).stdout
    lines = out.splitlines()
    seen = 0
    for i, ln in enumerate(lines):
        if "Function" in ln and ("sweep_tma_kernel" in ln or "sweep2d_tma_kernel" in ln):
            seen += 1
            stack = int(re.search(r"STACK:(\d+)", lines[i + 1]).group(1))
            assert stack <= 16, (ln, lines[i + 1])
    assert seen >= 16


def test_header_struct_sizes_match_binding():
    assert jb.jac_ipc_handle_bytes() == 256
    src = open(os.path.join(ROOT, "include", "jacobi3d.h")).read()
    assert len(J.STAT_NAMES) == int(re.search(r"JAC_STAT_N\s*=\s*(\d+)", src).group(1))
    # the binding's names follow the header's enum order
    names = re.findall(r"JAC_STAT_([A-Z_]+)\s*=\s*(\d+)", src)
    for name, idx in names:
        if name != "N":
            assert J.STAT_NAMES[int(idx)] == name.lower(), (name, idx)


@pytest.mark.parametrize("args,code", [
    ((0, 8, 8, 1, 1, 1, 1), J.JAC_EINVAL),
    ((8, 8, 8, 0, 1, 1, 1), J.JAC_EINVAL),
    ((8, 8, 8, 1, 1, 1, 0), J.JAC_EINVAL),
    ((9, 8, 8, 2, 1, 1, 1), J.JAC_EDECOMP),     # nx % bx
    ((8, 8, 8, 2, 1, 1, 3), J.JAC_EDECOMP),     # non-integral ODF
    ((8, 8, 8, 1, 1, 1, 2), J.JAC_EDECOMP),     # 1 block, 2 GPUs
])
def test_plan_errors(args, code):
    with pytest.raises(J.JacError) as ei:
        jb.jac_plan(*args)
    assert ei.value.code == code
    assert jb.jac_last_error()  # names the offending argument


def test_plan_error_names_argument():
    with pytest.raises(J.JacError, match="nz"):
        jb.jac_plan(8, 8, 0, 1, 1, 1, 1)
    with pytest.raises(J.JacError, match="ODF"):
        jb.jac_plan(8, 8, 8, 2, 1, 1, 3)


def test_plan_explicit_gpu_grid_checks():
    assert jb.jac_plan(16, 16, 16, 2, 2, 2, 4, (1, 2, 2)) == ((1, 2, 2), (8, 8, 8))
    with pytest.raises(J.JacError) as ei:
        jb.jac_plan(16, 16, 16, 2, 2, 2, 4, (1, 1, 2))   # product != n_gpus
    assert ei.value.code == J.JAC_EDECOMP
    with pytest.raises(J.JacError):
        jb.jac_plan(16, 16, 16, 1, 2, 4, 4, (2, 1, 2))   # bx % gx


@pytest.mark.parametrize("dims,blocks,n,grid", [
    # C3 weak scaling, ODF 8: 1x1x2, 1x2x2, 2x2x2
    ((768, 768, 1536), (2, 2, 4), 2, (1, 1, 2)),
    ((768, 1536, 1536), (2, 4, 4), 4, (1, 2, 2)),
    ((1536, 1536, 1536), (4, 4, 4), 8, (2, 2, 2)),
    # C4 strong scaling ODF 1 / 16
    ((1536, 1536, 1536), (1, 1, 2), 2, (1, 1, 2)),
    ((1536, 1536, 1536), (2, 4, 4), 2, (1, 1, 2)),
    ((1536, 1536, 1536), (2, 2, 2), 8, (2, 2, 2)),
    # C5 fine grain: 1024^3 with 32^3 blocks on 8 GPUs
    ((1024, 1024, 1024), (32, 32, 32), 8, (2, 2, 2)),
    ((512, 512, 512), (1, 1, 1), 1, (1, 1, 1)),
])
def test_plan_r10_min_surface_gpu_grid(dims, blocks, n, grid):
    g, e = jb.jac_plan(*dims, *blocks, n)
    assert g == grid
    assert e == tuple(dims[d] // blocks[d] for d in range(3))


def test_plan_face_kinds_symmetric():
    dims, blocks, n = (24, 16, 32), (3, 2, 4), 4
    g, _ = jb.jac_plan(*dims, *blocks, n)
    opp = [1, 0, 3, 2, 5, 4]
    seen = {0: 0, 1: 0, 2: 0}
    for iz in range(blocks[2]):
        for iy in range(blocks[1]):
            for ix in range(blocks[0]):
                for f in range(6):
                    kind, owner = jb.jac_plan_face(*dims, *blocks, n, None, ix, iy, iz, f)
                    seen[kind] += 1
                    nb = [ix, iy, iz]
                    nb[f >> 1] += 1 if f & 1 else -1
                    inside = all(0 <= nb[d] < blocks[d] for d in range(3))
                    assert (kind == J.JAC_FACE_BOUNDARY) == (not inside)
                    if inside:
                        k2, o2 = jb.jac_plan_face(*dims, *blocks, n, None, *nb, opp[f])
                        assert k2 == kind
                        me = jb.jac_plan_face(*dims, *blocks, n, None, *nb, opp[f])[1]
                        assert o2 == me
    # every interior face counted twice, boundary faces = 2*(bx*by + by*bz + bx*bz)
    assert seen[0] == 2 * (3 * 2 + 2 * 4 + 3 * 4)
    assert seen[2] > 0 and seen[1] > 0


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(J.JacError) as ei:
        jb.jac_create(8, 8, 8, 1, 1, 1)
    assert ei.value.code == J.JAC_EDEVICE


def test_null_safety():
    L = jb.load()
    assert L.jac_destroy(None) == 0
    assert L.jac_step(None, 1) == J.JAC_EINVAL
    assert L.jac_set_init(None, None) == J.JAC_EINVAL
    assert L.jac_get_block(None, 0, 0, 0, None) == J.JAC_EINVAL
    out = ctypes.c_void_p()
    assert L.jac_create(8, 8, 8, 1, 1, 1, 1, None, 0, None) == J.JAC_EINVAL
    assert L.jac_create(8, 8, 8, 1, 1, 1, 1, None, J.JAC_F_NCCL, ctypes.byref(out)) == J.JAC_EINVAL


def test_sass_no_fma_and_tma_present():
    """R5: the update has no a*b+c and the build uses -fmad=false, so the SASS must
    hold no DFMA; the TMA sweep must issue UTMALDG (cp.async.bulk.tensor)."""
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", J.lib_path()], capture_output=True, text=True).stdout
    assert "DFMA" not in sass
    funcs = sass.split("Function : ")
    tma = [f for f in funcs if f.startswith("_ZN3jac16sweep_tma_kernel")]
    assert len(tma) >= 6 and all("UTMALDG" in f and "UBLKCP" in f for f in tma)
    # programmatic dependent launch: every sweep instantiation waits on its predecessor
    assert all("ACQBULK" in f and "PREEXIT" in f for f in tma)
