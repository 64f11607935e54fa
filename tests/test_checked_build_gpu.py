"""Bounds-checked build (libjacobi3d_checked.so, -DJAC_CHECKED): the substitute for
compute-sanitizer, which is closed on this GPU pool (B200_PROFILING.md: runs under it
left GPUs needing a reset).  Every global store of every kernel is checked against the
context's allocation ranges (own + connected peers') and its alignment, every TMA
coordinate and x-ghost bulk-copy range is asserted; a violation is recorded (source
line, address) and the store skipped, and the call returns JAC_ECUDA naming it.

The small cases of tools/sanitize_cases.py (C1, 32^3 blocks, ragged, unfused pack,
plain loads, paper-style per-block streams, virtual 2x2x2 remote, NCCL layout, 2-D)
must run clean and bit-exact under it, and a deliberately corrupted face pointer
(experiment knob) must be caught."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _checked_lib():
    sys.path.insert(0, ROOT)
    from paper_2605_12734_b200 import build
    return build.build(checked=True)


def _run(args, env_extra=None):
    env = dict(os.environ)
    env["JAC_LIB"] = _checked_lib()
    env.update(env_extra or {})
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)


def test_checked_build_runs_clean_and_bit_exact():
    r = _run([os.path.join(ROOT, "tools", "sanitize_cases.py")])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("bit-exact") == 10 and "MISMATCH" not in r.stdout, r.stdout


def test_checked_build_loads_the_checked_library():
    code = ("import paper_2605_12734_b200 as jb; jb.load(); "
            "print(open('/proc/self/maps').read().count('libjacobi3d_checked.so') > 0)")
    r = _run(["-c", code])
    assert r.returncode == 0 and r.stdout.strip().endswith("True"), r.stdout + r.stderr


def test_checked_build_catches_a_wild_store():
    code = (
        "import jac_inputs as JI, paper_2605_12734_b200 as jb\n"
        "from paper_2605_12734_b200 import jacobi3d as J\n"
        "u0 = JI.hash_field(64, 64, 64, seed=1)\n"
        "with jb.Jacobi3D((64, 64, 64), (2, 2, 2)) as s:\n"
        "    s.set_init(u0)\n"
        "    try:\n"
        "        s.step(2)\n"
        "        print('NOT CAUGHT')\n"
        "    except J.JacError as e:\n"
        "        print('CAUGHT', e.code, e)\n"
        "    s.field(u0)\n"
        "    print('ALIVE')\n")
    r = _run(["-c", code], {"JAC_EXPERIMENT": "1", "JAC_CHECK_SELFTEST": "1"})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CAUGHT -5" in r.stdout and "out-of-range store" in r.stdout and "ALIVE" in r.stdout, r.stdout
