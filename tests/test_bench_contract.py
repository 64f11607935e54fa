"""bench.py contract on a CPU-only box: the reference arm (the oracle) prints the
driver's JSON line, and the product arm refuses to run without a GPU (no CPU
fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_reference_arm_json_line():
    p = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GLUP/s" and d["dtype"] == "f64"
    assert d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "jacobi3d_512^3_per_gpu_odf8"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"] > 0


def test_product_arm_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: the product arm runs")
    p = _run("--steps", "1", "--warmup", "3", "--no-sweep", "--no-cpu", timeout=300)
    assert p.returncode != 0
    assert "no CUDA device" in (p.stderr + p.stdout)


def test_multi_gpu_without_torchrun_is_a_single_process_run():
    """`bench.py --gpus N` without torchrun drives the N GPUs from one process
    (jac_create(n_gpus)); on a CPU box it stops at the missing device, not at a
    launcher complaint, and the reference arm prints its line."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = _run("--gpus", "2", "--steps", "1", "--warmup", "3", "--no-sweep", "--no-cpu", timeout=300)
    assert p.returncode != 0 and "no CUDA device" in (p.stderr + p.stdout)
    assert "torchrun" not in (p.stderr + p.stdout)
    p = _run("--impl", "reference", "--gpus", "4", "--steps", "1", "--warmup", "3")
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 4 and d["impl"] == "reference"


def test_workload_geometry():
    """Bench workloads follow readings R9 / R10 and the paper's grids."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.workload("c2", 1, 8)[:3] == ((512, 512, 512), (2, 2, 2), (1, 1, 1))
    assert bench.workload("c2", 4, 8)[:3] == ((512, 1024, 1024), (2, 4, 4), (1, 2, 2))
    assert bench.workload("c2", 8, 8)[:3] == ((1024, 1024, 1024), (4, 4, 4), (2, 2, 2))
    assert bench.workload("c4", 8, 16)[:3] == ((1536, 1536, 1536), (4, 4, 8), (2, 2, 2))
    # the paper's Jacobi2D strong grid: minimum cut splits x first (98304 < 131072)
    assert bench.workload("j2d_strong", 2, 1)[:3] == ((131072, 98304, 1), (2, 1, 1), (2, 1, 1))
    assert bench.workload("j2d_strong", 4, 8)[:3] == ((131072, 98304, 1), (8, 4, 1), (2, 2, 1))
    assert bench.workload("j2d_strong", 8, 16)[2] == (4, 2, 1)
    assert bench.gpu_grid_2d_r10(4, 131072, 98304) == (2, 2)
    assert bench.blocks_for_odf_2d((32768, 32768), 8) == (2, 4)
