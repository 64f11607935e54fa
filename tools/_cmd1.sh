F=gpurun_out/layouts2; mkdir -p $F
timeout 900 python -m pytest tests/test_layouts_gpu.py -m gpu -q 2>&1 | tail -15 > $F/pytest.log
