F=gpurun_out/mpfinal; mkdir -p $F
timeout 1500 python -m pytest tests/test_multigpu_gpu.py tests/test_parity_gpu.py -m gpu -q 2>&1 | tail -3 > $F/pytest.log
