timeout 1200 python -m pytest tests/test_multigpu_gpu.py -m gpu -q 2>&1 | tail -3 > gpurun_out/mp_tests.log
