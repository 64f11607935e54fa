timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x --durations=10 > gpurun_out/pytest_full.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full.log
