timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu2.log
