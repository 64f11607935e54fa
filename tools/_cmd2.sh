timeout 300 python -m pytest tests/test_microbench_gpu.py -q > gpurun_out/pytest_mb.log 2>&1; echo pytest=$? >> gpurun_out/pytest_mb.log
timeout 900 python tools/microbench.py > gpurun_out/microbench_r01.json 2> gpurun_out/microbench.err
