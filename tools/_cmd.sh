timeout 600 python -m pytest tests/test_parity2d_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config j2d --steps 50 --warmup 3 > gpurun_out/bench_j2d.json 2> gpurun_out/bench_j2d.err; echo rc=$? >> gpurun_out/bench_j2d.err
