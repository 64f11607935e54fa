timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for r in 1 2; do ITERS=40 timeout 200 python tools/quick_perf.py 2>&1 | cut -c1-100; FLAGS=512 ITERS=10 timeout 300 python tools/perf_shapes.py 32768x32768x1:2x4x1 2>&1 | cut -c1-110; done > gpurun_out/at.log
