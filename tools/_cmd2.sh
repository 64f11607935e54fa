timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu2.log
ITERS=40 timeout 200 python tools/quick_perf.py > gpurun_out/qp_final.log 2>&1
ITERS=30 timeout 600 python tools/perf_shapes.py 512x512x512:16x16x16 512x512x512:8x8x8 768x768x768:2x2x2 >> gpurun_out/qp_final.log 2>&1
