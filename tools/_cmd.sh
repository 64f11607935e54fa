timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
ITERS=30 timeout 300 python tools/perf_shapes.py 512x512x512:1x1x1 512x512x512:2x2x2 512x512x512:2x2x4 512x512x512:4x4x4 512x512x512:8x8x8 512x512x512:16x16x16 1024x1024x1024:32x32x32 64x64x64:2x2x2 2>&1 | cut -c1-100 > gpurun_out/final_shapes.log
