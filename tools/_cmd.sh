timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for r in 1 2; do
echo "== prev"; JAC_LIB=$PWD/build/ab/lib_prev.so ITERS=30 timeout 300 python tools/perf_shapes.py 512x512x512:1x1x1 512x512x512:2x2x2 512x512x512:4x4x4 512x512x512:8x8x8 512x512x512:16x16x16 2>&1 | cut -c1-90
echo "== cur"; ITERS=30 timeout 300 python tools/perf_shapes.py 512x512x512:1x1x1 512x512x512:2x2x2 512x512x512:4x4x4 512x512x512:8x8x8 512x512x512:16x16x16 2>&1 | cut -c1-90
done > gpurun_out/ab.log
