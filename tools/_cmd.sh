for z in 32 16 8 4 2; do echo "== zchunk $z"; JAC_ZCHUNK=$z ITERS=200 timeout 100 python tools/perf_shapes.py 64x64x64:2x2x2 64x64x64:1x1x1 128x128x128:2x2x2 2>&1 | cut -c1-100; done > gpurun_out/c1.log
echo "== default" >> gpurun_out/c1.log; ITERS=200 timeout 100 python tools/perf_shapes.py 64x64x64:2x2x2 64x64x64:1x1x1 128x128x128:2x2x2 2>&1 | cut -c1-100 >> gpurun_out/c1.log
echo "== default unroll 50" >> gpurun_out/c1.log; JAC_UNROLL=50 ITERS=200 timeout 100 python tools/perf_shapes.py 64x64x64:2x2x2 2>&1 | cut -c1-100 >> gpurun_out/c1.log
