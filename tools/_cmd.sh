FLAGS=512 ITERS=20 timeout 600 python tools/perf_shapes.py 32768x32768x1:1x1x1 32768x32768x1:2x4x1 32768x32768x1:4x4x1 32768x32768x1:8x8x1 32768x32768x1:32x32x1 8192x8192x1:4x4x1 > gpurun_out/j2d_shapes.log 2>&1
timeout 600 python bench.py --config j2d --steps 50 --warmup 3 > gpurun_out/bench_j2d.json 2> gpurun_out/bench_j2d.err; echo rc=$? >> gpurun_out/bench_j2d.err
