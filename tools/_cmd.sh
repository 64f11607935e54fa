timeout 500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for r in 1 2; do
echo "== prev"; JAC_LIB=$PWD/build/ab/lib_prev.so ITERS=40 ODFS=1 timeout 200 python tools/quick_perf.py 2>&1 | cut -c1-90
for d in 0 1 2 3; do echo "== dbg $d"; JAC_DBG=$d ITERS=40 ODFS=1,8 timeout 200 python tools/quick_perf.py 2>&1 | cut -c1-90; done
done > gpurun_out/ab.log
