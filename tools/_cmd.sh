timeout 300 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for gc in 0 100000 444 296 592; do echo "== GCOLS=$gc"; if [ $gc = 0 ]; then ITERS=40 timeout 200 python tools/quick_perf.py 2>&1; else JAC_GCOLS=$gc ITERS=40 timeout 200 python tools/quick_perf.py 2>&1; fi; done > gpurun_out/qp_gcols.log
