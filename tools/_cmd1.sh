F=gpurun_out/clean; mkdir -p $F
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_fuzz_gpu.py tests/test_parity2d_gpu.py tests/test_fullsize_gpu.py -m gpu -q 2>&1 | tail -2 > $F/pytest.log
VARS=0,5 BLOCKS=1x1x1,2x2x2 REPS=1 timeout 300 python tools/var_probe.py >> $F/pytest.log 2>&1
