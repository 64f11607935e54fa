F=gpurun_out/t128; mkdir -p $F
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_fuzz_gpu.py tests/test_parity2d_gpu.py tests/test_fullsize_gpu.py tests/test_abi_errors_gpu.py -m gpu -q 2>&1 | tail -3 > $F/parity.log
VARS=4,14 BLOCKS=8x8x8 timeout 300 python tools/var_probe.py > $F/probe2.log 2>&1
DIMS=64x64x64 VARS=3,13 BLOCKS=2x2x2 timeout 300 python tools/var_probe.py >> $F/probe2.log 2>&1
python bench.py --config c5 --no-sweep --no-cpu --no-e2e --no-sustained > $F/bench_c5.json 2>&1
