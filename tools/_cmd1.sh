F=gpurun_out/abi; mkdir -p $F
timeout 900 python -m pytest tests/test_abi_errors_gpu.py tests/test_parity_fuzz_gpu.py -m gpu -q 2>&1 | tail -30 > $F/pytest.log
