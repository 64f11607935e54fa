F=gpurun_out/gap; mkdir -p $F
timeout 900 python -m pytest tests/test_abi_errors_gpu.py -m gpu -q 2>&1 | tail -3 > $F/pytest.log
python bench.py --no-cpu --no-e2e --no-sustained > $F/bench.json 2> $F/bench.err
