F=gpurun_out/span; mkdir -p $F
timeout 1500 python -m pytest tests/test_abi_errors_gpu.py tests/test_parity_gpu.py tests/test_parity2d_gpu.py -m gpu -q 2>&1 | tail -2 > $F/pytest.log
python bench.py --no-cpu --no-e2e --no-sustained > $F/bench.json 2> $F/bench.err
python bench.py --config j2d --no-cpu --no-e2e --no-sustained --no-sweep > $F/bench_j2d.json 2> $F/bench_j2d.err
for b in "1 1 1" "2 2 2"; do python tools/profile_sweep.py --blocks $b --iters 20 >> $F/pytest.log 2>&1; done
