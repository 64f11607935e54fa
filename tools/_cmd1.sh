F=gpurun_out/c5tune; mkdir -p $F
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity2d_gpu.py tests/test_fullsize_gpu.py -m gpu -q 2>&1 | tail -2 > $F/parity.log
for lib in new prev new prev; do
  if [ $lib = prev ]; then export JAC_LIB=build/ab/lib_prev.so; else unset JAC_LIB; fi
  for b in "16 16 16" "8 8 8" "4 4 4" "2 2 2" "1 1 1"; do python tools/profile_sweep.py --blocks $b --iters 20 2>&1 | sed "s/^/$lib /"; done
  python tools/profile_sweep.py --dims 64 64 64 --blocks 2 2 2 --iters 50 2>&1 | sed "s/^/$lib /"
done > $F/time2.log
unset JAC_LIB
python bench.py --config c5 --no-sweep --no-cpu --no-e2e --no-sustained > $F/bench_c5.json 2>&1
