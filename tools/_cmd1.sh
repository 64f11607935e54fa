F=gpurun_out/at; mkdir -p $F
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity2d_gpu.py tests/test_fullsize_gpu.py -m gpu -q 2>&1 | tail -2 > $F/parity.log
for lib in new prev new prev; do
  if [ $lib = prev ]; then export JAC_LIB=build/ab/lib_prev.so; else unset JAC_LIB; fi
  python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 10 2>&1 | sed "s/^/$lib /"
  for b in "1 1 1" "2 2 2" "4 4 4"; do python tools/profile_sweep.py --blocks $b --iters 30 2>&1 | sed "s/^/$lib /"; done
done > $F/time.log
unset JAC_LIB
python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 3 > /dev/null 2>&1 && \
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum -k regex:sweep -c 1 python tools/profile_sweep.py --dims 32768 32768 1 --blocks 2 4 1 --flags 512 --iters 2 2>&1 | grep -E "inst_exec|duration" >> $F/time.log
