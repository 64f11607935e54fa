F=gpurun_out/j2d; mkdir -p $F
timeout 900 python -m pytest tests/test_parity2d_gpu.py tests/test_parity_gpu.py -m gpu -q 2>&1 | tail -2 > $F/parity.log
for lib in new prev new prev; do
  if [ $lib = prev ]; then export JAC_LIB=build/ab/lib_prev.so; export JAC_VARIANT=5; else unset JAC_LIB; unset JAC_VARIANT; fi
  CFG=j2d ODFS=1,8,64 SETTINGS="JAC_ZCHUNK=16" K=2 SETTLE=600 N=100 timeout 300 python tools/steady_probe.py 2>&1 | sed "s/^/$lib /"
done > $F/ab.log
